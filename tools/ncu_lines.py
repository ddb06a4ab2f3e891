"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export by
source line: warp-stall samples and executed instructions, top N lines.

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = []
    fname = None
    hdr = None
    with open(path) as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "File Path":
                fname = r[1].rsplit("/", 1)[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or r[0] == "" or r[0] == "Function Name":
                continue
            d = dict(zip(hdr[2:], r[2:]))
            try:
                samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                inst = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            rows.append((samp, inst, fname, r[0], r[1].strip()[:90]))
    ts = sum(r[0] for r in rows) or 1
    ti = sum(r[1] for r in rows) or 1
    print("total samples %d, warp instructions %d" % (ts, ti))
    for samp, inst, fn, ln, src in sorted(rows, reverse=True)[:top]:
        print("%5.1f%% samp %5.1f%% inst  %s:%s  %s" % (100 * samp / ts, 100 * inst / ti, fn, ln, src))


if __name__ == "__main__":
    main()
