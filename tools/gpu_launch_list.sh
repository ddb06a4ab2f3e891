#!/bin/bash
# ncu launch list (gpu__time_duration.sum per launch, no replay passes) of the
# bench command at reduced step counts; CSV + per-kernel summary in gpurun_out/.
#   tools/gpu_launch_list.sh 4   (config)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
c=${1:-4}
args="--config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-warm --level1-systems 0"
timeout 1500 python bench.py $args > gpurun_out/ll_bench_c$c.json 2> gpurun_out/ll_bench_c$c.err; echo "plain rc=$?"
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file /tmp/launches_c$c.csv python bench.py $args > gpurun_out/ll_ncu_c$c.log 2>&1; echo "ncu rc=$?"
python - <<PY
import csv, collections
rows = list(csv.reader(l for l in open("/tmp/launches_c$c.csv", errors="replace") if l.startswith('"')))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3, "nsecond": 1e-6}.get(u, 1e-6)
    nm = r[ki].split("(")[0][:90]
    a = tot.setdefault(nm, [0, 0.0])
    a[0] += 1
    a[1] += ms
allms = sum(a[1] for a in tot.values())
with open("gpurun_out/launches_c$c" + "_summary.txt", "w") as fh:
    fh.write("bench.py %s under ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launch times; shares only)\n" % "$args")
    fh.write("total %.1f ms over %d launches\n" % (allms, sum(a[0] for a in tot.values())))
    for nm, (cnt, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        fh.write("%6.2f%%  %10.3f ms  %5d launches  %s\n" % (100 * ms / allms, ms, cnt, nm))
print(open("gpurun_out/launches_c$c" + "_summary.txt").read()[:2500])
PY
head -c 3000000 /tmp/launches_c$c.csv | gzip > gpurun_out/launches_c$c.csv.gz
