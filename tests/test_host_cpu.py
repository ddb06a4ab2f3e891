"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, the host-side planning / sharding logic, and the
multi-rank (gloo, world_size 2) broadcast / gather path."""

import os
import json
import re
import socket

import numpy as np
import scipy.sparse as sp
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pmorb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1809_06574_b200 import _abi
    lib = _abi.load()
    names = _header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_abi.EXPORTS)
    assert lib.pmp_version() == 1
    # workspace queries are host-only and need no device
    assert lib.pmp_gram_workspace(1000, 10, 4) >= 256 + 8 * 40
    assert lib.pmp_ls_team_bytes(32, 64, 25, 7) > 0


def test_library_rejects_bad_arguments_without_device():
    from paper_1809_06574_b200 import _abi
    lib = _abi.load()
    assert lib.pmp_spmm(10, None, None, None, 40, None, 40, 1.0, 0.0, None, 0, None, 40,
                        None) == _abi.PMP_ERR_ARG
    assert lib.pmp_ls_columns(5, 32, 0, 64, 1, 1, 1, None, 1, None, None, None, None, None,
                              None, None, None, None, None, None, None, None, None, None, 0,
                              None) == _abi.PMP_ERR_ARG
    assert b"bad arguments" in lib.pmp_last_error()


def test_team_bytes_formula_matches_library():
    from paper_1809_06574_b200 import _abi
    from paper_1809_06574_b200.spai import _team_bytes
    lib = _abi.load()
    for l, m, n in ((64, 25, 7), (1024, 125, 27), (4096, 295, 80), (1, 0, 0)):
        assert lib.pmp_ls_team_bytes(32, l, m, n) == _team_bytes(l, m, n)


def test_tier_split_respects_limits():
    from paper_1809_06574_b200 import spai
    rng = np.random.default_rng(0)
    ncol = 5000
    cols = np.arange(ncol)
    nI = rng.integers(1, 240, ncol)
    m = nI * rng.integers(5, 60, ncol)
    lcap = spai._pow2(m * 3)
    # patch the device upload for a CPU run
    orig = spai.i32
    spai.i32 = lambda a, device=None: np.asarray(a)
    try:
        tiers = spai._split_tiers(cols, lcap, m, nI)
    finally:
        spai.i32 = orig
    seen = np.concatenate([t.cols_host for t in tiers])
    assert np.array_equal(np.sort(seen), cols)
    for t in tiers:
        limit = dict(((a, b), c) for a, b, c in spai._TIERS)[(t.team, t.glob)]
        if limit is not None:
            assert t.bytes <= limit
        sel = t.cols_host
        assert t.mcap == m[sel].max() and t.ncap == nI[sel].max()


def test_owned_systems_partition():
    from paper_1809_06574_b200.sequence import owned_systems
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i in owned_systems(40, r, world))
        assert got == list(range(40))
    assert owned_systems(5, 1, 2, "spai-update-second") == list(range(5))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_06574_b200.comm import column_bounds, get_comm
    from paper_1809_06574_b200.sequence import gather_records, owned_systems
    comm = get_comm()
    assert (comm.rank, comm.world, comm.uses_nccl) == (rank, world, False)
    vals = torch.arange(10, dtype=torch.float64) if rank == 0 else torch.zeros(10,
                                                                               dtype=torch.float64)
    comm.bcast(vals, 0)
    # column-sharded build exchange: rank r fills only its own range
    b = column_bounds(11, world)
    coef = torch.zeros(11, dtype=torch.float64)
    coef[b[rank]:b[rank + 1]] = 100.0 * (rank + 1) + torch.arange(b[rank], b[rank + 1])
    comm.allgatherv(coef, b)
    flags = torch.zeros(11, dtype=torch.int32)
    flags[b[rank]:b[rank + 1]] = rank + 1
    comm.allgatherv(flags, b)
    recs = [{"index": i, "iterations": 10 + i, "converged": True, "matvec_count": 3 * i,
             "precond_apply_count": 2 * i, "max_final_residual": 1e-9}
            for i in owned_systems(7, rank, world)]
    table = gather_records(recs, 7)
    q.put((rank, vals.tolist(), coef.tolist(), flags.tolist(),
           [(r["index"], r["iterations"], r["matvec_count"]) for r in table]))
    dist.destroy_process_group()


def test_gloo_two_ranks_broadcast_allgather_and_gather():
    """Host logic of the multi-GPU driver (comm.py, sequence.gather_records)
    over 2 gloo ranks: broadcast of P1, the column-sharded all-gather with
    uneven ranges, the per-system record table."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1809_06574_b200.comm import column_bounds
    b = column_bounds(11, world)
    want = [100.0 * (r + 1) + i for r in range(world) for i in range(b[r], b[r + 1])]
    wflags = [r + 1 for r in range(world) for i in range(b[r], b[r + 1])]
    for rank, vals, coef, flags, table in out:
        assert vals == list(range(10))
        assert coef == want
        assert flags == wflags
        assert table == [(i, 10 + i, 3 * i) for i in range(7)]


def test_inner_state_layout_matches_header(tmp_path):
    """ctypes mirror of PmpGcroInner == the C struct (gcc probe)."""
    import ctypes
    import subprocess
    from paper_1809_06574_b200.krylov import _InnerState as S
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pmorb200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(PmpGcroInner),'
                   ' offsetof(PmpGcroInner, mirror), offsetof(PmpGcroInner, bn),'
                   ' offsetof(PmpGcroInner, prev_max), offsetof(PmpGcroInner, steps_done));}\n')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(v) for v in got] == [ctypes.sizeof(S), S.mirror.offset, S.bn.offset,
                                     S.prev_max.offset, S.steps_done.offset]


def test_cycle_state_layout_matches_header(tmp_path):
    """ctypes mirror of PmpGcroCycle == the C struct (gcc probe)."""
    import ctypes
    import subprocess
    from paper_1809_06574_b200.krylov import _CycleState as S
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pmorb200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(PmpGcroCycle),'
                   ' offsetof(PmpGcroCycle, offB), offsetof(PmpGcroCycle, ws_bytes),'
                   ' offsetof(PmpGcroCycle, tol), offsetof(PmpGcroCycle, blocks_per_sm),'
                   ' offsetof(PmpGcroCycle, d_istate));}\n')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(v) for v in got] == [ctypes.sizeof(S), S.offB.offset, S.ws_bytes.offset,
                                     S.tol.offset, S.blocks_per_sm.offset, S.d_istate.offset]


def test_solve_batch_layout_matches_header(tmp_path):
    """ctypes mirrors of PmpSysDesc / PmpSolveBatch == the C structs."""
    import ctypes
    import subprocess
    from paper_1809_06574_b200.krylov import _SolveBatchArgs as S, _SysDesc as D
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pmorb200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(PmpSysDesc),'
                   ' offsetof(PmpSysDesc, B), sizeof(PmpSolveBatch),'
                   ' offsetof(PmpSolveBatch, tol), offsetof(PmpSolveBatch, oV),'
                   ' offsetof(PmpSolveBatch, pBmat), offsetof(PmpSolveBatch, stream));}\n')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(v) for v in got] == [ctypes.sizeof(D), D.B.offset, ctypes.sizeof(S), S.tol.offset,
                                     S.oV.offset, S.pBmat.offset, S.stream.offset]


def test_solve_layout_disjoint():
    from paper_1809_06574_b200.krylov import _solve_layout
    off, proj, total = _solve_layout(1000, 8, 68, 18, 74, 70, 2004)
    starts = sorted(off.values())
    assert starts[0] == 0 and all(b > a for a, b in zip(starts, starts[1:]))
    assert total > max(starts)
    assert all(v % 32 == 0 for v in off.values())


# ---------------------------------------------------------------------------
# persistence: Matrix Market interchange with the files the
# reference's own Preconditioner.save wrote (tests/golden/precond_ref)
# ---------------------------------------------------------------------------

GOLD_PRE = os.path.join(ROOT, "tests", "golden", "precond_ref")


def test_read_reference_matrix_market_files():
    import json
    import scipy.io
    from paper_1809_06574_b200 import mmio
    side = json.load(open(os.path.join(GOLD_PRE, "preconditioner.json")))
    assert side["kind"] == "factored" and side["factors"] == ["factor_00.mtx", "factor_01.mtx"]
    for name in side["factors"]:
        path = os.path.join(GOLD_PRE, name)
        M = mmio.read_matrix_market(path)
        R = sp.csr_matrix(scipy.io.mmread(path, spmatrix=False))
        assert M.dtype == np.float64 and M.has_sorted_indices
        assert np.abs(R.data.imag).max() == 0.0
        R = R.real.tocsr()
        R.eliminate_zeros()
        R.sort_indices()
        assert np.array_equal(M.indptr, R.indptr) and np.array_equal(M.indices, R.indices)
        assert np.array_equal(M.data, R.data)  # 17 digits: bit-exact


def test_matrix_market_round_trip_is_bit_exact(tmp_path):
    import scipy.io
    from paper_1809_06574_b200 import mmio
    M = mmio.read_matrix_market(os.path.join(GOLD_PRE, "factor_01.mtx"))
    out = tmp_path / "f.mtx"
    mmio.write_matrix_market(M, out)
    head = open(out).readline()
    assert head.startswith("%%MatrixMarket matrix coordinate complex general")
    # what the reference's reader (scipy.io.mmread + as_csr) sees
    R = sp.csr_matrix(scipy.io.mmread(str(out), spmatrix=False))
    assert np.array_equal(R.data.real, M.data) and np.abs(R.data.imag).max() == 0.0
    M2 = mmio.read_matrix_market(out)
    assert (M2 != M).nnz == 0 and np.array_equal(M2.data, M.data)
    # dense blocks
    X = np.random.default_rng(3).standard_normal((7, 3))
    mmio.write_dense_matrix_market(X, tmp_path / "x.mtx")
    assert np.array_equal(mmio.read_dense_matrix_market(tmp_path / "x.mtx"), X)


def test_matrix_market_complex_round_trip(tmp_path):
    """Complex files (sparsecore.py:250-285) read back bit-exactly as
    complex128; all-zero imaginary parts come back as float64."""
    import scipy.io
    import scipy.sparse as sp
    from paper_1809_06574_b200 import mmio
    A = sp.csr_matrix(np.array([[1.0 + 1.0 / 3.0j, 0], [0.1 - 2j, 2.0]]))
    mmio.write_matrix_market(A, tmp_path / "c.mtx")
    B = mmio.read_matrix_market(tmp_path / "c.mtx")
    assert B.dtype == np.complex128 and np.array_equal(B.toarray(), A.toarray())
    scipy.io.mmwrite(str(tmp_path / "r.mtx"), sp.csr_matrix(np.eye(2) * (1 + 0j)), field="complex")
    assert mmio.read_matrix_market(tmp_path / "r.mtx").dtype == np.float64
    X = np.array([[1.0 + 0.5j, 2.0], [0.25j, -1.0 / 7.0]])
    mmio.write_dense_matrix_market(X, tmp_path / "x.mtx")
    Y = mmio.read_dense_matrix_market(tmp_path / "x.mtx")
    assert Y.dtype == np.complex128 and np.array_equal(Y, X)
    (tmp_path / "bad.mtx").write_text("%%MatrixMarket matrix nonsense\n1 1 1\n")
    with pytest.raises(ValueError):
        mmio.read_matrix_market(tmp_path / "bad.mtx")


# ---------------------------------------------------------------------------
# experiment CLI: host-side pieces against the report the
# reference's own run_experiment wrote (tests/golden/cli_report.json)
# ---------------------------------------------------------------------------

def _golden_report():
    import json
    return json.load(open(os.path.join(ROOT, "tests", "golden", "cli_report.json")))


def test_cli_family_directory_loads_reference_files():
    from paper_1809_06574_b200 import cli
    man = os.path.join(ROOT, "tests", "golden", "cli_family")
    import json
    m = json.load(open(os.path.join(man, "manifest.json")))
    terms = [cli.mmio.read_matrix_market(os.path.join(man, t)) for t in m["terms"]]
    assert len(terms) == 3 and terms[0].shape == (144, 144)
    pts = [cli._values_from_json(p["values"]) for p in m["points"]]
    assert [p.real.tolist() for p in pts] == [[0.5, 0.2], [0.8, 0.3], [1.5, 0.7]]
    # the fingerprint the reference computed, recomputed here
    rep = _golden_report()
    fp = cli._config_hash({"model": rep["config"]["model"],
                           "points": [[[float(v.real), 0.0] for v in p] for p in pts]})
    assert fp == rep["family_fingerprint"]
    assert cli._config_hash(rep["config"]) == rep["config_hash"]


def test_cli_report_writer_round_trip(tmp_path):
    from paper_1809_06574_b200 import cli
    rep = _golden_report()
    cli.write_report(rep, tmp_path / "run")
    recs = cli.load_records_csv(tmp_path / "run" / "report.csv")
    assert recs == rep["records"]
    assert (tmp_path / "run" / "summary.txt").read_text().startswith("solver=block-gcro")
    b = json.loads(json.dumps(rep))
    for s in b["summary"]["per_step"].values():
        s["iterations"] -= 1
    b["summary"]["total_iterations"] -= 3
    d = cli.compare_reports(rep, b)
    assert len(d["steps"]) == 3 and d["totals"]["iterations_saving_pct"] > 0
    b["family_fingerprint"] = "x"
    with pytest.raises(ValueError):
        cli.compare_reports(rep, b)
    assert cli.main(["run"]) == cli.EXIT_USAGE


def test_solve_layout_and_size_table():
    """Host-side pieces of the persistent solve / LS planning: workspace
    offsets are 256-byte aligned, the control-state block is part of the
    projected-state area (offset 0 stays reserved: pCtl = 0 means "absent"),
    and the coarsening table equals the closed form."""
    from paper_1809_06574_b200 import krylov, spai
    off, proj, wsz = krylov._solve_layout(1000, 8, 68, 18, 49, 70, 2004, ctl=7536)
    assert all(v % 32 == 0 for v in off.values()) and wsz % 32 == 0
    assert all(v % 32 == 0 and v > 0 for v in proj.values())
    names = sorted(proj, key=proj.get)
    assert names[-1] == "pCtl"
    assert off["oLog"] - off["oProj"] >= proj["pCtl"] + 7536
    v = np.random.default_rng(0).integers(1, 5000, size=20000)

    def closed(x):
        x = np.maximum(np.asarray(x, dtype=np.int64), 8)
        p = 1 << (np.floor(np.log2(x)).astype(np.int64) - 2)
        return ((x + p - 1) // p) * p
    assert np.array_equal(spai._coarse(v), closed(v))          # table path
    assert np.array_equal(spai._coarse(v[:100]), closed(v[:100]))  # direct path
