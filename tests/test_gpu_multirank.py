"""Multi-rank sequence driver on the device.

* The pmp_nccl_* C-ABI collectives on a single-rank NCCL communicator (the
  pool has one GPU: NCCL refuses two ranks on one device).
* run_sequence sharded over 2 ranks that share the one GPU, over a gloo
  process group (comm.py's host path): the column-sharded base SPAI
  (level 0), the rank-0 build + structure broadcast (level 1, where the
  augmented supports make P1's structure differ from the level-0 pattern),
  round-robin systems and the gathered records -- everything must equal the
  single-rank run.  The ranks' kernels never wait on each other (only host
  collectives between launches).
"""

import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_06574_b200 as pm
    return pm


def test_nccl_abi_single_rank(pm):
    import torch
    from paper_1809_06574_b200 import _abi
    L = _abi.lib()
    assert L.pmp_nccl_available() == 1
    uid = (ctypes.c_ubyte * 128)()
    _abi.check(L.pmp_nccl_unique_id(uid), "uid")
    comm = ctypes.c_void_p()
    _abi.check(L.pmp_nccl_init(0, 1, uid, ctypes.byref(comm)), "init")
    try:
        t = torch.arange(100, dtype=torch.float64, device="cuda")
        _abi.check(L.pmp_nccl_bcast(t.data_ptr(), 800, 0, comm, _abi.stream()), "bcast")
        counts = (ctypes.c_size_t * 1)(800)
        displs = (ctypes.c_size_t * 1)(0)
        _abi.check(L.pmp_nccl_allgatherv(t.data_ptr(), counts, displs, 1, comm, _abi.stream()),
                   "allgatherv")
        _abi.check(L.pmp_nccl_allreduce_f64(t.data_ptr(), 100, comm, _abi.stream()),
                   "allreduce")
        torch.cuda.synchronize()
        assert torch.equal(t.cpu(), torch.arange(100, dtype=torch.float64))
    finally:
        _abi.check(L.pmp_nccl_destroy(comm), "destroy")
    with pytest.raises(ValueError):
        _abi.check(L.pmp_nccl_init(1, 1, uid, ctypes.byref(comm)), "init")


def _policy(pm, level):
    return pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=level),
                            update=pm.UpdateConfig(pattern_level=level))


def _workload():
    from paper_1809_06574_b200.workloads import make_config
    return make_config(2, scale=10)     # c2 stencil at n = 1000, 40 systems


def _rank_main(rank, world, port, level, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1809_06574_b200 as pm
    from paper_1809_06574_b200.comm import get_comm
    W = _workload()
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    sols = {}
    recs, info = pm.run_sequence(model, W.s_grid, W.p_grid, _policy(pm, level),
                                 pm.SolverConfig(tol=1e-8), rank=rank, world=world,
                                 on_solution=lambda i, X: sols.__setitem__(i, X.cpu().numpy()))
    allr = [(r["index"], r["iterations"], r["converged"]) for r in info["records_all"]]
    q.put((rank, [r["index"] for r in recs], allr, sols, get_comm().uses_nccl))
    dist.destroy_process_group()


@pytest.mark.parametrize("level", [0, 1])
def test_two_ranks_share_the_sequence(pm, level):
    import multiprocessing as mp
    W = _workload()
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    ref_sols = {}
    ref, _ = pm.run_sequence(model, W.s_grid, W.p_grid, _policy(pm, level),
                             pm.SolverConfig(tol=1e-8),
                             on_solution=lambda i, X: ref_sols.__setitem__(i, X.cpu().numpy()))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, level, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = [(r["index"], r["iterations"], r["converged"]) for r in ref]
    owned = set()
    for rank, mine, allr, sols, nccl in out:
        assert not nccl
        assert mine == list(range(rank, len(ref), 2))
        owned |= set(mine)
        assert allr == want
        for i, X in sols.items():
            # the same P1 (column-sharded build bitwise the single-rank one),
            # the same kernels: identical solutions
            assert np.array_equal(X, ref_sols[i]), i
    assert owned == set(range(len(ref)))
