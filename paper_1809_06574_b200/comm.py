"""Collectives of the multi-GPU sequence driver.

The first-approach sequence has exactly two exchanges: replicating the base
SPAI P1 (every system depends only on (A1, P1), rpmor.py:205-210) and
gathering the per-system scalar records at the end.  On GPUs both go through
NCCL behind the C-ABI (``pmp_nccl_*`` in libpmorb200, over NVLink /
NVSwitch); the torch.distributed process group only carries NCCL's 128-byte
unique id from rank 0 to the others (its store is the rendezvous).

With a ``gloo`` process group (the multi-process tests: CPU ranks, or
several ranks sharing one GPU, which NCCL refuses) the same operations run
as host copies through torch.distributed.
"""

import ctypes

import numpy as np
import torch

from . import _abi


class Comm:
    """rank / world plus broadcast, variable all-gather and sum-allreduce of
    device tensors."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.dist = dist
        self.active = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.active else 0
        self.world = dist.get_world_size(group) if self.active else 1
        self.backend = dist.get_backend(group) if self.active else None
        self._nccl = None
        if self.active and self.world > 1 and self.backend == "nccl":
            self._init_nccl()

    # -- NCCL through the C-ABI ------------------------------------------------
    def _init_nccl(self):
        L = _abi.lib()
        if not L.pmp_nccl_available():
            raise RuntimeError("pmp_nccl: " + L.pmp_last_error().decode(errors="replace"))
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _abi.check(L.pmp_nccl_unique_id(uid), "pmp_nccl_unique_id")
        obj = [bytes(uid)]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(obj[0])
        comm = ctypes.c_void_p()
        _abi.check(L.pmp_nccl_init(self.rank, self.world, uid, ctypes.byref(comm)),
                   "pmp_nccl_init")
        self._nccl = comm

    @property
    def uses_nccl(self):
        return self._nccl is not None

    def close(self):
        if self._nccl is not None:
            _abi.lib().pmp_nccl_destroy(self._nccl)
            self._nccl = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- operations ------------------------------------------------------------
    def bcast(self, t, root=0):
        """In place: t (contiguous, any dtype) from `root` to every rank."""
        if self.world <= 1:
            return t
        if self._nccl is not None:
            _abi.check(_abi.lib().pmp_nccl_bcast(t.data_ptr(), t.numel() * t.element_size(),
                                                 root, self._nccl, _abi.stream()),
                       "pmp_nccl_bcast")
            return t
        h = t.detach().cpu().contiguous()
        self.dist.broadcast(h, root, group=self.group)
        t.copy_(h)
        return t

    def allgatherv(self, t, bounds):
        """In place on a 1-D contiguous tensor: rank r's elements
        [bounds[r], bounds[r+1]) are replicated on every rank."""
        if self.world <= 1:
            return t
        es = t.element_size()
        if self._nccl is not None:
            counts = (ctypes.c_size_t * self.world)(*[(bounds[r + 1] - bounds[r]) * es
                                                      for r in range(self.world)])
            displs = (ctypes.c_size_t * self.world)(*[bounds[r] * es for r in range(self.world)])
            _abi.check(_abi.lib().pmp_nccl_allgatherv(t.data_ptr(), counts, displs, self.world,
                                                      self._nccl, _abi.stream()),
                       "pmp_nccl_allgatherv")
            return t
        h = t.detach().cpu().contiguous()
        for r in range(self.world):
            seg = h[bounds[r]:bounds[r + 1]].clone()
            self.dist.broadcast(seg, r, group=self.group)
            h[bounds[r]:bounds[r + 1]] = seg
        t.copy_(h)
        return t

    def allreduce_sum_f64(self, t):
        """In place element-wise sum over ranks of a float64 tensor."""
        if self.world <= 1:
            return t
        if self._nccl is not None and t.is_cuda:
            _abi.check(_abi.lib().pmp_nccl_allreduce_f64(t.data_ptr(), t.numel(), self._nccl,
                                                         _abi.stream()),
                       "pmp_nccl_allreduce_f64")
            return t
        h = t.detach().cpu().contiguous()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)
        return t


_COMMS = {}


def get_comm(group=None):
    """One Comm per process group (NCCL communicators are expensive)."""
    key = id(group)
    c = _COMMS.get(key)
    if c is None:
        c = _COMMS[key] = Comm(group)
    return c


def column_bounds(n, world):
    """Contiguous column ranges of a column-sharded build: rank r owns
    [b[r], b[r+1])."""
    return [(n * r) // world for r in range(world + 1)]


def record_table(records, n_systems, fields):
    table = np.zeros((n_systems, len(fields)), dtype=np.float64)
    for r in records:
        table[r["index"]] = [r[f] if f != "index" else r["index"] + 1 for f in fields]
    return table
