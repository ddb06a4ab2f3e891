"""ctypes binding of libpmorb200.so (include/pmorb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (plain
nvcc, sm_100a).  There is no CPU fallback: if the library is missing or
fails to load, every device entry point raises.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMP_LIB") or os.path.join(_HERE, "libpmorb200.so")

PMP_OK = 0
PMP_ERR_ARG = -1
PMP_ERR_CUDA = -2
PMP_ERR_WORKSPACE = -3

_lib = None

c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t

_SIGS = {
    "pmp_last_error": ([], ctypes.c_char_p),
    "pmp_version": ([], c_int),
    "pmp_assemble": ([c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_dbl, c_vp, c_vp, c_vp,
                      c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_assemble_multi": ([c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_int,
                            c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_compact_workspace": ([c_int], c_sz),
    "pmp_compact_zeros": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_transpose_workspace": ([c_int, c_int], c_sz),
    "pmp_transpose": ([c_int, c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                       c_vp], c_int),
    "pmp_permute": ([c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_permute_batch": ([c_int, c_vp, c_int, c_vp, ctypes.c_longlong, c_vp, ctypes.c_longlong, c_vp], c_int),
    "pmp_pattern_l0_workspace": ([c_int], c_sz),
    "pmp_pattern_l0": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_pattern_l0_ptr": ([c_int, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_ls_team_bytes": ([c_int, c_int, c_int, c_int], c_sz),
    "pmp_ls_columns_multi": ([c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp,
                              c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                              c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_ls_bound": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_ls_columns": ([c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp,
                        c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                        c_vp, c_sz, c_vp], c_int),
    "pmp_ls_columns_planned": ([c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_int,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_augment_team_bytes": ([c_int], c_sz),
    "pmp_augment": ([c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                     c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_spmm": ([c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_int, c_dbl, c_dbl, c_vp, c_int, c_vp,
                  c_int, c_vp], c_int),
    "pmp_gram_workspace": ([c_int, c_int, c_int], c_sz),
    "pmp_gram": ([c_int, c_int, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_tsmm": ([c_int, c_int, c_vp, c_int, c_int, c_vp, c_dbl, c_dbl, c_vp, c_int, c_vp], c_int),
    "pmp_tsqr_workspace": ([c_int, c_int], c_sz),
    "pmp_tsqr_r": ([c_int, c_int, c_vp, c_int, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_copy_cols": ([c_int, c_int, c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_vp], c_int),
    "pmp_axpby_cols": ([c_int, c_int, c_dbl, c_vp, c_int, c_vp, c_dbl, c_vp, c_int, c_vp, c_vp],
                       c_int),
    "pmp_count_flags": ([c_int, c_vp, c_int, c_vp, c_vp], c_int),
    "pmp_select_workspace": ([c_int], c_sz),
    "pmp_select_gt": ([c_int, c_vp, c_vp, c_dbl, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_scan_workspace": ([c_int], c_sz),
    "pmp_scan": ([c_int, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_merge_columns": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
                          c_int),
    "pmp_merge_sizes": ([c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_orth_workspace": ([c_int, c_int, c_int, c_int], c_sz),
    "pmp_orth_step": ([c_int, c_vp, c_int, c_int, c_vp, c_int, c_int, c_int, c_vp, c_int, c_int,
                       c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "pmp_fold_workspace": ([c_int, c_int], c_sz),
    "pmp_fold": ([c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_int, c_int, c_int, c_vp,
                  c_vp, c_sz, c_vp], c_int),
    "pmp_host_alloc_mapped": ([c_sz, c_vp], c_int),
    "pmp_host_free_mapped": ([c_vp], c_int),
    "pmp_host_device_ptr": ([c_vp, c_vp], c_int),
    "pmp_host_wait_flag": ([c_vp, c_dbl, ctypes.c_longlong, c_vp], c_int),
    "pmp_gcro_step": ([c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                       c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_vp,
                       c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_sz, c_vp, c_vp, c_vp],
                      c_int),
    "pmp_gcro_cycle_end": ([c_int, c_int, c_int, c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_int,
                            c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                            c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                            c_vp], c_int),
    "pmp_gcro_absorb": ([c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                         c_vp, c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                         c_vp], c_int),
    "pmp_bench_grid_sync": ([c_int, c_int, c_vp], c_int),
    "pmp_gcro_inner": ([c_vp], c_int),
    "pmp_cycle_workspace": ([c_int, c_int, c_int, c_int], c_sz),
    "pmp_gcro_cycle_dev": ([c_vp], c_int),
    "pmp_cycle_debug_stamps": ([c_vp, c_int], c_int),
    "pmp_solve_geometry": ([c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp],
                           c_int),
    "pmp_solve_batch": ([c_vp], c_int),
    "pmp_solve_ctl_doubles": ([c_int, c_int, c_int, c_int], c_sz),
    "pmp_set_coop_stream": ([c_vp], c_int),
    "pmp_orth_debug_stamps": ([c_vp, c_int], c_int),
    "pmp_host_deflate": ([c_int, c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_host_hls_append": ([c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                             c_vp, c_vp], c_int),
    "pmp_fp64_peak": ([c_int, c_int, c_vp, c_vp], c_int),
    "pmp_realify": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_realify_block": ([c_int, c_int, c_vp, c_vp, c_int, c_vp, c_int, c_vp], c_int),
    "pmp_derealify_block": ([c_int, c_int, c_vp, c_int, c_int, c_vp, c_vp, c_int, c_vp], c_int),
    "pmp_modulus": ([c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_pattern_realify": ([c_int, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_assemble_cplx": ([c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                           c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pmp_nccl_available": ([], c_int),
    "pmp_nccl_unique_id": ([c_vp], c_int),
    "pmp_nccl_init": ([c_int, c_int, c_vp, c_vp], c_int),
    "pmp_nccl_destroy": ([c_vp], c_int),
    "pmp_nccl_bcast": ([c_vp, c_sz, c_int, c_vp, c_vp], c_int),
    "pmp_nccl_allgatherv": ([c_vp, c_vp, c_vp, c_int, c_vp, c_vp], c_int),
    "pmp_nccl_allreduce_f64": ([c_vp, c_sz, c_vp, c_vp], c_int),
}

EXPORTS = tuple(_SIGS)


def load(path=None):
    """Load the library (no CUDA device needed to load it)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError("libpmorb200.so not built (%s): run __graft_entry__.build()" % p)
    lib = ctypes.CDLL(p)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def lib():
    return load()


def check(rc, what=""):
    if rc == PMP_OK:
        return
    msg = lib().pmp_last_error().decode(errors="replace")
    if rc == PMP_ERR_ARG:
        raise ValueError("%s: %s" % (what, msg))
    raise RuntimeError("%s failed (%d): %s" % (what, rc, msg))


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream():
    return torch.cuda.current_stream().cuda_stream


# kernel launches issued per ABI call (CUB scans launch an init + a scan
# kernel; the transpose launches count, scan, fill and sort kernels)
_LAUNCHES_PER_CALL = {"pmp_scan": 2, "pmp_transpose": 5, "pmp_pattern_l0": 5,
                      "pmp_pattern_l0_ptr": 3, "pmp_compact_zeros": 4, "pmp_select_gt": 4,
                      "pmp_augment": 1}
_NO_LAUNCH = {"pmp_last_error", "pmp_version", "pmp_host_deflate", "pmp_host_hls_append",
              "pmp_host_alloc_mapped", "pmp_host_free_mapped", "pmp_host_device_ptr",
              "pmp_host_wait_flag", "pmp_gcro_absorb", "pmp_orth_debug_stamps",
              "pmp_cycle_debug_stamps", "pmp_solve_geometry", "pmp_solve_ctl_doubles",
              "pmp_cycle_workspace", "pmp_nccl_available", "pmp_nccl_unique_id",
              "pmp_nccl_init", "pmp_nccl_destroy"}
# pmp_gcro_step launches the SpMM chain (1 + depth) and the orthogonalisation
_LAUNCHES_PER_CALL["pmp_gcro_step"] = 4


class MappedBuffer:
    """Pinned, device-mapped host memory (zero-copy results of the block
    step kernels); freed with the object."""

    def __init__(self, ndoubles):
        import numpy as np
        p = ctypes.c_void_p()
        check(lib().pmp_host_alloc_mapped(8 * ndoubles, ctypes.byref(p)), "pmp_host_alloc_mapped")
        self.ptr = p.value
        self.array = np.ctypeslib.as_array((ctypes.c_double * ndoubles).from_address(self.ptr))

    def __del__(self):
        try:
            if self.ptr:
                lib().pmp_host_free_mapped(self.ptr)
                self.ptr = None
        except Exception:
            pass

COUNTERS = {}          # name -> calls (enabled by count_launches())
_counting = False
_timed = {}            # name -> list of (start, end) CUDA events
_timing_names = ()


def count_launches(enable=True, timed=()):
    """Count ABI kernel launches (and optionally bracket the calls named in
    ``timed`` with CUDA events on the current stream)."""
    global _counting, _timing_names
    _counting = enable
    _timing_names = tuple(timed)
    COUNTERS.clear()
    _timed.clear()


def lib_seg_enabled():
    """The library's segmented least-squares tier is on (PMP_LS_REG != 0)."""
    return os.environ.get("PMP_LS_REG", "1")[:1] != "0"


def note_launches(k):
    """Record launches an ABI call made beyond one (calls whose launch count
    depends on their arguments, e.g. pmp_ls_columns_multi)."""
    if _counting:
        COUNTERS["_extra"] = COUNTERS.get("_extra", 0) + int(k)


def launches():
    return sum((1 if k == "_extra" else _LAUNCHES_PER_CALL.get(k, 1)) * v
               for k, v in COUNTERS.items() if k not in _NO_LAUNCH)


def timed_events():
    return _timed


def call(name, *args):
    if _counting:
        COUNTERS[name] = COUNTERS.get(name, 0) + 1
        if name in _timing_names:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            rc = getattr(lib(), name)(*args)
            b.record()
            _timed.setdefault(name, []).append((a, b, args))
            check(rc, name)
            return
    rc = getattr(lib(), name)(*args)
    check(rc, name)
