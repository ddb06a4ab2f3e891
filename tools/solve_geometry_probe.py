import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1809_06574_b200 import _abi
L = _abi.lib()
torch.cuda.init()
gsz, rows, cached = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
smem = ctypes.c_size_t()
for groups in (6,):
    rc = L.pmp_solve_geometry(32768, 8, 68, 18, 50, groups, ctypes.byref(gsz), ctypes.byref(rows), ctypes.byref(cached), ctypes.byref(smem))
    print(os.environ.get("PMP_LIB", "main"), "groups", groups, "rc", rc, "gsz", gsz.value, "rows", rows.value, "cached", cached.value, "smem", smem.value)
