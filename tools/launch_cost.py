"""Host cost per attention launch through the kernel-level C ABI (spattn_block_fwd on a tiny
problem, no synchronisation inside the loop; profiling helper).  python tools/launch_cost.py"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_22296_b200 import _lib as C  # noqa: E402

L, H, d = 256, 1, 128
q = torch.randn(1, L, H, d, device="cuda").bfloat16()
acc = torch.zeros(1, L, H, d, device="cuda")
lse = torch.full((1, L, H), float("-inf"), device="cuda")
pos = np.arange(L, dtype=np.int64)
pp = pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
s = torch.cuda.current_stream().cuda_stream
lib = C.lib()
fn = lib.spattn_block_fwd
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
               ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
               ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_int, ctypes.c_double,
               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]


def call():
    C.check(fn(s, 1, H, H, d, q.data_ptr(), pp, L, q.data_ptr(), q.data_ptr(), pp, L, 1, d ** -0.5,
               acc.data_ptr(), lse.data_ptr(), None))


for _ in range(50):
    call()
torch.cuda.synchronize()
n = 2000
t = time.perf_counter()
for _ in range(n):
    call()
host = (time.perf_counter() - t) / n * 1e6
torch.cuda.synchronize()
tot = (time.perf_counter() - t) / n * 1e6
print(f"host us per call {host:.1f}, wall us per call incl. GPU {tot:.1f}")
