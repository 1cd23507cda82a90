"""Forward / backward TFLOP/s of one ring step's block at the c4 SP=8 per-rank shape (q 16K rows
x k 8K rows, all admitted, 32q/8kv heads, d=128) through the kernel-level C ABI, against a long
causal block (profiling helper).  python tools/step_shape.py"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_22296_b200 import _lib as C  # noqa: E402

H, Hkv, d = 32, 8, 128
lib = C.lib()
I64 = ctypes.POINTER(ctypes.c_int64)
lib.spattn_block_bwd.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_void_p, I64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, I64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
lib.spattn_block_fwd.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_void_p, I64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, I64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p]


def run(lq, lk, q0, k0, reps=5):
    q = torch.randn(1, lq, H, d, device="cuda").bfloat16()
    k = torch.randn(1, lk, Hkv, d, device="cuda").bfloat16()
    v = torch.randn(1, lk, Hkv, d, device="cuda").bfloat16()
    acc = torch.zeros(1, lq, H, d, device="cuda")
    lse = torch.full((1, lq, H), float("-inf"), device="cuda")
    qp, kp = np.arange(q0, q0 + lq, dtype=np.int64), np.arange(k0, k0 + lk, dtype=np.int64)
    pairs = ctypes.c_int64()
    s = torch.cuda.current_stream().cuda_stream

    def call():
        C.check(lib.spattn_block_fwd(s, 1, H, Hkv, d, q.data_ptr(), qp.ctypes.data_as(I64), lq, k.data_ptr(),
                                     v.data_ptr(), kp.ctypes.data_as(I64), lk, 1, d ** -0.5, acc.data_ptr(),
                                     lse.data_ptr(), ctypes.byref(pairs)))
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = torch.randn(1, lq, H, d, device="cuda").bfloat16()
    lse2 = torch.randn(1, lq, H, device="cuda")
    dout = torch.randn(1, lq, H, d, device="cuda").bfloat16()
    dq = torch.zeros(1, lq, H, d, device="cuda")
    dk = torch.zeros(1, lk, Hkv, d, device="cuda")
    dv = torch.zeros(1, lk, Hkv, d, device="cuda")

    def bwd():
        C.check(lib.spattn_block_bwd(s, 1, H, Hkv, d, q.data_ptr(), qp.ctypes.data_as(I64), lq, k.data_ptr(),
                                     v.data_ptr(), kp.ctypes.data_as(I64), lk, 1, d ** -0.5, out.data_ptr(),
                                     lse2.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                     None))
    bwd()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        bwd()
    e1.record()
    torch.cuda.synchronize()
    bms = e0.elapsed_time(e1) / reps
    print(f"q {lq} x k {lk} (q0 {q0}, k0 {k0}): fwd {ms:.3f} ms {4 * d * pairs.value / ms / 1e9:.0f} TFLOP/s "
          f"(merge mode), bwd {bms:.3f} ms {10 * d * pairs.value / bms / 1e9:.0f} TFLOP/s (fp32 dq/dk/dv, incl. delta)",
          flush=True)


run(16384, 8192, 16384, 0)       # ring step block at c4 SP=8: all admitted
run(16384, 16384, 0, 0)          # diagonal-like causal block
run(32768, 32768, 0, 0, reps=2)  # long causal block (c2 size)
