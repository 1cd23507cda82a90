"""Do host->device DMA copies slow the attention kernels? c2 fwd+bwd kernel times (library CUDA
-event profiler) alone and with a side stream streaming pinned host rows into HBM (profiling
helper)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

L, H, Hkv, d = 32768, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
do = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
host = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def run(dma, reps=4):
    for i in range(reps + 1):
        if i == 1:
            torch.cuda.synchronize()
            C.check(C.lib().spattn_profile_enable(1))
        if dma:
            with torch.cuda.stream(side):
                for _ in range(3):  # ~15 ms of H2D per step, like the host step's 671 MB
                    dev.copy_(host, non_blocking=True)
        out = P.oracle_attention(q, k, v)
        out.backward(do)
    torch.cuda.synchronize()
    C.check(C.lib().spattn_profile_enable(0))
    ms, n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    C.check(C.lib().spattn_profile_read(ms, n))
    return ms[0] / reps, ms[1] / reps


for dma in (False, True, False, True):
    f, b = run(dma)
    print(f"dma={dma}: fwd {f:.2f} ms, bwd {b:.2f} ms")
