"""Per-kernel TFLOP/s of the attention kernels for one rank's shape (e.g. the per-GPU shape of
Ulysses SP=8 at c2: L=32768, 4 q heads, 1 kv head), via the library's CUDA-event profiler.
    python tools/shape_bench.py L H Hkv [d] [reps]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

P.set_kernel_family(os.environ.get("FAMILY", "tcgen05"))

L, H, Hkv = (int(x) for x in sys.argv[1:4])
d = int(sys.argv[4]) if len(sys.argv) > 4 else 128
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
# random upstream gradient (a constant one toggles fewer bits and runs at higher clocks under
# the power cap)
dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
for i in range(reps + 2):
    if i == 2:
        torch.cuda.synchronize()
        C.check(C.lib().spattn_profile_enable(1))
    out = P.oracle_attention(q, k, v)
    out.backward(dout)
torch.cuda.synchronize()
C.check(C.lib().spattn_profile_enable(0))
ms, n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
C.check(C.lib().spattn_profile_read(ms, n))
pairs = L * (L + 1) // 2 * H
f, b = ms[0] / reps, ms[1] / reps
print(f"L={L} H={H} Hkv={Hkv} d={d}: fwd {f:.3f} ms {4 * d * pairs / f / 1e9:.0f} TFLOP/s, "
      f"bwd {b:.3f} ms {10 * d * pairs / b / 1e9:.0f} TFLOP/s")
