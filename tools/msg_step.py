"""Ulysses SP=N step on the loopback fabric through the message path (pack -> send/recv ->
unpack, the NCCL rank's path): wall time of one fwd+bwd of the whole layer for all N ranks on one
GPU, and the copy-kernel launch count (profiling helper).  python tools/msg_step.py [sp]"""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

sp = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L, H, Hkv, d = 32768, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()


def step():
    out = P.engine_attention("ulysses", q, k, v, sp, force_messages=True)
    out.backward(dout)


for _ in range(2):
    step()
torch.cuda.synchronize()
n0 = C.lib().spattn_launch_count()
t = time.perf_counter()
for _ in range(3):
    step()
torch.cuda.synchronize()
print(f"sp={sp} message path: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms per layer step, "
      f"{(C.lib().spattn_launch_count() - n0) / 3:.0f} library launches")
