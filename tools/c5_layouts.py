"""c5 (neat-packed 256K, 32q/8kv, d=128) through the ring at SP=8 on the loopback fabric, per
layout: attention-kernel time (library CUDA-event profiler) and executed pairs, to separate the
kernels' efficiency from the rest of the step (profiling helper).
    python tools/c5_layouts.py [layouts...]"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "tools")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402
from sp_projection import c5_docs  # noqa: E402

L, H, Hkv, d, sp = 262144, 32, 8, 128, 8
docs = c5_docs(L)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
for lay in sys.argv[1:] or ["zigzag", "zigzag:4", "zigzag:16"]:
    fab = P.Fabric(sp)
    for rep in range(2):
        torch.cuda.synchronize()
        if rep:
            fab.reset_stats()
            C.check(C.lib().spattn_profile_enable(1))
        t0 = time.perf_counter()
        out = P.engine_attention("ring", q, k, v, sp, docs=docs, fabric=fab, layout=lay)
        out.backward(dout)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    C.check(C.lib().spattn_profile_enable(0))
    ms, n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    C.check(C.lib().spattn_profile_read(ms, n))
    fl = [fab.flops(i) for i in range(sp)]
    tot = sum(fl)
    print(f"{lay:10s} wall {t * 1e3:7.1f} ms  fwd kernels {ms[0]:7.1f} ms ({n[0]} launches)  "
          f"bwd kernels {ms[1]:7.1f} ms ({n[1]})  executed {tot / 1e12:.1f} TFLOP -> "
          f"{tot * 4 / 14 / ms[0] / 1e9:.0f} / {tot * 10 / 14 / ms[1] / 1e9:.0f} TFLOP/s, busiest {max(fl) / tot:.3f}")
