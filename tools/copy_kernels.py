"""Copy-kernel workload without RoPE (the bench's exchange copies): Ulysses SP=8 at c2 on the
loopback fabric through the NCCL-style message path (pack -> send/recv -> unpack), one fwd+bwd,
for ncu (profiling helper):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        -k regex:copy_rows --csv --log-file x.csv python tools/copy_kernels.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402

L, H, Hkv, d, sp = 32768, 32, 8, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
fab = P.Fabric(sp, force_messages=True)
out = P.engine_attention("ulysses", q, k, v, sp, fabric=fab)
out.backward(torch.ones_like(out))
torch.cuda.synchronize()
print("done")
