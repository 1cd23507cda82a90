"""Workload for the HBM-bound kernels of the SP layer (pack/permute/unpack copies with and
without fused RoPE, LSE merge, fp32->bf16 rounding), at the c2 shape (32q/8kv, d=128,
L=32768): Ulysses SP=8 on the loopback fabric (peer-read copies and the NCCL-style message
path), rope_apply, and spattn_lse_merge on a ring-step sized accumulator. Run under ncu:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        -k regex:"copy_rows|lse_merge|f32_to_bf16|rope|add_rows" --csv --log-file x.csv \\
        python tools/hbm_kernels.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

L, H, Hkv, d, sp = 32768, 32, 8, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
for messages in (False, True):
    fab = P.Fabric(sp, force_messages=messages)
    out = P.engine_attention("ulysses", q, k, v, sp, fabric=fab, position_ids=list(range(L)))
    out.backward(torch.ones_like(out))
    torch.cuda.synchronize()
x = P.rope_apply(q.detach(), list(range(L)))
# a ring step's merge: acc [L/8 rows x 32 heads x 128] fp32 with a fresh piece
rows = (L // sp) * H
acc = torch.randn(rows, d, device="cuda")
acc_lse = torch.randn(rows, device="cuda")
piece = torch.randn(rows, d, device="cuda")
piece_lse = torch.randn(rows, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    C.check(C.lib().spattn_lse_merge(s, acc.data_ptr(), acc_lse.data_ptr(), piece.data_ptr(),
                                     piece_lse.data_ptr(), rows, d))
torch.cuda.synchronize()
print("done")
