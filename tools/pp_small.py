import sys, torch
sys.path.insert(0, ".")
import paper_2505_22296_b200 as P
P.set_kernel_family("tcgen05_pp")
for L in (128, 256, 1024):
    q = torch.randn(1, L, 4, 64, device="cuda").bfloat16()
    k = torch.randn(1, L, 2, 64, device="cuda").bfloat16()
    out = P.oracle_attention(q, k, k)
    torch.cuda.synchronize()
    print("ok", L, flush=True)
