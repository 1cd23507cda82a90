"""One forward launch at c2 for ncu captures (profiling helper): python tools/fwd_one.py [family]."""
import sys, torch
sys.path.insert(0, ".")
import paper_2505_22296_b200 as P
P.set_kernel_family(sys.argv[1] if len(sys.argv) > 1 else "tcgen05_pp")
L, H, Hkv, d = 32768, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
for _ in range(2):
    P.oracle_attention(q, k, v)
torch.cuda.synchronize()
