import sys, torch
sys.path.insert(0, ".")
import paper_2505_22296_b200 as P
L = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, 2, 128, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, 1, 128, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, 1, 128, device="cuda", generator=g).bfloat16().requires_grad_(True)
P.oracle_attention(q, k, v).sum().backward()
torch.cuda.synchronize()
print("ok", q.grad.float().abs().sum().item())
