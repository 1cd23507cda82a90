"""Per-iteration globaltimer timeline of backward CTA 0 of the 128-query-tile kernel
(attn_bwd_q128.cu TR slots; profiling helper).  python tools/bwd_trace128.py [L]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

P.set_kernel_family("tcgen05")

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H, Hkv, d = 32, 8, 128
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
for traced in (False, True):
    if traced:
        C.check(C.lib().spattn_debug_bwd_trace(buf.data_ptr()))
    out = P.oracle_attention(q, k, v)
    out.backward(torch.randn_like(out))
    torch.cuda.synchronize()
C.check(C.lib().spattn_debug_bwd_trace(None))
t = buf.view(-1, 16).cpu().double()
n = int((t[:, 0] > 0).sum())
t = t[:n]
names = ["mma:iter", "mma:dsr_ok(dK)", "mma:pr+dof_ok(dV)", "mma:dqf_ok(dP)", "A:start", "B:start",
         "B:done", "dq:md_ok", "dq:dqf", "A:done"]
lo = min(50, n // 4)
print(f"iterations traced: {n}; ns per iteration (steady): {(t[n - 1, 0] - t[lo, 0]) / (n - 1 - lo):.0f}")
for i in range(lo, lo + 3):
    row = t[i] - t[i, 0]
    print(i, " ".join(f"{nm}={row[j]:.0f}" for j, nm in enumerate(names)))
def med(a, b, lag=0):
    return statistics.median([(t[i, b] - t[i - lag, a]).item() for i in range(lo + 1, n - 1)])
print("median ns: A start->A done", med(4, 9), " A done->B start", med(9, 5))
print("median ns: iter->dsr_ok", med(0, 1), " dsr_ok->pr_ok", med(1, 2), " pr_ok->dqf_ok", med(2, 3),
      " A start->B start", med(4, 5), " B start->done", med(5, 6), " md->dqf", med(7, 8))
print("cycles (clock64, same warp): phase A", med(10, 11), " wait A->B", med(11, 12), " phase B", med(12, 13),
      " B end -> next A start", statistics.median([(t[i + 1, 10] - t[i, 13]).item() for i in range(lo + 1, n - 2)]),
      " drain md->dqf", med(14, 15))
print("MMA thread cycles (clock64): per iteration", (t[n - 1, 0] - t[lo, 0]).item() / (n - 1 - lo),
      " iter->dsr_ok(B done)", med(0, 1), " dsr_ok->dqf_ok(drain done)", med(1, 3), " dqf_ok->pr_ok", med(3, 2),
      " pr_ok->next iter", statistics.median([(t[i + 1, 0] - t[i, 2]).item() for i in range(lo + 1, n - 2)]))
