"""Per-iteration clock64 timeline of the first CTA pair of the CTA-pair backward
(attn_bwd_pair.cu TC slots; profiling helper).  SPATTN_BWD_PAIR=1 python tools/bwd_trace_pair.py [L]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H, Hkv, d = 32, 8, 128
buf = torch.zeros(8192 * 32, dtype=torch.int64, device="cuda")
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
t = buf.view(-1, 2, 16).cpu().double()
n = int((t[:, 0, 0] > 0).sum())
lo, hi = min(50, n // 4), n - 2
def med(r, a, b, lag=0):
    return statistics.median([(t[i, r, b] - t[i - lag, r, a]).item() for i in range(lo + 1, hi)])
print(f"iterations {n}; leader MMA cycles per iteration {(t[hi, 0, 0] - t[lo, 0, 0]).item() / (hi - lo):.0f}")
print("leader MMA: iter->S issue", med(0, 0, 10), " iter->dQ issue (dS ready)", med(0, 0, 1),
      " dQ issue->dP issue (drained)", med(0, 1, 2), " dP issue->dV issue (P ready)", med(0, 2, 3),
      " dV issue->next iter", statistics.median([(t[i + 1, 0, 0] - t[i, 0, 3]).item() for i in range(lo, hi)]))
for r in (0, 1):
    print(f"rank {r} softmax: A", med(r, 4, 5), " A->B start", med(r, 5, 6), " B", med(r, 6, 7),
          " B end->next A", statistics.median([(t[i + 1, r, 4] - t[i, r, 7]).item() for i in range(lo, hi)]),
          " drain md->arrive", med(r, 8, 9))
    print(f"   rank {r}: B compute+stores", med(r, 6, 12), " wait_st+proxy fence", med(r, 12, 13), " arrive", med(r, 13, 7),
          " | A until wait_st", med(r, 4, 14), " A fence+arrive", med(r, 14, 5),
          " | drain ld", med(r, 8, 11), " drain fence+arrive", med(r, 11, 9))
print("leader: dQ issue -> drain sees dQ done", med(0, 1, 8), " drain arrive -> dP issue", med(0, 9, 2),
      " dP issue -> phase B start", med(0, 2, 6), " B end -> dQ issue", statistics.median([(t[i, 0, 1] - t[i, 0, 7]).item() for i in range(lo, hi)]))
