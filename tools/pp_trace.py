"""Per-tile event timeline of the ping-pong forward's CTA (0,0) (profiling helper)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

P.set_kernel_family("tcgen05_pp")
L, H, Hkv, d = 32768, 32, 8, 128
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
P.oracle_attention(q, k, v)
C.check(C.lib().spattn_debug_bwd_trace(buf.data_ptr()))
P.oracle_attention(q, k, v)
torch.cuda.synchronize()
C.check(C.lib().spattn_debug_bwd_trace(None))
t = buf.view(-1, 32).cpu().double()
n = int((t[:, 0] > 0).sum())
lo, hi = 20, n - 2
print("key tiles traced:", n, " cycles per key tile (2 tiles of work):", ((t[hi, 0] - t[lo, 0]) / (hi - lo)).item())
med = lambda f: statistics.median([f(i) for i in range(lo, hi)])  # noqa: E731
for x, nm in ((0, "A"), (1, "B")):
    print(f"{nm}: softmax S ready -> P arrive   ", med(lambda i: (t[i, 2 * x + 1] - t[i, 2 * x]).item()))
    print(f"{nm}: P arrive -> next S ready      ", med(lambda i: (t[i + 1, 2 * x] - t[i, 2 * x + 1]).item()))
    print(f"{nm}: MMA wait for P (PV issue span)", med(lambda i: (t[i, 5 + 2 * x] - t[i, 4 + 2 * x]).item()))
print("A warps 0-3 P arrive rel. to warp 0:", [med(lambda i: (t[i, 12 + w] - t[i, 12]).item()) for w in range(4)])
print("MMA: PV_A issued - last A warp arrive", med(lambda i: (t[i, 5] - max(t[i, 12:16])).item()))
print("MMA: P_A seen - last A warp arrive", med(lambda i: (t[i, 16] - max(t[i, 12:16])).item()))
print("MMA: PV_A issue (8 MMAs)", med(lambda i: (t[i, 5] - t[i, 16]).item()), " PV_B", med(lambda i: (t[i, 7] - t[i, 17]).item()))
for x in (0, 1):
    b = 18 + 4 * x
    print("ABx"[x], "phases: ld", med(lambda i: (t[i, b] - t[i, 2 * x]).item()), "max", med(lambda i: (t[i, b + 1] - t[i, b]).item()),
          "exp", med(lambda i: (t[i, b + 2] - t[i, b + 1]).item()), "st", med(lambda i: (t[i, b + 3] - t[i, b + 2]).item()),
          "arrive", med(lambda i: (t[i, 2 * x + 1] - t[i, b + 3]).item()))
print("MMA: wait K/V                       ", med(lambda i: (t[i, 9] - t[i, 8]).item()))
print("rescales A/B:", int((t[lo:hi, 10] > 0).sum()), int((t[lo:hi, 11] > 0).sum()))
for i in (100, 101, 102):
    b = t[100, 0]
    print(i, "A S", t[i, 0] - b, "A P", t[i, 1] - b, "B S", t[i, 2] - b, "B P", t[i, 3] - b,
          "PV_A issued", t[i, 5] - b, "PV_B issued", t[i, 7] - b)
