"""Per-tile event timeline of forward CTA (0,0) (profiling helper; shares the bwd trace hook)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

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
t = buf.view(-1, 16).cpu().double()
n = int((t[:, 0] > 0).sum())
print("tiles traced:", n, " cycles per tile:", ((t[n - 2, 0] - t[50, 0]) / (n - 52)).item())
med = lambda f: statistics.median([f(i) for i in range(50, n - 2)])  # noqa: E731
print("mma: wait K       ", med(lambda i: (t[i, 1] - t[i, 0]).item()), "(incl. S issue)")
print("mma: S(j) -> PV(j-1) wait start", med(lambda i: (t[i - 1, 2] - t[i, 1]).item()))
print("mma: wait P(j-1)  ", med(lambda i: (t[i, 3] - t[i, 2]).item()))
print("mma: PV issue     ", med(lambda i: (t[i, 4] - t[i, 3]).item()))
print("mma: PV(j-1) done -> S(j+1) start", med(lambda i: (t[i + 1, 0] - t[i, 4]).item()))
print("sm : wait S(j)    ", med(lambda i: (t[i, 6] - t[i, 5]).item()))
print("sm : compute      ", med(lambda i: (t[i, 7] - t[i, 6]).item()))
print("sm : -> next start", med(lambda i: (t[i + 1, 5] - t[i, 7]).item()))
print("sm : S ld+wait    ", med(lambda i: (t[i, 8] - t[i, 6]).item()))
print("sm : max+exchange ", med(lambda i: (t[i, 9] - t[i, 8]).item()))
print("sm : rescale+PVwait", med(lambda i: (t[i, 10] - t[i, 9]).item()))
print("sm : exp+P store  ", med(lambda i: (t[i, 11] - t[i, 10]).item()))
print("sm : fence+arrive ", med(lambda i: (t[i, 7] - t[i, 11]).item()))
print("mma: wait KF      ", med(lambda i: (t[i, 12] - t[i, 0]).item()))
print("mma: wait SFREE   ", med(lambda i: (t[i, 13] - t[i, 12]).item()))
print("mma: S issue      ", med(lambda i: (t[i, 1] - t[i, 13]).item()))
print("mma: S(j) issued -> P(j-2) wait start", med(lambda i: (t[i - 2, 2] - t[i, 1]).item()))
for i in (100, 101, 102, 103):
    print(i, "S issue start", t[i,0]-t[100,0], "S issued", t[i,1]-t[100,0], "sm has S", t[i,6]-t[100,0], "P ready", t[i,7]-t[100,0], "PV sees P", t[i,3]-t[100,0], "PV issued", t[i,4]-t[100,0])
