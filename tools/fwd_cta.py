"""Whole-grid timeline of the forward kernel at c2 (profiling helper): per-CTA globaltimer records
(spattn_debug_fwd_cta_trace) -> main-loop ns per tile, prologue/epilogue, SM occupancy gaps."""
import collections
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

L, H, Hkv, d = 32768, 32, 8, 128
if len(sys.argv) > 1:
    P.set_kernel_family(sys.argv[1])  # e.g. tcgen05_pp
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16()
ncta = (L // 128) * H
buf = torch.zeros(ncta * 8, dtype=torch.int64, device="cuda")
for _ in range(2):
    P.oracle_attention(q, k, v)
C.check(C.lib().spattn_debug_fwd_cta_trace(buf.data_ptr()))
P.oracle_attention(q, k, v)
torch.cuda.synchronize()
C.check(C.lib().spattn_debug_fwd_cta_trace(None))
t = [r for r in buf.view(-1, 8).cpu().tolist() if r[0] > 0]
t0 = min(r[0] for r in t)
span = max(r[3] for r in t) - t0
tiles = sum(r[4] for r in t)
loop = sum(r[2] - r[1] for r in t)
print(f"kernel span {span / 1e6:.3f} ms, CTAs {len(t)}, tiles {tiles}")
print(f"main loop ns/tile (sum over CTAs / tiles): {loop / tiles:.1f}  "
      f"-> {loop / tiles * 1.0:.0f} ns; x148 SMs ideal span {loop / 148 / 1e6:.3f} ms")
print(f"prologue (entry -> first S) median {statistics.median(r[1] - r[0] for r in t):.0f} ns, "
      f"epilogue (loop end -> exit) median {statistics.median(r[3] - r[2] for r in t):.0f} ns")
by_sm = collections.defaultdict(list)
for r in t:
    by_sm[r[5]].append(r)
busy, gaps = 0, []
for sm, rs in by_sm.items():
    rs.sort(key=lambda r: r[0])
    busy += sum(r[3] - r[0] for r in rs)
    gaps += [b[0] - a[3] for a, b in zip(rs, rs[1:])]
print(f"SMs used {len(by_sm)}, SM busy fraction {busy / (len(by_sm) * span):.3f}, "
      f"median inter-CTA gap {statistics.median(gaps):.0f} ns, mean {statistics.mean(gaps):.0f} ns")
ends = sorted(max(r[3] for r in rs) - t0 for rs in by_sm.values())
print(f"SM finish times: first {ends[0] / 1e6:.3f} ms, median {ends[len(ends) // 2] / 1e6:.3f}, "
      f"last {ends[-1] / 1e6:.3f}")
# loop ns/tile by CTA size
for lo, hi in ((1, 32), (32, 128), (128, 257)):
    sel = [r for r in t if lo <= r[4] < hi]
    if sel:
        print(f"  n_tiles in [{lo},{hi}): ns/tile {sum(r[2] - r[1] for r in sel) / sum(r[4] for r in sel):.1f}")
