"""Stream timeline of the ring engine's steps on the loopback fabric (profiling helper): per
rank, the attention kernels on the compute stream, the k|v and dk|dv hops on the comm stream and
the dk|dv adds, from spattn_debug_timeline. Prints, for the backward, the compute stream's idle
gap between consecutive step kernels and how much of each hop overlaps a kernel of the same rank.
    python tools/ring_timeline.py [sp] [L] [--messages]"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
sp = int(args[0]) if args else 4
L = int(args[1]) if len(args) > 1 else 65536
messages = "--messages" in sys.argv
H, Hkv, d = 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
fab = P.Fabric(sp, force_messages=messages)
for traced in (False, True):
    if traced:
        C.check(C.lib().spattn_debug_timeline(1))
    out = P.engine_attention("ring", q, k, v, sp, fabric=fab)
    out.backward(dout)
    torch.cuda.synchronize()
C.check(C.lib().spattn_debug_timeline(0))
N = 4096
st, en = (ctypes.c_double * N)(), (ctypes.c_double * N)()
kd, rk = (ctypes.c_int * N)(), (ctypes.c_int * N)()
n = ctypes.c_int64()
C.check(C.lib().spattn_debug_timeline_read(st, en, kd, rk, N, ctypes.byref(n)))
recs = [(st[i], en[i], kd[i], rk[i]) for i in range(min(n.value, N))]
names = {0: "fwd", 1: "bwd", 2: "kv-hop", 3: "dkdv-add", 4: "dkdv-hop"}
print(f"ring sp={sp} L={L} {'messages' if messages else 'peer reads'}: {len(recs)} records")
bwd0 = min(r[0] for r in recs if r[2] == 1)
for r in sorted(recs):
    if r[3] == 0 and r[0] >= bwd0 - 1e-3:
        print(f"  rank0 {names[r[2]]:9s} {r[0] - bwd0:9.3f} -> {r[1] - bwd0:9.3f} ms")


def overlap(a, b):
    return max(0.0, min(a[1], b[1]) - max(a[0], b[0]))


gaps, hidden = [], {2: [], 4: []}
for rank in range(sp):
    ks = sorted(r for r in recs if r[3] == rank and r[2] == 1)
    gaps += [ks[i + 1][0] - ks[i][1] for i in range(len(ks) - 1)]
    for kind in (2, 4):
        for h in (r for r in recs if r[3] == rank and r[2] == kind):
            dur = h[1] - h[0]
            if dur > 0:
                hidden[kind].append(sum(overlap(h, kk) for kk in ks) / dur)
# ordering evidence: does step s+1's kernel wait for step s's dk|dv hop (the r1 design did)?
early = []
for rank in range(sp):
    ks = sorted(r for r in recs if r[3] == rank and r[2] == 1)
    hs = sorted(r for r in recs if r[3] == rank and r[2] == 4)
    for s_ in range(min(len(ks) - 1, len(hs))):
        early.append(hs[s_][1] - ks[s_ + 1][0])  # > 0: next kernel started before the hop ended
print(f"step s+1 kernel start precedes the end of step s's dk|dv hop by median "
      f"{statistics.median(early):.3f} ms (min {min(early):.3f}; > 0 = the hop is off the compute stream's path)")
kt = [r[1] - r[0] for r in recs if r[2] == 1]
print(f"backward: median step kernel {statistics.median(kt):.3f} ms; median compute-stream gap between "
      f"step kernels {statistics.median(gaps):.3f} ms (max {max(gaps):.3f})")
for kind in (2, 4):
    if hidden[kind]:
        print(f"  {names[kind]}: median fraction overlapped by the same rank's kernels "
              f"{statistics.median(hidden[kind]):.2f}")
