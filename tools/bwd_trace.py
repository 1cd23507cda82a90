"""Per-iteration event timeline of backward CTA (0,0) (profiling helper).
    python tools/bwd_trace.py [L]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402

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
    out.backward(torch.ones_like(out))
    torch.cuda.synchronize()
C.check(C.lib().spattn_debug_bwd_trace(None))
t = buf.view(-1, 16).cpu()
n = int((t[:, 0] > 0).sum())
t = t[:n].double()
names = ["mma:wait_qf", "mma:qf_ok", "mma:S_issued", "mma:dqf_ok", "mma:dP_issued", "mma:wait_pr",
         "mma:pr_ok", "mma:tail_issued", "sm:start", "sm:inputs_ok", "sm:pr_done", "dq:md_ok",
         "dq:dqf_done", "dq:staged", "tma:wait_qe", "tma:qe_ok"]
base = t[0, 0]
print("iterations traced:", n)
per = (t[n - 1, 0] - t[100, 0]) / (n - 101)
print(f"cycles per iteration (steady): {per:.0f}")
for i in (200, 201, 202):
    row = t[i] - t[i, 0]
    print(f"iter {i}: " + " ".join(f"{nm}={row[j]:.0f}" for j, nm in enumerate(names)))
import statistics  # noqa: E402
def gap(a, b, lag=0):
    return statistics.median([(t[i, b] - t[i - lag, a]).item() for i in range(200, n - 1)])
print("median MMA wait for Q/dO (qf_ok - wait_qf):", gap(0, 1))
print("median MMA wait for dQ drain (dqf_ok - S_issued):", gap(2, 3))
print("median MMA wait for softmax (pr_ok - wait_pr):", gap(5, 6))
print("median softmax wait for inputs (inputs_ok - start):", gap(8, 9))
print("median softmax compute (pr_done - inputs_ok):", gap(9, 10))
print("median dq drain (staged - md_ok):", gap(11, 13))
print("absolute timeline (cycles from iter 200 start):")
b0 = t[200, 0]
ev = []
for i in range(200, 204):
    for j, nm in enumerate(names):
        ev.append(((t[i, j] - b0).item(), f"{nm}({i})"))
for x, nm in sorted(ev):
    print(f"  {x:8.0f}  {nm}")
print("MMA-thread gaps (median over iterations 200..n-2):")
pairs = [(0, 1, "wait Q/dO"), (1, 2, "issue S"), (2, 3, "wait dQ drain"), (3, 4, "issue dP"),
         (4, 5, "-> tail start"), (5, 6, "wait softmax"), (6, 7, "issue dV dK dQ")]
for a_, b_, nm in pairs:
    print(f"  {nm:16s} {gap(a_, b_):7.0f}")
print(f"  {'-> next iter':16s} {statistics.median([(t[i + 1, 0] - t[i, 7]).item() for i in range(200, n - 2)]):7.0f}  (tail(i) end -> iter i+2 start is: {statistics.median([(t[i + 2, 0] - t[i, 7]).item() for i in range(200, n - 3)]):.0f})")
d1 = statistics.median([(t[i - 1, 5] - t[i, 4]).item() for i in range(201, n - 1)])
d2 = statistics.median([(t[i + 1, 0] - t[i - 1, 7]).item() for i in range(201, n - 2)])
print(f"GAP dP(i) issued -> tail(i-1) start: {d1:.0f}; tail(i-1) end -> iter i+1 start: {d2:.0f}")
