"""Backward kernel check against a torch fp32 reference on a few shapes (ragged lengths, GQA,
causal / full), then c2 / 128K-shape timings of the backward. Run with and without
SPATTN_BWD_PAIR=1 to compare the CTA-pair backward with the single-CTA kernel.
    python tools/pair_check.py [quick]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402
from paper_2505_22296_b200 import _lib as C  # noqa: E402


def ref(q, k, v, dout, causal):
    qf, kf, vf = (x.detach().float().requires_grad_(True) for x in (q, k, v))
    rep = q.shape[2] // k.shape[2]
    ke, ve = kf.repeat_interleave(rep, 2), vf.repeat_interleave(rep, 2)
    s = torch.einsum("blhd,bmhd->bhlm", qf, ke) / q.shape[-1] ** 0.5
    if causal:
        L = q.shape[1]
        s = s.masked_fill(torch.ones(L, L, dtype=torch.bool, device=q.device).triu(1), float("-inf"))
    o = torch.einsum("bhlm,bmhd->blhd", s.softmax(-1), ve)
    o.backward(dout.float())
    return o, qf.grad, kf.grad, vf.grad


def run(L, H, Hkv, d, causal, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
    out = P.oracle_attention(q, k, v, causal=causal)
    out.backward(dout)
    torch.cuda.synchronize()
    ro, rq, rk, rv = ref(q, k, v, dout, causal)
    errs = []
    for got, want in ((out, ro), (q.grad, rq), (k.grad, rk), (v.grad, rv)):
        e = (got.float() - want).abs().max().item() / max(1.0, want.abs().max().item())
        errs.append(e)
    bad = any(e > 2e-2 or e != e for e in errs)
    print(f"L={L} H={H}/{Hkv} d={d} causal={causal}: out {errs[0]:.2e} dq {errs[1]:.2e} "
          f"dk {errs[2]:.2e} dv {errs[3]:.2e}{'  <-- FAIL' if bad else ''}", flush=True)
    return not bad


def timing(L, H, Hkv, d=128, reps=3):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
    for i in range(reps + 1):
        if i == 1:
            torch.cuda.synchronize()
            C.check(C.lib().spattn_profile_enable(1))
        P.oracle_attention(q, k, v).backward(dout)
    torch.cuda.synchronize()
    C.check(C.lib().spattn_profile_enable(0))
    ms, n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    C.check(C.lib().spattn_profile_read(ms, n))
    pairs = L * (L + 1) // 2 * H
    f, b = ms[0] / reps, ms[1] / reps
    print(f"TIMING L={L} H={H}/{Hkv}: fwd {f:.3f} ms {4 * d * pairs / f / 1e9:.0f} TFLOP/s, "
          f"bwd {b:.3f} ms {10 * d * pairs / b / 1e9:.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    print("pair backward:", bool(os.environ.get("SPATTN_BWD_PAIR")), flush=True)
    if len(sys.argv) > 1 and sys.argv[1] == "t":
        timing(32768, 32, 8)
        sys.exit(0)
    ok = True
    for L, H, Hkv, causal in ((128, 2, 1, True), (256, 4, 2, True), (200, 2, 2, True), (384, 4, 1, False),
                              (1000, 8, 2, True), (129, 1, 1, True), (777, 4, 4, False), (2048, 4, 1, True)):
        ok &= run(L, H, Hkv, 128, causal)
    if len(sys.argv) < 2 or sys.argv[1] != "quick":
        timing(32768, 32, 8)
        timing(131072, 32, 8, reps=1)
    print("ALL OK" if ok else "SOME FAILED")
