"""Parity at BASELINE.json's full sizes (configs c2-c5) through size-independent properties,
where the f64 oracle cannot run:

* row-stochastic softmax: for every kv head, the sum over keys of dV equals the sum over its
  query heads and query rows of dOut (P's rows sum to 1), and the sum over keys of dK is 0
  (dS's rows sum to 0, attention.cpp:190-209) — per neat-packed document for varlen;
* exact local blocks: causal rows whose dependencies are local are recomputed in fp32 torch —
  the first 128 query rows of out/lse/dq — and the last 128 rows' out/lse against all keys;
* engine agreement: Ring (zigzag) == Ulysses and Dummy-Head == XTuner on the same full-size
  inputs (different data movement and problem decomposition, same math).
Tolerances are bf16-operand level and written per check."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2505_22296_b200 as P

    P.set_kernel_family("tcgen05")
    return P


def inputs(L, H, Hkv, d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda h: torch.randn(1, L, h, d, device="cuda", generator=g).bfloat16()  # noqa: E731
    return mk(H), mk(Hkv), mk(Hkv), mk(H)


def run(P, engine, q, k, v, dout, sp, **kw):
    qt, kt, vt = (x.clone().requires_grad_(True) for x in (q, k, v))
    out, lse = P.engine_attention(engine, qt, kt, vt, sp, return_lse=True, **kw)
    out.backward(dout)
    torch.cuda.synchronize()
    return out, lse, qt.grad, kt.grad, vt.grad


def check_row_stochastic(dout, dk, dv, H, Hkv, docs=None):
    """sum_keys dV == sum_{queries, group heads} dOut; sum_keys dK == 0 (per document)."""
    rep = H // Hkv
    bounds = [0]
    for n in (docs or [dout.shape[1]]):
        bounds.append(bounds[-1] + n)
    for a, b in zip(bounds[:-1], bounds[1:]):
        do = dout[0, a:b].double().view(b - a, Hkv, rep, -1).sum(dim=(0, 2))
        sv = dv[0, a:b].double().sum(0)
        sk = dk[0, a:b].double().sum(0)
        scale = do.abs().max().item() + 1.0
        # bf16 rounding of each dV row (2^-9 relative) accumulates like a random walk
        tol = 4e-3 * math.sqrt(b - a) * dv[0, a:b].double().abs().max().item() + 1e-3 * scale
        assert (sv - do).abs().max().item() < tol, ((sv - do).abs().max().item(), tol)
        tol_k = 4e-3 * math.sqrt(b - a) * dk[0, a:b].double().abs().max().item() + 1e-3
        assert sk.abs().max().item() < tol_k, (sk.abs().max().item(), tol_k)


def torch_block(q, k, v, dout, scale):
    """fp32 causal attention of one local block (rows and keys aligned), with gradients."""
    qf, kf, vf = (t.float().requires_grad_(True) for t in (q, k, v))
    rep = qf.shape[1] // kf.shape[1]
    s = torch.einsum("lhd,mhd->hlm", qf, kf.repeat_interleave(rep, 1)) * scale
    n = qf.shape[0]
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=q.device), 1), float("-inf"))
    o = torch.einsum("hlm,mhd->lhd", torch.softmax(s, -1), vf.repeat_interleave(rep, 1))
    o.backward(dout.float())
    return o.detach(), torch.logsumexp(s, -1).T.detach(), qf.grad


def close(got, want, rel=2e-2):
    err = (got.float() - want.float()).abs().max().item()
    assert err <= rel * (want.abs().max().item() + 1e-6), (err, want.abs().max().item())


def test_c2_full_size(P):
    """c2: Llama-3-8B attention (32q/8kv, d=128), L=32768, causal — the bench workload."""
    L, H, Hkv, d = 32768, 32, 8, 128
    q, k, v, dout = inputs(L, H, Hkv, d, 2)
    out, lse, dq, dk, dv = run(P, "oracle", q, k, v, dout, 1, layout="naive")
    assert torch.isfinite(out).all() and torch.isfinite(dq).all()
    check_row_stochastic(dout, dk, dv, H, Hkv)
    scale = 1.0 / math.sqrt(d)
    # first 128 rows: causal dependencies are all local
    o, l, g = torch_block(q[0, :128], k[0, :128], v[0, :128], dout[0, :128], scale)
    close(out[0, :128], o)
    assert (lse[0, :128] - l).abs().max().item() < 2e-3
    close(dq[0, :128], g)
    # last 128 query rows: out and lse against all 32768 keys
    rep = H // Hkv
    ql = q[0, -128:].float()
    s = torch.einsum("lhd,mhd->hlm", ql, k[0].float().repeat_interleave(rep, 1)) * scale
    s[:, :, L - 128:] = s[:, :, L - 128:].masked_fill(
        torch.triu(torch.ones(128, 128, dtype=torch.bool, device="cuda"), 1), float("-inf"))
    lt = torch.logsumexp(s, -1)
    ot = torch.einsum("hlm,mhd->lhd", torch.softmax(s, -1), v[0].float().repeat_interleave(rep, 1))
    close(out[0, -128:], ot)
    assert (lse[0, -128:] - lt.T).abs().max().item() < 2e-3


def test_c4_ring_equals_ulysses_full_size(P):
    """c4: L=128K, Ring with zigzag balancing at SP=8 vs Ulysses SP=8 on the same inputs."""
    L, H, Hkv, d = 131072, 32, 8, 128
    q, k, v, dout = inputs(L, H, Hkv, d, 4)
    ring = run(P, "ring", q, k, v, dout, 8)
    check_row_stochastic(dout, ring[3], ring[4], H, Hkv)
    uly = run(P, "ulysses", q, k, v, dout, 8)
    for name, a, b in zip(("out", "lse", "dq", "dk", "dv"), ring, uly):
        if name == "lse":
            assert (a - b).abs().max().item() < 1e-3
        else:
            close(a, b, 1e-2)


def test_c3_dummy_head_equals_xtuner_full_size(P):
    """c3: Qwen2.5-7B attention (28q/4kv), L=64K, SP=8: Dummy-Head vs hidden-split."""
    L, H, Hkv, d = 65536, 28, 4, 128
    q, k, v, dout = inputs(L, H, Hkv, d, 3)
    dummy = run(P, "dummy_head", q, k, v, dout, 8)
    check_row_stochastic(dout, dummy[3], dummy[4], H, Hkv)
    xt = run(P, "xtuner", q, k, v, dout, 8)
    for name, a, b in zip(("out", "lse", "dq", "dk", "dv"), dummy, xt):
        if name == "lse":
            assert (a - b).abs().max().item() < 1e-3
        else:
            close(a, b, 1e-2)


def test_c5_varlen_full_size(P):
    """c5: neat-packed 256K tokens (documents of 1K-64K, reset positions), Ulysses vs Ring at
    SP=8; the row-stochastic identities hold per document."""
    import sys
    import os

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from sp_projection import c5_docs

    docs = c5_docs()
    L, H, Hkv, d = sum(docs), 32, 8, 128
    q, k, v, dout = inputs(L, H, Hkv, d, 5)
    uly = run(P, "ulysses", q, k, v, dout, 8, docs=docs)
    check_row_stochastic(dout, uly[3], uly[4], H, Hkv, docs)
    ring = run(P, "ring", q, k, v, dout, 8, docs=docs)
    for name, a, b in zip(("out", "lse", "dq", "dk", "dv"), uly, ring):
        if name == "lse":
            assert (a - b).abs().max().item() < 1e-3
        else:
            close(a, b, 1e-2)
    # the first document's first 128 rows are exact local blocks
    o, l, g = torch_block(q[0, :128], k[0, :128], v[0, :128], dout[0, :128], 1.0 / math.sqrt(d))
    close(uly[0][0, :128], o)
    close(uly[2][0, :128], g)
