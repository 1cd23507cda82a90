"""Shared helpers of the GPU parity tests: oracle-side data (reference Rng, bf16-rounded) and
the stated tolerance rule.

Tolerance: for out, lse, dq, dk, dv separately,
    max|gpu - oracle_f64| <= 2 * max|torch_fp32acc_bf16io - oracle_f64| + 1e-3 * max(1, max|oracle|)
where torch_fp32acc_bf16io is plain PyTorch attention computed in fp32 from the same
bf16-rounded inputs with its outputs rounded to bf16 (lse kept fp32). Permutations are
bit-exact (0 tolerance)."""
from __future__ import annotations

import math

import numpy as np
import torch

import seqpar_oracle as O


def to_dev(x: np.ndarray) -> torch.Tensor:
    """f64 values that are exactly bf16 -> bf16 CUDA tensor (exact)."""
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


def parity_inputs(seed, L, H, Hkv, d, bs=1):
    q, k, v, R = O.parity_data(seed, L, H, Hkv, d, bs)
    return tuple(O.bf16_round(x) for x in (q, k, v, R))


def oracle_all(q, k, v, R, causal=True, docs=None):
    if docs is None:
        return O.attention_fwd_bwd(q, k, v, R, causal=causal)
    return O.varlen_attention_fwd_bwd(q, k, v, R, docs, causal)


def torch_ref(q, k, v, R, causal=True, docs=None):
    """fp32 attention on bf16-rounded inputs, outputs rounded to bf16 (lse fp32)."""
    qt, kt, vt, Rt = (torch.from_numpy(x).float().cuda() for x in (q, k, v, R))
    qt.requires_grad_(True), kt.requires_grad_(True), vt.requires_grad_(True)
    bs, L, H, d = qt.shape
    rep = H // kt.shape[2]
    ke = kt.repeat_interleave(rep, dim=2)
    ve = vt.repeat_interleave(rep, dim=2)
    s = torch.einsum("blhd,bmhd->bhlm", qt, ke) / math.sqrt(d)
    allowed = torch.ones(L, L, dtype=torch.bool, device="cuda")
    if causal:
        allowed = torch.tril(allowed)
    if docs is not None:
        seg = torch.repeat_interleave(torch.arange(len(docs), device="cuda"),
                                      torch.tensor(docs, device="cuda"))
        allowed = allowed & (seg[:, None] == seg[None, :])
    s = s.masked_fill(~allowed, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    p = torch.softmax(s, dim=-1)
    out = torch.einsum("bhlm,bmhd->blhd", p, ve)
    (out * Rt).sum().backward()
    r = lambda t: t.detach().bfloat16().double().cpu().numpy()  # noqa: E731
    return {"out": r(out), "lse": lse.permute(0, 2, 1).detach().double().cpu().numpy(),
            "dq": r(qt.grad), "dk": r(kt.grad), "dv": r(vt.grad)}


def assert_close(name, gpu, oracle, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    oracle = np.asarray(oracle, dtype=np.float64)
    finite = np.isfinite(oracle)
    assert np.array_equal(np.isfinite(gpu), finite), f"{name}: non-finite pattern differs"
    err = np.max(np.abs(gpu[finite] - oracle[finite]), initial=0.0)
    ref_err = np.max(np.abs(ref[finite] - oracle[finite]), initial=0.0)
    bound = 2 * ref_err + 1e-3 * max(1.0, np.max(np.abs(oracle[finite]), initial=0.0))
    assert err <= bound, f"{name}: max err {err:.3e} > bound {bound:.3e} (torch ref err {ref_err:.3e})"
    return err, ref_err


def np_(t: torch.Tensor) -> np.ndarray:
    return t.detach().double().cpu().numpy()
