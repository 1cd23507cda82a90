"""Multi-tile shapes for the tcgen05 kernels (many 128-row query/key tiles, GQA, both head
dims, causal and full) against plain PyTorch fp32 attention on the same bf16 inputs — sizes the
f64 oracle cannot finish quickly. Tolerances are relative to bf16 operand rounding: relative
L2 error < 1e-2 and max abs error < 2e-2 * max|ref| for out, dq, dk, dv; lse within 1e-3."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def torch_attention(q, k, v, dout, causal):
    qf, kf, vf = (t.float().detach().requires_grad_(True) for t in (q, k, v))
    rep = q.shape[2] // k.shape[2]
    ke, ve = kf.repeat_interleave(rep, 2), vf.repeat_interleave(rep, 2)
    s = torch.einsum("blhd,bmhd->bhlm", qf, ke) / math.sqrt(q.shape[-1])
    if causal:
        L = q.shape[1]
        s = s.masked_fill(torch.triu(torch.ones(L, L, dtype=torch.bool, device=q.device), 1),
                          float("-inf"))
    lse = torch.logsumexp(s, -1)
    out = torch.einsum("bhlm,bmhd->blhd", torch.softmax(s, -1), ve)
    out.backward(dout.float())
    return out.detach(), lse.permute(0, 2, 1).detach(), qf.grad, kf.grad, vf.grad


def rel(a, b):
    return ((a.float() - b).norm() / b.norm()).item(), ((a.float() - b).abs().max() / b.abs().max()).item()


@pytest.mark.parametrize("L,H,Hkv,d,causal", [(2048, 8, 2, 128, True), (1536, 4, 4, 64, True),
                                              (1024, 4, 1, 128, False), (1920, 6, 2, 64, True)])
@pytest.mark.parametrize("family", ["tcgen05", "mma", "tcgen05_pp", "tcgen05_pair"])
def test_multi_tile_attention_vs_torch(L, H, Hkv, d, causal, family):
    import paper_2505_22296_b200 as P

    P.set_kernel_family(family)
    g = torch.Generator(device="cuda").manual_seed(L + H)
    q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
    out, lse = P.oracle_attention(q, k, v, causal=causal, return_lse=True)
    out.backward(dout)
    ro, rl, rdq, rdk, rdv = torch_attention(q, k, v, dout, causal)
    P.set_kernel_family("tcgen05")
    assert (lse - rl).abs().max().item() < 1e-3
    for name, got, want in (("out", out, ro), ("dq", q.grad, rdq), ("dk", k.grad, rdk),
                            ("dv", v.grad, rdv)):
        r2, rmax = rel(got, want)
        assert r2 < 1e-2 and rmax < 2e-2, (name, r2, rmax)
