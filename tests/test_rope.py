"""RoPE with global position ids (rope_apply, reference tensor.cpp:548-607; Model::forward's call
site model.cpp:339-344): the CPU oracle pinned to the unmodified reference
(tests/golden/reference_rope.npz, made by tests/golden/make_golden.py), the reference's own rope
properties (tests/test_tensor.cpp:133-190), and — on the GPU — the rotating copy kernels and the
engines with rope fused into the Ulysses all-to-all, against the oracle."""
import os

import numpy as np
import pytest

import seqpar_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
Z = np.load(os.path.join(GOLD, "reference_rope.npz"))
ROPE = sorted({k.split("/")[0] for k in Z.files if k.startswith("rope_L")})
ROPE_ENG = sorted({k.split("/")[0] for k in Z.files if k.startswith("rope_engine_")})


def _ids(L, scale, off, positions=None):
    p = np.arange(L) if positions is None else np.asarray(positions)
    return p * scale + off


# ------------------------------------------------------------------------------ CPU oracle
@pytest.mark.parametrize("name", ROPE)
def test_oracle_rope_matches_reference(name):
    L, h, d, sc, off, seed = (int(x) for x in Z[f"{name}/meta"])
    x, _, _, R = O.parity_data(seed, L, h, h, d)
    assert np.array_equal(x.ravel(), Z[f"{name}/x"])
    ids = _ids(L, sc, off)
    y = O.rope_apply(x, ids)
    assert np.max(np.abs(y.ravel() - Z[f"{name}/y"])) < 1e-12
    # tape backward of sum(y * R) = inverse rotation of R (tensor.cpp:589-600)
    dx = O.rope_apply(R, ids, inverse=True)
    assert np.max(np.abs(dx.ravel() - Z[f"{name}/dx"])) < 1e-12


@pytest.mark.parametrize("name", ROPE_ENG)
def test_oracle_rope_engines_match_reference(name):
    sp, L, h, kv, d, u, r, sc, off, seed = (int(x) for x in Z[f"{name}/meta"])
    q, k, v, R = O.parity_data(seed, L, h, kv, d)
    ids = _ids(L, sc, off)
    res = O.attention_fwd_bwd(O.rope_apply(q, ids), O.rope_apply(k, ids), v, R)
    assert np.max(np.abs(res["out"].ravel() - Z[f"{name}/out"])) < 1e-10
    dq = O.rope_apply(res["dq"], ids, inverse=True)
    dk = O.rope_apply(res["dk"], ids, inverse=True)
    for g, val in (("dq", dq), ("dk", dk), ("dv", res["dv"])):
        assert np.max(np.abs(val.ravel() - Z[f"{name}/{g}"])) < 1e-8, g


def test_rope_dot_products_depend_on_relative_position():
    # tests/test_tensor.cpp:133-151
    rng = np.random.default_rng(11)
    q, k = rng.uniform(-2, 2, (1, 1, 1, 8)), rng.uniform(-2, 2, (1, 1, 1, 8))
    dot = lambda m, n: float(np.sum(O.rope_apply(q, [m]) * O.rope_apply(k, [n])))  # noqa: E731
    assert abs(dot(3, 1) - dot(10, 8)) < 1e-10 and abs(dot(3, 1) - dot(103, 101)) < 1e-10


def test_rope_negated_positions_invert():
    # tests/test_tensor.cpp:153-162
    x = np.random.default_rng(13).uniform(-2, 2, (1, 4, 2, 6))
    pos = np.array([0, 5, 9, 2])
    back = O.rope_apply(O.rope_apply(x, pos), -pos)
    assert np.max(np.abs(back - x)) < 1e-12


def test_rope_preserves_norms():
    # tests/test_tensor.cpp:164-180
    x = np.random.default_rng(17).uniform(-2, 2, (1, 3, 2, 8))
    y = O.rope_apply(x, [7, 21, 2])
    assert np.max(np.abs(np.sum(x * x, -1) - np.sum(y * y, -1))) < 1e-10


def test_rope_validation():
    # tests/test_tensor.cpp:182-189
    with pytest.raises(O.ShapeError):
        O.rope_apply(np.zeros((1, 2, 1, 5)), [0, 1])
    with pytest.raises(O.ShapeError):
        O.rope_apply(np.zeros((1, 4, 1, 4)), [0, 1])


# ---------------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def P():
    import paper_2505_22296_b200 as P

    return P


def _bound(gpu, oracle, ulp_rel=2 ** -7):
    # bf16 outputs of an fp32 rotation: within one bf16 rounding of |value| (+ fp32 noise)
    return np.all(np.abs(gpu - oracle) <= ulp_rel * np.abs(oracle) + 1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("L,h,d,scale,off", [(64, 4, 128, 1, 0), (37, 3, 64, 1, 131000),
                                             (16, 2, 6, 7, 100000), (40, 5, 16, -3, 9)])
def test_gpu_rope_apply_matches_oracle(P, L, h, d, scale, off):
    import torch
    from gpu_util import np_, to_dev

    x, _, _, R = (O.bf16_round(a) for a in O.parity_data(29 + L, L, h, h, d, bs=2))
    ids = _ids(L, scale, off)
    xt = to_dev(x).requires_grad_(True)
    y = P.rope_apply(xt, ids.tolist())
    (y.float() * to_dev(R).float()).sum().backward()
    assert _bound(np_(y), O.rope_apply(x, ids))
    assert _bound(np_(xt.grad), O.rope_apply(R, ids, inverse=True))
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_gpu_rope_validation(P):
    import torch

    with pytest.raises(P.ShapeError):
        P.rope_apply(torch.zeros(1, 2, 1, 5, dtype=torch.bfloat16, device="cuda"), [0, 1])
    with pytest.raises(P.ShapeError):
        P.rope_apply(torch.zeros(1, 4, 1, 4, dtype=torch.bfloat16, device="cuda"), [0, 1])


ENGINE_ROPE_CASES = [
    # engine, sp, L, H, Hkv, d, extra kwargs
    ("ulysses", 2, 256, 4, 2, 128, {}), ("ulysses", 4, 256, 8, 2, 64, {}),
    ("dummy_head", 4, 256, 6, 2, 64, {}), ("dummy_head", 8, 256, 28, 4, 128, {}),
    ("xtuner", 4, 256, 6, 6, 64, {}), ("ring", 4, 256, 4, 2, 64, {}),
    ("usp", 4, 256, 4, 2, 64, dict(ulysses_degree=2, ring_degree=2)),
    ("oracle", 1, 200, 4, 2, 128, {}),
]


@pytest.mark.gpu
@pytest.mark.parametrize("engine,sp,L,H,Hkv,d,kw", ENGINE_ROPE_CASES)
@pytest.mark.parametrize("messages", [False, True])
@pytest.mark.parametrize("offset", [0, 70000])
def test_gpu_engines_with_fused_rope(P, engine, sp, L, H, Hkv, d, kw, messages, offset):
    """engine(rope(q), rope(k), v) with dq, dk pulled back through the rotation, against the
    oracle composition (pinned by test_oracle_rope_engines_match_reference)."""
    from gpu_util import assert_close, np_, parity_inputs, to_dev, torch_ref

    if engine == "oracle" and messages:
        pytest.skip("single device")
    P.set_kernel_family("tcgen05")
    q, k, v, R = parity_inputs(3000 + sp * 13 + H + offset, L, H, Hkv, d)
    ids = _ids(L, 1, offset)
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out, lse = P.engine_attention(engine, qt, kt, vt, sp, return_lse=True, position_ids=ids.tolist(),
                                  force_messages=messages, **kw)
    (out.float() * to_dev(R).float()).sum().backward()
    # oracle: f64 rotation of the bf16 inputs; the tolerance reference is torch fp32 attention
    # on the bf16-rounded rotated inputs (what a bf16 rope -> attention pipeline sees)
    qr, kr = O.rope_apply(q, ids), O.rope_apply(k, ids)
    orc = O.attention_fwd_bwd(qr, kr, v, R)
    orc["dq"] = O.rope_apply(orc["dq"], ids, inverse=True)
    orc["dk"] = O.rope_apply(orc["dk"], ids, inverse=True)
    # (a bf16 pipeline rounds dq/dk again after the inverse rotation, as the product does)
    ref = torch_ref(O.bf16_round(qr), O.bf16_round(kr), v, R)
    ref["dq"] = O.bf16_round(O.rope_apply(ref["dq"], ids, inverse=True))
    ref["dk"] = O.bf16_round(O.rope_apply(ref["dk"], ids, inverse=True))
    got = {"out": np_(out), "lse": np_(lse), "dq": np_(qt.grad), "dk": np_(kt.grad),
           "dv": np_(vt.grad)}
    for key in ("out", "lse", "dq", "dk", "dv"):
        assert_close(key, got[key], orc[key], ref[key])


@pytest.mark.gpu
def test_gpu_fused_rope_equals_separate_rope(P):
    """Ulysses with rope fused into the all-to-all gives bit-identical results to rope_apply
    followed by the engine (same fp32 rotation, same attention kernels)."""
    from gpu_util import np_, parity_inputs, to_dev

    q, k, v, R = parity_inputs(77, 256, 8, 2, 128)
    ids = list(range(5, 5 + 256))

    def run(fused):
        qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
        if fused:
            out = P.engine_attention("ulysses", qt, kt, vt, 4, position_ids=ids)
        else:
            out = P.engine_attention("ulysses", P.rope_apply(qt, ids), P.rope_apply(kt, ids), vt, 4)
        (out.float() * to_dev(R).float()).sum().backward()
        return [np_(t) for t in (out, qt.grad, kt.grad, vt.grad)]

    for a, b in zip(run(True), run(False)):
        assert np.array_equal(a, b)
