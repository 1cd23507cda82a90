"""Pins the CPU oracle (oracle/) against fixtures produced by the unmodified reference
(tests/golden/make_golden.py). CPU only."""
import json
import os

import numpy as np
import pytest

import seqpar_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
Z = np.load(os.path.join(GOLD, "reference_attention.npz"))
API = json.load(open(os.path.join(GOLD, "reference_api.json")))

ATTN = sorted({k.split("/")[0] for k in Z.files if k.startswith("attn_")})
ENG = sorted({k.split("/")[0] for k in Z.files if k.startswith("engine_")})


@pytest.mark.parametrize("name", ATTN)
def test_oracle_attention_matches_reference(name):
    L, h, kv, d, causal, seed = (int(x) for x in Z[f"{name}/meta"])
    q, k, v, R = O.parity_data(seed, L, h, kv, d)
    # the oracle's Rng port reproduces the reference's fixture stream bit for bit
    assert np.array_equal(q.ravel(), Z[f"{name}/q"]) and np.array_equal(R.ravel(), Z[f"{name}/R"])
    r = O.attention_fwd_bwd(q, k, v, R, causal=bool(causal))
    assert np.max(np.abs(r["out"].ravel() - Z[f"{name}/out"])) < 1e-12
    assert np.max(np.abs(r["lse"].ravel() - Z[f"{name}/lse"])) < 1e-12
    for g in ("dq", "dk", "dv"):
        assert np.max(np.abs(r[g].ravel() - Z[f"{name}/{g}"])) < 1e-10, g


@pytest.mark.parametrize("name", ENG)
def test_oracle_matches_reference_engines(name):
    sp, L, h, kv, d, u, r, seed = (int(x) for x in Z[f"{name}/meta"])
    q, k, v, R = O.parity_data(seed, L, h, kv, d)
    ref = O.attention_fwd_bwd(q, k, v, R)
    # every reference engine reproduces the single-device oracle (report.cpp:170-171)
    assert np.max(np.abs(ref["out"].ravel() - Z[f"{name}/out"])) < 1e-10
    for g in ("dq", "dk", "dv"):
        assert np.max(np.abs(ref[g].ravel() - Z[f"{name}/{g}"])) < 1e-8


def test_hand_computed_two_tokens():
    # tests/test_attention.cpp:216-231
    q = np.array([1.0, 2.0]).reshape(1, 2, 1, 1)
    k = np.array([0.5, -1.0]).reshape(1, 2, 1, 1)
    v = np.array([3.0, 5.0]).reshape(1, 2, 1, 1)
    out = O.attention_fwd_bwd(q, k, v)["out"].ravel()
    w0, w1 = np.exp(2 * 0.5), np.exp(2 * -1.0)
    assert out[0] == pytest.approx(3.0, rel=1e-14)
    assert out[1] == pytest.approx((3 * w0 + 5 * w1) / (w0 + w1), rel=1e-12)
    full = O.attention_fwd_bwd(q, k, v, causal=False)["out"].ravel()
    a0, a1 = np.exp(0.5), np.exp(-1.0)
    assert full[0] == pytest.approx((3 * a0 + 5 * a1) / (a0 + a1), rel=1e-12)


def test_block_split_merge_equals_whole():
    # tests/test_attention.cpp:263-305: merged halves == one block (1e-12); one piece bitwise
    q, k, v, R = O.parity_data(5, 24, 2, 2, 4)
    pos = np.arange(24)
    whole = O.finalize_piece(O.block_forward(q, pos, k, v, pos))
    acc = None
    for sl in (slice(0, 10), slice(10, 24)):
        acc = O.merge_piece(acc, O.block_forward(q, pos, k[:, sl], v[:, sl], pos[sl]))
    merged = O.finalize_piece(acc)
    assert np.max(np.abs(merged[0] - whole[0])) < 1e-12
    single = O.finalize_piece(O.merge_piece(None, O.block_forward(q, pos, k, v, pos)))
    assert np.array_equal(single[0], whole[0]) and np.array_equal(single[1], whole[1])


def test_c1_full_size_checksums():
    c1 = API["c1"]
    m = c1["meta"]
    q, k, v, R = O.parity_data(m["seed"], m["L"], m["heads"], m["kv"], m["dim"])
    r = O.attention_fwd_bwd(q, k, v, R)
    for key in ("out", "lse", "dq", "dk", "dv"):
        val = r[key].reshape(m["L"], m["heads"], -1)
        np.testing.assert_allclose(val.sum(axis=(0, 2)), c1[key]["sum_per_head"], rtol=1e-9,
                                   atol=1e-7)
        np.testing.assert_allclose(val[[0, 1, 4095]], np.array(c1[key]["rows_0_1_4095"]),
                                   rtol=1e-10, atol=1e-10)


def test_layouts_padding_insp_bytes_match_reference():
    api = API["api"]
    for key, per_rank in api["positions"].items():
        mode, L, sp, u, r = key.split("/")
        owned = O.layout_owned(mode, int(L), int(sp), int(u), int(r))
        assert [o.tolist() for o in owned] == per_rank, key
        assert [O.causal_pair_count(o) for o in owned] == api["causal_pairs"][key]
    for *args, want in api["pad_length"]:
        assert O.pad_length(*args) == want
    for *args, want in api["insp"]:
        assert O.pick_xtuner_insp(*args) == want
    for fn, args, want in api["bytes"]:
        assert getattr(O, fn)(*args) == want, fn


def test_layout_rejects_like_reference():
    # tests/test_partition.cpp:82-89
    for args in [("naive", 10, 4), ("zigzag", 12, 4), ("zigzag", 0, 2)]:
        with pytest.raises(ValueError):
            O.layout_owned(*args)
    with pytest.raises(ValueError):
        O.layout_owned("usp", 16, 0, 3, 2)
    with pytest.raises(ValueError):
        O.pick_xtuner_insp(3, 4, 9)


def test_all_to_all_examples():
    # tests/test_comm.cpp:29-45 two-rank example, and the bitwise inverse (:47-62)
    d = [np.array([[10.0], [11.0]]), np.array([[20.0], [21.0]])]
    assert O.all_to_all(d, 0, 0, 1).tolist() == [[10.0, 20.0]]
    assert O.all_to_all(d, 1, 0, 1).tolist() == [[11.0, 21.0]]
    rng = np.random.default_rng(0)
    xs = [rng.uniform(-3, 3, size=(2, 3, 8, 4)) for _ in range(4)]
    fwd = [O.all_to_all(xs, i, 2, 1) for i in range(4)]
    assert fwd[0].shape == (2, 12, 2, 4)
    back = [O.all_to_all(fwd, i, 1, 2) for i in range(4)]
    assert all(np.array_equal(a, b) for a, b in zip(back, xs))
