"""The remaining cases of the reference's own test strategy on the CUDA path:
batched inputs (bs=2), bidirectional engines, degenerate USP == the pure engines bitwise
(tests/test_attention.cpp:470-501), Ring at sp=1 == the single-device engine bitwise (:503-515),
and the paper's §5.2 position-id pitfall (tests/test_model.cpp:234-267): rotating with each
rank's local 0-based ids instead of the global ones changes the result."""
import numpy as np
import pytest

from gpu_util import assert_close, np_, oracle_all, parity_inputs, to_dev, torch_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2505_22296_b200 as P

    P.set_kernel_family("tcgen05")
    return P


def run(P, engine, q, k, v, R, sp, **kw):
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out, lse = P.engine_attention(engine, qt, kt, vt, sp, return_lse=True, **kw)
    (out.float() * to_dev(R).float()).sum().backward()
    return {"out": np_(out), "lse": np_(lse), "dq": np_(qt.grad), "dk": np_(kt.grad), "dv": np_(vt.grad)}


def check(res, q, k, v, R, causal=True):
    orc, ref = oracle_all(q, k, v, R, causal), torch_ref(q, k, v, R, causal)
    for key in ("out", "lse", "dq", "dk", "dv"):
        assert_close(key, res[key], orc[key], ref[key])


@pytest.mark.parametrize("engine,sp,kw", [("ulysses", 2, {}), ("dummy_head", 4, {}), ("ring", 2, {}),
                                          ("usp", 4, dict(ulysses_degree=2, ring_degree=2)),
                                          ("xtuner", 4, {}), ("oracle", 1, {}),
                                          ("ulysses", 2, dict(force_messages=True)),
                                          ("usp", 4, dict(ulysses_degree=2, ring_degree=2, force_messages=True))])
def test_batched_engines(P, engine, sp, kw):
    # tests/test_attention.cpp:317-396 mixes bs=2 into the engine grid; with force_messages the
    # bs=2 blocks take the staged (not in-place) message path
    H = 6 if engine in ("dummy_head", "xtuner") else 4
    q, k, v, R = parity_inputs(31 + sp, 256, H, 2, 64, bs=2)
    check(run(P, engine, q, k, v, R, sp, **kw), q, k, v, R)


@pytest.mark.parametrize("engine,sp,kw", [("ulysses", 4, {}), ("ring", 2, {}), ("dummy_head", 4, {}),
                                          ("usp", 4, dict(ulysses_degree=2, ring_degree=2))])
def test_bidirectional_engines(P, engine, sp, kw):
    # tests/test_attention.cpp:398-404
    H = 6 if engine == "dummy_head" else 4
    q, k, v, R = parity_inputs(41 + sp, 256, H, 2, 64)
    check(run(P, engine, q, k, v, R, sp, causal=False, **kw), q, k, v, R, causal=False)


def test_degenerate_usp_equals_pure_engines_bitwise(P):
    # tests/test_attention.cpp:470-501: usp(u=sp, r=1) == ulysses, usp(u=1, r=sp) == ring
    q, k, v, R = parity_inputs(51, 256, 4, 2, 64)
    uly = run(P, "ulysses", q, k, v, R, 4, layout="usp", ulysses_degree=4, ring_degree=1)
    usp_u = run(P, "usp", q, k, v, R, 4, ulysses_degree=4, ring_degree=1)
    ring = run(P, "ring", q, k, v, R, 4)
    usp_r = run(P, "usp", q, k, v, R, 4, ulysses_degree=1, ring_degree=4)
    for key in uly:
        assert np.array_equal(uly[key], usp_u[key]), key
    # the fp32 dQ/dK accumulations are order-dependent across launches; forward is bitwise
    for key in ("out", "lse"):
        assert np.array_equal(ring[key], usp_r[key]), key
    for key in ("dq", "dk", "dv"):
        assert np.max(np.abs(ring[key] - usp_r[key])) <= 1e-2 * max(1.0, np.max(np.abs(ring[key])))


def test_ring_sp1_equals_single_device_bitwise(P):
    # tests/test_attention.cpp:503-515
    q, k, v, R = parity_inputs(61, 256, 4, 2, 64)
    a = run(P, "ring", q, k, v, R, 1)
    b = run(P, "oracle", q, k, v, R, 1, layout="naive")
    for key in ("out", "lse"):
        assert np.max(np.abs(a[key] - b[key])) <= 1e-6 * max(1.0, np.max(np.abs(b[key]))), key
    check(a, q, k, v, R)


def test_local_position_ids_corrupt_the_rotary_phases(P):
    # tests/test_model.cpp:234-267 / the paper's §5.2 pitfall: at sp > 1 each rank must rotate
    # with the GLOBAL ids of its rows; local 0-based ids give a visibly different layer
    L, sp = 256, 4
    q, k, v, R = parity_inputs(71, L, 4, 2, 64)
    glob = run(P, "ulysses", q, k, v, R, sp, position_ids=list(range(L)))
    local = run(P, "ulysses", q, k, v, R, sp, position_ids=[i % (L // sp) for i in range(L)])
    assert np.max(np.abs(glob["out"] - local["out"])) > 1e-3
    # and the global-id run is the single-device rope + attention
    single = run(P, "oracle", q, k, v, R, 1, layout="naive", position_ids=list(range(L)))
    for key in ("out", "lse"):
        assert np.max(np.abs(glob[key] - single[key])) <= 2e-2 * max(1.0, np.max(np.abs(single[key]))), key


def test_rank_all_to_all_matches_fabric_driver(P):
    """spattn_all_to_all on each rank's context (one thread per rank, the call an NCCL rank makes)
    equals the fabric's group driver and the reference's a2a semantics (comm.cpp:278-321)."""
    import threading

    import torch

    from paper_2505_22296_b200 import _lib as C

    sp, L, H, d = 4, 64, 8, 16
    fab = P.Fabric(sp)
    xs = [torch.randn(1, L, H, d, device="cuda").bfloat16() for _ in range(sp)]
    want = fab.all_to_all(xs, 2, 1)
    outs = [torch.empty_like(w) for w in want]
    torch.cuda.synchronize()
    errs = []

    def rank(r):
        try:
            C.check(C.lib().spattn_all_to_all(fab.ctxs[r], xs[r].data_ptr(), outs[r].data_ptr(), 1, L, H, d, 2, 2, 1))
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(sp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    torch.cuda.synchronize()
    assert not errs, errs
    for a, b in zip(outs, want):
        assert torch.equal(a, b)


@pytest.mark.parametrize("engine,sp,messages", [("ulysses", 2, False), ("ring", 2, False), ("dummy_head", 4, False),
                                                ("ulysses", 2, True), ("dummy_head", 4, True)])
def test_batched_varlen_with_rope(P, engine, sp, messages):
    """bs=2 neat-packed batches (the same document cut for every batch entry) with RoPE at
    per-document reset ids, against the composed per-document oracle; with ``messages`` the
    grouped q|k|v / dq|dk|dv exchanges carry rotated, staged (bs=2) blocks."""
    import seqpar_oracle as O

    docs = [100, 60, 96]
    L = sum(docs)
    H = 6 if engine == "dummy_head" else 4
    q, k, v, R = parity_inputs(81 + sp, L, H, 2, 64, bs=2)
    ids = P.document_position_ids(docs)
    res = run(P, engine, q, k, v, R, sp, docs=docs, position_ids=ids,
              **(dict(force_messages=True) if messages else {}))
    qr, kr = O.rope_apply(q, ids), O.rope_apply(k, ids)
    orc = O.varlen_attention_fwd_bwd(qr, kr, v, R, docs)
    orc["dq"] = O.rope_apply(orc["dq"], ids, inverse=True)
    orc["dk"] = O.rope_apply(orc["dk"], ids, inverse=True)
    ref = torch_ref(O.bf16_round(qr), O.bf16_round(kr), v, R, docs=docs)
    ref["dq"] = O.bf16_round(O.rope_apply(ref["dq"], ids, inverse=True))
    ref["dk"] = O.bf16_round(O.rope_apply(ref["dk"], ids, inverse=True))
    for key in ("out", "dq", "dk", "dv"):
        assert_close(key, res[key], orc[key], ref[key])
