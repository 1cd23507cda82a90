"""GPU parity of the CUDA path against the CPU oracle (oracle/, pinned to the reference by
tests/test_oracle_golden.py). Every call goes through libspattn.so's C ABI."""
import numpy as np
import pytest
import torch

import seqpar_oracle as O
from gpu_util import assert_close, np_, oracle_all, parity_inputs, to_dev, torch_ref

pytestmark = pytest.mark.gpu

FAMILIES = ["tcgen05", "mma", "tcgen05_pp", "tcgen05_pair", "tcgen05_q64"]


@pytest.fixture(scope="module")
def P():
    import paper_2505_22296_b200 as P

    return P


def run_engine(P, engine, q, k, v, R, sp, causal=True, docs=None, **kw):
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out, lse = P.engine_attention(engine, qt, kt, vt, sp, causal=causal, docs=docs,
                                  return_lse=True, **kw)
    (out.float() * to_dev(R).float()).sum().backward()
    return {"out": np_(out), "lse": np_(lse), "dq": np_(qt.grad), "dk": np_(kt.grad),
            "dv": np_(vt.grad)}


def check_all(res, orc, ref, keys=("out", "lse", "dq", "dk", "dv")):
    for key in keys:
        assert_close(key, res[key], orc[key], ref[key])


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("L,H,Hkv,d,causal", [(256, 4, 4, 64, True), (320, 8, 2, 128, True),
                                              (200, 3, 1, 64, True), (192, 2, 2, 128, False),
                                              (130, 4, 2, 64, False)])
def test_oracle_engine_matches_oracle(P, family, L, H, Hkv, d, causal):
    P.set_kernel_family(family)
    q, k, v, R = parity_inputs(11 + L, L, H, Hkv, d)
    res = run_engine(P, "oracle", q, k, v, R, 1, causal)
    check_all(res, oracle_all(q, k, v, R, causal), torch_ref(q, k, v, R, causal))


# the reference parity grid shapes (report.cpp:295-297) scaled to kernel head dims
ENGINE_CASES = [
    ("ulysses", 2, 256, 4, 4, 64), ("ulysses", 4, 256, 8, 2, 64), ("ulysses", 2, 128, 4, 4, 128),
    ("dummy_head", 4, 256, 6, 6, 64), ("dummy_head", 4, 256, 6, 3, 64),
    ("dummy_head", 8, 256, 14, 2, 64), ("dummy_head", 8, 256, 28, 4, 64),
    ("xtuner", 4, 256, 6, 6, 64), ("xtuner", 4, 256, 6, 2, 64),
    ("ring", 2, 256, 4, 4, 64), ("ring", 4, 256, 4, 2, 64), ("ring", 8, 512, 2, 2, 128),
    ("usp", 4, 256, 4, 4, 64), ("usp", 8, 512, 6, 2, 64),
]


@pytest.mark.parametrize("engine,sp,L,H,Hkv,d", ENGINE_CASES)
@pytest.mark.parametrize("messages", [False, True])
def test_engines_match_oracle(P, engine, sp, L, H, Hkv, d, messages):
    P.set_kernel_family("tcgen05")
    kw = {}
    if engine == "usp":
        kw = dict(ulysses_degree=2, ring_degree=sp // 2)
    q, k, v, R = parity_inputs(1000003 + sp * 7 + H, L, H, Hkv, d)
    res = run_engine(P, engine, q, k, v, R, sp, force_messages=messages, **kw)
    check_all(res, oracle_all(q, k, v, R), torch_ref(q, k, v, R))


@pytest.mark.parametrize("engine", ["ring", "ulysses", "dummy_head"])
def test_one_member_engines_are_the_single_block(P, engine):
    # a one-member ring is its diagonal step alone (attention.cpp:279-291): the engines take the
    # single-block path (bf16 dK / dV, no ring accumulators) and agree with the oracle engine
    # bit for bit, and with the CPU oracle
    P.set_kernel_family("tcgen05")
    q, k, v, R = parity_inputs(41, 384, 8, 2, 128)
    a = run_engine(P, engine, q, k, v, R, 1)
    b = run_engine(P, "oracle", q, k, v, R, 1)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    check_all(a, oracle_all(q, k, v, R), torch_ref(q, k, v, R))


def test_dummy_head_equals_ulysses_bitwise_when_divisible(P):
    # tests/test_attention.cpp:455-468
    q, k, v, R = parity_inputs(3, 256, 8, 4, 64)
    a = run_engine(P, "ulysses", q, k, v, R, 4)
    b = run_engine(P, "dummy_head", q, k, v, R, 4)
    for key in a:
        assert np.array_equal(a[key], b[key]), key


def test_ulysses_accepts_zigzag_layout(P):
    # tests/test_attention.cpp:406-412: a2a engines accept the zigzag layout
    q, k, v, R = parity_inputs(5, 256, 4, 2, 64)
    res = run_engine(P, "ulysses", q, k, v, R, 4, layout="zigzag")
    check_all(res, oracle_all(q, k, v, R), torch_ref(q, k, v, R))


@pytest.mark.parametrize("engine,sp", [("ulysses", 2), ("ring", 2), ("ring", 4), ("oracle", 1)])
def test_varlen_docs_match_composed_oracle(P, engine, sp):
    docs = [70, 128, 30, 28]  # neat-packed documents, reset positions per document
    L = sum(docs)
    q, k, v, R = parity_inputs(77, L, 4, 2, 64)
    res = run_engine(P, engine, q, k, v, R, sp, docs=docs)
    check_all(res, oracle_all(q, k, v, R, docs=docs), torch_ref(q, k, v, R, docs=docs))


def test_infeasible_configs_raise(P):
    # tests/test_attention.cpp:414-453
    q, k, v, R = parity_inputs(1, 256, 6, 6, 64)
    with pytest.raises(ValueError):
        run_engine(P, "ulysses", q, k, v, R, 4)  # 6 heads % 4
    with pytest.raises(ValueError):
        run_engine(P, "ring", q, k, v, R, 4, layout="naive")  # ring needs zigzag
    with pytest.raises(ValueError):
        run_engine(P, "oracle", q, k, v, R, 2)


@pytest.mark.parametrize("dtype", [torch.float64, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("sp", [2, 4])
@pytest.mark.parametrize("messages", [False, True])
def test_all_to_all_bit_exact(P, dtype, sp, messages):
    # comm.cpp:278-321 semantics; round trip is the identity (tests/test_comm.cpp:47-62)
    rng = np.random.default_rng(sp)
    xs = [rng.uniform(-3, 3, size=(2, 12, 8, 4)) for _ in range(sp)]
    fab = P.Fabric(sp, force_messages=messages)
    dev = [torch.from_numpy(x).to(dtype).cuda() for x in xs]
    host = [t.double().cpu().numpy() for t in dev]
    fwd = fab.all_to_all(dev, 2, 1)
    for i in range(sp):
        want = O.all_to_all(host, i, 2, 1)
        assert np.array_equal(np_(fwd[i]), want)
    back = fab.all_to_all(fwd, 1, 2)
    for a, b in zip(back, dev):
        assert torch.equal(a, b)


@pytest.mark.parametrize("mode,L,sp,u,r", [("naive", 64, 4, 0, 0), ("zigzag", 64, 4, 0, 0),
                                           ("zigzag", 96, 8, 0, 0), ("usp", 64, 8, 2, 4)])
def test_shard_gather_rows_bit_exact(P, mode, L, sp, u, r):
    x = torch.randn(2, L, 3, 5, dtype=torch.float64, device="cuda")
    owned = O.layout_owned(mode, L, sp, u, r)
    shards = [P.shard_rows(x, mode, sp, i, u, r) for i in range(sp)]
    for i in range(sp):
        assert torch.equal(shards[i].cpu(), x.cpu()[:, torch.from_numpy(owned[i])])
    assert torch.equal(P.gather_rows(shards, mode, sp, u, r), x)


def test_lse_merge_matches_merge_piece(P):
    import ctypes

    from paper_2505_22296_b200 import _lib as C

    rng = np.random.default_rng(0)
    rows, d = 37, 64
    oa, ob = rng.standard_normal((rows, d)), rng.standard_normal((rows, d))
    la, lb = rng.standard_normal(rows), rng.standard_normal(rows)
    la[3] = -np.inf
    lb[5] = -np.inf
    acc_o, acc_l = torch.tensor(oa, dtype=torch.float32, device="cuda"), torch.tensor(la, dtype=torch.float32, device="cuda")
    po, pl = torch.tensor(ob, dtype=torch.float32, device="cuda"), torch.tensor(lb, dtype=torch.float32, device="cuda")
    C.check(C.lib().spattn_lse_merge(torch.cuda.current_stream().cuda_stream, acc_o.data_ptr(),
                                     acc_l.data_ptr(), po.data_ptr(), pl.data_ptr(), rows, d))
    # merge_piece (attention.cpp:117-149) on unnormalised pieces: num = out * e^lse, max=lse, norm=1
    mx = np.maximum(la, lb)
    want_l = np.where(np.isneginf(mx), -np.inf, mx + np.log(np.exp(la - mx) + np.exp(lb - mx)))
    wa = np.where(np.isneginf(la), 0, np.exp(la - want_l))
    wb = np.where(np.isneginf(lb), 0, np.exp(lb - want_l))
    want_o = oa * wa[:, None] + ob * wb[:, None]
    np.testing.assert_allclose(acc_o.cpu().numpy(), want_o, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(acc_l.cpu().numpy(), want_l, rtol=1e-6, atol=1e-6)


def test_block_merge_equals_whole(P):
    # tests/test_attention.cpp:263-305 on the kernel-level API (block fwd + merge + finalize)
    import ctypes

    from paper_2505_22296_b200 import _lib as C

    L, H, Hkv, d = 192, 2, 1, 64
    q, k, v, R = parity_inputs(5, L, H, Hkv, d)
    pos = np.arange(L, dtype=np.int64)
    s = torch.cuda.current_stream().cuda_stream
    qt, kt, vt = to_dev(q), to_dev(k), to_dev(v)
    accs = []
    for cuts in ([(0, L)], [(0, 70), (70, L)]):
        acc_o = torch.zeros(1, L, H, d, device="cuda")
        acc_l = torch.full((1, L, H), float("-inf"), device="cuda")
        for a, b in cuts:
            kp = np.ascontiguousarray(pos[a:b])
            C.check(C.lib().spattn_block_fwd(
                s, 1, H, Hkv, d, qt.data_ptr(), pos.ctypes.data_as(C._i64p), L,
                kt[:, a:b].contiguous().data_ptr(), vt[:, a:b].contiguous().data_ptr(),
                kp.ctypes.data_as(C._i64p), b - a, 1, 1 / np.sqrt(d), acc_o.data_ptr(),
                acc_l.data_ptr(), None))
        torch.cuda.synchronize()
        accs.append((acc_o.double().cpu().numpy(), acc_l.double().cpu().numpy()))
    orc = oracle_all(q, k, v, R)
    np.testing.assert_allclose(accs[0][0], orc["out"], atol=2e-2)
    # bf16 P differs with the tile split (different running max): bf16-level agreement
    np.testing.assert_allclose(accs[1][0], accs[0][0], atol=5e-3)
    np.testing.assert_allclose(accs[1][1], accs[0][1], atol=1e-4)


@pytest.mark.parametrize("d", [64, 128])
def test_block_backward_query_split_matches(P, d, monkeypatch):
    """A fully admitted block (every query sees every key: a ring step's off-diagonal block) on
    an fp32-accumulating backward launch of few CTAs is cut along the query range
    (engine.cpp split_query_ranges); its dq / dk / dv equal the uncut launch's up to fp32
    summation order, and the reference gradients of that block."""
    import ctypes

    from paper_2505_22296_b200 import _lib as C

    lq, lk, H, Hkv = 1000, 384, 4, 2
    rng = np.random.default_rng(17)
    bf = lambda *s: O.bf16_round(rng.uniform(-2, 2, s))  # noqa: E731
    q, k, v = bf(1, lq, H, d), bf(1, lk, Hkv, d), bf(1, lk, Hkv, d)
    R = rng.uniform(-1, 1, (1, lq, H, d))
    qpos = np.arange(lk, lk + lq, dtype=np.int64)  # queries after every key: all admitted
    kpos = np.arange(lk, dtype=np.int64)
    s = torch.cuda.current_stream().cuda_stream
    qt, kt, vt = to_dev(q), to_dev(k), to_dev(v)
    # forward of the block (merge into an empty accumulator), then its backward
    acc_o = torch.zeros(1, lq, H, d, device="cuda")
    acc_l = torch.full((1, lq, H), float("-inf"), device="cuda")
    C.check(C.lib().spattn_block_fwd(s, 1, H, Hkv, d, qt.data_ptr(), qpos.ctypes.data_as(C._i64p), lq,
                                     kt.data_ptr(), vt.data_ptr(), kpos.ctypes.data_as(C._i64p), lk, 1,
                                     1 / np.sqrt(d), acc_o.data_ptr(), acc_l.data_ptr(), None))
    out = acc_o.bfloat16()
    dout = to_dev(R).bfloat16()
    res = []
    for split in (True, False):
        if split:
            monkeypatch.delenv("SPATTN_BWD_NO_SPLIT", raising=False)
        else:
            monkeypatch.setenv("SPATTN_BWD_NO_SPLIT", "1")
        dq = torch.zeros(1, lq, H, d, device="cuda")
        dk = torch.zeros(1, lk, Hkv, d, device="cuda")
        dv = torch.zeros(1, lk, Hkv, d, device="cuda")
        C.check(C.lib().spattn_block_bwd(s, 1, H, Hkv, d, qt.data_ptr(), qpos.ctypes.data_as(C._i64p), lq,
                                         kt.data_ptr(), vt.data_ptr(), kpos.ctypes.data_as(C._i64p), lk, 1,
                                         1 / np.sqrt(d), out.data_ptr(), acc_l.data_ptr(), dout.data_ptr(),
                                         dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), None))
        torch.cuda.synchronize()
        res.append([x.double().cpu().numpy() for x in (dq, dk, dv)])
    for a, b, name in zip(res[0], res[1], ("dq", "dk", "dv")):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-5 * max(1.0, np.abs(b).max()), err_msg=name)
    # against torch fp32 on the same bf16 inputs (full attention of the block)
    qf, kf, vf = (torch.from_numpy(x).float().cuda().requires_grad_(True) for x in (q, k, v))
    rep = H // Hkv
    sc = torch.einsum("blhd,bmhd->bhlm", qf, kf.repeat_interleave(rep, 2)) / d ** 0.5
    o = torch.einsum("bhlm,bmhd->blhd", sc.softmax(-1), vf.repeat_interleave(rep, 2))
    o.backward(dout.float())
    for got, want, name in zip(res[0], (qf.grad, kf.grad, vf.grad), ("dq", "dk", "dv")):
        w = want.double().cpu().numpy()
        assert np.abs(got - w).max() <= 2e-2 * max(1.0, np.abs(w).max()), name


def test_flop_counters_match_reference_pairs(P):
    # the reference charges 4d fwd + 10d bwd per admitted pair (attention.cpp:113, :215)
    L, H, d = 256, 4, 64
    q, k, v, R = parity_inputs(9, L, H, H, d)
    for engine, sp in [("ulysses", 2), ("ring", 4)]:
        fab = P.Fabric(sp)
        qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
        out = P.engine_attention(engine, qt, kt, vt, sp, fabric=fab)
        out.float().sum().backward()
        total = sum(fab.flops(r) for r in range(sp))
        assert total == 14 * d * H * L * (L + 1) // 2


def test_native_bytes_closed_form(P):
    # measured per-rank bytes == the native (bf16, GQA-native) closed forms in DESIGN.md
    L, H, Hkv, d, sp = 256, 8, 4, 64, 4
    got = P.measure_engine_bytes("ulysses", L, H, Hkv, d, sp)
    X = L // sp
    # fwd q,k,v a2a + out a2a + lse a2a (fp32, 1 col/head); bwd dout a2a, dq, dk, dv reverse
    q_cols, kv_cols = H * d // sp, Hkv * d // sp
    per_peer = X * (4 * q_cols * 2 + 4 * kv_cols * 2 + (H // sp) * 4)
    assert got == (sp - 1) * per_peer
    got_r = P.measure_engine_bytes("ring", L, H, Hkv, d, sp)
    Xkv = X * Hkv * d
    # fwd: sp-1 k|v hops; bwd: sp-1 k|v hops (the home-coming k|v hop is skipped) and sp dk|dv
    # (fp32) hops, the last one bringing each rank's block home
    assert got_r == (sp - 1) * 2 * Xkv * 2 + (sp - 1) * 2 * Xkv * 2 + sp * 2 * Xkv * 4


@pytest.mark.parametrize("L,H,Hkv,d,groups", [(256, 8, 4, 128, 0), (256, 8, 4, 64, 2),
                                              (192, 4, 2, 128, 1), (320, 8, 8, 64, 4),
                                              (1000, 8, 2, 128, 1), (1000, 8, 2, 128, 2),
                                              (640, 4, 4, 64, 4)])
def test_host_step_matches_oracle(P, L, H, Hkv, d, groups):
    """spattn_step_host: host buffers in, host gradients out, copies pipelined over kv-head
    groups — the same math as the device path (the first and last groups run cut along the
    sequence: run_single_step_chunked)."""
    P.set_kernel_family("tcgen05")
    q, k, v, R = parity_inputs(500 + L + groups, L, H, Hkv, d)
    cpu = lambda x: torch.from_numpy(x).to(torch.bfloat16)  # noqa: E731
    dq, dk, dv, out, lse = P.attention_step_host("oracle", cpu(q), cpu(k), cpu(v), cpu(R),
                                                 groups=groups, want_out=True)
    res = {"out": np_(out), "lse": np_(lse), "dq": np_(dq), "dk": np_(dk), "dv": np_(dv)}
    check_all(res, oracle_all(q, k, v, R), torch_ref(q, k, v, R))


def test_host_step_ulysses_loopback_rejects_bad_groups(P):
    q = torch.zeros(1, 64, 6, 64, dtype=torch.bfloat16)
    k = torch.zeros(1, 64, 3, 64, dtype=torch.bfloat16)
    with pytest.raises(P.ConfigError):
        P.attention_step_host("oracle", q, k, k, q, groups=4)


@pytest.mark.parametrize("engine,sp,H,Hkv", [("ulysses", 2, 8, 4), ("dummy_head", 4, 6, 2),
                                             ("ring", 2, 4, 2)])
@pytest.mark.parametrize("messages", [False, True])
def test_host_step_sharded_on_loopback_ranks(P, engine, sp, H, Hkv, messages):
    """spattn_step_host on every rank of a loopback group (one thread per rank): the kv-head
    group split must respect each engine's head constraints and still match the oracle. With
    ``messages`` every exchange goes through send/recv messages paired in NCCL's order (the path
    an NCCL rank takes: no peer pointers)."""
    import threading
    import types

    P.set_kernel_family("tcgen05")
    L, d = 256, 64
    q, k, v, R = parity_inputs(700 + sp + H, L, H, Hkv, d)
    mode = "zigzag" if engine == "ring" else "naive"
    fab = P.Fabric(sp, force_messages=messages)
    shard = lambda x, i: P.shard_rows(to_dev(x), mode, sp, i).cpu()  # noqa: E731
    res, errs = [None] * sp, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            rc = types.SimpleNamespace(sp=sp, _h=fab.ctxs[r])
            res[r] = P.attention_step_host(engine, shard(q, r), shard(k, r), shard(v, r),
                                           shard(R, r), rank_ctx=rc, seq_len=L, want_out=True)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(sp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    gather = lambda i: P.gather_rows([res[r][i].cuda() for r in range(sp)], mode, sp)  # noqa: E731
    got = {"dq": np_(gather(0)), "dk": np_(gather(1)), "dv": np_(gather(2)), "out": np_(gather(3))}
    orc, ref = oracle_all(q, k, v, R), torch_ref(q, k, v, R)
    check_all(got, orc, ref, keys=("out", "dq", "dk", "dv"))
