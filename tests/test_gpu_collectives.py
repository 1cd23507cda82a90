"""The reference's public collectives beyond all_to_all (comm.hpp:131-140) through the C ABI:
all_gather (+ its reduce-scatter backward) and ring_shift, on loopback ranks (one Python thread
per rank, peer reads and NCCL-style messages) against the reference's own known answers
(tests/test_comm.cpp:110-172) and byte counters."""
import threading

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2505_22296_b200 as P

    return P


def on_ranks(fab, fn):
    res, errs = [None] * fab.world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            res[r] = fn(r)
            torch.cuda.current_stream().synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(fab.world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert not errs, errs
    return res


@pytest.mark.parametrize("messages", [False, True])
def test_all_gather_example_volume_and_order(P, messages):
    # tests/test_comm.cpp:110-125
    fab = P.Fabric(2, force_messages=messages)
    outs = on_ranks(fab, lambda r: P.all_gather((fab, r), torch.full((16,), float(r), dtype=torch.float64,
                                                                      device="cuda"), 0).cpu())
    for o in outs:
        assert o.shape == (32,) and o[0].item() == 0.0 and o[16].item() == 1.0
    for r in range(2):
        assert fab.stats(r)["all_gather"] == (1, 128)  # 16 * 8 * (2 - 1)


@pytest.mark.parametrize("messages", [False, True])
def test_all_gather_inner_axis_and_dtypes(P, messages):
    fab = P.Fabric(4, force_messages=messages)
    xs = [torch.randn(3, 5, 7, device="cuda").to(dt) for dt in (torch.bfloat16,) for _ in range(4)]
    outs = on_ranks(fab, lambda r: P.all_gather((fab, r), xs[r], 1))
    want = torch.cat(xs, 1)
    for o in outs:
        assert torch.equal(o, want)


@pytest.mark.parametrize("messages", [False, True])
def test_all_gather_backward_reduce_scatters(P, messages):
    # tests/test_comm.cpp:137-156: out = all_gather(x), loss = sum(out * w * (rank + 1))
    fab = P.Fabric(2, force_messages=messages)
    w = torch.tensor([1.0, 2.0, 3.0, 4.0], dtype=torch.float64, device="cuda")

    def rank(r):
        x = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")
        P.all_gather((fab, r), x, 0)
        return P.all_gather_backward((fab, r), w * (r + 1), x.shape, 0).cpu().tolist()

    grads = on_ranks(fab, rank)
    assert grads[0] == [3.0, 6.0] and grads[1] == [9.0, 12.0]
    # test_comm.cpp:154-155: the backward counts as a second all_gather at gather volume
    for r in range(2):
        assert fab.stats(r)["all_gather"] == (2, 2 * 16)
        assert fab.stats(r)["all_to_all"] == (0, 0)


def test_all_gather_autograd_single_member(P):
    fab = P.Fabric(1)
    x = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device="cuda", requires_grad=True)
    out = P.all_gather((fab, 0), x, 0)
    (out * torch.tensor([2.0, 3.0, 4.0], dtype=torch.float64, device="cuda")).sum().backward()
    assert x.grad.tolist() == [2.0, 3.0, 4.0]


@pytest.mark.parametrize("messages", [False, True])
def test_ring_shift_moves_one_hop_and_is_periodic(P, messages):
    # tests/test_comm.cpp:158-172
    fab = P.Fabric(4, force_messages=messages)

    def rank(r):
        cur = torch.tensor([float(r)], dtype=torch.float64, device="cuda")
        cur = P.ring_shift((fab, r), cur)
        first = cur.item()
        for _ in range(3):
            cur = P.ring_shift((fab, r), cur)
        return first, cur.item()

    res = on_ranks(fab, rank)
    for r, (first, back) in enumerate(res):
        assert first == float((r + 3) % 4) and back == float(r)
    assert res[2][0] == 1.0
    assert fab.stats(0)["p2p"] == (4, 4 * 8)


def test_asymmetric_failure_aborts_peers_instead_of_hanging(P):
    """tests/test_comm.cpp:290-300: one rank fails before the exchange (a null q); the others,
    already waiting in the all-to-all rendezvous, abort and the group call reports the root
    cause instead of hanging."""
    import ctypes

    from paper_2505_22296_b200 import _lib as C

    sp, L, H, d = 2, 256, 4, 64
    fab = P.Fabric(sp)
    mk = lambda h: torch.randn(1, L // sp, h, d, device="cuda").bfloat16()  # noqa: E731
    qs, ks, vs = [mk(H) for _ in range(sp)], [mk(2) for _ in range(sp)], [mk(2) for _ in range(sp)]
    outs = [torch.empty_like(x) for x in qs]
    lses = [torch.empty(1, L // sp, H, device="cuda") for _ in range(sp)]
    cfg, lay = C.make_config(H, 2, d, True), C.make_layout("naive", L, sp)
    saved = (ctypes.c_void_p * sp)()
    torch.cuda.synchronize()
    rc, err, msg = [None], [], [""]

    def call():
        try:
            rc[0] = C.lib().spattn_fabric_fwd_rope(
                fab._h, C.engine_id("ulysses"), ctypes.byref(cfg), ctypes.byref(lay), 1,
                C.ptr_array([qs[0].data_ptr(), 0]), C.ptr_array([x.data_ptr() for x in ks]),
                C.ptr_array([x.data_ptr() for x in vs]), C.ptr_array([x.data_ptr() for x in outs]),
                C.ptr_array([x.data_ptr() for x in lses]), None, 0, None, 10000.0, saved)
            msg[0] = C.lib().spattn_last_error().decode()  # thread-local: read on this thread
        except Exception as e:  # noqa: BLE001
            err.append(repr(e))

    t = threading.Thread(target=call)
    t.start()
    t.join(timeout=60)
    assert not t.is_alive(), "the group call hung"
    assert not err and rc[0] != 0
    assert msg[0] and "peer rank failed" not in msg[0], msg[0]  # the root cause, not the abort


@pytest.mark.parametrize("messages", [False, True])
def test_broadcast_replicates_the_root_payload(P, messages):
    # tests/test_comm.cpp:325-338 (root 0) and a non-zero root
    for root in (0, 2):
        fab = P.Fabric(4, force_messages=messages)
        got = on_ranks(fab, lambda r: P.broadcast_bytes((fab, r), bytes([1, 1, 0, 1]) if r == root else None,
                                                        root, 16))
        for r in range(4):
            assert got[r] == bytes([1, 1, 0, 1])
            assert fab.stats(r)["broadcast"] == (1, 4 * 3 // 4)


def test_group_of_one_is_identity_with_zero_bytes(P):
    # tests/test_comm.cpp:340-360
    fab = P.Fabric(1)
    x = torch.tensor([[1.0, 2.0], [3.0, 4.0]], dtype=torch.float64, device="cuda")
    assert torch.equal(P.all_gather((fab, 0), x, 0), x)
    assert torch.equal(P.ring_shift((fab, 0), x), x)
    assert P.broadcast_bytes((fab, 0), b"\x05\x06", 0, 8) == b"\x05\x06"
    assert all(b == 0 for _, b in fab.stats(0).values())


def test_broadcast_root_outside_group_raises(P):
    fab = P.Fabric(2, sp=1)  # two SP groups of one rank each
    with pytest.raises(ValueError):
        P.broadcast_bytes((fab, 0), b"x", 1, 8)
