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
