"""The per-rank multi-GPU path on the GPU box: torch.distributed (NCCL) carries the 128-byte
NCCL id, libspattn builds its own NCCL communicator (RankContext), and the autograd module
SequenceParallelAttention runs spattn_fwd/spattn_bwd on the caller's stream. World size 1 here
(one GPU per gpurun call); checked against the loopback engine and the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from gpu_util import np_, oracle_all, parity_inputs, to_dev, torch_ref, assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("engine", ["ulysses", "ring", "dummy_head", "oracle"])
def test_rank_context_module_matches_oracle(nccl_group, engine):
    import paper_2505_22296_b200 as P

    rc = P.RankContext()
    L, H, Hkv, d = 256, 4, 2, 64
    q, k, v, R = parity_inputs(21, L, H, Hkv, d)
    layer = P.SequenceParallelAttention(engine, H, Hkv, d, L, rc)
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out = layer(qt, kt, vt)
    (out.float() * to_dev(R).float()).sum().backward()
    torch.cuda.synchronize()
    res = {"out": np_(out), "dq": np_(qt.grad), "dk": np_(kt.grad), "dv": np_(vt.grad)}
    orc, ref = oracle_all(q, k, v, R), torch_ref(q, k, v, R)
    for key in res:
        assert_close(key, res[key], orc[key], ref[key])
    stats = rc.stats()
    assert all(b == 0 for _, b in stats.values())  # sp=1: nothing crosses NVLink


def test_nccl_transport_entry_points(nccl_group):
    """Every NCCL entry point the transport binds through dlopen (CommSplit, grouped Send/Recv on
    the split and the world communicator, CommDestroy) on the real library: a self message."""
    import paper_2505_22296_b200 as P
    from paper_2505_22296_b200 import _lib as C

    rc = P.RankContext()
    for nbytes in (1, 4096, 3 << 20):
        C.check(C.lib().spattn_debug_transport_selftest(rc._h, nbytes))


@pytest.mark.parametrize("messages", [False, True])
def test_loopback_transport_self_message(messages):
    import paper_2505_22296_b200 as P
    from paper_2505_22296_b200 import _lib as C

    fab = P.Fabric(1, force_messages=messages)
    C.check(C.lib().spattn_debug_transport_selftest(fab.ctxs[0], 1 << 16))


def test_rank_module_output_dropped_before_backward(nccl_group):
    """the saved state must outlive the returned ``out`` object — autograd drops it
    before running the backward in ``layer(q, k, v).sum().backward()``."""
    import gc

    import paper_2505_22296_b200 as P

    rc = P.RankContext()
    L, H, Hkv, d = 256, 4, 2, 64
    q, k, v, R = parity_inputs(22, L, H, Hkv, d)
    layer = P.SequenceParallelAttention("ulysses", H, Hkv, d, L, rc)
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    loss = (layer(qt, kt, vt).float() * to_dev(R).float()).sum()
    gc.collect()
    loss.backward()
    torch.cuda.synchronize()
    orc, ref = oracle_all(q, k, v, R), torch_ref(q, k, v, R)
    for key, got in (("dq", qt.grad), ("dk", kt.grad), ("dv", vt.grad)):
        assert_close(key, np_(got), orc[key], ref[key])
    assert rc._pending == []


def test_rank_module_double_backward_raises(nccl_group):
    import paper_2505_22296_b200 as P

    rc = P.RankContext()
    L, H, Hkv, d = 128, 2, 2, 64
    q, k, v, _ = parity_inputs(23, L, H, Hkv, d)
    layer = P.SequenceParallelAttention("ring", H, Hkv, d, L, rc)
    qt = to_dev(q).requires_grad_(True)
    out = layer(qt, to_dev(k), to_dev(v))
    out.float().sum().backward(retain_graph=True)
    with pytest.raises(P.StateError, match="twice"):
        out.float().sum().backward()


def test_rank_module_zero_participation(nccl_group):
    """attention.cpp:311-320: a forward whose output gets no gradient still runs its backward
    (zero upstream gradient) when the rank finishes its backward pass."""
    import paper_2505_22296_b200 as P

    rc = P.RankContext()
    L, H, Hkv, d = 128, 2, 1, 64
    q, k, v, R = parity_inputs(24, L, H, Hkv, d)
    layer = P.SequenceParallelAttention("ulysses", H, Hkv, d, L, rc)
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    used = layer(qt, kt, vt)
    unused = layer(qt, kt, vt)  # noqa: F841 (never reaches the loss)
    assert len(rc._pending) == 2
    (used.float() * to_dev(R).float()).sum().backward()
    assert len(rc._pending) == 1
    dq_used = qt.grad.clone()
    layer.finish_backward()
    torch.cuda.synchronize()
    assert rc._pending == []
    assert torch.equal(qt.grad, dq_used)  # the zero gradient adds nothing
    with torch.no_grad():
        layer(qt, kt, vt)
    assert rc._pending == []  # no-grad forwards are not tracked


@pytest.mark.parametrize("engine", ["oracle", "ring"])
def test_rank_module_misaligned_inputs_raise(nccl_group, engine):
    """A q/k/v the tcgen05 kernels cannot read through TMA (base not 16-byte aligned) raises
    instead of dropping to another kernel or leaving the output unwritten."""
    import paper_2505_22296_b200 as P

    rc = P.RankContext()
    L, H, Hkv, d = 128, 2, 2, 64
    q, k, v, _ = parity_inputs(25, L, H, Hkv, d)
    base = torch.empty(q.size + 8, dtype=torch.bfloat16, device="cuda")
    qm = base[1:1 + q.size].view(q.shape)  # 2-byte offset, still contiguous
    qm.copy_(to_dev(q))
    assert qm.is_contiguous() and qm.data_ptr() % 16 == 2
    layer = P.SequenceParallelAttention(engine, H, Hkv, d, L, rc)
    with pytest.raises(P.ShapeError, match="aligned"):
        layer(qm, to_dev(k), to_dev(v))
