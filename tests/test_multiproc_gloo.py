"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic: each process is one
SP rank; the exchange steps run over torch.distributed point-to-point messages exactly as the
NCCL transport orders them, the placement comes from this library's planners (C ABI, no GPU:
layouts, head windows, problem lists) and the compute is the f64 oracle. The assembled
per-rank results must equal the single-device oracle — i.e. the plans the CUDA engines run are
correct for real multi-process execution, not only for the single-GPU loopback fabric."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(sends, rank, world):
    """sends[j] (numpy f64) goes to rank j; returns the list received from every rank."""
    shapes = [None] * world
    meta = [torch.tensor(list(s.shape) + [0] * (4 - s.ndim), dtype=torch.int64) for s in sends]
    got_meta = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
    reqs = []
    for j in range(world):
        if j == rank:
            got_meta[j] = meta[j]
            continue
        reqs.append(dist.isend(meta[j], j))
        reqs.append(dist.irecv(got_meta[j], j))
    for r in reqs:
        r.wait()
    for j in range(world):
        shapes[j] = [int(x) for x in got_meta[j].tolist() if x > 0] if j != rank else list(sends[j].shape)
    out = [None] * world
    bufs = [torch.empty(int(np.prod(shapes[j])), dtype=torch.float64) for j in range(world)]
    reqs = []
    for j in range(world):
        if j == rank:
            out[j] = sends[j].copy()
            continue
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(sends[j]).ravel()), j))
        reqs.append(dist.irecv(bufs[j], j))
    for r in reqs:
        r.wait()
    for j in range(world):
        if j != rank:
            out[j] = bufs[j].numpy().reshape(shapes[j])
    return out


def _ulysses(rank, world):
    import seqpar_oracle as O

    import paper_2505_22296_b200 as P

    L, H, Hkv, d = 32, 6, 3, 8  # rep 2: rank 0 heads 0-2 -> kv 0,1; rank 1 heads 3-5 -> kv 1,2
    q, k, v, R = O.parity_data(1000003, L, H, Hkv, d)
    full = O.attention_fwd_bwd(q, k, v, R)
    pos = [np.array(P.shard_positions("zigzag", L, world, i)) for i in range(world)]
    mine = pos[rank]
    ql, kl, vl, Rl = (x[:, mine] for x in (q, k, v, R))
    qlo, qn, kvlo, kvn = P.plan_heads(H, Hkv, world)
    rep = H // Hkv

    def seq_to_heads(x, lo, n):
        parts = _exchange([x[:, :, lo[j]:lo[j] + n[j]] for j in range(world)], rank, world)
        g = np.zeros((1, L, n[rank], d))
        for i in range(world):
            g[:, pos[i]] = parts[i]
        return g

    qg, Rg = seq_to_heads(ql, qlo, qn), seq_to_heads(Rl, qlo, qn)
    kg, vg = seq_to_heads(kl, kvlo, kvn), seq_to_heads(vl, kvlo, kvn)
    idx = [(qlo[rank] + h) // rep - kvlo[rank] for h in range(qn[rank])]
    res = O.attention_fwd_bwd(qg, kg[:, :, idx], vg[:, :, idx], Rg)
    dkw, dvw = np.zeros(kg.shape), np.zeros(vg.shape)
    for h, i in enumerate(idx):  # repeat_heads backward: sum the group (tensor.cpp:437-447)
        dkw[:, :, i] += res["dk"][:, :, h]
        dvw[:, :, i] += res["dv"][:, :, h]

    def heads_to_seq(y, lo, n, width):
        parts = _exchange([y[:, pos[i]] for i in range(world)], rank, world)
        x = np.zeros((1, len(mine), width, d))
        for j in range(world):
            x[:, :, lo[j]:lo[j] + n[j]] += parts[j]  # overlapping kv windows add up
        return x

    out = heads_to_seq(res["out"], qlo, qn, H)
    dq = heads_to_seq(res["dq"], qlo, qn, H)
    dk = heads_to_seq(dkw, kvlo, kvn, Hkv)
    dv = heads_to_seq(dvw, kvlo, kvn, Hkv)
    for name, got in (("out", out), ("dq", dq), ("dk", dk), ("dv", dv)):
        err = np.max(np.abs(got - full[name][:, mine]))
        assert err < 1e-10, (name, err)


def _ring(rank, world):
    import seqpar_oracle as O

    import paper_2505_22296_b200 as P

    L, H, Hkv, d = 48, 4, 2, 8
    q, k, v, R = O.parity_data(1000008, L, H, Hkv, d)
    full = O.attention_fwd_bwd(q, k, v, R)
    pos = [np.array(P.shard_positions("zigzag", L, world, i)) for i in range(world)]
    mine = pos[rank]
    ql, kl, vl, Rl = (x[:, mine] for x in (q, k, v, R))
    n = len(mine)
    acc = None
    nxt, prv = (rank + 1) % world, (rank - 1) % world

    def shift(bufs):
        sends = [None] * world
        for j in range(world):
            sends[j] = bufs if j == nxt else np.zeros((0,))
        got = _exchange(sends, rank, world)
        return got[prv]

    pieces_rows = []
    kv = np.concatenate([kl, vl], axis=0)  # [2, n, Hkv, d]
    pairs_total = 0
    for s in range(world):
        if s > 0:
            kv = shift(kv)
        owner = (rank - s) % world
        probs, pairs = P.plan_problems(list(mine), list(pos[owner]))
        pairs_total += pairs
        for (q0, nq, k0, nk, off, causal) in probs:
            qp = np.arange(nq, dtype=np.int64) + off
            kp = np.arange(nk, dtype=np.int64)
            num, mx, nrm, _ = O.block_forward(ql[:, q0:q0 + nq], qp, kv[:1, k0:k0 + nk],
                                              kv[1:, k0:k0 + nk], kp, bool(causal))
            pieces_rows.append((q0, nq, (num, mx, nrm)))
    # merge every piece into a full-length accumulator (merge_piece, attention.cpp:117-149)
    num = np.zeros((1, n, H, d))
    mx = np.full((1, n, H), -np.inf)
    nrm = np.zeros((1, n, H))
    for q0, nq, piece in pieces_rows:
        a = (num[:, q0:q0 + nq], mx[:, q0:q0 + nq], nrm[:, q0:q0 + nq])
        empty = np.all(np.isneginf(a[1]))
        m = O.merge_piece(None if empty else a, piece)
        num[:, q0:q0 + nq], mx[:, q0:q0 + nq], nrm[:, q0:q0 + nq] = m
    out, lse = O.finalize_piece((num, mx, nrm))
    assert np.max(np.abs(out - full["out"][:, mine])) < 1e-10
    # backward: k|v|dk|dv circulate world times (attention.cpp:308-349)
    dq = np.zeros(ql.shape)
    buf = np.concatenate([kl, vl, np.zeros(kl.shape), np.zeros(vl.shape)], axis=0)
    for s in range(world):
        owner = (rank - s) % world
        probs, _ = P.plan_problems(list(mine), list(pos[owner]))
        for (q0, nq, k0, nk, off, causal) in probs:
            qp = np.arange(nq, dtype=np.int64) + off
            kp = np.arange(nk, dtype=np.int64)
            dqs = np.zeros((1, nq, H, d))
            dks, dvs = np.zeros((1, nk, Hkv, d)), np.zeros((1, nk, Hkv, d))
            O.block_backward(ql[:, q0:q0 + nq], qp, buf[0:1, k0:k0 + nk], buf[1:2, k0:k0 + nk], kp,
                             out[:, q0:q0 + nq], lse[:, q0:q0 + nq], Rl[:, q0:q0 + nq], dqs, dks, dvs,
                             bool(causal))
            dq[:, q0:q0 + nq] += dqs
            buf[2:3, k0:k0 + nk] += dks
            buf[3:4, k0:k0 + nk] += dvs
        buf = shift(buf)
    assert np.max(np.abs(dq - full["dq"][:, mine])) < 1e-9
    assert np.max(np.abs(buf[2:3] - full["dk"][:, mine])) < 1e-9
    assert np.max(np.abs(buf[3:4] - full["dv"][:, mine])) < 1e-9
    t = torch.tensor([pairs_total], dtype=torch.int64)
    dist.all_reduce(t)
    assert t.item() == H * 0 + L * (L + 1) // 2  # per-head admitted pairs over the ring


def _worker(rank, world, port, kind, errq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        {"ulysses": _ulysses, "ring": _ring}[kind](rank, world)
        dist.barrier()
    except Exception:  # noqa: BLE001
        errq.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["ulysses", "ring"])
def test_two_process_protocol_matches_oracle(kind):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, kind, errq)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(f"rank {r}:\n{tb}" for r, tb in errs)
    assert all(p.exitcode == 0 for p in procs)
