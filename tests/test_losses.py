"""The step after the model: per-position log-probs, exact sharded sums and
the grad-aware vs plain reductions (reference losses.cpp, exact_sum.cpp, comm.cpp:464-524).

* CPU: the oracle against fixtures of the unmodified reference (tests/golden/reference_loss.json,
  `oracle/_ref/ref_driver loss`, the reference's own test inputs); the library's ExactSum
  against math.fsum; two gloo processes reproducing the paper's §5.1 pitfall (8/12 vs 4/6,
  tests/test_comm.cpp:188-218) and the bit-exact sharded SFT / DPO losses and gradients.
* GPU: the fp64 row kernels and the device exact sum against the reference values, and sharded
  SFT on loopback ranks (one Python thread per rank)."""
import json
import math
import os
import random
import socket
import threading
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import seqpar_oracle as O
import paper_2505_22296_b200 as P

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_loss.json")))
T, V = 32, 11


def _naive(n, sp, i):
    return list(range(i * n // sp, (i + 1) * n // sp))


# -------------------------------------------------------------------------------- CPU
def test_oracle_matches_reference_losses():
    lg = np.array(G["logits"]).reshape(T, V)
    pp = O.logprob_per_position(lg, G["labels"])
    assert np.max(np.abs(pp - np.array(G["per_pos"]))) < 1e-14
    # every sharding of the reference gives the same loss bit for bit, and so does the oracle
    assert len(set(G["sft_losses"])) == 1
    assert O.sft_loss(G["per_pos"], G["labels"]) == G["sft_losses"][0]
    assert len(set(G["dpo_losses"])) == 1
    assert O.dpo_loss(G["pc"], G["pr"], G["rc"], G["rr"]) == G["dpo_losses"][0]
    # plain reduction scales the shard gradients by exactly 1/sp (tests/test_losses.cpp:171-193)
    aware, plain = np.array(G["sft_grad_sp4_aware"]), np.array(G["sft_grad_sp4_plain"])
    assert np.array_equal(aware, 4.0 * plain)
    assert np.max(np.abs(aware / 4.0 - np.array(G["sft_grad_sp1"]))) < 1e-15


def test_exact_sum_is_correctly_rounded_and_order_free():
    rng = random.Random(3)
    vals = [rng.uniform(-1, 1) * 10.0 ** rng.randint(-300, 300) for _ in range(3000)]
    vals += [5e-324, -2.5e-320, 1e308, -1e308, 1.0, -1.0, 0.0, -0.0]
    want = math.fsum(vals)
    for _ in range(3):
        rng.shuffle(vals)
        assert P.exact_sum(torch.tensor(vals, dtype=torch.float64)) == want
    # merging per-shard accumulators is exact too (exact_sum_all_reduce's merge)
    parts = [torch.tensor(vals[i::7], dtype=torch.float64) for i in range(7)]
    acc = P.losses._limbs()
    for p in parts:
        import ctypes  # noqa: F401

        from paper_2505_22296_b200 import _lib as C
        C.check(C.lib().spattn_exact_merge(acc, P.exact_sum_limbs(p)))
    assert P.exact_round(acc) == want
    # cancellation to exactly zero and a subnormal result
    assert P.exact_sum(torch.tensor([1e300, 3.0, -1e300, -3.0], dtype=torch.float64)) == 0.0
    assert P.exact_sum(torch.tensor([1e-310, -0.5e-310], dtype=torch.float64)) == math.fsum([1e-310, -0.5e-310])


def test_reduce_mode_validation():
    with pytest.raises(P.ConfigError):
        P.logprob_sum_allreduce(None, torch.zeros(2, dtype=torch.float64), "sum")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _toy(rank, world):
    # tests/test_comm.cpp:188-218: loss = 2*reduce(w*x) - 1, w = 1, x = 2 or 3
    for grad_aware, want in ((True, (8.0, 12.0)), (False, (4.0, 6.0))):
        w = torch.tensor([1.0], dtype=torch.float64, requires_grad=True)
        x = torch.tensor([2.0 if rank == 0 else 3.0], dtype=torch.float64)
        red = (P.all_reduce_grad_aware if grad_aware else P.all_reduce_plain)(dist.group.WORLD, w * x)
        loss = red * 2.0 - 1.0
        loss.sum().backward()
        assert loss.item() == 9.0
        assert w.grad.item() == want[rank], (grad_aware, w.grad.item())


def _sharded_losses(rank, world):
    grp = dist.group.WORLD
    # SFT from the reference's per-position values: exact sum -> loss equal to every reference
    # sharding bit for bit; d loss / d per_pos = -1/N (grad-aware sums the upstream over ranks)
    mine = _naive(T, world, rank)
    per_pos = torch.tensor([G["per_pos"][i] for i in mine], dtype=torch.float64, requires_grad=True)
    n_local = sum(1 for i in mine if G["labels"][i] != P.IGNORE_LABEL)
    n = P.all_reduce_count(grp, n_local)
    loss = P.logprob_sum_allreduce(grp, per_pos, "grad_aware") * (-1.0 / n)
    assert loss.item() == G["sft_losses"][0]
    loss.backward()
    assert torch.all(per_pos.grad == world * (-1.0 / n))
    # DPO (tests/test_losses.cpp:224-266): sharded == single device exactly, gradients too
    idx = _naive(24, world, rank)
    pick = lambda k, rg=False: torch.tensor([G[k][i] for i in idx], dtype=torch.float64,  # noqa: E731
                                            requires_grad=rg)
    pc, pr, rc, rr = pick("pc", True), pick("pr", True), pick("rc"), pick("rr")
    loss, sums = P.dpo_loss_sharded(grp, pc, pr, rc, rr, return_sums=True)
    assert loss.item() == G["dpo_losses"][0]
    loss.backward()
    assert np.max(np.abs(pc.grad.numpy() - np.array([G["dpo_grad_pc_sp2"][i] for i in idx]))) < 1e-15
    wrong = P.wrong_order_dpo_loss(grp, pick("pc"), pick("pr"), rc, rr)
    assert abs(wrong.item() - G["dpo_wrong_sp2"][0]) < 1e-12
    assert abs(wrong.item() - G["dpo_losses"][0]) > 1e-3


def _worker(rank, world, port, kind, errq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        {"toy": _toy, "sharded": _sharded_losses}[kind](rank, world)
        dist.barrier()
    except Exception:  # noqa: BLE001
        errq.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["toy", "sharded"])
def test_two_process_loss_reductions(kind):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(f"rank {r}:\n{tb}" for r, tb in errs)
    assert all(p.exitcode == 0 for p in procs)


# ---------------------------------------------------------------------------------- GPU
def _logits(dtype=torch.float64):
    return torch.tensor(G["logits"], dtype=torch.float64).reshape(T, V).to("cuda", dtype)


@pytest.mark.gpu
def test_gpu_logprob_kernels_match_reference():
    lg = _logits().requires_grad_(True)
    pp = P.sequence_logprob_per_position(lg, G["labels"])
    assert np.max(np.abs(pp.detach().cpu().numpy() - np.array(G["per_pos"]))) < 1e-14
    # single-device SFT through the kernels: loss and logits gradient of the reference
    fab = P.Fabric(1)
    loss = P.sft_loss_sharded((fab, 0), lg, G["labels"])
    assert abs(loss.item() - G["sft_losses"][0]) <= 4e-16 * abs(G["sft_losses"][0])
    loss.backward()
    assert np.max(np.abs(lg.grad.cpu().numpy().ravel() - np.array(G["sft_grad_sp1"]))) < 1e-15
    # bf16 / fp32 logits: same rows rounded, within the input rounding
    for dt, tol in ((torch.float32, 1e-6), (torch.bfloat16, 2e-2)):
        pp2 = P.sequence_logprob_per_position(_logits(dt), G["labels"])
        assert np.max(np.abs(pp2.cpu().numpy() - np.array(G["per_pos"]))) < tol


@pytest.mark.gpu
def test_gpu_exact_sum_matches_host():
    g = torch.Generator().manual_seed(5)
    x = (torch.rand(100000, generator=g, dtype=torch.float64) - 0.5) * torch.pow(
        10.0, torch.randint(-200, 200, (100000,), generator=g).double())
    assert P.exact_sum(x.cuda()) == P.exact_sum(x) == math.fsum(x.tolist())


@pytest.mark.gpu
@pytest.mark.parametrize("bad", [math.inf, -math.inf, math.nan])
def test_gpu_exact_sum_rejects_non_finite_like_host(bad):
    # ExactSum::add throws 'ExactSum requires finite values' (exact_sum.cpp); the device kernel
    # must not fold an exponent-0x7ff value in as a finite fixed-point chunk
    x = torch.tensor([1.0, 2.0, bad, 3.0], dtype=torch.float64)
    with pytest.raises(ValueError, match="finite"):
        P.exact_sum(x)
    with pytest.raises(ValueError, match="finite"):
        P.exact_sum(x.cuda())


def _run_ranks(sp, fn):
    fab = P.Fabric(sp)
    res, errs = [None] * sp, []

    def body(r):
        try:
            res[r] = fn(fab, r)
        except Exception:  # noqa: BLE001
            errs.append(traceback.format_exc())

    th = [threading.Thread(target=body, args=(r,)) for r in range(sp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs[0]
    return res, fab


@pytest.mark.gpu
@pytest.mark.parametrize("sp,mode", [(2, "grad_aware"), (4, "grad_aware"), (4, "plain")])
def test_gpu_sharded_sft_on_loopback_ranks(sp, mode):
    full = _logits()

    def rank(fab, r):
        torch.cuda.set_device(0)
        rows = _naive(T, sp, r)
        lg = full[rows].clone().requires_grad_(True)
        loss = P.sft_loss_sharded((fab, r), lg, [G["labels"][i] for i in rows], mode)
        loss.backward()
        torch.cuda.synchronize()
        return loss.item(), lg.grad.cpu().numpy()

    res, fab = _run_ranks(sp, rank)
    single, _ = _run_ranks(1, lambda f, r: P.sft_loss_sharded((f, r), full, G["labels"]).item())
    assert all(r[0] == single[0] for r in res)  # bit-exact for every sharding
    assert abs(single[0] - G["sft_losses"][0]) <= 4e-16 * abs(G["sft_losses"][0])
    grad = np.concatenate([r[1] for r in res]).ravel()
    want = np.array(G["sft_grad_sp4_aware" if mode == "grad_aware" else "sft_grad_sp4_plain"])
    if sp == 2:
        want = np.array(G["sft_grad_sp1"]) * 2.0
    assert np.max(np.abs(grad - want)) < 1e-15
    # the loss reduction is one 8-byte all-reduce (+ the count), as the reference counts it
    assert fab.stats(0)["all_reduce"][0] >= 2
