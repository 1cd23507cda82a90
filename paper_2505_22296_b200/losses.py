"""The step after the SP layer: per-position log-probs and the sharded losses whose backward
crosses ranks (reference proj/src/losses.cpp, exact_sum.cpp, comm.cpp:464-524; the paper's
§5.1 gradient pitfall).

* ``sequence_logprob_per_position`` runs the fp64 row kernels of ``libspattn.so`` on CUDA logits.
* Sums are exact (``ExactSum``: 2240-bit fixed point, rounded once), so a sharded loss equals
  the single-device loss bit for bit under any sharding.
* ``grad_aware`` reductions all-reduce the upstream gradient in backward (each rank's
  replicated loss consumed the group sum); ``plain`` passes it through, which scales every
  gradient by 1/sp once the trainer averages (the reference's ``ReduceMode``).

A *group* is a :class:`RankContext` (NCCL, one process per GPU), a ``(Fabric, rank)`` pair
(loopback ranks on one GPU, one Python thread per rank) or a ``torch.distributed`` process group
(e.g. gloo on CPU); every rank of the group makes the same calls in the same order."""
from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib as C
from ._lib import ConfigError, ShapeError

IGNORE_LABEL = -100
KLIMBS = 35
DPO_BETA_DEFAULT = 0.1  # kDpoBetaDefault (losses.hpp)
REDUCE_MODES = ("grad_aware", "plain")
_DTYPES = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2}


def _limbs(t=None):
    a = (ctypes.c_uint64 * KLIMBS)()
    if t is not None:
        for i, x in enumerate(t):
            a[i] = x
    return a


def _check_mode(mode):
    if mode not in REDUCE_MODES:  # reduce_mode_from_string (losses.cpp:15-19)
        raise ConfigError(f"unknown reduce mode '{mode}'")


# -------------------------------------------------------------------------------- groups
class _SpattnGroup:
    def __init__(self, handle, size):
        self.h, self.size = handle, size

    def exact_all_reduce(self, limbs):
        C.check(C.lib().spattn_exact_sum_all_reduce(self.h, limbs))
        return limbs

    def values(self, vals):
        arr = (ctypes.c_double * max(1, len(vals)))(*vals)
        C.check(C.lib().spattn_all_reduce_values(self.h, arr, len(vals)))
        return list(arr[:len(vals)])

    def count(self, n):
        v = ctypes.c_int64(n)
        C.check(C.lib().spattn_all_reduce_count(self.h, ctypes.byref(v)))
        return v.value


class _TorchGroup:
    def __init__(self, pg):
        import torch.distributed as dist

        self.dist, self.pg = dist, pg
        self.size = dist.get_world_size(pg)

    def _gather(self, t):
        dev = "cuda" if self.dist.get_backend(self.pg) == "nccl" else "cpu"
        t = t.to(dev)
        out = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.pg)
        return [o.cpu() for o in out]

    def exact_all_reduce(self, limbs):
        mine = torch.tensor([int(x) - (1 << 64) if int(x) >= (1 << 63) else int(x) for x in limbs],
                            dtype=torch.int64)
        acc = _limbs()
        for part in self._gather(mine):
            other = _limbs([int(x) & (2 ** 64 - 1) for x in part.tolist()])
            C.check(C.lib().spattn_exact_merge(acc, other))
        return acc

    def values(self, vals):
        parts = [p.tolist() for p in self._gather(torch.tensor(vals, dtype=torch.float64))]

        def tree(lo, hi):  # tree_sum_into (comm.cpp:323-337)
            if hi - lo == 1:
                return parts[lo]
            mid = lo + (hi - lo) // 2
            a, b = tree(lo, mid), tree(mid, hi)
            return [x + y for x, y in zip(a, b)]

        return tree(0, self.size)

    def count(self, n):
        return int(sum(int(p.item()) for p in self._gather(torch.tensor(n, dtype=torch.int64))))


def _group(group):
    from .seqpar import Fabric, RankContext

    if isinstance(group, RankContext):
        return _SpattnGroup(group._h, group.sp)
    if isinstance(group, tuple) and len(group) == 2 and isinstance(group[0], Fabric):
        fab, rank = group
        return _SpattnGroup(fab.ctxs[rank], fab.sp)
    if isinstance(group, (_SpattnGroup, _TorchGroup)):
        return group
    return _TorchGroup(group)


# ------------------------------------------------------------------------------- sums
def exact_sum_limbs(x: torch.Tensor):
    """ExactSum accumulator (35 uint64 limbs) of every element of a float64 tensor: the device
    kernel for CUDA tensors, host integer arithmetic for CPU tensors."""
    x = x.detach().contiguous().to(torch.float64).reshape(-1)
    acc = _limbs()
    if x.is_cuda:
        C.check(C.lib().spattn_exact_sum_device(torch.cuda.current_stream().cuda_stream,
                                                x.data_ptr(), x.numel(), acc))
    else:
        C.check(C.lib().spattn_exact_sum_host(x.data_ptr(), x.numel(), acc))
    return acc


def exact_round(limbs) -> float:
    out = ctypes.c_double()
    C.check(C.lib().spattn_exact_round(limbs, ctypes.byref(out)))
    return out.value


def exact_sum(x: torch.Tensor) -> float:
    """The exactly rounded sum of a float64 tensor (order-independent)."""
    return exact_round(exact_sum_limbs(x))


# --------------------------------------------------------------------------- log-probs
class _LogProb(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, labels):
        T, V = logits.shape
        out = torch.empty(T, dtype=torch.float64, device=logits.device)
        lse = torch.empty(T, dtype=torch.float64, device=logits.device)
        s = torch.cuda.current_stream().cuda_stream
        C.check(C.lib().spattn_logprob_fwd(s, logits.data_ptr(), _DTYPES[logits.dtype],
                                           T, V, labels.data_ptr(), out.data_ptr(), lse.data_ptr()))
        ctx.save_for_backward(logits, labels, lse)
        return out

    @staticmethod
    def backward(ctx, g):
        logits, labels, lse = ctx.saved_tensors
        T, V = logits.shape
        g = g.contiguous().to(torch.float64)
        d = torch.empty_like(logits)
        C.check(C.lib().spattn_logprob_bwd(torch.cuda.current_stream().cuda_stream,
                                           logits.data_ptr(), _DTYPES[logits.dtype],
                                           T, V, labels.data_ptr(), lse.data_ptr(), g.data_ptr(),
                                           d.data_ptr(), 0))
        return d, None


def sequence_logprob_per_position(logits: torch.Tensor, labels) -> torch.Tensor:
    """log softmax(logits)[t, label_t] in fp64 (losses.cpp:20-72); ignored labels give 0 and no
    gradient. logits: CUDA [T, V] float32, bfloat16 or float64."""
    if logits.dim() != 2:
        raise ShapeError("sequence_logprob: logits must be [T, V]")
    if not logits.is_cuda or logits.dtype not in _DTYPES:
        raise ShapeError("sequence_logprob: logits must be a float32/bfloat16/float64 CUDA tensor")
    labels = torch.as_tensor(labels, dtype=torch.int64).reshape(-1)
    T, V = logits.shape
    if labels.numel() != T:
        raise ShapeError(f"sequence_logprob: labels length {labels.numel()} does not match T {T}")
    bad = (labels != IGNORE_LABEL) & ((labels < 0) | (labels >= V))
    if bool(bad.any()):
        lab = int(labels[bad][0])
        raise ConfigError(f"sequence_logprob: label {lab} outside vocab of {V}")
    return _LogProb.apply(logits.contiguous(), labels.to(logits.device).contiguous())


def supervised_count(labels) -> int:
    labels = torch.as_tensor(labels)
    return int((labels != IGNORE_LABEL).sum())


# ----------------------------------------------------------------- cross-rank reductions
class _LogprobSum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, per_pos, grp, mode):
        total = exact_round(grp.exact_all_reduce(exact_sum_limbs(per_pos)))
        ctx.grp, ctx.mode, ctx.shape, ctx.device = grp, mode, per_pos.shape, per_pos.device
        # a host scalar, like the reference's loss: its backward (and the grad-aware
        # all-reduce in it) then runs on the calling thread, not on a shared device worker
        return torch.tensor(total, dtype=torch.float64)

    @staticmethod
    def backward(ctx, g):
        up = float(g)
        if ctx.mode == "grad_aware":  # losses.cpp:93-97
            up = ctx.grp.values([up])[0]
        return torch.full(ctx.shape, up, dtype=torch.float64, device=ctx.device), None, None


def logprob_sum_allreduce(group, per_pos: torch.Tensor, mode: str = "grad_aware") -> torch.Tensor:
    """logprob_sum_allreduce (losses.cpp:80-102): the exact group sum of every element, one
    8-byte all-reduce; backward adds the (grad-aware: group-summed) upstream to every element.
    Returns a 0-d float64 CPU tensor (the reference's host scalar)."""
    _check_mode(mode)
    return _LogprobSum.apply(per_pos, _group(group), mode)


class _AllReduce(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, grp, grad_aware):
        ctx.grp, ctx.grad_aware = grp, grad_aware
        out = grp.values(x.detach().to(torch.float64).reshape(-1).tolist())
        return torch.tensor(out, dtype=torch.float64, device=x.device).reshape(x.shape)

    @staticmethod
    def backward(ctx, g):
        if not ctx.grad_aware:
            return g, None, None
        red = ctx.grp.values(g.detach().to(torch.float64).reshape(-1).tolist())
        return torch.tensor(red, dtype=torch.float64, device=g.device).reshape(g.shape), None, None


def all_reduce_grad_aware(group, x: torch.Tensor) -> torch.Tensor:
    """all_reduce_grad_aware (comm.cpp:464-487): sum over the group; backward all-reduces the
    upstream gradient too."""
    return _AllReduce.apply(x, _group(group), True)


def all_reduce_plain(group, x: torch.Tensor) -> torch.Tensor:
    """all_reduce_plain: sum over the group; backward passes the gradient through (the §5.1
    pitfall: gradients come out 1/sp too small)."""
    return _AllReduce.apply(x, _group(group), False)


def all_reduce_count(group, n: int) -> int:
    return _group(group).count(int(n))


def sft_loss_sharded(group, logits: torch.Tensor, labels, mode: str = "grad_aware",
                     per_rank_mean: bool = False) -> torch.Tensor:
    """sft_loss_sharded (losses.cpp:104-119): -sum(logp) / N_global over the group's supervised
    positions (bit-identical to the single-device loss), or the mean of per-rank means."""
    _check_mode(mode)
    grp = _group(group)
    per_pos = sequence_logprob_per_position(logits, labels)
    local_n = supervised_count(labels)
    global_n = grp.count(local_n)
    if global_n == 0:
        raise ConfigError("sft loss: no supervised positions in the group")
    if per_rank_mean:
        inv = 1.0 / local_n if local_n > 0 else 0.0
        total = logprob_sum_allreduce(grp, per_pos * inv, mode)
        return total * (-1.0 / grp.size)
    return logprob_sum_allreduce(grp, per_pos, mode) * (-1.0 / global_n)


def _softplus(x):  # tensor.cpp:211-227
    return torch.log1p(torch.exp(-x.abs())) + x.clamp(min=0.0)


def dpo_loss_sharded(group, policy_chosen, policy_rejected, ref_chosen, ref_rejected,
                     beta: float = DPO_BETA_DEFAULT, return_sums: bool = False):
    """dpo_loss_sharded (losses.cpp:121-135): softplus(-beta * margin) with the margin built
    from exact group sums of the four per-position streams; policy sums reduce grad-aware."""
    grp = _group(group)
    pc = logprob_sum_allreduce(grp, policy_chosen, "grad_aware")
    pr = logprob_sum_allreduce(grp, policy_rejected, "grad_aware")
    rc = logprob_sum_allreduce(grp, ref_chosen, "plain")
    rr = logprob_sum_allreduce(grp, ref_rejected, "plain")
    loss = _softplus(((pc - pr) - (rc - rr)) * (-beta))
    if return_sums:
        return loss, tuple(float(x) for x in (pc, pr, rc, rr))
    return loss


def wrong_order_dpo_loss(group, policy_chosen, policy_rejected, ref_chosen, ref_rejected,
                         beta: float = DPO_BETA_DEFAULT):
    """The order-of-operations mistake (losses.cpp:137-147): the nonlinearity on each shard's
    local margin, averaged after — differs from dpo_loss_sharded whenever sp > 1."""
    grp = _group(group)
    margin = (policy_chosen.sum() - policy_rejected.sum()) - (ref_chosen.sum() - ref_rejected.sum())
    local = _softplus(margin * (-beta))
    return all_reduce_grad_aware(grp, local.reshape(1)).reshape(()) * (1.0 / grp.size)


__all__ = ["sequence_logprob_per_position", "supervised_count", "exact_sum", "exact_sum_limbs",
           "exact_round", "logprob_sum_allreduce", "all_reduce_grad_aware", "all_reduce_plain",
           "all_reduce_count", "sft_loss_sharded", "dpo_loss_sharded", "wrong_order_dpo_loss",
           "REDUCE_MODES", "DPO_BETA_DEFAULT"]


def _seq(xs: Sequence[float]):  # pragma: no cover - helper for interactive use
    return torch.tensor(list(xs), dtype=torch.float64)
