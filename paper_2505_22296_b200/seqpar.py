"""Python surface of the B200 SP attention layer, mirroring the reference module ``_seqpar``
(/root/reference/proj/bindings/py_module.cpp:315-401): same function names and argument
meaning, ValueError subclasses for configuration/shape errors. Differences: tensors are torch
CUDA tensors (bf16 compute), and ``engine_attention`` is differentiable (the reference binding
is forward-only, py_module.cpp:111-180).

Everything here calls libspattn.so through its C ABI (``_lib``); there is no CPU path."""
from __future__ import annotations

import ctypes
import dataclasses
import weakref
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as C
from ._lib import ConfigError, PeerAbort, ShapeError, StateError  # noqa: F401

__version__ = "0.1.0"


def _i64(n=1):
    return (ctypes.c_int64 * n)()


# ----------------------------------------------------------------------- layouts and counts
def engine_names() -> list[str]:
    return list(C.ENGINES)


def shard_positions(mode: str, len: int, sp: int, index: int, ulysses_degree: int = 0,
                    ring_degree: int = 0) -> list[int]:
    """ShardLayout::positions_of (reference partition.cpp:105-111)."""
    lay = C.make_layout(mode, len, sp, ulysses_degree, ring_degree)
    n = len // sp if sp > 0 else 0
    out = _i64(max(n, 1))
    C.check(C.lib().spattn_layout_positions(ctypes.byref(lay), index, out))
    return list(out[:n])


position_ids = shard_positions  # make_position_ids (partition.cpp:160-162)


def causal_pairs(mode: str, len: int, sp: int, index: int, ulysses_degree: int = 0,
                 ring_degree: int = 0) -> int:
    lay = C.make_layout(mode, len, sp, ulysses_degree, ring_degree)
    out = _i64()
    C.check(C.lib().spattn_causal_pairs(ctypes.byref(lay), index, out))
    return out[0]


def pad_length(len: int, sp: int, cutoff_len: int, pad_to_cutoff: bool = False) -> int:
    out = _i64()
    C.check(C.lib().spattn_pad_length(len, sp, cutoff_len, int(pad_to_cutoff), out))
    return out[0]


def balanced_zigzag_layout(docs: Sequence[int], sp: int, min_chunk: int = 1024) -> str:
    """Layout string for the ring over a neat-packed sequence (extension, no reference
    counterpart): "zigzag:B" with the fewest blocks B (a power of two, L divisible by 2*sp*B,
    chunks of at least ``min_chunk`` tokens: shorter chunks cost kernel efficiency) whose busiest
    rank carries within 2 % of the least share of the causal work those B reach (each query
    attends to the earlier keys of its own document). B = 1 is the reference zigzag."""
    lens = np.asarray(list(docs), dtype=np.int64)
    L = int(lens.sum())
    if sp <= 0 or L <= 0 or (lens <= 0).any():
        raise ConfigError("balanced_zigzag_layout: documents and sp must be positive")
    start = np.concatenate([[0], np.cumsum(lens)[:-1]])
    work = np.arange(L, dtype=np.int64) - np.repeat(start, lens) + 1
    best = []
    b = 1
    while L % (2 * sp * b) == 0 and (b == 1 or L // (2 * sp * b) >= min_chunk):
        share = max(int(work[np.asarray(shard_positions(f"zigzag:{b}", L, sp, i))].sum())
                    for i in range(sp)) / int(work.sum())
        best.append((share, b))
        b *= 2
    if not best:
        raise ConfigError(f"balanced_zigzag_layout: length {L} not divisible by 2*sp = {2 * sp}")
    lo = min(x for x, _ in best)
    return f"zigzag:{min(b for x, b in best if x <= lo * 1.02)}"


def pick_xtuner_insp(heads: int, sp: int, head_dim: int) -> int:
    out = ctypes.c_int()
    C.check(C.lib().spattn_pick_xtuner_insp(heads, sp, head_dim, ctypes.byref(out)))
    return out.value


def _ref_bytes(engine, bs, len, heads, head_dim, sp, u=0, r=0):
    out = _i64()
    C.check(C.lib().spattn_reference_bytes(C.engine_id(engine), bs, len, heads, head_dim, sp, u, r,
                                           out))
    return out[0]


def ulysses_bytes(bs, len, heads, head_dim, sp):
    return _ref_bytes("ulysses", bs, len, heads, head_dim, sp)


def ring_bytes(bs, len, heads, head_dim, sp):
    return _ref_bytes("ring", bs, len, heads, head_dim, sp)


def dummy_head_bytes(bs, len, heads, head_dim, sp):
    return _ref_bytes("dummy_head", bs, len, heads, head_dim, sp)


def xtuner_bytes(bs, len, heads, head_dim, sp):
    return _ref_bytes("xtuner", bs, len, heads, head_dim, sp)


def usp_bytes(bs, len, heads, head_dim, ulysses_degree, ring_degree):
    return _ref_bytes("usp", bs, len, heads, head_dim, ulysses_degree * ring_degree,
                      ulysses_degree, ring_degree)


def plan_heads(heads: int, kv_heads: int, group: int):
    """Head windows of the Ulysses moves per group member: (q_lo, q_n, kv_lo, kv_n) lists."""
    arrs = [(ctypes.c_int32 * group)() for _ in range(4)]
    C.check(C.lib().spattn_plan_heads(heads, kv_heads, group, *arrs))
    return tuple(list(a) for a in arrs)


def plan_problems(qpos, kpos, causal: bool = True, docs=None, max_problems: int = 4096):
    """Problem list (q_row0, nq, k_row0, nk, off, causal) for two position lists, and the
    admitted pair count."""
    qp = (ctypes.c_int64 * len(qpos))(*qpos)
    kp = (ctypes.c_int64 * len(kpos))(*kpos)
    nd = 0 if docs is None else len(docs)
    darr = None if docs is None else (ctypes.c_int64 * nd)(*docs)
    out = (ctypes.c_int32 * (6 * max_problems))()
    n, pairs = ctypes.c_int(), _i64()
    C.check(C.lib().spattn_plan_problems(qp, len(qpos), kp, len(kpos), int(causal), darr, nd, out,
                                         max_problems, ctypes.byref(n), pairs))
    return [tuple(out[6 * i:6 * i + 6]) for i in range(n.value)], pairs[0]


# ------------------------------------------------ batches, padding, neat-packing metadata
IGNORE_LABEL, NO_IMAGE, NO_SEGMENT = -100, -1, -1  # kIgnoreLabel / kNoImage / kNoSegment


@dataclasses.dataclass
class TrainBatch:
    """TrainBatch (reference partition.hpp:96-105): one packed sequence."""
    tokens: list
    labels: list
    position_ids: list
    segment_ids: list = dataclasses.field(default_factory=list)
    image_map: list = dataclasses.field(default_factory=list)

    def __len__(self):
        return len(self.tokens)

    def validate(self) -> None:  # partition.cpp:164-177
        n = len(self.tokens)
        if n == 0:
            raise ConfigError("batch has no tokens")
        if len(self.labels) != n:
            raise ConfigError("batch labels length does not match tokens")
        if len(self.position_ids) != n:
            raise ConfigError("batch position_ids length does not match tokens")
        if self.segment_ids and len(self.segment_ids) != n:
            raise ConfigError("batch segment_ids length does not match tokens")
        if self.image_map and len(self.image_map) != n:
            raise ConfigError("batch image_map length does not match tokens")


def pad_batch(batch: TrainBatch, sp: int, pad_token: int, cutoff_len: int,
              pad_to_cutoff: bool = False) -> TrainBatch:
    """pad_batch (partition.cpp:202-215): every field extended to pad_length(len, sp, ...)."""
    batch.validate()
    n = len(batch)
    target = pad_length(n, sp, cutoff_len, pad_to_cutoff)
    arr = lambda xs: _i64_array(xs) if xs else None  # noqa: E731
    outs = [_i64(max(1, target)) for _ in range(5)]
    out_len = _i64()
    C.check(C.lib().spattn_pad_batch(arr(batch.tokens), arr(batch.labels), arr(batch.position_ids),
                                     arr(batch.segment_ids), arr(batch.image_map), n, sp, pad_token,
                                     cutoff_len, int(pad_to_cutoff), out_len, *outs))
    t = out_len[0]
    return TrainBatch(list(outs[0][:t]), list(outs[1][:t]), list(outs[2][:t]),
                      list(outs[3][:t]) if batch.segment_ids else [],
                      list(outs[4][:t]) if batch.image_map else [])


def split_position_map(image_map: Sequence[int], mode: str, sp: int, index: int,
                       ulysses_degree: int = 0, ring_degree: int = 0) -> list[int]:
    """split_position_map (partition.cpp:217-220): the shard's entries of a per-position map."""
    lay = C.make_layout(mode, len(image_map), sp, ulysses_degree, ring_degree)
    n = len(image_map) // sp if sp > 0 else 0
    out = _i64(max(1, n))
    C.check(C.lib().spattn_split_position_map(ctypes.byref(lay), index, _i64_array(image_map), out))
    return list(out[:n])


def documents_from_segments(segment_ids: Sequence[int]) -> list[int]:
    """Neat-packing segment ids -> document lengths for the varlen kernels (``docs=``): runs of
    equal ids are documents, a -1 padding tail is one more document."""
    n = len(segment_ids)
    out = _i64(max(1, n))
    nd = ctypes.c_int()
    C.check(C.lib().spattn_documents_from_segments(_i64_array(segment_ids), n, out, max(1, n),
                                                   ctypes.byref(nd)))
    return list(out[:nd.value])


def document_position_ids(doc_lens: Sequence[int]) -> list[int]:
    """Per-document reset position ids (rope ids of a neat-packed sequence)."""
    ids = []
    for n in doc_lens:
        if n <= 0:
            raise ConfigError("documents: lengths must be positive")
        ids.extend(range(n))
    return ids


def set_kernel_family(name: str) -> None:
    """'tcgen05' (default where supported), 'mma', 'tcgen05_pp' (two-tile forward) or
    'tcgen05_pair' (CTA-pair cta_group::2 forward, d=128), 'tcgen05_q64' (the 64-query-tile
    backward for d=128 too; the default runs the 128-query-tile backward there)."""
    C.check(C.lib().spattn_set_kernel_family(
        {"tcgen05": 0, "mma": 1, "tcgen05_pp": 2, "tcgen05_pair": 3, "tcgen05_q64": 4}[name]))


def kernel_family() -> str:
    return ["tcgen05", "mma", "tcgen05_pp", "tcgen05_pair", "tcgen05_q64"][C.lib().spattn_get_kernel_family()]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# -------------------------------------------------------------------- row (re)distribution
def _layout_for(mode: str, engine: str, length: int, sp: int, u: int, r: int):
    if mode == "auto":  # py_module.cpp:39-47
        mode = "zigzag" if engine == "ring" else "usp" if engine == "usp" else "naive"
    return mode, C.make_layout(mode, length, sp, u, r)


def shard_rows(x: torch.Tensor, mode: str, sp: int, index: int, ulysses_degree: int = 0,
               ring_degree: int = 0) -> torch.Tensor:
    """shard_rows (partition.cpp:124-139) on a CUDA tensor [L, ...] or [bs, L, ...] (dim 1 is the
    sequence when x.dim() >= 3). Byte-exact for any dtype."""
    seq_dim = 0 if x.dim() <= 2 else 1
    L = x.shape[seq_dim]
    lay = C.make_layout(mode, L, sp, ulysses_degree, ring_degree)
    x = x.contiguous()
    bs = 1 if seq_dim == 0 else x.shape[0]
    row = x[0].numel() * x.element_size() if seq_dim == 0 else x[0, 0].numel() * x.element_size()
    shape = list(x.shape)
    shape[seq_dim] = L // sp
    out = torch.empty(shape, dtype=x.dtype, device=x.device)
    C.check(C.lib().spattn_shard_rows(_stream(), ctypes.byref(lay), index, bs, row, x.data_ptr(),
                                      out.data_ptr()))
    return out


def gather_rows(shards: Sequence[torch.Tensor], mode: str, sp: int, ulysses_degree: int = 0,
                ring_degree: int = 0) -> torch.Tensor:
    """gather_rows (partition.cpp:141-158): inverse of shard_rows."""
    if len(shards) != sp:
        raise ShapeError(f"gather: got {len(shards)} shards for sp {sp}")
    x0 = shards[0]
    seq_dim = 0 if x0.dim() <= 2 else 1
    L = x0.shape[seq_dim] * sp
    lay = C.make_layout(mode, L, sp, ulysses_degree, ring_degree)
    shape = list(x0.shape)
    shape[seq_dim] = L
    out = torch.empty(shape, dtype=x0.dtype, device=x0.device)
    bs = 1 if seq_dim == 0 else x0.shape[0]
    row = x0[0].numel() * x0.element_size() if seq_dim == 0 else x0[0, 0].numel() * x0.element_size()
    for i, s in enumerate(shards):
        s = s.contiguous()
        C.check(C.lib().spattn_gather_rows(_stream(), ctypes.byref(lay), i, bs, row, s.data_ptr(),
                                           out.data_ptr()))
    return out


# ---------------------------------------------------------------------------------- fabric
class Fabric:
    """Loopback CommFabric: ``world`` ranks as host threads sharing the current CUDA device
    (comm.hpp:86-140). ``force_messages`` routes collectives through pack -> send/recv ->
    unpack, the NCCL code path."""

    def __init__(self, world: int, sp: Optional[int] = None, device: Optional[int] = None,
                 force_messages: bool = False):
        self.world = world
        self.sp = sp or world
        dev = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        C.check(C.lib().spattn_fabric_create(dev, world, self.sp, int(force_messages),
                                             ctypes.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, C.lib().spattn_fabric_destroy, h)
        self.ctxs = []
        for r in range(world):
            c = ctypes.c_void_p()
            C.check(C.lib().spattn_fabric_ctx(h, r, ctypes.byref(c)))
            self.ctxs.append(c)

    def stats(self, rank: int) -> dict:
        out = {}
        for i, name in enumerate(C.PRIMITIVES):
            calls, nbytes = _i64(), _i64()
            C.check(C.lib().spattn_ctx_stats(self.ctxs[rank], i, calls, nbytes))
            out[name] = (calls[0], nbytes[0])
        return out

    def replicate_packing_mask(self, masks: Sequence[Optional[bytes]]) -> list[bytes]:
        """replicate_packing_mask (partition.cpp:222-227) on every rank: rank 0's bytes
        everywhere (counted as one broadcast)."""
        cap = max([len(m) for m in masks if m] + [1])
        bufs = [ctypes.create_string_buffer(m or b"", max(1, len(m or b""))) for m in masks]
        outs = [ctypes.create_string_buffer(cap) for _ in masks]
        lens = _i64_array([len(m or b"") for m in masks])
        out_lens = _i64(len(masks))
        C.check(C.lib().spattn_fabric_replicate_packing_mask(
            self._h, C.ptr_array([ctypes.addressof(b) for b in bufs]), lens,
            C.ptr_array([ctypes.addressof(o) for o in outs]), cap, out_lens))
        return [o.raw[:out_lens[i]] for i, o in enumerate(outs)]

    def total_bytes(self, rank: int) -> int:
        return sum(b for _, b in self.stats(rank).values())

    def flops(self, rank: int) -> int:
        f = _i64()
        C.check(C.lib().spattn_ctx_flops(self.ctxs[rank], f))
        return f[0]

    def reset_stats(self) -> None:
        for c in self.ctxs:
            C.check(C.lib().spattn_ctx_reset_stats(c))

    def all_to_all(self, locals_: Sequence[torch.Tensor], scatter_dim: int,
                   gather_dim: int) -> list[torch.Tensor]:
        """all_to_all (comm.cpp:357-379) of 4-D [bs, len, heads, dim] tensors, any dtype."""
        x0 = locals_[0]
        bs, L, H, D = x0.shape
        g = self.sp
        if scatter_dim == 2 and gather_dim == 1:
            shape = (bs, L * g, H // g if H % g == 0 else 0, D)
        elif scatter_dim == 1 and gather_dim == 2:
            shape = (bs, L // g if L % g == 0 else 0, H * g, D)
        else:
            raise ConfigError("all_to_all: unsupported dims")
        outs = [torch.empty(shape, dtype=x0.dtype, device=x0.device) for _ in locals_]
        torch.cuda.current_stream().synchronize()
        ins = [x.contiguous() for x in locals_]
        C.check(C.lib().spattn_fabric_all_to_all(
            self._h, C.ptr_array([x.data_ptr() for x in ins]),
            C.ptr_array([o.data_ptr() for o in outs]), bs, L, H, D, x0.element_size(),
            scatter_dim, gather_dim))
        return outs


class _Keep:
    """Per-rank shards the saved forward state points into (weak-referenceable holder)."""

    def __init__(self, *tensors):
        self.tensors = tensors


def _free_saved(handles):
    for h in handles:
        if h:
            C.lib().spattn_saved_free(h)


ROPE_BASE = 10000.0  # kRopeBase (reference tensor.hpp:141-144)


def _i64_array(xs):
    xs = [int(x) for x in xs]
    return (ctypes.c_int64 * max(1, len(xs)))(*xs)


class _Rope(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, pos, base):
        out = torch.empty_like(x)
        C.check(C.lib().spattn_rope_apply(_stream(), x.shape[0], x.shape[1], x.shape[2], x.shape[3],
                                          x.data_ptr(), pos, base, 0, out.data_ptr()))
        ctx.pos, ctx.base = pos, base
        return out

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        dx = torch.empty_like(g)
        C.check(C.lib().spattn_rope_apply(_stream(), g.shape[0], g.shape[1], g.shape[2], g.shape[3],
                                          g.data_ptr(), ctx.pos, ctx.base, 1, dx.data_ptr()))
        return dx, None, None


def rope_apply(x: torch.Tensor, position_ids: Sequence[int], base: float = ROPE_BASE):
    """rope_apply (reference tensor.cpp:548-607) on a bf16 CUDA tensor [bs, L, heads, dim] with
    one position id per sequence row; differentiable (the backward is the inverse rotation)."""
    if x.dim() != 4:
        raise ShapeError(f"rope_apply expects [bs, L, heads, dim], got {list(x.shape)}")
    if not x.is_cuda or x.dtype != torch.bfloat16:
        raise ShapeError("rope_apply: x must be a bf16 CUDA tensor")
    if len(position_ids) != x.shape[1]:
        raise ShapeError(f"position_ids length {len(position_ids)} does not match sequence "
                         f"extent {x.shape[1]}")
    return _Rope.apply(x.contiguous(), _i64_array(position_ids), float(base))


class _FabricEngine(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, fab, engine, cfg, lay, mode, u, r, docs, want_lse, pos=None):
        sp = fab.sp
        qs = [shard_rows(q, mode, sp, i, u, r) for i in range(sp)]
        ks = [shard_rows(k, mode, sp, i, u, r) for i in range(sp)]
        vs = [shard_rows(v, mode, sp, i, u, r) for i in range(sp)]
        outs = [torch.empty_like(x) for x in qs]
        lses = [torch.empty(x.shape[:3], dtype=torch.float32, device=x.device) for x in qs]
        torch.cuda.current_stream().synchronize()
        saved = (ctypes.c_void_p * sp)()
        nd = 0 if docs is None else len(docs)
        darr = None if docs is None else (ctypes.c_int64 * nd)(*docs)
        if pos is not None:  # each rank rotates with the global ids of its own rows
            lay_pos = [shard_positions(mode, q.shape[1], sp, i, u, r) for i in range(sp)]
            parts = [_i64_array([pos[p] for p in lp]) for lp in lay_pos]
            parr = (ctypes.POINTER(ctypes.c_int64) * sp)(
                *[ctypes.cast(a, ctypes.POINTER(ctypes.c_int64)) for a in parts])
        else:
            parr = None
        C.check(C.lib().spattn_fabric_fwd_rope(
            fab._h, C.engine_id(engine), ctypes.byref(cfg), ctypes.byref(lay), q.shape[0],
            C.ptr_array([x.data_ptr() for x in qs]), C.ptr_array([x.data_ptr() for x in ks]),
            C.ptr_array([x.data_ptr() for x in vs]), C.ptr_array([x.data_ptr() for x in outs]),
            C.ptr_array([x.data_ptr() for x in lses]), darr, nd, parr, ROPE_BASE, saved))
        handles = [saved[i] for i in range(sp)]
        ctx.fab, ctx.mode, ctx.u, ctx.r = fab, mode, u, r
        ctx.handles = handles
        ctx.keep = _Keep(qs, ks, vs, outs, lses)
        ctx.fin = weakref.finalize(ctx.keep, _free_saved, handles)
        out = gather_rows(outs, mode, sp, u, r)
        lse = gather_rows(lses, mode, sp, u, r) if want_lse else None
        ctx.mark_non_differentiable(*([lse] if lse is not None else []))
        return out, lse

    @staticmethod
    def backward(ctx, dout, _dlse):
        fab, mode, u, r = ctx.fab, ctx.mode, ctx.u, ctx.r
        sp = fab.sp
        if not ctx.fin.alive:
            raise StateError("engine_attention: backward ran twice over one forward; its saved "
                             "state was released by the first (retain_graph is not supported)")
        qs, ks, vs = ctx.keep.tensors[:3]
        dos = [shard_rows(dout.contiguous(), mode, sp, i, u, r) for i in range(sp)]
        dqs = [torch.empty_like(x) for x in qs]
        dks = [torch.empty_like(x) for x in ks]
        dvs = [torch.empty_like(x) for x in vs]
        torch.cuda.current_stream().synchronize()
        C.check(C.lib().spattn_fabric_bwd(
            fab._h, C.ptr_array(ctx.handles), C.ptr_array([x.data_ptr() for x in dos]),
            C.ptr_array([x.data_ptr() for x in dqs]), C.ptr_array([x.data_ptr() for x in dks]),
            C.ptr_array([x.data_ptr() for x in dvs])))
        ctx.fin()
        dq = gather_rows(dqs, mode, sp, u, r)
        dk = gather_rows(dks, mode, sp, u, r)
        dv = gather_rows(dvs, mode, sp, u, r)
        return dq, dk, dv, None, None, None, None, None, None, None, None, None, None


def engine_attention(engine: str, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, sp: int,
                     layout: str = "auto", causal: bool = True, ulysses_degree: int = 0,
                     ring_degree: int = 0, docs: Optional[Sequence[int]] = None,
                     fabric: Optional[Fabric] = None, force_messages: bool = False,
                     return_lse: bool = False, position_ids: Optional[Sequence[int]] = None):
    """Sharded attention across ``sp`` loopback ranks on the current GPU, gathered back to the
    full sequence (py_module.cpp:111-180), differentiable. q [bs, L, H, d] and k/v
    [bs, L, Hkv, d] are bf16 CUDA tensors; ``docs`` are neat-packed document lengths.
    ``position_ids`` (one global id per sequence row) applies rope_apply to q and k first, as
    Model::forward does (model.cpp:342-343) — fused into the all-to-all copy for Ulysses,
    Dummy-Head and USP; the gradients are those of the unrotated q and k."""
    for t in (q, k, v):
        if not t.is_cuda or t.dtype != torch.bfloat16:
            raise ShapeError("engine_attention: q, k, v must be bf16 CUDA tensors")
    bs, L, H, d = q.shape
    Hkv = k.shape[2]
    mode, lay = _layout_for(layout, engine, L, sp, ulysses_degree, ring_degree)
    cfg = C.make_config(H, Hkv, d, causal, ulysses_degree, ring_degree)
    fab = fabric or Fabric(sp, force_messages=force_messages)
    if fab.sp != sp:
        raise ConfigError("fabric sp does not match")
    if position_ids is not None and len(position_ids) != L:
        raise ShapeError(f"position_ids length {len(position_ids)} for {L} tokens")
    out, lse = _FabricEngine.apply(q.contiguous(), k.contiguous(), v.contiguous(), fab, engine,
                                   cfg, lay, mode, ulysses_degree, ring_degree,
                                   None if docs is None else list(docs), return_lse,
                                   None if position_ids is None else list(position_ids))
    return (out, lse) if return_lse else out


def oracle_attention(q, k, v, causal: bool = True, docs=None, return_lse: bool = False):
    """Single-device attention (oracle engine, attention.cpp:218-260) on the GPU kernels."""
    return engine_attention("oracle", q, k, v, 1, "naive", causal, docs=docs,
                            return_lse=return_lse)


def measure_engine_bytes(engine: str, len: int, heads: int, kv_heads: int, head_dim: int,
                         sp: int, ulysses_degree: int = 0, ring_degree: int = 0, seed: int = 1,
                         force_messages: bool = False) -> int:
    """Per-rank bytes this implementation moves for one fwd+bwd (report.cpp:977-991), bf16
    payloads and native GQA (the reference counts f64 and expanded KV); all ranks must agree."""
    fab = Fabric(sp, force_messages=force_messages)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.rand(1, len, heads, head_dim, device="cuda", generator=g).bfloat16() * 2 - 1
    k = torch.rand(1, len, kv_heads, head_dim, device="cuda", generator=g).bfloat16() * 2 - 1
    v = torch.rand(1, len, kv_heads, head_dim, device="cuda", generator=g).bfloat16() * 2 - 1
    q.requires_grad_(True)
    out = engine_attention(engine, q, k.requires_grad_(), v.requires_grad_(), sp,
                           ulysses_degree=ulysses_degree, ring_degree=ring_degree, fabric=fab)
    out.sum().backward()
    totals = [fab.total_bytes(r) for r in range(sp)]
    if len_set(totals) != 1:
        raise StateError(f"per-rank byte totals differ: {totals}")
    return totals[0]


def len_set(xs):
    return len(set(xs))


# ------------------------------------------------------------------- multi-GPU (NCCL) path
class RankContext:
    """One GPU's RankCtx over NCCL (one process per GPU). Built collectively from an existing
    torch.distributed process group, which only carries the 128-byte NCCL id."""

    def __init__(self, sp: Optional[int] = None):
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        self.sp = sp or world
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            C.check(C.lib().spattn_nccl_unique_id(buf))
            uid = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
        if dist.get_backend() == "nccl":
            uid = uid.cuda()
        dist.broadcast(uid, 0)
        raw = bytes(uid.cpu().tolist())
        h = ctypes.c_void_p()
        C.check(C.lib().spattn_ctx_create_nccl(torch.cuda.current_device(), rank, world, self.sp,
                                               raw, ctypes.byref(h)))
        self._h = h
        self.rank, self.world = rank, world
        self._pending = []  # _RankSaved of forwards whose backward has not run yet
        self._fin = weakref.finalize(self, C.lib().spattn_ctx_destroy, h)

    def finish_backward(self):
        """Zero participation (reference attention.cpp:311-320, comm.cpp:366-370): every forward
        of this rank whose output received no gradient — autograd never reaches its node when
        the output is unused — runs its backward with a zero upstream gradient, in forward
        order, so the peers' collectives complete; the gradients the peers send back still flow
        into q / k / v. Call it on every rank after ``loss.backward()`` (a no-op when every
        output was used)."""
        for e in list(self._pending):
            q, k, v = e.tensors[:3]
            grads = e.backward(torch.zeros_like(e.tensors[3]))
            pairs = [(t, g) for t, g in zip((q, k, v), grads) if t.requires_grad]
            if pairs:
                torch.autograd.backward([t for t, _ in pairs], [g for _, g in pairs])

    def replicate_packing_mask(self, mask: Optional[bytes], max_len: int) -> bytes:
        """replicate_packing_mask (partition.cpp:222-227) over NCCL: group index 0 supplies
        the mask, every rank returns it; ``max_len`` bounds the result buffer."""
        m = mask or b""
        buf = ctypes.create_string_buffer(m, max(1, len(m)))
        out = ctypes.create_string_buffer(max(1, max_len))
        n = _i64()
        C.check(C.lib().spattn_replicate_packing_mask(self._h, buf, len(m), out, max_len, n))
        return out.raw[:n[0]]

    def stats(self) -> dict:
        out = {}
        for i, name in enumerate(C.PRIMITIVES):
            calls, nbytes = _i64(), _i64()
            C.check(C.lib().spattn_ctx_stats(self._h, i, calls, nbytes))
            out[name] = (calls[0], nbytes[0])
        return out


def _rank_of(group):
    """(context handle, group size, index in the group) of a RankContext or a (Fabric, rank)."""
    if isinstance(group, RankContext):
        return group._h, group.sp, group.rank % group.sp
    if isinstance(group, tuple) and len(group) == 2 and isinstance(group[0], Fabric):
        fab, r = group
        return fab.ctxs[r], fab.sp, r % fab.sp
    raise ConfigError("expected a RankContext or a (Fabric, rank) pair")


def _around(x: torch.Tensor, dim: int):
    """x viewed as [outer, extent, inner_bytes] around axis `dim`."""
    outer = 1
    for n in x.shape[:dim]:
        outer *= n
    inner = x.element_size()
    for n in x.shape[dim + 1:]:
        inner *= n
    return outer, x.shape[dim], inner


def _tree_sum(parts):
    """tree_sum_into (comm.cpp:325-337): balanced pairwise sum in group order."""
    if len(parts) == 1:
        return parts[0]
    mid = len(parts) // 2
    return _tree_sum(parts[:mid]) + _tree_sum(parts[mid:])


class _AllGather(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, h, G, idx, dim):
        x = x.contiguous()
        outer, extent, inner = _around(x, dim)
        shape = list(x.shape)
        shape[dim] *= G
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
        C.check(C.lib().spattn_ctx_set_stream(h, _stream()))
        C.check(C.lib().spattn_all_gather(h, x.data_ptr(), out.data_ptr(), outer, extent, inner))
        ctx.meta = (h, G, dim, outer, extent, tuple(x.shape))
        return out

    @staticmethod
    def backward(ctx, gy):
        h, G, dim, outer, extent, xshape = ctx.meta
        return _reduce_scatter(h, G, gy, outer, extent).reshape(xshape), None, None, None, None


def _reduce_scatter(h, G, gy, outer, extent):
    """The all_gather backward (comm.cpp:415-443): one exchange hands every member its block of
    each member's gathered gradient, tree-summed in group order; counted as a second
    all_gather at gather volume (comm.cpp:418-420)."""
    gy = gy.contiguous()
    inner = gy.numel() * gy.element_size() // max(1, outer * G * extent)  # bytes after the axis
    buf = torch.empty((G, outer, extent, inner // gy.element_size()), dtype=gy.dtype,
                      device=gy.device)
    C.check(C.lib().spattn_ctx_set_stream(h, _stream()))
    C.check(C.lib().spattn_all_gather_backward(h, gy.data_ptr(), buf.data_ptr(), outer, extent,
                                               inner))
    return _tree_sum(list(buf.unbind(0)))


def all_gather_backward(group, grad_out: torch.Tensor, local_shape, dim: int) -> torch.Tensor:
    """Gradient of all_gather w.r.t. this member's input (what autograd calls; exposed for
    callers that drive backward themselves, e.g. one Python thread per loopback rank)."""
    h, G, idx = _rank_of(group)
    dim = dim % len(local_shape)
    outer = 1
    for n in local_shape[:dim]:
        outer *= n
    return _reduce_scatter(h, G, grad_out, outer, local_shape[dim]).reshape(local_shape)


def all_gather(group, x: torch.Tensor, dim: int):
    """all_gather (comm.hpp:136, comm.cpp:381-447) over the group of ``group`` (a RankContext
    or a (Fabric, rank) pair): members' tensors concatenated along ``dim`` in group order;
    differentiable (the backward reduce-scatters). Every member must call it."""
    h, G, idx = _rank_of(group)
    dim = dim % x.dim()
    return _AllGather.apply(x, h, G, idx, dim)


def ring_shift(group, payload: torch.Tensor) -> torch.Tensor:
    """ring_shift (comm.hpp:140, comm.cpp:449-460): group index i returns the payload of index
    i-1 (same shape and dtype on every member). Every member must call it."""
    h, G, idx = _rank_of(group)
    payload = payload.contiguous()
    out = torch.empty_like(payload)
    C.check(C.lib().spattn_ctx_set_stream(h, _stream()))
    C.check(C.lib().spattn_ring_shift(h, payload.data_ptr(), out.data_ptr(),
                                      payload.numel() * payload.element_size()))
    return out


def broadcast_bytes(group, payload: Optional[bytes], root: int, max_len: int) -> bytes:
    """broadcast_bytes (comm.hpp:159-161): the bytes of global rank ``root`` on every member of
    the group of ``group`` (a RankContext or a (Fabric, rank) pair); ``max_len`` bounds the
    result. Every member must call it."""
    h, _, _ = _rank_of(group)
    m = payload or b""
    buf = ctypes.create_string_buffer(m, max(1, len(m)))
    out = ctypes.create_string_buffer(max(1, max_len))
    n = _i64()
    C.check(C.lib().spattn_broadcast_bytes(h, buf, len(m), root, out, max_len, n))
    return out.raw[:n[0]]


def attention_step_host(engine: str, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                        dout: torch.Tensor, rank_ctx: Optional["RankContext"] = None,
                        seq_len: Optional[int] = None, layout: str = "auto", causal: bool = True,
                        ulysses_degree: int = 0, ring_degree: int = 0,
                        docs: Optional[Sequence[int]] = None, groups: int = 0,
                        want_out: bool = False):
    """One fwd+bwd step of the layer on HOST (CPU, ideally pinned) bf16 tensors of this rank's
    shard — run_attention_engine + the tape backward as the reference runs them on host
    tensors — with the H2D/D2H copies pipelined against the kernels over kv-head groups
    (spattn_step_host). Returns (dq, dk, dv) or (dq, dk, dv, out, lse) CPU tensors."""
    for t in (q, k, v, dout):
        if t.is_cuda or t.dtype != torch.bfloat16:
            raise ShapeError("attention_step_host: q, k, v, dout must be bf16 CPU tensors")
    bs, lloc, H, d = q.shape
    Hkv = k.shape[2]
    sp = rank_ctx.sp if rank_ctx is not None else 1
    mode, lay = _layout_for(layout, engine, seq_len or lloc * sp, sp, ulysses_degree, ring_degree)
    cfg = C.make_config(H, Hkv, d, causal, ulysses_degree, ring_degree)
    if rank_ctx is None:
        fab = Fabric(1)
        h = fab.ctxs[0]
    else:
        fab, h = None, rank_ctx._h
    C.check(C.lib().spattn_ctx_set_stream(h, _stream()))
    pin = lambda t: t.contiguous() if t.is_pinned() else t.contiguous().pin_memory()  # noqa: E731
    q, k, v, dout = (pin(t) for t in (q, k, v, dout))
    # results land in pinned buffers (torch's caching host allocator reuses them across steps)
    dq, dk, dv = (torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (q, k, v))
    out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True) if want_out else None
    lse = torch.empty(q.shape[:3], dtype=torch.float32, pin_memory=True) if want_out else None
    nd = 0 if docs is None else len(docs)
    darr = None if docs is None else (ctypes.c_int64 * nd)(*docs)
    C.check(C.lib().spattn_step_host(
        h, C.engine_id(engine), ctypes.byref(cfg), ctypes.byref(lay), bs, q.data_ptr(),
        k.data_ptr(), v.data_ptr(), dout.data_ptr(), out.data_ptr() if want_out else None,
        lse.data_ptr() if want_out else None, dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), darr, nd,
        groups))
    torch.cuda.current_stream().synchronize()
    del fab
    return (dq, dk, dv, out, lse) if want_out else (dq, dk, dv)


class _RankSaved:
    """One _RankEngine forward's library state (spattn_saved) and the tensors it points into.
    The handle is freed by the backward that consumes it, or when this holder is collected —
    never by the lifetime of the returned ``out`` object, which autograd may drop before it runs
    the backward."""

    def __init__(self, rc, h, q, k, v, out, lse):
        self.rc, self.h = rc, h
        self.tensors = (q, k, v, out, lse)
        self.done = False
        self._fin = weakref.finalize(self, C.lib().spattn_saved_free, h)

    def backward(self, dout):
        if self.done:
            raise StateError("SequenceParallelAttention: backward ran twice over one forward; its "
                             "saved state was released by the first (retain_graph is not "
                             "supported)")
        q, k, v = self.tensors[:3]
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        C.check(C.lib().spattn_ctx_set_stream(self.rc._h, _stream()))
        C.check(C.lib().spattn_bwd(self.rc._h, self.h, dout.contiguous().data_ptr(), dq.data_ptr(),
                                   dk.data_ptr(), dv.data_ptr()))
        self.done = True
        self.rc._pending = [e for e in self.rc._pending if e is not self]
        self.tensors = None
        self._fin()  # the state's buffers are not needed any more
        return dq, dk, dv


class _RankEngine(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, rc, engine, cfg, lay, docs, pos=None, track=False):
        out = torch.empty_like(q)
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
        C.check(C.lib().spattn_ctx_set_stream(rc._h, _stream()))
        saved = ctypes.c_void_p()
        nd = 0 if docs is None else len(docs)
        darr = None if docs is None else (ctypes.c_int64 * nd)(*docs)
        parr = None if pos is None else _i64_array(pos)
        C.check(C.lib().spattn_fwd_rope(rc._h, C.engine_id(engine), ctypes.byref(cfg),
                                        ctypes.byref(lay), q.shape[0], q.data_ptr(), k.data_ptr(),
                                        v.data_ptr(), out.data_ptr(), lse.data_ptr(), darr, nd,
                                        parr, ROPE_BASE, ctypes.byref(saved)))
        # the autograd ctx owns the holder (and so the handle); the rank context lists it until
        # a backward consumes it, so finish_backward() can make an unused output take part
        ctx.entry = _RankSaved(rc, saved, q, k, v, out, lse)
        if track:
            rc._pending.append(ctx.entry)
        return out

    @staticmethod
    def backward(ctx, dout):
        dq, dk, dv = ctx.entry.backward(dout)
        return dq, dk, dv, None, None, None, None, None, None, None


class SequenceParallelAttention(torch.nn.Module):
    """Per-rank SP attention layer (run_attention_engine, attention.hpp:90-92) over NCCL:
    every rank of the SP group calls it with its sequence shard."""

    def __init__(self, engine: str, heads: int, kv_heads: int, head_dim: int, seq_len: int,
                 rank_ctx: RankContext, layout: str = "auto", causal: bool = True,
                 ulysses_degree: int = 0, ring_degree: int = 0):
        super().__init__()
        self.engine = engine
        self.rc = rank_ctx
        self.mode, self.lay = _layout_for(layout, engine, seq_len, rank_ctx.sp, ulysses_degree,
                                          ring_degree)
        self.cfg = C.make_config(heads, kv_heads, head_dim, causal, ulysses_degree, ring_degree)

    def forward(self, q, k, v, docs: Optional[Sequence[int]] = None,
                position_ids: Optional[Sequence[int]] = None):
        """``position_ids``: the GLOBAL ids of this rank's rows; when given q and k are rotated
        (rope_apply) before attention — a local 0-based range would corrupt the rotary phases
        (reference model.cpp:313-318)."""
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        track = torch.is_grad_enabled() and any(t.requires_grad for t in (q, k, v))
        return _RankEngine.apply(q, k, v, self.rc, self.engine, self.cfg, self.lay,
                                 None if docs is None else list(docs),
                                 None if position_ids is None else list(position_ids), track)

    def finish_backward(self):
        """See RankContext.finish_backward."""
        self.rc.finish_backward()
