"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the sequence-parallel attention hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference legs may
import this module, and only as the checker: the product (``paper_2505_22296_b200``) never
imports anything under ``oracle/``.

Two halves:
  * f64 attention block math — plain C in ``oracle.c`` (``liboracle.so``), restating
    ``/root/reference/proj/src/attention.cpp:61-216``;
  * integer / permutation work — numpy restatements of ``partition.cpp``, ``comm.cpp`` and the
    ``tensor.cpp`` shape ops, each citing the line it follows.

Pinned against the reference itself: ``tests/golden/make_golden.py`` runs the unmodified
reference (``oracle/_ref``, compiled from /root/reference by ``oracle/Makefile``) and
``tests/test_oracle_golden.py`` checks this module against those fixtures.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


class ConfigError(ValueError):
    """Mirrors seqpar::ConfigError (tensor.hpp:24), surfaced as ValueError (py_module.cpp:320)."""


class ShapeError(ValueError):
    """Mirrors seqpar::ShapeError (tensor.hpp:18)."""


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)
        _LIB = ctypes.CDLL(path)
        _LIB.orc_rng_next.restype = ctypes.c_uint64
        _LIB.orc_rng_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        _LIB.orc_rng_fill_uniform.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_double,
                                              ctypes.c_double, _dp, ctypes.c_int64]
        fwd_args = [ctypes.c_int64] * 4 + [_dp, _ip, _ip, ctypes.c_int64, _dp, _dp, _ip, _ip,
                                           ctypes.c_int64, ctypes.c_int, ctypes.c_double]
        _LIB.orc_attn_block_forward.restype = ctypes.c_int64
        _LIB.orc_attn_block_forward.argtypes = fwd_args + [_dp, _dp, _dp]
        _LIB.orc_attn_block_backward.restype = ctypes.c_int64
        _LIB.orc_attn_block_backward.argtypes = fwd_args + [_dp, _dp, _dp, _dp, _dp, _dp]
        _LIB.orc_merge_piece.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _dp, _dp,
                                         _dp, _dp, _dp, _dp]
        _LIB.orc_finalize_piece.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, _dp, _dp, _dp,
                                            _dp]
    return _LIB


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _i(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


# ----------------------------------------------------------------------------- rng


class Rng:
    """splitmix64 + uniform_range, bit-exact with seqpar::Rng (tensor.cpp:724-739)."""

    def __init__(self, seed: int):
        self.state = ctypes.c_uint64(seed if seed else 0x9E3779B97F4A7C15)

    def next_u64(self) -> int:
        return int(lib().orc_rng_next(ctypes.byref(self.state)))

    def uniform_range(self, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        lib().orc_rng_fill_uniform(ctypes.byref(self.state), lo, hi, _d(out), n)
        return out

    def uniform_int(self, lo: int, hi: int) -> int:
        """tensor.cpp:757-761"""
        span = hi - lo + 1
        return lo + self.next_u64() % span


def parity_data(seed: int, L: int, heads: int, kv: int, dim: int, bs: int = 1):
    """q, k, v, R drawn in that order, uniform(-2, 2) (report.cpp:42-54)."""
    rng = Rng(seed)
    q = rng.uniform_range(-2, 2, bs * L * heads * dim).reshape(bs, L, heads, dim)
    k = rng.uniform_range(-2, 2, bs * L * kv * dim).reshape(bs, L, kv, dim)
    v = rng.uniform_range(-2, 2, bs * L * kv * dim).reshape(bs, L, kv, dim)
    R = rng.uniform_range(-2, 2, bs * L * heads * dim).reshape(bs, L, heads, dim)
    return q, k, v, R


# ----------------------------------------------------------------------------- layouts


def _check_divisible(length: int, sp: int, what: str):
    """partition.cpp:28-35"""
    if sp <= 0:
        raise ConfigError("sp must be positive")
    if length <= 0:
        raise ConfigError("sequence length must be positive")
    if length % sp:
        raise ConfigError(f"{what}: length {length} not divisible by sp {sp}")


def layout_owned(mode: str, length: int, sp: int, u: int = 0, r: int = 0) -> list[np.ndarray]:
    """ShardLayout::make_naive / make_zigzag / make_usp (partition.cpp:37-103)."""
    if mode == "naive":
        _check_divisible(length, sp, "naive split")
        local = length // sp
        return [np.arange(i * local, (i + 1) * local, dtype=np.int64) for i in range(sp)]
    if mode == "zigzag":
        _check_divisible(length, sp, "zigzag split")
        if length % (2 * sp):
            raise ConfigError(f"zigzag split: length {length} not divisible by 2*sp = {2 * sp}")
        chunk = length // (2 * sp)
        return [np.concatenate([np.arange(c * chunk, (c + 1) * chunk, dtype=np.int64)
                                for c in (i, 2 * sp - 1 - i)]) for i in range(sp)]
    if mode.startswith("zigzag:"):
        # extension with no reference counterpart (the repo's make_zigzag_blocks): zigzag within
        # each of B equal blocks; B = 1 is the reference zigzag above
        blocks = int(mode.split(":", 1)[1])
        if blocks <= 0:
            raise ConfigError("zigzag blocks: block count must be positive")
        if blocks == 1:
            return layout_owned("zigzag", length, sp)
        _check_divisible(length, sp, "zigzag split")
        if length % (2 * sp * blocks):
            raise ConfigError(f"zigzag blocks: length {length} not divisible by 2*sp*blocks = "
                              f"{2 * sp * blocks}")
        chunk, bl = length // (2 * sp * blocks), length // blocks
        return [np.concatenate([np.arange(b * bl + c * chunk, b * bl + (c + 1) * chunk, dtype=np.int64)
                                for b in range(blocks) for c in (i, 2 * sp - 1 - i)])
                for i in range(sp)]
    if mode == "usp":
        if u <= 0 or r <= 0:
            raise ConfigError("usp split: degrees must be positive")
        outer = layout_owned("zigzag", length, r)
        block = length // r
        if block % u:
            raise ConfigError(f"usp split: ring block {block} not divisible by ulysses degree {u}")
        local = block // u
        return [outer[rho][iota * local:(iota + 1) * local]
                for rho in range(r) for iota in range(u)]
    raise ConfigError(f"unknown split mode '{mode}'")


def causal_pair_count(owned: np.ndarray) -> int:
    """partition.cpp:118-122"""
    return int(np.sum(owned + 1))


def pad_length(length: int, sp: int, cutoff_len: int, pad_to_cutoff: bool = False) -> int:
    """partition.cpp:179-200"""
    if length <= 0:
        raise ConfigError("pad_length: length must be positive")
    if sp <= 0:
        raise ConfigError("pad_length: sp must be positive")
    quantum = 8 * sp
    if pad_to_cutoff:
        if cutoff_len % quantum:
            raise ConfigError(f"cutoff_len {cutoff_len} is not a multiple of 8*sp = {quantum}")
        if length > cutoff_len:
            raise ConfigError(f"sequence of length {length} exceeds cutoff_len {cutoff_len}")
        return cutoff_len
    padded = (length + quantum - 1) // quantum * quantum
    if padded > cutoff_len:
        raise ConfigError(f"padded length {padded} exceeds cutoff_len {cutoff_len}")
    return padded


def pick_xtuner_insp(heads: int, sp: int, head_dim: int) -> int:
    """attention.cpp:354-366"""
    if heads <= 0 or sp <= 0 or head_dim <= 0:
        raise ConfigError("xtuner: heads, sp, and head_dim must be positive")
    base = sp // math.gcd(heads, sp)
    insp = base
    while insp <= head_dim:
        if head_dim % insp == 0 and sp % insp == 0:
            return insp
        insp += base
    raise ConfigError(f"xtuner: no virtual-head factor for heads={heads}, sp={sp}, "
                      f"head_dim={head_dim}")


# ----------------------------------------------------------------------------- byte models
# report.cpp:906-941, f64 payloads (8 bytes per element), per rank, fwd + bwd.


def ulysses_bytes(bs, L, heads, head_dim, sp):
    local = bs * (L // sp) * heads * head_dim * 8
    return 8 * (local * (sp - 1) // sp)


def ring_bytes(bs, L, heads, head_dim, sp):
    local = bs * (L // sp) * heads * head_dim * 8
    return (6 * sp - 2) * local


def dummy_head_bytes(bs, L, heads, head_dim, sp):
    padded = (heads + sp - 1) // sp * sp
    return ulysses_bytes(bs, L, padded, head_dim, sp)


def xtuner_bytes(bs, L, heads, head_dim, sp):
    insp = pick_xtuner_insp(heads, sp, head_dim)
    local = bs * (L // sp) * heads * head_dim * 8
    return 8 * (local * (sp - 1) // sp) + 6 * local * (insp - 1)


def usp_bytes(bs, L, heads, head_dim, u, r):
    sp = u * r
    padded = (heads + u - 1) // u * u if u > 1 else heads
    local = bs * (L // sp) * padded * head_dim * 8
    total = 0
    if u > 1:
        total += 8 * (local * (u - 1) // u)
    if r > 1:
        total += (6 * r - 2) * local
    return total


# ----------------------------------------------------------------------------- permutations


def shard_rows(full: np.ndarray, owned: np.ndarray) -> np.ndarray:
    """shard_rows (partition.cpp:124-139) on [bs, L, ...]: rows at the owned positions."""
    return np.ascontiguousarray(full[:, owned])


def gather_rows(shards: Sequence[np.ndarray], owned: Sequence[np.ndarray], length: int):
    """gather_rows (partition.cpp:141-158) on [bs, l, ...] shards."""
    first = shards[0]
    out = np.empty((first.shape[0], length) + first.shape[2:], dtype=first.dtype)
    for s, pos in zip(shards, owned):
        out[:, pos] = s
    return out


def all_to_all(deposits: Sequence[np.ndarray], idx: int, scatter_dim: int, gather_dim: int):
    """all_to_all_values (comm.cpp:278-321): rank idx takes slice idx of scatter_dim from every
    peer j and places it at j*piece along gather_dim, in source-rank order (:314-319)."""
    g = len(deposits)
    shape = deposits[0].shape
    if shape[scatter_dim] % g:
        raise ShapeError(f"all_to_all: extent {shape[scatter_dim]} of axis {scatter_dim} not "
                         f"divisible by group size {g}")
    piece = shape[scatter_dim] // g
    parts = [np.take(d, np.arange(idx * piece, (idx + 1) * piece), axis=scatter_dim)
             for d in deposits]
    return np.concatenate(parts, axis=gather_dim)


def pad_axis_zeros(a: np.ndarray, axis: int, pad_after: int) -> np.ndarray:
    """tensor.cpp:390-416 (zeros appended after the axis' existing entries)"""
    if pad_after == 0:
        return a
    widths = [(0, 0)] * a.ndim
    widths[axis] = (0, pad_after)
    return np.pad(a, widths)


def slice_axis(a: np.ndarray, axis: int, start: int, length: int) -> np.ndarray:
    """tensor.cpp:360-388"""
    return np.ascontiguousarray(np.take(a, np.arange(start, start + length), axis=axis))


def repeat_heads(a: np.ndarray, rep: int) -> np.ndarray:
    """tensor.cpp:418-450: out head h reads input head h / rep."""
    return np.repeat(a, rep, axis=2)


def ring_shift(payloads: Sequence[np.ndarray]) -> list[np.ndarray]:
    """comm.cpp:449-460: index i receives the payload of index i-1."""
    g = len(payloads)
    return [payloads[(i - 1 + g) % g] for i in range(g)]


# ----------------------------------------------------------------------------- attention


def block_forward(q, qpos, k, v, kpos, causal=True, scale=None, qseg=None, kseg=None):
    """attn_block_forward (attention.cpp:61-115); q [bs,lq,h,d], k/v [bs,lk,hkv,d].
    Returns (numerator, row_max, row_norm, pairs) with rows ordered (b, i, h)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    bs, lq, h, d = q.shape
    lk, hkv = k.shape[1], k.shape[2]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    qpos = np.ascontiguousarray(qpos, dtype=np.int64)
    kpos = np.ascontiguousarray(kpos, dtype=np.int64)
    qseg = None if qseg is None else np.ascontiguousarray(qseg, dtype=np.int64)
    kseg = None if kseg is None else np.ascontiguousarray(kseg, dtype=np.int64)
    num = np.empty((bs, lq, h, d))
    mx = np.empty((bs, lq, h))
    nrm = np.empty((bs, lq, h))
    pairs = lib().orc_attn_block_forward(bs, h, hkv, d, _d(q), _i(qpos), _i(qseg), lq, _d(k),
                                         _d(v), _i(kpos), _i(kseg), lk, int(causal), scale,
                                         _d(num), _d(mx), _d(nrm))
    return num, mx, nrm, int(pairs)


def merge_piece(acc, piece):
    """merge_piece (attention.cpp:117-149); acc is None for an empty accumulator."""
    num, mx, nrm = (np.ascontiguousarray(x, dtype=np.float64) for x in piece[:3])
    if acc is None:
        return num.copy(), mx.copy(), nrm.copy()
    an, am, ar = (np.array(x, dtype=np.float64, copy=True) for x in acc[:3])
    rows, d = mx.size, num.shape[-1]
    lib().orc_merge_piece(rows, d, 0, _d(an), _d(am), _d(ar), _d(num), _d(mx), _d(nrm))
    return an, am, ar


def finalize_piece(piece):
    """finalize_piece (attention.cpp:151-165) -> (out, lse) with lse natural-log."""
    num, mx, nrm = (np.ascontiguousarray(x, dtype=np.float64) for x in piece[:3])
    out = np.empty_like(num)
    lse = np.empty_like(mx)
    lib().orc_finalize_piece(mx.size, num.shape[-1], _d(num), _d(mx), _d(nrm), _d(out), _d(lse))
    return out, lse


def block_backward(q, qpos, k, v, kpos, out, lse, dout, dq, dk, dv, causal=True, scale=None,
                   qseg=None, kseg=None):
    """attn_block_backward (attention.cpp:167-216); += into dq/dk/dv (float64, contiguous)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.ascontiguousarray(out, dtype=np.float64)
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    dout = np.ascontiguousarray(dout, dtype=np.float64)
    bs, lq, h, d = q.shape
    lk, hkv = k.shape[1], k.shape[2]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    qpos = np.ascontiguousarray(qpos, dtype=np.int64)
    kpos = np.ascontiguousarray(kpos, dtype=np.int64)
    qseg = None if qseg is None else np.ascontiguousarray(qseg, dtype=np.int64)
    kseg = None if kseg is None else np.ascontiguousarray(kseg, dtype=np.int64)
    pairs = lib().orc_attn_block_backward(bs, h, hkv, d, _d(q), _i(qpos), _i(qseg), lq, _d(k),
                                          _d(v), _i(kpos), _i(kseg), lk, int(causal), scale,
                                          _d(out), _d(lse), _d(dout), _d(dq), _d(dk), _d(dv))
    return int(pairs)


def attention_fwd_bwd(q, k, v, dout=None, positions=None, causal=True, segments=None):
    """oracle_attention (attention.cpp:218-260) fwd + the tape closure's bwd, GQA-aware.
    Returns dict(out, lse[bs,L,h], dq, dk, dv, pairs)."""
    bs, L, h, d = q.shape
    pos = np.arange(L, dtype=np.int64) if positions is None else np.asarray(positions, np.int64)
    num, mx, nrm, pairs = block_forward(q, pos, k, v, pos, causal, qseg=segments, kseg=segments)
    out, lse = finalize_piece((num, mx, nrm))
    res = {"out": out, "lse": lse, "pairs": pairs}
    if dout is not None:
        dq = np.zeros(q.shape)
        dk = np.zeros(k.shape)
        dv = np.zeros(v.shape)
        block_backward(q, pos, k, v, pos, out, lse, dout, dq, dk, dv, causal,
                       qseg=segments, kseg=segments)
        res.update(dq=dq, dk=dk, dv=dv)
    return res


def varlen_attention_fwd_bwd(q, k, v, dout, doc_lens: Sequence[int], causal=True):
    """Composed neat-packing oracle: the reference never wires segment ids into
    attention (model.cpp:339-351), so each document runs oracle_attention on its own contiguous
    rows with reset positions and the results are scattered back."""
    out = np.zeros(q.shape)
    lse = np.full(q.shape[:3], -np.inf)
    dq, dk, dv = np.zeros(q.shape), np.zeros(k.shape), np.zeros(v.shape)
    start = 0
    for n in doc_lens:
        sl = slice(start, start + n)
        r = attention_fwd_bwd(q[:, sl], k[:, sl], v[:, sl], dout[:, sl], None, causal)
        out[:, sl], lse[:, sl] = r["out"], r["lse"]
        dq[:, sl], dk[:, sl], dv[:, sl] = r["dq"], r["dk"], r["dv"]
        start += n
    return {"out": out, "lse": lse, "dq": dq, "dk": dk, "dv": dv}


IGNORE_LABEL, NO_IMAGE, NO_SEGMENT = -100, -1, -1  # partition.hpp:92-94


def pad_batch(tokens, labels, position_ids, segment_ids, image_map, sp, pad_token, cutoff_len,
              pad_to_cutoff=False):
    """pad_batch (partition.cpp:202-215): fields extended to pad_length with their sentinels;
    position ids become iota; absent (empty) segment_ids / image_map stay absent."""
    n = len(tokens)
    if n == 0:
        raise ConfigError("batch has no tokens")
    t = pad_length(n, sp, cutoff_len, pad_to_cutoff)
    ext = lambda xs, fill: list(xs) + [fill] * (t - len(xs)) if len(xs) else []  # noqa: E731
    return (ext(tokens, pad_token), ext(labels, IGNORE_LABEL), list(range(t)),
            ext(segment_ids, NO_SEGMENT), ext(image_map, NO_IMAGE))


def documents_from_segments(segment_ids):
    """Runs of equal segment ids -> document lengths (the B200 varlen bridge; the reference
    never consumes segment ids in attention, model.cpp:339-351)."""
    docs, seen, i = [], set(), 0
    seg = list(segment_ids)
    while i < len(seg):
        j = i + 1
        while j < len(seg) and seg[j] == seg[i]:
            j += 1
        if seg[i] != NO_SEGMENT:
            if seg[i] in seen:
                raise ConfigError(f"segment id {seg[i]} is not one contiguous run")
            seen.add(seg[i])
        docs.append(j - i)
        i = j
    return docs


def logprob_per_position(logits, labels):
    """sequence_logprob_per_position (losses.cpp:20-50): row[label] - (m + log(sum exp(row - m)))
    in f64, 0 for ignored labels."""
    logits = np.asarray(logits, dtype=np.float64)
    out = np.zeros(logits.shape[0])
    for t, lab in enumerate(labels):
        if lab == IGNORE_LABEL:
            continue
        row = logits[t]
        m = row.max()
        out[t] = row[lab] - (m + math.log(float(np.sum(np.exp(row - m)))))
    return out


def exact_sum(values) -> float:
    """ExactSum (exact_sum.hpp) rounds the exact sum once to nearest-even: math.fsum's contract."""
    return math.fsum(float(v) for v in np.asarray(values, dtype=np.float64).ravel())


def sft_loss(per_pos, labels) -> float:
    """sft_loss_sharded's value (losses.cpp:104-119, default weighting): -exact_sum / N_global,
    independent of the sharding."""
    n = sum(1 for lab in labels if lab != IGNORE_LABEL)
    if n == 0:
        raise ConfigError("sft loss: no supervised positions in the group")
    return exact_sum(per_pos) * (-1.0 / n)


def softplus(x: float) -> float:  # tensor.cpp:211-213
    return math.log1p(math.exp(-abs(x))) + max(x, 0.0)


def dpo_loss(pc, pr, rc, rr, beta=0.1) -> float:
    """dpo_loss_sharded's value (losses.cpp:121-135)."""
    margin = (exact_sum(pc) - exact_sum(pr)) - (exact_sum(rc) - exact_sum(rr))
    return softplus(margin * -beta)


ROPE_BASE = 10000.0  # kRopeBase (tensor.hpp:141-144)


def rope_apply(x: np.ndarray, position_ids, base: float = ROPE_BASE, inverse: bool = False):
    """rope_apply (tensor.cpp:548-607) on f64 [bs, L, heads, dim]: half-dim pairing
    (lo, hi) = (x[j], x[half + j]), theta_j = base^(-2j/dim) (:559-562), rotation by
    p*theta_j (:571-576). inverse=True is the tape backward (:589-600)."""
    if x.ndim != 4:
        raise ShapeError(f"rope_apply expects [bs, L, heads, dim], got {list(x.shape)}")
    bs, L, hs, dim = x.shape
    if dim % 2 != 0:
        raise ShapeError(f"rope head dim must be even, got {dim}")
    pos = np.asarray(position_ids, dtype=np.int64)
    if pos.shape != (L,):
        raise ShapeError(f"position_ids length {pos.size} does not match sequence extent {L}")
    half = dim // 2
    theta = np.array([math.pow(base, -2.0 * j / dim) for j in range(half)])
    ang = pos.astype(np.float64)[:, None] * theta[None, :]          # [L, half]
    c, s = np.cos(ang)[None, :, None, :], np.sin(ang)[None, :, None, :]
    if inverse:
        s = -s
    lo, hi = x[..., :half], x[..., half:]
    return np.concatenate([lo * c - hi * s, lo * s + hi * c], axis=-1)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (the inputs both sides see)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)
