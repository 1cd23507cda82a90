"""ctypes binding of libspattn.so (include/spattn.h). No torch types cross this boundary:
device buffers are passed as integer pointers, streams as cudaStream_t handles.

The library is built in-tree (``make -C paper_2505_22296_b200`` or ``__graft_entry__.build()``).
There is no fallback: a missing library is an ImportError at first use."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPATTN_LIB (development A/B builds) names another build of the library inside the package
LIB_PATH = os.path.join(_HERE, os.environ.get("SPATTN_LIB", "libspattn.so"))

OK, ERR_CONFIG, ERR_SHAPE, ERR_STATE, ERR_PEER = range(5)
ENGINES = ["oracle", "ulysses", "dummy_head", "xtuner", "ring", "usp"]
SPLITS = ["naive", "zigzag", "usp"]
PRIMITIVES = ["all_to_all", "all_gather", "p2p", "all_reduce", "broadcast"]

# Every entry point include/spattn.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "spattn_last_error", "spattn_abi_version", "spattn_layout_positions", "spattn_causal_pairs",
    "spattn_pad_length", "spattn_pick_xtuner_insp", "spattn_reference_bytes",
    "spattn_nccl_unique_id", "spattn_ctx_create_nccl", "spattn_ctx_destroy",
    "spattn_fabric_create", "spattn_fabric_destroy", "spattn_fabric_ctx", "spattn_ctx_set_stream",
    "spattn_ctx_stream", "spattn_ctx_stats", "spattn_ctx_flops", "spattn_ctx_reset_stats",
    "spattn_set_kernel_family", "spattn_get_kernel_family", "spattn_fwd", "spattn_bwd",
    "spattn_saved_free", "spattn_fabric_fwd", "spattn_fabric_bwd", "spattn_fabric_all_to_all",
    "spattn_block_fwd", "spattn_block_finalize", "spattn_lse_merge", "spattn_block_bwd",
    "spattn_shard_rows", "spattn_gather_rows", "spattn_launch_count", "spattn_profile_enable",
    "spattn_profile_read", "spattn_debug_timeline", "spattn_debug_timeline_read", "spattn_selftest_umma", "spattn_plan_heads", "spattn_plan_problems",
    "spattn_debug_bwd_trace", "spattn_debug_fwd_cta_trace", "spattn_debug_transport_selftest", "spattn_fwd_rope", "spattn_fabric_fwd_rope", "spattn_rope_apply",
    "spattn_step_host", "spattn_pick_step_groups", "spattn_pick_step_groups_len", "spattn_pad_batch",
    "spattn_split_position_map", "spattn_documents_from_segments", "spattn_replicate_packing_mask", "spattn_broadcast_bytes",
    "spattn_fabric_replicate_packing_mask", "spattn_logprob_fwd", "spattn_logprob_bwd",
    "spattn_exact_sum_device", "spattn_exact_sum_host", "spattn_exact_merge", "spattn_exact_round",
    "spattn_exact_sum_all_reduce", "spattn_all_reduce_count", "spattn_all_reduce_values",
    "spattn_all_to_all", "spattn_all_gather", "spattn_all_gather_backward", "spattn_ring_shift",
]


class ConfigError(ValueError):
    """seqpar::ConfigError (reference tensor.hpp:24; ValueError in py_module.cpp:320)."""


class ShapeError(ValueError):
    """seqpar::ShapeError (reference tensor.hpp:18)."""


class StateError(RuntimeError):
    """seqpar::StateError / CUDA / NCCL failure."""


class PeerAbort(RuntimeError):
    """A peer rank failed (reference comm.cpp:10-14)."""


class SpattnConfig(ctypes.Structure):
    _fields_ = [("heads", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("causal", ctypes.c_int32),
                ("ulysses_degree", ctypes.c_int32), ("ring_degree", ctypes.c_int32)]


class SpattnLayout(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("sp", ctypes.c_int32), ("global_len", ctypes.c_int64),
                ("u_degree", ctypes.c_int32), ("r_degree", ctypes.c_int32)]


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.c_int


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    try:  # share the CUDA runtime torch already mapped (same soname)
        import torch  # noqa: F401
    except Exception:  # pragma: no cover - torch is part of the image
        pass
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    L.spattn_last_error.restype = ctypes.c_char_p
    L.spattn_get_kernel_family.restype = _i32
    L.spattn_saved_free.restype = None
    L.spattn_saved_free.argtypes = [_vp]
    L.spattn_launch_count.restype = _i64
    L.spattn_launch_count.argtypes = []
    cfgp, layp = ctypes.POINTER(SpattnConfig), ctypes.POINTER(SpattnLayout)
    sig = {
        "spattn_layout_positions": [layp, _i32, _i64p],
        "spattn_causal_pairs": [layp, _i32, _i64p],
        "spattn_pad_length": [_i64, _i32, _i64, _i32, _i64p],
        "spattn_pick_xtuner_insp": [_i32, _i32, _i32, ctypes.POINTER(ctypes.c_int)],
        "spattn_reference_bytes": [_i32, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _i64p],
        "spattn_nccl_unique_id": [ctypes.c_char_p],
        "spattn_ctx_create_nccl": [_i32, _i32, _i32, _i32, ctypes.c_char_p, ctypes.POINTER(_vp)],
        "spattn_ctx_destroy": [_vp],
        "spattn_fabric_create": [_i32, _i32, _i32, _i32, ctypes.POINTER(_vp)],
        "spattn_fabric_destroy": [_vp],
        "spattn_fabric_ctx": [_vp, _i32, ctypes.POINTER(_vp)],
        "spattn_ctx_set_stream": [_vp, _vp],
        "spattn_ctx_stream": [_vp, ctypes.POINTER(_vp)],
        "spattn_ctx_stats": [_vp, _i32, _i64p, _i64p],
        "spattn_ctx_flops": [_vp, _i64p],
        "spattn_ctx_reset_stats": [_vp],
        "spattn_set_kernel_family": [_i32],
        "spattn_fwd": [_vp, _i32, cfgp, layp, _i64, _vp, _vp, _vp, _vp, _vp, _i64p, _i32,
                       ctypes.POINTER(_vp)],
        "spattn_fwd_rope": [_vp, _i32, cfgp, layp, _i64, _vp, _vp, _vp, _vp, _vp, _i64p, _i32,
                            _i64p, ctypes.c_double, ctypes.POINTER(_vp)],
        "spattn_bwd": [_vp, _vp, _vp, _vp, _vp, _vp],
        "spattn_fabric_fwd": [_vp, _i32, cfgp, layp, _i64, ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), _i64p, _i32, ctypes.POINTER(_vp)],
        "spattn_fabric_fwd_rope": [_vp, _i32, cfgp, layp, _i64, ctypes.POINTER(_vp),
                                   ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                   ctypes.POINTER(_vp), _i64p, _i32, ctypes.POINTER(_i64p),
                                   ctypes.c_double, ctypes.POINTER(_vp)],
        "spattn_pick_step_groups": [_i32, cfgp, _i32],
        "spattn_pick_step_groups_len": [_i32, cfgp, _i32, _i64],
        "spattn_logprob_fwd": [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp],
        "spattn_logprob_bwd": [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _i32],
        "spattn_exact_sum_device": [_vp, _vp, _i64, _vp],
        "spattn_exact_sum_host": [_vp, _i64, _vp],
        "spattn_exact_merge": [_vp, _vp],
        "spattn_exact_round": [_vp, ctypes.POINTER(ctypes.c_double)],
        "spattn_exact_sum_all_reduce": [_vp, _vp],
        "spattn_all_reduce_count": [_vp, _i64p],
        "spattn_all_reduce_values": [_vp, _vp, _i64],
        "spattn_pad_batch": [_i64p] * 5 + [_i64, _i32, _i64, _i64, _i32] + [_i64p] * 6,
        "spattn_split_position_map": [layp, _i32, _i64p, _i64p],
        "spattn_documents_from_segments": [_i64p, _i64, _i64p, _i32, ctypes.POINTER(ctypes.c_int)],
        "spattn_replicate_packing_mask": [_vp, _vp, _i64, _vp, _i64, _i64p],
        "spattn_broadcast_bytes": [_vp, _vp, _i64, _i32, _vp, _i64, _i64p],
        "spattn_fabric_replicate_packing_mask": [_vp, ctypes.POINTER(_vp), _i64p, ctypes.POINTER(_vp),
                                                 _i64, _i64p],
        "spattn_step_host": [_vp, _i32, cfgp, layp, _i64] + [_vp] * 9 + [_i64p, _i32, _i32],
        "spattn_rope_apply": [_vp, _i64, _i64, _i32, _i32, _vp, _i64p, ctypes.c_double, _i32, _vp],
        "spattn_fabric_bwd": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
        "spattn_all_to_all": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32],
        "spattn_all_gather": [_vp, _vp, _vp, _i64, _i64, _i64],
        "spattn_all_gather_backward": [_vp, _vp, _vp, _i64, _i64, _i64],
        "spattn_ring_shift": [_vp, _vp, _vp, _i64],
        "spattn_fabric_all_to_all": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, _i64,
                                     _i64, _i64, _i32, _i32, _i32],
        "spattn_block_fwd": [_vp, _i64, _i32, _i32, _i32, _vp, _i64p, _i64, _vp, _vp, _i64p,
                             _i64, _i32, ctypes.c_double, _vp, _vp, _i64p],
        "spattn_block_finalize": [_vp, _i64, _i32, _vp, _vp],
        "spattn_lse_merge": [_vp, _vp, _vp, _vp, _vp, _i64, _i32],
        "spattn_block_bwd": [_vp, _i64, _i32, _i32, _i32, _vp, _i64p, _i64, _vp, _vp, _i64p,
                             _i64, _i32, ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _i64p],
        "spattn_profile_enable": [_i32],
        "spattn_debug_bwd_trace": [_vp],
        "spattn_debug_fwd_cta_trace": [_vp],
        "spattn_debug_transport_selftest": [_vp, ctypes.c_int64],
        "spattn_plan_heads": [_i32, _i32, _i32] + [ctypes.POINTER(ctypes.c_int32)] * 4,
        "spattn_plan_problems": [_i64p, _i64, _i64p, _i64, _i32, _i64p, _i32,
                                 ctypes.POINTER(ctypes.c_int32), _i32, ctypes.POINTER(ctypes.c_int),
                                 _i64p],
        "spattn_selftest_umma": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
        "spattn_profile_read": [ctypes.POINTER(ctypes.c_double), _i64p],
        "spattn_debug_timeline": [_i32],
        "spattn_debug_timeline_read": [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _i32, _i64p],
        "spattn_shard_rows": [_vp, layp, _i32, _i64, _i64, _vp, _vp],
        "spattn_gather_rows": [_vp, layp, _i32, _i64, _i64, _vp, _vp],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _i32
    _lib = L
    return L


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().spattn_last_error().decode()
    raise {ERR_CONFIG: ConfigError, ERR_SHAPE: ShapeError, ERR_PEER: PeerAbort}.get(
        status, StateError)(msg)


ZIGZAG_BLOCKS = 3  # SPATTN_ZIGZAG_BLOCKS (extension): "zigzag:B" = zigzag within each of B blocks


def make_layout(mode: str, length: int, sp: int, u: int = 0, r: int = 0) -> SpattnLayout:
    if mode.startswith("zigzag:"):
        try:
            blocks = int(mode.split(":", 1)[1])
        except ValueError:
            raise ConfigError(f"unknown split mode '{mode}'") from None
        return SpattnLayout(ZIGZAG_BLOCKS, sp, length, blocks, 0)
    if mode not in SPLITS:
        raise ConfigError(f"unknown split mode '{mode}'")
    return SpattnLayout(SPLITS.index(mode), sp, length, u, r)


def make_config(heads, kv_heads, head_dim, causal=True, u=0, r=0) -> SpattnConfig:
    return SpattnConfig(heads, kv_heads, head_dim, int(bool(causal)), u, r)


def engine_id(name: str) -> int:
    if name not in ENGINES:
        raise ConfigError(f"unknown engine '{name}'")
    return ENGINES.index(name)


def ptr_array(ptrs):
    arr = (_vp * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
