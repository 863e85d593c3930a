"""ctypes binding of the C-ABI in include/fluxattn_b200.h.

The shared library is built in-tree (paper_2605_07719_b200/_lib/) by
``__graft_entry__.build()`` / ``make -C paper_2605_07719_b200/csrc``.  There
is no fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLUXATTN_B200_LIB", os.path.join(HERE, "_lib", "libfluxattn_b200.so"))

FX_OK = 0
FX_F32 = 0
FX_BF16 = 1
FX_PLAN_PROPS = 0
FX_PLAN_FIXED = 1
FX_PLAN_FULL = 2
FX_PLAN_GIVEN = 3
ABI_VERSION = 5
KERNELS = ("plan", "score", "select", "worklist", "attend", "metadata", "append", "merge")

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t


class Layout(C.Structure):
    """fx_layout: [batch][kv_heads][l_cap][head_dim] K/V, rows sink|cpu|local|new."""

    _fields_ = [("batch", _i32), ("kv_heads", _i32), ("group_size", _i32), ("head_dim", _i32),
                ("dtype", _i32), ("reserved", _i32), ("l_sink", _i64), ("l_cpu", _i64),
                ("l_local", _i64), ("l_cap", _i64)]


class StepArgs(C.Structure):
    _fields_ = [("k", _p), ("v", _p), ("meta", _p * 4), ("absmax", _p), ("l_new", _i64),
                ("q", _p), ("plan_mode", _i32), ("fixed_block_size", _i32),
                ("fixed_budget", C.c_double), ("bgt0", _p), ("kslope", _p), ("streaming", _p),
                ("plan_blk", _p), ("plan_budgets", _p), ("plan_volume", _p),
                ("plan_cand_volumes", _p), ("plan_kblocks", _p), ("sel_bits", _p),
                ("sel_words", _i32), ("o", _p), ("lse", _p),
                # context-parallel shard (C5); zero on a single device
                ("l_cpu_total", _i64), ("cpu_offset", _i64), ("sel_in", _p),
                # optional fused append of the previous step's token
                ("append_k", _p), ("append_v", _p)]


class WorkloadSpec(C.Structure):
    """fx_workload_spec (workload.hpp:16-54)."""

    _fields_ = [("seed", C.c_uint64), ("layers", _i32), ("heads", _i32), ("group_size", _i32),
                ("head_dim", _i32), ("context_len", _i32), ("sink_tokens", _i32),
                ("local_tokens", _i32), ("decode_steps", _i32), ("streaming_frac", C.c_double),
                ("retrieval_frac", C.c_double), ("sink_frac", C.c_double),
                ("diffuse_frac", C.c_double), ("needles", _i32), ("needle_tokens", _i32),
                ("needle_strength", C.c_double), ("payload_gain", C.c_double),
                ("local_boost", C.c_double), ("query_jitter", C.c_double),
                ("streaming_jitter", C.c_double), ("decoy_strength", C.c_double),
                ("decoy_payload_strength", C.c_double), ("decoy_tokens", _i32),
                ("decoy_payload_tokens", _i32), ("query_drift", C.c_double)]

    DEFAULTS = dict(seed=1, layers=4, heads=8, group_size=4, head_dim=64, context_len=4096,
                    sink_tokens=64, local_tokens=256, decode_steps=8, streaming_frac=0.5,
                    retrieval_frac=0.5, sink_frac=0.0, diffuse_frac=0.0, needles=1,
                    needle_tokens=16, needle_strength=10.0, payload_gain=3.0, local_boost=7.0,
                    query_jitter=0.2, streaming_jitter=0.45, decoy_strength=6.0,
                    decoy_payload_strength=4.0, decoy_tokens=160, decoy_payload_tokens=64,
                    query_drift=0.98)

    @classmethod
    def make(cls, **kw):
        d = dict(cls.DEFAULTS)
        d.update(kw)
        return cls(**d)


class TraceInfo(C.Structure):
    """fx_trace_info: the FXT1 header (workload.cpp:311-340)."""

    _fields_ = [("input_hash", C.c_uint64), ("seed", C.c_uint64), ("layers", _i32),
                ("heads", _i32), ("group_size", _i32), ("head_dim", _i32),
                ("context_len", _i32), ("sink_tokens", _i32), ("local_tokens", _i32),
                ("decode_steps", _i32)]


class CpPeer(C.Structure):
    """fx_cp_peer: one rank's exchange tables as seen from this device."""

    _fields_ = [("keys", _p), ("ids", _p), ("kth", _p), ("o", _p), ("lse", _p), ("flags", _p),
                ("cap", _i64), ("stats", _p), ("hist", _p), ("defc", _p)]


class NativeError(RuntimeError):
    """A non-zero fx_* status; the message carries the reference error code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


_SIGS = {
    "fx_last_error": (C.c_char_p, []),
    "fx_abi_version": (C.c_int, []),
    "fx_ctx_create": (C.c_int, [C.c_int, C.POINTER(_p)]),
    "fx_ctx_destroy": (C.c_int, [_p]),
    "fx_ctx_set_stream": (C.c_int, [_p, _p]),
    "fx_ctx_stream": (_p, [_p]),
    "fx_ctx_synchronize": (C.c_int, [_p]),
    "fx_ctx_launches": (C.c_uint64, [_p]),
    "fx_ctx_set_timing": (C.c_int, [_p, C.c_int]),
    "fx_ctx_kernel_time": (C.c_int, [_p, _i32, C.POINTER(C.c_double), C.POINTER(_i64)]),
    "fx_ctx_reset_timing": (C.c_int, [_p]),
    "fx_malloc": (C.c_int, [_p, _sz, C.POINTER(_p)]),
    "fx_free": (C.c_int, [_p, _p]),
    "fx_memcpy_h2d": (C.c_int, [_p, _p, _p, _sz]),
    "fx_memcpy_d2h": (C.c_int, [_p, _p, _p, _sz]),
    "fx_memset": (C.c_int, [_p, _p, C.c_int, _sz]),
    "fx_block_count": (_i64, [_i64, _i32]),
    "fx_meta_level_bytes": (_sz, [C.POINTER(Layout), _i32]),
    "fx_step_scratch_bytes": (_sz, [C.c_void_p, C.POINTER(Layout)]),
    "fx_build_metadata_levels": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _p, _p, _p, _p]),
    "fx_build_metadata": (C.c_int, [_p, _p, _i32, _i64, _i32, _i32, _p]),
    "fx_block_scores": (C.c_int, [_p, _p, _p, _i32, _i64, _i32, _p]),
    "fx_topk_blocks": (C.c_int, [_p, _p, _p, _i32, _i64, _i32, _i64, _p, C.POINTER(_i64),
                                 C.POINTER(_i32)]),
    "fx_approx_scores": (C.c_int, [_p, C.POINTER(Layout), _p * 4, _p, _p, _p,
                                   C.POINTER(C.c_double)]),
    "fx_plan_groups":(C.c_int, [_p, _i32, _i32, _i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "fx_blocks_for_budget": (C.c_int, [_p, _i32, _p, _p, _i64, _p]),
    "fx_model_create": (C.c_int, [_p] + [_p] * 8 + [C.POINTER(_p)]),
    "fx_model_destroy": (C.c_int, [_p]),
    "fx_predict": (C.c_int, [_p, _p, _i32, _p, _p, _p, _p, _p]),
    "fx_decode_step": (C.c_int, [_p, C.POINTER(Layout), C.POINTER(StepArgs)]),
    "fx_plan_select": (C.c_int, [_p, C.POINTER(Layout), C.POINTER(StepArgs)]),
    "fx_sparse_decode": (C.c_int, [_p, C.POINTER(Layout), C.POINTER(StepArgs)]),
    "fx_gathered_attention": (C.c_int, [_p, _p, _p, _p, _i32, _i64, _i32, _p, _i64, _p, _p]),
    "fx_merge_partials": (C.c_int, [_p, _i32, _i32, _p, _p, _p, _p]),
    "fx_append_kv": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _i64, _p, _p]),
    "fx_convert": (C.c_int, [_p, _p, _p, _i32, _sz]),
    "fx_cp_candidates": (C.c_int, [_p, C.POINTER(Layout), C.POINTER(StepArgs), _i64, _p, _p, _p, _p]),
    "fx_cp_threshold": (C.c_int, [_p, _i32, _i64, _i64, _p, _p, _p, _p]),
    "fx_cp_select": (C.c_int, [_p, C.POINTER(Layout), _i32, _i32, _i64, _p, _p, _p, _p, _p, _i64,
                               _p, _i32]),
    "fx_cp_combine": (C.c_int, [_p, _i32, _i64, _i32, _p, _p, _p, _p]),
    "fx_prefill_stats": (C.c_int, [_p, C.POINTER(Layout), _p, _p, C.POINTER(_p * 4), _p,
                                   C.c_double, _i32, _p]),
    "fx_decode_features": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _i64, _p, _p, _p]),
    "fx_memcpy_d2d": (C.c_int, [_p, _p, _p, _sz]),
    "fx_build_metadata_means": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _p, _p]),
    "fx_predict_props": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "fx_generate": (C.c_int, [_p, C.POINTER(WorkloadSpec), C.POINTER(Layout), _p, _p, _p, _p, _p,
                              _i32, _p, _p, _p, _p]),
    "fx_trace_info_read": (C.c_int, [C.c_char_p, C.POINTER(TraceInfo)]),
    "fx_trace_load": (C.c_int, [_p, C.c_char_p, _i32, C.POINTER(Layout), _i32, _p, _p, _p, _p,
                                _p, _p, _p]),
    "fx_trace_save": (C.c_int, [_p, C.c_char_p, C.POINTER(TraceInfo), C.POINTER(Layout), _p, _p,
                                _p, _p, _p, _p, _p, _p, _p, _p]),
    "fx_cp_signal": (C.c_int, [_p, _p, _i32, C.c_uint64]),
    "fx_cp_select_peer": (C.c_int, [_p, C.POINTER(Layout), _i32, _i32, _p, C.c_uint64, _p, _p, _i64,
                                    _p, _i32]),
    "fx_cp_dist_phase": (C.c_int, [_p, C.POINTER(Layout), C.POINTER(StepArgs), _i32, _i32, _i32, _p,
                                   C.c_uint64, _p, _i64]),
    "fx_cp_combine_peer": (C.c_int, [_p, _i32, _i64, _i32, _p, C.c_uint64, _p, _p]),
    "fx_ipc_handle": (C.c_int, [_p, C.c_char_p, C.POINTER(_i64)]),
    "fx_ipc_open": (C.c_int, [_p, C.c_char_p, C.POINTER(_p)]),
    "fx_ipc_close": (C.c_int, [_p, _p]),
    "fx_label_heads": (C.c_int, [_p, C.POINTER(Layout), _p, _p, _i64, C.POINTER(_p * 4), _p,
                                 C.c_double, _i32, _p, _p, _p, _p, _p, _p, _p]),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fx_abi_version() != ABI_VERSION:
        raise ImportError("fluxattn_b200 ABI version mismatch")
    return lib


LIB = load()


def check(status: int) -> None:
    if status != FX_OK:
        msg = LIB.fx_last_error()
        raise NativeError(status, msg.decode() if msg else f"fx status {status}")
