"""ctypes declarations of include/forkkv.h (argument marshalling only).

Loads the in-tree ``libforkkv.so``; raises ImportError if it is missing — there
is no fallback of any kind.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FKV_LIB_PATH: an alternative build of the same library (diagnostic A/B variants, tools/variants.sh)
LIB_PATH = os.environ.get("FKV_LIB_PATH") or os.path.join(HERE, "libforkkv.so")

OK = 0
E_INVALID = 1
E_NEEDS_EVICTION = 2
E_UNKNOWN_AGENT = 3
E_STALE = 4
E_READONLY = 5
E_NO_KEYS = 6
E_UNWRITTEN = 7
E_CUDA = 8
STATUS_NAMES = {0: "OK", 1: "E_INVALID", 2: "E_NEEDS_EVICTION", 3: "E_UNKNOWN_AGENT", 4: "E_STALE",
                5: "E_READONLY", 6: "E_NO_KEYS", 7: "E_UNWRITTEN", 8: "E_CUDA"}

DTYPE_BF16 = 0
DTYPE_F32 = 1
ROPE_NONE = 0
ROPE_DEFERRED = 1
KIND_BASE = 0
KIND_RES = 1
FORK_SHARE_RESIDUAL = 1
WRITE_KBASE, WRITE_VBASE, WRITE_RK, WRITE_RV = 1, 2, 4, 8
WRITE_ALL = 15
PLAN_CHECK_WRITTEN = 1
PLAN_FORCE_SIMT = 2
PLAN_FORCE_MMA = 4
PLAN_ROWS_KERNEL = 8


class fkv_config(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("rank", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("n_base_pages", ctypes.c_int64), ("n_res_pages", ctypes.c_int64), ("max_pos", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("rope_mode", ctypes.c_int32), ("device", ctypes.c_int32),
                ("alloc_order_seed", ctypes.c_uint64), ("kv_head_begin", ctypes.c_int32),
                ("kv_head_end", ctypes.c_int32)]


class fkv_buffers(ctypes.Structure):
    _fields_ = [("base_k", ctypes.c_void_p), ("base_v", ctypes.c_void_p), ("res_k", ctypes.c_void_p),
                ("res_v", ctypes.c_void_p), ("rope_cos", ctypes.c_void_p), ("rope_sin", ctypes.c_void_p)]


class fkv_seq(ctypes.Structure):
    _fields_ = [("agent", ctypes.c_int64), ("q_len", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class fkv_plan_info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_seqs", "n_rows", "n_segments", "n_items", "n_ctas", "n_warps",
                                               "n_entries", "key_tiles", "alg_bytes", "kernel", "device_bytes",
                                               "workspace_bytes", "alg_rank_bytes")]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_f32 = ctypes.c_float
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)

SIGNATURES = {
    "fkv_create": ([ctypes.POINTER(fkv_config), ctypes.POINTER(fkv_buffers), ctypes.POINTER(_vp)], _i32),
    "fkv_destroy": ([_vp], _i32),
    "fkv_last_error": ([_vp], ctypes.c_char_p),
    "fkv_version": ([], ctypes.c_char_p),
    "fkv_register_adapter": ([_vp, _i32, _vp, _vp], _i32),
    "fkv_create_root": ([_vp, _i64, _i32], _i32),
    "fkv_fork": ([_vp, _i64, _i64, _i64, _i32, _u32], _i32),
    "fkv_fork_tokens": ([_vp, _i64, _i32, _pi32, _i64, _pi64], _i32),
    "fkv_partition_keys": ([_i64, _i32, _i32, _i32, _pi64, _pi64], _i32),
    "fkv_plan_create_range": ([_vp, _i32, _vp, _u32, _i64, _i64, ctypes.POINTER(_vp)], _i32),
    "fkv_residual_attention_lse": ([_vp, _vp, _i32, _vp, _vp, _vp, _f32, _vp, ctypes.c_size_t, _vp], _i32),
    "fkv_merge_lse": ([_i32, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp], _i32),
    "fkv_register_adapter_down": ([_vp, _i32, _vp, _vp, _i32], _i32),
    "fkv_project_workspace_bytes": ([_vp, _i64, ctypes.POINTER(ctypes.c_size_t)], _i32),
    "fkv_project_kv": ([_vp, _i32, _i32, _pi64, _pi64, _pi32, _vp, _i32, _vp, _vp, _u32, _vp, ctypes.c_size_t, _vp],
                       _i32),
    "fkv_fork_resume": ([_vp, _i64, _i32, _i64, _pi32, _i64, _pi64, _pi64, _pi64], _i32),
    "fkv_evict": ([_vp, _i32, _i64, _pi64], _i32),
    "fkv_evictable_pages": ([_vp, _i32, _pi64], _i32),
    "fkv_append": ([_vp, _i32, _pi64, _pi32, _pi32, _vp], _i32),
    "fkv_write_kv": ([_vp, _i32, _i32, _pi64, _pi64, _pi32, _vp, _vp, _vp, _vp, _u32, _vp], _i32),
    "fkv_release": ([_vp, _i64], _i32),
    "fkv_get_table": ([_vp, _i64, _i64, _pi32, _pi32, _pi64, _pi64], _i32),
    "fkv_get_agent": ([_vp, _i64, _pi32, _pi64], _i32),
    "fkv_page_refcount": ([_vp, _i32, _i64, _pi32], _i32),
    "fkv_free_pages": ([_vp, _i32, _pi64], _i32),
    "fkv_dump": ([_vp, ctypes.c_char_p, _sz, ctypes.POINTER(_sz)], _i32),
    "fkv_take_copy_log": ([_vp, _pi32, _i64, _pi64], _i32),
    "fkv_plan_create": ([_vp, _i32, ctypes.POINTER(fkv_seq), _u32, ctypes.POINTER(_vp)], _i32),
    "fkv_plan_get_info": ([_vp, ctypes.POINTER(fkv_plan_info)], _i32),
    "fkv_plan_upload": ([_vp, _vp, _vp, _sz, _vp], _i32),
    "fkv_residual_attention": ([_vp, _vp, _i32, _vp, _vp, _f32, _vp, _sz, _vp], _i32),
    "fkv_residual_attention_phases": ([_vp, _vp, _i32, _vp, _vp, _f32, _vp, _sz, _vp, _u32], _i32),
    "fkv_residual_attention_host":([_vp, _vp, _i32, _vp, _vp, _vp, _vp, _f32, _vp, _sz, _vp], _i32),
    "fkv_plan_free": ([_vp], _i32),
    "fkv_build_rope_table": ([_i32, _i32, _f64, _i32, _f64, _f64, _f64, _f64, _vp, _vp], _i32),
    "fkv_synth_fill": ([_vp, _i32, _u64, _i32, _u64, _i32, _i64, _i32, _i32, _i32, _i32, _f32, _vp], _i32),
    "fkv_selftest_umma": ([_i32, _vp, _vp, _vp, _i32, _i32, _i32, _vp], _i32),
    "fkv_debug_timeline": ([_vp, _vp, _i32], _i32),
    "fkv_debug_hang_report": ([ctypes.c_char_p, _i64], _i32),
    "fkv_partition": ([_i32, _i32, _i64, _i64, _pi32, _pi32], _i32),
    "fkv_partition_shard": ([_i32, _i32, _i32, _i32, _i64, _pi32, _pi32, _pi64, _pi64], _i32),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2604_06370_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


class FkvError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
