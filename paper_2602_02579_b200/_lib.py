"""ctypes binding of the C-ABI library ``libpkv.so`` (include/pkv.h).

The product path has no CPU fallback: importing a device entry point without the
built library, or without a CUDA device, raises EngineError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import STATUS_TO_ERROR, EngineError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libpkv.so"

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t

PKV_QP_SCORES = 1
PKV_QP_RENORM = 2
PKV_QP_LOGITS = 4
PKV_QP_APPEND_KV = 8
PKV_QP_FROM_CHUNKS = 16
PKV_QP_PROBE = 32
PKV_QP_ROWS = 64
PKV_DT_F32, PKV_DT_F64, PKV_DT_BF16 = 0, 1, 2


class Config(ctypes.Structure):
    _fields_ = [("n_layers", c_i32), ("n_heads", c_i32), ("n_kv_heads", c_i32), ("head_dim", c_i32),
                ("hidden_dim", c_i32), ("ffn_dim", c_i32), ("vocab_size", c_i32),
                ("rope_theta", ctypes.c_double), ("norm_eps", ctypes.c_double)]


class LayerWeights(ctypes.Structure):
    _fields_ = [("attn_norm", c_vp), ("ffn_norm", c_vp), ("wqkv", c_vp), ("wo", c_vp), ("wgu", c_vp),
                ("wd", c_vp), ("wscale", ctypes.c_float * 4)]


class Weights(ctypes.Structure):
    _fields_ = [("embed", c_vp), ("final_norm", c_vp), ("lm_head", c_vp), ("layers", ctypes.POINTER(LayerWeights))]


class Cache(ctypes.Structure):
    _fields_ = [("k_pool", c_vp), ("v_pool", c_vp), ("pool_tokens", c_i64), ("page_table", c_vp), ("s", c_i32),
                ("token_ids", c_vp), ("rope_cos", c_vp), ("rope_sin", c_vp), ("rope_len", c_i32), ("recomputed", c_vp),
                ("k2_pool", c_vp), ("layer_ready", ctypes.POINTER(c_vp)),
                ("rope_cs32", c_vp), ("layer_done", ctypes.POINTER(c_vp)), ("nonfinite", c_vp),
                ("pool_heads", c_i32), ("head0", c_i32)]


class Chunks(ctypes.Structure):
    _fields_ = [("k_nr", c_vp), ("v", c_vp), ("chunk_len", c_vp), ("src_chunk", c_vp), ("src_local", c_vp),
                ("n_chunks", c_i32)]


_SIGS = {
    "pkv_layout": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(c_i32)]),
    "pkv_model_create": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Weights), ctypes.POINTER(c_vp)]),
    "pkv_model_destroy": (None, [c_vp]),
    "pkv_assemble": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Chunks), ctypes.POINTER(Cache), c_vp]),
    "pkv_assemble_layers": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Chunks), ctypes.POINTER(Cache), c_i32,
                                    c_i32, c_vp]),
    "pkv_query_pass_workspace": (c_sz, [c_vp, c_i32, c_i32, c_i32]),
    "pkv_query_pass": (c_i32, [c_vp, ctypes.POINTER(Cache), ctypes.POINTER(Chunks), c_vp, c_i32, c_i32, c_vp, c_vp,
                               c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pkv_select_workspace": (c_sz, [c_i32, c_i32]),
    "pkv_fuse_select": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pkv_topk": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "pkv_recompute_workspace": (c_sz, [c_vp, c_i32]),
    "pkv_recompute": (c_i32, [c_vp, ctypes.POINTER(Cache), c_vp, c_i32, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pkv_recompute_query_workspace": (c_sz, [c_vp, c_i32, c_i32]),
    "pkv_recompute_query": (c_i32, [c_vp, ctypes.POINTER(Cache), c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_sz, c_vp]),
    "pkv_recompute_rows_workspace": (c_sz, [c_vp, c_i32, c_i32, c_i32]),
    "pkv_recompute_rows": (c_i32, [c_vp, ctypes.POINTER(Cache), c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_sz,
                                   c_vp]),
    "pkv_full_prefill_workspace": (c_sz, [c_vp, c_i32]),
    "pkv_full_prefill": (c_i32, [c_vp, ctypes.POINTER(Cache), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pkv_replace_entries": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Cache), c_i32, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "pkv_cache_view": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Cache), ctypes.POINTER(Chunks), c_i32, c_i32, c_vp, c_vp]),
    "pkv_probe_accum": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "pkv_probe_scores": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Cache), c_vp, c_vp, c_vp, c_vp]),
    "pkv_gemm_bf16": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "pkv_proj_narrow": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "pkv_attention_sparse": (c_i32, [c_vp, ctypes.POINTER(Cache), c_i32, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "pkv_timing_enable": (c_i32, [c_i32]),
    "pkv_timing_collect": (c_i32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_i32), c_i32]),
    "pkv_nccl_load": (c_i32, [ctypes.c_char_p]),
    "pkv_comm_unique_id": (c_i32, [ctypes.c_char_p]),
    "pkv_comm_create_nccl": (c_i32, [ctypes.c_char_p, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "pkv_comm_create_local": (c_i32, [c_i32, ctypes.POINTER(c_vp)]),
    "pkv_comm_allreduce": (c_i32, [c_vp, c_vp, c_sz, c_i32, c_vp]),
    "pkv_comm_rank": (c_i32, [c_vp]),
    "pkv_comm_world": (c_i32, [c_vp]),
    "pkv_comm_destroy": (None, [c_vp]),
    "pkv_model_create_sharded": (c_i32, [ctypes.POINTER(Config), ctypes.POINTER(Weights), c_i32, c_i32, c_vp,
                                         ctypes.POINTER(c_vp)]),
    "pkv_last_error": (ctypes.c_char_p, []),
    "pkv_launch_count": (ctypes.c_uint64, []),
    "pkv_version": (c_i32, []),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes library handle. Raises EngineError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    # PKV_LIB: an alternative build of the same library (A/B timing of compile-time variants)
    p = Path(path) if path else Path(os.environ.get("PKV_LIB", LIB_PATH))
    if not p.exists():
        raise EngineError(f"CUDA extension {p} is not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        if not hasattr(lib, name) and "PKV_LIB" in os.environ and not path:
            continue  # an older build under A/B: entry points it lacks stay unbound
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status code onto the pikv exception taxonomy."""
    if rc == 0:
        return
    cls = STATUS_TO_ERROR.get(int(rc), EngineError)
    msg = load().pkv_last_error()
    raise cls(msg.decode() if msg else f"status {rc}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device: the B200 path has no CPU fallback")
    load()
    return torch


def stream_ptr(torch, stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def launch_count() -> int:
    return int(load().pkv_launch_count())


TIMER_NAMES = ("assemble", "qp_proj", "qp_attn", "qp_misc", "select", "rc_qkv", "rc_attn", "rc_o", "rc_gate_up",
               "rc_down", "rc_misc", "lm_head", "comm")


def timing(enable: bool) -> None:
    load().pkv_timing_enable(1 if enable else 0)


def timing_collect() -> dict:
    n = len(TIMER_NAMES)
    ms = (ctypes.c_double * n)()
    cnt = (c_i32 * n)()
    check(load().pkv_timing_collect(ms, cnt, n))
    return {name: (ms[i], cnt[i]) for i, name in enumerate(TIMER_NAMES)}
