"""The narrow query pass over an arbitrary host K/V state (reference model.py:362-402,
``query_pass`` / ``QueryPassResult``), on the device.

Callers outside the ProphetKV slice (the reference's scoring probes, loss probes and
tests) hand ``query_pass`` per-layer host K/V ``[t, Hkv, dk]`` (keys already rotated at
positions 0..t-1).  They are uploaded into paged fp16 pools with the keys' fp16 residual
plane (``pkv_replace_entries``), and the m query tokens at positions t..t+m-1 run through
the same fp32-faithful narrow-pass kernels as score_prophet / finalize_query, without
mutating the given state (reference: "without mutating it").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .chunkstore import QUERY_RESERVE, ctypes_ref
from .errors import ConfigError, NumericsError, ShapeError
from .model import FlopTally, ModelConfig, bill_query_pass, resolve_device_model
from .selection import check_tokens, workspace


@dataclass
class QueryPassResult:
    last_logits: np.ndarray      # [vocab], final query token
    rows: list | None            # per layer [m, t+m], head-averaged
    fresh_keys: list             # per layer [m, n_kv, d_k], rotated
    fresh_values: list           # per layer [m, n_kv, d_k]


def query_pass(weights, config: ModelConfig, kv_layers, kv_positions, query_tokens, capture_attn: bool = False,
               tally: FlopTally | None = None) -> QueryPassResult:
    """Run query tokens over a per-layer KV state (reference model.py:370-402)."""
    from .decode import DevicePools
    torch = _lib.require_cuda()
    ids = check_tokens(query_tokens, config)
    dm = resolve_device_model(weights, config)
    if getattr(dm, "tp_world", 1) > 1:
        raise ConfigError("query_pass over host K/V runs on an unsharded model")
    L, Hkv, dk = config.n_layers, config.n_kv_heads, config.head_dim
    if len(kv_layers) != L:
        raise ShapeError(f"{len(kv_layers)} KV layers for a {L}-layer model")
    keys = [np.asarray(k, dtype=np.float32) for k, _ in kv_layers]
    values = [np.asarray(v, dtype=np.float32) for _, v in kv_layers]
    t = int(keys[0].shape[0])
    for k, v in zip(keys, values):
        if k.shape != (t, Hkv, dk) or v.shape != (t, Hkv, dk):
            raise ShapeError(f"KV layer shapes {k.shape}/{v.shape}, expected {(t, Hkv, dk)}")
    pos = np.asarray(kv_positions, dtype=np.int64)
    if pos.shape != (t,):
        raise ShapeError(f"kv_positions shape {pos.shape}, expected ({t},)")
    if not np.array_equal(pos, np.arange(t)):
        raise ConfigError("the device path stores the KV state by position: kv_positions must be 0..t-1")
    m = int(ids.shape[0])
    dev = dm.device
    if t > 0:
        pools = DevicePools.from_host(config, keys, values, dev)
    else:
        pools = DevicePools(config, dev, QUERY_RESERVE)
    pools.ensure_room(m)
    flags = _lib.PKV_QP_LOGITS | (_lib.PKV_QP_ROWS if capture_attn else 0)
    fk = torch.empty((L, m, Hkv, dk), dtype=torch.float32, device=dev)
    fv = torch.empty_like(fk)
    logits = torch.empty(config.vocab_size, dtype=torch.float32, device=dev)
    rows = torch.empty((L, m, t + m), dtype=torch.float32, device=dev) if capture_attn else None
    d_ids = torch.from_numpy(ids.astype(np.int32)).to(dev)
    lib = _lib.load()
    ws = workspace(lib.pkv_query_pass_workspace(dm.handle, t, m, flags), "qp_host")
    c = pools.c_cache()
    _lib.check(lib.pkv_query_pass(dm.handle, ctypes_ref(c), None, d_ids.data_ptr(), m, flags,
                                  rows.data_ptr() if rows is not None else None, fk.data_ptr(), fv.data_ptr(),
                                  logits.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(torch)))
    bill_query_pass(tally, config, t, m)
    last = logits.cpu().numpy()
    if not np.isfinite(last).all():
        raise NumericsError("non-finite values in the query-pass logits")
    fkh, fvh = fk.cpu().numpy(), fv.cpu().numpy()
    rows_h = None
    if rows is not None:
        ra = rows.cpu().numpy()
        rows_h = [np.ascontiguousarray(ra[li]) for li in range(L)]
    return QueryPassResult(last_logits=last, rows=rows_h, fresh_keys=[fkh[li] for li in range(L)],
                           fresh_values=[fvh[li] for li in range(L)])
