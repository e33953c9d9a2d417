"""PKVC chunk files: the reference's on-disk chunk store format, plus a direct path into
pinned host memory in the device layout.

Format v1 (reference chunkstore.py:163-229, restated): ``b"PKVC"``, ``<u16 version=1``,
``<u32 header length``, a JSON header with sorted keys {fingerprint, head_dim,
n_kv_heads, n_layers, n_tokens, token_ids}, then per layer the unrotated keys and the
values as little-endian f32 ``[t][n_kv_heads][head_dim]``.  ``store_chunk`` /
``load_chunk`` are byte-compatible with the reference (tests/test_chunkfile.py stores
with one and loads with the other).

``load_chunk_pinned`` reads the same file straight into two pinned bf16 buffers in the
chunk-store layout of include/pkv.h (``[L][t][Hkv][dkp]``, RNE of the f32 payload, the
bf16 precision contract of the device path), so ``assemble`` can stream it to HBM layer
by layer while the scoring pass runs (chunkstore.assemble, pinned-host branch).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np

from .chunkstore import ChunkKV, chunk_content_id
from .errors import FormatError, ShapeError, TruncatedError
from .model import F32, Layout, ModelConfig

MAGIC = b"PKVC"
VERSION = 1
_FIXED = 10  # magic (4) + version (2) + header length (4)


def store_chunk(chunk, path) -> None:
    """Serialise a chunk (reference store_chunk, chunkstore.py:163-182)."""
    keys, values = chunk.keys_norope, chunk.values
    n_layers = len(keys)
    t = int(np.asarray(chunk.token_ids).shape[0])
    n_kv, d_k = (int(x) for x in np.asarray(keys[0]).shape[1:])
    header = {"fingerprint": chunk.config_fingerprint, "head_dim": d_k, "n_kv_heads": n_kv, "n_layers": n_layers,
              "n_tokens": t, "token_ids": [int(x) for x in np.asarray(chunk.token_ids)]}
    blob = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<HI", VERSION, len(blob)) + blob)
        for li in range(n_layers):
            for a in (keys[li], values[li]):
                arr = np.asarray(a)
                if arr.shape != (t, n_kv, d_k):
                    raise ShapeError(f"layer {li} tensor shape {arr.shape}, expected {(t, n_kv, d_k)}")
                f.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def _parse(data: bytes):
    if len(data) < _FIXED:
        raise TruncatedError("file ends inside the fixed header")
    if data[:4] != MAGIC:
        raise FormatError(f"bad magic {data[:4]!r}, expected {MAGIC!r}")
    version, hlen = struct.unpack_from("<HI", data, 4)
    if version != VERSION:
        raise FormatError(f"unsupported chunk file version {version}")
    if len(data) < _FIXED + hlen:
        raise TruncatedError("file ends inside the JSON header")
    try:
        h = json.loads(data[_FIXED:_FIXED + hlen])
        t, n_layers = int(h["n_tokens"]), int(h["n_layers"])
        n_kv, d_k = int(h["n_kv_heads"]), int(h["head_dim"])
        ids = np.asarray(h["token_ids"], dtype=np.int64)
        fp = str(h["fingerprint"])
    except (ValueError, KeyError, TypeError) as e:
        raise FormatError(f"corrupt chunk header: {e}") from e
    if ids.ndim != 1 or ids.shape[0] != t:
        raise FormatError("token_ids length disagrees with n_tokens")
    block = t * n_kv * d_k * 4
    need = _FIXED + hlen + 2 * n_layers * block
    if len(data) < need:
        raise TruncatedError(f"expected {need} bytes, file has {len(data)}")
    return fp, ids, t, n_layers, n_kv, d_k, _FIXED + hlen, block


def load_chunk(path) -> ChunkKV:
    """Read a chunk file into host f32 arrays (reference load_chunk, chunkstore.py:185-229)."""
    with open(path, "rb") as f:
        data = f.read()
    fp, ids, t, n_layers, n_kv, d_k, off, block = _parse(data)
    keys, values = [], []
    n = t * n_kv * d_k
    for _ in range(n_layers):
        for dst in (keys, values):
            dst.append(np.frombuffer(data, dtype="<f4", count=n, offset=off).reshape(t, n_kv, d_k).astype(F32))
            off += block
    return ChunkKV(chunk_content_id(fp, ids), fp, ids, keys, values)


def load_chunk_pinned(path, config: ModelConfig) -> ChunkKV:
    """Read a chunk file into pinned bf16 host buffers in the device chunk-store layout;
    ``assemble`` streams them to HBM layer by layer (overlapped with the scoring pass)."""
    import torch
    with open(path, "rb") as f:
        data = f.read()
    fp, ids, t, n_layers, n_kv, d_k, off, block = _parse(data)
    if (n_layers, n_kv, d_k) != (config.n_layers, config.n_kv_heads, config.head_dim):
        raise ShapeError(f"chunk file geometry {(n_layers, n_kv, d_k)} does not match the config")
    dkp = Layout.of(config).dkp
    payload = np.frombuffer(data, dtype="<f4", count=2 * n_layers * t * n_kv * d_k, offset=off)
    kv = torch.from_numpy(payload.reshape(n_layers, 2, t, n_kv, d_k).copy())
    k_host = torch.zeros((n_layers, t, n_kv, dkp), dtype=torch.bfloat16).pin_memory()
    v_host = torch.zeros((n_layers, t, n_kv, dkp), dtype=torch.bfloat16).pin_memory()
    k_host[..., :d_k] = kv[:, 0].to(torch.bfloat16)
    v_host[..., :d_k] = kv[:, 1].to(torch.bfloat16)
    return ChunkKV.from_pinned(chunk_content_id(fp, ids), fp, ids, k_host, v_host, d_k)


def chunk_path(store_dir, chunk_id: int) -> str:
    """Content-addressed file name used by the reference CLI (cli.py:97-101)."""
    return os.path.join(os.fspath(store_dir), f"{chunk_id:016x}.pkvc")
