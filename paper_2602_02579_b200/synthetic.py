"""Synthetic, CPU-reproducible benchmark inputs generated on the device ("SYN1").

The bench's random-init weights and chunk store must be checkable against the CPU
oracle, and at Llama-3-8B scale (8 B weights, 4.3 GB of chunk K/V) the reference's own
``random_weights`` PCG64 stream takes minutes on one host core.  SYN1 is a counter-based
generator that the device evaluates in milliseconds and numpy reproduces bit for bit
(``oracle/synthetic_inputs.py``, the same arithmetic):

  key(seed, tid) = mix32(seed * 0x9E3779B1 + tid * 0x85EBCA77 + 0x165667B1)
  u1 = mix32(i ^ key), u2 = mix32(u1 ^ 0x68E31DA4)          i = flat element index
  z  = lo16(u1) + hi16(u1) + lo16(u2) + hi16(u2) - 131070    (Irwin-Hall(4): mean 0, sd 37837.23)
  x  = bf16( f32(z) * f32(std / 37837.22703) )

mix32 is a 32-bit avalanche hash (xorshift-multiply).  Every step is integer or one
IEEE f32 multiply followed by RNE to bf16, so device and host agree exactly.  The values
follow the reference's initialisation scale (model.py:163-185: N(0,1)/sqrt(fan_in) for
projections, N(0,1) for the embedding); chunk keys/values are sd-1 like projected K/V.

Tensor ids (tid): layer l projection k (wq, wk, wv, wo, w_gate, w_up, w_down = 0..6) ->
16 l + k; embed 0x0FFFFFF0, lm_head 0x0FFFFFF1; chunk c layer l keys / values ->
0x10000000 + 2048 c + 2 l + (0 | 1); chunk c token ids 0x20000000 + c; query 0x30000000.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib

M32 = 0xFFFFFFFF
IH4_SD = 37837.22703  # sd of the sum of four uniform 16-bit integers
TID_EMBED, TID_HEAD = 0x0FFFFFF0, 0x0FFFFFF1
LAYER_TIDS = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "w_gate": 4, "w_up": 5, "w_down": 6}


def tid_chunk(c: int, layer: int, is_value: bool) -> int:
    return 0x10000000 + 2048 * c + 2 * layer + (1 if is_value else 0)


def tid_tokens(c: int) -> int:
    return 0x20000000 + c


TID_QUERY = 0x30000000


def key(seed: int, tid: int) -> int:
    return _mix32_int((seed * 0x9E3779B1 + tid * 0x85EBCA77 + 0x165667B1) & M32)


def _mix32_int(x: int) -> int:
    x ^= x >> 16
    x = (x * 0x7FEB352D) & M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & M32
    return x ^ (x >> 16)


def _mix32(x):
    """mix32 on an int64 torch tensor holding values in [0, 2^32)."""
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & M32  # int64 wrap-around keeps the low 32 bits exact
    return x ^ (x >> 16)


def _u12(torch, n: int, k: int, start: int, device):
    i = torch.arange(start, start + n, dtype=torch.int64, device=device)
    u1 = _mix32(i ^ k)
    u2 = _mix32(u1 ^ 0x68E31DA4)
    return u1, u2


def _torch_on(device):
    """torch and the target device (default: the current CUDA device; "cpu" is allowed so the
    CPU test suite can check this restatement against the numpy one)."""
    if device is not None and str(device) == "cpu":
        import torch
        return torch, torch.device("cpu")
    torch = _lib.require_cuda()
    return torch, device or torch.device("cuda", torch.cuda.current_device())


def normal_bf16(shape, seed: int, tid: int, std: float, device=None, block: int = 1 << 26):
    """bf16 tensor of `shape` (flat index order) with SYN1 values of sd `std`."""
    torch, device = _torch_on(device)
    n = math.prod(shape)
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    k = key(seed, tid)
    c = torch.tensor(float(np.float32(std / IH4_SD)), dtype=torch.float32, device=device)
    for s0 in range(0, n, block):
        nb = min(block, n - s0)
        u1, u2 = _u12(torch, nb, k, s0, device)
        z = (u1 & 0xFFFF) + (u1 >> 16) + (u2 & 0xFFFF) + (u2 >> 16) - 131070
        out[s0:s0 + nb] = (z.to(torch.float32) * c).to(torch.bfloat16)
    return out.view(shape)


def token_ids(n: int, vocab: int, seed: int, tid: int, device=None):
    """int64 ids in [0, vocab): u1 mod vocab."""
    torch, device = _torch_on(device)
    u1, _ = _u12(torch, n, key(seed, tid), 0, device)
    return u1 % vocab


def layer_weights(cfg, layer: int, seed: int, device=None) -> dict:
    """Reference-layout (input-major [fan_in, fan_out]) bf16 weights of one layer."""
    D, Q, KV, F = cfg.hidden_dim, cfg.n_heads * cfg.head_dim, cfg.kv_dim, cfg.ffn_dim
    shapes = {"wq": (D, Q), "wk": (D, KV), "wv": (D, KV), "wo": (Q, D), "w_gate": (D, F), "w_up": (D, F),
              "w_down": (F, D)}
    return {name: normal_bf16(shp, seed, 16 * layer + LAYER_TIDS[name], 1.0 / math.sqrt(shp[0]), device)
            for name, shp in shapes.items()}


def embed(cfg, seed: int, device=None):
    return normal_bf16((cfg.vocab_size, cfg.hidden_dim), seed, TID_EMBED, 1.0, device)


def lm_head(cfg, seed: int, device=None):
    return normal_bf16((cfg.hidden_dim, cfg.vocab_size), seed, TID_HEAD, 1.0 / math.sqrt(cfg.hidden_dim), device)


def chunk_kv(cfg, c: int, t: int, seed: int, device=None):
    """Chunk c's device store (K unrotated, V): bf16 [L][t][Hkv][dkp] each."""
    torch, device = _torch_on(device)
    lay = cfg.layout()
    L, Hkv, dk = cfg.n_layers, cfg.n_kv_heads, cfg.head_dim
    k = torch.zeros((L, t, Hkv, lay.dkp), dtype=torch.bfloat16, device=device)
    v = torch.zeros_like(k)
    for li in range(L):
        k[li, :, :, :dk] = normal_bf16((t, Hkv, dk), seed, tid_chunk(c, li, False), 1.0, device)
        v[li, :, :, :dk] = normal_bf16((t, Hkv, dk), seed, tid_chunk(c, li, True), 1.0, device)
    return k, v


def chunks(cfg, n_chunks: int, chunk_len: int, seed: int, fingerprint: str):
    """The synthetic request's chunk store as device ChunkKV objects."""
    from .chunkstore import ChunkKV
    out = []
    for c in range(n_chunks):
        k, v = chunk_kv(cfg, c, chunk_len, seed)
        ids = token_ids(chunk_len, cfg.vocab_size, seed, tid_tokens(c)).cpu().numpy()
        out.append(ChunkKV.from_device(c, fingerprint, ids, k, v, cfg.head_dim))
    return out


def query(cfg, m: int, seed: int):
    return token_ids(m, cfg.vocab_size, seed, TID_QUERY).cpu().numpy()
