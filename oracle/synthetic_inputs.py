"""Host (numpy) restatement of the SYN1 synthetic-input generator.

TEST INFRASTRUCTURE ONLY (like pikv_oracle.py): builds, on the CPU, exactly the weights,
chunk store and query that ``paper_2602_02579_b200/synthetic.py`` generates on the
device (the spec is in that module's docstring), so the oracle can check the bench's
own workload.  Bit-identity with the device generator is a test
(tests/test_synthetic_inputs.py on CPU vs the torch restatement, tests/test_gpu_anchor.py
on the device).
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import pikv_oracle as O

M32 = np.uint64(0xFFFFFFFF)
IH4_SD = 37837.22703
TID_EMBED, TID_HEAD, TID_QUERY = 0x0FFFFFF0, 0x0FFFFFF1, 0x30000000
LAYER_TIDS = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "w_gate": 4, "w_up": 5, "w_down": 6}


def tid_chunk(c, layer, is_value):
    return 0x10000000 + 2048 * c + 2 * layer + (1 if is_value else 0)


def tid_tokens(c):
    return 0x20000000 + c


def _mix32_int(x):
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    return x ^ (x >> 16)


def key(seed, tid):
    return _mix32_int((seed * 0x9E3779B1 + tid * 0x85EBCA77 + 0x165667B1) & 0xFFFFFFFF)


def _mix32(x):
    x = x ^ (x >> np.uint64(16))
    x = (x * np.uint64(0x7FEB352D)) & M32
    x = x ^ (x >> np.uint64(15))
    x = (x * np.uint64(0x846CA68B)) & M32
    return x ^ (x >> np.uint64(16))


def _u12(n, k, start):
    i = np.arange(start, start + n, dtype=np.uint64)
    u1 = _mix32(i ^ np.uint64(k))
    u2 = _mix32(u1 ^ np.uint64(0x68E31DA4))
    return u1, u2


_POOL = None


def normal_f32(shape, seed, tid, std, block=1 << 21):
    """float32 array (bf16-exact values) of the SYN1 stream (blocks on a thread pool:
    numpy releases the GIL inside the element-wise passes)."""
    global _POOL
    n = math.prod(shape)
    out = np.empty(n, dtype=np.float32)
    k = key(seed, tid)
    c = np.float32(std / IH4_SD)
    m16 = np.uint64(0xFFFF)

    def fill(s0):
        nb = min(block, n - s0)
        u1, u2 = _u12(nb, k, s0)
        z = ((u1 & m16) + (u1 >> np.uint64(16)) + (u2 & m16) + (u2 >> np.uint64(16))).astype(np.int64) - 131070
        out[s0:s0 + nb] = O.bf16_round(z.astype(np.float32) * c)

    starts = range(0, n, block)
    if n <= block:
        fill(0)
    else:
        if _POOL is None:
            from concurrent.futures import ThreadPoolExecutor
            _POOL = ThreadPoolExecutor(min(8, os.cpu_count() or 1))
        list(_POOL.map(fill, starts))
    return out.reshape(shape)


def token_ids(n, vocab, seed, tid):
    u1, _ = _u12(n, key(seed, tid), 0)
    return (u1 % np.uint64(vocab)).astype(np.int64)


def layer(cfg, li, seed):
    D, Q, KV, F = cfg.hidden_dim, cfg.n_heads * cfg.head_dim, cfg.kv_dim, cfg.ffn_dim
    shapes = {"wq": (D, Q), "wk": (D, KV), "wv": (D, KV), "wo": (Q, D), "w_gate": (D, F), "w_up": (D, F),
              "w_down": (F, D)}
    w = {name: normal_f32(shp, seed, 16 * li + LAYER_TIDS[name], 1.0 / math.sqrt(shp[0]))
         for name, shp in shapes.items()}
    ones = np.ones(D, np.float32)
    return O.Layer(attn_norm=ones, ffn_norm=ones.copy(), **w)


def weights(cfg, seed, layers=True):
    """O.Weights of the synthetic model (final / attention / ffn gains are ones)."""
    return O.Weights(embed=normal_f32((cfg.vocab_size, cfg.hidden_dim), seed, TID_EMBED, 1.0),
                     layers=[layer(cfg, li, seed) for li in range(cfg.n_layers)] if layers else [],
                     final_norm=np.ones(cfg.hidden_dim, np.float32),
                     lm_head=normal_f32((cfg.hidden_dim, cfg.vocab_size), seed, TID_HEAD,
                                        1.0 / math.sqrt(cfg.hidden_dim)))


def chunk_layer(cfg, c, t, li, seed):
    """(K_nr, V) f32 [t, Hkv, dk] of chunk c at layer li."""
    shp = (t, cfg.n_kv_heads, cfg.head_dim)
    return normal_f32(shp, seed, tid_chunk(c, li, False), 1.0), normal_f32(shp, seed, tid_chunk(c, li, True), 1.0)


def chunks(cfg, n_chunks, t, seed, fp="syn1"):
    out = []
    for c in range(n_chunks):
        kv = [chunk_layer(cfg, c, t, li, seed) for li in range(cfg.n_layers)]
        out.append(O.Chunk(chunk_id=c, fp=fp, token_ids=token_ids(t, cfg.vocab_size, seed, tid_tokens(c)),
                           k_nr=[a for a, _ in kv], v=[b for _, b in kv]))
    return out


def query(cfg, m, seed):
    return token_ids(m, cfg.vocab_size, seed, TID_QUERY)
