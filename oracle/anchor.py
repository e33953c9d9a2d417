"""Layer-streamed oracle run of the ProphetKV slice at full model scale.

TEST INFRASTRUCTURE ONLY.  ``pikv_oracle.prophet_ttft_slice`` keeps every layer's
weights, chunk store and cache resident (f32): at the Llama-3-8B / 32k target that is
~50 GB plus a dense [k, s] f64 score matrix per head.  This module runs the SAME
arithmetic -- it calls pikv_oracle's primitives (rmsnorm, qkv_proj, block_tail's mix,
masked_softmax64, mm) in the reference's order -- but streams one layer at a time:

* inputs are the SYN1 synthetic weights / chunk store (oracle/synthetic_inputs.py),
  regenerated per layer (counter-based, so any layer or embedding row is addressable);
* Stage-II attention (reference model.py:278-308 inside recompute.py:80-81) is evaluated
  per (head, block of selected rows) on a thread pool; a softmax row depends only on its
  own scores, so the blocks reproduce the unblocked rows (checked against the unblocked
  oracle in tests/test_anchor_oracle.py);
* only the selected rows' fresh K/V are kept between the repair and the final pass.

Outputs the reference-side numbers the GPU run is checked against (tests/golden/
make_anchor.py writes them as fixtures).
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import pikv_oracle as O
from . import synthetic_inputs as SO

f32, f64 = np.float32, np.float64


class SynRequest:
    """The synthetic request: config, seed, chunk geometry, query length."""

    def __init__(self, cfg, seed, n_chunks, chunk_len, m):
        self.cfg, self.seed, self.n_chunks, self.chunk_len, self.m = cfg, seed, n_chunks, chunk_len, m
        self.s = n_chunks * chunk_len
        self.positions = np.arange(self.s, dtype=np.int64)
        self.token_ids = np.concatenate([SO.token_ids(chunk_len, cfg.vocab_size, seed, SO.tid_tokens(c))
                                         for c in range(n_chunks)])
        self.query = SO.query(cfg, m, seed)

    def layer(self, li):
        return SO.layer(self.cfg, li, self.seed)

    def embed_rows(self, ids):
        """Rows of the SYN1 embedding (element index = row * D + col)."""
        D = self.cfg.hidden_dim
        k = SO.key(self.seed, SO.TID_EMBED)
        c = f32(1.0 / SO.IH4_SD)
        idx = (np.asarray(ids, dtype=np.uint64)[:, None] * np.uint64(D) + np.arange(D, dtype=np.uint64)[None, :])
        u1 = SO._mix32(idx ^ np.uint64(k))
        u2 = SO._mix32(u1 ^ np.uint64(0x68E31DA4))
        m16 = np.uint64(0xFFFF)
        z = ((u1 & m16) + (u1 >> np.uint64(16)) + (u2 & m16) + (u2 >> np.uint64(16))).astype(np.int64) - 131070
        return O.bf16_round(z.astype(f32) * c)

    def cache_layer(self, li):
        """Assembled layer li (chunkstore.py:123-127): rotated keys, values [s, Hkv, dk] f32."""
        kv = [SO.chunk_layer(self.cfg, c, self.chunk_len, li, self.seed) for c in range(self.n_chunks)]
        K = O.rope(np.concatenate([a for a, _ in kv], axis=0), self.positions, self.cfg.rope_theta)
        V = np.concatenate([b for _, b in kv], axis=0)
        return K, V


def _mix(lw, cfg, h, a):
    """block_tail's residual + SiLU FFN (model.py:311-323), the oracle's exact ops."""
    h = h + O.mm(a, lw.wo)
    y = O.rmsnorm(h, lw.ffn_norm, cfg.norm_eps)
    g = O.silu(O.mm(y, lw.w_gate))
    u = O.mm(y, lw.w_up)
    return h + O.mm(g * u, lw.w_down)


def attention_blocked(cfg, qr, K, V, pos_q, pos_kv, rows=256, threads=8):
    """O.attention without the head-mean rows, per (head, row block) on a thread pool."""
    n, H, dk = qr.shape
    grp = H // cfg.n_kv_heads
    scl = f32(1.0 / np.sqrt(dk))
    out = np.empty((n, H, dk), dtype=f32)
    Kt = [np.ascontiguousarray(K[:, g, :].T) for g in range(cfg.n_kv_heads)]
    Vg = [np.ascontiguousarray(V[:, g, :]) for g in range(cfg.n_kv_heads)]

    def unit(args):
        h, r0 = args
        r1 = min(n, r0 + rows)
        g = h // grp
        vis = pos_kv[None, :] <= pos_q[r0:r1, None]
        sc = O.mm(np.ascontiguousarray(qr[r0:r1, h, :]), Kt[g]) * scl
        p = O.masked_softmax64(sc, vis)
        out[r0:r1, h, :] = O.mm(p, Vg[g])

    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(1)
    except ImportError:
        limit = None
    try:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(unit, [(h, r0) for h in range(H) for r0 in range(0, n, rows)]))
    finally:
        if limit is not None:
            limit.restore_original_limits()
    return out.reshape(n, H * dk)


def narrow_layer(req, lw, li, h, K, V, want_rows):
    """One layer of query_pass (model.py:384-398) for the m query tokens."""
    cfg, m, s = req.cfg, req.m, req.s
    pq = s + np.arange(m, dtype=np.int64)
    pall = np.concatenate([req.positions, pq])
    x = O.rmsnorm(h, lw.attn_norm, cfg.norm_eps)
    qr, _, kr, v = O.qkv_proj(lw, cfg, x, pq, None)
    return O.block_tail(lw, cfg, h, qr, np.concatenate([K, kr], axis=0), np.concatenate([V, v], axis=0), pq, pall,
                        None, None, want_rows)


def run(req, p, kv_rows=None, log=print, threads=8, stage1_only=False):
    """assemble -> score_prophet -> select_top_p -> recompute_selected -> finalize_query.

    Returns dict(per_layer [L,s], fused [s], sel, k, first_logits [V], kv_k/kv_v
    [L][len(kv_rows)][Hkv][dk] fresh K/V of the selected rows kv_rows (indices into sel))."""
    cfg, s, L = req.cfg, req.s, req.cfg.n_layers
    t0 = time.time()
    # ---- Stage I (selection.py:64-86): the narrow pass with captured rows
    h = req.embed_rows(req.query)
    per = np.empty((L, s), dtype=f32)
    for li in range(L):
        lw = req.layer(li)
        K, V = req.cache_layer(li)
        h, rows = narrow_layer(req, lw, li, h, K, V, True)
        per[li] = rows[:, :s].astype(f64).mean(axis=0).astype(f32)
        log(f"[anchor] stage I layer {li} ({time.time() - t0:.0f}s)")
    fused = O.layer_mean(per)
    sel, k = O.select(fused, p)
    out = {"per_layer": per, "fused": fused, "sel": np.asarray(sel, dtype=np.int64), "k": k}
    if stage1_only:
        return out
    # ---- Stage II (recompute.py:43-82): write the fresh K/V first, then attend
    ix = out["sel"]
    ps = req.positions[ix]
    h = req.embed_rows(req.token_ids[ix])
    fresh = []
    kv_rows = np.arange(len(ix)) if kv_rows is None else np.asarray(kv_rows)
    kk, vv = [], []
    for li in range(L):
        lw = req.layer(li)
        K, V = req.cache_layer(li)
        x = O.rmsnorm(h, lw.attn_norm, cfg.norm_eps)
        qr, _, kr, v = O.qkv_proj(lw, cfg, x, ps, None)
        K[ix], V[ix] = kr, v
        fresh.append((kr, v))
        kk.append(kr[kv_rows])
        vv.append(v[kv_rows])
        if li < L - 1:  # the last layer's attention / MLP only feed the dropped residual
            a = attention_blocked(cfg, qr, K, V, ps, req.positions, threads=threads)
            h = _mix(lw, cfg, h, a)
        log(f"[anchor] stage II layer {li} ({time.time() - t0:.0f}s)")
    out["kv_k"], out["kv_v"], out["kv_rows"] = np.stack(kk), np.stack(vv), kv_rows
    # ---- finalize_query (recompute.py:105-125): the narrow pass over the repaired cache
    h = req.embed_rows(req.query)
    for li in range(L):
        lw = req.layer(li)
        K, V = req.cache_layer(li)
        K[ix], V[ix] = fresh[li]
        h, _ = narrow_layer(req, lw, li, h, K, V, False)
        log(f"[anchor] final layer {li} ({time.time() - t0:.0f}s)")
    lm_head = SO.normal_f32((cfg.hidden_dim, cfg.vocab_size), req.seed, SO.TID_HEAD, 1.0 / np.sqrt(cfg.hidden_dim))
    w_head = O.Weights(embed=None, layers=[], final_norm=np.ones(cfg.hidden_dim, f32), lm_head=lm_head)
    out["first_logits"] = O.logits_of(w_head, cfg, h, None)[-1]
    return out
