"""The layer-streamed oracle (oracle/anchor.py, used for the full-scale fixtures) is the
same computation as the oracle's resident slice (pikv_oracle.prophet_ttft_slice, pinned
to the reference) on the SYN1 inputs: bit-identical scores, selection, repaired K/V and
first logits, including the row-blocked Stage-II attention."""

import numpy as np

from oracle import anchor as A
from oracle import pikv_oracle as O
from oracle import synthetic_inputs as SO


def test_streamed_anchor_equals_resident_oracle():
    cfg = O.Cfg(3, 4, 2, 16, 64, 128, 97, rope_theta=500000.0)
    req = A.SynRequest(cfg, seed=3, n_chunks=3, chunk_len=100, m=7)
    got = A.run(req, 0.25, log=lambda *_: None, threads=3)
    w = SO.weights(cfg, 3)
    chunks = SO.chunks(cfg, 3, 100, 3)
    ref = O.prophet_ttft_slice(w, cfg, chunks, req.query.tolist(), 0.25)
    assert np.array_equal(got["per_layer"], ref["per_layer"])
    assert list(got["sel"]) == ref["sel"]
    for li in range(cfg.n_layers):
        assert np.array_equal(got["kv_k"][li], ref["fresh"]["k"][li])
        assert np.array_equal(got["kv_v"][li], ref["fresh"]["v"][li])
    assert np.array_equal(got["first_logits"], ref["first_logits"])


def test_blocked_attention_rows_equal_unblocked():
    rng = np.random.default_rng(0)
    cfg = O.Cfg(1, 4, 2, 32, 128, 64, 50)
    n, t = 300, 700
    qr = rng.standard_normal((n, 4, 32)).astype(np.float32)
    K = rng.standard_normal((t, 2, 32)).astype(np.float32)
    V = rng.standard_normal((t, 2, 32)).astype(np.float32)
    pos_q = np.sort(rng.choice(t, n, replace=False)).astype(np.int64)
    pos_kv = np.arange(t, dtype=np.int64)
    ref, _ = O.attention(cfg, qr, K, V, pos_q, pos_kv, None, None, False)
    got = A.attention_blocked(cfg, qr, K, V, pos_q, pos_kv, rows=37, threads=4)
    assert np.array_equal(got, ref)
