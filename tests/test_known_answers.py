"""Known-answer tests of the reference's own suite, applied to the oracle and to the
host-side drop-in API (reference tests/test_tensor.py, test_model.py)."""

import hashlib
import math

import numpy as np
import pytest

import paper_2602_02579_b200 as P
from oracle import pikv_oracle as O

TOKENS12 = [3, 17, 42, 0, 9, 31, 25, 7, 49, 13, 2, 38]
GOLDEN_LOGITS_DIGEST = "0977fbe50bbb2e0d"  # reference tests/test_model.py:18-22


def straight_line_forward(w, cfg, tokens):
    """Independent per-token float64 forward (same algorithm as the reference's
    test oracle ref_forward, tests/test_model.py:36-75), written from scratch."""
    x = w.embed[np.asarray(tokens)].astype(np.float64)
    n, grp, d = len(tokens), cfg.n_heads // cfg.n_kv_heads, cfg.head_dim

    def rot(vec, pos):
        out = np.array(vec, dtype=np.float64)
        for i in range(d // 2):
            ang = pos * cfg.rope_theta ** (-2.0 * i / d)
            c, s = math.cos(ang), math.sin(ang)
            a, b = out[2 * i], out[2 * i + 1]
            out[2 * i], out[2 * i + 1] = a * c - b * s, a * s + b * c
        return out

    def norm(v, g):
        return v / math.sqrt(float(np.mean(v * v)) + cfg.norm_eps) * g.astype(np.float64)

    for lw in w.layers:
        hn = np.stack([norm(x[i], lw.attn_norm) for i in range(n)])
        q, k, v = hn @ lw.wq.astype(np.float64), hn @ lw.wk.astype(np.float64), hn @ lw.wv.astype(np.float64)
        att = np.zeros((n, cfg.n_heads * d))
        for i in range(n):
            for hd in range(cfg.n_heads):
                gk = hd // grp
                qi = rot(q[i, hd * d:(hd + 1) * d], i)
                sc = [float(qi @ rot(k[j, gk * d:(gk + 1) * d], j)) / math.sqrt(d) for j in range(i + 1)]
                e = np.exp(np.array(sc) - max(sc))
                e /= e.sum()
                att[i, hd * d:(hd + 1) * d] = sum(e[j] * v[j, gk * d:(gk + 1) * d] for j in range(i + 1))
        x = x + att @ lw.wo.astype(np.float64)
        hn = np.stack([norm(x[i], lw.ffn_norm) for i in range(n)])
        gt, up = hn @ lw.w_gate.astype(np.float64), hn @ lw.w_up.astype(np.float64)
        x = x + (gt / (1 + np.exp(-gt)) * up) @ lw.w_down.astype(np.float64)
    hn = np.stack([norm(x[i], w.final_norm) for i in range(n)])
    return hn @ w.lm_head.astype(np.float64)


def test_golden_logits_digest_and_oracle_prefill():
    cfg = O.Cfg(n_layers=2, n_heads=2, n_kv_heads=1, head_dim=4, hidden_dim=8, ffn_dim=16, vocab_size=50)
    w = O.init_weights(cfg, 42)
    want = straight_line_forward(w, cfg, TOKENS12)
    assert hashlib.blake2b(np.round(want, 4).tobytes(), digest_size=8).hexdigest() == GOLDEN_LOGITS_DIGEST
    got = O.prefill(w, cfg, TOKENS12).logits
    np.testing.assert_allclose(got, want, atol=1e-4)


def test_rope_known_answers():
    x = np.zeros((1, 1, 4), np.float32)
    x[0, 0, :2] = 1.0, 2.0
    got = O.rope(x, [3], 10000.0)
    c, s = math.cos(3.0), math.sin(3.0)
    np.testing.assert_allclose(got[0, 0, :2], [c - 2 * s, s + 2 * c], atol=1e-6)
    rng = np.random.default_rng(3)
    y = rng.standard_normal((1, 2, 8)).astype(np.float32)
    assert np.array_equal(O.rope(y, [0], 10000.0), y)
    np.testing.assert_allclose(O.rope(O.rope(y, [5], 1e4), [-5], 1e4), y, atol=1e-5)


def test_top_k_ties_and_budget_known_answers():
    for topk in (O.topk_ascending,):
        assert topk([5.0, 5.0, 1.0], 1) == [0]
        assert topk([1.0, 5.0, 5.0], 1) == [1]
        assert topk([2.0, 2.0, 2.0], 2) == [0, 1]
        assert topk([0.1, 9.0, 3.0, 9.0, -2.0], 3) == [1, 2, 3]
    for budget in (O.budget, P.ratio_budget):
        assert budget(0.0, 100) == 0 and budget(1.0, 100) == 100
        assert budget(0.02, 100) == 2 and budget(0.021, 100) == 3
        assert budget(0.5, 7) == 4 and budget(0.2, 1) == 1
        assert budget(0.07, 100) == 8  # 0.07*100 == 7.000000000000001 in double
    with pytest.raises(P.ArgumentError):
        P.ratio_budget(1.01, 10)


def test_drop_in_host_types_match_oracle():
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, hidden_dim=32, ffn_dim=64, vocab_size=50)
    cfg_o = O.Cfg(**cfg.to_json_dict())
    w, wo = P.random_weights(cfg, 11), O.init_weights(cfg_o, 11)
    for (na, a), (nb, b) in zip(w.named_tensors(), wo.tensors()):
        assert na == nb and np.array_equal(a, b)
    assert w.fingerprint(cfg) == wo.fingerprint(cfg_o)
    # from_named round trip (reference model.py:124-145)
    named = dict(w.named_tensors())
    w2 = P.ModelWeights.from_named(cfg, named)
    assert w2.fingerprint(cfg) == w.fingerprint(cfg)
    with pytest.raises(P.ConfigError):
        P.ModelWeights.from_named(cfg, {k: v for k, v in named.items() if k != "layers.1.attn.wv"})
    with pytest.raises(P.ConfigError):
        P.ModelWeights.from_named(cfg, {**named, "lm_head.weight": named["lm_head.weight"][:, :7]})
    with pytest.raises(P.ConfigError):
        P.ModelConfig(n_layers=1, n_heads=3, n_kv_heads=2, head_dim=4, hidden_dim=12, ffn_dim=8, vocab_size=5)
    with pytest.raises(P.ConfigError):
        P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=3, hidden_dim=6, ffn_dim=8, vocab_size=5)


def test_value_scores_contract():
    per = np.array([[1.0, 2.0], [3.0, 4.0]], dtype=np.float32)
    P.ValueScores("x", per, np.array([2.0, 3.0], dtype=np.float32))
    with pytest.raises(P.ArgumentError):
        P.ValueScores("x", per, np.array([1.0, 4.0], dtype=np.float32))
    vs = P.ValueScores.from_vector("x", [1.0, 5.0, 2.0], 3)
    assert vs.per_layer.shape == (3, 3)


@pytest.mark.parametrize("s,m,k", [(15, 4, 5), (2048, 32, 410), (32768, 32, 6554)])
def test_mac_books_match_oracle_formulas(s, m, k):
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, hidden_dim=32, ffn_dim=64, vocab_size=50)
    cfg_o = O.Cfg(**cfg.to_json_dict())
    t = P.FlopTally()
    P.model.bill_query_pass(t, cfg, s, m)
    assert (t.total.multiply_accumulate_count, t.attn_scores.multiply_accumulate_count) == \
        O.macs_query_pass(cfg_o, s, m)
    t = P.FlopTally()
    P.model.bill_repair(t, cfg, s, k)
    assert (t.total.multiply_accumulate_count, t.attn_scores.multiply_accumulate_count) == O.macs_repair(cfg_o, s, k)
