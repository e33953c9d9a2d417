"""Oracle vs the real reference package, bit for bit (runs only where the
reference is importable, i.e. the build container)."""

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import pikv_oracle as O

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not mounted")


@pytest.fixture(scope="module")
def pikv():
    sys.path.insert(0, str(REF))
    import pikv as P
    return P


CFGS = [dict(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, hidden_dim=32, ffn_dim=64, vocab_size=50),
        dict(n_layers=3, n_heads=4, n_kv_heads=1, head_dim=6, hidden_dim=24, ffn_dim=40, vocab_size=37,
             rope_theta=5e5),
        dict(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=4, hidden_dim=8, ffn_dim=16, vocab_size=20)]


@pytest.mark.parametrize("ci", range(len(CFGS)))
@pytest.mark.parametrize("p", [0.0, 0.07, 0.3, 1.0])
def test_slice_bit_identical(pikv, ci, p):
    cfg_r = pikv.ModelConfig(**CFGS[ci])
    cfg_o = O.Cfg(**cfg_r.to_json_dict())
    wr, wo = pikv.random_weights(cfg_r, 3 + ci), O.init_weights(cfg_o, 3 + ci)
    assert wr.fingerprint(cfg_r) == wo.fingerprint(cfg_o)
    rng = np.random.default_rng(ci)
    units = [rng.integers(0, cfg_r.vocab_size, int(rng.integers(3, 9))).tolist() for _ in range(3)]
    query = rng.integers(0, cfg_r.vocab_size, 4).tolist()
    cr = [pikv.precompute_chunk(wr, cfg_r, u) for u in units]
    co = [O.make_chunk(wo, cfg_o, u) for u in units]
    for a, b in zip(cr, co):
        assert a.chunk_id == b.chunk_id
    car, cao = pikv.assemble(cr, cfg_r), O.stitch(co, cfg_o)
    for li in range(cfg_r.n_layers):
        assert np.array_equal(car.keys_rebased[li], cao.keys[li])
    for renorm in (False, True):
        sr = pikv.score_prophet(wr, cfg_r, car, query, renormalize_context_only=renorm)
        per, fused = O.prophet_scores(wo, cfg_o, cao, query, renorm=renorm)
        assert np.array_equal(sr.per_layer, per) and np.array_equal(sr.fused, fused)
    sr = pikv.score_prophet(wr, cfg_r, car, query)
    sel = pikv.select_top_p(sr, p)
    so, k = O.select(O.prophet_scores(wo, cfg_o, cao, query)[1], p)
    assert sel.indices == so and sel.k == k
    tr, to = pikv.FlopTally(), [0]
    pikv.recompute_selected(wr, cfg_r, car, pikv.RecomputePlan(sel), tally=tr)
    O.repair(wo, cfg_o, cao, so)
    assert tr.total.multiply_accumulate_count == O.macs_repair(cfg_o, car.context_length, k)[0]
    for li in range(cfg_r.n_layers):
        assert np.array_equal(car.keys_rebased[li], cao.keys[li])
        assert np.array_equal(car.values[li], cao.values[li])
    fr = pikv.finalize_query(wr, cfg_r, car, query)
    lo, _ = O.finalize(wo, cfg_o, cao, query)
    assert np.array_equal(fr.first_logits, lo)


def test_query_pass_books(pikv):
    cfg_r = pikv.ModelConfig(**CFGS[0])
    cfg_o = O.Cfg(**cfg_r.to_json_dict())
    wr = pikv.random_weights(cfg_r, 1)
    cr = [pikv.precompute_chunk(wr, cfg_r, u) for u in ([1, 2, 3, 4], [5, 6, 7])]
    for m in (1, 4):
        t = pikv.FlopTally()
        pikv.score_prophet(wr, cfg_r, pikv.assemble(cr, cfg_r), list(range(m)), tally=t)
        assert (t.total.multiply_accumulate_count, t.attn_scores.multiply_accumulate_count) == \
            O.macs_query_pass(cfg_o, 7, m)


def test_top_k_and_budget_match(pikv):
    from pikv.tensor import ratio_budget, top_k_indices
    rng = np.random.default_rng(9)
    for _ in range(200):
        n = int(rng.integers(1, 60))
        v = (rng.integers(-3, 4, n) / 3).astype(np.float32)
        k = int(rng.integers(0, n + 1))
        assert top_k_indices(v, k) == O.topk_ascending(v, k)
        p = float(rng.random())
        assert ratio_budget(p, n) == O.budget(p, n)


@pytest.mark.parametrize("ci", range(len(CFGS)))
def test_decode_and_full_prefill_bit_identical(pikv, ci):
    """The oracle's teacher-forced decode (used by tests/test_gpu_decode.py) and prefill
    reproduce the reference's decode_step / full_prefill bit for bit."""
    cfg_r = pikv.ModelConfig(**CFGS[ci])
    cfg_o = O.Cfg(**cfg_r.to_json_dict())
    wr, wo = pikv.random_weights(cfg_r, 5 + ci), O.init_weights(cfg_o, 5 + ci)
    rng = np.random.default_rng(ci)
    toks = rng.integers(0, cfg_r.vocab_size, 9).tolist()
    tr = pikv.full_prefill(wr, cfg_r, toks)
    to = O.prefill(wo, cfg_o, toks)
    assert np.array_equal(tr.logits, to.logits)
    for li in range(cfg_r.n_layers):
        assert np.array_equal(tr.keys[li], to.keys[li]) and np.array_equal(tr.values[li], to.values[li])
    cache = pikv.KVCache.from_prefill(tr)
    steps = [3, 1, 4]
    ref = []
    for i, t in enumerate(steps):
        lg, cache = pikv.decode_step(wr, cfg_r, cache, t, len(toks) + i)
        ref.append(lg)
    got = O.decode(wo, cfg_o, list(zip(to.keys, to.values)), np.arange(len(toks)), steps)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("ci", range(len(CFGS)))
def test_probe_baselines_bit_identical(pikv, ci):
    """The oracle's low-layer probe scores (cacheblend_l1 / kvshare_l1) and their MAC books
    reproduce the reference's selection.py:95-142."""
    cfg_r = pikv.ModelConfig(**CFGS[ci])
    cfg_o = O.Cfg(**cfg_r.to_json_dict())
    wr, wo = pikv.random_weights(cfg_r, 7 + ci), O.init_weights(cfg_o, 7 + ci)
    rng = np.random.default_rng(10 + ci)
    units = [rng.integers(0, cfg_r.vocab_size, int(rng.integers(3, 9))).tolist() for _ in range(3)]
    car = pikv.assemble([pikv.precompute_chunk(wr, cfg_r, u) for u in units], cfg_r)
    cao = O.stitch([O.make_chunk(wo, cfg_o, u) for u in units], cfg_o)
    for name, fn in (("score_cacheblend_l1", O.cacheblend_l1), ("score_kvshare_l1", O.kvshare_l1)):
        tr = pikv.FlopTally()
        ref = getattr(pikv.selection, name)(wr, cfg_r, car, tally=tr)
        macs = [0]
        got = fn(wo, cfg_o, cao, macs=macs)
        assert np.array_equal(ref.fused, got), name
        assert tr.total.multiply_accumulate_count == macs[0] == O.macs_probe(cfg_o, car.context_length)
