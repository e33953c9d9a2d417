"""The rest of the reference surface on the device: finalize_query(capture_attn=True)
rows, query_pass / QueryPassResult over host K/V (reference model.py:362-402),
score_prophet(renormalize_context_only=True) (selection.py:80-84), the check_finite ->
NumericsError contract of Stage II (tensor.py:31-34), the reference-typed inputs (duck-typed
pikv.ModelWeights / pikv.ChunkKV objects) and host-tier (pinned) chunks under every
strategy."""

import types

import numpy as np
import pytest

from oracle import pikv_oracle as O

from test_gpu_parity import COS_MIN, KV_ABS, REL_TOL, _cos, _device_inputs, _materialise, _selection_ok, _setup

pytestmark = pytest.mark.gpu
ROWS_ABS = 1e-5  # attention probabilities (fp32-faithful narrow pass)


@pytest.mark.parametrize("case", ["c1", "llama_width"])
def test_finalize_capture_attn_rows(built, case):
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg)
    sel = P.select_top_p(P.score_prophet(mw, cfg, cache, query), p)
    P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    fin = P.finalize_query(mw, cfg, cache, query, capture_attn=True)
    cache_o = O.stitch(chunks, cfg_o)
    O.repair(w, cfg_o, cache_o, sel.indices)
    _, res = O.finalize(w, cfg_o, cache_o, query, want_rows=True)
    assert len(fin.rows) == cfg.n_layers
    for li in range(cfg.n_layers):
        got, ref = fin.rows[li], res.rows[li]
        assert got.shape == ref.shape == (len(query), cache.context_length + len(query))
        assert np.abs(got - ref).max() <= ROWS_ABS, (li, np.abs(got - ref).max())
        assert np.allclose(got.sum(axis=1), 1.0, atol=1e-5)


@pytest.mark.parametrize("case", ["tiny_ref", "c1"])
def test_query_pass_over_host_kv(built, case):
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, _ = _device_inputs(P, cfg_o, w, chunks)
    ctx = [t for u in units for t in u]
    tr = O.prefill(w, cfg_o, ctx)
    kv = list(zip(tr.keys, tr.values))
    pos = np.arange(len(ctx))
    tally = P.FlopTally()
    got = P.query_pass(mw, cfg, kv, pos, query, capture_attn=True, tally=tally)
    ref = O.narrow_pass(w, cfg_o, kv, pos, query, want_rows=True)
    assert isinstance(got, P.QueryPassResult)
    assert np.abs(got.last_logits - ref.last_logits).max() <= KV_ABS
    assert _cos(got.last_logits, ref.last_logits) >= COS_MIN
    # the given values are stored fp16 on the device (keys carry a residual plane): the
    # fresh K/V of layers > 0 see that rounding (~1e-4 relative)
    for li in range(cfg.n_layers):
        assert np.abs(got.fresh_keys[li] - ref.fresh_k[li]).max() <= 2e-3
        assert np.abs(got.fresh_values[li] - ref.fresh_v[li]).max() <= 2e-3
        assert np.abs(got.rows[li] - ref.rows[li]).max() <= 1e-4
    assert tally.total.multiply_accumulate_count == O.macs_query_pass(cfg_o, len(ctx), len(query))[0]
    # the reference keeps the given state unchanged; positions must be 0..t-1 on the device
    with pytest.raises(P.ConfigError):
        P.query_pass(mw, cfg, kv, pos + 5, query)
    empty = P.query_pass(mw, cfg, [(k[:0], v[:0]) for k, v in kv], pos[:0], query)
    ref0 = O.narrow_pass(w, cfg_o, [(k[:0], v[:0]) for k, v in kv], pos[:0], query)
    assert np.abs(empty.last_logits - ref0.last_logits).max() <= KV_ABS


@pytest.mark.parametrize("case", ["c1", "llama_width", "mistral_width"])
def test_renormalized_scores(built, case):
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg)
    sc = P.score_prophet(mw, cfg, cache, query, renormalize_context_only=True)
    per_ref, fused_ref = O.prophet_scores(w, cfg_o, O.stitch(chunks, cfg_o), query, renorm=True)
    rel = np.abs(sc.per_layer - per_ref) / np.maximum(np.abs(per_ref), 1e-30)
    assert rel.max() <= REL_TOL, rel.max()
    sel_ref, k = O.select(fused_ref, p)
    assert _selection_ok(P.select_top_p(sc, p).indices, sel_ref, fused_ref, k)


def test_stage2_non_finite_raises(built):
    """A NaN weight makes the reference's matmul check fail (NumericsError); the device
    Stage-II epilogues flag it and finalize_query raises."""
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    bad = P.ModelWeights(embed=mw.embed, layers=list(mw.layers), final_norm=mw.final_norm, lm_head=mw.lm_head)
    lw = bad.layers[1]
    wg = lw.w_gate.copy()
    wg[3, 5] = np.nan
    bad.layers[1] = P.LayerWeights(**{**lw.__dict__, "w_gate": wg})
    cache = P.assemble(dch, cfg)
    sel = P.select_top_p(P.ValueScores.from_vector("x", np.arange(cache.context_length)[::-1], 1), p)
    P.recompute_selected(bad, cfg, cache, P.RecomputePlan(sel))
    with pytest.raises(P.NumericsError):
        P.finalize_query(bad, cfg, cache, query)
    # the clean model on a fresh cache does not trip the flag
    cache = P.assemble(dch, cfg)
    P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    assert np.isfinite(P.finalize_query(mw, cfg, cache, query).first_logits).all()


def test_reference_typed_inputs(built):
    """Objects shaped like the reference's pikv.ModelWeights / pikv.ChunkKV (plain attribute
    bags, as a reference caller passes them) run through the drop-in unchanged."""
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    fp = mw.fingerprint(cfg)
    ref_w = types.SimpleNamespace(embed=w.embed, final_norm=w.final_norm, lm_head=w.lm_head,
                                  layers=[types.SimpleNamespace(**lw.__dict__) for lw in w.layers],
                                  fingerprint=lambda config: fp)
    ref_chunks = [types.SimpleNamespace(chunk_id=c.chunk_id, config_fingerprint=fp, token_ids=c.token_ids,
                                        keys_norope=c.k_nr, values=c.v) for c in chunks]
    outs = []
    for weights, cks in ((mw, dch), (ref_w, ref_chunks)):
        cache = P.assemble(cks, cfg)
        sel = P.select_top_p(P.score_prophet(weights, cfg, cache, query), p)
        P.recompute_selected(weights, cfg, cache, P.RecomputePlan(sel))
        outs.append((sel.indices, P.finalize_query(weights, cfg, cache, query).first_logits))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])
    # a second config on the same weights object gets its own device image
    cfg2 = P.ModelConfig(**{**cfg_o.json(), "rope_theta": 20000.0})
    assert P.model.resolve_device_model(ref_w, cfg2) is not P.model.resolve_device_model(ref_w, cfg)


@pytest.mark.parametrize("strategy", ["epic", "random", "cacheblend_l1", "prophet"])
def test_pinned_chunks_every_strategy(built, strategy):
    """Host-tier chunks (pinned, streamed per layer) give the device-resident result for
    every strategy -- including the ones whose scores do not wait on the transfer."""
    import torch
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    outs = []
    for pinned in (False, True):
        src = [P.ChunkKV.from_pinned(c.chunk_id, c.config_fingerprint, c.token_ids,
                                     c.device_buffers(cfg)[0].cpu().pin_memory(),
                                     c.device_buffers(cfg)[1].cpu().pin_memory(), cfg.head_dim)
               for c in dch] if pinned else dch
        run = P.run_strategy(mw, cfg, src, query, strategy, p, seed=3, max_new_tokens=3)
        torch.cuda.synchronize()
        outs.append((run.selection.indices, run.first_logits, run.record.answer_tokens))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
