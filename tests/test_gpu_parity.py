"""End-to-end parity of the B200 path against the CPU oracle on identical inputs.

Contract:
  * fused scores: relative error <= 1e-4 (observed ~1e-6), per-layer likewise;
  * selection: |S_gpu| = k and S_gpu \\ B == S_ref \\ B, where B is the tie band
    {t : |f_ref(t) - kth| <= 1e-4 * kth}; inside the band the reference's own rule
    (equal f32 -> smaller index) decides, which the device applies bit-exactly to
    its own fused vector;
  * recomputed K/V (fp32 tap, before fp16 storage) and first-token logits:
    max abs <= 2e-2 and cosine >= 0.999, with the oracle run on the GPU's
    selection so selection and recompute parity decouple.
Inputs are bf16-exact (weights and chunk K/V rounded once, shared by both sides).
Full-depth / full-context cases on the bench's own inputs: tests/test_gpu_anchor.py.
"""

import numpy as np
import pytest

from oracle import pikv_oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
KV_ABS, COS_MIN = 2e-2, 0.999


def _setup(cfg_o, seed, units, query):
    w = O.init_weights(cfg_o, seed).rounded_bf16()
    chunks = []
    for u in units:
        c = O.make_chunk(w, cfg_o, u)
        c.k_nr = [O.bf16_round(x) for x in c.k_nr]
        c.v = [O.bf16_round(x) for x in c.v]
        chunks.append(c)
    return w, chunks


def _device_inputs(P, cfg_o, w, chunks):
    cfg = P.ModelConfig(**cfg_o.json())
    mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{k: getattr(lw, k) for k in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
        final_norm=w.final_norm, lm_head=w.lm_head)
    fp = mw.fingerprint(cfg)
    dch = [P.ChunkKV(c.chunk_id, fp, c.token_ids, c.k_nr, c.v) for c in chunks]
    return cfg, mw, dch


def _cos(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-300))


def _report(**kw):
    """Append measured parity numbers (DESIGN.md quotes them) to a JSONL report."""
    import json
    import os
    path = os.environ.get("PKV_PARITY_REPORT", "gpurun_out/parity_report.jsonl")
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        kw["s1_path"] = "simt" if os.environ.get("PKV_S1_SIMT") else "tcgen05-split3"
        with open(path, "a") as f:
            f.write(json.dumps({k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in kw.items()})
                    + "\n")
    except OSError:
        pass


def _selection_ok(sel_gpu, sel_ref, fused_ref, k):
    kth = np.sort(fused_ref)[::-1][k - 1] if k else 0.0
    band = np.abs(fused_ref - kth) <= REL_TOL * abs(kth)
    a, b = set(sel_gpu), set(sel_ref)
    return len(a) == k and {i for i in a if not band[i]} == {i for i in b if not band[i]}


CASES = {
    # reference test fixture tiny_cfg (conftest.py:17-20) with test_recompute UNITS/QUERY
    "tiny_ref": (O.Cfg(2, 2, 1, 4, 8, 16, 50), 42, [[3, 17, 42, 0, 9, 31], [25, 7, 49, 13], [2, 38, 11, 29, 6]],
                 [8, 19, 44, 1], 0.3),
    # BASELINE configs[0] (C1): L2 D256 H4 Hkv2 dk64 F1024 V1024, 8 x 256 + 32-token query
    "c1": (O.Cfg(2, 4, 2, 64, 256, 1024, 1024), 0, "8x256", 32, 0.2),
    # Llama-3-8B layer width, 2 layers, 8 x 256 context
    "llama_width": (O.Cfg(2, 32, 8, 128, 4096, 14336, 2048, rope_theta=500000.0), 0, "8x256", 32, 0.2),
    # BASELINE configs[3]: the recompute-ratio sweep end points (C1 shape)
    "c1_p05": (O.Cfg(2, 4, 2, 64, 256, 1024, 1024), 0, "8x256", 32, 0.05),
    "c1_p40": (O.Cfg(2, 4, 2, 64, 256, 1024, 1024), 0, "8x256", 32, 0.4),
    # configs[1] geometry: Mistral-7B layer width, theta 1e6, ragged chunks
    "mistral_width": (O.Cfg(2, 32, 8, 128, 4096, 14336, 2048, rope_theta=1000000.0), 3, "ragged", 24, 0.1),
    # edge cases: one chunk with a one-token query; a query longer than the 32-row narrow
    # tile (unfused projection path); four layers with odd chunk lengths
    "c1_single_m1": (O.Cfg(2, 4, 2, 64, 256, 1024, 1024), 5, "1x200", 1, 0.5),
    "c1_m40": (O.Cfg(2, 4, 2, 64, 256, 1024, 1024), 6, "4x128", 40, 0.2),
    "tiny_deep": (O.Cfg(4, 4, 2, 16, 64, 128, 256), 7, "5x37", 7, 0.25),
    # full depth: C1 width with the 32 layers of the target models (Llama width at 32 layers
    # and the 32k target itself: tests/test_gpu_anchor.py)
    "c1_deep32": (O.Cfg(32, 4, 2, 64, 256, 1024, 1024), 9, "8x256", 32, 0.2),
}


def _materialise(case):
    cfg_o, seed, units, query, p = CASES[case]
    rng = np.random.default_rng(1000 + seed)
    if units == "ragged":  # uneven chunk lengths (not multiples of the 64/128-token tiles)
        units = [rng.integers(0, cfg_o.vocab_size, t).tolist() for t in (300, 77, 513, 129, 255)]
    elif isinstance(units, str):
        n, t = map(int, units.split("x"))
        units = [rng.integers(0, cfg_o.vocab_size, t).tolist() for _ in range(n)]
    if isinstance(query, int):
        query = rng.integers(0, cfg_o.vocab_size, query).tolist()
    return cfg_o, seed, units, query, p


@pytest.mark.parametrize("case", list(CASES))
def test_prophet_slice_matches_oracle(built, case):
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cache_o = O.stitch(chunks, cfg_o)
    per_ref, fused_ref = O.prophet_scores(w, cfg_o, cache_o, query)
    sel_ref, k = O.select(fused_ref, p)

    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, fp32_taps=True)
    scores = P.score_prophet(mw, cfg, cache, query)
    rel = np.abs(scores.per_layer - per_ref) / np.maximum(np.abs(per_ref), 1e-30)
    frel = np.abs(scores.fused - fused_ref) / np.maximum(np.abs(fused_ref), 1e-30)
    sel = P.select_top_p(scores, p)
    kth = np.sort(fused_ref)[::-1][k - 1] if k else 0.0
    band = int(np.sum(np.abs(fused_ref - kth) <= REL_TOL * abs(kth)))
    sym = len(set(sel.indices) ^ set(sel_ref))
    assert rel.max() <= REL_TOL, f"per-layer score rel err {rel.max():.3e}"
    assert sel.k == k
    assert _selection_ok(sel.indices, sel_ref, fused_ref, k)
    # on identical fused input the device top-k is the reference rule, bit for bit
    assert P.top_k_indices(scores.fused, k) == O.topk_ascending(scores.fused, k)

    P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    fin = P.finalize_query(mw, cfg, cache, query)

    cap = {}
    O.repair(w, cfg_o, cache_o, sel.indices, capture=cap)
    lg_ref, _ = O.finalize(w, cfg_o, cache_o, query)
    ix = np.asarray(sel.indices)
    kv_err, kv_cos = 0.0, 1.0
    for li in range(cfg_o.n_layers):
        gk = cache.keys_rebased[li][ix]
        gv = cache.values[li][ix]
        kv_err = max(kv_err, np.abs(gk - cap["k"][li]).max(), np.abs(gv - cap["v"][li]).max())
        kv_cos = min(kv_cos, _cos(gk, cap["k"][li]), _cos(gv, cap["v"][li]))
        assert np.abs(gk - cap["k"][li]).max() <= KV_ABS and _cos(gk, cap["k"][li]) >= COS_MIN, li
        assert np.abs(gv - cap["v"][li]).max() <= KV_ABS and _cos(gv, cap["v"][li]) >= COS_MIN, li
        # untouched entries keep the exact assembled keys
        rest = np.setdiff1d(np.arange(cache.context_length), ix)
        assert np.array_equal(cache.keys_rebased[li][rest], cache_o.keys[li][rest])
    err = np.abs(fin.first_logits - lg_ref).max()
    _report(case=case, s=cache.context_length, k=k, per_layer_max_rel=rel.max(), fused_max_rel=frel.max(),
            tie_band=band, sel_symdiff=sym, kv_max_abs=kv_err, kv_min_cos=kv_cos, logits_max_abs=err,
            logits_cos=_cos(fin.first_logits, lg_ref))
    assert err <= KV_ABS and _cos(fin.first_logits, lg_ref) >= COS_MIN, err
    assert cache.recomputed[:, ix].all() and cache.recomputed.sum() == cfg_o.n_layers * len(ix)


def test_full_budget_repair_reproduces_joint_forward(built):
    """p = 1: the repaired cache equals a full prefill (reference test_recompute.py:29-38)."""
    P = built
    cfg_o, seed, units, query, _ = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, fp32_taps=True)
    scores = P.ValueScores.from_vector("x", np.arange(cache.context_length)[::-1], 1)
    sel = P.select_top_p(scores, 1.0)
    P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    ctx = [t for u in units for t in u]
    trace = O.prefill(w, cfg_o, ctx)
    for li in range(cfg_o.n_layers):
        assert np.abs(cache.keys_rebased[li] - trace.keys[li]).max() <= KV_ABS
        assert np.abs(cache.values[li] - trace.values[li]).max() <= KV_ABS
    assert cache.recomputed.all()
    fin = P.finalize_query(mw, cfg, cache, query)
    full = O.prefill(w, cfg_o, ctx + list(query))
    assert np.abs(fin.first_logits - full.logits[-1]).max() <= KV_ABS


def test_pinned_host_chunks_pipeline_is_identical(built):
    """Host-tier chunks (pinned bf16, streamed layer by layer and overlapped with the
    scoring pass) give exactly the device-resident result."""
    import torch
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    runs = []
    for pinned in (False, True):
        if pinned:
            src = [P.ChunkKV.from_pinned(c.chunk_id, c.config_fingerprint, c.token_ids,
                                         c.device_buffers(cfg)[0].cpu().pin_memory(),
                                         c.device_buffers(cfg)[1].cpu().pin_memory(), cfg.head_dim) for c in dch]
        else:
            src = dch
        cache = P.assemble(src, cfg, fp32_taps=False)
        sc = P.score_prophet(mw, cfg, cache, query)
        sel = P.select_top_p(sc, p)
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
        fin = P.finalize_query(mw, cfg, cache, query)
        torch.cuda.synchronize()
        runs.append((sc.per_layer, sel.indices, fin.first_logits))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][2], runs[1][2])


def test_final_pass_following_stage2_is_identical(built, monkeypatch):
    """finalize_query on its own stream, each layer released by Stage II's per-layer
    done event (PKV_FINAL_OVERLAP, default on), equals the serial order bit for bit --
    through the public API and through the graph-captured PrefillPipeline."""
    import torch

    from paper_2602_02579_b200.pipeline import PrefillPipeline
    P = built
    cfg_o, seed, units, query, p = _materialise("llama_width")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    monkeypatch.setenv("PKV_FUSED_FINAL", "0")  # the separate final pass (the fused one has none)
    runs = []
    for ov in ("0", "1"):
        monkeypatch.setenv("PKV_FINAL_OVERLAP", ov)
        cache = P.assemble(dch, cfg, fp32_taps=False)
        sc = P.score_prophet(mw, cfg, cache, query)
        sel = P.select_top_p(sc, p)
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
        fin = P.finalize_query(mw, cfg, cache, query)
        torch.cuda.synchronize()
        runs.append((sel.indices, fin.first_logits, cache.k_pool.clone()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    assert torch.equal(runs[0][2], runs[1][2])

    dm = P.DeviceModel.from_host(mw, cfg)
    outs = []
    for ov in (False, True):
        pipe = PrefillPipeline(dm, dch, len(query), p)
        pipe.final_overlap = ov
        pipe.set_query(query)
        pipe.step()
        pipe.capture()
        pipe.replay()
        torch.cuda.synchronize()
        outs.append((pipe.idx.clone(), pipe.logits.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("case", ["c1", "llama_width"])
def test_fused_finalize_matches_separate_pass(built, monkeypatch, case):
    """The query rows riding along Stage II (pkv_recompute_query, default) against the
    separate fp32-faithful final pass (PKV_FUSED_FINAL=0): the repaired context entries are
    bit-identical (each row of a GEMM / attention tile is computed independently of the rows
    added after it), the first-token logits and the appended query K/V agree within the
    contract, and both agree with the oracle -- through the public API and the pipeline."""
    import torch

    from paper_2602_02579_b200.pipeline import PrefillPipeline
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    ref = O.prophet_ttft_slice(w, cfg_o, chunks, query, p)
    runs = []
    for fused in ("0", "1"):
        monkeypatch.setenv("PKV_FUSED_FINAL", fused)
        cache = P.assemble(dch, cfg, fp32_taps=False)
        sc = P.score_prophet(mw, cfg, cache, query)
        sel = P.select_top_p(sc, p)
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
        fin = P.finalize_query(mw, cfg, cache, query)
        torch.cuda.synchronize()
        s, m = cache.context_length, len(query)
        runs.append((sel.indices, fin.first_logits, cache.k_pool[:, :, :s].clone(), cache.v_pool[:, :, :s].clone(),
                     cache.k_pool[:, :, s:s + m].float().clone(), fin.cache.keys, fin.cache.values))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][2], runs[1][2]) and torch.equal(runs[0][3], runs[1][3])
    for lg in (runs[0][1], runs[1][1]):
        assert np.abs(lg - ref["first_logits"]).max() <= KV_ABS and _cos(lg, ref["first_logits"]) >= COS_MIN
    assert float((runs[0][4] - runs[1][4]).abs().max()) <= KV_ABS
    for li in range(cfg.n_layers):  # the reference KVCache view: context + query rows
        assert np.abs(runs[0][5][li] - runs[1][5][li]).max() <= KV_ABS
        assert np.abs(runs[0][6][li] - runs[1][6][li]).max() <= KV_ABS
    _report(case=f"{case}_fused_final", logits_fused_max_abs=float(np.abs(runs[1][1] - ref["first_logits"]).max()),
            logits_separate_max_abs=float(np.abs(runs[0][1] - ref["first_logits"]).max()))

    dm = P.DeviceModel.from_host(mw, cfg)
    outs = []
    for fused in ("0", "1"):
        monkeypatch.setenv("PKV_FUSED_FINAL", fused)
        pipe = PrefillPipeline(dm, dch, len(query), p)
        pipe.set_query(query)
        pipe.step()
        pipe.capture()
        pipe.replay()
        torch.cuda.synchronize()
        outs.append((pipe.idx.clone(), pipe.logits.cpu().numpy()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert np.abs(outs[1][1] - ref["first_logits"]).max() <= KV_ABS


def test_deferred_norm_matches_standalone_norm(built, monkeypatch):
    """PKV_NORM_DEFER=1 (RMSNorm folded into the Stage-II GEMM epilogues) gives the same
    repaired cache and first-token logits within the Stage-II tolerance."""
    import torch
    P = built
    cfg_o, seed, units, query, p = _materialise("llama_width")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    runs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("PKV_NORM_DEFER", mode)
        cache = P.assemble(dch, cfg, fp32_taps=False)
        sc = P.score_prophet(mw, cfg, cache, query)
        sel = P.select_top_p(sc, p)
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
        fin = P.finalize_query(mw, cfg, cache, query)
        torch.cuda.synchronize()
        runs.append((sel.indices, fin.first_logits, cache.k_pool.float(), cache.v_pool.float()))
    assert runs[0][0] == runs[1][0]
    for a, b in ((runs[0][2], runs[1][2]), (runs[0][3], runs[1][3])):
        # two fp16 Stage-II rounding paths, each within KV_ABS of the fp32 reference
        assert float((a - b).abs().max()) <= 2 * KV_ABS
        assert float(torch.nn.functional.cosine_similarity(a.flatten(), b.flatten(), dim=0)) >= 0.9999
    assert np.abs(runs[0][1] - runs[1][1]).max() <= KV_ABS and _cos(runs[0][1], runs[1][1]) >= COS_MIN


def test_state_machine_and_errors(built):
    P = built
    cfg_o, seed, units, query, _ = CASES["tiny_ref"][0], 42, CASES["tiny_ref"][2], CASES["tiny_ref"][3], 0.3
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, track_access=True)
    sel = P.select_top_p(P.ValueScores.from_vector("x", np.arange(cache.context_length)[::-1], 1), 1.0)
    with pytest.raises(P.ArgumentError):
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(P.SelectionResult([3, 1], 0.2, 2)))
    out = P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    assert out is cache
    writes = [l for kind, l in cache.access_log if kind == "write"]
    assert writes == list(range(cfg.n_layers))
    with pytest.raises(P.StateError):
        P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
    P.finalize_query(mw, cfg, cache, query)
    with pytest.raises(P.StateError):
        P.finalize_query(mw, cfg, cache, query)
    with pytest.raises(P.InputError):
        P.score_prophet(mw, cfg, P.assemble(dch, cfg), [])
    with pytest.raises(P.InputError):
        P.assemble([], cfg)
    zero = P.select_top_p(P.ValueScores.from_vector("x", np.zeros(cache.context_length), 1), 0.0)
    fresh = P.assemble(dch, cfg)
    assert P.recompute_selected(mw, cfg, fresh, P.RecomputePlan(zero)) is fresh
    assert not fresh.recomputed.any()


def test_flop_books_follow_reference_formulas(built):
    P = built
    cfg_o, seed, units, query, _ = CASES["tiny_ref"][0], 42, CASES["tiny_ref"][2], CASES["tiny_ref"][3], 0.3
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg)
    s = cache.context_length
    for q in (query[:2], query):
        t = P.FlopTally()
        P.score_prophet(mw, cfg, cache, q, tally=t)
        m = len(q)
        assert t.attn_scores.multiply_accumulate_count == cfg.n_layers * cfg.n_heads * m * cfg.head_dim * (s + m)
        assert (t.total.multiply_accumulate_count, t.attn_scores.multiply_accumulate_count) == \
            O.macs_query_pass(cfg_o, s, m)


@pytest.mark.parametrize("case", ["tiny_ref", "c1", "llama_width"])
def test_kvshare_probe_matches_oracle(built, case):
    """score_kvshare_l1 (reference selection.py:136-142): layer-0 column sums x ||dV||_1."""
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, fp32_taps=False)
    tally = P.FlopTally()
    got = P.score_kvshare_l1(mw, cfg, cache, tally=tally).fused
    ref = O.kvshare_l1(w, cfg_o, O.stitch(chunks, cfg_o))
    assert tally.total.multiply_accumulate_count == O.macs_probe(cfg_o, cache.context_length)
    err = float(np.abs(got - ref).max()) / max(float(np.abs(ref).max()), 1e-30)
    assert err <= 1e-4, err
    sel_ref, k = O.select(ref, p)
    sel = P.select_top_p(P.ValueScores.from_vector("kvshare_l1", got, cfg.n_layers), p)
    assert _selection_ok(sel.indices, sel_ref, ref, k)
    _report(case=f"{case}_kvshare", s=cache.context_length, k=k, probe_max_rel=err,
            sel_symdiff=len(set(sel.indices) ^ set(sel_ref)))


@pytest.mark.parametrize("case", ["tiny_ref", "c1", "llama_width"])
def test_cacheblend_probe_matches_oracle(built, case):
    """score_cacheblend_l1 (reference selection.py:127-133): the fp32-faithful probe passes
    reproduce the oracle's ||dV||_2 and its MAC books, and select the same tokens."""
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, fp32_taps=False)
    tally = P.FlopTally()
    got = P.score_cacheblend_l1(mw, cfg, cache, tally=tally).fused
    macs = [0]
    ref = O.cacheblend_l1(w, cfg_o, O.stitch(chunks, cfg_o), macs=macs)
    assert tally.total.multiply_accumulate_count == macs[0] == O.macs_probe(cfg_o, cache.context_length)
    scale = max(float(np.abs(ref).max()), 1e-30)
    err = float(np.abs(got - ref).max()) / scale
    assert err <= 1e-4, err
    sel_ref, k = O.select(ref, p)
    sel = P.select_top_p(P.ValueScores.from_vector("cacheblend_l1", got, cfg.n_layers), p)
    assert _selection_ok(sel.indices, sel_ref, ref, k)
    _report(case=f"{case}_cacheblend", s=cache.context_length, k=k, probe_max_rel=err,
            sel_symdiff=len(set(sel.indices) ^ set(sel_ref)))
