"""Head-sharded (tensor-parallel) prefill on one GPU: W ranks as W host threads of an
in-process communicator group (paper_2602_02579_b200.tp.local_group), each with its
own stream, weight shard, chunk-store slice and paged cache -- the same stage loops
and exchange points the NCCL back end runs across GPUs.

Checked against the CPU oracle with the single-GPU contract (tests/test_gpu_parity.py):
per-layer scores rel err <= 1e-4, selection equal outside the 1e-4 tie band and
IDENTICAL on every rank, first-token logits max abs <= 2e-2 / cosine >= 0.999 against
the oracle run on the sharded selection; and against the unsharded device run: the
rank's cache slice (including the scattered Stage-II K/V) matches the W = 1 cache.
"""

import numpy as np
import pytest

from oracle import pikv_oracle as O

from test_gpu_parity import COS_MIN, KV_ABS, REL_TOL, _cos, _materialise, _report, _selection_ok, _setup

pytestmark = pytest.mark.gpu


def _run(P, dm, chunks, query, p):
    from paper_2602_02579_b200.pipeline import PrefillPipeline
    pipe = PrefillPipeline(dm, chunks, len(query), p)
    pipe.set_query(query)
    return pipe


@pytest.mark.parametrize("case,world", [("c1", 2), ("llama_width", 2), ("llama_width", 4)])
def test_head_sharded_prefill_matches_oracle(built, case, world):
    import torch

    from paper_2602_02579_b200 import tp
    P = built
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cache_o = O.stitch(chunks, cfg_o)
    per_ref, fused_ref = O.prophet_scores(w, cfg_o, cache_o, query)
    sel_ref, k = O.select(fused_ref, p)

    cfg = P.ModelConfig(**cfg_o.json())
    mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{n: getattr(lw, n) for n in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
        final_norm=w.final_norm, lm_head=w.lm_head)
    dm = P.DeviceModel.from_host(mw, cfg)
    fp = mw.fingerprint(cfg)
    dch = [P.ChunkKV(c.chunk_id, fp, c.token_ids, c.k_nr, c.v) for c in chunks]
    for c in dch:
        c.device_buffers(cfg)

    # unsharded device run (reference point for the cache slices)
    one = _run(P, dm, dch, query, p)
    one.step()
    torch.cuda.synchronize()

    comms = tp.local_group(world)
    shards = [dm.shard(c.rank, world, c.handle) for c in comms]
    pipes = [_run(P, shards[r], tp.shard_chunks(dch, r, world), query, p) for r in range(world)]
    torch.cuda.synchronize()
    tp.run_ranks([pipe.step for pipe in pipes])
    torch.cuda.synchronize()

    sels = [pipe.idx[:k].cpu().numpy().tolist() for pipe in pipes]
    for r in range(1, world):
        assert sels[r] == sels[0], f"rank {r} selected a different token set"
        assert torch.equal(pipes[r].per_layer, pipes[0].per_layer)
        assert torch.equal(pipes[r].logits, pipes[0].logits)
    per = pipes[0].per_layer.cpu().numpy()
    rel = np.abs(per - per_ref) / np.maximum(np.abs(per_ref), 1e-30)
    assert rel.max() <= REL_TOL, f"per-layer score rel err {rel.max():.3e}"
    assert _selection_ok(sels[0], sel_ref, fused_ref, k)

    # first-token logits vs the oracle on the sharded selection
    O.repair(w, cfg_o, cache_o, sels[0])
    lg_ref, _ = O.finalize(w, cfg_o, cache_o, query)
    lg = pipes[0].logits.cpu().numpy()
    err = float(np.abs(lg - lg_ref).max())
    cos = _cos(lg, lg_ref)
    assert err <= KV_ABS and cos >= COS_MIN, (err, cos)

    # each rank's cache slice == the unsharded cache's heads (Stage-II K/V scattered in place)
    # (fp16 storage: the fp32 sums differ from the unsharded order by ~1e-7 relative, so
    # an entry may round to a neighbouring fp16 value -> allow two fp16 ulps)
    s = one.s
    kl = cfg.n_kv_heads // world
    kv_err = 0.0
    same_sel = sels[0] == one.idx[:k].cpu().numpy().tolist()
    if same_sel:
        for r in range(world):
            for name in ("k_pool", "v_pool"):
                a = getattr(pipes[r].cache, name)[:, :, :s].float()
                b = getattr(one.cache, name)[:, r * kl:(r + 1) * kl, :s].float()
                ulp = torch.clamp(b.abs(), min=1.0) * 2.0 ** -10
                kv_err = max(kv_err, float(((a - b).abs() / ulp).max()))
        assert kv_err <= 2.0, f"cache slice differs from the unsharded cache by {kv_err:.2f} fp16 ulp"
    _report(case=f"{case}_tp{world}", s=s, k=k, per_layer_max_rel=rel.max(), sel_symdiff=len(set(sels[0]) ^ set(sel_ref)),
            logits_max_abs=err, logits_cos=cos, kv_vs_unsharded_max_abs=kv_err, same_sel_as_unsharded=same_sel)
    for c in comms:
        c.close()


def test_local_allreduce_sums_bit_identically(built):
    import torch

    from paper_2602_02579_b200 import tp
    world = 3
    comms = tp.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(0)
    bufs = [torch.randn(1000, generator=g, device="cuda", dtype=torch.float64) for _ in range(world)]
    want = bufs[0] + bufs[1] + bufs[2]
    torch.cuda.synchronize()
    tp.run_ranks([lambda r=r: comms[r].allreduce_(bufs[r]) for r in range(world)])
    for b in bufs:
        assert torch.equal(b, want)
    for c in comms:
        c.close()


@pytest.mark.parametrize("case,world", [("c1", 2), ("llama_width", 2), ("llama_width", 4), ("tiny_ref", 3)])
def test_token_parallel_stage2_is_bit_identical(built, case, world):
    """Token-parallel Stage II (DeviceModel.rows, pkv_recompute_rows): every rank holds the
    full model and cache, repairs its attention units of the selection and all-gathers the
    fresh entries per layer.  Each row is computed exactly as in the single-GPU run (a GEMM
    row and an attention tile do not depend on the other rows), so every rank's repaired
    cache and first-token logits equal the unsharded run's bit for bit -- through the
    graph-capturable pipeline and through the public API."""
    import torch

    import paper_2602_02579_b200 as P
    from paper_2602_02579_b200 import tp
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg = P.ModelConfig(**cfg_o.json())
    mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{n: getattr(lw, n) for n in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
        final_norm=w.final_norm, lm_head=w.lm_head)
    dm = P.DeviceModel.from_host(mw, cfg)
    fp = mw.fingerprint(cfg)
    dch = [P.ChunkKV(c.chunk_id, fp, c.token_ids, c.k_nr, c.v) for c in chunks]
    for c in dch:
        c.device_buffers(cfg)
    one = _run(P, dm, dch, query, p)
    one.step()
    torch.cuda.synchronize()

    comms = tp.local_group(world)
    pipes = [_run(P, dm.rows(c), dch, query, p) for c in comms]
    torch.cuda.synchronize()
    tp.run_ranks([pipe.step for pipe in pipes])
    torch.cuda.synchronize()
    s, k = one.s, one.k
    for r, pipe in enumerate(pipes):
        assert torch.equal(pipe.idx[:k], one.idx[:k]), r
        for name in ("k_pool", "v_pool", "k2_pool"):
            assert torch.equal(getattr(pipe.cache, name)[:, :, :s], getattr(one.cache, name)[:, :, :s]), (r, name)
        assert torch.equal(pipe.logits, one.logits), r
        assert torch.equal(pipe.cache.k_pool[:, :, s:s + len(query)], one.cache.k_pool[:, :, s:s + len(query)]), r

    # the public API on the same ranks: score -> select -> recompute -> finalize
    def api(c):
        def run():
            cache = P.assemble(dch, cfg, fp32_taps=False)
            sc = P.score_prophet(dm.rows(c), cfg, cache, query)
            sel = P.select_top_p(sc, p)
            P.recompute_selected(dm.rows(c), cfg, cache, P.RecomputePlan(sel))
            fin = P.finalize_query(dm.rows(c), cfg, cache, query)
            torch.cuda.current_stream().synchronize()
            return sel.indices, fin.first_logits, cache.k_pool[:, :, :s].clone()
        return run
    outs = tp.run_ranks([api(c) for c in comms])
    for sel_r, lg_r, kp_r in outs:
        assert sel_r == one.idx[:k].cpu().numpy().tolist()
        assert np.array_equal(lg_r, one.logits.cpu().numpy())
        assert torch.equal(kp_r, one.cache.k_pool[:, :, :s])
    _report(case=f"{case}_rows{world}", s=s, k=k, bit_identical=True)
    for c in comms:
        c.close()


def test_token_parallel_without_query_rows(built, monkeypatch):
    """Token-parallel Stage II with the separate final pass (PKV_FUSED_FINAL=0: no query rows
    ride along) and a rank that owns no selected rows: it still joins every per-layer
    all-gather and ends with the full repaired cache."""
    import torch

    import paper_2602_02579_b200 as P
    from paper_2602_02579_b200 import tp
    monkeypatch.setenv("PKV_FUSED_FINAL", "0")
    cfg_o, seed, units, query, p = _materialise("tiny_ref")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg = P.ModelConfig(**cfg_o.json())
    mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{n: getattr(lw, n) for n in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
        final_norm=w.final_norm, lm_head=w.lm_head)
    dm = P.DeviceModel.from_host(mw, cfg)
    fp = mw.fingerprint(cfg)
    dch = [P.ChunkKV(c.chunk_id, fp, c.token_ids, c.k_nr, c.v) for c in chunks]
    one = _run(P, dm, dch, query, p)
    one.step()
    torch.cuda.synchronize()
    comms = tp.local_group(3)
    pipes = [_run(P, dm.rows(c), dch, query, p) for c in comms]
    tp.run_ranks([pipe.step for pipe in pipes])
    torch.cuda.synchronize()
    s = one.s
    for pipe in pipes:
        for name in ("k_pool", "v_pool", "k2_pool"):
            assert torch.equal(getattr(pipe.cache, name)[:, :, :s], getattr(one.cache, name)[:, :, :s])
        assert torch.equal(pipe.logits, one.logits)
    for c in comms:
        c.close()


@pytest.mark.parametrize("case,world", [("llama_width", 2), ("llama_width", 4)])
def test_sharded_scoring_with_token_parallel_stage2(built, case, world):
    """Both multi-GPU splits at once (bench --mode tokens): the scoring pass head-sharded over
    each rank's head slice of its full cache (pkv_cache.pool_heads / head0, per-layer score
    all-reduce), Stage II token-parallel on the full model.  Every rank selects what the
    unsharded run selects and ends with its repaired cache and logits bit for bit."""
    import torch

    import paper_2602_02579_b200 as P
    from paper_2602_02579_b200 import tp
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg = P.ModelConfig(**cfg_o.json())
    mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{n: getattr(lw, n) for n in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
        final_norm=w.final_norm, lm_head=w.lm_head)
    dm = P.DeviceModel.from_host(mw, cfg)
    fp = mw.fingerprint(cfg)
    dch = [P.ChunkKV(c.chunk_id, fp, c.token_ids, c.k_nr, c.v) for c in chunks]
    one = _run(P, dm, dch, query, p)
    one.step()
    torch.cuda.synchronize()
    comms = tp.local_group(world)
    from paper_2602_02579_b200.pipeline import PrefillPipeline
    pipes = []
    for c in comms:
        pipe = PrefillPipeline(dm.rows(c), dch, len(query), p, stage1_dm=dm.shard(c.rank, world, c.handle))
        pipe.set_query(query)
        pipes.append(pipe)
    torch.cuda.synchronize()
    tp.run_ranks([pipe.step for pipe in pipes])
    torch.cuda.synchronize()
    s, k = one.s, one.k
    rel = float(((pipes[0].per_layer - one.per_layer).abs() / one.per_layer.abs().clamp_min(1e-30)).max())
    assert rel <= REL_TOL, rel
    for r, pipe in enumerate(pipes):
        assert torch.equal(pipe.per_layer, pipes[0].per_layer), r
        assert torch.equal(pipe.idx[:k], one.idx[:k]), r
        for name in ("k_pool", "v_pool", "k2_pool"):
            assert torch.equal(getattr(pipe.cache, name)[:, :, :s], getattr(one.cache, name)[:, :, :s]), (r, name)
        assert torch.equal(pipe.logits, one.logits), r
    _report(case=f"{case}_hybrid{world}", s=s, k=k, per_layer_rel_vs_unsharded=rel, bit_identical_stage2=True)
    for c in comms:
        c.close()
