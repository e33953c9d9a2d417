"""Device full prefill and chunk precompute against the oracle:
reference model.full_prefill (332-359) and chunkstore.precompute_chunk (52-62), with the
Stage-II tolerances (bf16 operands, fp32 accumulation: max abs <= 2e-2, cosine >= 0.999)."""

import numpy as np
import pytest

from oracle import pikv_oracle as O

from test_gpu_parity import COS_MIN, KV_ABS, _cos, _device_inputs, _materialise, _setup

pytestmark = pytest.mark.gpu


def test_precompute_chunk_matches_reference(built):
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    ref = O.make_chunk(w, cfg_o, units[0])
    got = P.precompute_chunk(mw, cfg, units[0])
    assert got.chunk_id == dch[0].chunk_id and got.config_fingerprint == dch[0].config_fingerprint
    for li in range(cfg.n_layers):
        for a, b in ((got.keys_norope[li], ref.k_nr[li]), (got.values[li], ref.v[li])):
            assert np.abs(a - b).max() <= KV_ABS and _cos(a, b) >= COS_MIN, li


def test_full_prefill_matches_reference_and_feeds_assembly(built):
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    toks = units[0] + units[1]
    ref = O.prefill(w, cfg_o, toks)
    t = P.FlopTally()
    got = P.full_prefill(mw, cfg, toks, capture_keys_norope=True, tally=t)
    for li in range(cfg.n_layers):
        assert np.abs(got.keys[li] - ref.keys[li]).max() <= KV_ABS
        assert np.abs(got.values[li] - ref.values[li]).max() <= KV_ABS
    rel = np.abs(got.logits - ref.logits).max() / np.abs(ref.logits).max()
    assert rel <= 2e-2 and _cos(got.logits, ref.logits) >= COS_MIN, rel
    assert t.total.multiply_accumulate_count == O.macs_query_pass(cfg_o, 0, len(toks))[0]
    # a device-produced chunk assembles exactly like the same bytes uploaded from the host
    chunk = P.precompute_chunk(mw, cfg, units[0])
    host = P.ChunkKV(chunk.chunk_id, chunk.config_fingerprint, chunk.token_ids, chunk.keys_norope, chunk.values)
    k_dev = P.assemble([chunk], cfg, fp32_taps=False).keys_rebased[1]
    k_host = P.assemble([host], cfg, fp32_taps=False).keys_rebased[1]
    assert np.array_equal(k_dev, k_host)
