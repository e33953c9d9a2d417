"""The CPU oracle reproduces reference-generated golden outputs bit for bit.

Fixtures: tests/golden/*.npz, produced by tests/golden/make_golden.py running the
real reference package.  Inputs are regenerated here from the recorded seeds with
the oracle, so this also pins the oracle's weight init and chunk precompute.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import pikv_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"
# anchor_*.npz: the SYN1 full-scale fixtures of tests/golden/make_anchor.py (tests/test_gpu_anchor.py)
NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith("anchor_"))


def oracle_run(meta):
    cfg = O.Cfg(**meta["cfg"])
    w = O.init_weights(cfg, meta["seed"])
    if meta["bf16"]:
        w = w.rounded_bf16()
    chunks = []
    for u in meta["units"]:
        c = O.make_chunk(w, cfg, u)
        if meta["bf16"]:
            c.k_nr = [O.bf16_round(x) for x in c.k_nr]
            c.v = [O.bf16_round(x) for x in c.v]
        chunks.append(c)
    cache = O.stitch(chunks, cfg)
    keys0 = np.stack([k.copy() for k in cache.keys])
    per, fused = O.prophet_scores(w, cfg, cache, meta["query"])
    sel, k = O.select(fused, meta["p"])
    O.repair(w, cfg, cache, sel)
    logits, _ = O.finalize(w, cfg, cache, meta["query"])
    ix = np.asarray(sel, dtype=np.int64)
    return w, cfg, {"per_layer": per, "fused": fused, "sel": ix, "first_logits": logits, "assembled_keys": keys0,
                    "repaired_k": np.stack([kk[ix] for kk in cache.keys]),
                    "repaired_v": np.stack([v[ix] for v in cache.values])}


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_golden(name):
    meta = json.loads((GOLDEN / f"{name}.json").read_text())
    gold = np.load(GOLDEN / f"{name}.npz")
    w, cfg, got = oracle_run(meta)
    assert w.fingerprint(cfg) == meta["fingerprint"]
    for key in gold.files:
        assert np.array_equal(got[key], gold[key]), key
    assert len(got["sel"]) == meta["k"]


def test_golden_fixtures_present():
    assert {"tiny_ref", "c1_bf16", "task_gqa"} <= set(NAMES)
