"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py

The fixtures pin the oracle (tests/test_oracle_golden.py) on machines where the
reference is absent, e.g. the GPU box.  Inputs are regenerated deterministically
from the seeds recorded here (reference random_weights / precompute_chunk), so only
outputs are stored.
"""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

SCENARIOS = {
    # reference conftest tiny_cfg + test_recompute UNITS/QUERY
    "tiny_ref": dict(cfg=dict(n_layers=2, n_heads=2, n_kv_heads=1, head_dim=4, hidden_dim=8, ffn_dim=16,
                              vocab_size=50), seed=42,
                     units=[[3, 17, 42, 0, 9, 31], [25, 7, 49, 13], [2, 38, 11, 29, 6]], query=[8, 19, 44, 1],
                     p=0.3, bf16=False),
    # BASELINE configs[0]-shaped (C1), bf16-rounded weights and chunk K/V (the GPU parity inputs)
    "c1_bf16": dict(cfg=dict(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64, hidden_dim=256, ffn_dim=1024,
                             vocab_size=1024), seed=0, units="8x256", query=32, p=0.2, bf16=True),
    # GQA task-size model (reference conftest task_cfg shape, vocab 64)
    "task_gqa": dict(cfg=dict(n_layers=3, n_heads=4, n_kv_heads=2, head_dim=8, hidden_dim=32, ffn_dim=64,
                              vocab_size=64), seed=7, units="4x24", query=6, p=0.25, bf16=False),
}


def bf16(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def materialise(sc):
    rng = np.random.default_rng(1000 + sc["seed"])
    units = sc["units"]
    if isinstance(units, str):
        n, t = map(int, units.split("x"))
        units = [rng.integers(0, sc["cfg"]["vocab_size"], t).tolist() for _ in range(n)]
    query = sc["query"]
    if isinstance(query, int):
        query = rng.integers(0, sc["cfg"]["vocab_size"], query).tolist()
    return units, query


def run(name, sc):
    sys.path.insert(0, str(REF))
    import pikv
    cfg = pikv.ModelConfig(**sc["cfg"])
    w = pikv.random_weights(cfg, sc["seed"])
    if sc["bf16"]:
        for lw in w.layers:
            for k in ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down"):
                setattr(lw, k, bf16(getattr(lw, k)))
        w.embed, w.final_norm, w.lm_head = bf16(w.embed), bf16(w.final_norm), bf16(w.lm_head)
        w._fingerprint = None
    units, query = materialise(sc)
    chunks = [pikv.precompute_chunk(w, cfg, u) for u in units]
    if sc["bf16"]:
        for c in chunks:
            c.keys_norope = [bf16(x) for x in c.keys_norope]
            c.values = [bf16(x) for x in c.values]
    cache = pikv.assemble(chunks, cfg)
    keys0 = [k.copy() for k in cache.keys_rebased]
    scores = pikv.score_prophet(w, cfg, cache, query)
    sel = pikv.select_top_p(scores, sc["p"])
    pikv.recompute_selected(w, cfg, cache, pikv.RecomputePlan(sel))
    fin = pikv.finalize_query(w, cfg, cache, query)
    ix = np.asarray(sel.indices, dtype=np.int64)
    arrays = {
        "per_layer": scores.per_layer, "fused": scores.fused, "sel": ix, "first_logits": fin.first_logits,
        "assembled_keys": np.stack(keys0), "repaired_k": np.stack([k[ix] for k in cache.keys_rebased]),
        "repaired_v": np.stack([v[ix] for v in cache.values]),
    }
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    meta = dict(sc, units=units, query=query, k=sel.k, fingerprint=w.fingerprint(cfg),
                sha={k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16] for k, v in arrays.items()})
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(name, "k =", sel.k, "s =", cache.context_length)


if __name__ == "__main__":
    if not REF.exists():
        sys.exit("reference package not found; fixtures can only be regenerated in the build container")
    for n, sc in SCENARIOS.items():
        run(n, sc)
