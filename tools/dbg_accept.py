"""Diagnostic: total-recompute first-logit gaps per seed, f32 weights vs bf16-exact weights."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import __graft_entry__
__graft_entry__.build()
import paper_2602_02579_b200 as P
from oracle import pikv_oracle as O
import test_gpu_acceptance as T

for rnd in (False, True):
    for i in range(50):
        cfg, w, units, query = T._random_setup(P, 1000 + i)
        if rnd:
            w = P.ModelWeights(embed=O.bf16_round(w.embed), final_norm=O.bf16_round(w.final_norm),
                               lm_head=O.bf16_round(w.lm_head),
                               layers=[P.LayerWeights(**{k: O.bf16_round(getattr(lw, k)) for k in (
                                   "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")})
                                   for lw in w.layers])
        cfg_o, w_o = T._oracle(cfg, w)
        ref_logits, ref_ans, margins = T._greedy_ref(w_o, cfg_o, [t for u in units for t in u] + list(query), 6)
        run = P.run_strategy(w, cfg, T._chunks(P, cfg, w, units), query, T.STRATEGIES[i % 5], 1.0, seed=i,
                             max_new_tokens=6)
        gap = float(np.abs(run.first_logits - ref_logits).max())
        print(f"rnd={rnd} i={i} cfg={cfg.to_json_dict()} gap={gap:.4f} maxlogit={np.abs(ref_logits).max():.3f} "
              f"ans_ok={T._answers_agree(run.record.answer_tokens, ref_ans, margins)}", flush=True)
