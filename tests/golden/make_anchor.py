"""Generate the full-scale parity fixtures (the oracle run on the SYN1 synthetic inputs).

    python tests/golden/make_anchor.py sel32k_l4 llama_l32_2k c3 [--threads 8]

Each fixture is the layer-streamed oracle (oracle/anchor.py, bit-identical to the
resident oracle, which is pinned to the reference) on the SYN1 weights / chunk store /
query (oracle/synthetic_inputs.py == paper_2602_02579_b200/synthetic.py on the device):
per-layer and fused scores, the selection, the first-token logits and the fresh K/V of
16 evenly spaced selected rows at every layer.  tests/test_gpu_anchor.py and bench.py
check the GPU path against them.  CPU cost here (8 cores): sel32k_l4 ~1 min,
llama_l32_2k ~10 min, c3 ~1 h.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import anchor as A  # noqa: E402
from oracle import pikv_oracle as O  # noqa: E402

LLAMA = dict(n_heads=32, n_kv_heads=8, head_dim=128, hidden_dim=4096, ffn_dim=14336, rope_theta=500000.0)
SPECS = {
    # selection parity at the target context: Llama width, 4 layers, 16 x 2048 + 32, p = 0.2 (Stage I only)
    "sel32k_l4": dict(cfg=dict(n_layers=4, vocab_size=128256, **LLAMA), n_chunks=16, chunk_len=2048, m=32, p=0.2,
                      stage1_only=True),
    # full depth at Llama width: 32 layers, 8 x 256 + 32, p = 0.2
    "llama_l32_2k": dict(cfg=dict(n_layers=32, vocab_size=8192, **LLAMA), n_chunks=8, chunk_len=256, m=32, p=0.2),
    # the bench's workload (BASELINE configs[2] / C3): Llama-3-8B shape, 16 x 2048 + 32, p = 0.2
    "c3": dict(cfg=dict(n_layers=32, vocab_size=128256, **LLAMA), n_chunks=16, chunk_len=2048, m=32, p=0.2),
}


def make(name, threads, seed=0):
    sp = SPECS[name]
    cfg = O.Cfg(**sp["cfg"])
    req = A.SynRequest(cfg, seed, sp["n_chunks"], sp["chunk_len"], sp["m"])
    t0 = time.time()
    k = O.budget(sp["p"], req.s)
    rows = np.unique(np.linspace(0, k - 1, 16).round().astype(np.int64))
    out = A.run(req, sp["p"], kv_rows=rows, threads=threads, stage1_only=sp.get("stage1_only", False),
                log=lambda msg: print(msg, flush=True))
    meta = dict(name=name, cfg=sp["cfg"], seed=seed, n_chunks=sp["n_chunks"], chunk_len=sp["chunk_len"], m=sp["m"],
                p=sp["p"], k=int(out["k"]), inputs="SYN1 (oracle/synthetic_inputs.py)",
                oracle="oracle/anchor.py (layer-streamed pikv_oracle)", cpu_seconds=round(time.time() - t0, 1))
    arrays = {k_: v for k_, v in out.items() if isinstance(v, np.ndarray)}
    arrays["sel"] = arrays["sel"].astype(np.int32)
    path = Path(__file__).with_name(f"anchor_{name}.npz")
    np.savez_compressed(path, meta=json.dumps(meta), **arrays)
    print(f"wrote {path} ({path.stat().st_size / 1e6:.1f} MB) in {meta['cpu_seconds']} s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+", choices=list(SPECS))
    ap.add_argument("--threads", type=int, default=8)
    a = ap.parse_args()
    for n in a.names:
        make(n, a.threads)
