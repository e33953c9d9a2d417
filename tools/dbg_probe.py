import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import __graft_entry__; __graft_entry__.build()
import paper_2602_02579_b200 as P
from oracle import pikv_oracle as O
from test_gpu_parity import _materialise, _setup, _device_inputs
for case in ("tiny_ref", "c1"):
    cfg_o, seed, units, query, p = _materialise(case)
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    cache = P.assemble(dch, cfg, fp32_taps=False)
    got = P.score_cacheblend_l1(mw, cfg, cache).fused
    ref = O.cacheblend_l1(w, cfg_o, O.stitch(chunks, cfg_o))
    print(case, cache.context_length, "max ref", ref.max())
    d = np.abs(got - ref)
    idx = np.argsort(-d)[:8]
    print(" worst", idx.tolist(), got[idx].round(5).tolist(), ref[idx].round(5).tolist())
    print(" first tokens", got[:6].round(5).tolist(), ref[:6].round(5).tolist())
    for b in range(0, cache.context_length, 256):
        print("  block", b, float(d[b:b+256].max()))
