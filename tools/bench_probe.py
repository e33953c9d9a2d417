"""Time the probe baselines (score_cacheblend_l1 / score_kvshare_l1, reference
selection.py:95-142) on the device at the C3 shape (Llama-3-8B width, 32k context of 16
SYN1 chunks): 1024 per-block fp32-faithful narrow passes over the truncated cache, device
f64 column sums and norms, one read-back.  python tools/bench_probe.py [n_chunks]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from paper_2602_02579_b200 import synthetic as S  # noqa: E402

n_chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.synthetic(cfg, seed=0)
chunks = S.chunks(cfg, n_chunks, 2048, 0, dm.fingerprint)
res = {"s": n_chunks * 2048}
for name, fn in (("cacheblend_l1", P.score_cacheblend_l1), ("kvshare_l1", P.score_kvshare_l1)):
    cache = P.assemble(chunks, cfg, fp32_taps=False)
    fn(dm, cfg, cache)  # warm-up (workspace, kernel attributes)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sc = fn(dm, cfg, cache)
    torch.cuda.synchronize()
    res[name + "_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    res[name + "_finite"] = bool(torch.isfinite(torch.as_tensor(sc.fused)).all())
print(json.dumps(res))
