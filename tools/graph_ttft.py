"""Graph-replayed TTFT of the Llama-3-8B 32k prefill (one process per setting: env knobs
such as PKV_PDL / PKV_ASM_PIPE are read once).  python tools/graph_ttft.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from paper_2602_02579_b200.pipeline import PrefillPipeline, random_device_chunks  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.random(cfg, seed=0)
chunks = random_device_chunks(cfg, 16, 2048, seed=1)
pipe = PrefillPipeline(dm, chunks, 32, float(os.environ.get("P", "0.2")))
pipe.set_query(np.random.default_rng(7).integers(0, cfg.vocab_size, 32))
for _ in range(2):
    pipe.step()
pipe.capture()
for _ in range(3):
    pipe.replay()
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pipe.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / steps)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PKV_") or k == "P"},
                  "ttft_ms": [round(x, 3) for x in res]}), flush=True)
