"""Run the benchmark pipeline for a few steps (target of ncu captures).

    ncu --set full -k regex:<kernel> -s <skip> -c 1 -o out python tools/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from paper_2602_02579_b200.pipeline import PrefillPipeline, random_device_chunks  # noqa: E402

steps = int(os.environ.get("STEPS", "2"))
cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.random(cfg, seed=0)
chunks = random_device_chunks(cfg, 16, 2048, seed=1)
pipe = PrefillPipeline(dm, chunks, 32, 0.2)
pipe.set_query(np.random.default_rng(7).integers(0, cfg.vocab_size, 32))
for _ in range(steps):
    pipe.step()
torch.cuda.synchronize()
print("done")
