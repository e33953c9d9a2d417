"""Per-phase device times (native timers) of the Llama-3-8B 32k prefill step, optionally
under a sweep of an environment knob:  python tools/phase_times.py [VAR v1 v2 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from paper_2602_02579_b200 import _lib  # noqa: E402
from paper_2602_02579_b200.pipeline import PrefillPipeline, random_device_chunks  # noqa: E402

cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.random(cfg, seed=0)
chunks = random_device_chunks(cfg, 16, 2048, seed=1)
pipe = PrefillPipeline(dm, chunks, 32, float(os.environ.get("P", "0.2")))
pipe.set_query(np.random.default_rng(7).integers(0, cfg.vocab_size, 32))
var, vals = (sys.argv[1], sys.argv[2:]) if len(sys.argv) > 2 else (None, [None])
for v in vals:
    if var:
        os.environ[var] = v
    for _ in range(2):
        pipe.step()
    torch.cuda.synchronize()
    _lib.timing(True)
    n = 3
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(n):
        pipe.step()
    ev1.record()
    torch.cuda.synchronize()
    ph = _lib.timing_collect()
    _lib.timing(False)
    tot = ev0.elapsed_time(ev1) / n
    print(json.dumps({"var": var, "value": v, "step_ms": round(tot, 3),
                      **{k: round(t / n, 3) for k, (t, c) in ph.items() if c}}), flush=True)
