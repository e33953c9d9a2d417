"""Graph-replayed time of each prefill phase (Llama-3-8B 32k, p = 0.2): the scoring
narrow pass, Stage II, the final narrow pass.  python tools/graph_phases.py"""
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
from paper_2602_02579_b200.chunkstore import ctypes_ref  # noqa: E402
from paper_2602_02579_b200.pipeline import PrefillPipeline, random_device_chunks  # noqa: E402

cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.random(cfg, seed=0)
chunks = random_device_chunks(cfg, 16, 2048, seed=1)
pipe = PrefillPipeline(dm, chunks, 32, float(os.environ.get("P", "0.2")))
pipe.set_query(np.random.default_rng(7).integers(0, cfg.vocab_size, 32))
for _ in range(2):
    pipe.step()
torch.cuda.synchronize()
lib = _lib.load()
c = pipe.cache
_cc = _lib.Cache.from_buffer_copy(c.c_cache)
_cc.layer_ready = None  # no cross-capture event waits (each phase is its own graph)
cc, ch = ctypes_ref(_cc), ctypes_ref(c.c_chunks)


def score(st):
    _lib.check(lib.pkv_query_pass(dm.handle, cc, ch, pipe.query.data_ptr(), pipe.m, pipe.flags_score,
                                  pipe.per_layer.data_ptr(), None, None, None, pipe.ws_qp.data_ptr(),
                                  pipe.ws_qp.numel(), st))


def recompute(st):
    _lib.check(lib.pkv_recompute(dm.handle, cc, pipe.idx.data_ptr(), pipe.k, None, None, pipe.ws_rc.data_ptr(),
                                 pipe.ws_rc.numel(), st))


def final(st):
    _lib.check(lib.pkv_query_pass(dm.handle, cc, ch, pipe.query.data_ptr(), pipe.m, pipe.flags_final, None, None,
                                  None, pipe.logits.data_ptr(), pipe.ws_qp.data_ptr(), pipe.ws_qp.numel(), st))


out = {}
for name, fn in (("score_pass", score), ("stage2", recompute), ("final_pass", final)):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            fn(side.cuda_stream)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    n = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / n, 3)
print(json.dumps(out))
