"""Graph-timed Stage-II attention at the C3 shape (32 heads, 8 KV heads, dk 128, s = 32768,
6554 selected queries at sorted random positions).  Env knobs of attn_tc.cu apply
(PKV_ATTN_POLY, PKV_ATTN_SPLIT).  python tools/bench_attn.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from test_gpu_kernels import _attn_setup  # noqa: E402

H, Hkv, dk, s, n_q = 32, 8, 128, 32768, 6554
cfg, dm, lay, kp, vp, pages, pos, q, cache = _attn_setup(torch, P, H, Hkv, dk, s, n_q, False, seed=3)
out = torch.zeros((n_q, H, lay.dkp), dtype=torch.bfloat16, device="cuda")
lib = P._lib.load()
side = torch.cuda.Stream()


def run(st):
    P._lib.check(lib.pkv_attention_sparse(dm.handle, ctypes.byref(cache), 1, q.data_ptr(), out.data_ptr(),
                                          pos.data_ptr(), n_q, st))


run(side.cuda_stream)
torch.cuda.synchronize()
n = 10
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side):
    for _ in range(n):
        run(side.cuda_stream)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
flops = 4.0 * H * dk * float((pos.long() + 1).sum())
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PKV_")}, "ms": round(ms, 3),
                  "tflops": round(flops / ms / 1e9, 1)}))
