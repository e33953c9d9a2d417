"""Isolated timing of the narrow-pass projection (EPI_PROJ GEMM) per Llama layer shape and
split count, weights rotated over copies larger than L2.  python tools/bench_proj.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import __graft_entry__

__graft_entry__.build()
from paper_2602_02579_b200 import _lib  # noqa: E402

lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
shapes = {"wqkv": (6144, 4096), "wo": (4096, 4096), "wgu": (28672, 4096), "wd": (4096, 14336)}
splits = [int(x) for x in os.environ.get("SPLITS", "0,-64,-74,-96,-112,-128,-140,3").split(",")]
resid = int(os.environ.get("RESID", "0"))
for name, (N, K) in shapes.items():
    copies = max(2, int(400e6 // (N * K * 2)))
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
    x3 = torch.randn(96, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(32, N, device="cuda")
    part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
    cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
    for sp in splits:
        for i in range(3):
            _lib.check(lib.pkv_proj_narrow(Ws[i % copies].data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, resid,
                                           part.data_ptr(), cnt.data_ptr(), sp, st))
        torch.cuda.synchronize()
        n = 20
        # graph-captured so host-side launch cost (tensor-map encodes) cannot pace the GPU
        side = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(n):
                _lib.check(lib.pkv_proj_narrow(Ws[i % copies].data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(),
                                               N, resid, part.data_ptr(), cnt.data_ptr(), sp, side.cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        print(json.dumps({"w": name, "splits": sp, "us": round(us, 2), "GBps": round(N * K * 2 / us / 1e3, 1)}),
              flush=True)
    # correctness vs fp32 (x = sum of planes)
    x = x3[:32].float() + x3[32:64].float() + x3[64:].float()
    want = x @ Ws[(n - 1) % copies].float().t()
    if not resid:
        print(json.dumps({"w": name, "max_rel_err": float(((out - want).abs().max() / want.abs().max()).item())}))
    del Ws
    torch.cuda.empty_cache()
