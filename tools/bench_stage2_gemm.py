"""Graph-timed Stage-II GEMM shapes (k = 6554 selected rows, Llama-3-8B) through
pkv_gemm_bf16 (EPI=0: EPI_F32, EPI=2: EPI_RESID).  PKV_GEMM_SK=1 enables the stream-K tail,
PKV_GEMM_RASTER=g the grouped raster, PKV_LIB an alternative build."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib  # noqa: E402
lib = _lib.load()
M = int(os.environ.get("M", "6554"))
EPI = int(os.environ.get("EPI", "0"))
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
res = {}
for name, (N, K) in shapes.items():
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
    C = torch.zeros(M, N, device="cuda")
    side = torch.cuda.Stream()
    def run(i, st):
        _lib.check(lib.pkv_gemm_bf16(A.data_ptr(), K, Ws[i % 2].data_ptr(), K, M, N, K, C.data_ptr(), N, 256, EPI, st))
    C.zero_(); run(0, side.cuda_stream); torch.cuda.synchronize()
    want = A[:300].float() @ Ws[0][:].float().t()
    err = float((C[:300] - want).abs().max() / want.abs().max())
    n = 10
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for i in range(n):
            run(i, side.cuda_stream)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    res[name] = {"us": round(us, 1), "tflops": round(2 * M * N * K / us / 1e6, 1), "rel_err": err}
    del A, Ws, C
print(json.dumps({"lib": os.environ.get("PKV_LIB", "default"), "epi": EPI, **res}))
