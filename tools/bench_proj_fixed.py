import json, os, sys
sys.path.insert(0, '/root/repo')
import torch
import __graft_entry__; __graft_entry__.build()
from paper_2602_02579_b200 import _lib
lib = _lib.load()
for (N, K, sp) in [(128, 64, 1), (4096, 64, 1), (4096, 512, 1), (4096, 4096, 1), (4096, 4096, 4), (128, 4096, 1), (128, 4096, 4), (4096, 1024, 1), (18944, 4096, 1)]:
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    x3 = torch.randn(96, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(32, N, device="cuda")
    part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
    cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    for _ in range(2):
        _lib.check(lib.pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, 0, part.data_ptr(), cnt.data_ptr(), sp, side.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    n = 20
    with torch.cuda.graph(g, stream=side):
        for i in range(n):
            _lib.check(lib.pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, 0, part.data_ptr(), cnt.data_ptr(), sp, side.cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(json.dumps({"N": N, "K": K, "splits": sp, "us": round(e0.elapsed_time(e1) / n * 1e3, 2), "MB": N*K*2/1e6}), flush=True)
