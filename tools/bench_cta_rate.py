"""Single-CTA streaming rate of the tcgen05 GEMM for different tile widths (what bounds
the narrow projections): M = 128 (one CTA), K large, operands L2-resident."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib
lib = _lib.load()
for bn, N in [(96, 96), (128, 128), (256, 256), (256, 512)]:
    K = 8192
    A = torch.randn(128, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.zeros(128, N, device="cuda")
    side = torch.cuda.Stream()
    for _ in range(2):
        _lib.check(lib.pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, 128, N, K, C.data_ptr(), N, bn, 0, side.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(10):
            _lib.check(lib.pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, 128, N, K, C.data_ptr(), N, bn, 0, side.cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    ctas = (N + bn - 1) // bn
    per_cta_bytes = (128 + bn) * K * 2
    print(json.dumps({"bn": bn, "N": N, "ctas": ctas, "us": round(us, 2), "per_cta_GBps": round(per_cta_bytes / us / 1e3, 1),
                      "per_ktile_ns": round(us * 1e3 / (K / 64), 1)}), flush=True)
