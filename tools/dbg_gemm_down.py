import os, sys
sys.path.insert(0, '/root/repo')
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib
lib = _lib.load()
for (M, N, K) in [(512, 4096, 14336), (6554, 4096, 14336), (6554, 4096, 4096), (512, 256, 14336)]:
    torch.manual_seed(0)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.zeros(M, N, device="cuda")
    _lib.check(lib.pkv_gemm_bf16(A.data_ptr(), K, W.data_ptr(), K, M, N, K, C.data_ptr(), N, 256, 0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = A.float() @ W.float().t()
    print(M, N, K, "nan_C", bool(C.isnan().any()), "nan_want", bool(want.isnan().any()), "err", float((C - want).abs().max() / want.abs().max()))
