"""Does tcgen05.mma kind::f16 accept A = fp16 with B = bf16 (idesc a_fmt 0, b_fmt 1)?
Runs the Stage-II GEMM kernel with the A-format bit cleared on fp16 data."""
import sys
sys.path.insert(0, ".")
import torch
import __graft_entry__ as G
G.build()
import paper_2602_02579_b200 as P
for (M, N, K) in [(128, 256, 64), (300, 512, 4096), (6554, 6144, 4096)]:
    A = (torch.randn((M, K), device="cuda") * 3).half()
    B = torch.randn((N, K), device="cuda").to(torch.bfloat16)
    C = torch.full((M, N), float("nan"), device="cuda")
    P._lib.check(P._lib.load().pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, M, N, K, C.data_ptr(), N, 256, 0x100,
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = A.double() @ B.double().t()
    wrong = A.view(torch.bfloat16).double() @ B.double().t()
    print(M, N, K, "err vs fp16-A", (C.double() - want).abs().max().item(), "scale", want.abs().max().item(),
          "err vs bf16-reinterpret", (C.double() - wrong).abs().max().item())
