"""Eager narrow-projection launches for an ncu duration list (tools/proj_durations.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib  # noqa: E402
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
cfgs = [(128, 64, 1), (128, 256, 1), (128, 1024, 1), (128, 4096, 1), (128, 4096, 2), (128, 4096, 4),
        (4096, 4096, 1), (4096, 4096, 2), (4096, 4096, 4), (28672, 4096, 1)]
for (N, K, sp) in cfgs:
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    x3 = torch.randn(96, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(32, N, device="cuda")
    part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
    cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    print("cfg", N, K, sp, flush=True)
    for _ in range(4):
        _lib.check(lib.pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, 0,
                                       part.data_ptr(), cnt.data_ptr(), sp, st))
    torch.cuda.synchronize()
