"""One narrow-projection launch per shape for ncu (python tools/ncu_proj.py; SHAPE=wo SPLITS=2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib  # noqa: E402
lib = _lib.load()
shapes = {"wqkv": (6144, 4096), "wo": (4096, 4096), "wgu": (28672, 4096), "wd": (4096, 14336)}
N, K = shapes[os.environ.get("SHAPE", "wo")]
sp = int(os.environ.get("SPLITS", "2"))
W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
x3 = torch.randn(96, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(32, N, device="cuda")
part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(lib.pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, 0, part.data_ptr(),
                                   cnt.data_ptr(), sp, st))
torch.cuda.synchronize()
