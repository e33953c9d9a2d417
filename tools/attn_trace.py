"""Per-page timeline of one Stage-II attention CTA (PKV_ATTN_TRACE=1 python tools/attn_trace.py)."""
import ctypes
import os
import sys

os.environ["PKV_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from test_gpu_kernels import _attn_setup  # noqa: E402

H, Hkv, dk, s, n_q = 32, 8, 128, 32768, 6554
cfg, dm, lay, kp, vp, pages, pos, q, cache = _attn_setup(torch, P, H, Hkv, dk, s, n_q, False, seed=3)
out = torch.zeros((n_q, H, lay.dkp), dtype=torch.bfloat16, device="cuda")
lib = P._lib.load()
buf = np.zeros((9, 64), dtype=np.uint64)
for it in range(3):
    P._lib.check(lib.pkv_attention_sparse(dm.handle, ctypes.byref(cache), 1, q.data_ptr(), out.data_ptr(),
                                          pos.data_ptr(), n_q, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
lib.pkv_debug_attn_trace(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.astype(np.int64)
t0 = t[0, 0]
names = ["sA", "sB", "pA", "pB", "pvA", "pvB", "kv", "ldK", "ldV"]
print("page  " + "  ".join(f"{n:>7s}" for n in names) + "   smA   smB  wakeA wakeB  periodA (ns)")
for j in range(8, 24):
    row = [t[e, j] - t0 for e in range(9)]
    smA, smB = t[2, j] - t[0, j], t[3, j] - t[1, j]
    wA, wB = t[4, j] - t[2, j], t[5, j] - t[3, j]
    per = t[0, j + 1] - t[0, j]
    lat = t[6, j] - t[7, j + 1]  # page j+1: issue -> seen ready by the MMA warp
    print(f"{j:4d}  " + "  ".join(f"{v:7d}" for v in row) + f"  {smA:5d} {smB:5d} {wA:6d} {wB:5d} {per:7d}  ld{j+1}->{lat}")
