"""Per-CTA timeline of narrow-projection launches (PKV_GEMM_TRACE=1 python tools/proj_trace.py)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PKV_GEMM_TRACE"] = "1"
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2602_02579_b200 import _lib  # noqa: E402
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
names = ["entry", "prologue", "acc_ready", "part_stored", "cnt_acq", "reduced", "written"]
for (N, K, sp) in [(128, 4096, 0), (4096, 4096, 0), (6144, 4096, 0), (4096, 14336, 0), (28672, 4096, 0), (4096, 14336, 3)]:
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    x3 = torch.randn(96, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(32, N, device="cuda")
    part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
    cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
    buf = np.zeros((1024, 8), dtype=np.uint64)
    for it in range(3):
        lib.pkv_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)
        _lib.check(lib.pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, 32, out.data_ptr(), N, 0,
                                       part.data_ptr(), cnt.data_ptr(), sp, st))
        lib.pkv_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)
    rows = buf[buf[:, 0] > 0].astype(np.int64)
    t0 = rows[:, 0].min()
    rel = np.where(rows > 0, rows - t0, -1)
    print(f"N={N} K={K} sp={sp} ctas={len(rows)}")
    for i, nm in enumerate(names):
        col = rel[:, i][rel[:, i] >= 0]
        if len(col):
            print(f"  {nm:12s} n={len(col):4d} min={col.min()/1e3:7.2f} med={np.median(col)/1e3:7.2f} max={col.max()/1e3:7.2f} us")
    if len(rows) <= 4:
        print("  per-CTA:", (rel[:, :7] / 1e3).round(2).tolist())
