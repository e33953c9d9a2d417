"""Per-CTA timeline of one Stage-II attention launch at the C3 shape (PKV_ATTN_CTA_TRACE=1):
SM occupancy over the launch, gaps between consecutive CTAs of an SM, the tail, and the
time per K/V page of each CTA.  python tools/attn_cta_trace.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ["PKV_ATTN_CTA_TRACE"] = "1"
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
for _ in range(3):
    P._lib.check(lib.pkv_attention_sparse(dm.handle, ctypes.byref(cache), 1, q.data_ptr(), out.data_ptr(),
                                          pos.data_ptr(), n_q, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
T = 128 // (H // Hkv)
n_ctas = -(-(-(-n_q // T)) // 2) * Hkv
buf = np.zeros((n_ctas, 4), dtype=np.uint64)
lib.pkv_debug_attn_cta_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.pkv_debug_attn_cta_trace(buf.ctypes.data_as(ctypes.c_void_p), n_ctas) == 0
st, en, sm, pg = buf[:, 0].astype(np.int64), buf[:, 1].astype(np.int64), buf[:, 2], buf[:, 3].astype(np.int64)
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3
span = en.max()
busy = {}
gaps = []
for smid in np.unique(sm):
    idx = np.where(sm == smid)[0]
    idx = idx[np.argsort(st[idx])]
    busy[int(smid)] = float(np.sum(en[idx] - st[idx]))
    gaps += list(st[idx][1:] - en[idx][:-1])
last_end = np.array([max(en[sm == x]) for x in np.unique(sm)])
dur = en - st
res = {"ctas": int(n_ctas), "sms": int(len(busy)), "span_us": round(float(span), 1),
       "busy_frac": round(sum(busy.values()) / (span * len(busy)), 4),
       "median_gap_us": round(float(np.median(gaps)), 2), "max_gap_us": round(float(np.max(gaps)), 2),
       "first_sm_done_us": round(float(last_end.min()), 1), "sm_done_p10_us": round(float(np.percentile(last_end, 10)), 1),
       "us_per_page_median": round(float(np.median(dur / pg)), 3),
       "us_per_page_p10_p90": [round(float(np.percentile(dur / pg, 10)), 3), round(float(np.percentile(dur / pg, 90)), 3)],
       "fixed_us_fit": None}
A = np.vstack([pg, np.ones_like(pg)]).T.astype(np.float64)
coef = np.linalg.lstsq(A, dur, rcond=None)[0]
res["fixed_us_fit"] = {"us_per_page": round(float(coef[0]), 3), "us_per_cta": round(float(coef[1]), 2)}
print(json.dumps(res))
