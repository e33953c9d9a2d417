"""Per-tile %globaltimer timeline of one narrow-pass attention CTA (PKV_S1_TRACE=1): the C3
scoring pass is run once; the trace is the last launch's CTA (0,0,0).
    python tools/s1_trace.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PKV_S1_TRACE"] = "1"
import numpy as np
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2602_02579_b200 as P  # noqa: E402
from paper_2602_02579_b200.pipeline import PrefillPipeline, random_device_chunks  # noqa: E402

cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.random(cfg, seed=0)
chunks = random_device_chunks(cfg, 16, 2048, seed=1)
pipe = PrefillPipeline(dm, chunks, 32, 0.2)
pipe.set_query(np.random.default_rng(7).integers(0, cfg.vocab_size, 32))
pipe.score_select()
pipe.score_select()
torch.cuda.synchronize()
lib = P._lib.load()
buf = np.zeros(6 * 64, dtype=np.uint64)
lib.pkv_debug_s1_trace.argtypes = [ctypes.c_void_p]
assert lib.pkv_debug_s1_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf.reshape(6, 64).astype(np.int64)
t0 = t[t > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
names = ["softmax saw S", "softmax P done", "mma saw K/V", "mma issued PV", "tma issued", "markers"]
n = int(np.sum(t[0] > 0))
print(f"tiles traced: {n}; markers (prologue done, softmax loop done, partials written): {rel[5, :3].round(2)}; "
      f"fresh-key CTA start / staged / end: {rel[5, [4, 6, 5]].round(2)}")
for j in range(n):
    print(f"j={j:2d} " + "  ".join(f"{names[e][:14]:>14s} {rel[e, j]:7.2f}" for e in range(5)))
d = np.diff(rel[0, :n])
print(f"softmax period median {np.nanmedian(d):.3f} us; P(j) - S(j) median {np.nanmedian(rel[1, :n] - rel[0, :n]):.3f} us; "
      f"S(j+1) - P(j) median {np.nanmedian(rel[0, 1:n] - rel[1, :n - 1]):.3f} us")

# scoring pass 2 (s1_score_tc_kernel), CTA (0,0,0): start, Q planes in TMEM, S(j) seen, done
sb = np.zeros(64, dtype=np.uint64)
lib.pkv_debug_s1_score_trace.argtypes = [ctypes.c_void_p]
if lib.pkv_debug_s1_score_trace(sb.ctypes.data_as(ctypes.c_void_p)) == 0 and sb[0] > 0:
    t = sb.astype(np.int64)
    rel2 = np.where(t > 0, (t - t[0]) / 1e3, np.nan)
    nt = int(np.sum(t[4:] > 0))
    d2 = np.diff(rel2[4:4 + nt])
    print(f"score pass 2: Q in TMEM {rel2[1]:.2f} us, tiles {nt}, first S {rel2[4]:.2f}, done {rel2[2]:.2f}, "
          f"tile period median {np.nanmedian(d2):.3f} us")
