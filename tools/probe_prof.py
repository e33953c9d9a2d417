import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
import __graft_entry__
__graft_entry__.build()
import paper_2602_02579_b200 as P
from paper_2602_02579_b200 import synthetic as S, _lib
cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
dm = P.DeviceModel.synthetic(cfg, seed=0)
chunks = S.chunks(cfg, 4, 2048, 0, dm.fingerprint)
cache = P.assemble(chunks, cfg, fp32_taps=False)
P.score_kvshare_l1(dm, cfg, cache); torch.cuda.synchronize()
_lib.timing(True)
t0=time.perf_counter(); P.score_kvshare_l1(dm, cfg, cache); torch.cuda.synchronize(); t1=time.perf_counter()
ph=_lib.timing_collect(); _lib.timing(False)
print("kvshare 8k", round((t1-t0)*1e3,1), "ms", {k:(round(v[0],2), v[1]) for k,v in ph.items() if v[1]})
_lib.timing(True)
t0=time.perf_counter(); P.score_cacheblend_l1(dm, cfg, cache); torch.cuda.synchronize(); t1=time.perf_counter()
ph=_lib.timing_collect(); _lib.timing(False)
print("cacheblend 8k", round((t1-t0)*1e3,1), "ms", {k:(round(v[0],2), v[1]) for k,v in ph.items() if v[1]})
