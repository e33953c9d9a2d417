import ctypes, sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import __graft_entry__; __graft_entry__.build()
import paper_2602_02579_b200 as P
from test_gpu_kernels import _attn_setup, _attn_reference
for (H,Hkv,dk,s,n_q,perm) in [(32,8,128,4096,819,False),(8,8,128,1000,100,True),(32,8,128,8192,1639,False)]:
    cfg, dm, lay, kp, vp, pages, pos, q, cache = _attn_setup(torch, P, H, Hkv, dk, s, n_q, perm, seed=H + s)
    out = torch.zeros((n_q, H, lay.dkp), dtype=torch.bfloat16, device="cuda")
    P._lib.check(P._lib.load().pkv_attention_sparse(dm.handle, ctypes.byref(cache), 1, q.data_ptr(), out.data_ptr(), pos.data_ptr(), n_q, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = _attn_reference(torch, 1, kp, vp, pages, pos, q, H, Hkv, dk, s)
    got = out[..., :dk].float()
    e = (got - want).abs()
    print(H,Hkv,dk,s,n_q, "max", e.max().item(), "mean", e.mean().item())
    er = e.amax(dim=(1,2))
    idx = torch.argsort(er, descending=True)[:8]
    print(" worst rows", idx.tolist(), "pos", pos[idx].tolist(), er[idx].tolist())
    eh = e.amax(dim=(0,2)); print(" per head max", [round(x,3) for x in eh.tolist()[:8]])
    # error vs position bucket
    for b in range(0, s, s//8):
        m = (pos >= b) & (pos < b + s//8)
        if m.any(): print("  pos", b, round(e[m].max().item(),4), round(e[m].mean().item(),5))
