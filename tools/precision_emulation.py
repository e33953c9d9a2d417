"""Stage-II precision emulation at depth (CPU, torch): which operand format keeps the
recomputed K/V within the north star's max-abs 2e-2 at L = 32?

Runs the reference arithmetic (f64 accumulation, f32 storage) next to GPU-like schemes
on the same weights / context / selection, layer by layer, and prints per-layer K/V
max-abs errors (fp32 tap and stored) plus first-logit errors of an fp32-faithful final
pass over each scheme's repaired cache.  Weights are N(0,1)/sqrt(fan_in) rounded to
bf16 (the shared inputs); chunk K/V are N(0,1) bf16.  Not the reference's RNG stream:
this is a numerics study, not a parity test.

Schemes (operand format of every tensor-core input; accumulation fp32 everywhere):
  bf16        current Stage II: bf16 activations / P / attention out, bf16 cache
  bf16_kv32   bf16, but the K/V projection on exact fp32 activations
  fp16        fp16 activations / P / attention out, fp16 cache (weights exact in fp16)
  fp16_bfc    fp16 activations, bf16 cache storage
  bf16x2      bf16 hi+lo split of every activation (2 MMAs per GEMM), bf16 cache
"""
import argparse
import math
import time

import torch

f64, f32 = torch.float64, torch.float32


def rnd(x, fmt):
    if fmt == "f32":
        return x.to(f32)
    if fmt == "bf16":
        return x.to(f32).to(torch.bfloat16).to(f32)
    if fmt == "fp16":
        return x.to(f32).to(torch.float16).to(f32)
    if fmt == "bf16x2":
        x = x.to(f32)
        hi = x.to(torch.bfloat16).to(f32)
        return hi + (x - hi).to(torch.bfloat16).to(f32)
    raise ValueError(fmt)


def rope(x, pos, theta):  # x [n, heads, d] -> rotated, f64 factors
    d = x.shape[-1]
    inv = theta ** (-torch.arange(0, d, 2, dtype=f64) / d)
    ang = pos.to(f64)[:, None] * inv[None, :]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    w = x.to(f64)
    out = torch.empty_like(w)
    out[..., 0::2] = w[..., 0::2] * c - w[..., 1::2] * s
    out[..., 1::2] = w[..., 0::2] * s + w[..., 1::2] * c
    return out


def rms(h, eps=1e-5):
    w = h.to(f64)
    return (w / torch.sqrt((w * w).mean(-1, keepdim=True) + eps)).to(f32)


def attend(q, K, V, pos_q, pos_kv, grp, fmt_q, fmt_p, ref):
    """q [n,H,dk] K/V [t,Hkv,dk] -> [n, H*dk] (f32)."""
    n, H, dk = q.shape
    vis = pos_kv[None, :] <= pos_q[:, None]
    scl = 1.0 / math.sqrt(dk)
    out = torch.empty((n, H, dk), dtype=f32)
    for h in range(H):
        g = h // grp
        if ref:
            sc = (q[:, h].to(f64) @ K[:, g].to(f64).T).to(f32).to(f64) * float(torch.tensor(scl, dtype=f32))
            sc[~vis] = -math.inf
            e = torch.exp(sc - sc.max(1, keepdim=True).values)
            p = (e / e.sum(1, keepdim=True)).to(f32)
            out[:, h] = (p.to(f64) @ V[:, g].to(f64)).to(f32)
        else:
            sc = rnd(q[:, h], fmt_q) @ K[:, g].T * scl  # fp32 accumulate
            sc[~vis] = -math.inf
            e = torch.exp(sc - sc.max(1, keepdim=True).values)
            l = e.sum(1, keepdim=True)
            out[:, h] = (rnd(e, fmt_p) @ V[:, g]) / l
    return out.reshape(n, H * dk)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--D", type=int, default=4096)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--Hkv", type=int, default=8)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--V", type=int, default=4096)
    ap.add_argument("--s", type=int, default=2048)
    ap.add_argument("--k", type=int, default=410)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--theta", type=float, default=5e5)
    ap.add_argument("--schemes", default="bf16,bf16_kv32,fp16,fp16_bfc,bf16x2")
    a = ap.parse_args()
    torch.manual_seed(0)
    L, D, H, Hkv, F, s, k, m = a.L, a.D, a.H, a.Hkv, a.F, a.s, a.k, a.m
    dk = D // H
    grp = H // Hkv
    bfw = lambda r, c: (torch.randn(r, c, dtype=f32) / math.sqrt(r)).to(torch.bfloat16).to(f32)
    embed = torch.randn(a.V, D, dtype=f32).to(torch.bfloat16).to(f32)
    head = bfw(D, a.V)
    tok = torch.randint(0, a.V, (s,))
    qtok = torch.randint(0, a.V, (m,))
    sel = torch.sort(torch.randperm(s)[:k]).values
    pos = torch.arange(s)
    ps = pos[sel]
    schemes = a.schemes.split(",")
    fmt = {"bf16": ("bf16", "bf16", "bf16"), "bf16_kv32": ("bf16", "f32", "bf16"), "fp16": ("fp16", "fp16", "fp16"),
           "fp16_bfc": ("fp16", "fp16", "bf16"), "bf16x2": ("bf16x2", "bf16x2", "bf16")}
    # state per scheme: residual h, cache K/V (stored format)
    h = {"ref": embed[tok[sel]].clone()}
    for sc in schemes:
        h[sc] = embed[tok[sel]].clone()
    caches = {}
    layers = []
    t0 = time.time()
    for l in range(L):
        W = dict(wq=bfw(D, H * dk), wk=bfw(D, Hkv * dk), wv=bfw(D, Hkv * dk), wo=bfw(H * dk, D), wg=bfw(D, F),
                 wu=bfw(D, F), wd=bfw(F, D))
        layers.append(W)
        knr = torch.randn(s, Hkv, dk, dtype=f32).to(torch.bfloat16).to(f32)
        vctx = torch.randn(s, Hkv, dk, dtype=f32).to(torch.bfloat16).to(f32)
        krot = rope(knr, pos, a.theta).to(f32)
        # reference
        x = rms(h["ref"])
        mm = lambda A, B: (A.to(f64) @ B.to(f64)).to(f32)
        q = rope(mm(x, W["wq"]).view(k, H, dk), ps, a.theta).to(f32)
        kk = rope(mm(x, W["wk"]).view(k, Hkv, dk), ps, a.theta).to(f32)
        vv = mm(x, W["wv"]).view(k, Hkv, dk)
        K = krot.clone()
        Vc = vctx.clone()
        K[sel], Vc[sel] = kk, vv
        caches.setdefault("ref", []).append((K, Vc))
        att = attend(q, K, Vc, ps, pos, grp, None, None, True)
        hr = h["ref"] + mm(att, W["wo"])
        y = rms(hr)
        g = mm(y, W["wg"]).to(f64)
        act = (g / (1 + torch.exp(-g))).to(f32) * mm(y, W["wu"])
        h["ref"] = hr + mm(act, W["wd"])
        ref_k, ref_v = kk, vv
        line = [f"L{l:02d}"]
        for sc in schemes:
            fa, fkv, fc = fmt[sc]
            x = rms(h[sc])
            xa = rnd(x, fa)
            q = rope((xa @ W["wq"]).view(k, H, dk), ps, a.theta).to(f32)
            xk = rnd(x, fkv)
            kk = rope((xk @ W["wk"]).view(k, Hkv, dk), ps, a.theta).to(f32)
            vv = (xk @ W["wv"]).view(k, Hkv, dk)
            K = rnd(krot, fc)
            Vc = rnd(vctx, fc)
            K[sel], Vc[sel] = rnd(kk, fc), rnd(vv, fc)
            caches.setdefault(sc, []).append((K, Vc))
            ek = max((kk - ref_k).abs().max().item(), (vv - ref_v).abs().max().item())
            es = max((K[sel] - ref_k).abs().max().item(), (Vc[sel] - ref_v).abs().max().item())
            att = attend(q, K, Vc, ps, pos, grp, fa, fa if fa != "bf16x2" else "bf16x2", False)
            hr = h[sc] + rnd(att, fa) @ W["wo"]
            y = rnd(rms(hr), fa)
            g = (y @ W["wg"]).to(f64)
            act = (g / (1 + torch.exp(-g))).to(f32) * (y @ W["wu"])
            h[sc] = hr + rnd(act, fa) @ W["wd"]
            line.append(f"{sc}: tap {ek:.4f} stored {es:.4f}")
        print(" | ".join(line), f"({time.time() - t0:.0f}s)", flush=True)
    # fp32-faithful final pass (reference arithmetic) over each scheme's cache
    def final(cache):
        hq = embed[qtok].clone()
        pq = s + torch.arange(m)
        pall = torch.cat([pos, pq])
        mm = lambda A, B: (A.to(f64) @ B.to(f64)).to(f32)
        for l, W in enumerate(layers):
            x = rms(hq)
            q = rope(mm(x, W["wq"]).view(m, H, dk), pq, a.theta).to(f32)
            kk = rope(mm(x, W["wk"]).view(m, Hkv, dk), pq, a.theta).to(f32)
            vv = mm(x, W["wv"]).view(m, Hkv, dk)
            K, Vc = cache[l]
            att = attend(q, torch.cat([K, kk]), torch.cat([Vc, vv]), pq, pall, grp, None, None, True)
            hr = hq + mm(att, W["wo"])
            y = rms(hr)
            g = mm(y, W["wg"]).to(f64)
            hq = hr + mm((g / (1 + torch.exp(-g))).to(f32) * mm(y, W["wu"]), W["wd"])
        return mm(rms(hq[-1:]), head)[0]
    lr = final(caches["ref"])
    for sc in schemes:
        lg = final(caches[sc])
        cos = float((lg.to(f64) @ lr.to(f64)) / (lg.to(f64).norm() * lr.to(f64).norm()))
        print(f"logits {sc}: max abs {(lg - lr).abs().max().item():.5f} cos {cos:.8f}", flush=True)


if __name__ == "__main__":
    main()
