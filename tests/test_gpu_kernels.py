"""Kernel-level GPU tests: each sm_100a kernel against a plain fp32 torch
reference (GEMM, attention) or the CPU oracle (assembly, top-k)."""

import ctypes

import numpy as np
import pytest

from oracle import pikv_oracle as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (300, 512, 4096, 256), (7, 8, 8, 256),
                                      (1000, 640, 448, 128), (6144, 96, 4096, 96), (129, 96, 72, 96)])
def test_gemm_matches_fp32_reference(built, M, N, K, bn):
    torch = _torch()
    P = built
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K), generator=g, device="cuda").to(torch.bfloat16)
    C = torch.full((M, N), float("nan"), device="cuda")
    rc = P._lib.load().pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, M, N, K, C.data_ptr(), N, bn, 0,
                                     torch.cuda.current_stream().cuda_stream)
    P._lib.check(rc)
    torch.cuda.synchronize()
    want = A.float() @ B.float().t()
    err = (C - want).abs().max().item()
    assert err <= 1e-3 * max(1.0, want.abs().max().item()), err


@pytest.mark.parametrize("M,N,K,epi", [(128, 256, 64, 0), (300, 512, 4096, 2), (6554, 512, 4096, 0), (7, 8, 8, 2)])
def test_gemm_fp16_operands(built, M, N, K, epi):
    """The Stage-II operand format: fp16 A and B (epilogue bit 0x100), fp32 accumulation."""
    torch = _torch()
    P = built
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (torch.randn((M, K), generator=g, device="cuda") * 4).half()
    B = (torch.randn((N, K), generator=g, device="cuda") * 300).half()  # pre-scaled weights span ~2^8
    C0 = torch.randn((M, N), generator=g, device="cuda")
    C = C0.clone() if epi == 2 else torch.full((M, N), float("nan"), device="cuda")
    P._lib.check(P._lib.load().pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, M, N, K, C.data_ptr(), N, 256,
                                             0x100 | epi, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = A.double() @ B.double().t() + (C0.double() if epi == 2 else 0)
    err = ((C.double() - want).abs().max() / want.abs().max()).item()
    assert err < 1e-5, err


def test_gemm_residual_epilogue(built):
    torch = _torch()
    P = built
    M, N, K = 200, 512, 256
    A = torch.randn((M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K), device="cuda").to(torch.bfloat16)
    C0 = torch.randn((M, N), device="cuda")
    C = C0.clone()
    P._lib.check(P._lib.load().pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, M, N, K, C.data_ptr(), N, 256, 2,
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = C0 + A.float() @ B.float().t()
    assert (C - want).abs().max().item() < 1e-3


def _attn_setup(torch, P, H, Hkv, dk, s, n_q, perm_pages, seed):
    cfg = P.ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hkv, head_dim=dk, hidden_dim=H * dk, ffn_dim=256,
                        vocab_size=64)
    dm = P.DeviceModel.random(cfg, seed=1)
    lay = cfg.layout()
    g = torch.Generator(device="cuda").manual_seed(seed)
    pool_tokens = -(-s // 128) * 128
    n_pages = pool_tokens // 128
    L = cfg.n_layers
    kp = torch.zeros((L, Hkv, pool_tokens, lay.dkp), dtype=torch.float16, device="cuda")
    vp = torch.zeros_like(kp)
    kp[..., :dk] = torch.randn((L, Hkv, pool_tokens, dk), generator=g, device="cuda").half()
    vp[..., :dk] = torch.randn((L, Hkv, pool_tokens, dk), generator=g, device="cuda").half()
    pages = torch.randperm(n_pages, generator=g, device="cuda").int() if perm_pages else \
        torch.arange(n_pages, dtype=torch.int32, device="cuda")
    pos = torch.sort(torch.randperm(s, generator=g, device="cuda")[:n_q])[0].int()
    q = torch.zeros((n_q, H, lay.dkp), dtype=torch.float16, device="cuda")
    q[..., :dk] = torch.randn((n_q, H, dk), generator=g, device="cuda").half()
    cache = P._lib.Cache(kp.data_ptr(), vp.data_ptr(), pool_tokens, pages.data_ptr(), s, 0, 0, 0, 0, 0)
    return cfg, dm, lay, kp, vp, pages, pos, q, cache


def _attn_reference(torch, layer, kp, vp, pages, pos, q, H, Hkv, dk, s):
    # logical token t -> slot pages[t//128]*128 + t%128
    t = torch.arange(s, device="cuda")
    slot = pages.long()[t // 128] * 128 + t % 128
    K = kp[layer][:, slot, :dk].float()   # [Hkv, s, dk]
    V = vp[layer][:, slot, :dk].float()
    G = H // Hkv
    out = torch.empty((q.shape[0], H, dk), device="cuda")
    mask = t[None, :] <= pos.long()[:, None]
    for h in range(H):
        sc = (q[:, h, :dk].float() @ K[h // G].t()) / dk ** 0.5
        sc = sc.masked_fill(~mask, float("-inf"))
        out[:, h] = torch.softmax(sc, dim=-1) @ V[h // G]
    return out


@pytest.mark.parametrize("H,Hkv,dk,s,n_q,perm", [(32, 8, 128, 4096, 819, False), (4, 2, 64, 2048, 410, True),
                                                 (8, 8, 128, 1000, 100, True), (2, 1, 4, 300, 64, False)])
def test_sparse_attention_matches_fp32_reference(built, H, Hkv, dk, s, n_q, perm):
    torch = _torch()
    P = built
    cfg, dm, lay, kp, vp, pages, pos, q, cache = _attn_setup(torch, P, H, Hkv, dk, s, n_q, perm, seed=H + s)
    out = torch.zeros((n_q, H, lay.dkp), dtype=torch.float16, device="cuda")
    layer = 1
    P._lib.check(P._lib.load().pkv_attention_sparse(dm.handle, ctypes.byref(cache), layer, q.data_ptr(),
                                                    out.data_ptr(), pos.data_ptr(), n_q,
                                                    torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = _attn_reference(torch, layer, kp, vp, pages, pos, q, H, Hkv, dk, s)
    got = out[..., :dk].float()
    err = (got - want).abs().max().item()
    cos = torch.nn.functional.cosine_similarity(got.flatten(), want.flatten(), dim=0).item()
    # fp16 P and output (2^-11 relative), fp32 accumulation
    assert err < 5e-3 and cos > 0.99999, (err, cos)


@pytest.mark.parametrize("hkv,dk,lens", [(2, 128, [300, 1, 517, 128]),    # 8 tokens per TMA group
                                          (8, 128, [3, 1, 2, 261, 130]),     # Llama geometry, 4 per group
                                          (4, 64, [1, 1, 1, 1, 1, 1, 1, 77])])  # one run per token
def test_assembly_is_fp16_of_reference_keys(built, hkv, dk, lens):
    """The assembly (ragged chunk boundaries, a context length that is not a multiple of the
    TMA-staged form's token group) is the reference's stitch + RoPE rebase, rounded to fp16
    bit for bit.  The TMA-staged form runs in a subprocess (its switch is read once)."""
    torch = _torch()
    P = built
    cfg_o = O.Cfg(n_layers=3, n_heads=4 * hkv, n_kv_heads=hkv, head_dim=dk, hidden_dim=4 * hkv * dk, ffn_dim=256,
                  vocab_size=64, rope_theta=500000.0)
    rng = np.random.default_rng(5)
    chunks = []
    for ci, t in enumerate(lens):
        kn = [O.bf16_round(rng.standard_normal((t, hkv, dk)).astype(np.float32) * 3) for _ in range(3)]
        vv = [O.bf16_round(rng.standard_normal((t, hkv, dk)).astype(np.float32)) for _ in range(3)]
        chunks.append(O.Chunk(chunk_id=ci, fp="fp", token_ids=rng.integers(0, 64, t), k_nr=kn, v=vv))
    ref = O.stitch(chunks, cfg_o)
    cfg = P.ModelConfig(**cfg_o.json())
    dch = [P.ChunkKV(c.chunk_id, "fp", c.token_ids, c.k_nr, c.v) for c in chunks]
    cache = P.assemble(dch, cfg)
    torch.cuda.synchronize()
    s = cache.context_length
    kp = cache.k_pool[:, :, :s, :dk].permute(0, 2, 1, 3)  # [L, s, Hkv, dk]
    vp = cache.v_pool[:, :, :s, :dk].permute(0, 2, 1, 3)
    for li in range(3):
        want_k = torch.from_numpy(ref.keys[li]).cuda().half()
        want_v = torch.from_numpy(ref.values[li]).cuda().half()
        assert torch.equal(kp[li].view(torch.int16), want_k.view(torch.int16))  # RNE of the f32 key
        assert torch.equal(vp[li].view(torch.int16), want_v.view(torch.int16))
        # key + residual plane = the reference's f32 key to 2^-22 relative (2^-25 absolute
        # where the residual is an fp16 subnormal)
        k2 = cache.k2_pool[li, :, :s, :dk].permute(1, 0, 2).float()
        planes = (kp[li].float() + k2).double().cpu().numpy()
        refk = ref.keys[li].astype(np.float64)
        assert np.all(np.abs(planes - refk) <= np.abs(refk) * 2.0 ** -22 + 2.0 ** -25)
        # the f32 view equals the reference's keys_rebased bit for bit
        assert np.array_equal(cache.keys_rebased[li], ref.keys[li])
        assert np.array_equal(cache.values[li], ref.values[li])


@pytest.mark.parametrize("n,k,mode", [(32768, 6554, "rand"), (2048, 410, "ties"), (5, 0, "rand"), (5, 5, "rand"),
                                      (3000, 1, "ties"), (100000, 26215, "rand"), (7, 3, "allequal"),
                                      (1000, 500, "signed")])
def test_topk_matches_reference_rule(built, n, k, mode):
    P = built
    rng = np.random.default_rng(n + k)
    if mode == "rand":
        v = rng.random(n).astype(np.float32)
    elif mode == "ties":
        v = rng.integers(0, 20, n).astype(np.float32) / 7
    elif mode == "allequal":
        v = np.full(n, 0.25, dtype=np.float32)
    else:
        v = (rng.standard_normal(n) * 3).astype(np.float32)
        v[::17] = 0.0
        v[::19] = -0.0
    assert P.top_k_indices(v, k) == O.topk_ascending(v, k)


def test_topk_rejects_non_finite(built):
    P = built
    with pytest.raises(P.NumericsError):
        P.top_k_indices(np.array([np.nan, 1.0], dtype=np.float32), 1)


def test_fuse_layers_bit_exact(built):
    P = built
    rng = np.random.default_rng(3)
    per = rng.random((32, 4096)).astype(np.float32) * 1e-3
    assert np.array_equal(P.fuse_layers(per), O.layer_mean(per))


@pytest.mark.parametrize("N,K,m,splits,resid", [(4096, 4096, 32, 0, 0), (384, 1024, 7, 3, 1), (6144, 4096, 32, 1, 0),
                                                  # stream-K: one m-tile cut into 15 pieces; wd shape on 96 CTAs
                                                  (128, 4096, 5, 0, 1), (4096, 14336, 32, -96, 1)])
def test_narrow_projection_is_fp32_faithful(built, N, K, m, splits, resid):
    """EPI_PROJ: out (+)= x . W^T for <= 32 fp32 rows given as 3 exact scaled fp16 planes
    (x = hi + 2^-11 mid + 2^-22 lo, include/pkv.h)."""
    torch = _torch()
    P = built
    g = torch.Generator(device="cuda").manual_seed(N + K)
    W = (torch.randn((N, K), generator=g, device="cuda") * 64).half()
    x = torch.randn((m, K), generator=g, device="cuda")
    x[:, ::7] *= 1e-3  # small activations: their lower planes exercise the plane scales
    hi = x.half()
    r1 = (x - hi.float()) * 2048
    mid = r1.half()
    lo = ((r1 - mid.float()) * 2048).half()
    # exact, except below ~2^-22 where the planes are subnormal (error <= 2^-46)
    rec = hi.double() + mid.double() / 2048 + lo.double() / 2048 ** 2
    assert float((rec - x.double()).abs().max()) <= 2.0 ** -46
    x3 = torch.zeros((96, K), dtype=torch.float16, device="cuda")
    x3[:m], x3[32:32 + m], x3[64:64 + m] = hi, mid, lo
    out = torch.randn((m, N), generator=g, device="cuda")
    base = out.clone()
    part = torch.empty(16 * ((N + 127) // 128) * 128 * 32, device="cuda")
    cnt = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
    P._lib.check(P._lib.load().pkv_proj_narrow(W.data_ptr(), N, K, x3.data_ptr(), K, m, out.data_ptr(), N, resid,
                                                part.data_ptr(), cnt.data_ptr(), splits,
                                                torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = x.double() @ W.double().t() + (base.double() if resid else 0)
    err = ((out.double() - want).abs().max() / want.abs().max()).item()
    assert err < 1e-5, err
    assert int(cnt.sum().item()) == 0  # split counters are reset for the next launch


_SK_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import torch
import paper_2602_02579_b200 as P
lib = P._lib.load()
M, N, K = 6554, 6144, 1024   # 26 x 24 = 624 tiles: a 32-tile tail on 74 CTA pairs
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
B = torch.randn((N, K), generator=g, device="cuda").to(torch.bfloat16)
outs = []
for _ in range(2):
    C = torch.full((M, N), float("nan"), device="cuda")
    P._lib.check(lib.pkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, M, N, K, C.data_ptr(), N, 256, 0,
                                   torch.cuda.current_stream().cuda_stream))
    outs.append(C)
torch.cuda.synchronize()
want = A.float() @ B.float().t()
err = (outs[0] - want).abs().max().item()
assert err <= 1e-3 * want.abs().max().item(), err
assert torch.equal(outs[0], outs[1]), "stream-K tail is not deterministic"
print("ok", err)
"""


def test_gemm_stream_k_tail_opt_in(built, tmp_path):
    """PKV_GEMM_SK=1 (read once per process, hence the subprocess): the last wave's
    tiles split into k pieces over all CTA pairs, summed in piece order."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "sk.py"
    script.write_text(_SK_SCRIPT)
    env = dict(os.environ, PKV_GEMM_SK="1")
    r = subprocess.run([sys.executable, str(script), root], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_opt_in_variants():
    """The opt-in kernel variants whose switches are read once per process -- the TMA-staged
    assembly (PKV_ASM_TMA=1), the grouped GEMM raster (PKV_GEMM_RASTER=2: partial groups
    on every GEMM test shape), the one-tile attention (PKV_ATTN_ONE=1) and the
    one-thread-per-row attention (PKV_ATTN_ROW=1) -- rerun the kernel tests in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PKV_ASM_TMA="1", PKV_GEMM_RASTER="2", PKV_ATTN_ONE="1", PKV_ATTN_PERSIST="0")
    tests = ["tests/test_gpu_kernels.py::test_assembly_is_fp16_of_reference_keys",
             "tests/test_gpu_kernels.py::test_sparse_attention_matches_fp32_reference",
             "tests/test_gpu_kernels.py::test_gemm_matches_fp32_reference",
             "tests/test_gpu_kernels.py::test_gemm_fp16_operands", "tests/test_gpu_kernels.py::test_gemm_residual_epilogue"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *tests], cwd=root,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    # one thread per Q-tile row, one CTA per unit (PKV_ATTN_PERSIST=0 PKV_ATTN_ROW=1), and the
    # round-1 two-tile kernel with 8 softmax warps per tile (PKV_ATTN_PERSIST=0)
    # and the persistent kernel with S(j+1) in two key halves (PKV_ATTN_SPLIT_S=1)
    for extra in ({"PKV_ATTN_PERSIST": "0", "PKV_ATTN_ROW": "1"}, {"PKV_ATTN_PERSIST": "0"},
                  {"PKV_ATTN_SPLIT_S": "1"}):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                            "tests/test_gpu_kernels.py::test_sparse_attention_matches_fp32_reference"], cwd=root,
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    env = dict(os.environ, PKV_ATTN_ROW="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_kernels.py::test_sparse_attention_matches_fp32_reference"], cwd=root,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
