// K1: position-independent KV assembly (reference chunkstore.py:99-140 with
// rope_apply tensor.py:89-114) and the K8 standalone scatter (replace_entries,
// chunkstore.py:143-160).
//
// Chunk store layout (input): per chunk, bf16 [L][t_c][Hkv][dkp], keys unrotated.
// Paged cache (output):       fp16 [L][Hkv][pool_tokens][dkp]; slot of token t is
//                             page_table[t/128]*128 + t%128.
// Keys are rotated with the float64 cos/sin table (identical bytes to the
// oracle's rope_cos_sin), products and the difference rounded exactly like the
// reference's float64 numpy expression, then rounded f64->f32->fp16: the stored
// key is fp16(reference f32 key) bit for bit, and the residual plane k2 holds
// fp16(f32 key - key) for the fp32-faithful narrow passes.  Values are copied
// (bf16 -> fp16 is exact for |v| >= 2^-14 and within 2^-25 below).
#include "kernels.cuh"

namespace pkv {


__device__ __forceinline__ void rope_pair64(float e, float o, double c, double s, float& oe, float& oo) {
  double de = (double)e, dd = (double)o;
  oe = (float)__dsub_rn(__dmul_rn(de, c), __dmul_rn(dd, s));
  oo = (float)__dadd_rn(__dmul_rn(de, s), __dmul_rn(dd, c));
}

// one thread = one (token, 16-byte column vector); loops over layers and heads
__global__ void __launch_bounds__(128) assemble_kernel(ChunkView cv, int s, int l0, int l1, int Hkv, int dkp,
                                                       int head_dim,
                                                       const double* __restrict__ rcos,
                                                       const double* __restrict__ rsin, const int32_t* page_table,
                                                       __half* k_pool, __half* v_pool,
                                                       long pool_tokens, __half* k2_pool) {
  pdl_entry();
  const int vecs = dkp / 8;
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)s * vecs) return;
  const int t = (int)(gid / vecs);
  const int c = (int)(gid - (long)t * vecs);
  const int ch = cv.src_chunk[t];
  const int loc = cv.src_local[t];
  const int tc = cv.chunk_len[ch];
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(cv.k_nr[ch]);
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(cv.v[ch]);
  const long slot = (long)page_table[t >> 7] * 128 + (t & 127);
  const int half = head_dim >> 1;
  // this thread's 4 pairs of cos/sin stay in registers for all L*Hkv rows
  double cs[4], sn[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    int i = c * 4 + p;
    cs[p] = i < half ? rcos[(long)t * half + i] : 1.0;
    sn[p] = i < half ? rsin[(long)t * half + i] : 0.0;
  }
  for (int l = l0; l < l1; ++l) {
    const long src_row = ((long)l * tc + loc) * Hkv;
    const long dst_layer = (long)l * Hkv * pool_tokens;
    for (int h = 0; h < Hkv; ++h) {
      const long so = (src_row + h) * dkp + c * 8;
      uint4 kv = __ldg(reinterpret_cast<const uint4*>(kb + so));
      uint4 vv = __ldg(reinterpret_cast<const uint4*>(vb + so));
      uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w}, vw[4] = {vv.x, vv.y, vv.z, vv.w}, o[4], o2[4], ov[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float e = bf16_lo(w[p]), od = bf16_hi(w[p]);
        float re = e, ro = od;
        if (2 * (c * 4 + p) < head_dim) rope_pair64(e, od, cs[p], sn[p], re, ro);
        // the fp16 cache key is RNE(f32 key); the residual plane carries the rest
        split2h_pack(re, ro, o[p], o2[p]);
        ov[p] = pack_f16(bf16_lo(vw[p]), bf16_hi(vw[p]));
      }
      const long dofs = (dst_layer + (long)h * pool_tokens + slot) * dkp + c * 8;
      *reinterpret_cast<uint4*>(k_pool + dofs) = make_uint4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<uint4*>(v_pool + dofs) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
      if (k2_pool != nullptr) *reinterpret_cast<uint4*>(k2_pool + dofs) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
    }
  }
}

// TMA-staged form (opt-in, PKV_ASM_TMA=1; see assemble_launch).  CTA = a group of TG consecutive context tokens (TG | 128,
// so the group's cache slots are consecutive inside one page) over layers l0..l1:
//   loads   per layer, one 1-D bulk copy per run of tokens from the same chunk (a token's
//           row [Hkv][dkp] is contiguous in the chunk store and consecutive tokens of a
//           chunk are adjacent) for K and for V -> a 3-stage shared-memory ring
//           completing on an mbarrier's transaction count;
//   compute 16-byte vectors from shared memory: RoPE in float64 (as above), fp16 key +
//           fp16 residual, bf16 -> fp16 values, into a double-buffered output tile
//           [plane][Hkv][TG][dkp];
//   stores  per layer, 3*Hkv bulk copies shared -> global (TG*dkp*2 contiguous bytes per
//           head and plane), left in flight while the next layer is computed.
// Every HBM byte moves through the TMA engine in >= 1 KB transactions; the SM only
// touches shared memory.
constexpr int ASM_STAGES = 3;
constexpr int ASM_THREADS = 128;

__host__ __device__ inline int asm_tg(int Hkv, int dkp) {  // tokens per CTA: ~8 KB per plane and layer
  const int row = Hkv * dkp * 2;
  int tg = 8;
  while (tg > 1 && tg * row > 8192) tg >>= 1;
  return tg;
}
__host__ __device__ inline int asm_smem(int Hkv, int dkp, int head_dim) {
  const int plane = asm_tg(Hkv, dkp) * Hkv * dkp * 2;
  return ASM_STAGES * 2 * plane + 2 * 3 * plane + 2 * asm_tg(Hkv, dkp) * (head_dim / 2) * 8 + ASM_STAGES * 8 + 16;
}

__global__ void __launch_bounds__(ASM_THREADS) assemble_tma_kernel(ChunkView cv, int s, int l0, int l1, int Hkv,
                                                                   int dkp, int head_dim,
                                                                   const double* __restrict__ rcos,
                                                                   const double* __restrict__ rsin,
                                                                   const int32_t* page_table, __half* k_pool,
                                                                   __half* v_pool, long pool_tokens,
                                                                   __half* k2_pool) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int TG = asm_tg(Hkv, dkp);
  const int C = dkp / 8;  // 16-byte vectors per head row
  const int row_b = Hkv * dkp * 2;
  const int plane = TG * row_b;
  const int half = head_dim >> 1;
  const int t0 = blockIdx.x * TG;
  const int nt = min(TG, s - t0);
  const int nl = l1 - l0;
  uint8_t* in = smem;                              // [STAGES][K|V][TG][Hkv][dkp] bf16
  uint8_t* out = in + ASM_STAGES * 2 * plane;      // [2][K|V|K2][Hkv][TG][dkp] fp16
  double* tcs = reinterpret_cast<double*>(out + 2 * 3 * plane);  // [TG][half]
  double* tsn = tcs + TG * half;
  uint64_t* full = reinterpret_cast<uint64_t*>(tsn + TG * half);
  const int tid = threadIdx.x;
  const int planes_out = k2_pool != nullptr ? 3 : 2;

  // runs of tokens that are adjacent in one chunk (thread 0 only; at most TG runs)
  int run_tok[8], run_ch[8], run_loc[8], run_len[8], n_runs = 0;
  if (tid == 0) {
    for (int j = 0; j < ASM_STAGES; ++j) mbar_init(&full[j], 1);
    fence_barrier_init();
  }
  pdl_entry();
  if (tid == 0) {
    for (int j = 0; j < nt; ++j) {
      const int ch = cv.src_chunk[t0 + j], loc = cv.src_local[t0 + j];
      if (n_runs > 0 && run_ch[n_runs - 1] == ch && run_loc[n_runs - 1] + run_len[n_runs - 1] == loc) {
        ++run_len[n_runs - 1];
      } else {
        run_tok[n_runs] = j;
        run_ch[n_runs] = ch;
        run_loc[n_runs] = loc;
        run_len[n_runs] = 1;
        ++n_runs;
      }
    }
  }
  auto issue = [&](int i) {  // layer l0 + i -> stage i % STAGES (thread 0)
    const int l = l0 + i, st = i % ASM_STAGES;
    uint8_t* dk = in + st * 2 * plane;
    mbar_expect_tx(&full[st], (uint32_t)(2 * nt * row_b));
    for (int r = 0; r < n_runs; ++r) {
      const int tc = cv.chunk_len[run_ch[r]];
      const long src = ((long)l * tc + run_loc[r]) * Hkv * dkp;
      const uint32_t bytes = (uint32_t)(run_len[r] * row_b);
      bulk_g2s(dk + run_tok[r] * row_b, reinterpret_cast<const __nv_bfloat16*>(cv.k_nr[run_ch[r]]) + src, bytes,
               &full[st]);
      bulk_g2s(dk + plane + run_tok[r] * row_b, reinterpret_cast<const __nv_bfloat16*>(cv.v[run_ch[r]]) + src,
               bytes, &full[st]);
    }
  };
  if (tid == 0)
    for (int i = 0; i < nl && i < ASM_STAGES; ++i) issue(i);
  for (int e = tid; e < nt * half; e += ASM_THREADS) {
    const int j = e / half, i = e - j * half;
    tcs[e] = rcos[(long)(t0 + j) * half + i];
    tsn[e] = rsin[(long)(t0 + j) * half + i];
  }
  const long slot0 = (long)page_table[t0 >> 7] * 128 + (t0 & 127);
  const int nvec = nt * Hkv * C;
  __syncthreads();  // barriers initialised

  for (int i = 0; i < nl; ++i) {
    const int st = i % ASM_STAGES, ob = i & 1, l = l0 + i;
    mbar_wait(&full[st], (uint32_t)((i / ASM_STAGES) & 1));
    const uint8_t* ik = in + st * 2 * plane;
    // a thread's vectors: v = tid + ASM_THREADS * j (<= 4 per thread at the default sizes)
    constexpr int VMAX = 8;
    uint4 kr[VMAX], vr[VMAX];
#pragma unroll
    for (int j = 0; j < VMAX; ++j) {
      const int v = tid + ASM_THREADS * j;
      if (v < nvec) {
        kr[j] = *reinterpret_cast<const uint4*>(ik + (long)v * 16);
        vr[j] = *reinterpret_cast<const uint4*>(ik + plane + (long)v * 16);
      }
    }
    if (tid < planes_out * Hkv) bulk_wait_read<1>();  // this thread's stores of layer i-2 have left out[ob]
    __syncthreads();                    // in[st] consumed, out[ob] free, cos/sin staged
    if (tid == 0 && i + ASM_STAGES < nl) issue(i + ASM_STAGES);
    uint8_t* o = out + ob * 3 * plane;
#pragma unroll
    for (int j = 0; j < VMAX; ++j) {
      const int v = tid + ASM_THREADS * j;
      if (v < nvec) {
        const int c = v % C, h = (v / C) % Hkv, tok = v / (C * Hkv);
        const uint32_t w[4] = {kr[j].x, kr[j].y, kr[j].z, kr[j].w}, vw[4] = {vr[j].x, vr[j].y, vr[j].z, vr[j].w};
        uint32_t ok[4], o2[4], ov[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int pi = c * 4 + p;
          float re = bf16_lo(w[p]), ro = bf16_hi(w[p]);
          if (pi < half) rope_pair64(re, ro, tcs[tok * half + pi], tsn[tok * half + pi], re, ro);
          split2h_pack(re, ro, ok[p], o2[p]);
          ov[p] = pack_f16(bf16_lo(vw[p]), bf16_hi(vw[p]));
        }
        const long oo = ((long)(h * TG + tok) * C + c) * 16;
        *reinterpret_cast<uint4*>(o + oo) = make_uint4(ok[0], ok[1], ok[2], ok[3]);
        *reinterpret_cast<uint4*>(o + plane + oo) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
        *reinterpret_cast<uint4*>(o + 2 * plane + oo) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid < planes_out * Hkv) {  // one bulk store per (plane, head)
      const int pl = tid / Hkv, h = tid - pl * Hkv;
      __half* pool = pl == 0 ? k_pool : pl == 1 ? v_pool : k2_pool;
      const long dofs = (((long)l * Hkv + h) * pool_tokens + slot0) * dkp;
      bulk_s2g(pool + dofs, o + pl * plane + (long)h * TG * dkp * 2, (uint32_t)(nt * dkp * 2));
      bulk_commit();
    }
  }
  if (tid < planes_out * Hkv) bulk_wait<0>();
}

int assemble_launch(const ChunkView& cv, int s, int l0, int l1, int Hkv, int dkp, int head_dim, const double* rcos,
                    const double* rsin, const int32_t* page_table, void* k_pool, void* v_pool, long pool_tokens,
                    void* k2_pool, cudaStream_t stream) {
  if (s <= 0) return PKV_OK;
  // the TMA-staged form is opt-in: on the C3 step it measured no faster than the
  // LDG/STG.128 kernel below (that one already moves 10.7 GB at ~89 % of the copy peak,
  // profiles/r02/ncu_summary.json), score pass 8.0 vs 7.4 ms (profiles/r02/ab_ttft_r02d.txt)
  static const bool tma = getenv("PKV_ASM_TMA") && getenv("PKV_ASM_TMA")[0] == '1';
  const int tg = asm_tg(Hkv, dkp);
  if (tma && tg * Hkv * (dkp / 8) <= 8 * ASM_THREADS) {
    const int smem = asm_smem(Hkv, dkp, head_dim);
    static int configured = 0;
    if (smem > configured) {
      cudaFuncSetAttribute(assemble_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured = smem;
    }
    launch_k(assemble_tma_kernel, (unsigned)ceil_div((long)s, tg), ASM_THREADS, smem, stream, cv, s, l0, l1, Hkv, dkp,
             head_dim, rcos, rsin, page_table, reinterpret_cast<__half*>(k_pool), reinterpret_cast<__half*>(v_pool),
             pool_tokens, reinterpret_cast<__half*>(k2_pool));
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("assemble_tma_kernel");
    return PKV_OK;
  }
  const long threads = (long)s * (dkp / 8);
  launch_k(assemble_kernel, ceil_div(threads, 128), 128, 0, stream, 
      cv, s, l0, l1, Hkv, dkp, head_dim, rcos, rsin, page_table, reinterpret_cast<__half*>(k_pool),
      reinterpret_cast<__half*>(v_pool), pool_tokens, reinterpret_cast<__half*>(k2_pool));
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("assemble_kernel");
  return PKV_OK;
}

// f32 view of one cache layer as the reference stores it ([s][Hkv][dk]).
// Keys of entries not yet recomputed are re-derived exactly from the chunk store
// (rotation in float64 -> f32, bit-identical to keys_rebased); recomputed entries
// and values come from the fp32 taps when given, else from the fp16 cache (keys: the
// fp16 key plus its residual plane).
__global__ void cache_view_kernel(ChunkView cv, int use_chunks, int s, int layer, int Hkv, int dkp, int head_dim,
                                  const double* rcos, const double* rsin, const int32_t* page_table,
                                  const __half* pool, const __half* pool2, long pool_tokens, int is_key, float* out) {
  pdl_entry();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)s * Hkv * head_dim;
  if (gid >= total) return;
  const int d = (int)(gid % head_dim);
  const long th = gid / head_dim;
  const int h = (int)(th % Hkv);
  const int t = (int)(th / Hkv);
  if (use_chunks) {
    const int ch = cv.src_chunk[t], loc = cv.src_local[t], tc = cv.chunk_len[ch];
    const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(is_key ? cv.k_nr[ch] : cv.v[ch]);
    const long row = (((long)layer * tc + loc) * Hkv + h) * dkp;
    if (!is_key) {
      out[gid] = __bfloat162float(base[row + d]);
      return;
    }
    const int i = d >> 1, half = head_dim >> 1;
    float e = __bfloat162float(base[row + 2 * i]), o = __bfloat162float(base[row + 2 * i + 1]);
    float re, ro;
    rope_pair64(e, o, rcos[(long)t * half + i], rsin[(long)t * half + i], re, ro);
    out[gid] = (d & 1) ? ro : re;
  } else {
    const long slot = (long)page_table[t >> 7] * 128 + (t & 127);
    const long o = (((long)layer * Hkv + h) * pool_tokens + slot) * dkp + d;
    out[gid] = __half2float(pool[o]) + (pool2 != nullptr ? __half2float(pool2[o]) : 0.f);
  }
}

int cache_view_launch(const ChunkView& cv, int use_chunks, int s, int layer, int Hkv, int dkp, int head_dim,
                      const double* rcos, const double* rsin, const int32_t* page_table, const void* pool,
                      const void* pool2, long pool_tokens, int is_key, float* out, cudaStream_t stream) {
  const long total = (long)s * Hkv * head_dim;
  if (total <= 0) return PKV_OK;
  launch_k(cache_view_kernel, ceil_div(total, 256), 256, 0, stream, cv, use_chunks, s, layer, Hkv, dkp, head_dim, rcos,
                                                             rsin, page_table,
                                                             reinterpret_cast<const __half*>(pool),
                                                             reinterpret_cast<const __half*>(pool2), pool_tokens,
                                                             is_key, out);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("cache_view_kernel");
  return PKV_OK;
}

// scatter fp32 rows [n][Hkv][dk] into the fp16 cache at token indices idx
__global__ void scatter_kernel(const int32_t* idx, int n, int layer, int Hkv, int dkp, int head_dim,
                               const float* src, const int32_t* page_table, __half* pool,
                               long pool_tokens, __half* pool2) {
  pdl_entry();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)n * Hkv * (dkp / 2);
  if (gid >= total) return;
  const int d = 2 * (int)(gid % (dkp / 2));
  const long rh = gid / (dkp / 2);
  const int h = (int)(rh % Hkv);
  const int r = (int)(rh / Hkv);
  const int t = idx[r];
  const long slot = (long)page_table[t >> 7] * 128 + (t & 127);
  const float* row = src + ((long)r * Hkv + h) * head_dim;
  const float v0 = d < head_dim ? row[d] : 0.f, v1 = d + 1 < head_dim ? row[d + 1] : 0.f;
  uint32_t p1, p2;
  split2h_pack(v0, v1, p1, p2);
  const long o = (((long)layer * Hkv + h) * pool_tokens + slot) * dkp + d;
  *reinterpret_cast<uint32_t*>(pool + o) = p1;
  if (pool2 != nullptr) *reinterpret_cast<uint32_t*>(pool2 + o) = p2;
}

// pool2 (nullable): residual plane of a key pool
int scatter_launch(const int32_t* idx, int n, int layer, int Hkv, int dkp, int head_dim, const float* src,
                   const int32_t* page_table, void* pool, long pool_tokens, void* pool2, cudaStream_t stream) {
  const long total = (long)n * Hkv * (dkp / 2);
  if (total <= 0) return PKV_OK;
  launch_k(scatter_kernel, ceil_div(total, 256), 256, 0, stream, idx, n, layer, Hkv, dkp, head_dim, src, page_table,
                                                          reinterpret_cast<__half*>(pool), pool_tokens,
                                                          reinterpret_cast<__half*>(pool2));
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("scatter_kernel");
  return PKV_OK;
}

}  // namespace pkv
