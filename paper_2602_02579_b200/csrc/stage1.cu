// Narrow query pass kernels (reference model.py:370-402 query_pass; scoring
// selection.py:64-86; finalize recompute.py:105-125).  Everything here is
// fp32-faithful: the m query rows stay fp32, projections run on tcgen05 with a
// scaled 3-way fp16 split of the activations (x = hi + 2^-11 mid + 2^-22 lo exactly,
// split3s in common.cuh) against the pre-scaled fp16 weights, attention runs on
// tcgen05 with fp16 planes (s1_attn_tc.cu) or fp32 SIMT, and the per-token score
// reductions run in float64 like the reference.
#include <algorithm>
#include <mutex>
#include "kernels.cuh"
#include "comm.cuh"

namespace pkv {

// --------------------------------------------------------------- split / norm
__device__ __forceinline__ void split3(float x, __half& hi, __half& mid, __half& lo) { split3s(x, hi, mid, lo); }

// x [m][ld] fp32 (first `cols` valid) -> X3 [96][ldx] fp16 rows i, 32+i, 64+i
__global__ void split3_kernel(const float* x, int m, int cols, long ld, __half* x3, long ldx) {
  pdl_entry();
  const int i = blockIdx.y;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ldx; c += gridDim.x * blockDim.x) {
    float v = (i < m && c < cols) ? x[(long)i * ld + c] : 0.f;
    __half a, b, d;
    split3(v, a, b, d);
    x3[(long)i * ldx + c] = a;
    x3[(long)(32 + i) * ldx + c] = b;
    x3[(long)(64 + i) * ldx + c] = d;
  }
}

int split3_launch(const float* x, int m, int cols, long ld, void* x3, long ldx, cudaStream_t st) {
  dim3 grid(ceil_div(ldx, 256) > 64 ? 64 : ceil_div(ldx, 256), 32);
  launch_k(split3_kernel, grid, 256, 0, st, x, m, cols, ld, reinterpret_cast<__half*>(x3), ldx);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("split3_kernel");
  return PKV_OK;
}

// RMSNorm of each row in float64 (reference tensor.py:78-86), output fp32 and/or
// the scaled fp16 3-way split (rows >= m of X3 are zero-filled by this kernel) and/or a
// 16-bit copy (fp16, or bf16 when y16_bf16).
__global__ void rmsnorm_kernel(const float* h, int m, int D, long ld, const float* gain, double eps, float* y,
                               __half* x3, long ldx, void* y16, int y16_bf16) {
  pdl_entry();
  const int i = blockIdx.x;
  __shared__ double red[32];
  double acc = 0.0;
  if (i < m) {
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      double v = (double)h[(long)i * ld + c];
      acc += v * v;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double inv = 1.0 / sqrt(red[0] / (double)D + eps);
  // columns of this CTA: gridDim.y column chunks of the row (the next GEMM reads
  // x3 columns [0, ld) only); every chunk recomputes the row's sum of squares
  const long cw = (ld + gridDim.y - 1) / gridDim.y;
  const long c0 = blockIdx.y * cw, c1 = min(ld, c0 + cw);
  for (long c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    float out = 0.f;
    if (i < m && c < D) out = (float)((double)h[(long)i * ld + c] * inv * (double)gain[c]);
    if (y && c < ld) y[(long)i * ld + c] = out;
    if (y16 && c < ld) {
      if (y16_bf16) reinterpret_cast<__nv_bfloat16*>(y16)[(long)i * ld + c] = __float2bfloat16_rn(out);
      else reinterpret_cast<__half*>(y16)[(long)i * ld + c] = __float2half_rn(out);
    }
    if (x3) {
      __half a, b, d;
      split3(out, a, b, d);
      x3[(long)i * ldx + c] = a;
      x3[(long)(32 + i) * ldx + c] = b;
      x3[(long)(64 + i) * ldx + c] = d;
    }
  }
}

// narrow-pass rows -> the 3 fp16 planes of the next projection's B operand only: one
// 256-thread CTA per plane row (32 rows; rows >= m zero-filled), the row in registers as
// float4 vectors, one f64 block reduction, 8-byte plane stores
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_x3_kernel(const float* __restrict__ h, int m, int D, long ld,
                                                         const float* __restrict__ gain, double eps,
                                                         __half* __restrict__ x3, long ldx) {
  pdl_entry();
  const int i = blockIdx.x;
  const int nvec = (int)(ld >> 2);
  float4 v[NV];
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = j * 256 + threadIdx.x;
    v[j] = (i < m && c < nvec) ? __ldg(reinterpret_cast<const float4*>(h + (long)i * ld) + c)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    acc += (double)v[j].x * v[j].x + (double)v[j].y * v[j].y + (double)v[j].z * v[j].z + (double)v[j].w * v[j].w;
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const double inv = 1.0 / sqrt(tot / (double)D + eps);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = j * 256 + threadIdx.x;
    if (c >= nvec) continue;
    const float4 g = __ldg(g4 + c);
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    if (i < m) {
      o[0] = (4 * c + 0 < D) ? (float)((double)v[j].x * inv * (double)g.x) : 0.f;
      o[1] = (4 * c + 1 < D) ? (float)((double)v[j].y * inv * (double)g.y) : 0.f;
      o[2] = (4 * c + 2 < D) ? (float)((double)v[j].z * inv * (double)g.z) : 0.f;
      o[3] = (4 * c + 3 < D) ? (float)((double)v[j].w * inv * (double)g.w) : 0.f;
    }
    uint32_t h0, m0, l0, h1, m1, l1;
    split3s_pack(o[0], o[1], h0, m0, l0);
    split3s_pack(o[2], o[3], h1, m1, l1);
    *reinterpret_cast<uint2*>(x3 + (long)i * ldx + 4 * c) = make_uint2(h0, h1);
    *reinterpret_cast<uint2*>(x3 + (long)(32 + i) * ldx + 4 * c) = make_uint2(m0, m1);
    *reinterpret_cast<uint2*>(x3 + (long)(64 + i) * ldx + 4 * c) = make_uint2(l0, l1);
  }
}

// Stage-II rows (16-bit GEMM operand only: fp16, or bf16 for the full-prefill lm_head):
// one 128-thread CTA per row, the row held in registers as float4 vectors (one coalesced
// read of h), f64 sum of squares as above
template <int NV, bool BF>
__global__ void __launch_bounds__(128) rmsnorm_y16_kernel(const float* __restrict__ h, int D, long ld,
                                                          const float* __restrict__ gain, double eps,
                                                          void* __restrict__ y16) {
  pdl_entry();
  const long i = blockIdx.x;
  const float4* src = reinterpret_cast<const float4*>(h + i * ld);
  const int nvec = (int)(ld >> 2);
  float4 v[NV];
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = j * 128 + threadIdx.x;
    v[j] = c < nvec ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc += (double)v[j].x * v[j].x + (double)v[j].y * v[j].y + (double)v[j].z * v[j].z + (double)v[j].w * v[j].w;
  }
  __shared__ double red[4];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  const double inv = 1.0 / sqrt((red[0] + red[1] + red[2] + red[3]) / (double)D + eps);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  uint2* dst = reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(y16) + i * ld);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = j * 128 + threadIdx.x;
    if (c < nvec) {
      const float4 g = __ldg(g4 + c);
      const float o0 = (4 * c + 0 < D) ? (float)((double)v[j].x * inv * (double)g.x) : 0.f;
      const float o1 = (4 * c + 1 < D) ? (float)((double)v[j].y * inv * (double)g.y) : 0.f;
      const float o2 = (4 * c + 2 < D) ? (float)((double)v[j].z * inv * (double)g.z) : 0.f;
      const float o3 = (4 * c + 3 < D) ? (float)((double)v[j].w * inv * (double)g.w) : 0.f;
      dst[c] = BF ? make_uint2(pack_bf16(o0, o1), pack_bf16(o2, o3)) : make_uint2(pack_f16(o0, o1), pack_f16(o2, o3));
    }
  }
}

// rows = max(m, 32) blocks when x3 is given so that the padding rows get zeros
template <bool BF>
static void launch_rms_y16(int nv, int m, cudaStream_t st, const float* h, int D, long ld, const float* gain,
                           double eps, void* out) {
  if (nv <= 2) launch_k(rmsnorm_y16_kernel<2, BF>, m, 128, 0, st, h, D, ld, gain, eps, out);
  else if (nv <= 4) launch_k(rmsnorm_y16_kernel<4, BF>, m, 128, 0, st, h, D, ld, gain, eps, out);
  else if (nv <= 8) launch_k(rmsnorm_y16_kernel<8, BF>, m, 128, 0, st, h, D, ld, gain, eps, out);
  else launch_k(rmsnorm_y16_kernel<16, BF>, m, 128, 0, st, h, D, ld, gain, eps, out);
}

int rmsnorm_launch(const float* h, int m, int D, long ld, const float* gain, double eps, float* y, void* x3, long ldx,
                   void* ybf, cudaStream_t st, int y16_bf16) {
  if (m <= 0 && !x3) return PKV_OK;  // e.g. a token-parallel rank without rows
  if (ybf && !y && !x3 && ld % 4 == 0 && ld <= 128 * 4 * 16) {
    const int nv = ceil_div(ld / 4, 128);
    if (y16_bf16) launch_rms_y16<true>(nv, m, st, h, D, ld, gain, eps, ybf);
    else launch_rms_y16<false>(nv, m, st, h, D, ld, gain, eps, ybf);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("rmsnorm_y16_kernel");
    return PKV_OK;
  }
  int rows = x3 ? 32 : m;
  if (x3 && ld > ldx) return set_error(PKV_ERR_SHAPE, "rmsnorm: plane width %ld < row width %ld", ldx, ld);
  if (x3 && !y && !ybf && m <= 32 && ld % 4 == 0 && ldx % 4 == 0 && ld <= 256 * 4 * 8) {
    const int nv = ceil_div(ld / 4, 256);
    auto* o = reinterpret_cast<__half*>(x3);
    if (nv <= 1) launch_k(rmsnorm_x3_kernel<1>, 32, 256, 0, st, h, m, D, ld, gain, eps, o, ldx);
    else if (nv <= 2) launch_k(rmsnorm_x3_kernel<2>, 32, 256, 0, st, h, m, D, ld, gain, eps, o, ldx);
    else if (nv <= 4) launch_k(rmsnorm_x3_kernel<4>, 32, 256, 0, st, h, m, D, ld, gain, eps, o, ldx);
    else launch_k(rmsnorm_x3_kernel<8>, 32, 256, 0, st, h, m, D, ld, gain, eps, o, ldx);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("rmsnorm_x3_kernel");
    return PKV_OK;
  }
  const int chunks = x3 ? std::max(1, std::min(8, (int)(ld / 512))) : 1;
  if (rows <= 0) return PKV_OK;
  launch_k(rmsnorm_kernel, dim3(rows, chunks), 256, 0, st, h, m, D, ld, gain, eps, y, reinterpret_cast<__half*>(x3), ldx,
           ybf, y16_bf16);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("rmsnorm_kernel");
  return PKV_OK;
}

// split-K partials P [splits][N][96] (the 3 scaled fp16 planes' products, already times the
// weight scale) -> Y[i][n] (mode 0: store, 1: += residual)
__global__ void splitk_reduce_kernel(const float* part, int splits, int N, int m, float* y, long ldy, int mode) {
  pdl_entry();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)N * m) return;
  const int i = (int)(gid / N);
  const int n = (int)(gid - (long)i * N);
  float acc = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float* p = part + ((long)s * N + n) * 96;
    acc += fmaf(p[64 + i], 1.f / X3_LO, fmaf(p[32 + i], 1.f / X3_MID, p[i]));
  }
  float* dst = y + (long)i * ldy + n;
  if (mode == 1) *dst = *dst + acc;
  else *dst = acc;
}

int splitk_reduce_launch(const float* part, int splits, int N, int m, float* y, long ldy, int mode, cudaStream_t st) {
  const long total = (long)N * m;
  launch_k(splitk_reduce_kernel, ceil_div(total, 256), 256, 0, st, part, splits, N, m, y, ldy, mode);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("splitk_reduce_kernel");
  return PKV_OK;
}

// ------------------------------------------------------------ q/k/v of queries
// qkv fp32 [m][NQKV] (padded-head layout) -> rotated q [m][H][dkp], k [m][Hkv][dkp],
// v [m][Hkv][dkp] at positions pos0 + i; optionally append k/v (fp16, key residual plane)
// to the cache pool and emit the fp32 fresh K/V as the reference returns them ([m][Hkv][dk]).
__global__ void query_qkv_kernel(const float* qkv, int m, int H, int Hkv, int dk, int dkp, int pos0,
                                 const double* rcos, const double* rsin, float* q, float* k, float* v,
                                 __half* k_pool, __half* v_pool, long pool_tokens,
                                 const int32_t* page_table, float* fresh_k, float* fresh_v, __half* k2_pool,
                                 __half* q3, int G, int RB) {
  pdl_entry();
  const int heads = H + 2 * Hkv;
  const long total = (long)m * heads * (dkp / 2);
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int pi = (int)(gid % (dkp / 2));
  const long rh = gid / (dkp / 2);
  const int hh = (int)(rh % heads);
  const int i = (int)(rh / heads);
  const int pos = pos0 + i;
  const float* src = qkv + ((long)i * heads + hh) * dkp + 2 * pi;
  float e = src[0], o = src[1];
  const bool is_v = hh >= H + Hkv;
  if (!is_v && 2 * pi < dk) {
    const int half = dk >> 1;
    double c = rcos[(long)pos * half + pi], s = rsin[(long)pos * half + pi];
    double de = e, dd = o;
    float re = (float)__dsub_rn(__dmul_rn(de, c), __dmul_rn(dd, s));
    float ro = (float)__dadd_rn(__dmul_rn(de, s), __dmul_rn(dd, c));
    e = re;
    o = ro;
  }
  if (hh < H) {
    float* d = q + ((long)i * H + hh) * dkp + 2 * pi;
    d[0] = e;
    d[1] = o;
    if (q3 != nullptr) {  // the tensor-core attention's Q planes (s1_qprep_kernel's layout)
      const int g = hh / G, rr = (hh - g * G) * m + i;
      uint32_t ph, pm, pl;
      split3h_pack(e * 64.f, o * 64.f, ph, pm, pl);
      const long base = (((long)g * RB + (rr >> 7)) * 3) * 128 + (rr & 127);
      reinterpret_cast<uint32_t*>(q3 + base * dkp)[pi] = ph;
      reinterpret_cast<uint32_t*>(q3 + (base + 128) * dkp)[pi] = pm;
      reinterpret_cast<uint32_t*>(q3 + (base + 256) * dkp)[pi] = pl;
    }
    return;
  }
  const int g = is_v ? hh - H - Hkv : hh - H;
  float* d = (is_v ? v : k) + ((long)i * Hkv + g) * dkp + 2 * pi;
  d[0] = e;
  d[1] = o;
  if (k_pool != nullptr) {
    const long slot = (long)page_table[pos >> 7] * 128 + (pos & 127);
    const long po = ((long)g * pool_tokens + slot) * dkp + 2 * pi;
    uint32_t p1, p2;
    split2h_pack(e, o, p1, p2);
    *reinterpret_cast<uint32_t*>((is_v ? v_pool : k_pool) + po) = p1;
    if (!is_v && k2_pool != nullptr) *reinterpret_cast<uint32_t*>(k2_pool + po) = p2;
  }
  float* fr = is_v ? fresh_v : fresh_k;
  if (fr != nullptr && 2 * pi < dk) {
    float* fd = fr + ((long)i * Hkv + g) * dk + 2 * pi;
    fd[0] = e;
    fd[1] = o;
  }
}

int query_qkv_launch(const float* qkv, int m, int H, int Hkv, int dk, int dkp, int pos0, const double* rcos,
                     const double* rsin, float* q, float* k, float* v, void* k_pool, void* v_pool, long pool_tokens,
                     const int32_t* page_table, float* fresh_k, float* fresh_v, void* k2_pool, cudaStream_t st,
                     void* q3) {
  const long total = (long)m * (H + 2 * Hkv) * (dkp / 2);
  const int G = H / Hkv, RB = ceil_div(m * G, 128);
  launch_k(query_qkv_kernel, ceil_div(total, 256), 256, 0, st, 
      qkv, m, H, Hkv, dk, dkp, pos0, rcos, rsin, q, k, v, reinterpret_cast<__half*>(k_pool),
      reinterpret_cast<__half*>(v_pool), pool_tokens, page_table, fresh_k, fresh_v, reinterpret_cast<__half*>(k2_pool),
      reinterpret_cast<__half*>(q3), G, RB);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("query_qkv_kernel");
  return PKV_OK;
}

// Low-layer probe (selection.py:95-124): the probed context tokens attend to the
// ASSEMBLED layer-0 entries, their own included -- overwrite the pass's fresh K (rotated)
// and V of the m rows at positions pos0.. with the cache's f32 key (fp16 k + residual
// plane k2) and value.
__global__ void probe_cache_kv_kernel(float* k, float* v, int m, int Hkv, int dk, int dkp, int pos0,
                                      const __half* k_pool, const __half* k2_pool, const __half* v_pool,
                                      long pool_tokens, const int32_t* page_table) {
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)m * Hkv * dk) return;
  const int d = (int)(gid % dk);
  const long rg = gid / dk;
  const int g = (int)(rg % Hkv), i = (int)(rg / Hkv);
  const int pos = pos0 + i;
  const long slot = (long)page_table[pos >> 7] * 128 + (pos & 127);
  const long po = ((long)g * pool_tokens + slot) * dkp + d;
  k[((long)i * Hkv + g) * dkp + d] = __half2float(k_pool[po]) + __half2float(k2_pool[po]);
  v[((long)i * Hkv + g) * dkp + d] = __half2float(v_pool[po]);
}

// Low-layer probe, kvshare (selection.py:136-142): the block's own keys' share of the
// layer-0 attention column sums, out[t] = sum_{q >= t} rows[q][t] over the block's queries
// (rows = f32 head mean of the probabilities, reference model.py:296-305).  Scores are
// recomputed exactly as s1_attn_pass1 forms the fresh-key scores (sequential f32 FMAs over
// the padded head dim, then * scale) and normalised with the pass's final row max / sum.
// kvshare: the block keys' own column sums (reference _low_layer_probe: rows of the
// block's queries over its own keys, causal).  One CTA per block key t: the (query, head)
// terms exp(s - M) / L are formed in parallel into shared memory, then summed in the
// round-1 kernel's order -- per query the heads in order in f64, rounded to f32 after the
// head mean; the queries in order in f64 -- so the result is unchanged bit for bit.
__global__ void __launch_bounds__(256) probe_diag_colsum_kernel(const float* q, const float* k, const float* Mfin,
                                                                const float* Lfin, int m, int H, int Hkv, int dk,
                                                                int dkp, float scale, float* out) {
  extern __shared__ float term[];  // [m][H]
  __shared__ float rowv[128];
  const int t = blockIdx.x;
  constexpr float LOG2E = 1.4426950408889634f;
  const int G = H / Hkv, R = m * G;
  for (int pidx = threadIdx.x; pidx < m * H; pidx += blockDim.x) {
    const int qi = pidx / H, h = pidx - qi * H;
    if (qi < t) continue;
    const int g = h / G, j = h - g * G;
    const float* qp = q + ((long)qi * H + h) * dkp;
    const float* kp = k + ((long)t * Hkv + g) * dkp;
    float sc = 0.f;
    for (int d = 0; d < dkp; ++d) sc = fmaf(qp[d], kp[d], sc);
    const float sv = sc * scale;
    const int r = g * R + j * m + qi;
    term[pidx] = ex2(fmaf(sv, LOG2E, -Mfin[r] * LOG2E)) * (1.f / Lfin[r]);
  }
  __syncthreads();
  for (int qi = t + (int)threadIdx.x; qi < m; qi += blockDim.x) {
    double acc = 0.0;
    for (int h = 0; h < H; ++h) acc += (double)term[qi * H + h];
    rowv[qi] = (float)(acc / (double)H);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double col = 0.0;
    for (int qi = t; qi < m; ++qi) col += (double)rowv[qi];
    out[t] = (float)col;
  }
}

int probe_diag_colsum_launch(const float* q, const float* k, const float* Mfin, const float* Lfin, int m, int H,
                             int Hkv, int dk, int dkp, float scale, float* out, cudaStream_t st) {
  if (m <= 0) return PKV_OK;
  if (m > 128 || (size_t)m * H * sizeof(float) > 48 * 1024)
    return set_error(PKV_ERR_ARGUMENT, "probe block of %d rows x %d heads", m, H);
  probe_diag_colsum_kernel<<<m, 256, (size_t)m * H * sizeof(float), st>>>(q, k, Mfin, Lfin, m, H, Hkv, dk, dkp, scale,
                                                                          out);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("probe_diag_colsum_kernel");
  return PKV_OK;
}

int probe_cache_kv_launch(float* k, float* v, int m, int Hkv, int dk, int dkp, int pos0, const void* k_pool,
                          const void* k2_pool, const void* v_pool, long pool_tokens, const int32_t* page_table,
                          cudaStream_t st) {
  const long total = (long)m * Hkv * dk;
  probe_cache_kv_kernel<<<ceil_div(total, 256), 256, 0, st>>>(
      k, v, m, Hkv, dk, dkp, pos0, reinterpret_cast<const __half*>(k_pool), reinterpret_cast<const __half*>(k2_pool),
      reinterpret_cast<const __half*>(v_pool), pool_tokens, page_table);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("probe_cache_kv_kernel");
  return PKV_OK;
}

// gate/up interleaved per 256 columns -> act = f32(silu64(gate)) * up
// (reference model.py:260-262 and 318-321)
// act (nullable) fp32 [m][Fp]; x3 (nullable): the 3 scaled fp16 planes of act for the next
// projection, rows i / 32+i / 64+i (valid rows only)
__global__ void silu_act_kernel(const float* gu, int m, int F, int Fp, float* act, __half* x3, long ldx) {
  pdl_entry();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)m * Fp) return;
  const int i = (int)(gid / Fp), f = (int)(gid - (long)i * Fp);
  float a = 0.f;
  if (f < F) {
    const int b = f >> 7, j = f & 127;
    const float g = gu[(long)i * 2 * Fp + b * 256 + j];
    const float u = gu[(long)i * 2 * Fp + b * 256 + 128 + j];
    const double gd = (double)g;
    a = (float)(gd / (1.0 + exp(-gd))) * u;
  }
  if (act) act[gid] = a;
  if (x3) {
    __half p, q, r;
    split3(a, p, q, r);
    x3[(long)i * ldx + f] = p;
    x3[(long)(32 + i) * ldx + f] = q;
    x3[(long)(64 + i) * ldx + f] = r;
  }
}

int silu_act_launch(const float* gu, int m, int F, int Fp, float* act, cudaStream_t st, void* x3, long ldx) {
  const long total = (long)m * Fp;
  launch_k(silu_act_kernel, ceil_div(total, 256), 256, 0, st, gu, m, F, Fp, act, reinterpret_cast<__half*>(x3),
                                                        ldx);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("silu_act_kernel");
  return PKV_OK;
}

// ------------------------------------------------------------ attention pass 1
// One CTA: KV head g, a contiguous key range, up to 128 rows r = j*m + i (head
// g*G + j, query i).  Keys t < s come from the chunk store (unrotated, rotated
// here in float64 -- exactly the reference's keys_rebased) or from the cache
// pool; keys s..s+m-1 are the queries' own fresh K/V.  Scores (already scaled,
// masked -> -inf) are written to S[g][r][t] for the scoring reduction; per-split
// online-softmax partials (m, l, O) go to the combine kernel.

// RPT rows per thread: a CTA covers ROWS = 32*RPT rows (RPT = 1 for the short fresh-key
// split next to the tensor-core path -> 4x more CTAs; 4 for long SIMT key ranges)
template <int DKP, int RPT>
__global__ void __launch_bounds__(256) s1_attn_pass1(S1Attn a) {
  pdl_entry();
  constexpr int LDQ = DKP + 4;
  constexpr int NQ = DKP / 32;  // float4 groups of output dims per thread
  constexpr int ROWS = 32 * RPT;
  extern __shared__ float sm[];
  float* Qs = sm;                  // [ROWS][LDQ]
  float* Ks = Qs + ROWS * LDQ;     // [32][LDQ]
  float* Vs = Ks + 32 * LDQ;       // [32][LDQ]
  float* Ps = Vs + 32 * LDQ;       // [ROWS][33]
  const int g = blockIdx.y;
  const int split = blockIdx.x;
  const int r0 = blockIdx.z * ROWS;
  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;

  // Q rows of this block
  for (int e = tid; e < ROWS * (DKP / 4); e += 256) {
    const int rr = e / (DKP / 4), c4 = e - rr * (DKP / 4);
    const int r = r0 + rr;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < a.R) {
      const int j = r / a.m, i = r - j * a.m;
      v = *reinterpret_cast<const float4*>(a.q + ((long)i * a.H + g * a.G + j) * DKP + c4 * 4);
    }
    *reinterpret_cast<float4*>(Qs + rr * LDQ + c4 * 4) = v;
  }

  float mrow[RPT], lrow[RPT], o[RPT][NQ][4];
#pragma unroll
  for (int x = 0; x < RPT; ++x) {
    mrow[x] = -INFINITY;
    lrow[x] = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[x][q][e] = 0.f;
  }
  int qi[RPT];  // query index of each of this thread's rows (for the causal part)
#pragma unroll
  for (int x = 0; x < RPT; ++x) {
    const int r = r0 + ty * RPT + x;
    qi[x] = r < a.R ? r % a.m : -1;
  }

  const int k_begin = a.key_base + split * a.keys_per_split;
  const int k_end = min(k_begin + a.keys_per_split, a.s_tot);
  const int half = a.dk >> 1;

  for (int t0 = k_begin; t0 < k_end; t0 += 32) {
    __syncthreads();
    // ---- K/V tile -> smem fp32
    for (int e = tid; e < 32 * (DKP / 8); e += 256) {
      const int kr = e / (DKP / 8), c8 = e - kr * (DKP / 8);
      const int t = t0 + kr;
      float kf[8], vf[8];
      if (t < k_end && t < a.s) {
        uint4 kraw, vraw, k2raw = make_uint4(0, 0, 0, 0);
        const bool from_chunk = a.src_chunks && !(a.recomp != nullptr && a.recomp[t]);
        if (from_chunk) {
          const int ch = a.src_chunk[t], loc = a.src_local[t], tc = a.chunk_len[ch];
          const long off = (((long)a.layer * tc + loc) * a.Hkv + g) * DKP + c8 * 8;
          kraw = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.ck[ch]) + off);
          vraw = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.cv[ch]) + off);
        } else {
          const long slot = (long)a.page_table[t >> 7] * 128 + (t & 127);
          const long off = ((long)g * a.pool_tokens + slot) * DKP + c8 * 8;
          kraw = *reinterpret_cast<const uint4*>(a.k_pool + off);
          vraw = *reinterpret_cast<const uint4*>(a.v_pool + off);
          k2raw = a.k2_pool != nullptr ? *reinterpret_cast<const uint4*>(a.k2_pool + off) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t kw[4] = {kraw.x, kraw.y, kraw.z, kraw.w};
        const uint32_t k2w[4] = {k2raw.x, k2raw.y, k2raw.z, k2raw.w};
        const uint32_t vw[4] = {vraw.x, vraw.y, vraw.z, vraw.w};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float e0, e1;
          const int pi = c8 * 4 + p;
          if (from_chunk) {  // bf16 chunk store, rotated here exactly like keys_rebased
            e0 = bf16_lo(kw[p]);
            e1 = bf16_hi(kw[p]);
            if (pi < half) {
              const double c = a.rcos[(long)t * half + pi], sn = a.rsin[(long)t * half + pi];
              const double de = e0, dd = e1;
              e0 = (float)__dsub_rn(__dmul_rn(de, c), __dmul_rn(dd, sn));
              e1 = (float)__dadd_rn(__dmul_rn(de, sn), __dmul_rn(dd, c));
            }
            vf[2 * p] = bf16_lo(vw[p]);
            vf[2 * p + 1] = bf16_hi(vw[p]);
          } else {  // fp16 pool key + residual plane, fp16 value
            e0 = f16_lo(kw[p]) + f16_lo(k2w[p]);
            e1 = f16_hi(kw[p]) + f16_hi(k2w[p]);
            vf[2 * p] = f16_lo(vw[p]);
            vf[2 * p + 1] = f16_hi(vw[p]);
          }
          kf[2 * p] = e0;
          kf[2 * p + 1] = e1;
        }
      } else if (t < k_end) {
        const int i = t - a.s;
        const float* ks = a.fk + ((long)i * a.Hkv + g) * DKP + c8 * 8;
        const float* vs = a.fv + ((long)i * a.Hkv + g) * DKP + c8 * 8;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          kf[p] = ks[p];
          vf[p] = vs[p];
        }
      } else {
#pragma unroll
        for (int p = 0; p < 8; ++p) kf[p] = vf[p] = 0.f;
      }
      float* kd = Ks + kr * LDQ + c8 * 8;
      float* vd = Vs + kr * LDQ + c8 * 8;
      *reinterpret_cast<float4*>(kd) = make_float4(kf[0], kf[1], kf[2], kf[3]);
      *reinterpret_cast<float4*>(kd + 4) = make_float4(kf[4], kf[5], kf[6], kf[7]);
      *reinterpret_cast<float4*>(vd) = make_float4(vf[0], vf[1], vf[2], vf[3]);
      *reinterpret_cast<float4*>(vd + 4) = make_float4(vf[4], vf[5], vf[6], vf[7]);
    }
    __syncthreads();

    // ---- scores: rows ty*4+x, keys b*8+tx
    float acc[RPT][4];
#pragma unroll
    for (int x = 0; x < RPT; ++x)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[x][b] = 0.f;
#pragma unroll 4
    for (int d = 0; d < DKP; d += 4) {
      float4 qv[RPT], kv[4];
#pragma unroll
      for (int x = 0; x < RPT; ++x) qv[x] = *reinterpret_cast<const float4*>(Qs + (ty * RPT + x) * LDQ + d);
#pragma unroll
      for (int b = 0; b < 4; ++b) kv[b] = *reinterpret_cast<const float4*>(Ks + (b * 8 + tx) * LDQ + d);
#pragma unroll
      for (int x = 0; x < RPT; ++x)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          acc[x][b] = fmaf(qv[x].x, kv[b].x, acc[x][b]);
          acc[x][b] = fmaf(qv[x].y, kv[b].y, acc[x][b]);
          acc[x][b] = fmaf(qv[x].z, kv[b].z, acc[x][b]);
          acc[x][b] = fmaf(qv[x].w, kv[b].w, acc[x][b]);
        }
    }
    // ---- scale, mask, store S, online softmax
#pragma unroll
    for (int x = 0; x < RPT; ++x) {
      const int r = r0 + ty * RPT + x;
      float tmax = -INFINITY;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int t = t0 + b * 8 + tx;
        const bool vis = qi[x] >= 0 && t < k_end && (t < a.s || (t - a.s) <= qi[x]);
        const float sv = vis ? acc[x][b] * a.scale : -INFINITY;
        acc[x][b] = sv;
        if (a.S != nullptr && r < a.R && t < k_end && t < a.s) a.S[((long)g * a.s + t) * a.R + r] = sv;
        tmax = fmaxf(tmax, sv);
      }
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
      const float m_new = fmaxf(mrow[x], tmax);
      const float corr = (mrow[x] == -INFINITY) ? 0.f : expf(mrow[x] - m_new);
      float psum = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float p = (acc[x][b] == -INFINITY) ? 0.f : expf(acc[x][b] - m_new);
        psum += p;
        Ps[(ty * RPT + x) * 33 + b * 8 + tx] = p;
      }
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
      if (m_new != -INFINITY) {
        lrow[x] = lrow[x] * corr + psum;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) o[x][q][e] *= corr;
        mrow[x] = m_new;
      }
    }
    __syncthreads();
    // ---- O += P V : rows ty*4+x, dims tx*4 + 32q + e
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
      float p[RPT];
#pragma unroll
      for (int x = 0; x < RPT; ++x) p[x] = Ps[(ty * RPT + x) * 33 + c];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 vv = *reinterpret_cast<const float4*>(Vs + c * LDQ + tx * 4 + 32 * q);
#pragma unroll
        for (int x = 0; x < RPT; ++x) {
          o[x][q][0] = fmaf(p[x], vv.x, o[x][q][0]);
          o[x][q][1] = fmaf(p[x], vv.y, o[x][q][1]);
          o[x][q][2] = fmaf(p[x], vv.z, o[x][q][2]);
          o[x][q][3] = fmaf(p[x], vv.w, o[x][q][3]);
        }
      }
    }
  }
  // ---- partials
#pragma unroll
  for (int x = 0; x < RPT; ++x) {
    const int r = r0 + ty * RPT + x;
    if (r >= a.R) continue;
    const long base = ((long)(a.split_base + split) * a.Hkv + g) * a.R + r;
    float* od = a.Opart + base * DKP;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      *reinterpret_cast<float4*>(od + tx * 4 + 32 * q) = make_float4(o[x][q][0], o[x][q][1], o[x][q][2], o[x][q][3]);
    if (tx == 0) {
      a.Mpart[base] = mrow[x];
      a.Lpart[base] = lrow[x];
    }
  }
}

// combine split partials -> attention output [m][H][dkp] fp32 and the final
// per-row (max, denominator) used by the scoring reduction
// Cfin (nullable): the row's probability mass on the context keys (splits [0, n_ctx)),
// for the context-renormalised scores
__global__ void s1_attn_combine(const float* Opart, const float* Mpart, const float* Lpart, int splits, int Hkv,
                                int R, int m, int G, int H, int dkp, float* out, float* Mfin, float* Lfin,
                                __half* x3, long ldx, int n_ctx, float* Cfin) {
  pdl_entry();
  extern __shared__ float wsp[];  // [splits rounded up to 8] rescale weight of each split (0 past splits:
                                  // the unrolled loop below reads it in 16-byte vectors)
  __shared__ float sM, sL, sC;
  const int r = blockIdx.x, g = blockIdx.y;
  if (threadIdx.x < 32) {
    float M = -INFINITY;
    for (int sp = threadIdx.x; sp < splits; sp += 32) M = fmaxf(M, Mpart[((long)sp * Hkv + g) * R + r]);
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f, Lc = 0.f;
    for (int sp = threadIdx.x; sp < splits; sp += 32) {
      const long b = ((long)sp * Hkv + g) * R + r;
      const float w = Mpart[b] != -INFINITY ? expf(Mpart[b] - M) : 0.f;
      wsp[sp] = w;
      L += Lpart[b] * w;
      if (sp < n_ctx) Lc += Lpart[b] * w;
    }
    for (int sp = splits + threadIdx.x; sp < ((splits + 7) & ~7); sp += 32) wsp[sp] = 0.f;
    for (int o = 16; o > 0; o >>= 1) {
      L += __shfl_xor_sync(0xffffffffu, L, o);
      Lc += __shfl_xor_sync(0xffffffffu, Lc, o);
    }
    if (threadIdx.x == 0) {
      sM = M;
      sL = L;
      sC = Lc / L;
    }
  }
  __syncthreads();
  const float M = sM, L = sL;
  const int j = r / m, i = r - j * m;
  for (int d = threadIdx.x; d < dkp; d += blockDim.x) {
    float acc = 0.f;
    const float* op = Opart + ((long)g * R + r) * dkp + d;
    const long sstride = (long)Hkv * R * dkp;
#pragma unroll 8
    for (int sp = 0; sp < splits; ++sp) {
      const float w = wsp[sp];  // 0 for empty splits, whose partials may be garbage
      const float v = __ldg(op + sp * sstride);
      acc = w != 0.f ? fmaf(v, w, acc) : acc;
    }
    const float o = acc / L;
    const long col = (long)(g * G + j) * dkp + d;
    out[(long)i * H * dkp + col] = o;
    if (x3 != nullptr) {  // the o-projection's B operand (3 scaled fp16 planes, rows i/32+i/64+i)
      __half p, q, rr;
      split3(o, p, q, rr);
      x3[(long)i * ldx + col] = p;
      x3[(long)(32 + i) * ldx + col] = q;
      x3[(long)(64 + i) * ldx + col] = rr;
    }
  }
  if (threadIdx.x == 0 && Mfin != nullptr) {
    Mfin[(long)g * R + r] = M;
    Lfin[(long)g * R + r] = L;
    if (Cfin != nullptr) Cfin[(long)g * R + r] = sC;
  }
}

// Combine fused with the m fresh query keys (keys s..s+m-1, fp32 K/V, causal within the
// query) when the context keys ran on the tensor cores: each CTA (row r, KV head g) scores
// its row against the fresh keys itself (a 32 x dk dot product set) instead of a separate
// SIMT split kernel, then merges them with the split partials exactly like a split.
__global__ void s1_attn_combine_fresh(const float* Opart, const float* Mpart, const float* Lpart, int splits,
                                      int Hkv, int R, int m, int G, int H, int dkp, const float* __restrict__ q,
                                      const float* __restrict__ fk, const float* __restrict__ fv, float scale,
                                      float* out, float* Mfin, float* Lfin, __half* x3, long ldx) {
  pdl_entry();
  extern __shared__ float shc[];  // wsp[splits] | sS[m] (scores, then probabilities) | sV[m][dkp]
  float* wsp = shc;
  float* sS = shc + splits;
  float* sV = sS + m;
  __shared__ float sM, sL, sWf;
  const int r = blockIdx.x, g = blockIdx.y;
  const int j = r / m, i = r - j * m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* qr = q + ((long)i * H + g * G + j) * dkp;
  for (int e = threadIdx.x; e < m * dkp; e += blockDim.x) {  // the fresh values of head g -> smem
    const int kk = e / dkp, d = e - kk * dkp;
    sV[e] = fv[((long)kk * Hkv + g) * dkp + d];
  }
  for (int kk = warp; kk < m; kk += (int)(blockDim.x >> 5)) {  // S = f32(q.k) * scale, causal
    const float* kr = fk + ((long)kk * Hkv + g) * dkp;
    float part = 0.f;
    for (int d = lane; d < dkp; d += 32) part = fmaf(qr[d], kr[d], part);
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) sS[kk] = kk <= i ? part * scale : -INFINITY;
  }
  __syncthreads();
  if (warp == 0) {
    float mf = -INFINITY;
    for (int kk = lane; kk < m; kk += 32) mf = fmaxf(mf, sS[kk]);
    for (int o = 16; o > 0; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, o));
    float M = mf;  // finite: key 0 of the query is always visible
    for (int sp = lane; sp < splits; sp += 32) M = fmaxf(M, Mpart[((long)sp * Hkv + g) * R + r]);
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f, lf = 0.f;
    for (int sp = lane; sp < splits; sp += 32) {
      const long b = ((long)sp * Hkv + g) * R + r;
      const float w = Mpart[b] != -INFINITY ? expf(Mpart[b] - M) : 0.f;
      wsp[sp] = w;
      L += Lpart[b] * w;
    }
    for (int kk = lane; kk < m; kk += 32) {
      const float p = sS[kk] == -INFINITY ? 0.f : expf(sS[kk] - mf);
      sS[kk] = p;
      lf += p;
    }
    for (int o = 16; o > 0; o >>= 1) {
      L += __shfl_xor_sync(0xffffffffu, L, o);
      lf += __shfl_xor_sync(0xffffffffu, lf, o);
    }
    if (lane == 0) {
      const float wf = expf(mf - M);
      sM = M;
      sL = L + lf * wf;
      sWf = wf;
    }
  }
  __syncthreads();
  const float M = sM, L = sL, wf = sWf;
  for (int d = threadIdx.x; d < dkp; d += blockDim.x) {
    float acc = 0.f;
    const float* op = Opart + ((long)g * R + r) * dkp + d;
    const long sstride = (long)Hkv * R * dkp;
#pragma unroll 8
    for (int sp = 0; sp < splits; ++sp) {
      const float w = wsp[sp];
      const float v = __ldg(op + sp * sstride);
      acc = w != 0.f ? fmaf(v, w, acc) : acc;
    }
    float of = 0.f;  // fresh keys' P.V, as its own split
    for (int kk = 0; kk <= i && kk < m; ++kk) of = fmaf(sS[kk], sV[kk * dkp + d], of);
    acc = fmaf(of, wf, acc);
    const float o = acc / L;
    const long col = (long)(g * G + j) * dkp + d;
    out[(long)i * H * dkp + col] = o;
    if (x3 != nullptr) {
      __half p, qq, rr;
      split3(o, p, qq, rr);
      x3[(long)i * ldx + col] = p;
      x3[(long)(32 + i) * ldx + col] = qq;
      x3[(long)(64 + i) * ldx + col] = rr;
    }
  }
  if (threadIdx.x == 0 && Mfin != nullptr) {
    Mfin[(long)g * R + r] = M;
    Lfin[(long)g * R + r] = L;
  }
}

// Scores of one layer from the key-major S [Hkv][s][R] (model.py:294, 303-307 and
// selection.py:79-86):
//   rows[i][t]      = f32( sum_h f64(p_{h,i,t}) / H ),  p = exp(S - M) / L
//   per_layer[t]    = f32( mean_i f64(rows[i][t]) )
// One warp per context token, lane = query i (S loads of 32 consecutive rows).  p is
// evaluated as 2^(S*log2e - M*log2e) * (1/L) (rel. error ~3e-7, far inside the 1e-4
// score tolerance); the query mean is a fixed-order f64 warp reduction.
//   MODE 0: per_layer directly;  MODE 1: rows [m][ld] f32 (renormalised scoring: ld = s;
//           capture_attn: ld = s + m, the fresh-key columns by s1_fresh_rows_kernel);
//   MODE 2: this rank's head sums rows64 [s][m] f64 (tensor parallel; summed over ranks,
//           then s1_scores_finish applies the mean over all H heads).
enum { SC_MEAN = 0, SC_ROWS = 1, SC_PARTIAL = 2 };

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) s1_scores_kernel(const float* __restrict__ S, const float* __restrict__ Mfin,
                                                        const float* __restrict__ Lfin, int Hkv, int G, int R, int m,
                                                        int s, int H_total, float* out, double* out64, long ld) {
  pdl_entry();
  extern __shared__ float2 shn[];  // [Hkv*R]: (M*log2e, 1/L) per row g*R + r
  constexpr float LOG2E = 1.4426950408889634f;
  for (int q = threadIdx.x; q < Hkv * R; q += blockDim.x) shn[q] = make_float2(Mfin[q] * LOG2E, 1.f / Lfin[q]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < s; t += gridDim.x * wpb) {
    double tok = 0.0;
    for (int i0 = 0; i0 < m; i0 += 32) {
      const int i = i0 + lane;
      double acc = 0.0;
      if (i < m) {
        if (G == 4 && (Hkv & 1) == 0) {
          // common GQA case: 8 independent loads in flight per step, two f64 chains
          double acc2 = 0.0;
          for (int g = 0; g < Hkv; g += 2) {
            const float* c0 = S + ((long)g * s + t) * R + i;
            const float* c1 = c0 + (long)s * R;
            float v[8];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v[j] = __ldg(c0 + j * m);
              v[4 + j] = __ldg(c1 + j * m);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 n0 = shn[g * R + j * m + i], n1 = shn[(g + 1) * R + j * m + i];
              acc += (double)(ex2(fmaf(v[j], LOG2E, -n0.x)) * n0.y);
              acc2 += (double)(ex2(fmaf(v[4 + j], LOG2E, -n1.x)) * n1.y);
            }
          }
          acc += acc2;
        } else {
          for (int g = 0; g < Hkv; ++g) {
            const float* col = S + ((long)g * s + t) * R;
#pragma unroll 4
            for (int j = 0; j < G; ++j) {
              const int r = j * m + i;
              const float2 n = shn[g * R + r];
              acc += (double)(ex2(fmaf(__ldg(col + r), LOG2E, -n.x)) * n.y);
            }
          }
        }
      }
      if (MODE == SC_PARTIAL) {
        if (i < m) out64[(long)t * m + i] = acc;
      } else {
        const float rv = (float)(acc / (double)H_total);
        if (MODE == SC_ROWS) {
          if (i < m) out[(long)i * ld + t] = rv;
        } else if (i < m) {
          tok += (double)rv;
        }
      }
    }
    if (MODE == SC_MEAN) {
      tok = warp_sum_f64(tok);
      if (lane == 0) out[t] = (float)(tok / (double)m);
    }
  }
}

// after the rank sum: rows64 [s][m] -> MODE 0 per_layer / MODE 1 rows [m][s]
template <int MODE>
__global__ void __launch_bounds__(256) s1_scores_finish(const double* __restrict__ rows64, int m, int s, int H_total,
                                                        float* out, long ld) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < s; t += gridDim.x * wpb) {
    double tok = 0.0;
    for (int i = lane; i < m; i += 32) {
      const float rv = (float)(rows64[(long)t * m + i] / (double)H_total);
      if (MODE == SC_ROWS) out[(long)i * ld + t] = rv;
      else tok += (double)rv;
    }
    if (MODE == SC_MEAN) {
      tok = warp_sum_f64(tok);
      if (lane == 0) out[t] = (float)(tok / (double)m);
    }
  }
}

// capture_attn rows, the query's own keys (columns s..s+m-1 of rows [m][ld]): the head mean
// of p = exp(S - M) / L with S recomputed exactly as the fresh-key split forms it
// (sequential f32 FMAs over the padded head dim, then * scale) and the final row max /
// sum; causal within the query (j > i: 0)
__global__ void s1_fresh_rows_kernel(const float* q, const float* k, const float* Mfin, const float* Lfin, int m,
                                     int H, int Hkv, int dkp, float scale, int s, float* out, long ld) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (j >= m) return;
  constexpr float LOG2E = 1.4426950408889634f;
  const int G = H / Hkv, R = m * G;
  float rv = 0.f;
  if (j <= i) {
    double acc = 0.0;
    for (int h = 0; h < H; ++h) {
      const int g = h / G, jh = h - g * G;
      const float* qp = q + ((long)i * H + h) * dkp;
      const float* kp = k + ((long)j * Hkv + g) * dkp;
      float sc = 0.f;
      for (int d = 0; d < dkp; ++d) sc = fmaf(qp[d], kp[d], sc);
      const int r = g * R + jh * m + i;
      acc += (double)(ex2(fmaf(sc * scale, LOG2E, -Mfin[r] * LOG2E)) * (1.f / Lfin[r]));
    }
    rv = (float)(acc / (double)H);
  }
  out[(long)i * ld + s + j] = rv;
}

// optional context-only renormalisation denominators (selection.py:80-84)
__global__ void s1_row_sums_kernel(const float* rows, int s, double* denom) {
  pdl_entry();
  const int i = blockIdx.x;
  __shared__ double red[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < s; t += blockDim.x) acc += (double)rows[(long)i * s + t];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
    denom[i] = v > 1e-30 ? v : 1e-30;
  }
}

// per_layer[t] = f32( mean_i f64(rows[i][t]) )  (selection.py:79-86)
__global__ void s1_query_mean_kernel(const float* rows, const double* denom, int m, int s, float* out) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  double acc = 0.0;
  for (int i = 0; i < m; ++i) {
    double v = (double)rows[(long)i * s + t];
    if (denom) v = v / denom[i];
    acc += v;
  }
  out[t] = (float)(acc / (double)m);
}

// row weights of the second scoring pass: w = 1 / (L * H * m), divided by the query's
// context-only denominator when renormalising (selection.py:80-84: denom_i = sum over the
// context of the head-mean row = (1/H) sum_h C_{h,i}, C = the row's context mass)
__global__ void s1_row_weights_kernel(const float* Lfin, const float* Cfin, int Hkv, int G, int R, int m, int H_total,
                                      float* W) {
  pdl_entry();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Hkv * R) return;
  const int r = idx % R;
  double w = 1.0 / ((double)Lfin[idx] * (double)H_total * (double)m);
  if (Cfin != nullptr) {
    const int i = r % m;
    double d = 0.0;
    for (int g = 0; g < Hkv; ++g)
      for (int j = 0; j < G; ++j) d += (double)Cfin[(long)g * R + j * m + i];
    d /= (double)H_total;
    w /= (d > 1e-30 ? d : 1e-30);
  }
  W[idx] = (float)w;
}

// per_layer[t] = f32( sum over (row block, KV head) of the pass-2 column sums ), fixed
// order in f64;  MODE 1: the f64 sums of this rank's heads (summed over ranks, then
// rounded by s1_f64_to_f32_kernel)
template <int MODE>
__global__ void s1_colsum_finish(const float* __restrict__ part, int nparts, int s, float* out, double* out64) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  double acc = 0.0;
  for (int p = 0; p < nparts; ++p) acc += (double)__ldg(part + (long)p * s + t);
  if (MODE == 0) out[t] = (float)acc;
  else out64[t] = acc;
}
__global__ void s1_f64_to_f32_kernel(const double* x, int n, float* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = (float)x[t];
}

int s1_attention_launch(const S1Attn& a_in, float* attn_out, float* Mfin, float* Lfin, float* rows, double* denom,
                        float* per_layer, int renorm, int H_total, double* rows64, pkv_comm* comm, cudaStream_t st,
                        float* capture_rows) {
  S1Attn a = a_in;
  const int row_blocks = ceil_div(a.R, 128);
  int total_splits = a.n_splits;
  const size_t fresh_smem = (a.tc_splits + a.m + (size_t)a.m * a.dkp) * sizeof(float);
  bool combined = false, fresh_done = false;
  // scores by the second pass over the keys (no score matrix) unless the rows themselves
  // are wanted (capture_attn) or the renormalised scores need other ranks' heads
  const bool pass2 = a.tc_splits > 0 && per_layer != nullptr && capture_rows == nullptr && a.s > 0 &&
                     a.sc_part != nullptr && !(renorm && comm_world(comm) > 1);
  if (a.tc_splits > 0) {
    // context keys [0, s) on the tensor cores (fp16 planes, fp32-faithful)
    S1TcArgs t{};
    t.q = a.q;
    t.m = a.m;
    t.H = a.H;
    t.Hkv = a.Hkv;
    t.G = a.G;
    t.dk = a.dk;
    t.R = a.R;
    t.s = a.s;
    t.s_tot = a.s_tot;
    t.keys_per_split = a.tc_keys_per_split;
    t.n_splits = a.tc_splits;
    t.scale = a.scale;
    t.q3 = a.q3;
    t.q3_ready = a.q3_ready;
    t.kv_row0 = ((long)a.layer * a.pool_heads + a.head0) * a.pool_tokens;
    t.pool_tokens = a.pool_tokens;
    t.page_table = a.page_table;
    t.S = pass2 ? nullptr : a.S;
    t.Opart = a.Opart;
    t.Mpart = a.Mpart;
    t.Lpart = a.Lpart;
    // the fresh query keys ride along as an extra CTA slot of the same launch
    static const bool fused_fresh_env = getenv("PKV_FRESH_FUSED") && getenv("PKV_FRESH_FUSED")[0] == '1';
    t.fresh = (a.m <= 128 && !fused_fresh_env) ? 1 : 0;
    t.fk = a.fk;
    t.fv = a.fv;
    int rc = s1_attn_tc_launch(t, a.k1_all, a.k2_all, a.v_all, a.pool_rows_total, a.dkp, st);
    if (rc) return rc;
    // fused fresh keys + combine: measured neutral (each CTA re-reads the head's fresh V),
    // so opt-in (PKV_FRESH_FUSED=1)
    if (fused_fresh_env && fresh_smem <= 160 * 1024 && !(pass2 && renorm)) {
      // the m fresh query keys are merged inside the combine (one kernel instead of a
      // SIMT split + combine)
      static std::once_flag once_fresh;
      std::call_once(once_fresh, [] {
        cudaFuncSetAttribute(s1_attn_combine_fresh, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      });
      launch_k(s1_attn_combine_fresh, dim3(a.R, a.Hkv), 128, fresh_smem, st, a.Opart, a.Mpart, a.Lpart,
               a.tc_splits, a.Hkv, a.R, a.m, a.G, a.H, a.dkp, a.q, a.fk, a.fv, a.scale, attn_out, Mfin, Lfin,
               reinterpret_cast<__half*>(a.x3_out), a.x3_ld);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_attn_combine_fresh");
      combined = true;
    } else {  // the fresh keys as one extra split (inside the launch above, or SIMT)
      fresh_done = t.fresh != 0;
      a.key_base = a.s;
      a.keys_per_split = a.m;
      a.n_splits = 1;
      a.split_base = a.tc_splits;
      total_splits = a.tc_splits + 1;
    }
  }
  if (!combined) {
  if (!fresh_done) {
  // short fresh-key split: 32-row CTAs (4x the parallelism); long SIMT ranges: 128 rows
  const bool small = a.tc_splits > 0;
  const int rows_per_cta = small ? 32 : 128;
  dim3 grid(a.n_splits, a.Hkv, ceil_div(a.R, rows_per_cta));
  const int smem = (rows_per_cta * (a.dkp + 4) + 2 * 32 * (a.dkp + 4) + rows_per_cta * 33) * 4;
  if (a.dkp == 128) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_pass1<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
      cudaFuncSetAttribute(s1_attn_pass1<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    });
    if (small) launch_k(s1_attn_pass1<128, 1>, grid, 256, smem, st, a);
    else launch_k(s1_attn_pass1<128, 4>, grid, 256, smem, st, a);
  } else if (a.dkp == 64) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_pass1<64, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
      cudaFuncSetAttribute(s1_attn_pass1<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    });
    if (small) launch_k(s1_attn_pass1<64, 1>, grid, 256, smem, st, a);
    else launch_k(s1_attn_pass1<64, 4>, grid, 256, smem, st, a);
  } else {
    return set_error(PKV_ERR_CONFIG, "narrow pass: padded head dim %d unsupported", a.dkp);
  }
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("s1_attn_pass1");
  }
  launch_k(s1_attn_combine, dim3(a.R, a.Hkv), 128, ((total_splits + 7) & ~7) * sizeof(float), st, a.Opart, a.Mpart, a.Lpart, total_splits, a.Hkv, a.R, a.m, a.G, a.H,
                                                    a.dkp, attn_out, Mfin, Lfin,
                                                    reinterpret_cast<__half*>(a.x3_out), a.x3_ld, a.tc_splits,
                                                    (pass2 && renorm) ? a.sc_c : (float*)nullptr);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("s1_attn_combine");
  }
  if (pass2) {
    const int nrw = a.Hkv * a.R;
    launch_k(s1_row_weights_kernel, ceil_div(nrw, 128), 128, 0, st, (const float*)Lfin,
             renorm ? (const float*)a.sc_c : (const float*)nullptr, a.Hkv, a.G, a.R, a.m, H_total, a.sc_w);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("s1_row_weights_kernel");
    S1ScoreArgs sa{};
    sa.q3 = a.q3;
    sa.Hkv = a.Hkv;
    sa.R = a.R;
    sa.s = a.s;
    sa.keys_per_split = a.sc_keys_per_split;
    sa.n_splits = a.sc_splits;
    sa.scale = a.scale;
    sa.kv_row0 = ((long)a.layer * a.pool_heads + a.head0) * a.pool_tokens;
    sa.pool_tokens = a.pool_tokens;
    sa.page_table = a.page_table;
    sa.Mfin = Mfin;
    sa.W = a.sc_w;
    sa.part = a.sc_part;
    int rc = s1_score_tc_launch(sa, a.k1_all, a.k2_all, a.pool_rows_total, a.dkp, st);
    if (rc) return rc;
    const int nparts = row_blocks * a.Hkv;
    if (comm_world(comm) > 1) {
      launch_k(s1_colsum_finish<1>, ceil_div(a.s, 256), 256, 0, st, (const float*)a.sc_part, nparts, a.s,
               (float*)nullptr, rows64);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_colsum_finish");
      rc = comm_allreduce(comm, rows64, (size_t)a.s, PKV_DT_F64, st);
      if (rc) return rc;
      launch_k(s1_f64_to_f32_kernel, ceil_div(a.s, 256), 256, 0, st, (const double*)rows64, a.s, per_layer);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_f64_to_f32_kernel");
    } else {
      launch_k(s1_colsum_finish<0>, ceil_div(a.s, 256), 256, 0, st, (const float*)a.sc_part, nparts, a.s, per_layer,
               (double*)nullptr);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_colsum_finish");
    }
    return PKV_OK;
  }
  if (a.S == nullptr && (capture_rows != nullptr || per_layer != nullptr) && a.s > 0)
    return set_error(PKV_ERR_ARGUMENT, "narrow pass: the score path needs the score workspace");
  if (a.S != nullptr && capture_rows != nullptr) {  // capture_attn: head-mean rows [m][s + m]
    const long ld = a.s + a.m;
    if (comm_world(comm) > 1) return set_error(PKV_ERR_CONFIG, "capture_attn is not supported head-sharded");
    if (a.s > 0) {
      const int sgrid = std::min(ceil_div(a.s, 8), 8 * num_sms());
      const size_t ssmem = (size_t)a.Hkv * a.R * sizeof(float2);
      static std::once_flag once_c;
      std::call_once(once_c, [] {
        cudaFuncSetAttribute(s1_scores_kernel<SC_ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      });
      launch_k(s1_scores_kernel<SC_ROWS>, sgrid, 256, ssmem, st, a.S, Mfin, Lfin, a.Hkv, a.G, a.R, a.m, a.s, H_total,
               capture_rows, (double*)nullptr, ld);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_scores_kernel");
    }
    if (a.m > 1024) return set_error(PKV_ERR_SHAPE, "capture_attn: query longer than 1024 tokens");
    s1_fresh_rows_kernel<<<a.m, ((a.m + 31) / 32) * 32, 0, st>>>(a.q, a.fk, Mfin, Lfin, a.m, a.H, a.Hkv, a.dkp,
                                                                 a.scale, a.s, capture_rows, ld);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("s1_fresh_rows_kernel");
  } else if (a.S != nullptr && per_layer != nullptr && a.s > 0) {  // (s = 0: no context keys to score)
    const int sgrid = std::min(ceil_div(a.s, 8), 8 * num_sms());
    const size_t ssmem = (size_t)a.Hkv * a.R * sizeof(float2);
    if (ssmem > 48 * 1024) {
      static std::once_flag once;
      std::call_once(once, [] {
        for (auto f : {s1_scores_kernel<SC_MEAN>, s1_scores_kernel<SC_ROWS>, s1_scores_kernel<SC_PARTIAL>})
          cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      });
    }
    float* target = renorm ? rows : per_layer;
    if (comm_world(comm) > 1) {
      // per-token score exchange before the global top-k: sum the ranks' head partials
      launch_k(s1_scores_kernel<SC_PARTIAL>, sgrid, 256, ssmem, st, a.S, Mfin, Lfin, a.Hkv, a.G, a.R, a.m, a.s, H_total,
               (float*)nullptr, rows64, (long)a.s);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_scores_kernel");
      int rc = comm_allreduce(comm, rows64, (size_t)a.m * a.s, PKV_DT_F64, st);
      if (rc) return rc;
      if (renorm) launch_k(s1_scores_finish<SC_ROWS>, sgrid, 256, 0, st, rows64, a.m, a.s, H_total, target, (long)a.s);
      else launch_k(s1_scores_finish<SC_MEAN>, sgrid, 256, 0, st, rows64, a.m, a.s, H_total, target, (long)a.s);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_scores_finish");
    } else {
      if (renorm)
        launch_k(s1_scores_kernel<SC_ROWS>, sgrid, 256, ssmem, st, a.S, Mfin, Lfin, a.Hkv, a.G, a.R, a.m, a.s, H_total,
                 target, (double*)nullptr, (long)a.s);
      else
        launch_k(s1_scores_kernel<SC_MEAN>, sgrid, 256, ssmem, st, a.S, Mfin, Lfin, a.Hkv, a.G, a.R, a.m, a.s, H_total,
                 target, (double*)nullptr, (long)a.s);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_scores_kernel");
    }
    if (renorm) {
      launch_k(s1_row_sums_kernel, a.m, 256, 0, st, rows, a.s, denom);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_row_sums_kernel");
      launch_k(s1_query_mean_kernel, ceil_div(a.s, 256), 256, 0, st, rows, denom, a.m, a.s, per_layer);
      PKV_LAUNCHED();
      PKV_CHECK_LAUNCH("s1_query_mean_kernel");
    }
  }
  return PKV_OK;
}

// ------------------------------------------------------------------ lm_head
// logits[n] = dot(x, W[n]) over D, fp32 accumulation (x = final-normed last row)
// R output rows per warp pass (16-byte loads of R rows, UNR k-steps in flight per lane,
// independent accumulators); x (fp32, final-normed) staged in shared memory.  R = 2: with
// 4 rows per pass the 128k-row vocabulary split into 3.4 passes per warp (85 % balance)
template <int R, int UNR>
__global__ void __launch_bounds__(256) gemv_rows_kernel(const float* x, const __nv_bfloat16* __restrict__ W, int N,
                                                        int D, long ldw, float* out) {
  pdl_entry();
  extern __shared__ float xs[];
  for (int c = threadIdx.x; c < D; c += blockDim.x) xs[c] = x[c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const bool vec = (D % 8 == 0) && (ldw % 8 == 0);
  for (int n0 = (blockIdx.x * wpb + warp) * R; n0 < N; n0 += gridDim.x * wpb * R) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    if (vec) {
#pragma unroll UNR
      for (int c = lane * 8; c < D; c += 256) {
        uint4 u[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
          u[r] = n0 + r < N ? __ldg(reinterpret_cast<const uint4*>(W + (long)(n0 + r) * ldw + c)) : make_uint4(0, 0, 0, 0);
        const float4 xa = *reinterpret_cast<const float4*>(xs + c);
        const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r] = fmaf(xa.x, bf16_lo(u[r].x), acc[r]);
          acc[r] = fmaf(xa.y, bf16_hi(u[r].x), acc[r]);
          acc[r] = fmaf(xa.z, bf16_lo(u[r].y), acc[r]);
          acc[r] = fmaf(xa.w, bf16_hi(u[r].y), acc[r]);
          acc[r] = fmaf(xb.x, bf16_lo(u[r].z), acc[r]);
          acc[r] = fmaf(xb.y, bf16_hi(u[r].z), acc[r]);
          acc[r] = fmaf(xb.z, bf16_lo(u[r].w), acc[r]);
          acc[r] = fmaf(xb.w, bf16_hi(u[r].w), acc[r]);
        }
      }
    } else {
      for (int r = 0; r < R && n0 + r < N; ++r)
        for (int c = lane; c < D; c += 32) acc[r] = fmaf(xs[c], __bfloat162float(W[(long)(n0 + r) * ldw + c]), acc[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float v = acc[r];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && n0 + r < N) out[n0 + r] = v;
    }
  }
}

// one row per warp pass with the whole row's NV 16-byte loads per lane issued up front
// (D = 256 * NV): fine-grained rows balance the 128k-row vocabulary over the warps (14 vs
// 13.5 passes) while each lane keeps NV * 16 B in flight.  Same per-lane summation order
// as gemv_rows_kernel (column blocks lane*8 + 256*i in increasing i), so bit-identical.
template <int NV>
__global__ void __launch_bounds__(256) gemv_row1_kernel(const float* x, const __nv_bfloat16* __restrict__ W, int N,
                                                        long ldw, float* out) {
  pdl_entry();
  __shared__ __align__(16) float xs[NV * 256];
  for (int c = threadIdx.x; c < NV * 256; c += blockDim.x) xs[c] = x[c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int n = blockIdx.x * (blockDim.x >> 5) + warp; n < N; n += nw) {
    const uint4* row = reinterpret_cast<const uint4*>(W + (long)n * ldw) + lane;
    uint4 u[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) u[i] = __ldg(row + i * 32);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float* xp = xs + i * 256 + lane * 8;
      const float4 xa = *reinterpret_cast<const float4*>(xp);
      const float4 xb = *reinterpret_cast<const float4*>(xp + 4);
      acc = fmaf(xa.x, bf16_lo(u[i].x), acc);
      acc = fmaf(xa.y, bf16_hi(u[i].x), acc);
      acc = fmaf(xa.z, bf16_lo(u[i].y), acc);
      acc = fmaf(xa.w, bf16_hi(u[i].y), acc);
      acc = fmaf(xb.x, bf16_lo(u[i].z), acc);
      acc = fmaf(xb.y, bf16_hi(u[i].z), acc);
      acc = fmaf(xb.z, bf16_lo(u[i].w), acc);
      acc = fmaf(xb.w, bf16_hi(u[i].w), acc);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[n] = acc;
  }
}

int gemv_launch(const float* x, const void* W, int N, int D, long ldw, float* out, cudaStream_t st) {
  if (D % 256 == 0 && ldw % 8 == 0 && !getenv("PKV_GEMV_ROWS")) {
    const int blocks = std::min(ceil_div(N, 8), num_sms() * 8);
    auto* w = reinterpret_cast<const __nv_bfloat16*>(W);
    switch (D / 256) {
      case 1: launch_k(gemv_row1_kernel<1>, blocks, 256, 0, st, x, w, N, ldw, out); break;
      case 2: launch_k(gemv_row1_kernel<2>, blocks, 256, 0, st, x, w, N, ldw, out); break;
      case 4: launch_k(gemv_row1_kernel<4>, blocks, 256, 0, st, x, w, N, ldw, out); break;
      case 8: launch_k(gemv_row1_kernel<8>, blocks, 256, 0, st, x, w, N, ldw, out); break;
      case 16: launch_k(gemv_row1_kernel<16>, blocks, 256, 0, st, x, w, N, ldw, out); break;
      default: goto rows_kernel;
    }
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("gemv_row1_kernel");
    return PKV_OK;
  }
rows_kernel:
  static const int rows = getenv("PKV_GEMV_ROWS") ? atoi(getenv("PKV_GEMV_ROWS")) : 4;
  const int per_block = 8 * rows;
  const int blocks = std::min(ceil_div(N, per_block), num_sms() * 8);
  auto* w = reinterpret_cast<const __nv_bfloat16*>(W);
  if (rows == 4) launch_k(gemv_rows_kernel<4, 2>, blocks, 256, D * sizeof(float), st, x, w, N, D, ldw, out);
  else if (rows == 1) launch_k(gemv_rows_kernel<1, 8>, blocks, 256, D * sizeof(float), st, x, w, N, D, ldw, out);
  else launch_k(gemv_rows_kernel<2, 4>, blocks, 256, D * sizeof(float), st, x, w, N, D, ldw, out);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("gemv_rows_kernel");
  return PKV_OK;
}

// Deferred RMSNorm after the tensor-parallel all-reduce of h: the xg = fp16(h * g) and
// per-256-column-tile fp32 sums of h^2 that the EPI_RESID epilogue writes on one GPU, in the
// same (increasing column) order, so head-sharded and unsharded Stage II normalise alike.
__global__ void norm_defer_kernel(const float* __restrict__ h, long ld, int N, const float* __restrict__ g,
                                  __half* __restrict__ xg, long ldxg, float* __restrict__ ssq, int ssq_ld) {
  pdl_entry();
  const long row = blockIdx.x;
  const int c0 = threadIdx.x * 256;
  if (c0 >= N) return;
  const float* hr = h + row * ld;
  float acc = 0.f;
  const int c1 = min(c0 + 256, N);
  for (int c = c0; c < c1; ++c) {
    const float v = hr[c];
    acc = fmaf(v, v, acc);
    xg[row * ldxg + c] = __float2half_rn(v * g[c]);
  }
  ssq[row * ssq_ld + threadIdx.x] = acc;
}

int norm_defer_launch(const float* h, int m, long ld, int N, const float* g, void* xg, long ldxg, float* ssq,
                      int ssq_ld, cudaStream_t st) {
  if (m <= 0) return PKV_OK;
  const int threads = ceil_div(N, 256);
  if (threads > 1024) return set_error(PKV_ERR_SHAPE, "norm_defer: row too wide");
  launch_k(norm_defer_kernel, m, threads, 0, st, h, ld, N, g, reinterpret_cast<__half*>(xg), ldxg, ssq, ssq_ld);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("norm_defer_kernel");
  return PKV_OK;
}

// embedding rows (bf16 table) -> fp32 [n][ld]
__global__ void embed_gather_kernel(const __nv_bfloat16* embed, long lde, const int32_t* ids, const int32_t* sel,
                                    int n, int D, float* out, long ldo) {
  pdl_entry();
  const int r = blockIdx.x;
  if (r >= n) return;
  const int tok = sel ? ids[sel[r]] : ids[r];
  for (int c = threadIdx.x; c < ldo; c += blockDim.x)
    out[(long)r * ldo + c] = c < D ? __bfloat162float(embed[(long)tok * lde + c]) : 0.f;
}

int embed_gather_launch(const void* embed, long lde, const int32_t* ids, const int32_t* sel, int n, int D, float* out,
                        long ldo, cudaStream_t st) {
  if (n <= 0) return PKV_OK;
  launch_k(embed_gather_kernel, n, 256, 0, st, reinterpret_cast<const __nv_bfloat16*>(embed), lde, ids, sel, n, D, out, ldo);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("embed_gather_kernel");
  return PKV_OK;
}

}  // namespace pkv

namespace pkv {

// ------------------------------------------------------ probe baselines (selection.py:95-142)
// kvshare column sums: block [p0, p0+n) adds n * (its mean row over keys < p0) and its own
// diagonal part, in f64, one launch per block in block order (deterministic)
__global__ void probe_accum_kernel(const float* __restrict__ part, int p0, int n, double* colsum) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p0 + n) return;
  const double v = (double)part[t];
  colsum[t] += t < p0 ? v * (double)n : v;
}

// per context token t (one warp): dV = v1[t] - assembled layer-1 value (fp16 pool = the
// chunk store's bf16 value exactly), f64 norms; out = f32(colsum[t] * ||dV||_1) (kvshare)
// or f32(||dV||_2) (cacheblend, colsum == nullptr)
__global__ void probe_scores_kernel(const float* __restrict__ v1, const __half* __restrict__ vp1,
                                    const int32_t* page_table, long pool_tokens, int s, int Hkv, int dk, int dkp,
                                    const double* __restrict__ colsum, float* out) {
  pdl_entry();
  const int t = (int)(((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (t >= s) return;
  const long slot = (long)page_table[t >> 7] * 128 + (t & 127);
  double acc = 0.0;
  for (int e = lane; e < Hkv * dk; e += 32) {
    const int h = e / dk, d = e - h * dk;
    const double dv = (double)v1[(long)t * Hkv * dk + e] - (double)__half2float(vp1[((long)h * pool_tokens + slot) * dkp + d]);
    acc += colsum != nullptr ? fabs(dv) : dv * dv;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[t] = colsum != nullptr ? (float)(colsum[t] * acc) : (float)sqrt(acc);
}

int probe_accum_launch(const float* part, int p0, int n, double* colsum, cudaStream_t st) {
  if (p0 + n <= 0) return PKV_OK;
  launch_k(probe_accum_kernel, ceil_div(p0 + n, 256), 256, 0, st, part, p0, n, colsum);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("probe_accum_kernel");
  return PKV_OK;
}

int probe_scores_launch(const float* v1, const void* vp1, const int32_t* page_table, long pool_tokens, int s, int Hkv,
                        int dk, int dkp, const double* colsum, float* out, cudaStream_t st) {
  if (s <= 0) return PKV_OK;
  launch_k(probe_scores_kernel, ceil_div((long)s * 32, 256), 256, 0, st, v1, reinterpret_cast<const __half*>(vp1),
           page_table, pool_tokens, s, Hkv, dk, dkp, colsum, out);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("probe_scores_kernel");
  return PKV_OK;
}

}  // namespace pkv
