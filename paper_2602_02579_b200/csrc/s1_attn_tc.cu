// fp32-faithful narrow-pass attention on tcgen05 (reference model.py:278-308 as
// called by query_pass model.py:370-402, i.e. score_prophet and finalize_query).
//
// The reference computes q.k and p.v in float64 on f32 inputs.  On the fp16 tensor
// cores with fp32 accumulation in TMEM every fp32 operand is split into unscaled fp16
// planes that share ONE accumulator (split3h_pack / split2h_pack, common.cuh):
//     Q' = 2^6 q  = Qh + Qm + Ql         (three planes; the 2^6 pre-scale keeps the
//                                         residual planes out of the fp16 subnormals)
//     K  = Kh + Kl                        (the fp16 cache key k_pool + its residual plane
//                                         k2_pool: 2^-22 relative, 2^-25 absolute)
//     Q' K^T = Qh Kh + Qm Kh + Qh Kl   (the dropped Ql Kh, Qm Kl, Ql Kl are < 2^-21 of
//                                       |q||k|, the key planes' own truncation is 2^-22)
//     P' V   = Ph V + Pm V,  P' = 2^10 p         (V: fp16 cache values, exact for
//                                                       the chunk store's bf16 values)
// so scores and outputs are f32-faithful to ~5e-7 of |q||k| (far inside the 1e-4
// selection tie band).  Only the context keys [0, s) run here; the m fresh query keys (fp32 K/V)
// are one extra SIMT split.
//
// CTA = (KV head g, key split): 128 rows r = j*m + i (query head g*G+j, query i),
// 64-key tiles (half a cache page), 2-stage TMA ring.
//   warps 0-7  softmax: warp w owns TMEM lane quarter w%4 (32 rows) and key
//              columns [32*(w/4), +32) of each tile; the two warps of a quarter
//              exchange their row maxima through smem.  Q planes -> smem once;
//              per tile: S from TMEM, scale + mask, exact online softmax,
//              scores -> S workspace, P split -> TMEM (A operand of PV),
//              O rescale in TMEM when the row max grows
//   warp 8     TMA producer: Kh, Km, Kl, V tiles
//   warp 9     TMEM owner + MMA issuer (3 + 2 products per tile)
#include <mutex>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace pkv {

template <int DKP>
struct S1TcCfg {
  static constexpr int ATOMS = DKP / 64;
  static constexpr int KT = 64;                 // keys per tile
  static constexpr int QSPLIT = 128 * DKP * 2;  // one Q plane (128 rows)
  static constexpr int PLANE = KT * DKP * 2;    // one K plane / the V tile
  static constexpr int ATOM_Q = 128 * 128;      // bytes per 64-col atom of a Q plane
  static constexpr int ATOM_K = KT * 128;       // bytes per 64-col atom of a K/V plane
  static constexpr int STAGE = 3 * PLANE;       // Kh, Kl, V
  // The Q planes live in TMEM (A operand of the S MMAs), which frees shared memory for
  // the K/V ring: with two stages the softmax waited for S ~45 % of the time behind the
  // TMA (ncu, profiles/r01), the memory pipeline being too shallow.
  static constexpr int STAGES = DKP == 128 ? 4 : 6;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  // TMEM columns: Q planes [0,192) (plane x at 64x, DKP/2 columns each), S [192,256),
  // O [256,256+DKP), P planes [384,480)
  static constexpr int T_Q = 0, Q_PLANE = 64, T_S = 192, T_O = 256, T_P = 384;
  // two P buffers (2 fp16 planes x 32 columns each) when they fit: the softmax writes P(j)
  // while PV(j-1) still reads P(j-1), and waits for PV(j-1) only to rescale O
  static constexpr int P_BUFS = 2;  // set below per datapath

  static constexpr int SOFTMAX_WARPS = 8;
};

// Q planes: q3[((g*RB + rb)*3 + plane)*128 + r][DKP] fp16 planes of 2^6 q, row r of row
// block rb = query head g*G + j, query i with rb*128 + r = j*m + i (zero padded)
constexpr float S1_QSCALE = 64.f, S1_PSCALE = 1024.f;
// plane products of S = Q'K^T, in order of significance: QhKh, QmKh, QhKl (each ~2^-11
// below the previous level), then QlKh, QmKl (~2^-22 of |q||k|).  Three keep the score to
// ~2^-21 of |q||k| -- the key planes themselves stop at 2^-22 -- for 3/5 of the MMAs
// (ncu: with 5 QK + 3 PV products the narrow attention was tensor-bound, 69 us per layer
// for 201 MB of K/V).  P' is two planes (2^-22).  PKV_S1_FULL_PLANES=1 at build time
// restores 5 + 3 (the round-1 datapath).
#ifdef PKV_S1_FULL_PLANES
constexpr int S1_QK_PROD = 5, S1_P_PLANES = 3;
#else
constexpr int S1_QK_PROD = 3, S1_P_PLANES = 2;
#endif
constexpr int S1_Q_PLANES = S1_QK_PROD > 3 ? 3 : 2;
constexpr int S1_P_BUFS = S1_P_PLANES == 2 ? 2 : 1;  // P buffers in TMEM [384, 512)

__global__ void s1_qprep_kernel(const float* q, int m, int H, int G, int R, int RB, int dkp, __half* q3) {
  pdl_entry();
  const int g = blockIdx.y, rr = blockIdx.x;  // rr = rb*128 + r
  const int rb = rr >> 7, r = rr & 127;
  const bool valid = rr < R;
  const int jh = valid ? rr / m : 0, qi = valid ? rr - jh * m : 0;
  const float* src = q + ((long)qi * H + g * G + jh) * dkp;
  for (int d2 = threadIdx.x; d2 < dkp / 2; d2 += blockDim.x) {
    float x0 = valid ? src[2 * d2] * S1_QSCALE : 0.f, x1 = valid ? src[2 * d2 + 1] * S1_QSCALE : 0.f;
    uint32_t h, mi, l;
    split3h_pack(x0, x1, h, mi, l);
    const long base = (((long)g * RB + rb) * 3) * 128 + r;
    reinterpret_cast<uint32_t*>(q3 + base * dkp)[d2] = h;
    reinterpret_cast<uint32_t*>(q3 + (base + 128) * dkp)[d2] = mi;
    reinterpret_cast<uint32_t*>(q3 + (base + 256) * dkp)[d2] = l;
  }
}

// The m fresh query keys of one (KV head, row block) as split a.n_splits, on the CTA slot
// the launch adds after the context splits (so no separate SIMT launch).  S = f32(q.k) *
// scale (model.py:291, 298), causal within the query; partials in the context splits' form
// (O unnormalised, M, L).  Warp per row with lane = KEY (keys lane, lane + 32, ...): every
// lane forms whole dot products from shared memory (key rows padded to DKP + 4 floats, so
// the lanes' 16-byte reads of 32 different keys hit distinct banks), one max / sum
// reduction per row, then lane = 4 output dims.  (Round 1's lane = 4 dims with a
// shuffle-reduced dot product per key made this CTA the launch's critical path: 60 us
// against ~43 us for the context splits, tools/s1_trace.py.)
template <int DKP>
__device__ __noinline__ void s1_fresh_cta(const S1TcArgs& a, uint8_t* smem) {
  constexpr int KS = DKP + 4, DPL = DKP / 32;
  const int g = blockIdx.y, rb = blockIdx.z;
  const int m = a.m;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* sk = reinterpret_cast<float*>(smem);
  float* sv = sk + (long)m * KS;
  float* qs = sv + (long)m * KS;  // [128][DKP] the CTA's query rows, then [nw][32] probabilities
  // float4 copies, 4 in flight per thread (a load per element had taken 9 us, latency-bound)
  const int nv4 = m * (DKP / 4);
  for (int e0 = threadIdx.x; e0 < nv4; e0 += 4 * blockDim.x) {
    float4 kv[4], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < nv4) {
        const int kk = e / (DKP / 4), d4 = e - kk * (DKP / 4);
        const long src = ((long)kk * a.Hkv + g) * DKP + 4 * d4;
        kv[u] = *reinterpret_cast<const float4*>(a.fk + src);
        vv[u] = *reinterpret_cast<const float4*>(a.fv + src);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < nv4) {
        const int kk = e / (DKP / 4), d4 = e - kk * (DKP / 4);
        *reinterpret_cast<float4*>(sk + kk * KS + 4 * d4) = kv[u];
        *reinterpret_cast<float4*>(sv + kk * KS + 4 * d4) = vv[u];
      }
    }
  }
  for (int e0 = threadIdx.x; e0 < 128 * (DKP / 4); e0 += 4 * blockDim.x) {  // the 128 query rows
    float4 qv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x, r = e / (DKP / 4), d4 = e - r * (DKP / 4), row = rb * 128 + r;
      qv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < 128 * (DKP / 4) && row < a.R) {
        const int jh = row / m, i = row - jh * m;
        qv[u] = *reinterpret_cast<const float4*>(a.q + ((long)i * a.H + g * a.G + jh) * DKP + 4 * d4);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < 128 * (DKP / 4)) reinterpret_cast<float4*>(qs)[e] = qv[u];
    }
  }
  __syncthreads();
  if (a.trace != nullptr && g == 0 && rb == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[5 * 64 + 6] = t;  // fresh-key CTA: K/V staged
  }
  float* pw = qs + 128 * DKP + warp * 32;  // this warp's probabilities of one key block
  for (int r = warp; r < 128; r += nw) {
    const int row = rb * 128 + r;
    if (row >= a.R) break;
    const int i = row % m;
    const float* qw = qs + r * DKP;
    float sc[4];
    float mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int kk = lane + 32 * t;
      sc[t] = -INFINITY;
      if (kk < m && kk <= i) {
        const float4* kr = reinterpret_cast<const float4*>(sk + kk * KS);
        const float4* q4 = reinterpret_cast<const float4*>(qw);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};  // four independent chains, summed in a fixed order
#pragma unroll 8
        for (int d = 0; d < DKP / 4; ++d) {
          const float4 x = q4[d], y = kr[d];
          acc[0] = fmaf(x.x, y.x, acc[0]);
          acc[1] = fmaf(x.y, y.y, acc[1]);
          acc[2] = fmaf(x.z, y.z, acc[2]);
          acc[3] = fmaf(x.w, y.w, acc[3]);
        }
        sc[t] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * a.scale;
      }
      mx = fmaxf(mx, sc[t]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    float pk[4], l = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      pk[t] = sc[t] == -INFINITY ? 0.f : expf(sc[t] - mx);
      l += pk[t];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    float o[DPL];
#pragma unroll
    for (int d = 0; d < DPL; ++d) o[d] = 0.f;
    const int nk = min(i + 1, m);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (32 * t >= m) break;  // (m is uniform: no dynamic indexing of pk)
      // all 32 lanes' probabilities of this key block to shared memory (reuses the query
      // row slot, read by this warp only), then 4 keys per step: independent loads in flight
      __syncwarp();
      pw[lane] = pk[t];
      __syncwarp();
      const int k1 = min(nk, 32 * t + 32);
      int kk = 32 * t;
      for (; kk + 4 <= k1; kk += 4) {
        const float4 pv = *reinterpret_cast<const float4*>(pw + (kk - 32 * t));
        const float* vr = sv + kk * KS + lane * DPL;
#pragma unroll
        for (int d = 0; d < DPL; ++d) {
          o[d] = fmaf(pv.x, vr[d], o[d]);
          o[d] = fmaf(pv.y, vr[KS + d], o[d]);
          o[d] = fmaf(pv.z, vr[2 * KS + d], o[d]);
          o[d] = fmaf(pv.w, vr[3 * KS + d], o[d]);
        }
      }
      for (; kk < k1; ++kk) {
        const float pv = pw[kk - 32 * t];
        const float* vr = sv + kk * KS + lane * DPL;
#pragma unroll
        for (int d = 0; d < DPL; ++d) o[d] = fmaf(pv, vr[d], o[d]);
      }
    }
    const long base = ((long)a.n_splits * a.Hkv + g) * a.R + row;
    float* od = a.Opart + base * DKP + lane * DPL;
#pragma unroll
    for (int d = 0; d < DPL; ++d) od[d] = o[d];
    if (lane == 0) {
      a.Mpart[base] = mx;
      a.Lpart[base] = l;
    }
    __syncwarp();
  }
}

// trace[ev * 64 + j], tile j < 64 of CTA (0,0,0) (tools/s1_trace.py):
//   ev 0: softmax warp 0 saw S(j)   ev 1: softmax warp 0 arrived P(j)   ev 2: MMA warp saw K/V(j)
//   ev 3: MMA warp issued PV(j)     ev 4: producer issued tile j        ev 5: j=0 prologue done,
//   j=1 softmax loop done, j=2 partials written, j=4/5 fresh-key CTA of KV head 0 start/end
__device__ __forceinline__ void s1_stamp(const S1TcArgs& a, int ev, int j) {
  if (a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[ev * 64 + j] = t;
  }
}

template <int DKP>
__global__ void __launch_bounds__(320, 1)
    s1_attn_tc_kernel(const __grid_constant__ CUtensorMap tK1, const __grid_constant__ CUtensorMap tK2,
                      const __grid_constant__ CUtensorMap tV, S1TcArgs a) {
  using C = S1TcCfg<DKP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if (a.fresh && blockIdx.x == (unsigned)a.n_splits) {  // the fresh query keys' split
    griddep_wait();
    const bool tr = a.trace != nullptr && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0;
    unsigned long long t0 = 0, t1 = 0;
    if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    s1_fresh_cta<DKP>(a, smem);
    if (tr) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      a.trace[5 * 64 + 4] = t0;  // fresh-key CTA of KV head 0: start / end
      a.trace[5 * 64 + 5] = t1;
    }
    return;
  }
  uint8_t* sKV = smem;  // STAGES x {Kh, Kl, V}
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::STAGES * C::STAGE);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + C::STAGES;
  uint64_t* s_full = bars + 2 * C::STAGES;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;   // [2]: per P buffer
  uint64_t* pv_full = p_full + 2;  // [2]: PV of the P buffer done
  uint64_t* q_full = pv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.y;
  const int split = blockIdx.x;
  const int r0 = blockIdx.z * 128;
  const int k_begin = split * a.keys_per_split;
  const int k_end = min(k_begin + a.keys_per_split, a.s);
  const int n_tiles = (k_end - k_begin + C::KT - 1) / C::KT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, C::SOFTMAX_WARPS);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&p_full[b], C::SOFTMAX_WARPS);
      mbar_init(&pv_full[b], 1);
    }
    mbar_init(q_full, C::SOFTMAX_WARPS);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: the Q planes come from the previous kernel
  griddep_launch();

  if (warp == 8) {
    // ----------------------------------------------------------- TMA producer
    if (elect_one()) {
      tma_prefetch(&tK1);
      tma_prefetch(&tK2);
      tma_prefetch(&tV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % C::STAGES;
        mbar_wait(&kv_empty[st], ((uint32_t)(j / C::STAGES) & 1) ^ 1);
        const int t0 = k_begin + j * C::KT;  // 64-aligned: inside one 128-token page
        const int row = (int)(head_row + (long)a.page_table[t0 >> 7] * 128 + (t0 & 127));
        uint8_t* base = sKV + st * C::STAGE;
        s1_stamp(a, 4, j);
        mbar_expect_tx(&kv_full[st], C::STAGE);
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at) {
          tma_load_2d(base + at * C::ATOM_K, &tK1, &kv_full[st], at * 64, row);
          tma_load_2d(base + C::PLANE + at * C::ATOM_K, &tK2, &kv_full[st], at * 64, row);
          tma_load_2d(base + 2 * C::PLANE + at * C::ATOM_K, &tV, &kv_full[st], at * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = make_idesc_f16(128, C::KT);
    constexpr uint32_t idesc_o = make_idesc_f16(128, DKP, /*b_mn_major=*/true);
    constexpr int NPROD = S1_QK_PROD;
    constexpr int PA[5] = {0, 1, 0, 2, 1};
    constexpr int PB[5] = {0, 0, 1, 0, 1};
    mbar_wait(q_full, 0);
    tc_fence_after();
    for (int j = 0; j <= n_tiles; ++j) {
      if (j < n_tiles) {
        const int st = j % C::STAGES;
        mbar_wait(&kv_full[st], (uint32_t)(j / C::STAGES) & 1);
        if (lane == 0) s1_stamp(a, 2, j);
        if (j >= 1) mbar_wait(s_free, (uint32_t)(j - 1) & 1);  // S(j-1) is in the softmax's registers
        tc_fence_after();
        if (elect_one()) {
          const uint32_t k_addr = smem_u32(sKV + st * C::STAGE);
          int n = 0;
#pragma unroll
          for (int pr = 0; pr < NPROD; ++pr)
#pragma unroll
            for (int kk = 0; kk < DKP / 16; ++kk, ++n) {
              const uint32_t ko = PB[pr] * C::PLANE + (kk >> 2) * C::ATOM_K + (kk & 3) * 32;
              umma_ts(tmem + C::T_S, tmem + C::T_Q + PA[pr] * C::Q_PLANE + kk * 8,
                           sdesc_sw128(k_addr + ko, 16, 1024), idesc_s, n > 0 ? 1u : 0u);
            }
          umma_commit(s_full);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jp = j - 1;
        const int st = jp % C::STAGES;
        // P buffer b holds P(b), P(b + B), ...: P(jp) is its (jp / B)-th fill
        const int pb = jp % S1_P_BUFS;
        mbar_wait(&p_full[pb], (uint32_t)(jp / S1_P_BUFS) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = smem_u32(sKV + st * C::STAGE + 2 * C::PLANE);
          int n = 0;
#pragma unroll
          for (int x = 0; x < S1_P_PLANES; ++x)
#pragma unroll
            for (int kk = 0; kk < C::KT / 16; ++kk, ++n)
              umma_ts(tmem + C::T_O, tmem + C::T_P + pb * 64 + x * (C::KT / 2) + kk * 8,
                           sdesc_sw128(v_addr + kk * 16 * 128, C::ATOM_K, 1024), idesc_o,
                           (jp > 0 || n > 0) ? 1u : 0u);
          umma_commit(&pv_full[pb]);
          umma_commit(&kv_empty[st]);
          s1_stamp(a, 3, jp);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax
    constexpr float LOG2E = 1.4426950408889634f;
    const int quarter = warp & 3, hc = warp >> 2;
    const int r = quarter * 32 + lane;  // TMEM lane == tile row
    const int row = r0 + r;
    const bool valid = row < a.R;
    const uint32_t lb = (uint32_t)(quarter * 32) << 16;
    constexpr int HC = C::KT / 2;  // columns per warp
    {  // this warp's half of the row's Q planes -> TMEM (lane = row): A operand of S = Q K^T
      const __half* q3 = reinterpret_cast<const __half*>(a.q3);
      if (hc * 32 < DKP / 2) {
#pragma unroll 1
        for (int x = 0; x < S1_Q_PLANES; ++x) {
          const uint4* src = reinterpret_cast<const uint4*>(
              q3 + ((((long)g * gridDim.z + blockIdx.z) * 3 + x) * 128 + r) * DKP + hc * 64);
          uint32_t u[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = src[c];
            u[4 * c] = v.x; u[4 * c + 1] = v.y; u[4 * c + 2] = v.z; u[4 * c + 3] = v.w;
          }
          tmem_st32(tmem + lb + C::T_Q + x * C::Q_PLANE + hc * 32, u);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    float m_run = -INFINITY, l_run = 0.f;  // l_run: this warp's half of the row sum
    // scores, key-major S[g][t][r] (t < s): one warp store = 32 consecutive rows = 128 B
    float* scol = (a.S != nullptr && valid) ? a.S + (long)g * a.s * a.R + row : nullptr;
    if (warp == 0 && lane == 0) s1_stamp(a, 5, 0);
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(s_full, (uint32_t)j & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0) s1_stamp(a, 0, j);
      // both warps of a quarter read the whole 64-key row (cheap TMEM reads) so each
      // has the tile max without an exchange; each then handles its 32 columns
      float sv[HC];
      float tmax = -INFINITY;
      const int key0 = k_begin + j * C::KT + hc * HC;
      {
        uint32_t u[32], w[32];
        tmem_ld32(tmem + lb + C::T_S + hc * HC, u);
        tmem_ld32(tmem + lb + C::T_S + (hc ^ 1) * HC, w);
        tmem_ld_wait();
        // reference: f32(q.k) * F32(1/sqrt(dk)), model.py:291,298.  The accumulator holds
        // 2^6 q.k, so acc * (2^-6 scale) rounds exactly like (acc * 2^-6) * scale, and as the
        // factor is positive the max of the rounded scores is the rounded max accumulator
        const float c = a.scale * (1.f / S1_QSCALE);
        if (k_begin + (j + 1) * C::KT <= k_end) {  // whole tile (warp-uniform): no mask
          float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < HC; ++i) {
            sv[i] = __uint_as_float(u[i]) * c;
            mx[i & 3] = fmaxf(mx[i & 3], fmaxf(__uint_as_float(u[i]), __uint_as_float(w[i])));
          }
          tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * c;
        } else {
          const int okey0 = k_begin + j * C::KT + (hc ^ 1) * HC;
#pragma unroll
          for (int i = 0; i < HC; ++i) {
            const float x = (key0 + i < k_end) ? __uint_as_float(u[i]) * c : -INFINITY;
            const float y = (okey0 + i < k_end) ? __uint_as_float(w[i]) * c : -INFINITY;
            sv[i] = x;
            tmax = fmaxf(tmax, fmaxf(x, y));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      if (scol != nullptr) {
        if (key0 + HC <= k_end) {
#pragma unroll
          for (int i = 0; i < HC; ++i) scol[(long)(key0 + i) * a.R] = sv[i];
        } else {
#pragma unroll
          for (int i = 0; i < HC; ++i)  // (predicated, not a data-dependent trip count: sv stays in registers)
            if (key0 + i < k_end) scol[(long)(key0 + i) * a.R] = sv[i];
        }
      }
      // lazy rescale: the running max moves (and O / l are rescaled) only when a row's max
      // grows by more than 2^5 in p; P' = 2^10 p then stays below 2^15 (fp16), and the
      // pass's (M, L) stay a consistent pair for the split combine and scoring pass 2
      const float m_new = fmaxf(m_run, tmax);
      const bool grow = (m_new - m_run) * LOG2E > 5.f;  // also true on the first tile (m_run = -inf)
      const float m_use = grow ? m_new : m_run;
      const float corr = (m_run == -INFINITY) ? 0.f : ex2((m_run - m_use) * LOG2E);
      const float mb = m_use * LOG2E;
      float psum = 0.f;
      uint32_t ph[HC / 2], pm[HC / 2], pl[HC / 2];
#pragma unroll
      for (int i = 0; i < HC / 2; ++i) {
        const float p0 = ex2(fmaf(sv[2 * i], LOG2E, -mb)), p1 = ex2(fmaf(sv[2 * i + 1], LOG2E, -mb));
        psum += p0 + p1;
        if constexpr (S1_P_PLANES == 3) split3h_pack(p0 * S1_PSCALE, p1 * S1_PSCALE, ph[i], pm[i], pl[i]);
        else split2h_pack(p0 * S1_PSCALE, p1 * S1_PSCALE, ph[i], pm[i]);
      }
      const int pb = j % S1_P_BUFS;
      if (j >= S1_P_BUFS) {  // PV(j - B) has read this P buffer
        mbar_wait(&pv_full[pb], (uint32_t)((j - S1_P_BUFS) / S1_P_BUFS) & 1);
        tc_fence_after();
      }
      if (j >= 1 && __any_sync(0xffffffffu, grow)) {  // rescale O: PV(j-1) must have accumulated
        {
          const int jq = j - 1;
          mbar_wait(&pv_full[jq % S1_P_BUFS], (uint32_t)(jq / S1_P_BUFS) & 1);
          tc_fence_after();
        }
        {
          const float f = grow ? corr : 1.f;
#pragma unroll 1
          for (int c = hc * DKP / 64; c < (hc + 1) * DKP / 64; ++c) {
            uint32_t u[32];
            tmem_ld32(tmem + lb + C::T_O + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * f);
            tmem_st32(tmem + lb + C::T_O + c * 32, u);
          }
        }
      }
      l_run = l_run * (grow ? corr : 1.f) + psum;
      m_run = m_use;
      const uint32_t tP = tmem + lb + C::T_P + pb * 64;
      tmem_st16(tP + hc * (HC / 2), ph);
      tmem_st16(tP + C::KT / 2 + hc * (HC / 2), pm);
      if constexpr (S1_P_PLANES == 3) tmem_st16(tP + C::KT + hc * (HC / 2), pl);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
      if (warp == 0 && lane == 0) s1_stamp(a, 1, j);
    }
    if (warp == 0 && lane == 0) s1_stamp(a, 5, 1);
    if (n_tiles > 0) {
      const int jq = n_tiles - 1;  // the last PV completes after all earlier ones
      mbar_wait(&pv_full[jq % S1_P_BUFS], (uint32_t)(jq / S1_P_BUFS) & 1);
      tc_fence_after();
    }
    const long base = ((long)split * a.Hkv + g) * a.R + row;
#pragma unroll 1
    for (int c = hc * DKP / 64; c < (hc + 1) * DKP / 64; ++c) {
      uint32_t u[32];
      tmem_ld32(tmem + lb + C::T_O + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        float* od = a.Opart + base * DKP + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 4)  // the accumulator holds 2^10 p.v
          *reinterpret_cast<float4*>(od + i) =
              make_float4(__uint_as_float(u[i]) * (1.f / S1_PSCALE), __uint_as_float(u[i + 1]) * (1.f / S1_PSCALE),
                          __uint_as_float(u[i + 2]) * (1.f / S1_PSCALE), __uint_as_float(u[i + 3]) * (1.f / S1_PSCALE));
      }
    }
    // row sum = both halves (all MMAs and TMA loads are done: reuse the K/V ring)
    float* red = reinterpret_cast<float*>(sKV);
    red[hc * 128 + r] = l_run;
    named_bar_sync(1 + quarter, 64);
    if (valid && hc == 0) {
      a.Mpart[base] = n_tiles > 0 ? m_run : -INFINITY;
      a.Lpart[base] = l_run + red[128 + r];
    }
    if (warp == 0 && lane == 0) s1_stamp(a, 5, 2);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static unsigned long long* g_s1_trace = nullptr;

int s1_attn_tc_launch(const S1TcArgs& a_in, const void* k1, const void* k2, const void* v, long pool_rows_total,
                      int dkp, cudaStream_t st) {
  S1TcArgs a = a_in;
  if (a.n_splits <= 0) return PKV_OK;
  {
    static const bool tr = getenv("PKV_S1_TRACE") && getenv("PKV_S1_TRACE")[0] == '1';
    if (tr && g_s1_trace == nullptr && cudaMalloc(&g_s1_trace, 6 * 64 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(g_s1_trace, 0, 6 * 64 * sizeof(unsigned long long));
    a.trace = tr ? g_s1_trace : nullptr;
  }
  if (a.keys_per_split % 64 != 0) return set_error(PKV_ERR_ARGUMENT, "narrow pass: split not 64-aligned");
  const int RB = ceil_div(a.R, 128);
  dim3 grid(a.n_splits + (a.fresh ? 1 : 0), a.Hkv, RB);
  if (a.fresh && (a.m > 128 || (2L * a.m * (dkp + 4) + 128L * dkp + 10L * 32) * 4 > S1TcCfg<128>::SMEM - 2048))
    return set_error(PKV_ERR_ARGUMENT, "narrow pass: fused fresh split needs m <= 128");
  if (!a.q3_ready) {
    launch_k(s1_qprep_kernel, dim3(RB * 128, a.Hkv), 64, 0, st, a.q, a.m, a.H, a.G, a.R, RB, dkp,
             reinterpret_cast<__half*>(a.q3));
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("s1_qprep_kernel");
  }
  CUtensorMap m1, m2, mv;
  if (!cached_tmap(&m1, k1, pool_rows_total, dkp, dkp, 64) || !cached_tmap(&m2, k2, pool_rows_total, dkp, dkp, 64) ||
      !cached_tmap(&mv, v, pool_rows_total, dkp, dkp, 64))
    return set_error(PKV_ERR_CUDA, "narrow pass: TMA encode failed");
  if (dkp == 128) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, S1TcCfg<128>::SMEM);
    });
    launch_k(s1_attn_tc_kernel<128>, grid, 320, S1TcCfg<128>::SMEM, st, m1, m2, mv, a);
  } else if (dkp == 64) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, S1TcCfg<64>::SMEM);
    });
    launch_k(s1_attn_tc_kernel<64>, grid, 320, S1TcCfg<64>::SMEM, st, m1, m2, mv, a);
  } else {
    return set_error(PKV_ERR_CONFIG, "narrow pass: padded head dim %d unsupported", dkp);
  }
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("s1_attn_tc_kernel");
  return PKV_OK;
}


// ---------------------------------------------------------------------------------
// Scoring pass 2 (reference selection.py:76-86 over model.py:294-307):
// the context keys' scores without the [Hkv][s][R] fp32 score matrix.  Pass 1
// (s1_attn_tc_kernel with S = null) leaves the final per-row max M and denominator L;
// this kernel recomputes Q'K^T with the SAME fp16 plane products (identical
// accumulator), forms p = 2^(S log2e - M log2e) * w with w = 1 / (L H m) (or the
// context-renormalised weight, s1_row_weights_kernel) and sums p over the CTA's 128 rows
// = (G query heads x m queries) for every key of its split: a warp transposes-and-adds
// its 32 x 32 block with 31 shuffles (lane c ends with column c), the four TMEM lane
// quarters add through shared memory in a fixed order.  One f32 per (row block, KV
// head, key) goes to HBM instead of 128.
//
// CTA = (key split, KV head g, row block); 128-key tiles = one cache page, 3-stage TMA
// ring of the two key planes, S double-buffered in TMEM so the MMAs of page j+1 run
// under the reduction of page j.
//   warps 0-7  reduction: warp w owns lane quarter w%4 and columns [64*(w/4), +64)
//   warp 8     TMA producer (Kh, Kl)       warp 9  TMEM owner + MMA issuer
template <int DKP>
struct S1ScCfg {
  static constexpr int ATOMS = DKP / 64;
  static constexpr int KT = 128;
  static constexpr int PLANE = KT * DKP * 2;
  static constexpr int ATOM_K = KT * 128;
  static constexpr int STAGE = 2 * PLANE;
  static constexpr int STAGES = DKP == 128 ? 3 : 6;
  static constexpr int RED = 2 * 4 * KT * 4;  // double-buffered [4 quarters][KT] f32
  static constexpr int SMEM = STAGES * STAGE + RED + 1024 + 256;
  static constexpr int T_Q = 0, Q_PLANE = 64, T_S = 256;
};

// lane c returns sum over the warp's 32 lanes of v[c] (v is clobbered)
__device__ __forceinline__ float warp_colsum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool up = (lane & k) != 0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = up ? v[i] : v[i + k];
      const float keep = up ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

template <int DKP>
__global__ void __launch_bounds__(320, 1)
    s1_score_tc_kernel(const __grid_constant__ CUtensorMap tK1, const __grid_constant__ CUtensorMap tK2,
                       S1ScoreArgs a) {
  using C = S1ScCfg<DKP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  float* red = reinterpret_cast<float*>(sK + C::STAGES * C::STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(red) + C::RED);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + C::STAGES;
  uint64_t* s_full = bars + 2 * C::STAGES;  // [2]
  uint64_t* s_free = s_full + 2;            // [2]
  uint64_t* q_full = s_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.y, split = blockIdx.x, rb = blockIdx.z;
  if (a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[0] = t;
  }
  const int k_begin = split * a.keys_per_split;
  const int k_end = min(k_begin + a.keys_per_split, a.s);
  const int n_tiles = (k_end - k_begin + C::KT - 1) / C::KT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 8);
    }
    mbar_init(q_full, 8);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();
  griddep_launch();

  if (warp == 8) {
    if (elect_one()) {
      tma_prefetch(&tK1);
      tma_prefetch(&tK2);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % C::STAGES;
        mbar_wait(&kv_empty[st], ((uint32_t)(j / C::STAGES) & 1) ^ 1);
        const int t0 = k_begin + j * C::KT;  // page-aligned
        const int row = (int)(head_row + (long)a.page_table[t0 >> 7] * 128);
        uint8_t* base = sK + st * C::STAGE;
        mbar_expect_tx(&kv_full[st], C::STAGE);
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at) {
          tma_load_2d(base + at * C::ATOM_K, &tK1, &kv_full[st], at * 64, row);
          tma_load_2d(base + C::PLANE + at * C::ATOM_K, &tK2, &kv_full[st], at * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idesc = make_idesc_f16(128, C::KT);
    constexpr int NPROD = S1_QK_PROD;  // the first pass's products, same order
    constexpr int PA[5] = {0, 1, 0, 2, 1};
    constexpr int PB[5] = {0, 0, 1, 0, 1};
    mbar_wait(q_full, 0);
    tc_fence_after();
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j % C::STAGES, b = j & 1;
      mbar_wait(&kv_full[st], (uint32_t)(j / C::STAGES) & 1);
      if (j >= 2) mbar_wait(&s_free[b], (uint32_t)((j - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k_addr = smem_u32(sK + st * C::STAGE);
        int n = 0;
#pragma unroll
        for (int pr = 0; pr < NPROD; ++pr)
#pragma unroll
          for (int kk = 0; kk < DKP / 16; ++kk, ++n) {
            const uint32_t ko = PB[pr] * C::PLANE + (kk >> 2) * C::ATOM_K + (kk & 3) * 32;
            umma_ts(tmem + C::T_S + b * C::KT, tmem + C::T_Q + PA[pr] * C::Q_PLANE + kk * 8,
                    sdesc_sw128(k_addr + ko, 16, 1024), idesc, n > 0 ? 1u : 0u);
          }
        umma_commit(&s_full[b]);
        umma_commit(&kv_empty[st]);
      }
      __syncwarp();
    }
  } else {
    constexpr float LOG2E = 1.4426950408889634f;
    const int quarter = warp & 3, hc = warp >> 2;
    const int r = quarter * 32 + lane;
    const int row = rb * 128 + r;
    const bool valid = row < a.R;
    const uint32_t lb = (uint32_t)(quarter * 32) << 16;
    {  // Q planes -> TMEM, as in the first pass
      const __half* q3 = reinterpret_cast<const __half*>(a.q3);
      if (hc * 32 < DKP / 2) {
#pragma unroll 1
        for (int x = 0; x < S1_Q_PLANES; ++x) {
          const uint4* src = reinterpret_cast<const uint4*>(
              q3 + ((((long)g * gridDim.z + rb) * 3 + x) * 128 + r) * DKP + hc * 64);
          uint32_t u[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = src[c];
            u[4 * c] = v.x; u[4 * c + 1] = v.y; u[4 * c + 2] = v.z; u[4 * c + 3] = v.w;
          }
          tmem_st32(tmem + lb + C::T_Q + x * C::Q_PLANE + hc * 32, u);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    const float mb = valid ? a.Mfin[(long)g * a.R + row] * LOG2E : 0.f;
    const float wr = valid ? a.W[(long)g * a.R + row] : 0.f;
    const float c1 = (a.scale * (1.f / S1_QSCALE)) * LOG2E;
    float* out = a.part + ((long)rb * a.Hkv + g) * a.s;
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && warp == 0 &&
                    lane == 0;
    auto stamp = [&](int i) {
      if (tr && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[i] = t;
      }
    };
    stamp(1);
    for (int j = 0; j < n_tiles; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (uint32_t)(j >> 1) & 1);
      tc_fence_after();
      stamp(4 + j);
      uint32_t u0[32], u1[32];
      tmem_ld32(tmem + lb + C::T_S + b * C::KT + hc * 64, u0);
      tmem_ld32(tmem + lb + C::T_S + b * C::KT + hc * 64 + 32, u1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[b]);
      const int key0 = k_begin + j * C::KT + hc * 64;
      float* rq = red + (b * 4 + quarter) * C::KT + hc * 64;
      {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          v[i] = (valid && key0 + i < k_end) ? ex2(fmaf(__uint_as_float(u0[i]), c1, -mb)) * wr : 0.f;
        rq[lane] = warp_colsum32(v);
      }
      {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          v[i] = (valid && key0 + 32 + i < k_end) ? ex2(fmaf(__uint_as_float(u1[i]), c1, -mb)) * wr : 0.f;
        rq[32 + lane] = warp_colsum32(v);
      }
      named_bar_sync(1, 256);
      if (quarter == 0) {
        const float* rr = red + b * 4 * C::KT + hc * 64;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = h2 * 32 + lane;
          const float sum = ((rr[c] + rr[C::KT + c]) + rr[2 * C::KT + c]) + rr[3 * C::KT + c];
          if (key0 + c < k_end) out[key0 + c] = sum;
        }
      }
    }
    stamp(2);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static unsigned long long* g_s1s_trace = nullptr;

int s1_score_tc_launch(const S1ScoreArgs& a_in, const void* k1, const void* k2, long pool_rows_total, int dkp,
                       cudaStream_t st) {
  S1ScoreArgs a = a_in;
  if (a.n_splits <= 0) return PKV_OK;
  {
    static const bool tr = getenv("PKV_S1_TRACE") && getenv("PKV_S1_TRACE")[0] == '1';
    if (tr && g_s1s_trace == nullptr && cudaMalloc(&g_s1s_trace, 64 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(g_s1s_trace, 0, 64 * sizeof(unsigned long long));
    a.trace = tr ? g_s1s_trace : nullptr;
  }
  if (a.keys_per_split % 128 != 0) return set_error(PKV_ERR_ARGUMENT, "score pass: split not page-aligned");
  const int RB = ceil_div(a.R, 128);
  dim3 grid(a.n_splits, a.Hkv, RB);
  CUtensorMap m1, m2;
  if (!cached_tmap(&m1, k1, pool_rows_total, dkp, dkp, 128) || !cached_tmap(&m2, k2, pool_rows_total, dkp, dkp, 128))
    return set_error(PKV_ERR_CUDA, "score pass: TMA encode failed");
  if (dkp == 128) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_score_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, S1ScCfg<128>::SMEM);
    });
    launch_k(s1_score_tc_kernel<128>, grid, 320, S1ScCfg<128>::SMEM, st, m1, m2, a);
  } else if (dkp == 64) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_score_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, S1ScCfg<64>::SMEM);
    });
    launch_k(s1_score_tc_kernel<64>, grid, 320, S1ScCfg<64>::SMEM, st, m1, m2, a);
  } else {
    return set_error(PKV_ERR_CONFIG, "score pass: padded head dim %d unsupported", dkp);
  }
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("s1_score_tc_kernel");
  return PKV_OK;
}

}  // namespace pkv

extern "C" int pkv_debug_s1_trace(unsigned long long* host) {
  if (pkv::g_s1_trace == nullptr) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, pkv::g_s1_trace, 6 * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}

extern "C" int pkv_debug_s1_score_trace(unsigned long long* host) {
  if (pkv::g_s1s_trace == nullptr) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, pkv::g_s1s_trace, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}
