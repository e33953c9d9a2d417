// Sparse-query causal attention on tcgen05 (Stage II, reference recompute.py:80-81
// -> model.py:_attend 278-308 with pos_q = positions of the selected tokens and
// pos_kv = 0..s-1 over the repaired cache).
//
// One CTA = one KV head g and a block of T = 128/G selected tokens; its 128 MMA rows
// are the G query heads sharing g (GQA packing), row r = j*T + i (head g*G+j,
// token b*T+i).  KV tiles are 128-token pages of the paged cache, TMA-loaded.
//
//   warps 0-7  softmax: warp w owns TMEM lane quarter w%4 (32 rows) and key
//              columns [64*(w/4), +64) of each tile; both warps of a quarter read
//              the full S row for the max (no exchange), then exponentiate their
//              half in the log2 domain, P -> smem (bf16, SW128 K-major atom w/4),
//              conditional O rescale in TMEM (only when the max grows by > 2^8)
//   warp 8     TMA producer: K and V pages, 2-stage ring
//   warp 9     TMEM owner + MMA issuer: S = Q K^T (double-buffered in TMEM),
//              O += P V (V as MN-major B operand)
#include <mutex>
#include "kernels.cuh"
#include "gemm_tc.cuh"

namespace pkv {

struct AttnArgs {
  const __nv_bfloat16* q;    // [n_q][H][DKP]
  __nv_bfloat16* out;        // [n_q][H][DKP]
  const int32_t* pos;        // [n_q] ascending
  const int32_t* page_table; // logical page -> physical page
  int n_q, H, Hkv, G, T, n_tiles;
  long kv_row0;              // first pool row of this layer: layer * Hkv * pool_tokens
  long pool_tokens;
  float scale_log2;          // log2(e) / sqrt(head_dim)
};

template <int DKP>
struct AttnCfg {
  static constexpr int ATOMS = DKP / 64;
  static constexpr int Q_BYTES = 128 * DKP * 2;
  static constexpr int KV_BYTES = 128 * DKP * 2;  // one K or V page
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int STAGES = 2;
  static constexpr int SMEM = Q_BYTES + STAGES * 2 * KV_BYTES + P_BYTES + 1024 + 256;
  static constexpr int SOFTMAX_WARPS = 8;
};

template <int DKP>
__global__ void __launch_bounds__(320, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  using Cfg = AttnCfg<DKP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + Cfg::Q_BYTES;  // stage s: K at sKV + s*2*KV_BYTES, V right after
  uint8_t* sP = sKV + Cfg::STAGES * 2 * Cfg::KV_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + Cfg::P_BYTES);
  uint64_t* kv_full = bars;                    // [STAGES]
  uint64_t* kv_empty = bars + Cfg::STAGES;     // [STAGES]
  uint64_t* s_full = bars + 2 * Cfg::STAGES;   // [2]
  uint64_t* s_free = s_full + 2;               // [2]
  uint64_t* p_full = s_free + 2;
  uint64_t* pv_full = p_full + 1;
  uint64_t* q_full = pv_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % a.Hkv;
  const int b = a.n_tiles - 1 - blockIdx.x / a.Hkv;  // heaviest token blocks first (LPT)
  const int tok0 = b * a.T;
  const int last_tok = min(tok0 + a.T, a.n_q) - 1;
  const int max_pos = a.pos[last_tok];
  const int min_pos = a.pos[tok0];
  const int n_kv_tiles = max_pos / 128 + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], Cfg::SOFTMAX_WARPS);
    }
    mbar_init(p_full, Cfg::SOFTMAX_WARPS);
    mbar_init(pv_full, 1);
    mbar_init(q_full, Cfg::SOFTMAX_WARPS);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;          // S buffers at cols 0 and 128
  const uint32_t tO = tmem + 256;    // O accumulator

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_kv_tiles; ++j) {
        const int st = j % Cfg::STAGES;
        const uint32_t ph = (uint32_t)(j / Cfg::STAGES) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        uint8_t* sk = sKV + st * 2 * Cfg::KV_BYTES;
        uint8_t* sv = sk + Cfg::KV_BYTES;
        const int row = (int)(head_row + (long)a.page_table[j] * 128);
        mbar_expect_tx(&kv_full[st], 2 * Cfg::KV_BYTES);
#pragma unroll
        for (int at = 0; at < Cfg::ATOMS; ++at) {
          tma_load_2d(sk + at * 16384, &tmK, &kv_full[st], at * 64, row);
          tma_load_2d(sv + at * 16384, &tmV, &kv_full[st], at * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, DKP, /*b_mn_major=*/true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    const uint32_t p_addr = smem_u32(sP);
    for (int j = 0; j <= n_kv_tiles; ++j) {
      if (j < n_kv_tiles) {
        const int st = j % Cfg::STAGES;
        mbar_wait(&kv_full[st], (uint32_t)(j / Cfg::STAGES) & 1);
        if (j >= 2) mbar_wait(&s_free[j & 1], (uint32_t)((j - 2) >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t k_addr = smem_u32(sKV + st * 2 * Cfg::KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < DKP / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_bf16(tS + (j & 1) * 128, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024),
                      idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[j & 1]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jp = j - 1;
        const int st = jp % Cfg::STAGES;
        mbar_wait(p_full, (uint32_t)jp & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = smem_u32(sKV + st * 2 * Cfg::KV_BYTES + Cfg::KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t a_off = (kk >> 2) * 16384 + (kk & 3) * 32;  // P: K-major, 64-col atoms
            const uint32_t b_off = kk * 16 * 128;                       // V: 16 kv rows per step
            umma_bf16(tO, sdesc_sw128(p_addr + a_off, 16, 1024), sdesc_sw128(v_addr + b_off, 16384, 1024), idesc_o,
                      (jp > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(pv_full);
          umma_commit(&kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax
    const int quarter = warp & 3, hc = warp >> 2;
    const int r = quarter * 32 + lane;  // 0..127 == TMEM lane
    const int hj = r / a.T;
    const int ti = r - hj * a.T;
    const int tok = tok0 + ti;
    const bool valid = hj < a.G && tok < a.n_q;
    const int head = g * a.G + hj;
    const int my_pos = valid ? a.pos[tok] : max_pos;
    const uint32_t lane_base = (uint32_t)((quarter * 32) << 16);
    const float sl2 = a.scale_log2;

    // Q row -> smem (this warp: 64-column atom hc), 128B-swizzled K-major
    if (hc < Cfg::ATOMS) {
      const uint4* src = valid ? reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) : nullptr;
#pragma unroll
      for (int c = hc * 8; c < hc * 8 + 8; ++c) {
        uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
        const int ch = (c & 7) ^ (r & 7);
        *reinterpret_cast<uint4*>(sQ + hc * 16384 + r * 128 + ch * 16) = v;
      }
      fence_proxy_async_smem();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(q_full);

    float m_run = -INFINITY, l_run = 0.f;  // m in log2 units; l: this warp's half of the row sum
    for (int j = 0; j < n_kv_tiles; ++j) {
      mbar_wait(&s_full[j & 1], (uint32_t)(j >> 1) & 1);
      tc_fence_after();
      const int key0 = j * 128;
      const bool unmasked = key0 + 127 <= min_pos;
      // the partner half only contributes to the max
      float omax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        const int col = (hc ^ 1) * 64 + c * 32;
        tmem_ld32(tS + lane_base + (j & 1) * 128 + col, u);
        tmem_ld_wait();
        if (unmasked) {
#pragma unroll
          for (int i = 0; i < 32; ++i) omax = fmaxf(omax, __uint_as_float(u[i]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (key0 + col + i <= my_pos) omax = fmaxf(omax, __uint_as_float(u[i]));
        }
      }
      float s[64];
      float lmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        const int col = hc * 64 + c * 32;
        tmem_ld32(tS + lane_base + (j & 1) * 128 + col, u);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float x = (unmasked || key0 + col + i <= my_pos) ? __uint_as_float(u[i]) : -INFINITY;
          s[c * 32 + i] = x;
          lmax = fmaxf(lmax, x);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[j & 1]);

      const float m_new = fmaxf(m_run, fmaxf(lmax, omax) * sl2);
      const bool grow = (m_new - m_run) > 8.0f;  // also true on the first tile (m_run = -inf)
      const float m_use = grow ? m_new : m_run;
      float rsum = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float p0 = ex2(fmaf(s[2 * i], sl2, -m_use)), p1 = ex2(fmaf(s[2 * i + 1], sl2, -m_use));
        rsum += p0 + p1;
        pk[i] = pack_bf16(p0, p1);
      }
      // previous PV must be done before P is overwritten and before O is rescaled
      if (j >= 1) {
        mbar_wait(pv_full, (uint32_t)(j - 1) & 1);
        tc_fence_after();
      }
      const bool any_grow = __any_sync(0xffffffffu, grow && j > 0) != 0;
      if (any_grow) {
        const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
        for (int c = hc * DKP / 64; c < (hc + 1) * DKP / 64; ++c) {
          uint32_t u[32];
          tmem_ld32(tO + lane_base + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st32(tO + lane_base + c * 32, u);
        }
        tmem_st_wait();
      }
      if (grow && j > 0) l_run *= ex2(m_run - m_use);
      if (grow) m_run = m_use;
      l_run += rsum;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int ch = c ^ (r & 7);
        *reinterpret_cast<uint4*>(sP + hc * 16384 + r * 128 + ch * 16) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(pv_full, (uint32_t)(n_kv_tiles - 1) & 1);
    tc_fence_after();
    // row sum = both halves; all MMAs are done, so the P buffer is free for the exchange
    float* red = reinterpret_cast<float*>(sP);
    red[hc * 128 + r] = l_run;
    named_bar_sync(1 + quarter, 64);
    const float inv_l = 1.f / (red[r] + red[128 + r]);
#pragma unroll 1
    for (int c = hc * DKP / 64; c < (hc + 1) * DKP / 64; ++c) {
      uint32_t u[32];
      tmem_ld32(tO + lane_base + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(__uint_as_float(u[8 * i]) * inv_l, __uint_as_float(u[8 * i + 1]) * inv_l),
                              pack_bf16(__uint_as_float(u[8 * i + 2]) * inv_l, __uint_as_float(u[8 * i + 3]) * inv_l),
                              pack_bf16(__uint_as_float(u[8 * i + 4]) * inv_l, __uint_as_float(u[8 * i + 5]) * inv_l),
                              pack_bf16(__uint_as_float(u[8 * i + 6]) * inv_l, __uint_as_float(u[8 * i + 7]) * inv_l));
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
template <int DKP>
static int launch_attn(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream) {
  using Cfg = AttnCfg<DKP>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(attn_tc_kernel<DKP>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn smem attr: %s", cudaGetErrorString(err));
  attn_tc_kernel<DKP><<<a.n_tiles * a.Hkv, 320, Cfg::SMEM, stream>>>(tk, tv, a);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_tc_kernel");
  return PKV_OK;
}

// q/out: [n_q][H][dkp] bf16; k_pool/v_pool: [L][Hkv][pool_tokens][dkp] bf16 (whole pool)
int attn_tc_launch(const void* q, void* out, const int32_t* pos, int n_q, int H, int Hkv, int head_dim, int dkp,
                   const void* k_pool, const void* v_pool, long pool_rows_total, long pool_tokens, int layer,
                   const int32_t* page_table, cudaStream_t stream) {
  if (n_q <= 0) return PKV_OK;
  const int G = H / Hkv;
  if (G > 128) return set_error(PKV_ERR_CONFIG, "attention: group size %d > 128", G);
  AttnArgs a;
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.pos = pos;
  a.page_table = page_table;
  a.n_q = n_q;
  a.H = H;
  a.Hkv = Hkv;
  a.G = G;
  a.T = 128 / G;
  a.n_tiles = ceil_div(n_q, a.T);
  a.kv_row0 = (long)layer * Hkv * pool_tokens;
  a.pool_tokens = pool_tokens;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  CUtensorMap tk, tv;
  if (!cached_tmap(&tk, k_pool, pool_rows_total, dkp, dkp, 128) ||
      !cached_tmap(&tv, v_pool, pool_rows_total, dkp, dkp, 128))
    return set_error(PKV_ERR_CUDA, "attention: TMA encode failed");
  if (dkp == 128) return launch_attn<128>(tk, tv, a, stream);
  if (dkp == 64) return launch_attn<64>(tk, tv, a, stream);
  return set_error(PKV_ERR_CONFIG, "attention: padded head dim %d unsupported", dkp);
}

}  // namespace pkv
