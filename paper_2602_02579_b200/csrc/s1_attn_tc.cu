// fp32-faithful narrow-pass attention on tcgen05 (reference model.py:278-308 as
// called by query_pass model.py:370-402, i.e. score_prophet and finalize_query).
//
// The reference computes q.k and p.v in float64 on f32 inputs.  Here every fp32
// operand x is split exactly into three bf16 planes x = xh + xm + xl (24 bits of
// significand), so
//     Q K^T  = Qh Kh + Qh Km + Qm Kh + Qh Kl + Qm Km + Ql Kh   (+ terms < 2^-24 rel.)
//     P V    = Ph V + Pm V + Pl V                                (V is bf16-exact)
// on the bf16 tensor cores with fp32 accumulation in TMEM.  Only the context keys
// [0, s) run here; the m fresh query keys (fp32 V) are a separate SIMT split.
//
// CTA = (KV head g, key split): 128 rows r = j*m + i (query head g*G+j, query i),
// 64-key tiles, 2-stage smem ring.
//   warps 0-3  producers: load K (chunk store: unrotated bf16 + float64 RoPE, or
//              the repaired pool entry), split 3-way, write SW128 K-major planes
//              and the V tile (MN-major for the PV MMA)
//   warps 4-7  softmax: S row from TMEM, scale+mask, exact online softmax
//              (expf), scores -> S workspace, P split -> TMEM (A operand of PV)
//   warp 8     TMEM owner + MMA issuer
#include <mutex>

#include "kernels.cuh"

namespace pkv {


template <int DKP>
struct S1TcCfg {
  static constexpr int ATOMS = DKP / 64;
  static constexpr int KT = 64;                       // keys per tile
  static constexpr int QSPLIT = 128 * DKP * 2;        // one Q plane (128 rows)
  static constexpr int PLANE = KT * DKP * 2;          // one K plane / the V tile
  static constexpr int ATOM_Q = 128 * 128;            // bytes per 64-col atom of a Q plane
  static constexpr int ATOM_K = KT * 128;             // bytes per 64-col atom of a K/V plane
  static constexpr int STAGE = 4 * PLANE;             // Kh, Km, Kl, V
  static constexpr int STAGES = 2;
  static constexpr int SMEM = 3 * QSPLIT + STAGES * STAGE + 1024 + 256;
  // TMEM columns: S0 [0,64) S1 [64,128) O [128,128+DKP) P planes [256,352)
  static constexpr int T_S = 0, T_O = 128, T_P = 256;
};

__device__ __forceinline__ void split3_bf(float x, uint32_t& h, uint32_t& m, uint32_t& l) {
  __nv_bfloat16 a = __float2bfloat16_rn(x);
  float r1 = x - __bfloat162float(a);
  __nv_bfloat16 b = __float2bfloat16_rn(r1);
  float r2 = r1 - __bfloat162float(b);
  __nv_bfloat16 c = __float2bfloat16_rn(r2);
  h = *reinterpret_cast<uint16_t*>(&a);
  m = *reinterpret_cast<uint16_t*>(&b);
  l = *reinterpret_cast<uint16_t*>(&c);
}

template <int DKP>
__global__ void __launch_bounds__(288, 1) s1_attn_tc_kernel(S1TcArgs a) {
  using C = S1TcCfg<DKP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                     // 3 planes
  uint8_t* sKV = smem + 3 * C::QSPLIT;    // STAGES x {Kh, Km, Kl, V}
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::STAGES * C::STAGE);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + C::STAGES;
  uint64_t* s_full = bars + 2 * C::STAGES;
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_free + 2;
  uint64_t* pv_full = p_full + 1;
  uint64_t* q_full = pv_full + 1;
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
      mbar_init(&kv_full[i], 4);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_full, 1);
    mbar_init(q_full, 4);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------- producers
    const int tid = threadIdx.x;  // 0..127
    constexpr int VECS = DKP / 8;
    const int half = a.dk >> 1;
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j % C::STAGES;
      mbar_wait(&kv_empty[st], ((uint32_t)(j / C::STAGES) & 1) ^ 1);
      uint8_t* base = sKV + st * C::STAGE;
      for (int e = tid; e < C::KT * VECS; e += 128) {
        const int kr = e / VECS, c8 = e - kr * VECS;
        const int t = k_begin + j * C::KT + kr;
        uint32_t kh[4], km[4], kl[4];
        uint4 vraw = make_uint4(0, 0, 0, 0);
        if (t < k_end) {
          const bool from_chunk = a.src_chunks && !(a.recomp != nullptr && a.recomp[t]);
          uint4 kraw;
          if (from_chunk) {
            const int ch = a.src_chunk[t], loc = a.src_local[t], tc = a.chunk_len[ch];
            const long off = (((long)a.layer * tc + loc) * a.Hkv + g) * DKP + c8 * 8;
            kraw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.ck[ch]) + off));
            vraw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.cv[ch]) + off));
          } else {
            const long slot = (long)a.page_table[t >> 7] * 128 + (t & 127);
            const long off = ((long)g * a.pool_tokens + slot) * DKP + c8 * 8;
            kraw = *reinterpret_cast<const uint4*>(a.k_pool + off);
            vraw = *reinterpret_cast<const uint4*>(a.v_pool + off);
          }
          const uint32_t kw[4] = {kraw.x, kraw.y, kraw.z, kraw.w};
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            float e0 = bf16_lo(kw[p]), e1 = bf16_hi(kw[p]);
            const int pi = c8 * 4 + p;
            if (from_chunk && pi < half) {
              const double cs = a.rcos[(long)t * half + pi], sn = a.rsin[(long)t * half + pi];
              const double de = e0, dd = e1;
              e0 = (float)__dsub_rn(__dmul_rn(de, cs), __dmul_rn(dd, sn));
              e1 = (float)__dadd_rn(__dmul_rn(de, sn), __dmul_rn(dd, cs));
            }
            uint32_t h0, m0, l0, h1, m1, l1;
            split3_bf(e0, h0, m0, l0);
            split3_bf(e1, h1, m1, l1);
            kh[p] = h0 | (h1 << 16);
            km[p] = m0 | (m1 << 16);
            kl[p] = l0 | (l1 << 16);
          }
        } else {
#pragma unroll
          for (int p = 0; p < 4; ++p) kh[p] = km[p] = kl[p] = 0u;
        }
        const uint32_t off = (c8 >> 3) * C::ATOM_K + sw128_offset(kr, (c8 & 7) * 8);
        *reinterpret_cast<uint4*>(base + off) = make_uint4(kh[0], kh[1], kh[2], kh[3]);
        *reinterpret_cast<uint4*>(base + C::PLANE + off) = make_uint4(km[0], km[1], km[2], km[3]);
        *reinterpret_cast<uint4*>(base + 2 * C::PLANE + off) = make_uint4(kl[0], kl[1], kl[2], kl[3]);
        *reinterpret_cast<uint4*>(base + 3 * C::PLANE + off) = vraw;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&kv_full[st]);
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16(128, C::KT);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, DKP, /*b_mn_major=*/true);
    constexpr int PA[6] = {0, 0, 1, 0, 1, 2};  // Q plane of each product
    constexpr int PB[6] = {0, 1, 0, 2, 1, 0};  // K plane of each product
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    for (int j = 0; j <= n_tiles; ++j) {
      if (j < n_tiles) {
        const int st = j % C::STAGES;
        mbar_wait(&kv_full[st], (uint32_t)(j / C::STAGES) & 1);
        if (j >= 2) mbar_wait(&s_free[j & 1], (uint32_t)((j - 2) >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t k_addr = smem_u32(sKV + st * C::STAGE);
          int n = 0;
#pragma unroll
          for (int pr = 0; pr < 6; ++pr)
#pragma unroll
            for (int kk = 0; kk < DKP / 16; ++kk, ++n) {
              const uint32_t qo = PA[pr] * C::QSPLIT + (kk >> 2) * C::ATOM_Q + (kk & 3) * 32;
              const uint32_t ko = PB[pr] * C::PLANE + (kk >> 2) * C::ATOM_K + (kk & 3) * 32;
              umma_bf16(tmem + C::T_S + (j & 1) * C::KT, sdesc_sw128(q_addr + qo, 16, 1024),
                        sdesc_sw128(k_addr + ko, 16, 1024), idesc_s, n > 0 ? 1u : 0u);
            }
          umma_commit(&s_full[j & 1]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jp = j - 1;
        const int st = jp % C::STAGES;
        mbar_wait(p_full, (uint32_t)jp & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = smem_u32(sKV + st * C::STAGE + 3 * C::PLANE);
          int n = 0;
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int kk = 0; kk < C::KT / 16; ++kk, ++n)
              umma_bf16_ts(tmem + C::T_O, tmem + C::T_P + x * (C::KT / 2) + kk * 8,
                           sdesc_sw128(v_addr + kk * 16 * 128, C::ATOM_K, 1024), idesc_o,
                           (jp > 0 || n > 0) ? 1u : 0u);
          umma_commit(pv_full);
          umma_commit(&kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // TMEM lane == tile row
    const int row = r0 + r;
    const bool valid = row < a.R;
    const int jh = valid ? row / a.m : 0, qi = valid ? row - jh * a.m : 0;
    const uint32_t lb = (uint32_t)(quarter * 32) << 16;
    {  // Q planes
      const float* src = a.q + ((long)qi * a.H + g * a.G + jh) * DKP;
#pragma unroll 1
      for (int c8 = 0; c8 < DKP / 8; ++c8) {
        uint32_t h[4], m[4], l[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float e0 = valid ? src[c8 * 8 + 2 * p] : 0.f, e1 = valid ? src[c8 * 8 + 2 * p + 1] : 0.f;
          uint32_t h0, m0, l0, h1, m1, l1;
          split3_bf(e0, h0, m0, l0);
          split3_bf(e1, h1, m1, l1);
          h[p] = h0 | (h1 << 16);
          m[p] = m0 | (m1 << 16);
          l[p] = l0 | (l1 << 16);
        }
        const uint32_t off = (c8 >> 3) * C::ATOM_Q + sw128_offset(r, (c8 & 7) * 8);
        *reinterpret_cast<uint4*>(sQ + off) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(sQ + C::QSPLIT + off) = make_uint4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<uint4*>(sQ + 2 * C::QSPLIT + off) = make_uint4(l[0], l[1], l[2], l[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    float m_run = -INFINITY, l_run = 0.f;
    float* srow = (a.S != nullptr && valid) ? a.S + ((long)g * a.R + row) * a.s_tot : nullptr;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&s_full[j & 1], (uint32_t)(j >> 1) & 1);
      tc_fence_after();
      float sv[C::KT];
#pragma unroll
      for (int c = 0; c < C::KT / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tmem + lb + C::T_S + (j & 1) * C::KT + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(u[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[j & 1]);
      const int key0 = k_begin + j * C::KT;
      float tmax = -INFINITY;
#pragma unroll
      for (int i = 0; i < C::KT; ++i) {
        const float x = (key0 + i < k_end) ? sv[i] * a.scale : -INFINITY;
        sv[i] = x;
        tmax = fmaxf(tmax, x);
      }
      if (srow != nullptr) {
        if (key0 + C::KT <= k_end) {
#pragma unroll
          for (int i = 0; i < C::KT; i += 4)
            *reinterpret_cast<float4*>(srow + key0 + i) = make_float4(sv[i], sv[i + 1], sv[i + 2], sv[i + 3]);
        } else {
          for (int i = 0; i < C::KT && key0 + i < k_end; ++i) srow[key0 + i] = sv[i];
        }
      }
      const float m_new = fmaxf(m_run, tmax);
      const bool grow = m_new > m_run;
      const float corr = (m_run == -INFINITY) ? 0.f : expf(m_run - m_new);
      float psum = 0.f;
      uint32_t ph[C::KT / 2], pm[C::KT / 2], pl[C::KT / 2];
#pragma unroll
      for (int i = 0; i < C::KT / 2; ++i) {
        const float p0 = expf(sv[2 * i] - m_new), p1 = expf(sv[2 * i + 1] - m_new);
        psum += p0 + p1;
        uint32_t h0, m0, l0, h1, m1, l1;
        split3_bf(p0, h0, m0, l0);
        split3_bf(p1, h1, m1, l1);
        ph[i] = h0 | (h1 << 16);
        pm[i] = m0 | (m1 << 16);
        pl[i] = l0 | (l1 << 16);
      }
      if (j >= 1) {
        mbar_wait(pv_full, (uint32_t)(j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow)) {
          const float f = grow ? corr : 1.f;
#pragma unroll 1
          for (int c = 0; c < DKP / 32; ++c) {
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
      m_run = m_new;
      tmem_st32(tmem + lb + C::T_P, ph);
      tmem_st32(tmem + lb + C::T_P + C::KT / 2, pm);
      tmem_st32(tmem + lb + C::T_P + C::KT, pl);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    if (n_tiles > 0) {
      mbar_wait(pv_full, (uint32_t)(n_tiles - 1) & 1);
      tc_fence_after();
    }
    const long base = ((long)split * a.Hkv + g) * a.R + row;
#pragma unroll 1
    for (int c = 0; c < DKP / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tmem + lb + C::T_O + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        float* od = a.Opart + base * DKP + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(od + i) = make_float4(__uint_as_float(u[i]), __uint_as_float(u[i + 1]),
                                                           __uint_as_float(u[i + 2]), __uint_as_float(u[i + 3]));
      }
    }
    if (valid) {
      a.Mpart[base] = n_tiles > 0 ? m_run : -INFINITY;
      a.Lpart[base] = l_run;
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int s1_attn_tc_launch(const S1TcArgs& a, cudaStream_t st) {
  dim3 grid(a.n_splits, a.Hkv, ceil_div(a.R, 128));
  if (a.n_splits <= 0) return PKV_OK;
  if (a.dk > 128) return set_error(PKV_ERR_CONFIG, "head_dim > 128");
  // the kernel template follows the padded head dim of the cache layout
  const int dkp = a.dk <= 64 ? 64 : 128;
  if (dkp == 128) {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           S1TcCfg<128>::SMEM);
    });
    s1_attn_tc_kernel<128><<<grid, 288, S1TcCfg<128>::SMEM, st>>>(a);
  } else {
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(s1_attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, S1TcCfg<64>::SMEM);
    });
    s1_attn_tc_kernel<64><<<grid, 288, S1TcCfg<64>::SMEM, st>>>(a);
  }
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("s1_attn_tc_kernel");
  return PKV_OK;
}

}  // namespace pkv
