// Sparse-query causal attention on tcgen05 (Stage II, reference recompute.py:80-81
// -> model.py:_attend 278-308 with pos_q = positions of the selected tokens and
// pos_kv = 0..s-1 over the repaired cache).  Q, K, V and P are fp16 (fp32 accumulation).
//
// GQA packing: a 128-row Q tile = the G query heads sharing KV head g for a block of
// T = 128/G selected tokens, row r = j*T + i (head g*G+j, token b*T+i).
// One CTA = KV head g and TWO consecutive token blocks (tiles A, B): every 128-token
// K/V page is TMA-loaded once and used by both tiles, which halves L2->SM traffic
// per FLOP (the per-SM L2 read budget, not the tensor pipe, bounded the one-tile
// design).
//
//   warps 0-7  softmax of tile A, warps 8-15 softmax of tile B; per tile, the two
//              warps on a TMEM lane quarter split the 128 key columns: pass 1
//              reads the whole S row for the max, pass 2 exponentiates the warp's
//              64 keys in the log2 domain (1/8 of them with a degree-3 polynomial
//              on the FMA pipe to offload MUFU) and writes P (fp16) back into the
//              first 64 TMEM columns of its S buffer (A operand of the PV MMA);
//              O is rescaled in TMEM only when the max grows by > 2^8
//   warp 16    TMA producer: K and V pages, 2-stage ring
//   warp 17    TMEM owner + MMA issuer, pipe order per page j:
//              PV_A(j), S_A(j+1), PV_B(j), S_B(j+1)
// TMEM: S_A [0,128) S_B [128,256) O_A [256,256+DKP) O_B [384,384+DKP).
#include <mutex>
#include <type_traits>
#include "kernels.cuh"
#include "gemm_tc.cuh"

namespace pkv {

struct AttnArgs {
  const __half* q;           // [n_q][H][DKP] fp16
  __half* out;               // [n_q][H][DKP] fp16
  const int32_t* pos;        // [n_q] ascending
  const int32_t* page_table; // logical page -> physical page
  int n_q, H, Hkv, G, T, n_tiles, n_pairs;
  int hg;                    // KV heads per scheduling group (divides Hkv), see below
  long kv_row0;              // first pool row of this layer: layer * Hkv * pool_tokens
  long pool_tokens;
  float scale_log2;          // log2(e) / sqrt(head_dim)
  unsigned long long* trace; // debug (PKV_ATTN_TRACE=1): %globaltimer per page of CTA 0, see below
  unsigned long long* cta_trace;  // debug (PKV_ATTN_CTA_TRACE=1): per CTA {start, end, smid, pages}
  int* ticket;                    // attn_ps_kernel: next work unit (zeroed before the launch)
};

// trace[ev * 64 + j] for page j < 64 of blockIdx.x == 0 (tools/attn_trace.py):
//   ev 0/1: tile A/B softmax saw S(j) (warp 0 / 8, lane 0)   ev 2/3: A/B arrived P(j)
//   ev 4/5: MMA warp issued PV_A(j) / PV_B(j)                ev 6: MMA warp saw K/V page j+1
//   ev 7: producer issued the K/V loads of page j
// Measured (C3 shape, tools/attn_trace.py + tools/bench_attn.py): a page takes ~1.7 us;
// each softmax ~0.87 us; the MMA warp waits ~0.32 us per page for K/V(j+1) and S(j+1)
// reaches the softmax ~0.2 us after its MMA.  A 64 KB page load takes ~0.9 us; issued
// earlier (separate K / V rings, K(j+2) right after S_B(j+1)) it took ~2.3 us instead --
// the SM's K/V stream is throughput-bound (~40 GB/s per SM with all SMs streaming), not
// latency-bound (1.40 vs 1.36 ms).  Diagnostics: no exponentials -4.5 %, no half-row max
// exchange -3 %, no V loads -8 %: no single stage dominates the S -> softmax -> PV chain.
__device__ __forceinline__ void attn_stamp(const AttnArgs& a, int ev, int j) {
  if (a.trace != nullptr && blockIdx.x == 0 && j < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[ev * 64 + j] = t;
  }
}

template <int DKP>
struct AttnCfg {
  static constexpr int ATOMS = DKP / 64;
  static constexpr int Q_BYTES = 128 * DKP * 2;   // one Q tile
  static constexpr int KV_BYTES = 128 * DKP * 2;  // one K or V page
  static constexpr int STAGES = 2;
  static constexpr int SMEM = 2 * Q_BYTES + STAGES * 2 * KV_BYTES + 1024 + 256 + 4096;  // + max exchange
};

// packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f32x2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f32x2_unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x without the XU pipe (MUFU.EX2, FRND and F2I all issue there; with every
// exponential on MUFU the XU pipe, not the tensor pipe, bounds this kernel):
// round-to-nearest via the 1.5*2^23 magic add (FADD), degree-3 minimax polynomial
// for 2^f on [-0.5, 0.5] (max relative error 7.5e-5; P is rounded to fp16, 2^-11, afterwards),
// exponent added as an integer taken from the magic sum's low mantissa bits.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517606f, f, 0.24261151f), f, 0.69326018f), f, 0.99992803f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void unpack_f16x2(uint32_t v, float& lo, float& hi) {
  asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
      : "=f"(lo), "=f"(hi) : "r"(v));
}

// POLY of every 8 exponentials go to the FMA-pipe polynomial, the rest to MUFU.EX2;
// POLY < 0: packed half-precision MUFU.EX2 (two exponentials per op)
// PAIR = 1: CTA pairs (cluster of 2, tcgen05 cta_group::2).  The pair's CTAs take two
// adjacent query-pair blocks of the same KV head; every MMA is M = 256 (both CTAs' tiles)
// and its B operand is split along N across the pair -- each CTA loads 64 of a page's
// 128 keys of K and 64 of the 128 dims of V -- so per SM the K/V stream halves (it bounds
// the page loop: ~40 GB/s per SM with every SM streaming) and the ring gets 4 stages.
// tmK is then a 64-row-box map.  Only the leader's MMA warp issues.  Opt-in
// (PKV_ATTN_PAIR=1): correct, and the K/V wait disappears, but every PV now waits for the
// other CTA's softmax through a remote mbarrier arrive (~0.35 us on the critical chain),
// so a page takes ~2.08 instead of ~1.70 us (1.59 vs 1.40 ms for the C3 layer).
template <int DKP, int POLY, int PAIR = 0>
__global__ void __launch_bounds__(576, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  using Cfg = AttnCfg<DKP>;
  static_assert(!PAIR || DKP == 128, "CTA-pair attention for head dim 128");
  constexpr int NST = PAIR ? 2 * Cfg::STAGES : Cfg::STAGES;    // K/V ring stages
  constexpr int KVB = PAIR ? Cfg::KV_BYTES / 2 : Cfg::KV_BYTES;  // this CTA's K (or V) bytes per page
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // tile A at +0, tile B at +Q_BYTES
  uint8_t* sKV = sQ + 2 * Cfg::Q_BYTES;    // stage s: K at sKV + s*2*KV_BYTES, V right after
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NST * 2 * KVB);
  uint64_t* kv_full = bars;                 // [NST]
  uint64_t* kv_empty = bars + NST;          // [NST]
  uint64_t* s_full = bars + 2 * NST;          // [2] per tile
  uint64_t* p_full = s_full + 2;              // [2]
  uint64_t* pv_full = p_full + 2;             // [2]
  uint64_t* q_full = pv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA order: KV-head groups of hg heads one after the other, inside a group heaviest
  // pairs first (LPT).  All heads at once keep every head's K/V pages live -- 134 MB per
  // layer at 32k, more than L2 -- while a group's K/V fits and is re-read from L2.
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int n_units = PAIR ? (a.n_pairs + 1) >> 1 : a.n_pairs;  // query-pair blocks (pairs of them)
  const int per_group = a.hg * n_units;
  const int grp = cid / per_group, rem_ = cid - grp * per_group;
  const int g = grp * a.hg + rem_ % a.hg;
  const int unit = rem_ / a.hg;  // 0 = heaviest
  const int pair = PAIR ? a.n_pairs - 1 - (2 * unit + (int)rank) : a.n_pairs - 1 - unit;  // < 0: no rows
  const int lead_pair = PAIR ? a.n_pairs - 1 - 2 * unit : pair;  // sets the pages both CTAs walk

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8 * (PAIR + 1));
      mbar_init(&pv_full[i], 1);
    }
    mbar_init(q_full, 16 * (PAIR + 1));
    fence_barrier_init();
  }
  if constexpr (PAIR) {
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive / TMA
    if (warp == 17) tmem_alloc_cg2(tmem_slot, 512);
  } else {
    if (warp == 17) tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: q / the scattered K/V come from the previous kernel
  griddep_launch();
  // last valid token of the pair decides how many KV pages the CTA walks
  const int last_tok = min((2 * lead_pair + 2) * a.T, a.n_q) - 1;
  const int n_kv_tiles = a.pos[last_tok] / 128 + 1;
  if (a.cta_trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    uint32_t sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.cta_trace[blockIdx.x * 4 + 0] = t;
    a.cta_trace[blockIdx.x * 4 + 2] = sm;
    a.cta_trace[blockIdx.x * 4 + 3] = (unsigned long long)n_kv_tiles;
  }

  if (warp == 16) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_kv_tiles; ++j) {
        const int st = j % NST;
        const uint32_t ph = (uint32_t)(j / NST) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        attn_stamp(a, 7, j);
        uint8_t* sk = sKV + st * 2 * KVB;
        uint8_t* sv = sk + KVB;
        const int row = (int)(head_row + (long)a.page_table[j] * 128);
        if constexpr (PAIR) {
          // keys [64 rank, +64) of K (2 atoms of 64 rows), dims [64 rank, +64) of V; all
          // four halves land on the leader's barrier (only its MMA waits)
          if (rank == 0) mbar_expect_tx(&kv_full[st], 4 * KVB);
          tma_load_2d_cg2(sk, &tmK, &kv_full[st], 0, row + (int)rank * 64);
          tma_load_2d_cg2(sk + 8192, &tmK, &kv_full[st], 64, row + (int)rank * 64);
          tma_load_2d_cg2(sv, &tmV, &kv_full[st], (int)rank * 64, row);
        } else {
          mbar_expect_tx(&kv_full[st], 2 * Cfg::KV_BYTES);
#pragma unroll
          for (int at = 0; at < Cfg::ATOMS; ++at) {
            tma_load_2d(sk + at * 16384, &tmK, &kv_full[st], at * 64, row);
            tma_load_2d(sv + at * 16384, &tmV, &kv_full[st], at * 64, row);
          }
        }
      }
    }
  } else if (warp == 17) {
   if (!PAIR || rank == 0) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_f16(128 * (PAIR + 1), 128);
    constexpr uint32_t idesc_o = make_idesc_f16(128 * (PAIR + 1), DKP, /*b_mn_major=*/true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR) umma_commit_cg2(bar);  // arrives in both CTAs
      else umma_commit(bar);
    };
    auto issue_s = [&](int t, int j) {  // S_t(j) = Q_t K_j^T
      const int st = j % NST;
      const uint32_t k_addr = smem_u32(sKV + st * 2 * KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * (PAIR ? 8192 : 16384) + (kk & 3) * 32;
          if constexpr (PAIR)
            umma_ss_cg2(tmem + t * 128, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                          sdesc_sw128(k_addr + koff, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
          else
            umma_ss(tmem + t * 128, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                      sdesc_sw128(k_addr + koff, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        commit(&s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j, P from TMEM
      const int st = j % NST;
      const uint32_t v_addr = smem_u32(sKV + st * 2 * KVB + KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if constexpr (PAIR)
            umma_ts_cg2(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                             sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          else
            umma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                         sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        commit(&pv_full[t]);
      }
      __syncwarp();
    };
    mbar_wait(&kv_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < n_kv_tiles; ++j) {
      const bool more = j + 1 < n_kv_tiles;
      mbar_wait(&p_full[0], (uint32_t)j & 1);
      tc_fence_after();
      if (lane == 0) attn_stamp(a, 4, j);
      issue_pv(0, j);
      if (more) {
        mbar_wait(&kv_full[(j + 1) % NST], (uint32_t)((j + 1) / NST) & 1);
        tc_fence_after();
        if (lane == 0) attn_stamp(a, 6, j);
        issue_s(0, j + 1);  // in-order after PV_A(j): P_A's TMEM columns are free again
      }
      mbar_wait(&p_full[1], (uint32_t)j & 1);
      tc_fence_after();
      if (lane == 0) attn_stamp(a, 5, j);
      issue_pv(1, j);
      if (elect_one()) commit(&kv_empty[j % NST]);
      __syncwarp();
      if (more) issue_s(1, j + 1);
    }
   }
  } else {
    // ---------------------------------------------------------------- softmax
    // warp w: tile t = w/8, TMEM lane quarter w%4, key-column half h = (w/4)%2
    const int t = warp >> 3;
    const int quarter = warp & 3;
    const int h = (warp >> 2) & 1;
    const int r = quarter * 32 + lane;  // 0..127 == TMEM lane
    const int bar_id = 1 + t * 4 + quarter;  // the two column halves of these 32 rows
    const int b = 2 * pair + t;
    const bool has_tile = pair >= 0 && b < a.n_tiles;  // (a pair CTA may have no rows)
    const int hj = r / a.T;
    const int ti = r - hj * a.T;
    const int tok = b * a.T + ti;
    const bool valid = has_tile && hj < a.G && tok < a.n_q;
    const int head = g * a.G + hj;
    const int tile_last = min((b + 1) * a.T, a.n_q) - 1;
    const int min_pos = has_tile ? a.pos[b * a.T] : 0x7fffffff;
    const int my_pos = valid ? a.pos[tok] : (has_tile ? a.pos[tile_last] : 0x7fffffff);
    const uint32_t lb = (uint32_t)((quarter * 32) << 16);
    const uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
    const float sl2 = a.scale_log2;

    if (h < Cfg::ATOMS) {  // Q row, this warp's 64-column atom -> smem (128B-swizzled K-major)
      uint4 v[8];
      const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) + h * 8;
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = valid ? src[c] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int ch = c ^ (r & 7);
        *reinterpret_cast<uint4*>(sQ + t * Cfg::Q_BYTES + h * 16384 + r * 128 + ch * 16) = v[c];
      }
      fence_proxy_async_smem();
    }
    __syncwarp();
    if (lane == 0) {
      if (PAIR && rank != 0) mbar_arrive_cluster(q_full, 0);  // the leader's MMA waits
      else mbar_arrive(q_full);
    }

    float m_run = -INFINITY, l_run = 0.f;  // m in log2 units; l: this half's row sum
    float* red = reinterpret_cast<float*>(sKV + Cfg::STAGES * 2 * Cfg::KV_BYTES + 256);  // [2][2 tiles][2][128]
    for (int j = 0; j < n_kv_tiles; ++j) {
      mbar_wait(&s_full[t], (uint32_t)j & 1);  // also implies PV_t(j-1) is complete
      tc_fence_after();
      if ((warp & 7) == 0 && lane == 0) attn_stamp(a, t, j);
      const int key0 = j * 128 + h * 64;
      // pass 1: this half's 64 scores -> registers (masked -> -inf only on diagonal pages)
      float sv[64];
      {
        uint32_t u[32], w[32];
        tmem_ld32(tS + lb + h * 64, u);
        tmem_ld32(tS + lb + h * 64 + 32, w);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          sv[i] = __uint_as_float(u[i]);
          sv[32 + i] = __uint_as_float(w[i]);
        }
      }
      if (key0 + 63 > min_pos) {
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = (key0 + i <= my_pos) ? sv[i] : -INFINITY;
      }
      // 4 independent max chains (a single 32-deep dependent chain is pure latency)
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; i += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(sv[i + 2 * q], sv[i + 2 * q + 1]));
      const float hmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      // exchange the half-row maxima with the partner warp (same rows, other 64 keys)
      float* rb = red + ((j & 1) * 2 + t) * 256;
      rb[h * 128 + r] = hmax;
      named_bar_sync(bar_id, 64);  // both halves have their S in registers from here on
      const float tmax = fmaxf(hmax, rb[(h ^ 1) * 128 + r]);
      const float m_new = fmaxf(m_run, tmax * sl2);
      const bool grow = (m_new - m_run) > 8.0f;  // also true on the first tile (m_run = -inf)
      const float m_use = grow ? m_new : m_run;
      // pass 2: P = 2^(s*sl2 - m) with packed f32x2 FMA/ADD; 1/4 of the exponentials on
      // the FMA pipe.  P of keys [64h, 64h+64) -> TMEM columns [32h, 32h+32) of the S
      // buffer (safe: the partner's S is in its registers since the barrier)
      const uint64_t sl2x2 = f32x2(sl2, sl2), negm = f32x2(-m_use, -m_use);
      uint64_t rsum2 = f32x2(0.f, 0.f), rsum2b = f32x2(0.f, 0.f);  // two sum chains
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = ffma2(f32x2(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]), sl2x2, negm);
          float x0, x1;
          f32x2_unpack(x, x0, x1);
          float p0, p1;
          constexpr uint32_t kPolyMask = POLY >= 4 ? 0xAAu : POLY == 3 ? 0x94u : POLY == 2 ? 0x88u : POLY == 1 ? 0x80u : 0u;
          if constexpr (POLY < 0) {
            // two exponentials per MUFU op (ex2.approx.f16x2): the argument is rounded to
            // f16 (|x| < 1: 2^-11 relative; larger |x| only for P < 2^-4) and P is rounded
            // to fp16 for the MMA anyway
            const uint32_t hx = pack_f16x2(x0, x1);
            uint32_t hp;
            asm("ex2.approx.f16x2 %0, %1;" : "=r"(hp) : "r"(hx));
            unpack_f16x2(hp, p0, p1);
          } else if ((kPolyMask >> (i & 7)) & 1u) {
            p0 = exp2_poly(x0);
            p1 = exp2_poly(x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          if (i & 1) rsum2b = fadd2(rsum2b, f32x2(p0, p1));
          else rsum2 = fadd2(rsum2, f32x2(p0, p1));
          pk[i] = pack_f16(p0, p1);
        }
        tmem_st16(tS + lb + h * 32 + c * 16, pk);
      }
      float rs0, rs1;
      f32x2_unpack(fadd2(rsum2, rsum2b), rs0, rs1);
      const float rsum = rs0 + rs1;
      if (__any_sync(0xffffffffu, grow && j > 0)) {
        const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
        for (int c = h * DKP / 64; c < (h + 1) * DKP / 64; ++c) {
          uint32_t u[32];
          tmem_ld32(tO + lb + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st32(tO + lb + c * 32, u);
        }
      }
      if (grow && j > 0) l_run *= ex2(m_run - m_use);
      if (grow) m_run = m_use;
      l_run += rsum;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && rank != 0) mbar_arrive_cluster(&p_full[t], 0);  // remote: the leader's MMA waits
        else mbar_arrive(&p_full[t]);
      }
      if ((warp & 7) == 0 && lane == 0) attn_stamp(a, 2 + t, j);
    }
    mbar_wait(&pv_full[t], (uint32_t)(n_kv_tiles - 1) & 1);
    tc_fence_after();
    // row sum = both halves; every MMA has completed, so the Q tile is free scratch
    float* lred = reinterpret_cast<float*>(sQ + t * Cfg::Q_BYTES);
    lred[h * 128 + r] = l_run;
    named_bar_sync(bar_id, 64);
    const float inv_l = 1.f / (lred[r] + lred[128 + r]);
#pragma unroll 1
    for (int c = h * DKP / 64; c < (h + 1) * DKP / 64; ++c) {
      uint32_t u[32];
      tmem_ld32(tO + lb + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_f16(__uint_as_float(u[8 * i]) * inv_l, __uint_as_float(u[8 * i + 1]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 2]) * inv_l, __uint_as_float(u[8 * i + 3]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 4]) * inv_l, __uint_as_float(u[8 * i + 5]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 6]) * inv_l, __uint_as_float(u[8 * i + 7]) * inv_l));
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (a.cta_trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.cta_trace[blockIdx.x * 4 + 1] = t;
  }
  if constexpr (PAIR) cluster_sync();  // no TMEM use or remote arrive left in either CTA
  if (warp == 17) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_cg2(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}


// Three key-column slices per TMEM lane quarter (48 + 48 + 32 keys of each 128-key page):
// 24 softmax warps + TMA + MMA = 832 threads.  The page loop of a tile is a chain
// softmax(j) -> PV(j), S(j+1) -> softmax(j+1); spreading the softmax of a page over three
// warps per 32 rows (instead of two) shortens that chain.  Each slice writes its P into
// its OWN S columns (cols [48c, 48c + W/2)), so the PV MMA reads P at slice offsets.
// DKP = 128 only (O columns split 48/48/32 the same way).
template <int POLY>
__global__ void __launch_bounds__(832, 1)
    attn_tc3_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  constexpr int DKP = 128;
  using Cfg = AttnCfg<DKP>;
  constexpr int TMA_WARP = 24, MMA_WARP = 25;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + 2 * Cfg::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + Cfg::STAGES * 2 * Cfg::KV_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + Cfg::STAGES;
  uint64_t* s_full = bars + 2 * Cfg::STAGES;
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_full = p_full + 2;
  uint64_t* q_full = pv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA order: KV-head groups of hg heads one after the other, inside a group heaviest
  // pairs first (LPT).  All heads at once keep every head's K/V pages live -- 134 MB per
  // layer at 32k, more than L2 -- while a group's K/V fits and is re-read from L2.
  const int per_group = a.hg * a.n_pairs;
  const int grp = blockIdx.x / per_group, rem_ = blockIdx.x - grp * per_group;
  const int g = grp * a.hg + rem_ % a.hg;
  const int pair = a.n_pairs - 1 - rem_ / a.hg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 12);
      mbar_init(&pv_full[i], 1);
    }
    mbar_init(q_full, 24);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();
  griddep_launch();
  const int last_tok = min((2 * pair + 2) * a.T, a.n_q) - 1;
  const int n_kv_tiles = a.pos[last_tok] / 128 + 1;

  if (warp == TMA_WARP) {
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_kv_tiles; ++j) {
        const int st = j % Cfg::STAGES;
        mbar_wait(&kv_empty[st], ((uint32_t)(j / Cfg::STAGES) & 1) ^ 1);
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
  } else if (warp == MMA_WARP) {
    constexpr uint32_t idesc_s = make_idesc_f16(128, 128);
    constexpr uint32_t idesc_o = make_idesc_f16(128, DKP, /*b_mn_major=*/true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    auto issue_s = [&](int t, int j) {
      const uint32_t k_addr = smem_u32(sKV + (j % Cfg::STAGES) * 2 * Cfg::KV_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + t * 128, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                    sdesc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {  // P of keys 16kk.. sits in its slice's S columns
      const uint32_t v_addr = smem_u32(sKV + (j % Cfg::STAGES) * 2 * Cfg::KV_BYTES + Cfg::KV_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t pcol = kk < 3 ? kk * 8 : (kk < 6 ? 48 + (kk - 3) * 8 : 96 + (kk - 6) * 8);
          umma_ts(tmem + 256 + t * 128, tmem + t * 128 + pcol,
                       sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&pv_full[t]);
      }
      __syncwarp();
    };
    mbar_wait(&kv_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < n_kv_tiles; ++j) {
      const bool more = j + 1 < n_kv_tiles;
      mbar_wait(&p_full[0], (uint32_t)j & 1);
      tc_fence_after();
      issue_pv(0, j);
      if (more) {
        mbar_wait(&kv_full[(j + 1) % Cfg::STAGES], (uint32_t)((j + 1) / Cfg::STAGES) & 1);
        tc_fence_after();
        issue_s(0, j + 1);
      }
      mbar_wait(&p_full[1], (uint32_t)j & 1);
      tc_fence_after();
      issue_pv(1, j);
      if (elect_one()) umma_commit(&kv_empty[j % Cfg::STAGES]);
      __syncwarp();
      if (more) issue_s(1, j + 1);
    }
  } else {
    const int t = warp / 12;
    const int idx = warp - t * 12;
    const int quarter = idx & 3;  // == warp % 4 (TMEM lane quarter rule)
    const int c3 = idx >> 2;      // key-column slice 0..2
    const int col0 = c3 * 48;
    const int r = quarter * 32 + lane;
    const int bar_id = 1 + t * 4 + quarter;  // the three slices of these 32 rows
    const int b = 2 * pair + t;
    const int hj = r / a.T;
    const int ti = r - hj * a.T;
    const int tok = b * a.T + ti;
    const bool valid = hj < a.G && tok < a.n_q && b < a.n_tiles;
    const int head = g * a.G + hj;
    const int tile_last = min((b + 1) * a.T, a.n_q) - 1;
    const int min_pos = b < a.n_tiles ? a.pos[b * a.T] : 0x7fffffff;
    const int my_pos = valid ? a.pos[tok] : (b < a.n_tiles ? a.pos[tile_last] : 0x7fffffff);
    const uint32_t lb = (uint32_t)((quarter * 32) << 16);
    const uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
    const float sl2 = a.scale_log2;

    if (c3 < Cfg::ATOMS) {  // Q row atom c3 -> smem (128B-swizzled K-major)
      uint4 v[8];
      const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) + c3 * 8;
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = valid ? src[c] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int ch = c ^ (r & 7);
        *reinterpret_cast<uint4*>(sQ + t * Cfg::Q_BYTES + c3 * 16384 + r * 128 + ch * 16) = v[c];
      }
      fence_proxy_async_smem();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(q_full);

    float m_run = -INFINITY, l_run = 0.f;
    float* red = reinterpret_cast<float*>(sKV + Cfg::STAGES * 2 * Cfg::KV_BYTES + 256);  // [2][2 tiles][3][128]

    auto page = [&](int j, auto WC) {
      constexpr int W = decltype(WC)::value;  // keys of this slice
      const int key0 = j * 128 + col0;
      float sv[W];
      {
        uint32_t u[W];
#pragma unroll
        for (int c = 0; c < W / 16; ++c) tmem_ld16(tS + lb + col0 + c * 16, u + c * 16);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < W; ++i) sv[i] = __uint_as_float(u[i]);
      }
      if (key0 + W - 1 > min_pos) {
#pragma unroll
        for (int i = 0; i < W; ++i) sv[i] = (key0 + i <= my_pos) ? sv[i] : -INFINITY;
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < W; i += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(sv[i + 2 * q], sv[i + 2 * q + 1]));
      const float hmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      float* rb = red + ((j & 1) * 2 + t) * 384;
      rb[c3 * 128 + r] = hmax;
      named_bar_sync(bar_id, 96);
      const float tmax = fmaxf(fmaxf(rb[r], rb[128 + r]), rb[256 + r]);
      const float m_new = fmaxf(m_run, tmax * sl2);
      const bool grow = (m_new - m_run) > 8.0f;
      const float m_use = grow ? m_new : m_run;
      const uint64_t sl2x2 = f32x2(sl2, sl2), negm = f32x2(-m_use, -m_use);
      uint64_t rsum2 = f32x2(0.f, 0.f), rsum2b = f32x2(0.f, 0.f);
      uint32_t pk[W / 2];
#pragma unroll
      for (int i = 0; i < W / 2; ++i) {
        const uint64_t x = ffma2(f32x2(sv[2 * i], sv[2 * i + 1]), sl2x2, negm);
        float x0, x1;
        f32x2_unpack(x, x0, x1);
        float p0, p1;
        constexpr uint32_t kPolyMask = POLY >= 4 ? 0xAAu : POLY == 3 ? 0x94u : POLY == 2 ? 0x88u : POLY == 1 ? 0x80u : 0u;
        if ((kPolyMask >> (i & 7)) & 1u) {
          p0 = exp2_poly(x0);
          p1 = exp2_poly(x1);
        } else {
          p0 = ex2(x0);
          p1 = ex2(x1);
        }
        if (i & 1) rsum2b = fadd2(rsum2b, f32x2(p0, p1));
        else rsum2 = fadd2(rsum2, f32x2(p0, p1));
        pk[i] = pack_f16(p0, p1);
      }
      // P of this slice -> its own S columns [col0, col0 + W/2) (no other slice reads them)
      tmem_st16p(tS + lb + col0, pk);
      if constexpr (W / 2 > 16) tmem_st8(tS + lb + col0 + 16, pk + 16);
      float rs0, rs1;
      f32x2_unpack(fadd2(rsum2, rsum2b), rs0, rs1);
      if (__any_sync(0xffffffffu, grow && j > 0)) {
        const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
        for (int c = 0; c < W / 16; ++c) {
          uint32_t u[16];
          tmem_ld16(tO + lb + col0 + c * 16, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st16p(tO + lb + col0 + c * 16, u);
        }
      }
      if (grow && j > 0) l_run *= ex2(m_run - m_use);
      if (grow) m_run = m_use;
      l_run += rs0 + rs1;
    };

    for (int j = 0; j < n_kv_tiles; ++j) {
      mbar_wait(&s_full[t], (uint32_t)j & 1);
      tc_fence_after();
      if (c3 < 2) page(j, std::integral_constant<int, 48>{});
      else page(j, std::integral_constant<int, 32>{});
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    mbar_wait(&pv_full[t], (uint32_t)(n_kv_tiles - 1) & 1);
    tc_fence_after();
    float* lred = reinterpret_cast<float*>(sQ + t * Cfg::Q_BYTES);
    lred[c3 * 128 + r] = l_run;
    named_bar_sync(bar_id, 96);
    const float inv_l = 1.f / ((lred[r] + lred[128 + r]) + lred[256 + r]);
    const int W = c3 < 2 ? 48 : 32;
#pragma unroll 1
    for (int c = 0; c < W / 16; ++c) {
      uint32_t u[16];
      tmem_ld16(tO + lb + col0 + c * 16, u);
      tmem_ld_wait();
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + col0 + c * 16);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          dst[i] = make_uint4(pack_f16(__uint_as_float(u[8 * i]) * inv_l, __uint_as_float(u[8 * i + 1]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 2]) * inv_l, __uint_as_float(u[8 * i + 3]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 4]) * inv_l, __uint_as_float(u[8 * i + 5]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 6]) * inv_l, __uint_as_float(u[8 * i + 7]) * inv_l));
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
// One 128-row Q tile per CTA with S double-buffered in TMEM (PKV_ATTN_ONE=1).  The two-tile
// kernel above keeps one S buffer per tile because two tiles' S and O fill all 512 TMEM
// columns, so each tile's page loop is the chain softmax(j) -> PV(j) -> S(j+1) ->
// softmax(j+1) (ncu: the softmax warps wait for S 39 % of the time, tensor pipe 63 %).
// With one tile the columns hold S(j) and S(j+1) [0,256), O [256,384) and two P buffers
// [384,512), so S(j+1) is computed while the softmax of page j runs and the softmax runs
// back to back; the cost is that every CTA streams its own K/V pages (twice the L2 -> SM
// traffic per flop of the two-tile form).
//   warps 0-7  softmax: warp w owns TMEM lane quarter w%4 and keys [64h, 64h+64), h = w/4
//   warp 8     TMA producer (3-stage K/V ring)
//   warp 9     TMEM owner + MMA issuer: S(0), S(1), then per page j: PV(j), S(j+2)
constexpr int ATTN1_NST = 3;
constexpr int ATTN1_NEED = 128 * 128 * 2 /*Q*/ + ATTN1_NST * 2 * 128 * 128 * 2 /*K/V*/ + 2048 /*max exchange*/ +
                           16 * 8 /*barriers*/ + 16;
constexpr int ATTN1_SMEM = 232448;  // the per-block maximum; the kernel checks the aligned fit

template <int POLY>
__global__ void __launch_bounds__(320, 1)
    attn_tc1_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  constexpr int DKP = 128, KVB = 128 * DKP * 2, NST = ATTN1_NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0 && (smem - smem_raw) + ATTN1_NEED > ATTN1_SMEM) __trap();
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + KVB;  // stage s: K at sKV + 2*s*KVB, V right after
  float* red = reinterpret_cast<float*>(sKV + NST * 2 * KVB);  // [2 parity][2 halves][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 512);
  uint64_t* kv_full = bars;         // [NST]
  uint64_t* kv_empty = bars + NST;  // [NST]
  uint64_t* s_full = bars + 2 * NST;  // [2] per S buffer
  uint64_t* s_free = s_full + 2;      // [2]
  uint64_t* p_full = s_free + 2;      // [2] per P buffer
  uint64_t* pv_full = p_full + 2;     // [2]
  uint64_t* q_full = pv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);
  constexpr uint32_t T_O = 256, T_P = 384;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA order: KV-head groups of hg heads, inside a group the heaviest tiles first (LPT)
  const int per_group = a.hg * a.n_tiles;
  const int grp = (int)blockIdx.x / per_group, rem_ = (int)blockIdx.x - grp * per_group;
  const int g = grp * a.hg + rem_ % a.hg;
  const int b = a.n_tiles - 1 - rem_ / a.hg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_full[i], 1);
    }
    mbar_init(q_full, 8);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: q / the scattered K/V come from the previous kernel
  griddep_launch();
  const int tile_last = min((b + 1) * a.T, a.n_q) - 1;
  const int n_kv = a.pos[tile_last] / 128 + 1;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NST;
        mbar_wait(&kv_empty[st], ((uint32_t)(j / NST) & 1) ^ 1);
        uint8_t* sk = sKV + st * 2 * KVB;
        const int row = (int)(head_row + (long)a.page_table[j] * 128);
        mbar_expect_tx(&kv_full[st], 2 * KVB);
#pragma unroll
        for (int at = 0; at < 2; ++at) {
          tma_load_2d(sk + at * 16384, &tmK, &kv_full[st], at * 64, row);
          tma_load_2d(sk + KVB + at * 16384, &tmV, &kv_full[st], at * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_f16(128, 128);
    constexpr uint32_t idesc_o = make_idesc_f16(128, DKP, /*b_mn_major=*/true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    auto issue_s = [&](int j) {  // S(j) = Q K_j^T -> S buffer j % 2
      mbar_wait(&kv_full[j % NST], (uint32_t)(j / NST) & 1);
      tc_fence_after();
      const uint32_t k_addr = smem_u32(sKV + (j % NST) * 2 * KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + (j & 1) * 128, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024),
                  idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    issue_s(0);
    if (n_kv > 1) issue_s(1);
    for (int j = 0; j < n_kv; ++j) {
      const int pb = j & 1;
      mbar_wait(&p_full[pb], (uint32_t)(j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_addr = smem_u32(sKV + (j % NST) * 2 * KVB + KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tmem + T_O, tmem + T_P + pb * 64 + kk * 8, sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024), idesc_o,
                  (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&pv_full[pb]);
        umma_commit(&kv_empty[j % NST]);
      }
      __syncwarp();
      if (j + 2 < n_kv) {
        mbar_wait(&s_free[pb], (uint32_t)(j >> 1) & 1);  // the softmax has S(j) in registers
        issue_s(j + 2);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax
    const int quarter = warp & 3, h = warp >> 2;
    const int r = quarter * 32 + lane;  // TMEM lane == tile row
    const int bar_id = 1 + quarter;     // the two key halves of these 32 rows
    const int hj = r / a.T, ti = r - hj * a.T;
    const int tok = b * a.T + ti;
    const bool valid = hj < a.G && tok < a.n_q;
    const int head = g * a.G + hj;
    const int min_pos = a.pos[b * a.T];
    const int my_pos = valid ? a.pos[tok] : a.pos[tile_last];
    const uint32_t lb = (uint32_t)((quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    {  // Q row, this warp's 64-column atom -> smem (128B-swizzled K-major)
      uint4 v[8];
      const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) + h * 8;
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = valid ? src[c] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int ch = c ^ (r & 7);
        *reinterpret_cast<uint4*>(sQ + h * 16384 + r * 128 + ch * 16) = v[c];
      }
      fence_proxy_async_smem();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(q_full);

    float m_run = -INFINITY, l_run = 0.f;  // m in log2 units; l: this half's row sum
    for (int j = 0; j < n_kv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (uint32_t)(j >> 1) & 1);
      tc_fence_after();
      const int key0 = j * 128 + h * 64;
      float sv[64];
      {
        uint32_t u[32], w[32];
        tmem_ld32(tmem + sb * 128 + lb + h * 64, u);
        tmem_ld32(tmem + sb * 128 + lb + h * 64 + 32, w);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          sv[i] = __uint_as_float(u[i]);
          sv[32 + i] = __uint_as_float(w[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[sb]);  // S(j + 2) may overwrite this buffer
      if (key0 + 63 > min_pos) {
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = (key0 + i <= my_pos) ? sv[i] : -INFINITY;
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; i += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(sv[i + 2 * q], sv[i + 2 * q + 1]));
      const float hmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      float* rb = red + sb * 256;
      rb[h * 128 + r] = hmax;
      named_bar_sync(bar_id, 64);
      const float tmax = fmaxf(hmax, rb[(h ^ 1) * 128 + r]);
      const float m_new = fmaxf(m_run, tmax * sl2);
      const bool grow = (m_new - m_run) > 8.0f;  // also true on the first page (m_run = -inf)
      const float m_use = grow ? m_new : m_run;
      const uint64_t sl2x2 = f32x2(sl2, sl2), negm = f32x2(-m_use, -m_use);
      uint64_t rsum2 = f32x2(0.f, 0.f), rsum2b = f32x2(0.f, 0.f);
      uint32_t pk[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = ffma2(f32x2(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]), sl2x2, negm);
          float x0, x1;
          f32x2_unpack(x, x0, x1);
          float p0, p1;
          constexpr uint32_t kPolyMask = POLY >= 4 ? 0xAAu : POLY == 3 ? 0x94u : POLY == 2 ? 0x88u : POLY == 1 ? 0x80u : 0u;
          if ((kPolyMask >> (i & 7)) & 1u) {
            p0 = exp2_poly(x0);
            p1 = exp2_poly(x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          if (i & 1) rsum2b = fadd2(rsum2b, f32x2(p0, p1));
          else rsum2 = fadd2(rsum2, f32x2(p0, p1));
          pk[c][i] = pack_f16(p0, p1);
        }
      }
      const int pb = j & 1;
      if (j >= 2) {  // PV(j-2) has read this P buffer
        mbar_wait(&pv_full[pb], (uint32_t)((j - 2) >> 1) & 1);
        tc_fence_after();
      }
      tmem_st16(tmem + T_P + pb * 64 + lb + h * 32, pk[0]);
      tmem_st16(tmem + T_P + pb * 64 + lb + h * 32 + 16, pk[1]);
      float rs0, rs1;
      f32x2_unpack(fadd2(rsum2, rsum2b), rs0, rs1);
      const float rsum = rs0 + rs1;
      if (__any_sync(0xffffffffu, grow && j > 0)) {  // O rescale: PV(j-1) must have accumulated
        mbar_wait(&pv_full[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1);
        tc_fence_after();
        const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
        for (int c = h * DKP / 64; c < (h + 1) * DKP / 64; ++c) {
          uint32_t u[32];
          tmem_ld32(tmem + T_O + lb + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st32(tmem + T_O + lb + c * 32, u);
        }
      }
      if (grow && j > 0) l_run *= ex2(m_run - m_use);
      if (grow) m_run = m_use;
      l_run += rsum;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
    }
    mbar_wait(&pv_full[(n_kv - 1) & 1], (uint32_t)((n_kv - 1) >> 1) & 1);
    tc_fence_after();
    // row sum = both halves; every MMA has completed, so the Q tile is free scratch
    float* lred = reinterpret_cast<float*>(sQ);
    lred[h * 128 + r] = l_run;
    named_bar_sync(bar_id, 64);
    const float inv_l = 1.f / (lred[r] + lred[128 + r]);
#pragma unroll 1
    for (int c = h * DKP / 64; c < (h + 1) * DKP / 64; ++c) {
      uint32_t u[32];
      tmem_ld32(tmem + T_O + lb + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_f16(__uint_as_float(u[8 * i]) * inv_l, __uint_as_float(u[8 * i + 1]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 2]) * inv_l, __uint_as_float(u[8 * i + 3]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 4]) * inv_l, __uint_as_float(u[8 * i + 5]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 6]) * inv_l, __uint_as_float(u[8 * i + 7]) * inv_l));
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

static int launch_attn1(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(attn_tc1_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ATTN1_SMEM);
  });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn1 smem attr: %s", cudaGetErrorString(err));
  launch_k(attn_tc1_kernel<1>, a.n_tiles * a.Hkv, 320, ATTN1_SMEM, stream, tk, tv, a);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_tc1_kernel");
  return PKV_OK;
}

// One thread per Q-tile row (PKV_ATTN_ROW=1): the two-tile kernel above with 4 softmax
// warps per tile instead of 8 -- each thread reads its row's 128 scores, takes the max
// in registers (no half-row exchange through shared memory and no named barrier per
// page) and exponentiates all 128 keys; warps 0-3 tile A, 4-7 tile B, 8 TMA, 9 MMA.
template <int POLY>
__global__ void __launch_bounds__(320, 1)
    attn_row_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  constexpr int DKP = 128;
  using Cfg = AttnCfg<DKP>;
  constexpr int NST = Cfg::STAGES, KVB = Cfg::KV_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + 2 * Cfg::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NST * 2 * KVB);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + NST;
  uint64_t* s_full = bars + 2 * NST;  // [2] per tile
  uint64_t* p_full = s_full + 2;      // [2]
  uint64_t* pv_full = p_full + 2;     // [2]
  uint64_t* q_full = pv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cid = (int)blockIdx.x;
  const int per_group = a.hg * a.n_pairs;
  const int grp = cid / per_group, rem_ = cid - grp * per_group;
  const int g = grp * a.hg + rem_ % a.hg;
  const int pair = a.n_pairs - 1 - rem_ / a.hg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_full[i], 1);
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
  const int last_tok = min((2 * pair + 2) * a.T, a.n_q) - 1;
  const int n_kv_tiles = a.pos[last_tok] / 128 + 1;

  if (warp == 8) {
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
      for (int j = 0; j < n_kv_tiles; ++j) {
        const int st = j % NST;
        mbar_wait(&kv_empty[st], ((uint32_t)(j / NST) & 1) ^ 1);
        uint8_t* sk = sKV + st * 2 * KVB;
        uint8_t* sv = sk + KVB;
        const int row = (int)(head_row + (long)a.page_table[j] * 128);
        mbar_expect_tx(&kv_full[st], 2 * KVB);
#pragma unroll
        for (int at = 0; at < Cfg::ATOMS; ++at) {
          tma_load_2d(sk + at * 16384, &tmK, &kv_full[st], at * 64, row);
          tma_load_2d(sv + at * 16384, &tmV, &kv_full[st], at * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idesc_s = make_idesc_f16(128, 128);
    constexpr uint32_t idesc_o = make_idesc_f16(128, DKP, /*b_mn_major=*/true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    auto issue_s = [&](int t, int j) {
      const uint32_t k_addr = smem_u32(sKV + (j % NST) * 2 * KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + t * 128, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                  sdesc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {
      const uint32_t v_addr = smem_u32(sKV + (j % NST) * 2 * KVB + KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024),
                  idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&pv_full[t]);
      }
      __syncwarp();
    };
    mbar_wait(&kv_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < n_kv_tiles; ++j) {
      const bool more = j + 1 < n_kv_tiles;
      mbar_wait(&p_full[0], (uint32_t)j & 1);
      tc_fence_after();
      issue_pv(0, j);
      if (more) {
        mbar_wait(&kv_full[(j + 1) % NST], (uint32_t)((j + 1) / NST) & 1);
        tc_fence_after();
        issue_s(0, j + 1);
      }
      mbar_wait(&p_full[1], (uint32_t)j & 1);
      tc_fence_after();
      issue_pv(1, j);
      if (elect_one()) umma_commit(&kv_empty[j % NST]);
      __syncwarp();
      if (more) issue_s(1, j + 1);
    }
  } else {
    const int t = warp >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int b = 2 * pair + t;
    const bool has_tile = pair >= 0 && b < a.n_tiles;
    const int hj = r / a.T, ti = r - hj * a.T;
    const int tok = b * a.T + ti;
    const bool valid = has_tile && hj < a.G && tok < a.n_q;
    const int head = g * a.G + hj;
    const int tile_last = min((b + 1) * a.T, a.n_q) - 1;
    const int min_pos = has_tile ? a.pos[b * a.T] : 0x7fffffff;
    const int my_pos = valid ? a.pos[tok] : (has_tile ? a.pos[tile_last] : 0x7fffffff);
    const uint32_t lb = (uint32_t)((quarter * 32) << 16);
    const uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
    const float sl2 = a.scale_log2;
#pragma unroll 1
    for (int h = 0; h < Cfg::ATOMS; ++h) {  // this row's Q -> smem (both 64-column atoms)
      uint4 v[8];
      const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) + h * 8;
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = valid ? src[c] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sQ + t * Cfg::Q_BYTES + h * 16384 + r * 128 + ((c ^ (r & 7)) * 16)) = v[c];
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(q_full);

    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_kv_tiles; ++j) {
      mbar_wait(&s_full[t], (uint32_t)j & 1);  // also implies PV_t(j-1) is complete
      tc_fence_after();
      const int key0 = j * 128;
      float sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t u[32];
        tmem_ld32(tS + lb + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(u[i]);
      }
      if (key0 + 127 > min_pos) {
#pragma unroll
        for (int i = 0; i < 128; ++i) sv[i] = (key0 + i <= my_pos) ? sv[i] : -INFINITY;
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 128; i += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(sv[i + 2 * q], sv[i + 2 * q + 1]));
      const float tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      const float m_new = fmaxf(m_run, tmax * sl2);
      const bool grow = (m_new - m_run) > 8.0f;
      const float m_use = grow ? m_new : m_run;
      const uint64_t sl2x2 = f32x2(sl2, sl2), negm = f32x2(-m_use, -m_use);
      uint64_t rsum2 = f32x2(0.f, 0.f), rsum2b = f32x2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = ffma2(f32x2(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]), sl2x2, negm);
          float x0, x1;
          f32x2_unpack(x, x0, x1);
          float p0, p1;
          constexpr uint32_t kPolyMask = POLY >= 4 ? 0xAAu : POLY == 3 ? 0x94u : POLY == 2 ? 0x88u : POLY == 1 ? 0x80u : 0u;
          if ((kPolyMask >> (i & 7)) & 1u) {
            p0 = exp2_poly(x0);
            p1 = exp2_poly(x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          if (i & 1) rsum2b = fadd2(rsum2b, f32x2(p0, p1));
          else rsum2 = fadd2(rsum2, f32x2(p0, p1));
          pk[i] = pack_f16(p0, p1);
        }
        tmem_st16(tS + lb + c * 16, pk);  // P of keys [32c, 32c+32): the S columns are in registers
      }
      float rs0, rs1;
      f32x2_unpack(fadd2(rsum2, rsum2b), rs0, rs1);
      if (__any_sync(0xffffffffu, grow && j > 0)) {
        const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
        for (int c = 0; c < DKP / 32; ++c) {
          uint32_t u[32];
          tmem_ld32(tO + lb + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st32(tO + lb + c * 32, u);
        }
      }
      if (grow && j > 0) l_run *= ex2(m_run - m_use);
      if (grow) m_run = m_use;
      l_run += rs0 + rs1;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    mbar_wait(&pv_full[t], (uint32_t)(n_kv_tiles - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l_run;
#pragma unroll 1
    for (int c = 0; c < DKP / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tO + lb + c * 32, u);
      tmem_ld_wait();
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_f16(__uint_as_float(u[8 * i]) * inv_l, __uint_as_float(u[8 * i + 1]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 2]) * inv_l, __uint_as_float(u[8 * i + 3]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 4]) * inv_l, __uint_as_float(u[8 * i + 5]) * inv_l),
                              pack_f16(__uint_as_float(u[8 * i + 6]) * inv_l, __uint_as_float(u[8 * i + 7]) * inv_l));
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

// Persistent form of attn_row_kernel (PKV_ATTN_PERSIST=1): one CTA per SM walks its share of
// the work units (KV head, pair of 32-token blocks) -- zigzag over the LPT-ordered list --
// instead of one CTA per unit.  The per-CTA timeline (tools/attn_cta_trace.py) had put
// ~11.5 us of fixed cost on every unit (barrier init, TMEM alloc, Q tiles, the first K/V
// pages, the output) plus ~3.7 us between consecutive CTAs of an SM; persistent, the K/V
// ring keeps streaming across units (the next unit's first pages arrive while this one
// drains) and only the Q load and the output remain per unit.  Barrier phases run on
// the CTA-global page count (every tile walks every page of its unit).
// Units are handed out dynamically in LPT order (a global ticket, as the hardware scheduler
// does for one CTA per unit): the producer warp takes the next ticket when it reaches the
// unit and publishes it through a 4-slot ring in shared memory to the MMA and softmax warps.
constexpr int ATTN_PS_RING = 4;

template <int POLY, int SPLIT>
__global__ void __launch_bounds__(320, 1)
    attn_ps_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  constexpr int DKP = 128;
  using Cfg = AttnCfg<DKP>;
  constexpr int NST = Cfg::STAGES, KVB = Cfg::KV_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + 2 * Cfg::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NST * 2 * KVB);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + NST;
  uint64_t* s_full = bars + 2 * NST;  // [2] per tile
  uint64_t* p_full = s_full + 2;      // [2]
  uint64_t* pv_full = p_full + 2;     // [2]
  uint64_t* q_full = pv_full + 2;
  uint64_t* u_full = q_full + 1;              // [RING] unit ticket published
  uint64_t* u_empty = u_full + ATTN_PS_RING;  // [RING] read by the MMA warp and the 8 softmax warps
  uint64_t* s_free = u_empty + ATTN_PS_RING;  // [2] SPLIT: the tile's S(j) is in the softmax's registers
  int* u_ids = reinterpret_cast<int*>(s_free + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u_ids + ATTN_PS_RING);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_units = a.n_pairs * a.Hkv;
  // the k-th unit of this CTA (consumers: wait for the producer's ticket, release the slot)
  auto take_unit = [&](int k) -> int {
    const int slot = k % ATTN_PS_RING;
    mbar_wait(&u_full[slot], (uint32_t)(k / ATTN_PS_RING) & 1);
    const int u = *reinterpret_cast<volatile int*>(&u_ids[slot]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&u_empty[slot]);
    return u;
  };
  const int per_group = a.hg * a.n_pairs;
  auto unit_of = [&](int u, int& g, int& pair, int& n_kv) {
    const int grp = u / per_group, rem_ = u - grp * per_group;
    g = grp * a.hg + rem_ % a.hg;
    pair = a.n_pairs - 1 - rem_ / a.hg;
    n_kv = a.pos[min((2 * pair + 2) * a.T, a.n_q) - 1] / 128 + 1;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(q_full, 8);
    for (int i = 0; i < ATTN_PS_RING; ++i) {
      mbar_init(&u_full[i], 1);
      mbar_init(&u_empty[i], 9);
    }
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
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      int jg = 0;  // pages loaded by this CTA so far
      for (int k = 0;; ++k) {
        const int slot = k % ATTN_PS_RING;
        mbar_wait(&u_empty[slot], ((uint32_t)(k / ATTN_PS_RING) & 1) ^ 1);
        const int u = atomicAdd(a.ticket, 1);
        *reinterpret_cast<volatile int*>(&u_ids[slot]) = u;
        mbar_arrive(&u_full[slot]);  // (release: the ticket is visible to the waiting warps)
        if (u >= n_units) break;
        int g, pair, n_kv;
        unit_of(u, g, pair, n_kv);
        const long head_row = a.kv_row0 + (long)g * a.pool_tokens;
        for (int j = 0; j < n_kv; ++j, ++jg) {
          const int st = jg % NST;
          mbar_wait(&kv_empty[st], ((uint32_t)(jg / NST) & 1) ^ 1);
          uint8_t* sk = sKV + st * 2 * KVB;
          const int row = (int)(head_row + (long)a.page_table[j] * 128);
          mbar_expect_tx(&kv_full[st], 2 * KVB);
#pragma unroll
          for (int at = 0; at < Cfg::ATOMS; ++at) {
            tma_load_2d(sk + at * 16384, &tmK, &kv_full[st], at * 64, row);
            tma_load_2d(sk + KVB + at * 16384, &tmV, &kv_full[st], at * 64, row);
          }
        }
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idesc_s = make_idesc_f16(128, 128);
    constexpr uint32_t idesc_o = make_idesc_f16(128, DKP, /*b_mn_major=*/true);
    const uint32_t q_addr = smem_u32(sQ);
    auto issue_s = [&](int t, int jg) {
      const uint32_t k_addr = smem_u32(sKV + (jg % NST) * 2 * KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + t * 128, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                  sdesc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    // keys [64 half, +64) of page jg -> S columns [64 half, +64); commits s_full when last
    auto issue_s_half = [&](int t, int jg, int half, bool last) {
      constexpr uint32_t idesc_h = make_idesc_f16(128, 64);
      const uint32_t k_addr = smem_u32(sKV + (jg % NST) * 2 * KVB) + half * 8192;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DKP / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + t * 128 + half * 64, sdesc_sw128(q_addr + t * Cfg::Q_BYTES + off, 16, 1024),
                  sdesc_sw128(k_addr + off, 16, 1024), idesc_h, kk > 0 ? 1u : 0u);
        }
        if (last) umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j, int jg) {
      const uint32_t v_addr = smem_u32(sKV + (jg % NST) * 2 * KVB + KVB);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc_sw128(v_addr + kk * 16 * 128, 16384, 1024),
                  idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&pv_full[t]);
      }
      __syncwarp();
    };
    int jg = 0;
    for (int k = 0;; ++k) {
      const int u = take_unit(k);
      if (u >= n_units) break;
      int g, pair, n_kv;
      unit_of(u, g, pair, n_kv);
      mbar_wait(q_full, (uint32_t)k & 1);  // both tiles' Q of this unit are in shared memory
      tc_fence_after();
      mbar_wait(&kv_full[jg % NST], (uint32_t)(jg / NST) & 1);
      tc_fence_after();
      issue_s(0, jg);
      issue_s(1, jg);
      if constexpr (SPLIT) {
        // P(j) occupies S columns [0, 64) only: keys [64, 128) of S(j+1) go into columns
        // [64, 128) as soon as the softmax holds S(j) in registers, so after P(j) only PV(j)
        // and the other half of S(j+1) stand between two softmax passes of a tile
        for (int j = 0; j < n_kv; ++j, ++jg) {
          const bool more = j + 1 < n_kv;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&s_free[t], (uint32_t)jg & 1);
            if (more) {
              if (t == 0) mbar_wait(&kv_full[(jg + 1) % NST], (uint32_t)((jg + 1) / NST) & 1);
              tc_fence_after();
              issue_s_half(t, jg + 1, 1, false);
            }
            mbar_wait(&p_full[t], (uint32_t)jg & 1);
            tc_fence_after();
            issue_pv(t, j, jg);
            if (t == 1) {
              if (elect_one()) umma_commit(&kv_empty[jg % NST]);
              __syncwarp();
            }
            if (more) issue_s_half(t, jg + 1, 0, true);
          }
        }
      } else {
      for (int j = 0; j < n_kv; ++j, ++jg) {
        const bool more = j + 1 < n_kv;
        mbar_wait(&p_full[0], (uint32_t)jg & 1);
        tc_fence_after();
        issue_pv(0, j, jg);
        if (more) {
          mbar_wait(&kv_full[(jg + 1) % NST], (uint32_t)((jg + 1) / NST) & 1);
          tc_fence_after();
          issue_s(0, jg + 1);
        }
        mbar_wait(&p_full[1], (uint32_t)jg & 1);
        tc_fence_after();
        issue_pv(1, j, jg);
        if (elect_one()) umma_commit(&kv_empty[jg % NST]);
        __syncwarp();
        if (more) issue_s(1, jg + 1);
      }
      }
    }
  } else {
    const int t = warp >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lb = (uint32_t)((quarter * 32) << 16);
    const uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
    const float sl2 = a.scale_log2;
    const int hj = r / a.T, ti = r - hj * a.T;
    int jg = 0;
    for (int k = 0;; ++k) {
      const int u = take_unit(k);
      if (u >= n_units) break;
      int g, pair, n_kv;
      unit_of(u, g, pair, n_kv);
      const int b = 2 * pair + t;
      const bool has_tile = b < a.n_tiles;
      const int tok = b * a.T + ti;
      const bool valid = has_tile && hj < a.G && tok < a.n_q;
      const int head = g * a.G + hj;
      const int tile_last = min((b + 1) * a.T, a.n_q) - 1;
      const int min_pos = has_tile ? a.pos[b * a.T] : 0x7fffffff;
      const int my_pos = valid ? a.pos[tok] : (has_tile ? a.pos[tile_last] : 0x7fffffff);
#pragma unroll 1
      for (int h = 0; h < Cfg::ATOMS; ++h) {  // this row's Q -> smem (both 64-column atoms)
        uint4 v[8];
        const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long)tok * a.H + head) * DKP) + h * 8;
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = valid ? src[c] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(sQ + t * Cfg::Q_BYTES + h * 16384 + r * 128 + ((c ^ (r & 7)) * 16)) = v[c];
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);

      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n_kv; ++j, ++jg) {
        mbar_wait(&s_full[t], (uint32_t)jg & 1);  // also implies PV_t(j-1) is complete
        tc_fence_after();
        const int key0 = j * 128;
        float sv[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[32];
          tmem_ld32(tS + lb + c * 32, w);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(w[i]);
        }
        if constexpr (SPLIT) {  // S(j) is in registers: columns [64, 128) may take S(j+1)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[t]);
        }
        if (key0 + 127 > min_pos) {
#pragma unroll
          for (int i = 0; i < 128; ++i) sv[i] = (key0 + i <= my_pos) ? sv[i] : -INFINITY;
        }
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 128; i += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], fmaxf(sv[i + 2 * q], sv[i + 2 * q + 1]));
        const float tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        const float m_new = fmaxf(m_run, tmax * sl2);
        const bool grow = (m_new - m_run) > 8.0f;
        const float m_use = grow ? m_new : m_run;
        const uint64_t sl2x2 = f32x2(sl2, sl2), negm = f32x2(-m_use, -m_use);
        uint64_t rsum2 = f32x2(0.f, 0.f), rsum2b = f32x2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint64_t x = ffma2(f32x2(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]), sl2x2, negm);
            float x0, x1;
            f32x2_unpack(x, x0, x1);
            float p0, p1;
            constexpr uint32_t kPolyMask = POLY >= 4 ? 0xAAu : POLY == 3 ? 0x94u : POLY == 2 ? 0x88u : POLY == 1 ? 0x80u : 0u;
            if ((kPolyMask >> (i & 7)) & 1u) {
              p0 = exp2_poly(x0);
              p1 = exp2_poly(x1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            if (i & 1) rsum2b = fadd2(rsum2b, f32x2(p0, p1));
            else rsum2 = fadd2(rsum2, f32x2(p0, p1));
            pk[i] = pack_f16(p0, p1);
          }
          tmem_st16(tS + lb + c * 16, pk);
        }
        float rs0, rs1;
        f32x2_unpack(fadd2(rsum2, rsum2b), rs0, rs1);
        if (__any_sync(0xffffffffu, grow && j > 0)) {
          const float alpha = (grow && j > 0) ? ex2(m_run - m_use) : 1.f;
#pragma unroll 1
          for (int c = 0; c < DKP / 32; ++c) {
            uint32_t w[32];
            tmem_ld32(tO + lb + c * 32, w);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
            tmem_st32(tO + lb + c * 32, w);
          }
        }
        if (grow && j > 0) l_run *= ex2(m_run - m_use);
        if (grow) m_run = m_use;
        l_run += rs0 + rs1;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      mbar_wait(&pv_full[t], (uint32_t)(jg - 1) & 1);  // the unit's last PV of this tile
      tc_fence_after();
      const float inv_l = 1.f / l_run;
#pragma unroll 1
      for (int c = 0; c < DKP / 32; ++c) {
        uint32_t w[32];
        tmem_ld32(tO + lb + c * 32, w);
        tmem_ld_wait();
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(a.out + ((long)tok * a.H + head) * DKP + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_f16(__uint_as_float(w[8 * i]) * inv_l, __uint_as_float(w[8 * i + 1]) * inv_l),
                                pack_f16(__uint_as_float(w[8 * i + 2]) * inv_l, __uint_as_float(w[8 * i + 3]) * inv_l),
                                pack_f16(__uint_as_float(w[8 * i + 4]) * inv_l, __uint_as_float(w[8 * i + 5]) * inv_l),
                                pack_f16(__uint_as_float(w[8 * i + 6]) * inv_l, __uint_as_float(w[8 * i + 7]) * inv_l));
        }
      }
      tc_fence_before();
      __syncwarp();
    }
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int POLY, int SPLIT = 0>
static int launch_attn_ps(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream,
                          int* ticket_ws) {
  using Cfg = AttnCfg<128>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(attn_ps_kernel<POLY, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn_ps smem attr: %s", cudaGetErrorString(err));
  const int units = a.n_pairs * a.Hkv;
  // the caller's workspace ticket (Stage II: one per repair, so concurrent in-process ranks do
  // not share it); else one per process for the standalone entry point
  static int* own = nullptr;
  int* ticket = ticket_ws;
  if (ticket == nullptr) {
    if (own == nullptr && cudaMalloc(&own, sizeof(int)) != cudaSuccess)
      return set_error(PKV_ERR_CUDA, "attn_ps: ticket allocation");
    ticket = own;
  }
  cudaMemsetAsync(ticket, 0, sizeof(int), stream);
  AttnArgs b = a;
  b.ticket = ticket;
  launch_k(attn_ps_kernel<POLY, SPLIT>, std::min(units, num_sms()), 320, Cfg::SMEM, stream, tk, tv, b);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_ps_kernel");
  return PKV_OK;
}

static int launch_attn_row(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream) {
  using Cfg = AttnCfg<128>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(attn_row_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn_row smem attr: %s", cudaGetErrorString(err));
  launch_k(attn_row_kernel<1>, a.n_pairs * a.Hkv, 320, Cfg::SMEM, stream, tk, tv, a);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_row_kernel");
  return PKV_OK;
}

template <int DKP, int POLY>
static int launch_attn(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream) {
  using Cfg = AttnCfg<DKP>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(attn_tc_kernel<DKP, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn smem attr: %s", cudaGetErrorString(err));
  launch_k(attn_tc_kernel<DKP, POLY>, a.n_pairs * a.Hkv, 576, Cfg::SMEM, stream, tk, tv, a);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_tc_kernel");
  return PKV_OK;
}

// CTA-pair launch: clusters of 2, grid = 2 * Hkv * ceil(n_pairs / 2)
template <int POLY>
static int launch_attn_pair(const CUtensorMap& tk64, const CUtensorMap& tv, const AttnArgs& a, cudaStream_t stream) {
  using Cfg = AttnCfg<128>;
  auto kern = attn_tc_kernel<128, POLY, 1>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&] { err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM); });
  if (err != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn pair smem attr: %s", cudaGetErrorString(err));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * a.Hkv * ((a.n_pairs + 1) / 2));
  cfg.blockDim = dim3(576);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, tk64, tv, a);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("attn_tc_kernel (CTA pairs)");
  return PKV_OK;
}

static unsigned long long* g_attn_trace = nullptr;
static unsigned long long* g_attn_cta_trace = nullptr;

// q/out: [n_q][H][dkp] fp16; k_pool/v_pool: [L][Hkv][pool_tokens][dkp] fp16 (whole pool)
int attn_tc_launch(const void* q, void* out, const int32_t* pos, int n_q, int H, int Hkv, int head_dim, int dkp,
                   const void* k_pool, const void* v_pool, long pool_rows_total, long pool_tokens, int layer,
                   const int32_t* page_table, cudaStream_t stream, int* ticket) {
  if (n_q <= 0) return PKV_OK;
  const int G = H / Hkv;
  if (G > 128) return set_error(PKV_ERR_CONFIG, "attention: group size %d > 128", G);
  AttnArgs a;
  a.q = reinterpret_cast<const __half*>(q);
  a.out = reinterpret_cast<__half*>(out);
  a.pos = pos;
  a.page_table = page_table;
  a.n_q = n_q;
  a.H = H;
  a.Hkv = Hkv;
  a.G = G;
  a.T = 128 / G;
  a.n_tiles = ceil_div(n_q, a.T);
  a.n_pairs = ceil_div(a.n_tiles, 2);
  {
    static const int hg_env = getenv("PKV_ATTN_HG") ? atoi(getenv("PKV_ATTN_HG")) : 4;
    int hg = std::max(1, std::min(hg_env, Hkv));
    while (Hkv % hg) --hg;
    a.hg = hg;
  }
  a.kv_row0 = (long)layer * Hkv * pool_tokens;
  a.pool_tokens = pool_tokens;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  a.trace = nullptr;
  a.cta_trace = nullptr;
  {
    static const bool ct = getenv("PKV_ATTN_CTA_TRACE") && getenv("PKV_ATTN_CTA_TRACE")[0] == '1';
    if (ct && g_attn_cta_trace == nullptr &&
        cudaMalloc(&g_attn_cta_trace, 16384 * 4 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(g_attn_cta_trace, 0, 16384 * 4 * sizeof(unsigned long long));
    if (ct && (long)a.n_pairs * Hkv <= 16384) a.cta_trace = g_attn_cta_trace;
  }
  {
    static const bool tr = getenv("PKV_ATTN_TRACE") && getenv("PKV_ATTN_TRACE")[0] == '1';
    static unsigned long long* buf = nullptr;
    if (tr && buf == nullptr && cudaMalloc(&buf, 8 * 64 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(buf, 0, 8 * 64 * sizeof(unsigned long long));
    if (tr) a.trace = buf;
    g_attn_trace = buf;
  }
  CUtensorMap tk, tv;
  if (!cached_tmap(&tk, k_pool, pool_rows_total, dkp, dkp, 128) ||
      !cached_tmap(&tv, v_pool, pool_rows_total, dkp, dkp, 128))
    return set_error(PKV_ERR_CUDA, "attention: TMA encode failed");
  const char* env = getenv("PKV_ATTN_POLY");  // tuning override: exponentials on the FMA pipe per 8
  const int poly = env ? atoi(env) : 1;
  static const int split = getenv("PKV_ATTN_SPLIT") ? atoi(getenv("PKV_ATTN_SPLIT")) : 2;
  if (dkp == 128 && split == 3) {
    using Cfg = AttnCfg<128>;
    constexpr int smem3 = Cfg::SMEM + 2048;  // 3-slice max exchange
    static std::once_flag once3;
    static cudaError_t err3 = cudaSuccess;
    std::call_once(once3, [] {
      err3 = cudaFuncSetAttribute(attn_tc3_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    });
    if (err3 != cudaSuccess) return set_error(PKV_ERR_CUDA, "attn3 smem attr: %s", cudaGetErrorString(err3));
    launch_k(attn_tc3_kernel<1>, a.n_pairs * a.Hkv, 832, smem3, stream, tk, tv, a);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("attn_tc3_kernel");
    return PKV_OK;
  }
  static const bool pair_env = getenv("PKV_ATTN_PAIR") && getenv("PKV_ATTN_PAIR")[0] == '1';
  if (dkp == 128 && pair_env && poly == 1) {
    CUtensorMap tk64;
    if (!cached_tmap(&tk64, k_pool, pool_rows_total, dkp, dkp, 64))
      return set_error(PKV_ERR_CUDA, "attention: TMA encode failed");
    return launch_attn_pair<1>(tk64, tv, a, stream);
  }
  // persistent, dynamically scheduled form by default (1.393 vs 1.410 ms per C3 layer,
  // tools/bench_attn.py); PKV_ATTN_PERSIST=0 launches one CTA per unit
  static const bool ps_env = !(getenv("PKV_ATTN_PERSIST") && getenv("PKV_ATTN_PERSIST")[0] == '0');
  // S(j+1) issued in two key halves, one of them during the softmax of page j
  static const bool split_env = getenv("PKV_ATTN_SPLIT_S") && getenv("PKV_ATTN_SPLIT_S")[0] == '1';
  if (dkp == 128 && ps_env && split_env && poly == 1) return launch_attn_ps<1, 1>(tk, tv, a, stream, ticket);
  if (dkp == 128 && ps_env && poly == 0) return launch_attn_ps<0>(tk, tv, a, stream, ticket);
  if (dkp == 128 && ps_env && poly == 1) return launch_attn_ps<1>(tk, tv, a, stream, ticket);
  if (dkp == 128 && ps_env && poly == 2) return launch_attn_ps<2>(tk, tv, a, stream, ticket);
  if (dkp == 128 && ps_env && poly == 3) return launch_attn_ps<3>(tk, tv, a, stream, ticket);
  static const bool row_env = getenv("PKV_ATTN_ROW") && getenv("PKV_ATTN_ROW")[0] == '1';
  if (dkp == 128 && row_env && poly == 1) return launch_attn_row(tk, tv, a, stream);
  static const bool one_env = getenv("PKV_ATTN_ONE") && getenv("PKV_ATTN_ONE")[0] == '1';
  if (dkp == 128 && one_env && poly == 1) return launch_attn1(tk, tv, a, stream);
  if (dkp == 128) {
    if (poly == 1) return launch_attn<128, 1>(tk, tv, a, stream);
    if (poly < 0) return launch_attn<128, -1>(tk, tv, a, stream);
    return launch_attn<128, 2>(tk, tv, a, stream);
  }
  if (dkp == 64) return launch_attn<64, 2>(tk, tv, a, stream);
  return set_error(PKV_ERR_CONFIG, "attention: padded head dim %d unsupported", dkp);
}

}  // namespace pkv

extern "C" int pkv_debug_attn_trace(unsigned long long* host) {
  if (pkv::g_attn_trace == nullptr) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, pkv::g_attn_trace, 8 * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}

extern "C" int pkv_debug_attn_cta_trace(unsigned long long* host, int n_ctas) {
  if (pkv::g_attn_cta_trace == nullptr) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, pkv::g_attn_cta_trace, (size_t)std::min(n_ctas, 16384) * 4 * sizeof(unsigned long long),
             cudaMemcpyDeviceToHost);
  return 0;
}
