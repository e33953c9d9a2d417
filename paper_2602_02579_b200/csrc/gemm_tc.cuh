// Persistent, warp-specialised tcgen05 GEMM:  D[M,N] = A[M,K] . B[N,K]^T
// (both operands K-major, both fp16 or both bf16, fp32 accumulation in TMEM) with
// fused epilogues.  fp16 weights are stored pre-scaled by a power of two (see
// DeviceModel); every epilogue multiplies the accumulator by acc_scale first.
//
//   warp 0      TMA producer (one elected lane) -> smem ring of STAGES (A,B) tiles
//   warp 1      TMEM allocator + MMA issuer (one elected lane), 2 TMEM accumulators
//   warps 2..5  epilogue: tcgen05.ld a row per thread, apply EPI, store to HBM
//
// Used by Stage II (recompute_selected, reference recompute.py:55-82: QKV / o /
// gate-up / down projections) with A = activations of the k selected tokens and
// B = transposed weights, and by the fp32-faithful narrow pass with A = weights
// and B = a scaled 3-way fp16 split of the fp32 activations (split3s, common.cuh).
#pragma once
#include "common.cuh"

namespace pkv {

enum GemmEpi : int {
  EPI_F32 = 0,      // C (+ split * M * ldc) = acc               (fp32 partials / plain store)
  EPI_BF16 = 1,     // C = bf16(acc)
  EPI_RESID = 2,    // C += acc                                    (fp32 residual stream)
  EPI_SILU = 3,     // C[:, n/2..] = fp16(silu(gate) * up), gate/up interleaved per 128 cols
  EPI_QKV = 4,      // rope(q), rope(k) at token positions; q -> fp16 buffer; k, v -> paged fp16 cache
  EPI_PROJ = 5,     // narrow pass (BN = 96): y[i][n] = (acc[n][i] + 2^-11 acc[n][32+i]) + 2^-22 acc[n][64+i]
                    // (the 3 scaled fp16 planes of 32 fp32 rows), stored / added to out[i][n]; split-K
                    // partials are reduced in split order by the last-arriving CTA of each M tile
};

struct GemmArgs {
  int M, N, K;
  int k_tiles_per_split;  // in units of 64
  int n_splits;
  void* C;                // output (see GemmEpi)
  long ldc;               // elements
  // EPI_QKV -----------------------------------------------------------------
  const int32_t* pos;         // [M] token positions (also cache slot via page table)
  const double* rope_cos;     // [n_pos][dk/2]
  const double* rope_sin;
  const float2* rope_cs32;    // optional f32 (cos, sin) [n_pos][dk/2]: fp32 rotation (fp16 Stage II)
  int head_dim, dkp, n_heads, n_kv_heads;
  __half* k_pool;             // layer base: [Hkv][pool_tokens][dkp] fp16
  __half* v_pool;
  long pool_tokens;
  const int32_t* page_table;
  float* tap_k;               // optional fp32 [M][Hkv][dk]
  float* tap_v;
  int tap_rows;               // with qtap_*: rows >= tap_rows tap into qtap_* at row - tap_rows instead
  float* qtap_k;              // (the query rows riding along a Stage-II repair, pkv_recompute_query)
  float* qtap_v;
  __half* kvc;                // optional compact copy of the cache entries [M][3][Hkv][dkp] fp16 (K, K
                              // residual, V) for the token-parallel exchange (pkv_recompute_rows)
  __half* k2_pool;            // optional residual key plane fp16(k - k_pool) (layer base), see s1_attn_tc.cu
  __nv_bfloat16* knr_out;     // optional bf16 [M][Hkv][dkp]: keys BEFORE RoPE (chunk-store layout)
  __nv_bfloat16* vcap_out;    // optional bf16 [M][Hkv][dkp]: values (chunk-store layout)
  int head0;                  // first head of the GEMM's N range (H: K and V rows only)
  // EPI_PROJ ---------------------------------------------------------------
  float* out;                 // [mrows][ldo]
  long ldo;
  int mrows;                  // valid query rows (<= 32)
  int resid;                  // 1: out += y
  float* part;                // split-K partials [n_splits][tiles_m*128][32]
  int* cnt;                   // [tiles_m] arrival counters (zero; reset by the reducing CTA)
  unsigned long long* trace;  // debug (PKV_GEMM_TRACE=1): per-CTA globaltimer stamps [grid][8]
  int stream_k;               // EPI_PROJ: 1 = stream-K (CTA c owns k units [c*U/G, (c+1)*U/G))
  // Stage-II stream-K tail (CTA pairs): the T % P tiles of the last, partial wave are cut
  // into k pieces over the first sk_pairs pairs, before the T - T % P whole tiles
  int sk_pairs;               // 0 = off
  float* sk_part;             // [rem tiles][SK_MAXP][CG][BN cols][128 rows] fp32 pieces
  int* sk_cnt;                // [rem tiles][CG] arrival counters (zeroed; reset by the reducer)
  int sk_maxp;                // piece stride per tail tile (<= SK_MAXP)
  // deferred RMSNorm (Stage II).  rmsnorm(h) . W = ((h * g) . W) / rms(h) row by row, so
  // an EPI_RESID producer writes xg = fp16(h_new * ng) and the fp32 sums of h_new^2 of each
  // (row, BN-column tile) -- sequentially over the tile's columns -- and the next GEMM
  // (EPI_QKV / EPI_SILU) scales its accumulator rows by 1 / sqrt(sum / norm_D + eps).
  // Replaces a standalone norm pass over h (read 4 B + write 2 B per element) per norm.
  const float* ng;            // producer: gain of the next norm [N] (nullptr: off)
  __half* xg;                 // producer: [M][ldxg] fp16(h_new * ng)
  long ldxg;
  float* ssq;                 // producer: [M][ssq_ld] per-tile sums of h_new^2 (fp32, in column order)
  int ssq_ld;
  const float* ssq_in;        // consumer: [M][ssq_ld] (nullptr: input already normalised)
  int ssq_n;                  // consumer: tiles to sum (in order)
  int norm_D;                 // consumer: mean divisor (the unpadded hidden size)
  float norm_eps;
  int f16;                    // operands fp16 (Stage II, narrow projections) instead of bf16
  float acc_scale;            // accumulator multiplier (2^-e of the pre-scaled fp16 weights)
  int raster_gm;              // tile-mode order: m-tiles per raster group (0 = all, m fastest)
  int* nonfinite;             // nullable: OR-ed with 1 when EPI_QKV / EPI_SILU / EPI_RESID write a
                              // non-finite value (the reference's check_finite, tensor.py:31-34)
};
constexpr int SK_MAXP = 8;    // pieces per tail tile (host plan guarantees)

__device__ __forceinline__ void gemm_stamp(const GemmArgs& a, int i) {
  if (a.trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 8 + i] = t;
  }
}

// BK = k extent of one pipeline stage (SW128 atoms of 64 bf16); MT = 128-row sub-tiles of
// A per CTA tile sharing each B tile (EPI_PROJ only).  Measured on the narrow-pass
// projections (tools/bench_proj.py, graph-captured): BK = 128 and MT = 2 were both slower
// or neutral (per-SM smem fill, not the barrier round trip or the B traffic, bounds them),
// so both stay at 1 atom / 1 sub-tile; the knobs are kept for re-tuning.
// PKV_PROJ_MT (compile time): weight sub-tiles per narrow-projection CTA.  2 (44 KB stages,
// 27 % less activation fill per weight byte) measured 1.5-2x slower with stream-K
// (tools/bench_proj.py: wgu 62 vs 46 us, wd 41 vs 27 us), so the stage count and not the
// activation share of the fill sets the per-CTA stream rate.
#ifndef PKV_PROJ_MT
#define PKV_PROJ_MT 1
#endif
constexpr int gemm_bk(int bn) { return 64; }
constexpr int gemm_mt(int bn, int epi) { return (bn == 96 && epi == 5 /*EPI_PROJ*/) ? PKV_PROJ_MT : 1; }
// CG = 2: CTA pair (cluster of 2, cta_group::2).  One MMA tile is 256 x BN: each CTA
// loads its 128 rows of A and HALF of B (BN/2 rows), the leader issues M = 256 MMAs that
// read both CTAs' shared memory, and each CTA's TMEM receives its 128 rows x BN.  Per SM
// this halves the B fill per MMA flop (the Stage-II GEMMs move 48 -> 32 KB per 64-deep
// k step), the canonical Blackwell GEMM shape.
template <int BN, int EPI, int CG = 1>
struct GemmCfg {
  static constexpr int BM = 128, BK = gemm_bk(BN), MT = CG == 2 ? 1 : gemm_mt(BN, EPI), BMT = BM * MT * CG;
  static constexpr int BN_CTA = BN / CG;                            // B rows held by one CTA
  static constexpr int ATOMS = BK / 64;
  static constexpr int A_ATOM = BM * 128, B_ATOM = BN_CTA * 128;  // bytes of one 64-column atom
  static constexpr int A_SUB = BM * BK * 2;                        // one 128-row sub-tile
  static constexpr int A_BYTES = MT * A_SUB;
  static constexpr int B_BYTES = BN_CTA * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 2 ? 6 : (BN >= 256) ? 4 : (BN >= 128 ? 6 : (MT == 2 ? 5 : 7));
  static_assert(CG == 1 || MT == 1, "CTA pairs with one A sub-tile per CTA");
  static_assert(MT == 1 || EPI == EPI_PROJ, "sub-tiled A only for the narrow projection epilogue");
  static constexpr int ACC_STRIDE = MT * (BN <= 128 ? 128 : 256);
  static constexpr int TMEM_COLS = 2 * ACC_STRIDE;
  // fp32 stores (EPI_F32 / EPI_RESID): a 32 x 32 fp32 transpose tile per epilogue warp, so the
  // residual stream is read and written a whole 128-byte row segment per 8 lanes instead of
  // one row per lane (32 lines per warp instruction)
  static constexpr int EPI_STAGE = (EPI == 0 /*EPI_F32*/ || EPI == 2 /*EPI_RESID*/) ? 4 * 32 * 32 * 4 : 0;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE;
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

// Narrow-pass projections (EPI_PROJ): every M tile streams its own weights but all of
// them read the SAME activation tile at a given k, so in lock-step the whole grid hits
// the few L2 slices holding that tile.  Each M tile therefore walks its k range from a
// different starting point (fixed per tile: deterministic fp32 order).
template <int EPI>
__device__ __forceinline__ int k_rotation_t(int mb, int nk) {
  if constexpr (EPI == EPI_PROJ) return nk > 0 ? (mb * 5) % nk : 0;
  return 0;
}
#define k_rotation(mb, nk) k_rotation_t<EPI>(mb, nk)

// CK = 1 (EPI_PROJ only): split-K across a thread-block cluster of n_splits CTAs (one
// m-tile per cluster, rank = split); the partial results are summed through distributed
// shared memory by rank 0 in split order -- no global partials, fences or atomics.
template <int BN, int EPI, int CG, int CK = 0>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
  using Cfg = GemmCfg<BN, EPI, CG>;
  static_assert(CK == 0 || (EPI == EPI_PROJ && CG == 1), "cluster split-K is for the narrow projection");
  const uint32_t rank = (CG == 2 || CK) ? cluster_ctarank() : 0;  // CTA of the pair / k split
  int cta_id = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  int n_ctas = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  if constexpr (CK) {  // exactly one tile per CTA: (m-tile = cluster, split = rank)
    const int tiles_m_ = (args.M + Cfg::BMT - 1) / Cfg::BMT;
    cta_id = (int)(blockIdx.x / args.n_splits) + tiles_m_ * (int)rank;
    n_ctas = 1 << 30;
  }
  if (threadIdx.x == 64) gemm_stamp(args, 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int tiles_m = (args.M + Cfg::BMT - 1) / Cfg::BMT;
  const int subtiles_m = (args.M + Cfg::BM - 1) / Cfg::BM;  // EPI_PROJ partial / counter index space
  const int tiles_n = (args.N + BN - 1) / BN;
  const int total_tiles = tiles_m * tiles_n * args.n_splits;
  const int k_tiles_total = (args.K + Cfg::BK - 1) / Cfg::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4 * CG);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_barrier_init();
  }
  if constexpr (CG == 2) {
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive / TMA
    if (warp == 1) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
  } else {
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: the prologue above overlapped the previous kernel; from here on we read its outputs
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 64) gemm_stamp(args, 1);

  // tile order: m fastest, in groups of raster_gm m-tiles (all n of a group before the next
  // group) so that a wave of concurrent tiles reads few distinct A panels when A does not
  // fit in L2 (Stage-II down projection: A = 6554 x 14336 fp16 = 188 MB)
  const int gm = (args.raster_gm > 0 && args.raster_gm < tiles_m) ? args.raster_gm : tiles_m;
  auto tile_coords = [&](int t, int& mb, int& nb, int& sp) {
    const int mn = tiles_m * tiles_n;
    sp = t / mn;
    const int r = t - sp * mn;
    const int g0 = (r / (gm * tiles_n)) * gm;  // first m-tile of the group
    const int gsz = min(gm, tiles_m - g0);
    const int ri = r - g0 * tiles_n;
    mb = g0 + ri % gsz;
    nb = ri / gsz;
  };

  // Work items.  Tile mode: tile t = (m, n, split) strided over the grid.  Stream-K
  // (narrow projection): the U = tiles_m * k_tiles units (m-tile, 64-deep k step) are cut
  // into G equal contiguous ranges, one per CTA; a range covers the tail of one m-tile,
  // whole tiles and the head of another.  Piece idx of an m-tile is its idx-th owner, so
  // the split points -- and the fixed-order sum of the pieces -- depend only on (U, G).
  struct Work { int mb, nb, k0, k1, idx, nseg, slot; };
  const bool sk = (EPI == EPI_PROJ && CG == 1 && CK == 0) && args.stream_k;
  const long U = (long)tiles_m * k_tiles_total;
  auto sk_start = [&](int c) -> long { return (long)c * U / n_ctas; };
  auto sk_owner = [&](long u) -> int {
    int c = (int)((u * n_ctas) / U);
    if (c >= n_ctas) c = n_ctas - 1;
    while (c + 1 < n_ctas && sk_start(c + 1) <= u) ++c;
    while (c > 0 && sk_start(c) > u) --c;
    return c;
  };
  // Stage-II tail: phase 0 walks this pair's share of the rem tail tiles' k units
  // (tiles T-rem..T-1), phase 1 the whole tiles 0..T-rem-1 strided over the pairs.
  const int skp = (CG == 2 && EPI != EPI_PROJ) ? args.sk_pairs : 0;
  const int sk_rem = skp ? (tiles_m * tiles_n) % n_ctas : 0;
  const long Usk = (long)sk_rem * k_tiles_total;
  auto t_start = [&](int c) -> long { return skp ? (long)c * Usk / skp : 0; };
  auto t_owner = [&](long u) -> int {
    int c = (int)((u * skp) / Usk);
    if (c >= skp) c = skp - 1;
    while (c + 1 < skp && t_start(c + 1) <= u) ++c;
    while (c > 0 && t_start(c) > u) --c;
    return c;
  };
  int phase0 = (skp && cta_id < skp) ? 1 : 0;
  auto first_pos = [&]() -> long {
    phase0 = (skp && cta_id < skp) ? 1 : 0;
    return sk ? sk_start(cta_id) : (phase0 ? t_start(cta_id) : (long)cta_id);
  };
  auto next_work = [&](long& pos, Work& w) -> bool {
    w.slot = -1;
    if (phase0) {
      const long u1 = t_start(cta_id + 1);
      if (pos < u1) {
        const int sl = (int)(pos / k_tiles_total);
        int sp_;
        tile_coords(tiles_m * tiles_n - sk_rem + sl, w.mb, w.nb, sp_);
        w.k0 = (int)(pos - (long)sl * k_tiles_total);
        w.k1 = (int)min((long)k_tiles_total, (long)w.k0 + (u1 - pos));
        const long tb = (long)sl * k_tiles_total;
        const int o0 = t_owner(tb);
        w.idx = cta_id - o0;
        w.nseg = t_owner(tb + k_tiles_total - 1) - o0 + 1;
        w.slot = sl;
        pos += w.k1 - w.k0;
        return true;
      }
      phase0 = 0;
      pos = cta_id;
    }
    if (sk) {
      const long u1 = sk_start(cta_id + 1);
      if (pos >= u1) return false;
      w.mb = (int)(pos / k_tiles_total);
      w.nb = 0;
      w.k0 = (int)(pos - (long)w.mb * k_tiles_total);
      w.k1 = (int)min((long)k_tiles_total, (long)w.k0 + (u1 - pos));
      const long tb = (long)w.mb * k_tiles_total;
      const int o0 = sk_owner(tb);
      w.idx = cta_id - o0;
      w.nseg = sk_owner(tb + k_tiles_total - 1) - o0 + 1;
      pos += w.k1 - w.k0;
      return true;
    }
    if (pos >= total_tiles - sk_rem) return false;
    int sp;
    tile_coords((int)pos, w.mb, w.nb, sp);
    w.k0 = sp * args.k_tiles_per_split;
    w.k1 = min(w.k0 + args.k_tiles_per_split, k_tiles_total);
    w.idx = sp;
    w.nseg = args.n_splits;
    pos += n_ctas;
    return true;
  };

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      long pos = first_pos();
      Work w;
      while (next_work(pos, w)) {
        const int mb = w.mb, nb = w.nb, k0 = w.k0;
        const int nk = w.k1 - k0, rot = k_rotation(mb, nk);
        for (int i = 0; i < nk; ++i) {
          const int kt = k0 + (i + rot) % nk;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if constexpr (CG == 2) {
            // both CTAs' bytes land on the leader's full barrier (only the leader's MMA waits)
            if (rank == 0) mbar_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
#pragma unroll
            for (int at = 0; at < Cfg::ATOMS; ++at) {
              tma_load_2d_cg2(sa + at * Cfg::A_ATOM, &tmA, &full_bar[stage], kt * Cfg::BK + at * 64,
                              mb * Cfg::BMT + (int)rank * Cfg::BM);
              tma_load_2d_cg2(sb + at * Cfg::B_ATOM, &tmB, &full_bar[stage], kt * Cfg::BK + at * 64,
                              nb * BN + (int)rank * Cfg::BN_CTA);
            }
          } else {
            mbar_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
#pragma unroll
            for (int at = 0; at < Cfg::ATOMS; ++at) {
#pragma unroll
              for (int j = 0; j < Cfg::MT; ++j)
                tma_load_2d(sa + j * Cfg::A_SUB + at * Cfg::A_ATOM, &tmA, &full_bar[stage], kt * Cfg::BK + at * 64,
                            mb * Cfg::BMT + j * Cfg::BM);
              tma_load_2d(sb + at * Cfg::B_ATOM, &tmB, &full_bar[stage], kt * Cfg::BK + at * 64, nb * BN);
            }
          }
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && (CG == 1 || rank == 0)) {  // the pair's MMAs are issued by the leader
    const uint32_t idesc = make_idesc(128 * CG, BN, args.f16 != 0);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    long pos = first_pos();
    Work w;
    for (; next_work(pos, w); ++local) {
      const int k0 = w.k0, k1 = w.k1;
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      mbar_wait(&tempty_bar[acc], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * Cfg::ACC_STRIDE;
      const int nk = k1 - k0;
      for (int i = 0; i < nk; ++i) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t b_addr = a_addr + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < Cfg::BK / 16; ++kk) {
            uint64_t bd = sdesc_sw128(b_addr + (kk >> 2) * Cfg::B_ATOM + (kk & 3) * 32, 16, 1024);
#pragma unroll
            for (int j = 0; j < Cfg::MT; ++j) {
              uint64_t ad = sdesc_sw128(a_addr + j * Cfg::A_SUB + (kk >> 2) * Cfg::A_ATOM + (kk & 3) * 32, 16, 1024);
              if constexpr (CG == 2)
                umma_ss_cg2(d_tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
              else
                umma_ss(d_tmem + j * (Cfg::ACC_STRIDE / Cfg::MT), ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
            }
          }
          if constexpr (CG == 2) umma_commit_cg2(&empty_bar[stage]);  // frees the stage in both CTAs
          else umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) {
        if constexpr (CG == 2) umma_commit_cg2(&tfull_bar[acc]);
        else umma_commit(&tfull_bar[acc]);
      }
      __syncwarp();
    }
  } else if (warp >= 2) {
    // ---------------------------------------------------------------- epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = quarter * 32 + lane;
    const float asc = args.acc_scale;
    int local = 0;
    long pos = first_pos();
    Work w;
    for (; next_work(pos, w); ++local) {
      const int mb = w.mb, nb = w.nb;
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      // EPI_PROJ residual (out += y): a whole-tile item fetches out[.][n] while its MMAs
      // run; a split tile's reducer fetches it with the pieces (one round trip either way)
      [[maybe_unused]] float rres[32];
      [[maybe_unused]] bool have_r = false;
      if constexpr (EPI == EPI_PROJ && CG == 1 && Cfg::MT == 1) {
        const int n = mb * Cfg::BM + (warp & 3) * 32 + lane;
        if (args.resid && w.nseg == 1 && n < args.M) {
#pragma unroll
          for (int i = 0; i < 32; ++i) rres[i] = i < args.mrows ? __ldcg(args.out + (long)i * args.ldo + n) : 0.f;
          have_r = true;
        }
      }
      mbar_wait(&tfull_bar[acc], use & 1);
      tc_fence_after();
      const int row = mb * Cfg::BMT + (int)rank * Cfg::BM + row_in_tile;
      const bool row_ok = row < args.M;
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * Cfg::ACC_STRIDE;
      bool do_epi = true;
      if constexpr (CG == 2 && EPI != EPI_PROJ) {
        if (w.slot >= 0 && w.nseg > 1) {
          // tail piece: store the raw fp32 accumulator (coalesced: [col][row]); the last
          // piece to arrive sums all pieces in piece order (deterministic) back into its
          // TMEM accumulator and runs the normal epilogue on it
          __shared__ int s_last2;
          const long pstride = (long)CG * BN * 128;
          const float* pbase = args.sk_part + (long)w.slot * args.sk_maxp * pstride + (long)rank * BN * 128 + row_in_tile;
          float* mine = const_cast<float*>(pbase) + w.idx * pstride;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t a[32];
            __syncwarp();
            tmem_ld32(t_row + c * 32, a);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) __stcg(mine + (long)(c * 32 + i) * 128, __uint_as_float(a[i]));
          }
          named_bar_sync(1, 128);
          if (threadIdx.x == 64)
            s_last2 = atom_add_acq_rel_gpu(&args.sk_cnt[w.slot * CG + (int)rank], 1) == w.nseg - 1 ? 1 : 0;
          named_bar_sync(1, 128);
          if (!s_last2) {
            do_epi = false;
          } else {
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              float sum[32];
#pragma unroll 2
              for (int j = 0; j < w.nseg; ++j) {
                const float* pj = pbase + j * pstride + (long)c * 32 * 128;
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __ldcg(pj + (long)i * 128);
#pragma unroll
                for (int i = 0; i < 32; ++i) sum[i] = j == 0 ? v[i] : sum[i] + v[i];
              }
              uint32_t r[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(sum[i]);
              __syncwarp();
              tmem_st32(t_row + c * 32, r);
            }
            tmem_st_wait();
            if (threadIdx.x == 64) args.sk_cnt[w.slot * CG + (int)rank] = 0;
          }
        }
      }
      bool bad = false;  // a non-finite output in this work item (nonfinite flag)
      if (do_epi) {
      [[maybe_unused]] float rnorm = 1.f;
      if constexpr (EPI == EPI_QKV || EPI == EPI_SILU) {
        if (args.ssq_in != nullptr && row_ok) {
          // the tile sums in order; loads issued 8 at a time (one round trip for D <= 2048)
          const float* sp = args.ssq_in + (long)row * args.ssq_ld;
          float sq = 0.f;
          for (int t0 = 0; t0 < args.ssq_n; t0 += 8) {
            float part[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) part[q] = t0 + q < args.ssq_n ? sp[t0 + q] : 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (t0 + q < args.ssq_n) sq += part[q];
          }
          rnorm = 1.f / sqrtf(sq / (float)args.norm_D + args.norm_eps);
        }
      }

      if constexpr (EPI == EPI_PROJ) {
       __shared__ int s_last;
       if (threadIdx.x == 64) gemm_stamp(args, 2);
#pragma unroll 1
       for (int j = 0; j < Cfg::MT; ++j) {
        // one thread = one output feature n; the 96 accumulator columns are the hi/mid/lo
        // planes of the 32 query rows
        const int msub = (mb * CG + (int)rank) * Cfg::MT + j;  // 128-row sub-tile
        uint32_t a0[32], a1[32], a2[32];
        __syncwarp();
        const uint32_t t_sub = t_row + j * (Cfg::ACC_STRIDE / Cfg::MT);
        tmem_ld32(t_sub, a0);
        tmem_ld32(t_sub + 32, a1);
        tmem_ld32(t_sub + 64, a2);
        tmem_ld_wait();
        if (CG == 1 && j == Cfg::MT - 1) {  // accumulator drained: the next item's MMAs may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        }
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          y[i] = fmaf(__uint_as_float(a2[i]), 1.f / X3_LO, fmaf(__uint_as_float(a1[i]), 1.f / X3_MID,
                                                                __uint_as_float(a0[i]))) * asc;
        const int n = msub * Cfg::BM + row_in_tile;  // GEMM row == output feature
        bool write = w.nseg == 1;
        if constexpr (CK) {  // partial -> own smem (the pipeline ring is drained); reduced below
          float* xb = reinterpret_cast<float*>(smem) + row_in_tile * 33;
#pragma unroll
          for (int i = 0; i < 32; ++i) xb[i] = y[i];
          write = false;
        } else if (!write) {
          // partial piece, row-major [32 query rows][128 features]: coalesced stores/loads
          float* mine = args.part + (long)(w.idx * subtiles_m + msub) * 4096 + row_in_tile;
#pragma unroll
          for (int i = 0; i < 32; ++i) __stcg(mine + i * 128, y[i]);
          // release/acquire hand-off: the barrier orders the 128 threads' partial stores
          // before thread 64's acq_rel atomic (cumulative), and the last CTA's reads after
          // its acquire.  (__threadfence() here was a MEMBAR.SC.GPU + L1 invalidate per
          // thread, several microseconds per launch.)
          named_bar_sync(1, 128);
          if (threadIdx.x == 64) gemm_stamp(args, 3);
          if (threadIdx.x == 64) s_last = (atom_add_acq_rel_gpu(&args.cnt[msub], 1) == w.nseg - 1) ? 1 : 0;
          named_bar_sync(1, 128);
          if (threadIdx.x == 64) gemm_stamp(args, 4);
          if (s_last) {
            // fixed piece order -> bit-identical regardless of which CTA arrives last;
            // four pieces' loads in flight per round trip
            if (CG == 1 && Cfg::MT == 1 && args.resid && n < args.M) {
#pragma unroll
              for (int i = 0; i < 32; ++i) rres[i] = i < args.mrows ? __ldcg(args.out + (long)i * args.ldo + n) : 0.f;
              have_r = true;
            }
#pragma unroll 1
            for (int s0 = 0; s0 < w.nseg; s0 += 4) {
              float v[4][32];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (s0 + q < w.nseg) {
                  const float* p = args.part + (long)((s0 + q) * subtiles_m + msub) * 4096 + row_in_tile;
#pragma unroll
                  for (int i = 0; i < 32; ++i) v[q][i] = __ldcg(p + i * 128);
                }
              }
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (s0 + q < w.nseg) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) y[i] = (s0 + q == 0) ? v[q][i] : y[i] + v[q][i];
                }
              }
            }
            if (threadIdx.x == 64) args.cnt[msub] = 0;
            write = true;
            if (threadIdx.x == 64) gemm_stamp(args, 5);
          }
        }
        if (write && n < args.M) {
          if (args.resid && !have_r) {
#pragma unroll
            for (int i = 0; i < 32; ++i) rres[i] = i < args.mrows ? __ldcg(args.out + (long)i * args.ldo + n) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {  // constant indices keep y in registers
            if (i < args.mrows) args.out[(long)i * args.ldo + n] = args.resid ? rres[i] + y[i] : y[i];
          }
        }
        if (threadIdx.x == 64) gemm_stamp(args, 6);
       }
      } else if constexpr (EPI == EPI_SILU) {
        // gate columns [0,BN/2), up columns [BN/2,BN) of this tile feed BN/2 outputs
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          uint32_t g[32], u[32];
          __syncwarp();
          tmem_ld32(t_row + c * 32, g);
          tmem_ld32(t_row + BN / 2 + c * 32, u);
          tmem_ld_wait();
          const int col = nb * (BN / 2) + c * 32;
          if (row_ok && col < args.N / 2) {
            uint32_t packed[16];
            const float sc = rnorm * asc;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float a0 = silu_f(__uint_as_float(g[2 * j]) * sc) * (__uint_as_float(u[2 * j]) * sc);
              float a1 = silu_f(__uint_as_float(g[2 * j + 1]) * sc) * (__uint_as_float(u[2 * j + 1]) * sc);
              bad |= !(fabsf(a0) <= 65504.f) || !(fabsf(a1) <= 65504.f);  // non-finite or fp16 overflow
              packed[j] = pack_f16(a0, a1);
            }
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(args.C) + (long)row * args.ldc + col);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
          }
        }
      } else {
        [[maybe_unused]] float ssacc = 0.f;  // deferred norm: sum of h_new^2 over this tile
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          __syncwarp();
          tmem_ld32(t_row + c * 32, r);
          tmem_ld_wait();
          const int col0 = nb * BN + c * 32;
          if constexpr (EPI == EPI_F32 || EPI == EPI_RESID) {
            if (args.xg == nullptr && col0 + 32 <= args.N && (args.ldc & 3) == 0) {
              // transpose through shared memory: lane = row on the TMEM side, 8 lanes = one
              // row's 32 columns (128 B) on the global side; float4 slots XOR-swizzled by row
              float* stg = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 256) + quarter * 1024;
              float* base = reinterpret_cast<float*>(args.C) + (long)(w.slot >= 0 ? 0 : w.idx) * args.M * args.ldc + col0;
              const int row0 = mb * Cfg::BMT + (int)rank * Cfg::BM + quarter * 32;
              const int cc = lane & 7;
              [[maybe_unused]] float4 o[8];
              if constexpr (EPI == EPI_RESID) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int gr = row0 + i * 4 + (lane >> 3);
                  if (gr < args.M) o[i] = __ldcg(reinterpret_cast<const float4*>(base + (long)gr * args.ldc) + cc);
                }
              }
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) * 4)) =
                    make_float4(__uint_as_float(r[4 * j]) * asc, __uint_as_float(r[4 * j + 1]) * asc,
                                __uint_as_float(r[4 * j + 2]) * asc, __uint_as_float(r[4 * j + 3]) * asc);
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rr = i * 4 + (lane >> 3), gr = row0 + rr;
                float4 v = *reinterpret_cast<const float4*>(stg + rr * 32 + ((cc ^ (rr & 7)) * 4));
                if (gr < args.M) {
                  if constexpr (EPI == EPI_RESID) {
                    v.x += o[i].x; v.y += o[i].y; v.z += o[i].z; v.w += o[i].w;
                    bad |= !isfinite(v.x + v.y + v.z + v.w);
                  }
                  reinterpret_cast<float4*>(base + (long)gr * args.ldc)[cc] = v;
                }
              }
              __syncwarp();
              continue;
            }
          }
          if (!row_ok || col0 >= args.N) continue;
          const bool full = col0 + 32 <= args.N && (args.ldc & 7) == 0;  // vector stores need aligned rows
          if constexpr (EPI == EPI_F32 || EPI == EPI_RESID) {
            float* dst = reinterpret_cast<float*>(args.C) + (long)(w.slot >= 0 ? 0 : w.idx) * args.M * args.ldc + (long)row * args.ldc + col0;
            if (full) {
              // all residual loads first: a store through another pointer (xg) between
              // them would otherwise serialise every load behind the previous store
              [[maybe_unused]] float4 o[8];
              if constexpr (EPI == EPI_RESID) {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = reinterpret_cast<const float4*>(dst)[j];
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float4 v = make_float4(__uint_as_float(r[4 * j]) * asc, __uint_as_float(r[4 * j + 1]) * asc,
                                       __uint_as_float(r[4 * j + 2]) * asc, __uint_as_float(r[4 * j + 3]) * asc);
                if constexpr (EPI == EPI_RESID) {
                  v.x += o[j].x; v.y += o[j].y; v.z += o[j].z; v.w += o[j].w;
                  bad |= !isfinite(v.x + v.y + v.z + v.w);
                  r[4 * j] = __float_as_uint(v.x);
                  r[4 * j + 1] = __float_as_uint(v.y);
                  r[4 * j + 2] = __float_as_uint(v.z);
                  r[4 * j + 3] = __float_as_uint(v.w);
                }
                reinterpret_cast<float4*>(dst)[j] = v;
              }
              if constexpr (EPI == EPI_RESID) {
                if (args.xg != nullptr) {
                  float4 gg[8];
#pragma unroll
                  for (int j = 0; j < 8; ++j) gg[j] = __ldg(reinterpret_cast<const float4*>(args.ng + col0) + j);
                  uint2* xd = reinterpret_cast<uint2*>(args.xg + (long)row * args.ldxg + col0);
#pragma unroll
                  for (int j = 0; j < 8; ++j) {
                    const float a = __uint_as_float(r[4 * j]), b = __uint_as_float(r[4 * j + 1]);
                    const float c2 = __uint_as_float(r[4 * j + 2]), d = __uint_as_float(r[4 * j + 3]);
                    ssacc = fmaf(a, a, ssacc);
                    ssacc = fmaf(b, b, ssacc);
                    ssacc = fmaf(c2, c2, ssacc);
                    ssacc = fmaf(d, d, ssacc);
                    xd[j] = make_uint2(pack_f16(a * gg[j].x, b * gg[j].y), pack_f16(c2 * gg[j].z, d * gg[j].w));
                  }
                }
              }
            } else {
              // (fully unrolled with a predicate: a data-dependent trip count would index r[]
              // dynamically and put every accumulator chunk of the kernel in local memory)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (col0 + j >= args.N) continue;
                float v = __uint_as_float(r[j]) * asc;
                if constexpr (EPI == EPI_RESID) {
                  v += dst[j];
                  if (args.xg != nullptr) {
                    ssacc = fmaf(v, v, ssacc);
                    args.xg[(long)row * args.ldxg + col0 + j] = __float2half_rn(v * args.ng[col0 + j]);
                  }
                }
                dst[j] = v;
              }
            }
          } else if constexpr (EPI == EPI_BF16) {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.C) + (long)row * args.ldc + col0;
            if (full) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                reinterpret_cast<uint4*>(dst)[j] =
                    make_uint4(pack_bf16(__uint_as_float(r[8 * j]) * asc, __uint_as_float(r[8 * j + 1]) * asc),
                               pack_bf16(__uint_as_float(r[8 * j + 2]) * asc, __uint_as_float(r[8 * j + 3]) * asc),
                               pack_bf16(__uint_as_float(r[8 * j + 4]) * asc, __uint_as_float(r[8 * j + 5]) * asc),
                               pack_bf16(__uint_as_float(r[8 * j + 6]) * asc, __uint_as_float(r[8 * j + 7]) * asc));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < args.N) dst[j] = __float2bfloat16_rn(__uint_as_float(r[j]) * asc);
            }
          } else if constexpr (EPI == EPI_QKV) {
            // a 32-column chunk never straddles a head (dkp is 64 or 128)
            const int dkp = args.dkp;
            const int d0 = col0 % dkp;
            const int head_all = col0 / dkp + args.head0;  // 0..H+2Hkv-1
            const int H = args.n_heads, Hkv = args.n_kv_heads;
            const int pos = args.pos[row];
            const bool is_v = head_all >= H + Hkv;
            float vals[32];
            const float sc = rnorm * asc;
#pragma unroll
            for (int j = 0; j < 32; ++j) vals[j] = __uint_as_float(r[j]) * sc;
            if (head_all >= H) {  // precompute_chunk captures: unrotated keys / values
              __nv_bfloat16* cap = is_v ? args.vcap_out : args.knr_out;
              if (cap != nullptr) {
                const int gk = is_v ? head_all - H - Hkv : head_all - H;
                uint4* cd = reinterpret_cast<uint4*>(cap + ((long)row * Hkv + gk) * dkp + d0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  cd[j] = make_uint4(pack_bf16(vals[8 * j], vals[8 * j + 1]), pack_bf16(vals[8 * j + 2], vals[8 * j + 3]),
                                     pack_bf16(vals[8 * j + 4], vals[8 * j + 5]),
                                     pack_bf16(vals[8 * j + 6], vals[8 * j + 7]));
              }
            }
            if (!is_v && args.rope_cs32 != nullptr) {
              // interleaved-pair RoPE (reference tensor.py:104-113) in fp32 with the float64
              // factors rounded to f32: Stage II stores fp16, so the f64 rotation buys
              // nothing here and would make the FP64 pipe the epilogue's bottleneck
              const int half = args.head_dim >> 1;
              const float2* cs = args.rope_cs32 + (long)pos * half;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int i = (d0 >> 1) + j;
                if (2 * i < args.head_dim) {
                  const float2 f = __ldg(cs + i);
                  const float e = vals[2 * j], o = vals[2 * j + 1];
                  vals[2 * j] = fmaf(e, f.x, -o * f.y);
                  vals[2 * j + 1] = fmaf(e, f.y, o * f.x);
                }
              }
            } else if (!is_v) {
              // interleaved-pair RoPE with float64 factors (reference tensor.py:104-113)
              const int half = args.head_dim >> 1;
              const double* cs = args.rope_cos + (long)pos * half;
              const double* sn = args.rope_sin + (long)pos * half;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                int i = (d0 >> 1) + j;
                if (2 * i < args.head_dim) {
                  double c = cs[i], s = sn[i];
                  double e = (double)vals[2 * j], o = (double)vals[2 * j + 1];
                  vals[2 * j] = (float)__dsub_rn(__dmul_rn(e, c), __dmul_rn(o, s));
                  vals[2 * j + 1] = (float)__dadd_rn(__dmul_rn(e, s), __dmul_rn(o, c));
                }
              }
            }
            // q -> fp16 operand buffer; k -> fp16 pool + fp16 residual plane; v -> fp16 pool
            uint32_t packed[16], pk2[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              bad |= !(fabsf(vals[2 * j]) <= 65504.f) || !(fabsf(vals[2 * j + 1]) <= 65504.f);
              split2h_pack(vals[2 * j], vals[2 * j + 1], packed[j], pk2[j]);
            }
            __half* dst;
            if (head_all < H) {
              dst = reinterpret_cast<__half*>(args.C) + (long)row * args.ldc + col0;
            } else {
              const int g = is_v ? head_all - H - Hkv : head_all - H;
              const long slot = (long)args.page_table[pos >> 7] * 128 + (pos & 127);
              __half* pool = is_v ? args.v_pool : args.k_pool;
              const long po = ((long)g * args.pool_tokens + slot) * dkp + d0;
              dst = pool + po;
              if (args.kvc != nullptr) {  // compact copy for the token-parallel exchange
                uint4* kc = reinterpret_cast<uint4*>(args.kvc + (((long)row * 3 + (is_v ? 2 : 0)) * Hkv + g) * dkp + d0);
#pragma unroll
                for (int j = 0; j < 4; ++j) kc[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
                if (!is_v) {
                  uint4* k2c = reinterpret_cast<uint4*>(args.kvc + (((long)row * 3 + 1) * Hkv + g) * dkp + d0);
#pragma unroll
                  for (int j = 0; j < 4; ++j) k2c[j] = make_uint4(pk2[4 * j], pk2[4 * j + 1], pk2[4 * j + 2], pk2[4 * j + 3]);
                }
              }
              if (!is_v && args.k2_pool != nullptr) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  reinterpret_cast<uint4*>(args.k2_pool + po)[j] =
                      make_uint4(pk2[4 * j], pk2[4 * j + 1], pk2[4 * j + 2], pk2[4 * j + 3]);
              }
              float* tap = is_v ? args.tap_v : args.tap_k;
              long trow = row;
              if ((args.qtap_k != nullptr || args.qtap_v != nullptr) && row >= args.tap_rows) {
                tap = is_v ? args.qtap_v : args.qtap_k;
                trow = row - args.tap_rows;
              }
              if (tap != nullptr) {
                float* tp = tap + (trow * Hkv + g) * args.head_dim;
                for (int j = 0; j < 32; ++j)
                  if (d0 + j < args.head_dim) tp[d0 + j] = vals[j];
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              reinterpret_cast<uint4*>(dst)[j] =
                  make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
          }
        }
        if constexpr (EPI == EPI_RESID) {
          if (args.xg != nullptr && row_ok && nb * BN < args.N) args.ssq[(long)row * args.ssq_ld + nb] = ssacc;
        }
      }
      }  // do_epi
      if constexpr (EPI == EPI_QKV || EPI == EPI_SILU || EPI == EPI_RESID) {
        if (args.nonfinite != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(args.nonfinite, 1);
      }
      if constexpr (EPI != EPI_PROJ || CG == 2) {  // (EPI_PROJ, CG = 1 released it above)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(&tempty_bar[acc], 0);  // the leader's MMA waits
          else mbar_arrive(&tempty_bar[acc]);
        }
      }
    }
  }

  __syncthreads();
  if constexpr (CK) {
    cluster_sync();  // every split's partial is in its shared memory
    if (rank == 0 && warp >= 2) {
      const int row_in_tile = (warp & 3) * 32 + (threadIdx.x & 31);
      const int n = (cta_id % ((args.M + Cfg::BMT - 1) / Cfg::BMT)) * Cfg::BM + row_in_tile;
      float y[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) y[i] = 0.f;
      const uint32_t local = smem_u32(reinterpret_cast<float*>(smem) + row_in_tile * 33);
#pragma unroll 1
      for (int s2 = 0; s2 < args.n_splits; ++s2) {  // fixed split order: deterministic
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(s2));
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float v;
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote + 4 * i));
          y[i] += v;
        }
      }
      if (n < args.M) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i < args.mrows) {
            float* dst = args.out + (long)i * args.ldo + n;
            *dst = args.resid ? *dst + y[i] : y[i];
          }
        }
      }
    }
    cluster_sync();  // peers keep their shared memory until rank 0 has read it
  }
  if constexpr (CG == 2) cluster_sync();  // no TMEM use or remote arrive left in either CTA
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// host launcher (gemm_tc.cu)
// Stage-II stream-K tail plan for an M x N x K GEMM on CTA pairs (256 x 256 tiles):
// pairs sharing the tail (0 = off), tail tiles and the most pieces any tail tile gets.
int gemm_sk_plan(int M, int N, int K, int* rem_out, int* maxp_out);
// workspace for the tail pieces + counters of such a GEMM (0 when the plan is off)
size_t gemm_sk_ws_floats(int M, int N, int K);
int gemm_tc_launch(int epi, int bn, const void* A, long lda_rows, const void* B, long ldb_rows, int K, GemmArgs args,
                   cudaStream_t stream);
bool make_tmap_2d(CUtensorMap* map, const void* base, long rows, long cols, long row_stride_elems, int box_rows,
                  int box_cols);
// encoded once per (buffer, shape), 128B swizzle, 64-column boxes
bool cached_tmap(CUtensorMap* out, const void* base, long rows, long cols, long stride, int box_rows);

}  // namespace pkv
