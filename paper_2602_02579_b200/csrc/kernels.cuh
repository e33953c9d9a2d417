// Launcher declarations and the argument structs shared between translation units.
#pragma once
#include "common.cuh"

namespace pkv {

struct ChunkView {
  const uint64_t* k_nr;
  const uint64_t* v;
  const int32_t* src_chunk;
  const int32_t* src_local;
  const int32_t* chunk_len;
};
int assemble_launch(const ChunkView& cv, int s, int l0, int l1, int Hkv, int dkp, int head_dim, const double* rcos,
                    const double* rsin, const int32_t* page_table, void* k_pool, void* v_pool, long pool_tokens,
                    void* k2_pool, cudaStream_t stream);
int cache_view_launch(const ChunkView& cv, int use_chunks, int s, int layer, int Hkv, int dkp, int head_dim,
                      const double* rcos, const double* rsin, const int32_t* page_table, const void* pool,
                      const void* pool2, long pool_tokens, int is_key, float* out, cudaStream_t stream);
int scatter_launch(const int32_t* idx, int n, int layer, int Hkv, int dkp, int head_dim, const float* src,
                   const int32_t* page_table, void* pool, long pool_tokens, void* pool2, cudaStream_t stream);
int mark_launch(const int32_t* idx, int n, uint8_t* flags, cudaStream_t st);
int split3_launch(const float* x, int m, int cols, long ld, void* x3, long ldx, cudaStream_t st);
// ybf (nullable): the normalised rows as a 16-bit GEMM operand, fp16 (Stage II) or bf16 (y16_bf16 = 1: the
// full-prefill lm_head GEMM, whose weights stay bf16)
int rmsnorm_launch(const float* h, int m, int D, long ld, const float* gain, double eps, float* y, void* x3, long ldx,
                   void* ybf, cudaStream_t st, int y16_bf16 = 0);
int splitk_reduce_launch(const float* part, int splits, int N, int m, float* y, long ldy, int mode, cudaStream_t st);
int query_qkv_launch(const float* qkv, int m, int H, int Hkv, int dk, int dkp, int pos0, const double* rcos,
                     const double* rsin, float* q, float* k, float* v, void* k_pool, void* v_pool, long pool_tokens,
                     const int32_t* page_table, float* fresh_k, float* fresh_v, void* k2_pool, cudaStream_t st,
                     void* q3 = nullptr);
int silu_act_launch(const float* gu, int m, int F, int Fp, float* act, cudaStream_t st, void* x3 = nullptr,
                    long ldx = 0);

// SIMT fp32 narrow-pass attention (all keys, or only the fresh query keys when
// the context keys run on the tensor cores)
struct S1Attn {
  const float* q;
  int m, H, Hkv, G, dk, dkp, s, s_tot, R, keys_per_split, n_splits;
  int key_base, split_base;          // first key / first partial index of this launch
  int tc_splits, tc_keys_per_split;  // >0: context keys on tcgen05 (s1_attn_tc), fresh keys here
  float scale;
  int src_chunks;
  const uint8_t* recomp;  // nullable [s]: repaired entries come from the pool
  const uint64_t* ck;
  const uint64_t* cv;
  const int32_t* src_chunk;
  const int32_t* src_local;
  const int32_t* chunk_len;
  const double* rcos;
  const double* rsin;
  const __half* k_pool;  // layer base (fp16)
  const __half* v_pool;
  const __half* k2_pool;  // layer base, nullable: residual key plane
  long pool_tokens;
  const int32_t* page_table;
  int layer;
  int pool_heads, head0;  // the pools' head layout (a head-slice view of a larger cache)
  const float* fk;
  const float* fv;
  float* S;
  float* Opart;
  float* Mpart;
  float* Lpart;
  // whole-pool bases for the tensor-core path (TMA) and its Q-plane workspace
  void* q3;
  int q3_ready;  // the Q planes were written by query_qkv_kernel (R % 128 == 0)
  void* x3_out;  // nullable: also write the output as 3 scaled fp16 planes (next projection's B operand)
  long x3_ld;
  const void* k1_all;
  const void* k2_all;
  const void* v_all;
  long pool_rows_total;
  // scoring pass 2 (s1_score_tc_kernel) workspace; sc_part == null: score-matrix path
  float* sc_w;     // [Hkv][R] row weights
  float* sc_c;     // [Hkv][R] context mass of each row
  float* sc_part;  // [RB][Hkv][s] column sums
  int sc_splits, sc_keys_per_split;
};

// tensor-core narrow-pass attention over the context keys [0, s)
struct S1TcArgs {
  const float* q;  // [m][H][DKP] rotated fp32
  void* q3;        // workspace: fp16 Q planes [Hkv][RB][3][128][DKP]
  int q3_ready;    // already written (fused into query_qkv_kernel)
  int m, H, Hkv, G, dk, R, s, s_tot, keys_per_split, n_splits;
  float scale;
  long kv_row0;  // first pool row of this layer: layer * Hkv * pool_tokens
  long pool_tokens;
  const int32_t* page_table;
  float* S;  // key-major scores [Hkv][s][R] (context keys only) or null
  float* Opart;
  float* Mpart;
  float* Lpart;
  // fresh = 1: one extra CTA per (KV head, row block) at blockIdx.x == n_splits scores the
  // m fresh query keys (fp32 K/V [m][Hkv][DKP], causal) as split n_splits (m <= 128)
  int fresh;
  const float* fk;
  const float* fv;
  unsigned long long* trace;  // debug (PKV_S1_TRACE=1): %globaltimer per tile of CTA (0,0,0), s1_attn_tc.cu
};
int s1_attn_tc_launch(const S1TcArgs& a, const void* k1, const void* k2, const void* v, long pool_rows_total, int dkp,
                      cudaStream_t st);

// second pass of the scoring (K2b): QK^T recomputed exactly as the first pass forms it,
// p = exp(S - M) * w with the final per-row max M and weight w = 1 / (L * H * m) (or the
// context-renormalised weight), summed over the CTA's 128 rows per context key
struct S1ScoreArgs {
  const void* q3;         // the first pass's fp16 Q planes [Hkv][RB][3][128][DKP]
  int Hkv, R, s, keys_per_split, n_splits;
  float scale;
  long kv_row0, pool_tokens;
  const int32_t* page_table;
  const float* Mfin;      // [Hkv][R]
  const float* W;         // [Hkv][R] row weights
  float* part;            // [RB][Hkv][s] per-row-block column sums
  unsigned long long* trace;  // debug (PKV_S1_TRACE=1): CTA (0,0,0) start, Q in TMEM, S(j) seen, end
};
int s1_score_tc_launch(const S1ScoreArgs& a, const void* k1, const void* k2, long pool_rows_total, int dkp,
                       cudaStream_t st);
int s1_attention_launch(const S1Attn& a, float* attn_out, float* Mfin, float* Lfin, float* rows, double* denom,
                        float* per_layer, int renorm, int H_total, double* rows64, pkv_comm* comm, cudaStream_t st,
                        float* capture_rows = nullptr);
int gemv_launch(const float* x, const void* W, int N, int D, long ldw, float* out, cudaStream_t st);
int norm_defer_launch(const float* h, int m, long ld, int N, const float* g, void* xg, long ldxg, float* ssq,
                      int ssq_ld, cudaStream_t st);
int probe_diag_colsum_launch(const float* q, const float* k, const float* Mfin, const float* Lfin, int m, int H,
                             int Hkv, int dk, int dkp, float scale, float* out, cudaStream_t st);
int probe_accum_launch(const float* part, int p0, int n, double* colsum, cudaStream_t st);
int probe_scores_launch(const float* v1, const void* vp1, const int32_t* page_table, long pool_tokens, int s, int Hkv,
                        int dk, int dkp, const double* colsum, float* out, cudaStream_t st);
int probe_cache_kv_launch(float* k, float* v, int m, int Hkv, int dk, int dkp, int pos0, const void* k_pool,
                          const void* k2_pool, const void* v_pool, long pool_tokens,
                          const int32_t* page_table, cudaStream_t st);
int embed_gather_launch(const void* embed, long lde, const int32_t* ids, const int32_t* sel, int n, int D, float* out,
                        long ldo, cudaStream_t st);
int fuse_layers_launch(const float* per_layer, int L, int s, float* fused, cudaStream_t st);
int topk_launch(const float* v, int n, int k, int32_t* out, int32_t* status, cudaStream_t st);
int attn_tc_launch(const void* q, void* out, const int32_t* pos, int n_q, int H, int Hkv, int head_dim, int dkp,
                   const void* k_pool, const void* v_pool, long pool_rows_total, long pool_tokens, int layer,
                   const int32_t* page_table, cudaStream_t stream, int* ticket = nullptr);

}  // namespace pkv
