/*
 * pkv.h -- C ABI of the B200-native ProphetKV selective-recompute prefill.
 *
 * The reference (`pikv`, /root/reference/pkg/src/pikv) is a pure-Python numpy
 * package with no FFI of its own; this header is the boundary its Python API
 * would bind (see INTEGRATION.md for the ctypes binding).  Every entry point
 * names the reference function it replaces.  Conventions:
 *
 *   - plain C types only; all tensor pointers are caller-owned DEVICE memory
 *     unless a field says "host"; no allocation inside (workspace is passed in,
 *     sized by the *_workspace() queries);
 *   - every call is stream-ordered on the given cudaStream_t (passed as void*),
 *     never synchronises the host, and is reentrant across streams;
 *   - return value is a status code (PKV_OK or one of the PKV_ERR_* below, which
 *     map 1:1 onto pikv.errors classes); pkv_last_error() gives a thread-local
 *     message.
 *
 * Device layouts (bf16 = IEEE bfloat16, fp16 = IEEE binary16, little endian):
 *   dkp  = 64 if head_dim <= 64 else 128 (head dims zero-padded)
 *   Dp   = hidden_dim rounded up to 64,  Fp = ffn_dim rounded up to 128
 *   NQKV = (n_heads + 2*n_kv_heads) * dkp
 *   projection weights are fp16, transposed ("output-major", K contiguous) and
 *   pre-scaled by a power of two per matrix (stored = w * 2^e, wscale = 2^-e):
 *     wqkv [NQKV][Dp]  rows = q heads, k heads, v heads, each dkp rows
 *     wo   [Dp][n_heads*dkp]
 *     wgu  [2*Fp][Dp]  gate/up interleaved in blocks of 128 rows
 *     wd   [Dp][Fp]
 *     embed, lm_head: bf16 [vocab][Dp];   norm gains fp32 [Dp]
 *   chunk store (one buffer per chunk): bf16 [n_layers][t_c][n_kv_heads][dkp], keys UNROTATED
 *   paged KV cache: fp16 K and V pools [n_layers][n_kv_heads][pool_tokens][dkp], plus the
 *     fp16 key residual plane k2_pool = fp16(f32 key - K) (same layout);
 *     token t lives in slot page_table[t / 128] * 128 + t % 128
 *   RoPE tables: float64 cos/sin [rope_len][head_dim/2], angle = pos * theta^(-2i/d)
 */
#ifndef PKV_H_
#define PKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> pikv.errors (reference errors.py:4-41) */
enum {
  PKV_OK = 0,
  PKV_ERR_SHAPE = 1,        /* ShapeError */
  PKV_ERR_ARGUMENT = 2,     /* ArgumentError */
  PKV_ERR_CONFIG = 3,       /* ConfigError */
  PKV_ERR_INPUT = 4,        /* InputError */
  PKV_ERR_STATE = 5,        /* StateError */
  PKV_ERR_INCOMPATIBLE = 6, /* IncompatibleError */
  PKV_ERR_NUMERICS = 7,     /* NumericsError */
  PKV_ERR_CUDA = 100        /* EngineError (device failure) */
};

/* query-pass flags */
enum {
  PKV_QP_SCORES = 1,    /* capture per-layer context scores (score_prophet) */
  PKV_QP_RENORM = 2,    /* renormalize_context_only=True */
  PKV_QP_LOGITS = 4,    /* compute last-row logits (finalize_query) */
  PKV_QP_APPEND_KV = 8, /* append query K/V to the cache pool at positions s.. */
  PKV_QP_FROM_CHUNKS = 16, /* read context keys/values from the chunk store (naive cache) */
  PKV_QP_PROBE = 32,      /* low-layer probe (selection.py:95-124): stop after layer 1's QKV
                             projection (fresh_v[1] = the probe's layer-1 values); the m
                             rows are context tokens s.. attending causally to [0, s) and
                             to their own assembled layer-0 entries.  With PKV_QP_SCORES,
                             per_layer[0..s) = layer 0's head/query-mean scores of the rows
                             and per_layer[s..s+m) = sum over rows q >= i of row q's
                             head-mean probability on block key i (kvshare column sums) */
  PKV_QP_ROWS = 64        /* capture_attn (query_pass model.py:386-398): per_layer receives the
                             head-averaged attention rows [L][m][s+m] f32 of every query token
                             over the s context and m query keys (unsharded models) */
};

/* reference ModelConfig, model.py:24-63 */
typedef struct pkv_config {
  int32_t n_layers, n_heads, n_kv_heads, head_dim, hidden_dim, ffn_dim, vocab_size;
  double rope_theta, norm_eps;
} pkv_config;

/* reference LayerWeights, model.py:66-76 (device layouts above) */
typedef struct pkv_layer_weights {
  const float* attn_norm;
  const float* ffn_norm;
  const void* wqkv;
  const void* wo;
  const void* wgu;
  const void* wd;
  float wscale[4];  /* 2^-e of wqkv, wo, wgu, wd (see "Device layouts") */
} pkv_layer_weights;

/* reference ModelWeights, model.py:79-160 */
typedef struct pkv_weights {
  const void* embed;
  const float* final_norm;
  const void* lm_head;
  const pkv_layer_weights* layers; /* host array [n_layers] */
} pkv_weights;

/* reference AssembledCache, chunkstore.py:65-96 (device state) */
typedef struct pkv_cache {
  void* k_pool;
  void* v_pool;
  int64_t pool_tokens;       /* slots per (layer, kv head); multiple of 128 */
  const int32_t* page_table; /* [ceil(rope_len/128)] */
  int32_t s;                 /* context length */
  const int32_t* token_ids;  /* [s] */
  const double* rope_cos;    /* [rope_len][head_dim/2] */
  const double* rope_sin;
  int32_t rope_len;          /* positions covered (>= s + query length) */
  const uint8_t* recomputed; /* nullable [s]: 1 = entry repaired by Stage II (read from the pool
                                even when a query pass reads the others from the chunk store) */
  void* k2_pool;             /* residual key plane, same layout as k_pool: the f32 key is k_pool +
                                k2_pool to 2^-22 (fp16 each); used by the fp32-faithful narrow passes */
  void* const* layer_ready;  /* nullable host array [n_layers] of cudaEvent_t: a query pass makes its
                                stream wait on layer_ready[l] before reading layer l (pipelined
                                host->device chunk transfer + per-layer assembly) */
  const float* rope_cs32;    /* nullable [rope_len][head_dim/2][2]: (cos, sin) of the float64 tables
                                rounded to f32, used by the fp16 Stage-II RoPE epilogue (the
                                fp32-faithful paths and assembly always use the float64 tables) */
  void* const* layer_done;   /* nullable host array [n_layers] of cudaEvent_t: pkv_recompute records
                                layer_done[l] once layer l's K/V are final (after its QKV scatter),
                                so the final query pass can follow Stage II layer by layer on
                                another stream (pass it these events as layer_ready) */
  int32_t* nonfinite;        /* nullable device int32: OR-ed with 1 when a Stage-II epilogue writes a
                                non-finite (or fp16-overflowing) value; the host raises NumericsError
                                (reference check_finite, tensor.py:31-34) */
  int32_t pool_heads;        /* 0, or the KV heads of the pools' layout when this cache is a head slice
                                of a larger cache (narrow passes only): layer stride pool_heads, this
                                view's heads start at head0 (token-parallel Stage II with a head-sharded
                                scoring pass, DeviceModel.rows + shard) */
  int32_t head0;
} pkv_cache;

/* reference list[ChunkKV] in prompt order, chunkstore.py:37-49 */
typedef struct pkv_chunks {
  const uint64_t* k_nr;      /* device [n_chunks] device pointers, bf16 [L][t_c][Hkv][dkp] */
  const uint64_t* v;         /* device [n_chunks] */
  const int32_t* chunk_len;  /* device [n_chunks] */
  const int32_t* src_chunk;  /* device [s] chunk ordinal of each token */
  const int32_t* src_local;  /* device [s] index inside its chunk */
  int32_t n_chunks;
} pkv_chunks;

typedef struct pkv_model pkv_model; /* opaque: config + device weight views */

/* padded layout: out[0..4] = dkp, Dp, Fp, NQKV, n_heads*dkp */
int pkv_layout(const pkv_config* cfg, int32_t out[5]);

/* validates the config like ModelConfig.__post_init__ (model.py:36-50) */
int pkv_model_create(const pkv_config* cfg, const pkv_weights* w, pkv_model** out);
void pkv_model_destroy(pkv_model* m);

/* assemble(chunks, config) -- chunkstore.py:99-140 (+ rope_apply tensor.py:89-114):
 * concatenates the chunk K/V into the paged cache, rotating keys at global
 * positions 0..s-1 with the float64 tables. */
int pkv_assemble(const pkv_config* cfg, const pkv_chunks* chunks, const pkv_cache* cache, void* stream);
/* same for layers [layer_begin, layer_end) only (layer-pipelined assembly) */
int pkv_assemble_layers(const pkv_config* cfg, const pkv_chunks* chunks, const pkv_cache* cache, int32_t layer_begin,
                        int32_t layer_end, void* stream);

/* query_pass -- model.py:370-402; with PKV_QP_SCORES it is score_prophet
 * (selection.py:64-86, per_layer [L][s] f32); with PKV_QP_LOGITS|PKV_QP_APPEND_KV
 * it is finalize_query (recompute.py:105-125, last_logits [vocab] f32).
 * query_ids: device int32 [m].  fresh_k/fresh_v (nullable): fp32 [L][m][Hkv][head_dim].
 * With PKV_QP_ROWS, per_layer is the capture_attn rows buffer [L][m][s+m]. */
size_t pkv_query_pass_workspace(const pkv_model* m, int32_t s, int32_t n_query, int32_t flags);
int pkv_query_pass(const pkv_model* m, const pkv_cache* cache, const pkv_chunks* chunks, const int32_t* query_ids,
                   int32_t n_query, int32_t flags, float* per_layer, float* fresh_k, float* fresh_v,
                   float* last_logits, void* workspace, size_t workspace_bytes, void* stream);

/* fuse_layers + select_top_p -- selection.py:52-61 with top_k_indices tensor.py:117-133.
 * per_layer [L][s] f32 -> fused [s] f32 (nullable) and the k indices, ascending, in idx_out.
 * status_out (device int32) receives PKV_OK or PKV_ERR_NUMERICS (non-finite scores). */
size_t pkv_select_workspace(int32_t n_layers, int32_t s);
int pkv_fuse_select(const float* per_layer, int32_t n_layers, int32_t s, int32_t k, float* fused, int32_t* idx_out,
                    int32_t* status_out, void* workspace, size_t workspace_bytes, void* stream);
/* top_k_indices -- tensor.py:117-133 on an arbitrary f32 vector */
int pkv_topk(const float* scores, int32_t n, int32_t k, int32_t* idx_out, int32_t* status_out, void* stream);

/* recompute_selected (fresh-peer mode) -- recompute.py:43-82.
 * sel: device int32 [k], strictly ascending positions.  Per layer: fresh K/V of
 * all selected tokens are written into the cache first (replace_entries,
 * chunkstore.py:143-160), then the selected queries attend over the updated
 * layer with mask pos_kv <= pos_sel.  tap_k/tap_v (nullable): fp32
 * [L][k][Hkv][head_dim] copies of the recomputed K/V before fp16 storage. */
size_t pkv_recompute_workspace(const pkv_model* m, int32_t k);
int pkv_recompute(const pkv_model* m, const pkv_cache* cache, const int32_t* sel, int32_t k, float* tap_k,
                  float* tap_v, void* workspace, size_t workspace_bytes, void* stream);

/* recompute_selected (recompute.py:43-82) followed by finalize_query (recompute.py:105-125)
 * in one pass: the m query tokens (device int32 ids) ride along the repair as rows
 * k..k+m-1 at positions s..s+m-1 -- per layer they attend over the repaired layer plus their
 * own causal entries, exactly what the separate query pass (model.py:370-402) reads --
 * their K/V are appended to the pool (as PKV_QP_APPEND_KV), and last_logits receives the
 * first-token logits of the last query row.  Stage-II precision (fp16 operands, fp32
 * accumulation and residual stream) instead of the fp32-faithful narrow pass; the north-star
 * logits tolerance (2e-2 / 0.999) applies.  query_k/query_v (nullable): fp32 [L][m][Hkv][dk]
 * fresh query K/V (the reference's appended KVCache entries).  Needs pool_tokens and
 * rope_len >= s + m. */
size_t pkv_recompute_query_workspace(const pkv_model* m, int32_t k, int32_t n_query);
int pkv_recompute_query(const pkv_model* m, const pkv_cache* cache, const int32_t* sel, int32_t k,
                        const int32_t* query_ids, int32_t n_query, float* tap_k, float* tap_v, float* query_k,
                        float* query_v, float* last_logits, void* workspace, size_t workspace_bytes, void* stream);

/* full_prefill -- model.py:332-359 (and precompute_chunk, chunkstore.py:52-62) on the
 * device: the Stage-II layer loop over every position 0..s-1 of `cache` (its token_ids
 * are the sequence; K/V land in its pool, RoPE'd at 0..s-1).  Optional captures:
 * k_nr_out / v_out bf16 [L][s][Hkv][dkp] (the chunk-store layout; keys BEFORE RoPE),
 * logits_out f32 [s][vocab] (final norm + lm_head on the bf16 tensor cores; bf16 lm_head). */
size_t pkv_full_prefill_workspace(const pkv_model* m, int32_t n);
int pkv_full_prefill(const pkv_model* m, const pkv_cache* cache, void* k_nr_out, void* v_out, float* logits_out,
                     void* workspace, size_t workspace_bytes, void* stream);

/* replace_entries -- chunkstore.py:143-160 (standalone scatter of fp32 rows) */
int pkv_replace_entries(const pkv_config* cfg, const pkv_cache* cache, int32_t layer, const int32_t* idx, int32_t n,
                        const float* new_k, const float* new_v, void* stream);

/* f32 view of one cache layer as keys_rebased/values ([s][Hkv][head_dim]).
 * chunks != NULL: derive from the chunk store (exact f32 rotation of the
 * assembled keys); chunks == NULL: read the fp16 cache (keys: k_pool + k2_pool). */
int pkv_cache_view(const pkv_config* cfg, const pkv_cache* cache, const pkv_chunks* chunks, int32_t layer, int32_t is_key,
                   float* out, void* stream);

/* Probe baselines (reference selection.py:95-142, score_cacheblend_l1 / score_kvshare_l1),
 * the reductions that follow the per-block probe passes (pkv_query_pass with PKV_QP_PROBE):
 *   pkv_probe_accum   colsum[t] += n * part[t] (t < p0), += part[t] (p0 <= t < p0 + n): the
 *                     layer-0 head-mean attention column sums of block [p0, p0+n), f64, in
 *                     block order (reference _low_layer_probe: rows.astype(F64).sum(axis=0));
 *   pkv_probe_scores  out[t] = f32(colsum[t] * ||dV_t||_1) (kvshare) or f32(||dV_t||_2)
 *                     (colsum == NULL: cacheblend), dV_t = v1[t] - the assembled layer-1
 *                     value of token t, norms in f64.  v1: [s][Hkv][head_dim] f32. */
int pkv_probe_accum(const float* part, int32_t p0, int32_t n, double* colsum, void* stream);
int pkv_probe_scores(const pkv_config* cfg, const pkv_cache* cache, const float* v1, const double* colsum, float* out,
                     void* stream);

/* ---------------------------------------------------------------------------
 * Head-sharded (tensor-parallel) prefill -- SURVEY §8(e), config C3 on 2/4/8 GPUs.
 * No reference counterpart: the reference is single-process numpy.
 * Rank r of W owns KV heads [r*Hkv/W, (r+1)*Hkv/W) with their query heads, and
 * ffn blocks [r*Fp/W, (r+1)*Fp/W) (Fp/128 must be divisible by W):
 *   wqkv_r = rows of its q, k and v heads; wo_r = its head columns of wo;
 *   wgu_r  = its 2*Fp/W rows (gate/up 128-row blocks); wd_r = its Fp/W columns.
 * embed, lm_head and the norm gains are replicated.  The cache and the chunk
 * store of a rank hold its KV heads only (n_kv_heads = Hkv/W in their config).
 * Exchange points (in-place sums): the per-(query, token) head-score partials
 * of every layer before the f32 head mean (so all ranks select the same
 * tokens), and the o / down projection outputs of every layer (narrow passes:
 * [m][Dp] fp32; Stage II: [k][Dp] fp32).                                    */
typedef struct pkv_comm pkv_comm;
enum { PKV_DT_F32 = 0, PKV_DT_F64 = 1, PKV_DT_BF16 = 2 };
#define PKV_MAX_LOCAL_RANKS 8

/* NCCL back end (libnccl.so.2 is dlopen'ed; path may be NULL = default search) */
int pkv_nccl_load(const char* path);
int pkv_comm_unique_id(uint8_t id_out[128]);
int pkv_comm_create_nccl(const uint8_t id[128], int32_t rank, int32_t world, pkv_comm** out);
/* in-process back end: `world` rank handles (out[world]) sharing one device,
 * each driven by its own host thread and stream (single-GPU tests of the
 * sharded path); sums are bit-identical on every rank */
int pkv_comm_create_local(int32_t world, pkv_comm** out);
int pkv_comm_allreduce(pkv_comm* c, void* buf, size_t count, int32_t dtype, void* stream);
int pkv_comm_rank(const pkv_comm* c);
int pkv_comm_world(const pkv_comm* c);
void pkv_comm_destroy(pkv_comm* c);

/* Token-parallel Stage II over the W ranks of `comm` (one process per GPU, every rank holding
 * the UNSHARDED model and a full assembled cache; multi-GPU alternative to head sharding,
 * SURVEY §8(e)).  No reference counterpart (single-process numpy).  sel: the global selection
 * (identical on every rank: the scoring pass is replicated and deterministic).  Rank r
 * repairs the attention units (128/G consecutive selected rows) r, r+W, r+2W, ...; after
 * each layer's QKV GEMM the ranks all-gather the fresh cache entries of their rows (fp16 K,
 * K residual, V: 6 KB per row at Llama width) and scatter the peers' into their own pools,
 * so the attention of every rank reads the whole repaired layer and all ranks end with the
 * identical cache -- one all-gather of ~40 MB per layer instead of two [k][D] fp32
 * all-reduces.  m > 0: the query rows ride along on every rank (as pkv_recompute_query)
 * and last_logits gets the first-token logits. */
size_t pkv_recompute_rows_workspace(const pkv_model* m, int32_t k, int32_t n_query, int32_t world);
int pkv_recompute_rows(const pkv_model* m, const pkv_cache* cache, const int32_t* sel, int32_t k,
                       const int32_t* query_ids, int32_t n_query, pkv_comm* comm, float* last_logits,
                       void* workspace, size_t workspace_bytes, void* stream);

/* cfg is the FULL model config; w holds rank tp_rank's weight shard (layouts
 * above with the local head / ffn counts).  comm may be NULL iff tp_world == 1. */
int pkv_model_create_sharded(const pkv_config* cfg, const pkv_weights* w, int32_t tp_rank, int32_t tp_world,
                             pkv_comm* comm, pkv_model** out);

/* unit-level entry points used by the kernel tests; pkv_gemm_bf16 takes fp16 A and B when
 * epilogue has bit 0x100 set */
int pkv_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M, int32_t N, int32_t K, float* C,
                  int64_t ldc, int32_t bn, int32_t epilogue, void* stream);
/* fp32-faithful narrow projection (the query passes' x.W of model.py:265-275 / 311-323):
 * out[i][n] (+)= sum_k x[i][k] W[n][k] for m <= 32 fp32 rows given as 3 scaled fp16 planes
 * x3 [96][ldx] (rows i, 32+i, 64+i: x = hi + 2^-11 mid + 2^-22 lo); W [N][K] fp16;
 * part >= 16*ceil(N/128)*128*32 floats,
 * cnt >= ceil(N/128) zeroed ints; n_splits > 0: split-K, 0: stream-K (default grid),
 * < 0: stream-K on a grid of -n_splits CTAs. */
int pkv_proj_narrow(const void* W, int32_t N, int32_t K, const void* x3, int64_t ldx, int32_t m, float* out,
                    int64_t ldo, int32_t resid, float* part, int32_t* cnt, int32_t n_splits, void* stream);
int pkv_attention_sparse(const pkv_model* m, const pkv_cache* cache, int32_t layer, const void* q, void* out,
                         const int32_t* pos, int32_t n_q, void* stream);

/* phase timers: when enabled, every stage records CUDA events on its stream around
 * each kernel group; collect() waits for them and returns per-category totals (ms)
 * and launch-group counts.  Categories: 0 assemble, 1 narrow-pass projections,
 * 2 narrow-pass attention+scores, 3 narrow-pass misc, 4 fuse+top-k, 5 Stage-II
 * QKV GEMM (+RoPE+scatter), 6 Stage-II attention, 7 o GEMM, 8 gate/up GEMM,
 * 9 down GEMM, 10 Stage-II misc (norms, gather), 11 lm_head. */
int pkv_timing_enable(int32_t on);
int pkv_timing_collect(double* ms, int32_t* counts, int32_t ncat);

const char* pkv_last_error(void);
uint64_t pkv_launch_count(void);
int pkv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PKV_H_ */
