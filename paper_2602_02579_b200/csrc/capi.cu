// C-ABI entry points (include/pkv.h): validation, workspace carving and the
// per-layer launch sequences of the three stages.  The host loop lives here (C++),
// so Python makes one call per stage.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.cuh"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

struct pkv_model {
  pkv_config cfg;       // the full model
  int dkp, Dp, Fp, NQKV, HQ;
  int H, Hkv, F;        // this rank's query heads, KV heads and ffn width (== cfg when unsharded);
                        // Fp, NQKV and HQ above are the local padded sizes
  int tp_rank = 0, tp_world = 1;
  pkv_comm* comm = nullptr;
  pkv_weights w;
  std::vector<pkv_layer_weights> layers;
};

namespace pkv {

// ---- error state / bookkeeping
static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// PDL is off by default: measured neutral without an early trigger and ~3% slower with
// one (dependents parked on busy SMs); PKV_PDL=1 enables it
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PKV_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

// ---- workspace carving
struct Carver {
  uint8_t* base;
  size_t off = 0, cap;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += n * sizeof(T);
    return p;
  }
};

static int layout_of(const pkv_config* c, int out[5]) {
  if (c->n_layers <= 0 || c->n_heads <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0 || c->ffn_dim <= 0 ||
      c->vocab_size <= 0)
    return set_error(PKV_ERR_CONFIG, "all model dimensions must be positive");
  if (c->n_heads % c->n_kv_heads != 0) return set_error(PKV_ERR_CONFIG, "n_heads not divisible by n_kv_heads");
  if (c->hidden_dim != c->n_heads * c->head_dim) return set_error(PKV_ERR_CONFIG, "hidden_dim != n_heads*head_dim");
  if (c->head_dim % 2 != 0) return set_error(PKV_ERR_CONFIG, "head_dim must be even");
  if (!(c->rope_theta > 0) || !(c->norm_eps > 0)) return set_error(PKV_ERR_CONFIG, "rope_theta/norm_eps must be > 0");
  if (c->head_dim > 128) return set_error(PKV_ERR_CONFIG, "head_dim > 128 not supported by the sm_100a kernels");
  if (c->n_heads / c->n_kv_heads > 128) return set_error(PKV_ERR_CONFIG, "GQA group larger than 128");
  const int dkp = c->head_dim <= 64 ? 64 : 128;
  out[0] = dkp;
  out[1] = (c->hidden_dim + 63) / 64 * 64;
  out[2] = (c->ffn_dim + 127) / 128 * 128;
  out[3] = (c->n_heads + 2 * c->n_kv_heads) * dkp;
  out[4] = c->n_heads * dkp;
  return PKV_OK;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- native phase timers (pkv_timing_enable / pkv_timing_collect): CUDA events
// recorded on the launching stream around each kernel group when enabled.
enum TimerCat { T_ASSEMBLE = 0, T_QP_PROJ, T_QP_ATTN, T_QP_MISC, T_SELECT, T_RC_QKV, T_RC_ATTN, T_RC_O, T_RC_GU,
                T_RC_DOWN, T_RC_MISC, T_LMHEAD, T_COMM, T_NCAT };
struct TimerRec {
  int cat;
  cudaEvent_t a, b;
};
static std::mutex g_tm_mu;
static std::vector<TimerRec> g_tm;
static std::vector<cudaEvent_t> g_ev_pool;
static std::atomic<int> g_timing{0};

static cudaEvent_t ev_get() {
  std::lock_guard<std::mutex> lk(g_tm_mu);
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ScopedTimer {
  int cat;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ScopedTimer(int c, cudaStream_t s) : cat(c), st(s) {
    if (g_timing.load(std::memory_order_relaxed)) {
      a = ev_get();
      cudaEventRecord(a, st);
    }
  }
  ~ScopedTimer() {
    if (a) {
      cudaEvent_t b = ev_get();
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_tm_mu);
      g_tm.push_back({cat, a, b});
    }
  }
};
#define TTRY(cat, x)                     \
  do {                                   \
    ::pkv::ScopedTimer t__(cat, st);     \
    if ((rc = (x)) != 0) return rc;      \
  } while (0)

int mark_launch(const int32_t* idx, int n, uint8_t* flags, cudaStream_t st);


// fp32-faithful projection of m (<= any) fp32 rows: out[m][N] (=|+=) x[m][K] . W[N][K]^T
// via tcgen05 on the 3-way bf16 split of x, split-K partials and a reduce.
struct ProjWs {
  void* x3;        // bf16 [96][Kmax]
  long ldx;
  float* part;     // [8][Nmax][96]
  int* cnt;        // [Nmax/128] split-K arrival counters (EPI_PROJ)
};
// split-K count of a narrow-pass projection (N output features of K inputs, 128 x 64
// weight tiles streamed once): the persistent grid runs ceil(tiles / SMs) rounds of
// k_tiles/splits tiles each plus a fixed per-tile cost (pipeline fill + split fixup),
// so pick the split that minimises rounds * (k per split + overhead).
static int choose_splits(int N, int K) {
  const char* env = getenv("PKV_PROJ_SPLITS");  // tuning override
  const int forced = env ? atoi(env) : 0;
  const int m_tiles = ceil_div(N, 128 * gemm_mt(96, EPI_PROJ)), k_tiles = ceil_div(K, gemm_bk(96));
  if (forced > 0) return std::min(std::min(forced, 16), k_tiles);
  int best = 1;
  double best_cost = 1e30;
  for (int sp = 1; sp <= 16 && k_tiles / sp >= 2; ++sp) {
    const int per = ceil_div(k_tiles, sp);
    const int nsp = ceil_div(k_tiles, per);
    const int rounds = ceil_div((long)m_tiles * nsp, num_sms());
    const double cost = rounds * (per + 3.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = nsp;
    }
  }
  return best;
}
static int proj_f32(const void* W, float wsc, int N, int K, const float* x, long ldx_src, int m, float* out, long ldo,
                    int mode, const ProjWs& ws, cudaStream_t st) {
  for (int r0 = 0; r0 < m; r0 += 32) {
    const int rows = std::min(32, m - r0);
    int rc = split3_launch(x + (long)r0 * ldx_src, rows, K, ldx_src, ws.x3, ws.ldx, st);
    if (rc) return rc;
    GemmArgs g{};
    g.M = N;
    g.N = 96;
    const int sp = choose_splits(N, K);
    g.n_splits = sp;
    g.k_tiles_per_split = 0;  // gemm_tc_launch splits the k range evenly
    g.C = ws.part;
    g.ldc = 96;
    g.f16 = 1;
    g.acc_scale = wsc;
    rc = gemm_tc_launch(EPI_F32, 96, W, K, ws.x3, ws.ldx, K, g, st);
    if (rc) return rc;
    const int ktt = ceil_div(K, gemm_bk(96)), nsp = ceil_div(ktt, ceil_div(ktt, sp));  // as gemm_tc_launch
    rc = splitk_reduce_launch(ws.part, nsp, N, rows, out + (long)r0 * ldo, ldo, mode, st);
    if (rc) return rc;
  }
  return PKV_OK;
}

// m <= 32: the producer already wrote x's 3 bf16 planes into ws.x3; one GEMM launch sums
// the planes and the split-K partials (deterministically) and stores / accumulates out.
static int proj_fused(const void* W, float wsc, int N, int K, int m, float* out, long ldo, int resid, const ProjWs& ws,
                      cudaStream_t st) {
  GemmArgs g{};
  g.f16 = 1;
  g.acc_scale = wsc;
  g.M = N;
  g.N = 96;
  // stream-K (balanced k ranges over the whole grid) unless a split count is forced
  static const bool forced = getenv("PKV_PROJ_SPLITS") != nullptr;
  g.stream_k = forced ? 0 : 1;
  g.n_splits = forced ? choose_splits(N, K) : 1;
  g.k_tiles_per_split = 0;  // gemm_tc_launch splits the k range evenly
  g.out = out;
  g.ldo = ldo;
  g.mrows = m;
  g.resid = resid;
  g.part = ws.part;
  g.cnt = ws.cnt;
  return gemm_tc_launch(EPI_PROJ, 96, W, K, ws.x3, ws.ldx, K, g, st);
}

}  // namespace pkv

using namespace pkv;

extern "C" {

int pkv_version(void) { return 1; }

int pkv_timing_enable(int32_t on) {
  g_timing.store(on ? 1 : 0);
  return PKV_OK;
}

int pkv_timing_collect(double* ms, int32_t* counts, int32_t ncat) {
  std::vector<TimerRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_tm_mu);
    recs.swap(g_tm);
  }
  for (int i = 0; i < ncat; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  int rc = PKV_OK;
  for (auto& r : recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) rc = set_error(PKV_ERR_CUDA, "timer event failed");
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cat < ncat) {
      ms[r.cat] += t;
      counts[r.cat] += 1;
    }
  }
  std::lock_guard<std::mutex> lk(g_tm_mu);
  for (auto& r : recs) {
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  return rc;
}
const char* pkv_last_error(void) { return g_err; }
uint64_t pkv_launch_count(void) { return g_launches.load(); }

int pkv_layout(const pkv_config* cfg, int32_t out[5]) {
  int o[5];
  int rc = layout_of(cfg, o);
  if (rc) return rc;
  for (int i = 0; i < 5; ++i) out[i] = o[i];
  return PKV_OK;
}

int pkv_model_create_sharded(const pkv_config* cfg, const pkv_weights* w, int32_t tp_rank, int32_t tp_world,
                             pkv_comm* comm, pkv_model** out) {
  if (!cfg || !out) return set_error(PKV_ERR_ARGUMENT, "null argument");
  int o[5];
  int rc = layout_of(cfg, o);
  if (rc) return rc;
  if (!w || !w->layers || !w->embed || !w->lm_head || !w->final_norm)
    return set_error(PKV_ERR_ARGUMENT, "null weight pointer");
  if (tp_world < 1 || tp_rank < 0 || tp_rank >= tp_world) return set_error(PKV_ERR_ARGUMENT, "bad tp rank");
  if (tp_world > 1) {
    if (!comm) return set_error(PKV_ERR_ARGUMENT, "sharded model needs a communicator");
    if (comm_world(comm) != tp_world || comm_rank(comm) != tp_rank)
      return set_error(PKV_ERR_ARGUMENT, "communicator rank/size do not match the shard");
    if (cfg->n_kv_heads % tp_world != 0) return set_error(PKV_ERR_CONFIG, "n_kv_heads not divisible by tp size");
    if ((o[2] / 128) % tp_world != 0) return set_error(PKV_ERR_CONFIG, "ffn blocks not divisible by tp size");
  }
  pkv_model* m = new pkv_model();
  m->cfg = *cfg;
  m->dkp = o[0];
  m->Dp = o[1];
  m->H = cfg->n_heads / tp_world;
  m->Hkv = cfg->n_kv_heads / tp_world;
  m->Fp = o[2] / tp_world;
  m->F = tp_world == 1 ? cfg->ffn_dim : m->Fp;  // shards carry zero-padded columns, silu(0)*0 = 0
  m->NQKV = (m->H + 2 * m->Hkv) * m->dkp;
  m->HQ = m->H * m->dkp;
  m->tp_rank = tp_rank;
  m->tp_world = tp_world;
  m->comm = tp_world > 1 ? comm : nullptr;
  m->layers.assign(w->layers, w->layers + cfg->n_layers);
  for (auto& l : m->layers)
    if (!l.wqkv || !l.wo || !l.wgu || !l.wd || !l.attn_norm || !l.ffn_norm) {
      delete m;
      return set_error(PKV_ERR_ARGUMENT, "null layer weight pointer");
    }
  m->w = *w;
  m->w.layers = m->layers.data();
  *out = m;
  return PKV_OK;
}

int pkv_model_create(const pkv_config* cfg, const pkv_weights* w, pkv_model** out) {
  return pkv_model_create_sharded(cfg, w, 0, 1, nullptr, out);
}

void pkv_model_destroy(pkv_model* m) { delete m; }

int pkv_assemble_layers(const pkv_config* cfg, const pkv_chunks* ch, const pkv_cache* c, int32_t l0, int32_t l1,
                        void* stream) {
  if (!cfg || !ch || !c) return set_error(PKV_ERR_ARGUMENT, "null argument");
  int lay[5];
  int rc = layout_of(cfg, lay);
  if (rc) return rc;
  if (ch->n_chunks <= 0) return set_error(PKV_ERR_INPUT, "assemble needs at least one chunk");
  if (c->pool_tokens % 128 != 0 || c->pool_tokens < c->s) return set_error(PKV_ERR_SHAPE, "pool too small");
  if (c->rope_len < c->s) return set_error(PKV_ERR_SHAPE, "rope table shorter than the context");
  if (l0 < 0 || l1 > cfg->n_layers || l0 >= l1) return set_error(PKV_ERR_ARGUMENT, "bad layer range");
  ChunkView cv{ch->k_nr, ch->v, ch->src_chunk, ch->src_local, ch->chunk_len};
  cudaStream_t st = S(stream);
  if (c->recomputed && l0 == 0) cudaMemsetAsync(const_cast<uint8_t*>(c->recomputed), 0, (size_t)c->s, st);
  ScopedTimer t__(T_ASSEMBLE, st);
  return assemble_launch(cv, c->s, l0, l1, cfg->n_kv_heads, lay[0], cfg->head_dim, c->rope_cos, c->rope_sin,
                         c->page_table, c->k_pool, c->v_pool, c->pool_tokens, c->k2_pool, st);
}

int pkv_assemble(const pkv_config* cfg, const pkv_chunks* ch, const pkv_cache* c, void* stream) {
  if (!cfg) return set_error(PKV_ERR_ARGUMENT, "null argument");
  return pkv_assemble_layers(cfg, ch, c, 0, cfg->n_layers, stream);
}

int pkv_cache_view(const pkv_config* cfg, const pkv_cache* c, const pkv_chunks* ch, int32_t layer, int32_t is_key,
                   float* out, void* stream) {
  int lay[5];
  int rc = layout_of(cfg, lay);
  if (rc) return rc;
  if (layer < 0 || layer >= cfg->n_layers) return set_error(PKV_ERR_ARGUMENT, "layer out of range");
  ChunkView cv{};
  if (ch) cv = ChunkView{ch->k_nr, ch->v, ch->src_chunk, ch->src_local, ch->chunk_len};
  const void* pool = is_key ? c->k_pool : c->v_pool;
  return cache_view_launch(cv, ch != nullptr, c->s, layer, cfg->n_kv_heads, lay[0], cfg->head_dim, c->rope_cos,
                           c->rope_sin, c->page_table, pool, is_key ? c->k2_pool : nullptr, c->pool_tokens, is_key,
                           out, S(stream));
}

int pkv_probe_accum(const float* part, int32_t p0, int32_t n, double* colsum, void* stream) {
  if (!part || !colsum) return set_error(PKV_ERR_ARGUMENT, "null argument");
  if (p0 < 0 || n < 0) return set_error(PKV_ERR_ARGUMENT, "bad block");
  return probe_accum_launch(part, p0, n, colsum, S(stream));
}

int pkv_probe_scores(const pkv_config* cfg, const pkv_cache* c, const float* v1, const double* colsum, float* out,
                     void* stream) {
  if (!cfg || !c || !v1 || !out) return set_error(PKV_ERR_ARGUMENT, "null argument");
  int lay[5];
  int rc = layout_of(cfg, lay);
  if (rc) return rc;
  if (cfg->n_layers < 2) return set_error(PKV_ERR_ARGUMENT, "the probe scores need layer 1");
  const long layer_pool = (long)cfg->n_kv_heads * c->pool_tokens * lay[0];
  return probe_scores_launch(v1, reinterpret_cast<const __half*>(c->v_pool) + layer_pool, c->page_table,
                             c->pool_tokens, c->s, cfg->n_kv_heads, cfg->head_dim, lay[0], colsum, out, S(stream));
}

int pkv_replace_entries(const pkv_config* cfg, const pkv_cache* c, int32_t layer, const int32_t* idx, int32_t n,
                        const float* new_k, const float* new_v, void* stream) {
  int lay[5];
  int rc = layout_of(cfg, lay);
  if (rc) return rc;
  if (layer < 0 || layer >= cfg->n_layers) return set_error(PKV_ERR_ARGUMENT, "layer out of range");
  rc = scatter_launch(idx, n, layer, cfg->n_kv_heads, lay[0], cfg->head_dim, new_k, c->page_table, c->k_pool,
                      c->pool_tokens, c->k2_pool, S(stream));
  if (rc) return rc;
  if (c->recomputed && (rc = mark_launch(idx, n, const_cast<uint8_t*>(c->recomputed), S(stream))) != 0) return rc;
  return scatter_launch(idx, n, layer, cfg->n_kv_heads, lay[0], cfg->head_dim, new_v, c->page_table, c->v_pool,
                        c->pool_tokens, nullptr, S(stream));
}

// ------------------------------------------------------------------ query pass
struct QpWs {
  float *h, *x, *qkv, *q, *k, *v, *attn, *gu, *act, *S, *Opart, *Mpart, *Lpart, *Mfin, *Lfin, *rows, *xl;
  double* denom;
  double* rows64;  // tensor-parallel: per-(query, token) head-sum partials, all-reduced
  __half* q3;
  float *sc_w, *sc_c, *sc_part;  // scoring pass 2
  int sc_splits, sc_keys_per_split;
  ProjWs proj;
  int n_splits, keys_per_split, tc_splits, tc_keys_per_split;
};

static QpWs carve_qp(const pkv_model* md, int s, int m, int flags, void* base, size_t* total) {
  const int H = md->H, Hkv = md->Hkv, G = H / Hkv, dkp = md->dkp;
  const int R = m * G;
  const int s_tot = s + m;
  QpWs w{};
  Carver cv{reinterpret_cast<uint8_t*>(base), 0, 0};
  const long kmax = std::max({(long)md->Dp, (long)md->HQ, (long)md->Fp});
  const long nmax = std::max({(long)md->NQKV, (long)md->Dp, 2L * md->Fp});
  w.h = cv.take<float>((size_t)m * md->Dp);
  w.x = cv.take<float>((size_t)m * md->Dp);
  w.qkv = cv.take<float>((size_t)m * md->NQKV);
  w.q = cv.take<float>((size_t)m * H * dkp);
  w.k = cv.take<float>((size_t)m * Hkv * dkp);
  w.v = cv.take<float>((size_t)m * Hkv * dkp);
  w.attn = cv.take<float>((size_t)m * H * dkp);
  w.gu = cv.take<float>((size_t)m * 2 * md->Fp);
  w.act = cv.take<float>((size_t)m * md->Fp);
  w.proj.x3 = cv.take<__half>((size_t)96 * kmax);
  w.proj.ldx = kmax;
  w.proj.part = cv.take<float>((size_t)16 * nmax * 96);  // up to 16 split-K partials
  w.proj.cnt = cv.take<int>((size_t)ceil_div(nmax, 128));
  w.keys_per_split = 512;
  w.n_splits = ceil_div(s_tot, w.keys_per_split);
  {
    // tensor-core split of the context keys: one wave of (KV head x split) CTAs (measured
    // best of 1..4 waves; PKV_S1_WAVES overrides)
    static const bool simt_only = getenv("PKV_S1_SIMT") != nullptr;
    const int row_blocks = ceil_div(R, 128);
    static const int waves = getenv("PKV_S1_WAVES") ? std::max(1, atoi(getenv("PKV_S1_WAVES"))) : 1;
    int target = std::max(1, waves * num_sms() / std::max(1, Hkv * row_blocks));
    // the fused fresh-key split takes one CTA slot per (KV head, row block): keep the
    // launch inside one wave (152 CTAs on 148 SMs doubled the kernel's time)
    if (m <= 128 && target > 1 && !(getenv("PKV_FRESH_FUSED") && getenv("PKV_FRESH_FUSED")[0] == '1')) target -= 1;
    w.tc_keys_per_split = std::max(64, ceil_div(ceil_div(s, target), 64) * 64);
    w.tc_splits = (simt_only || s == 0) ? 0 : ceil_div(s, w.tc_keys_per_split);
    // partial buffers sized for either path (the caller's cache decides which runs)
    w.n_splits = std::max(w.n_splits, w.tc_splits + 1);
  }
  const int row_blocks = ceil_div(R, 128);
  (void)row_blocks;
  if (flags & (PKV_QP_SCORES | PKV_QP_ROWS)) {
    // the [Hkv][s][R] score matrix only for capture_attn rows, the SIMT path and the
    // head-sharded renormalised scores; otherwise the second pass reduces p per key
    const bool need_S = (flags & PKV_QP_ROWS) || w.tc_splits == 0 || ((flags & PKV_QP_RENORM) && md->tp_world > 1);
    if (need_S) w.S = cv.take<float>((size_t)Hkv * R * s_tot);
    if (w.tc_splits > 0 && s > 0) {
      const int target = std::max(1, num_sms() / std::max(1, Hkv * row_blocks));
      w.sc_keys_per_split = std::max(128, ceil_div(ceil_div(s, target), 128) * 128);
      w.sc_splits = ceil_div(s, w.sc_keys_per_split);
      w.sc_w = cv.take<float>((size_t)Hkv * R);
      w.sc_c = cv.take<float>((size_t)Hkv * R);
      w.sc_part = cv.take<float>((size_t)row_blocks * Hkv * s);
    }
    w.rows = cv.take<float>((size_t)m * s);
    w.denom = cv.take<double>((size_t)m);
    if (md->tp_world > 1) w.rows64 = cv.take<double>((size_t)m * s);
  }
  w.Opart = cv.take<float>((size_t)w.n_splits * Hkv * R * dkp);
  w.Mpart = cv.take<float>((size_t)w.n_splits * Hkv * R);
  w.Lpart = cv.take<float>((size_t)w.n_splits * Hkv * R);
  w.Mfin = cv.take<float>((size_t)Hkv * R);
  w.Lfin = cv.take<float>((size_t)Hkv * R);
  w.xl = cv.take<float>((size_t)md->Dp);
  w.q3 = cv.take<__half>((size_t)Hkv * ceil_div(R, 128) * 3 * 128 * dkp);
  *total = cv.off + 256;
  return w;
}

size_t pkv_query_pass_workspace(const pkv_model* m, int32_t s, int32_t n_query, int32_t flags) {
  size_t total = 0;
  carve_qp(m, s, n_query, flags, nullptr, &total);
  return total;
}

int pkv_query_pass(const pkv_model* md, const pkv_cache* c, const pkv_chunks* ch, const int32_t* query_ids,
                   int32_t m, int32_t flags, float* per_layer, float* fresh_k, float* fresh_v, float* last_logits,
                   void* workspace, size_t ws_bytes, void* stream) {
  if (!md || !c || !query_ids) return set_error(PKV_ERR_ARGUMENT, "null argument");
  if (m <= 0) return set_error(PKV_ERR_INPUT, "token sequence must be non-empty");
  const pkv_config& cf = md->cfg;
  const int s = c->s;
  if (c->rope_len < s + m) return set_error(PKV_ERR_SHAPE, "rope table shorter than context + query");
  if ((flags & PKV_QP_FROM_CHUNKS) && !ch) return set_error(PKV_ERR_ARGUMENT, "chunk view required");
  if ((flags & PKV_QP_APPEND_KV) && c->pool_tokens < s + m) return set_error(PKV_ERR_SHAPE, "pool too small to append");
  if ((flags & PKV_QP_ROWS) && (flags & (PKV_QP_SCORES | PKV_QP_PROBE)))
    return set_error(PKV_ERR_ARGUMENT, "PKV_QP_ROWS excludes PKV_QP_SCORES / PKV_QP_PROBE");
  size_t need = 0;
  QpWs w = carve_qp(md, s, m, flags, workspace, &need);
  if (ws_bytes < need) return set_error(PKV_ERR_ARGUMENT, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = S(stream);
  const int H = md->H, Hkv = md->Hkv, G = H / Hkv, dk = cf.head_dim, dkp = md->dkp;
  const int Dp = md->Dp, Fp = md->Fp;
  // row-parallel o / down projections: rank 0 adds its partial into the replicated
  // residual stream, the other ranks overwrite it with theirs, and the in-place sum
  // over ranks yields h + sum of partials everywhere
  const int resid = md->tp_rank == 0 ? 1 : 0;
  pkv_comm* comm = md->comm;
  int rc;
#define TRY(x)             \
  do {                     \
    if ((rc = (x)) != 0) return rc; \
  } while (0)
  TTRY(T_QP_MISC, embed_gather_launch(md->w.embed, Dp, query_ids, nullptr, m, cf.hidden_dim, w.h, Dp, st));
  // a head-slice view of a larger cache (pool_heads > 0): layer stride over all its heads,
  // this view's heads from head0
  const int HP = c->pool_heads > 0 ? c->pool_heads : Hkv, h0 = c->pool_heads > 0 ? c->head0 : 0;
  if (h0 < 0 || h0 + Hkv > HP) return set_error(PKV_ERR_ARGUMENT, "head slice [%d, %d) of %d heads", h0, h0 + Hkv, HP);
  if (c->pool_heads > 0 && (flags & (PKV_QP_PROBE | PKV_QP_ROWS)))
    return set_error(PKV_ERR_ARGUMENT, "probe / row capture passes need the whole cache");
  const long layer_pool = (long)HP * c->pool_tokens * dkp, head_off = (long)h0 * c->pool_tokens * dkp;
  // m <= 32: producers write the bf16 planes of the next GEMM input directly and the
  // projection epilogue reduces planes + split-K partials itself (one launch each)
  const bool fused = m <= 32;
  if (fused) cudaMemsetAsync(w.proj.cnt, 0, sizeof(int) * ceil_div(std::max({(long)md->NQKV, (long)Dp, 2L * Fp}), 128), st);
  void* x3 = fused ? w.proj.x3 : nullptr;
  const long ldx = w.proj.ldx;
  for (int l = 0; l < cf.n_layers; ++l) {
    const pkv_layer_weights& lw = md->layers[l];
    TTRY(T_QP_MISC, rmsnorm_launch(w.h, m, cf.hidden_dim, Dp, lw.attn_norm, cf.norm_eps, fused ? nullptr : w.x, x3,
                                   ldx, nullptr, st));
    if (fused) TTRY(T_QP_PROJ, proj_fused(lw.wqkv, lw.wscale[0], md->NQKV, Dp, m, w.qkv, md->NQKV, 0, w.proj, st));
    else TTRY(T_QP_PROJ, proj_f32(lw.wqkv, lw.wscale[0], md->NQKV, Dp, w.x, Dp, m, w.qkv, md->NQKV, 0, w.proj, st));
    __half* kp = reinterpret_cast<__half*>(c->k_pool) + l * layer_pool + head_off;
    __half* vp = reinterpret_cast<__half*>(c->v_pool) + l * layer_pool + head_off;
    const bool append = (flags & PKV_QP_APPEND_KV) != 0;
    const bool planes = c->k2_pool != nullptr;
    __half* k2p = planes ? reinterpret_cast<__half*>(c->k2_pool) + l * layer_pool + head_off : nullptr;
    // the tensor-core attention's Q planes straight from the RoPE kernel when no row block
    // needs zero padding
    const bool q3_fused = planes && w.tc_splits > 0 && (m * G) % 128 == 0 && !(flags & PKV_QP_PROBE);
    TTRY(T_QP_MISC, query_qkv_launch(w.qkv, m, H, Hkv, dk, dkp, s, c->rope_cos, c->rope_sin, w.q, w.k, w.v,
                                     append ? kp : nullptr, append ? vp : nullptr, c->pool_tokens, c->page_table,
                                     fresh_k ? fresh_k + (long)l * m * Hkv * dk : nullptr,
                                     fresh_v ? fresh_v + (long)l * m * Hkv * dk : nullptr, append ? k2p : nullptr,
                                     st, q3_fused ? w.q3 : nullptr));
    if ((flags & PKV_QP_PROBE) && l == 1) break;  // the probe only needs layer 1's fresh values
    if ((flags & PKV_QP_PROBE) && l == 0) {
      if (!planes) return set_error(PKV_ERR_ARGUMENT, "probe needs the cache's key plane");
      TTRY(T_QP_MISC, probe_cache_kv_launch(w.k, w.v, m, Hkv, dk, dkp, s, kp, k2p, vp, c->pool_tokens, c->page_table,
                                            st));
    }
    S1Attn a{};
    a.q = w.q;
    a.m = m;
    a.H = H;
    a.Hkv = Hkv;
    a.G = G;
    a.dk = dk;
    a.dkp = dkp;
    a.s = s;
    a.s_tot = s + m;
    a.R = m * G;
    const int tc_splits = planes ? w.tc_splits : 0;  // the tensor-core path needs the key plane
    a.keys_per_split = w.keys_per_split;
    a.n_splits = tc_splits > 0 ? 1 : ceil_div(s + m, w.keys_per_split);
    a.key_base = 0;
    a.split_base = 0;
    a.tc_splits = tc_splits;
    a.tc_keys_per_split = w.tc_keys_per_split;
    a.q3 = w.q3;
    a.q3_ready = q3_fused ? 1 : 0;
    a.k1_all = c->k_pool;
    a.k2_all = c->k2_pool;
    a.v_all = c->v_pool;
    a.pool_rows_total = (long)cf.n_layers * HP * c->pool_tokens;
    a.pool_heads = HP;
    a.head0 = h0;
    a.scale = (float)(1.0 / std::sqrt((double)dk));
    a.src_chunks = (flags & PKV_QP_FROM_CHUNKS) ? 1 : 0;
    a.recomp = c->recomputed;
    if (ch) {
      a.ck = ch->k_nr;
      a.cv = ch->v;
      a.src_chunk = ch->src_chunk;
      a.src_local = ch->src_local;
      a.chunk_len = ch->chunk_len;
    }
    a.rcos = c->rope_cos;
    a.rsin = c->rope_sin;
    a.k_pool = kp;
    a.v_pool = vp;
    a.k2_pool = k2p;
    a.pool_tokens = c->pool_tokens;
    a.page_table = c->page_table;
    a.layer = l;
    a.fk = w.k;
    a.fv = w.v;
    const bool scores = (flags & PKV_QP_SCORES) && per_layer;
    const bool capture = (flags & PKV_QP_ROWS) && per_layer;
    a.S = (scores || capture) ? w.S : nullptr;
    a.sc_w = w.sc_w;
    a.sc_c = w.sc_c;
    a.sc_part = (scores && tc_splits > 0) ? w.sc_part : nullptr;
    a.sc_splits = w.sc_splits;
    a.sc_keys_per_split = w.sc_keys_per_split;
    // pipelined transfer: layer l of the cache may still be in flight
    if (c->layer_ready != nullptr && c->layer_ready[l] != nullptr)
      cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(c->layer_ready[l]), 0);
    a.Opart = w.Opart;
    a.Mpart = w.Mpart;
    a.Lpart = w.Lpart;
    a.x3_out = x3;
    a.x3_ld = ldx;
    TTRY(T_QP_ATTN, s1_attention_launch(a, w.attn, w.Mfin, w.Lfin, w.rows, w.denom, scores ? per_layer + (long)l * s : nullptr,
                            (flags & PKV_QP_RENORM) ? 1 : 0, cf.n_heads, w.rows64, comm, st,
                            capture ? per_layer + (long)l * m * (s + m) : nullptr));
    if ((flags & PKV_QP_PROBE) && scores && l == 0)  // block keys' column sums after the context's
      TTRY(T_QP_MISC, probe_diag_colsum_launch(w.q, w.k, w.Mfin, w.Lfin, m, H, Hkv, dk, dkp, a.scale, per_layer + s, st));
    // without logits (score_prophet) the last layer's o-projection and MLP only feed a
    // residual stream nobody reads: the per-layer scores are complete here
    if (l == cf.n_layers - 1 && !(flags & PKV_QP_LOGITS)) break;
    if (fused) {
      TTRY(T_QP_PROJ, proj_fused(lw.wo, lw.wscale[1], Dp, md->HQ, m, w.h, Dp, resid, w.proj, st));
      if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h, (size_t)m * Dp, PKV_DT_F32, st));
      TTRY(T_QP_MISC, rmsnorm_launch(w.h, m, cf.hidden_dim, Dp, lw.ffn_norm, cf.norm_eps, nullptr, x3, ldx, nullptr, st));
      TTRY(T_QP_PROJ, proj_fused(lw.wgu, lw.wscale[2], 2 * Fp, Dp, m, w.gu, 2 * Fp, 0, w.proj, st));
      TTRY(T_QP_MISC, silu_act_launch(w.gu, m, md->F, Fp, nullptr, st, x3, ldx));
      TTRY(T_QP_PROJ, proj_fused(lw.wd, lw.wscale[3], Dp, Fp, m, w.h, Dp, resid, w.proj, st));
      if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h, (size_t)m * Dp, PKV_DT_F32, st));
    } else {
      TTRY(T_QP_PROJ, proj_f32(lw.wo, lw.wscale[1], Dp, md->HQ, w.attn, md->HQ, m, w.h, Dp, resid, w.proj, st));
      if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h, (size_t)m * Dp, PKV_DT_F32, st));
      TTRY(T_QP_MISC, rmsnorm_launch(w.h, m, cf.hidden_dim, Dp, lw.ffn_norm, cf.norm_eps, w.x, nullptr, 0, nullptr, st));
      TTRY(T_QP_PROJ, proj_f32(lw.wgu, lw.wscale[2], 2 * Fp, Dp, w.x, Dp, m, w.gu, 2 * Fp, 0, w.proj, st));
      TTRY(T_QP_MISC, silu_act_launch(w.gu, m, md->F, Fp, w.act, st));
      TTRY(T_QP_PROJ, proj_f32(lw.wd, lw.wscale[3], Dp, Fp, w.act, Fp, m, w.h, Dp, resid, w.proj, st));
      if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h, (size_t)m * Dp, PKV_DT_F32, st));
    }
  }
  if ((flags & PKV_QP_LOGITS) && last_logits) {
    TTRY(T_LMHEAD, rmsnorm_launch(w.h + (long)(m - 1) * Dp, 1, cf.hidden_dim, Dp, md->w.final_norm, cf.norm_eps, w.xl, nullptr, 0,
                       nullptr, st));
    TTRY(T_LMHEAD, gemv_launch(w.xl, md->w.lm_head, cf.vocab_size, Dp, Dp, last_logits, st));
  }
  return PKV_OK;
}

// ------------------------------------------------------------------- selection
size_t pkv_select_workspace(int32_t n_layers, int32_t s) { return ((size_t)s * 4 + 255) & ~size_t(255); }

int pkv_fuse_select(const float* per_layer, int32_t L, int32_t s, int32_t k, float* fused, int32_t* idx_out,
                    int32_t* status_out, void* workspace, size_t ws_bytes, void* stream) {
  if (k < 0 || k > s) return set_error(PKV_ERR_ARGUMENT, "k=%d outside [0, %d]", k, s);
  float* f = fused;
  if (!f) {
    if (ws_bytes < (size_t)s * 4) return set_error(PKV_ERR_ARGUMENT, "workspace too small");
    f = reinterpret_cast<float*>(workspace);
  }
  cudaStream_t st = S(stream);
  ScopedTimer t__(T_SELECT, st);
  int rc = fuse_layers_launch(per_layer, L, s, f, st);
  if (rc) return rc;
  return topk_launch(f, s, k, idx_out, status_out, st);
}

int pkv_topk(const float* scores, int32_t n, int32_t k, int32_t* idx_out, int32_t* status_out, void* stream) {
  if (k < 0 || k > n) return set_error(PKV_ERR_ARGUMENT, "k=%d outside [0, %d]", k, n);
  return topk_launch(scores, n, k, idx_out, status_out, S(stream));
}

// ------------------------------------------------------------------- recompute
struct RcWs {
  float* h;
  __half *xb, *qb, *ab, *act;  // fp16 GEMM / attention operands
  float* sk_part;  // stream-K tail pieces of the Stage-II GEMMs (shared: they run in order)
  int* sk_cnt;
  size_t sk_cnt_n;
  float* ssq;      // deferred RMSNorm: [k][ceil(Dp/256)] per-tile sums of h^2
  int* ticket;     // work ticket of the persistent attention (attn_ps_kernel)
};
static RcWs carve_rc(const pkv_model* md, int k, void* base, size_t* total) {
  Carver cv{reinterpret_cast<uint8_t*>(base), 0, 0};
  RcWs w{};
  w.h = cv.take<float>((size_t)k * md->Dp);
  w.xb = cv.take<__half>((size_t)k * md->Dp);
  w.qb = cv.take<__half>((size_t)k * md->HQ);
  w.ab = cv.take<__half>((size_t)k * md->HQ);
  w.act = cv.take<__half>((size_t)k * md->Fp);
  w.ssq = cv.take<float>((size_t)k * ceil_div(md->Dp, 256));
  w.ticket = cv.take<int>(1);
  const size_t skf = std::max(std::max(gemm_sk_ws_floats(k, md->NQKV, md->Dp), gemm_sk_ws_floats(k, md->Dp, md->HQ)),
                              std::max(gemm_sk_ws_floats(k, 2 * md->Fp, md->Dp), gemm_sk_ws_floats(k, md->Dp, md->Fp)));
  if (skf > 0) {
    w.sk_cnt_n = (size_t)2 * (num_sms() / 2);
    w.sk_cnt = cv.take<int>(w.sk_cnt_n);
    w.sk_part = cv.take<float>(skf);
  }
  *total = cv.off + 256;
  return w;
}

size_t pkv_recompute_workspace(const pkv_model* m, int32_t k) {
  size_t t = 0;
  carve_rc(m, k, nullptr, &t);
  return t;
}

// the Stage-II layer loop over the k rows `sel` (recompute_selected, and with sel = all
// positions full_prefill / precompute_chunk); leaves the final residual stream in w.h
// need_final_h = false: the last layer stops after its QKV projection + scatter.  Its
// attention / o / MLP only update the residual stream, which recompute_selected drops
// after the loop (reference recompute.py:57-82 returns the cache; the K/V writes are the
// only observable result), so that work is dead.  full_prefill keeps it for the logits.
//
// Query rows (q.m > 0, pkv_recompute_query): the m query tokens of finalize_query
// (reference recompute.py:105-125 -> model.py query_pass 370-402) ride along as rows
// k..k+m-1 at positions s..s+m-1.  Layer by layer they see exactly what the separate query
// pass would see -- the repaired layer (every selected entry written by this layer's QKV
// GEMM before its attention) plus their own causal K/V, appended to the pool -- so the
// final query pass disappears (it had to run after, or interleaved with, Stage II).  The
// last layer computes attention / o / MLP for the query rows only; then final norm and
// lm_head on the last query row.  (Stage-II precision: fp16 operands, fp32 accumulation
// and residual stream, instead of the fp32-faithful narrow pass.)
struct QueryRows {
  const int32_t* ids = nullptr;  // [m] device token ids
  int m = 0;
  int32_t* pos = nullptr;        // workspace [k + m]: sel, then s..s+m-1
  float* tap_k = nullptr;        // optional fp32 [L][m][Hkv][dk] fresh query K / V
  float* tap_v = nullptr;
  float* logits = nullptr;       // [vocab] first-token logits
  float* xl = nullptr;           // workspace [Dp]: normalised last row
};
// Token-parallel Stage II (pkv_recompute_rows): rank r of W repairs the 128/G-row attention
// units r, r+W, r+2W, ... of the selection with the full model; after each layer's QKV GEMM
// the ranks all-gather the fresh cache entries of their rows (fp16 K, K residual, V) and
// scatter the others' into their own pools, so every rank's attention reads the whole
// repaired layer and every rank ends with the identical repaired cache.
struct RowsMode {
  pkv_comm* comm = nullptr;           // null: off
  const int32_t* sel_global = nullptr;
  int k_global = 0, T = 32, kmax = 0;
  __half* kvc = nullptr;              // [kmax + m][3][Hkv][dkp] this rank's rows
  __half* recv = nullptr;             // [W][kmax][3][Hkv][dkp]
};
__host__ __device__ inline int rows_global(int j, int i, int W, int T) { return (j + W * (i / T)) * T + i % T; }
__global__ void rows_local_kernel(const int32_t* sel, int T, int W, int r, int kr, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kr) out[i] = sel[rows_global(r, i, W, T)];
}
__global__ void rows_scatter_kernel(const uint4* __restrict__ recv, int W, int kmax, int me, const int32_t* sel, int k,
                                    int T, int Hkv, int dkp, const int32_t* page_table, long pool_tokens, __half* kp,
                                    __half* k2p, __half* vp) {
  const int vpr = 3 * Hkv * dkp / 8;  // 16-byte vectors per row
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)W * kmax * vpr) return;
  const int j = (int)(gid / ((long)kmax * vpr));
  const long rem = gid - (long)j * kmax * vpr;
  const int i = (int)(rem / vpr), v = (int)(rem - (long)i * vpr);
  if (j == me) return;
  const int g = rows_global(j, i, W, T);
  if (g >= k) return;
  const int plane = v / (Hkv * dkp / 8), h = (v / (dkp / 8)) % Hkv, c = v % (dkp / 8);
  __half* base = plane == 0 ? kp : plane == 1 ? k2p : vp;
  if (base == nullptr) return;
  const int pos = sel[g];
  const long slot = (long)page_table[pos >> 7] * 128 + (pos & 127);
  reinterpret_cast<uint4*>(base + ((long)h * pool_tokens + slot) * dkp)[c] = recv[gid];
}
static void rows_counts(int k, int T, int W, int* kr) {  // rows per rank
  for (int j = 0; j < W; ++j) kr[j] = 0;
  for (int u = 0; u * T < k; ++u) kr[u % W] += std::min(T, k - u * T);
}

__global__ void iota_from_kernel(int32_t* v, int n, int base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = base + i;
}

static int recompute_core(const pkv_model* md, const pkv_cache* c, const int32_t* sel, int32_t k, float* tap_k,
                          float* tap_v, void* knr_out, void* v_out, const RcWs& w, cudaStream_t st,
                          bool need_final_h, const QueryRows& q = QueryRows(), const RowsMode& rows = RowsMode()) {
  const pkv_config& cf = md->cfg;
  const int H = md->H, Hkv = md->Hkv, dk = cf.head_dim, dkp = md->dkp, Dp = md->Dp, Fp = md->Fp;
  // row-parallel o / down GEMMs under tensor parallelism: rank 0 accumulates into the
  // residual stream, the others store their partial there; the sum restores h + sum
  const int epi_resid = md->tp_rank == 0 ? EPI_RESID : EPI_F32;
  pkv_comm* comm = md->comm;
  const long layer_pool = (long)Hkv * c->pool_tokens * dkp;
  int rc;
  const int m = q.m;
  const int n = k + m;  // rows of the layer loop
  const int32_t* pos = sel;
  if (m > 0) {  // positions of all rows: the selection, then the query at s..s+m-1
    cudaMemcpyAsync(q.pos, sel, sizeof(int32_t) * k, cudaMemcpyDeviceToDevice, st);
    iota_from_kernel<<<ceil_div(m, 128), 128, 0, st>>>(q.pos + k, m, c->s);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("iota_from_kernel");
    pos = q.pos;
  }
  // deferred RMSNorm (opt-in PKV_NORM_DEFER=1): the o / down GEMM epilogues (or,
  // head-sharded, a small pass after the all-reduce) write bf16(h * g) and per-tile sums of
  // h^2; the QKV / gate-up epilogues scale by 1/rms, so only layer 0's attention norm runs
  // as its own kernel.  Measured +1 ms per prefill (fp32 sums; +15 ms with f64 sums): the
  // extra epilogue stores compete with the mainloop's TMA fill, which costs more than the
  // 2 ms of standalone norm passes it removes.
  const bool defer = m == 0 && getenv("PKV_NORM_DEFER") && getenv("PKV_NORM_DEFER")[0] == '1';
  const int ntile = ceil_div(Dp, 256);
  auto consume = [&](GemmArgs& a) {
    a.ssq_in = w.ssq;
    a.ssq_n = ntile;
    a.ssq_ld = ntile;
    a.norm_D = cf.hidden_dim;
    a.norm_eps = (float)cf.norm_eps;
  };
  auto produce = [&](GemmArgs& a, const float* gain) {
    a.ng = gain;
    a.xg = w.xb;
    a.ldxg = Dp;
    a.ssq = w.ssq;
    a.ssq_ld = ntile;
  };
  if (w.sk_cnt) cudaMemsetAsync(w.sk_cnt, 0, w.sk_cnt_n * sizeof(int), st);
  TTRY(T_RC_MISC, embed_gather_launch(md->w.embed, Dp, c->token_ids, sel, k, cf.hidden_dim, w.h, Dp, st));
  if (m > 0)
    TTRY(T_RC_MISC, embed_gather_launch(md->w.embed, Dp, q.ids, nullptr, m, cf.hidden_dim, w.h + (long)k * Dp, Dp, st));
  for (int l = 0; l < cf.n_layers; ++l) {
    const pkv_layer_weights& lw = md->layers[l];
    const bool last = l == cf.n_layers - 1;
    // the scatter must land after this layer's (possibly pipelined) assembly
    if (c->layer_ready != nullptr && c->layer_ready[l] != nullptr)
      cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(c->layer_ready[l]), 0);
    // the repaired-entry flags: after layer 0's assembly, which clears them (a pipelined
    // host-tier assembly runs on another stream)
    if (l == 0 && c->recomputed)
      TTRY(T_RC_MISC, rows.comm ? mark_launch(rows.sel_global, rows.k_global, const_cast<uint8_t*>(c->recomputed), st)
                                : mark_launch(sel, k, const_cast<uint8_t*>(c->recomputed), st));
    if (l == 0 || !defer)
      TTRY(T_RC_MISC, rmsnorm_launch(w.h, n, cf.hidden_dim, Dp, lw.attn_norm, cf.norm_eps, nullptr, nullptr, 0, w.xb, st));
    GemmArgs g{};
    if (defer && l > 0) consume(g);
    g.f16 = 1;
    g.nonfinite = c->nonfinite;
    g.acc_scale = lw.wscale[0];
    g.sk_part = w.sk_part;
    g.sk_cnt = w.sk_cnt;
    g.M = n;
    g.N = md->NQKV;
    g.n_splits = 1;
    g.C = w.qb;
    g.ldc = md->HQ;
    g.pos = pos;
    g.rope_cos = c->rope_cos;
    g.rope_sin = c->rope_sin;
    g.rope_cs32 = reinterpret_cast<const float2*>(c->rope_cs32);
    g.head_dim = dk;
    g.dkp = dkp;
    g.n_heads = H;
    g.n_kv_heads = Hkv;
    g.k_pool = reinterpret_cast<__half*>(c->k_pool) + l * layer_pool;
    g.v_pool = reinterpret_cast<__half*>(c->v_pool) + l * layer_pool;
    g.pool_tokens = c->pool_tokens;
    g.page_table = c->page_table;
    g.tap_k = tap_k ? tap_k + (long)l * k * Hkv * dk : nullptr;
    g.tap_v = tap_v ? tap_v + (long)l * k * Hkv * dk : nullptr;
    if (m > 0) {
      g.tap_rows = k;
      g.qtap_k = q.tap_k ? q.tap_k + (long)l * m * Hkv * dk : nullptr;
      g.qtap_v = q.tap_v ? q.tap_v + (long)l * m * Hkv * dk : nullptr;
    }
    g.knr_out = knr_out ? reinterpret_cast<__nv_bfloat16*>(knr_out) + (long)l * k * Hkv * dkp : nullptr;
    g.vcap_out = v_out ? reinterpret_cast<__nv_bfloat16*>(v_out) + (long)l * k * Hkv * dkp : nullptr;
    if (c->k2_pool != nullptr) g.k2_pool = reinterpret_cast<__half*>(c->k2_pool) + l * layer_pool;
    g.kvc = rows.kvc;
    // K/V of every selected token are in the cache before this layer's attention.  The last
    // layer of a repair only scatters K/V (its attention / o / MLP are dead, below): skip
    // the query rows of wqkv.
    if (last && !need_final_h) {
      GemmArgs gq = g;  // (the query rows' own QKV, below)
      g.M = k;
      g.N = 2 * Hkv * dkp;
      g.head0 = H;
      TTRY(T_RC_QKV, gemm_tc_launch(EPI_QKV, 256, w.xb, Dp,
                                    reinterpret_cast<const __half*>(lw.wqkv) + (long)H * dkp * Dp, Dp, Dp, g,
                                    st));
      if (m > 0) {  // the query rows need their q as well: the full wqkv for those m rows only
        gq.M = m;
        gq.pos = pos + k;
        gq.C = w.qb + (long)k * md->HQ;
        gq.tap_k = gq.tap_v = nullptr;
        gq.tap_rows = 0;
        gq.kvc = nullptr;  // (replicated on every rank: not exchanged)
        TTRY(T_RC_QKV, gemm_tc_launch(EPI_QKV, 256, w.xb + (long)k * Dp, Dp, lw.wqkv, Dp, Dp, gq, st));
      }
    } else {
      TTRY(T_RC_QKV, gemm_tc_launch(EPI_QKV, 256, w.xb, Dp, lw.wqkv, Dp, Dp, g, st));
    }
    if (rows.comm) {  // every rank's fresh entries of this layer into every pool
      const size_t bytes = (size_t)rows.kmax * 3 * Hkv * dkp * sizeof(__half);
      TTRY(T_COMM, comm_allgather(rows.comm, rows.kvc, rows.recv, bytes, st));
      const int W = comm_world(rows.comm);
      const long nvec = (long)W * rows.kmax * 3 * Hkv * dkp / 8;
      if (nvec > 0) {
        rows_scatter_kernel<<<ceil_div(nvec, 256), 256, 0, st>>>(
            reinterpret_cast<const uint4*>(rows.recv), W, rows.kmax, comm_rank(rows.comm), rows.sel_global,
            rows.k_global, rows.T, Hkv, dkp, c->page_table, c->pool_tokens, g.k_pool, g.k2_pool, g.v_pool);
        PKV_LAUNCHED();
        PKV_CHECK_LAUNCH("rows_scatter_kernel");
      }
    }
    if (c->layer_done != nullptr && c->layer_done[l] != nullptr)
      cudaEventRecord(reinterpret_cast<cudaEvent_t>(c->layer_done[l]), st);
    if (last && !need_final_h && m == 0) break;
    // rows [r0, n) continue: all of them, or on the last layer of a repair with query rows
    // only the query rows (the selected rows' last attention / o / MLP are dead)
    const int r0 = (last && !need_final_h) ? k : 0, nr = n - r0;
    TTRY(T_RC_ATTN, attn_tc_launch(w.qb + (long)r0 * md->HQ, w.ab + (long)r0 * md->HQ, pos + r0, nr, H, Hkv, dk, dkp,
                                   c->k_pool, c->v_pool, (long)cf.n_layers * Hkv * c->pool_tokens, c->pool_tokens, l,
                                   c->page_table, st, w.ticket));
    GemmArgs go{};
    go.f16 = 1;
    go.nonfinite = c->nonfinite;
    go.acc_scale = lw.wscale[1];
    go.sk_part = w.sk_part;
    go.sk_cnt = w.sk_cnt;
    go.M = nr;
    go.N = Dp;
    go.n_splits = 1;
    go.C = w.h + (long)r0 * Dp;
    go.ldc = Dp;
    if (defer && !comm) produce(go, lw.ffn_norm);
    TTRY(T_RC_O, gemm_tc_launch(epi_resid, 256, w.ab + (long)r0 * md->HQ, md->HQ, lw.wo, md->HQ, md->HQ, go, st));
    if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h + (long)r0 * Dp, (size_t)nr * Dp, PKV_DT_F32, st));
    if (!defer)
      TTRY(T_RC_MISC, rmsnorm_launch(w.h + (long)r0 * Dp, nr, cf.hidden_dim, Dp, lw.ffn_norm, cf.norm_eps, nullptr,
                                     nullptr, 0, w.xb + (long)r0 * Dp, st));
    else if (comm)
      TTRY(T_RC_MISC, norm_defer_launch(w.h, n, Dp, Dp, lw.ffn_norm, w.xb, Dp, w.ssq, ntile, st));
    GemmArgs gg{};
    gg.f16 = 1;
    gg.nonfinite = c->nonfinite;
    gg.acc_scale = lw.wscale[2];
    gg.sk_part = w.sk_part;
    gg.sk_cnt = w.sk_cnt;
    gg.M = nr;
    gg.N = 2 * Fp;
    gg.n_splits = 1;
    gg.C = w.act + (long)r0 * Fp;
    gg.ldc = Fp;
    if (defer) consume(gg);
    TTRY(T_RC_GU, gemm_tc_launch(EPI_SILU, 256, w.xb + (long)r0 * Dp, Dp, lw.wgu, Dp, Dp, gg, st));
    GemmArgs gd{};
    gd.f16 = 1;
    gd.nonfinite = c->nonfinite;
    gd.acc_scale = lw.wscale[3];
    gd.sk_part = w.sk_part;
    gd.sk_cnt = w.sk_cnt;
    gd.M = nr;
    gd.N = Dp;
    gd.n_splits = 1;
    gd.C = w.h + (long)r0 * Dp;
    gd.ldc = Dp;
    const float* next_norm = l + 1 < cf.n_layers ? md->layers[l + 1].attn_norm : nullptr;
    if (defer && !comm && next_norm) produce(gd, next_norm);
    TTRY(T_RC_DOWN, gemm_tc_launch(epi_resid, 256, w.act + (long)r0 * Fp, Fp, lw.wd, Fp, Fp, gd, st));
    if (comm) TTRY(T_COMM, comm_allreduce(comm, w.h + (long)r0 * Dp, (size_t)nr * Dp, PKV_DT_F32, st));
    if (defer && comm && next_norm)
      TTRY(T_RC_MISC, norm_defer_launch(w.h, n, Dp, Dp, next_norm, w.xb, Dp, w.ssq, ntile, st));
  }
  if (m > 0 && q.logits != nullptr) {  // _head_logits (model.py:326-329) of the last query row
    TTRY(T_LMHEAD, rmsnorm_launch(w.h + (long)(n - 1) * Dp, 1, cf.hidden_dim, Dp, md->w.final_norm, cf.norm_eps, q.xl,
                                  nullptr, 0, nullptr, st));
    TTRY(T_LMHEAD, gemv_launch(q.xl, md->w.lm_head, cf.vocab_size, Dp, Dp, q.logits, st));
  }
  return PKV_OK;
}

int pkv_recompute(const pkv_model* md, const pkv_cache* c, const int32_t* sel, int32_t k, float* tap_k, float* tap_v,
                  void* workspace, size_t ws_bytes, void* stream) {
  if (k == 0) return PKV_OK;
  if (k < 0 || k > c->s) return set_error(PKV_ERR_ARGUMENT, "bad selection size %d", k);
  size_t need = 0;
  RcWs w = carve_rc(md, k, workspace, &need);
  if (ws_bytes < need) return set_error(PKV_ERR_ARGUMENT, "workspace too small (%zu < %zu)", ws_bytes, need);
  return recompute_core(md, c, sel, k, tap_k, tap_v, nullptr, nullptr, w, S(stream), /*need_final_h=*/false);
}

size_t pkv_recompute_query_workspace(const pkv_model* md, int32_t k, int32_t m) {
  size_t t = 0;
  carve_rc(md, k + m, nullptr, &t);
  return t + ((size_t)(k + m) * sizeof(int32_t) + 255) / 256 * 256 + ((size_t)md->Dp * sizeof(float) + 255) / 256 * 256;
}

int pkv_recompute_query(const pkv_model* md, const pkv_cache* c, const int32_t* sel, int32_t k,
                        const int32_t* query_ids, int32_t m, float* tap_k, float* tap_v, float* query_k,
                        float* query_v, float* last_logits, void* workspace, size_t ws_bytes, void* stream) {
  if (!md || !c || !sel || !query_ids || !last_logits) return set_error(PKV_ERR_ARGUMENT, "null argument");
  if (k < 0 || k > c->s) return set_error(PKV_ERR_ARGUMENT, "bad selection size %d", k);
  if (m <= 0) return set_error(PKV_ERR_INPUT, "token sequence must be non-empty");
  if (c->pool_tokens < c->s + m || c->rope_len < c->s + m) return set_error(PKV_ERR_SHAPE, "pool too small to append");
  if (ws_bytes < pkv_recompute_query_workspace(md, k, m))
    return set_error(PKV_ERR_ARGUMENT, "workspace too small");
  size_t used = 0;
  RcWs w = carve_rc(md, k + m, workspace, &used);
  uint8_t* tail = reinterpret_cast<uint8_t*>(workspace) + used;
  QueryRows q;
  q.ids = query_ids;
  q.m = m;
  q.pos = reinterpret_cast<int32_t*>(tail);
  q.xl = reinterpret_cast<float*>(tail + ((size_t)(k + m) * sizeof(int32_t) + 255) / 256 * 256);
  q.tap_k = query_k;
  q.tap_v = query_v;
  q.logits = last_logits;
  return recompute_core(md, c, sel, k, tap_k, tap_v, nullptr, nullptr, w, S(stream), /*need_final_h=*/false, q);
}

// token-parallel workspace: Stage-II buffers for kmax + m rows, positions, the normalised
// last row, the local selection, this rank's compact entries and the gathered ones
static size_t rows_ws(const pkv_model* md, int k, int m, int world, RcWs* w, QueryRows* q, RowsMode* rm,
                      int32_t** local, void* base) {
  const int G = md->H / md->Hkv, T = std::max(1, 128 / std::max(1, G));
  std::vector<int> kr(std::max(1, world));
  rows_counts(k, T, std::max(1, world), kr.data());
  const int kmax = *std::max_element(kr.begin(), kr.end());
  size_t used = 0;
  RcWs ww = carve_rc(md, kmax + m, base, &used);
  Carver cv{reinterpret_cast<uint8_t*>(base), used, 0};
  int32_t* pos = cv.take<int32_t>((size_t)kmax + m);
  float* xl = cv.take<float>((size_t)md->Dp);
  int32_t* loc = cv.take<int32_t>((size_t)std::max(kmax, 1));
  const size_t row_elems = (size_t)3 * md->Hkv * md->dkp;
  __half* kvc = cv.take<__half>((size_t)(kmax + m) * row_elems);
  __half* recv = cv.take<__half>((size_t)std::max(1, world) * kmax * row_elems);
  if (w) *w = ww;
  if (q) {
    q->pos = pos;
    q->xl = xl;
  }
  if (rm) {
    rm->T = T;
    rm->kmax = kmax;
    rm->kvc = kvc;
    rm->recv = recv;
  }
  if (local) *local = loc;
  return cv.off + 256;
}

size_t pkv_recompute_rows_workspace(const pkv_model* md, int32_t k, int32_t m, int32_t world) {
  return rows_ws(md, k, m, world, nullptr, nullptr, nullptr, nullptr, nullptr);
}

int pkv_recompute_rows(const pkv_model* md, const pkv_cache* c, const int32_t* sel, int32_t k,
                       const int32_t* query_ids, int32_t m, pkv_comm* comm, float* last_logits, void* workspace,
                       size_t ws_bytes, void* stream) {
  if (!md || !c || !sel) return set_error(PKV_ERR_ARGUMENT, "null argument");
  if (md->tp_world != 1) return set_error(PKV_ERR_ARGUMENT, "token-parallel Stage II needs the unsharded model");
  if (k < 0 || k > c->s) return set_error(PKV_ERR_ARGUMENT, "bad selection size %d", k);
  if (m < 0 || (m > 0 && (!query_ids || !last_logits))) return set_error(PKV_ERR_ARGUMENT, "query rows");
  if (m > 0 && (c->pool_tokens < c->s + m || c->rope_len < c->s + m))
    return set_error(PKV_ERR_SHAPE, "pool too small to append");
  const int W = comm_world(comm), r = comm_rank(comm);
  if (ws_bytes < pkv_recompute_rows_workspace(md, k, m, W)) return set_error(PKV_ERR_ARGUMENT, "workspace too small");
  RcWs w;
  QueryRows q;
  RowsMode rm;
  int32_t* local = nullptr;
  rows_ws(md, k, m, W, &w, &q, &rm, &local, workspace);
  std::vector<int> kr(W);
  rows_counts(k, rm.T, W, kr.data());
  cudaStream_t st = S(stream);
  if (kr[r] > 0) {
    rows_local_kernel<<<ceil_div(kr[r], 128), 128, 0, st>>>(sel, rm.T, W, r, kr[r], local);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("rows_local_kernel");
  }
  rm.comm = comm;
  rm.sel_global = sel;
  rm.k_global = k;
  q.ids = query_ids;
  q.m = m;
  q.logits = last_logits;
  return recompute_core(md, c, local, kr[r], nullptr, nullptr, nullptr, nullptr, w, st, /*need_final_h=*/false, q, rm);
}

// ------------------------------------------------------------------ full prefill
__global__ void iota_kernel(int32_t* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

static size_t full_ws(const pkv_model* md, int n, RcWs* w, int32_t** sel, __nv_bfloat16** xl, void* base) {
  // xl: the final-normed rows in bf16, the A operand of the bf16 lm_head GEMM
  size_t rc_bytes = 0;
  carve_rc(md, n, nullptr, &rc_bytes);
  Carver cv{reinterpret_cast<uint8_t*>(base), 0, 0};
  uint8_t* rc_base = cv.take<uint8_t>(rc_bytes);
  *sel = cv.take<int32_t>((size_t)n);
  *xl = cv.take<__nv_bfloat16>((size_t)n * md->Dp);
  if (base) {
    size_t t = 0;
    *w = carve_rc(md, n, rc_base, &t);
  }
  return cv.off + 256;
}

size_t pkv_full_prefill_workspace(const pkv_model* m, int32_t n) {
  RcWs w{};
  int32_t* sel;
  __nv_bfloat16* xl;
  return full_ws(m, n, &w, &sel, &xl, nullptr);
}

int pkv_full_prefill(const pkv_model* md, const pkv_cache* c, void* k_nr_out, void* v_out, float* logits_out,
                     void* workspace, size_t ws_bytes, void* stream) {
  if (!md || !c) return set_error(PKV_ERR_ARGUMENT, "null argument");
  const int n = c->s;
  if (n <= 0) return set_error(PKV_ERR_INPUT, "token sequence must be non-empty");
  if (c->rope_len < n || c->pool_tokens < n) return set_error(PKV_ERR_SHAPE, "cache too small for the sequence");
  RcWs w{};
  int32_t* sel;
  __nv_bfloat16* xl;
  if (ws_bytes < full_ws(md, n, &w, &sel, &xl, nullptr))
    return set_error(PKV_ERR_ARGUMENT, "workspace too small");
  full_ws(md, n, &w, &sel, &xl, workspace);
  cudaStream_t st = S(stream);
  iota_kernel<<<ceil_div(n, 256), 256, 0, st>>>(sel, n);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("iota_kernel");
  int rc = recompute_core(md, c, sel, n, nullptr, nullptr, k_nr_out, v_out, w, st, logits_out != nullptr);
  if (rc) return rc;
  if (logits_out) {  // _head_logits (model.py:326-329) for every row: final norm, then lm_head
    const pkv_config& cf = md->cfg;
    TTRY(T_LMHEAD, rmsnorm_launch(w.h, n, cf.hidden_dim, md->Dp, md->w.final_norm, cf.norm_eps, nullptr, nullptr, 0,
                                  xl, st, /*y16_bf16=*/1));
    GemmArgs g{};
    g.M = n;
    g.N = cf.vocab_size;
    g.n_splits = 1;
    g.C = logits_out;
    g.ldc = cf.vocab_size;
    TTRY(T_LMHEAD, gemm_tc_launch(EPI_F32, 256, xl, md->Dp, md->w.lm_head, md->Dp, md->Dp, g, st));
  }
  return PKV_OK;
}

// ------------------------------------------------------------------ unit entry
int pkv_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M, int32_t N, int32_t K, float* C,
                  int64_t ldc, int32_t bn, int32_t epi, void* stream) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.n_splits = 1;
  g.C = C;
  g.ldc = ldc;
  g.f16 = (epi & 0x100) ? 1 : 0;  // 0x100: fp16 operands
  epi &= 0xff;
  if (epi != EPI_F32 && epi != EPI_RESID && epi != EPI_BF16) return set_error(PKV_ERR_ARGUMENT, "epilogue");
  // the stream-K tail needs piece storage: a per-device scratch grown on demand (unit
  // tests / microbenchmarks only; the prefill path carves it from its workspace)
  static float* sk_part[64] = {};
  static int* sk_cnt[64] = {};
  static size_t sk_cap[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = gemm_sk_ws_floats(M, N, K);
  if (need > 0 && dev < 64) {
    if (need > sk_cap[dev]) {
      if (sk_part[dev]) cudaFree(sk_part[dev]);
      if (!sk_cnt[dev]) {
        if (cudaMalloc(&sk_cnt[dev], 1024 * sizeof(int)) != cudaSuccess) return set_error(PKV_ERR_CUDA, "sk alloc");
        cudaMemset(sk_cnt[dev], 0, 1024 * sizeof(int));
      }
      if (cudaMalloc(&sk_part[dev], need * sizeof(float)) != cudaSuccess) return set_error(PKV_ERR_CUDA, "sk alloc");
      sk_cap[dev] = need;
    }
    g.sk_part = sk_part[dev];
    g.sk_cnt = sk_cnt[dev];
  }
  return gemm_tc_launch(epi, bn, A, lda, B, ldb, K, g, S(stream));
}

int pkv_proj_narrow(const void* W, int32_t N, int32_t K, const void* x3, int64_t ldx, int32_t m, float* out,
                    int64_t ldo, int32_t resid, float* part, int32_t* cnt, int32_t n_splits, void* stream) {
  if (m <= 0 || m > 32) return set_error(PKV_ERR_ARGUMENT, "narrow projection takes 1..32 rows");
  if (K % 64 != 0 || ldx < K) return set_error(PKV_ERR_SHAPE, "narrow projection: K must be a multiple of 64");
  GemmArgs g{};
  g.M = N;
  g.N = 96;
  // n_splits > 0: split-K with that many splits; 0: stream-K on the default grid;
  // < 0: stream-K on a grid of -n_splits CTAs (tuning)
  g.stream_k = n_splits > 0 ? 0 : (n_splits < 0 ? -n_splits : 1);
  g.n_splits = n_splits > 0 ? std::min(n_splits, 16) : 1;
  g.k_tiles_per_split = 0;  // gemm_tc_launch splits the k range evenly
  g.out = out;
  g.ldo = ldo;
  g.mrows = m;
  g.resid = resid;
  g.part = part;
  g.cnt = cnt;
  g.f16 = 1;
  return gemm_tc_launch(EPI_PROJ, 96, W, K, x3, ldx, K, g, S(stream));
}

int pkv_attention_sparse(const pkv_model* md, const pkv_cache* c, int32_t layer, const void* q, void* out,
                         const int32_t* pos, int32_t n_q, void* stream) {
  const pkv_config& cf = md->cfg;
  return attn_tc_launch(q, out, pos, n_q, md->H, md->Hkv, cf.head_dim, md->dkp, c->k_pool, c->v_pool,
                        (long)cf.n_layers * md->Hkv * c->pool_tokens, c->pool_tokens, layer, c->page_table,
                        S(stream));
}

}  // extern "C"
