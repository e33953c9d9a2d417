// Host side of the tcgen05 GEMM: TMA descriptor encoding (cached per buffer) and
// launch dispatch over (BN, epilogue).
#include <mutex>
#include <unordered_map>

#include "gemm_tc.cuh"

namespace pkv {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// row-major 16-bit (bf16 or fp16: TMA moves bytes) matrix [rows][cols] with the given row stride; box = box_rows x box_cols,
// 128-byte swizzle (box_cols must be 64). Out-of-range rows/cols read as zero.
bool make_tmap_2d(CUtensorMap* map, const void* base, long rows, long cols, long row_stride_elems, int box_rows,
                  int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
struct MapKey {
  const void* p;
  long rows, cols, stride;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && stride == o.stride && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.p);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull;
    h ^= (size_t)k.cols * 0xC2B2AE3D27D4EB4Full + (size_t)k.stride * 31 + (size_t)k.box_rows;
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;
}  // namespace

bool cached_tmap(CUtensorMap* out, const void* base, long rows, long cols, long stride, int box_rows) {
  MapKey key{base, rows, cols, stride, box_rows};
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) {
    *out = it->second;
    return true;
  }
  if (g_maps.size() > 4096) g_maps.clear();
  if (!make_tmap_2d(out, base, rows, cols, stride, box_rows, 64)) return false;
  g_maps.emplace(key, *out);
  return true;
}

template <int BN, int EPI, int CG = 1>
static int launch_one(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t stream) {
  using Cfg = GemmCfg<BN, EPI, CG>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (attr_err != cudaSuccess) return set_error(PKV_ERR_CUDA, "gemm smem attr: %s", cudaGetErrorString(attr_err));
  long tiles = (long)ceil_div(args.M, Cfg::BMT) * ceil_div(args.N, BN) * args.n_splits;
  if (tiles <= 0) return PKV_OK;
  if constexpr (CG == 2) {  // persistent CTA pairs, one cluster of 2 per TPC
    const int pairs = (int)std::min<long>(tiles, num_sms() / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(192);
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
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, EPI, CG>, ta, tb, args);
    PKV_LAUNCHED();
    PKV_CHECK_LAUNCH("gemm_tc_kernel (CTA pairs)");
    return PKV_OK;
  }
  int grid = (int)std::min<long>(tiles, num_sms());
  if (EPI == EPI_PROJ && CG == 1 && args.stream_k) grid = args.stream_k;  // stream-K grid (see gemm_tc_launch)
  launch_k(gemm_tc_kernel<BN, EPI, CG>, grid, 192, Cfg::SMEM, stream, ta, tb, args);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("gemm_tc_kernel");
  return PKV_OK;
}

// narrow projection with split-K over a cluster of n_splits CTAs (DSMEM reduction)
static int launch_proj_cluster(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args,
                               cudaStream_t stream) {
  using Cfg = GemmCfg<96, EPI_PROJ, 1>;
  auto kern = gemm_tc_kernel<96, EPI_PROJ, 1, 1>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  });
  if (attr_err != cudaSuccess) return set_error(PKV_ERR_CUDA, "gemm smem attr: %s", cudaGetErrorString(attr_err));
  const int tiles_m = ceil_div(args.M, Cfg::BMT);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles_m * args.n_splits);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = args.n_splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, ta, tb, args);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("gemm_tc_kernel (cluster split-K)");
  return PKV_OK;
}

// Debug: PKV_GEMM_TRACE=1 makes the narrow projection stamp %globaltimer per CTA
// (kernel entry, prologue done, accumulator ready, partial stored, counter acquired,
// reduced, written) into a static buffer read back by pkv_debug_gemm_trace.
static unsigned long long* g_trace = nullptr;
static constexpr int kTraceCtas = 1024;
static unsigned long long* gemm_trace_buffer() {
  static const bool on = getenv("PKV_GEMM_TRACE") && getenv("PKV_GEMM_TRACE")[0] == '1';
  if (!on) return nullptr;
  if (g_trace == nullptr) {
    if (cudaMalloc(&g_trace, kTraceCtas * 8 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(g_trace, 0, kTraceCtas * 8 * sizeof(unsigned long long));
  }
  return g_trace;
}

int gemm_sk_plan(int M, int N, int K, int* rem_out, int* maxp_out) {
  // opt-in (PKV_GEMM_SK=1): correct and deterministic, but measured 2-4 % slower on the
  // qkv / o shapes and neutral on gate_up / down (tools/bench_stage2_gemm.py): under the
  // power cap a partial last wave runs at higher clocks, so the tail costs less than its
  // tile count suggests, and the pieces lose the cross-pair B-tile sharing in L2
  static const bool off = !(getenv("PKV_GEMM_SK") && getenv("PKV_GEMM_SK")[0] == '1');
  *rem_out = 0;
  *maxp_out = 0;
  if (off || M <= 0 || N <= 0) return 0;
  const int P = num_sms() / 2;
  const long tiles = (long)ceil_div(M, 256) * ceil_div(N, 256);
  const int kt = ceil_div(K, 64);
  if (P <= 0 || tiles < P || kt < 8) return 0;
  const int rem = (int)(tiles % P);
  if (rem == 0) return 0;
  const long U = (long)rem * kt;
  // <= 4 tail tiles' worth of pairs per tile keeps pieces >= kt/4 deep
  const int skp = (int)std::min<long>(P, std::min<long>(4L * rem, U));
  auto start = [&](int c) { return (long)c * U / skp; };
  auto owner = [&](long u) {
    int c = (int)((u * skp) / U);
    if (c >= skp) c = skp - 1;
    while (c + 1 < skp && start(c + 1) <= u) ++c;
    while (c > 0 && start(c) > u) --c;
    return c;
  };
  int maxp = 0;
  for (int sl = 0; sl < rem; ++sl) maxp = std::max(maxp, owner((long)sl * kt + kt - 1) - owner((long)sl * kt) + 1);
  if (maxp > SK_MAXP) return 0;
  *rem_out = rem;
  *maxp_out = maxp;
  return skp;
}

size_t gemm_sk_ws_floats(int M, int N, int K) {
  int rem, maxp;
  if (!gemm_sk_plan(M, N, K, &rem, &maxp)) return 0;
  return (size_t)rem * maxp * 2 * 256 * 128;
}

// A: [M][K], B: [N][K], both bf16 or both fp16 (args.f16), row strides lda / ldb elements.
int gemm_tc_launch(int epi, int bn, const void* A, long lda, const void* B, long ldb, int K, GemmArgs args,
                   cudaStream_t stream) {
  if (args.M <= 0 || args.N <= 0) return PKV_OK;
  if (K <= 0) return set_error(PKV_ERR_SHAPE, "gemm: K must be positive");
  if ((lda * 2) % 16 != 0 || (ldb * 2) % 16 != 0)
    return set_error(PKV_ERR_SHAPE, "gemm: row strides must be multiples of 8 elements");
  args.K = K;
  if (args.acc_scale == 0.f) args.acc_scale = 1.f;  // value-initialised GemmArgs: unscaled
  int kt = ceil_div(K, gemm_bk(bn));
  if (args.n_splits <= 0) args.n_splits = 1;
  if (args.k_tiles_per_split <= 0) args.k_tiles_per_split = ceil_div(kt, args.n_splits);
  args.n_splits = ceil_div(kt, args.k_tiles_per_split);  // no empty splits
  if (epi == EPI_PROJ) args.trace = gemm_trace_buffer();
  if (epi == EPI_PROJ && args.stream_k) {
    // stream-K grid G (stream_k > 1: requested G): every CTA gets >= 1 unit and an m-tile is cut into <= 16 pieces
    // (the partial buffer holds 16 per tile).  PKV_PROJ_SK_GRID overrides (tuning).
    const long tm = ceil_div(args.M, 128 * gemm_mt(96, EPI_PROJ));  // m-tiles of the kernel
    const long units = tm * kt;
    static const int g_env = getenv("PKV_PROJ_SK_GRID") ? atoi(getenv("PKV_PROJ_SK_GRID")) : 0;
    // 128 CTAs measured best on B200 for all four Llama-8B shapes (tools/bench_proj.py:
    // 101 us per layer vs 107 on all 148 SMs and 127 for the old split-K cost model)
    long g = args.stream_k > 1 ? args.stream_k : (g_env > 0 ? g_env : std::min(128, num_sms()));
    g = std::min(g, units);
    g = std::min(g, 15L * tm);
    args.stream_k = (int)std::max(1L, g);
    args.n_splits = 1;
    args.k_tiles_per_split = kt;
  }
  CUtensorMap ta, tb;
  // Stage-II GEMMs (BN = 256) on CTA pairs unless PKV_GEMM_CG=1
  static const int cg_env = getenv("PKV_GEMM_CG") ? atoi(getenv("PKV_GEMM_CG")) : 2;
  static const int proj_cg_env = getenv("PKV_PROJ_CG") ? atoi(getenv("PKV_PROJ_CG")) : 1;
  const int cg = ((bn == 256 && cg_env == 2) || (bn == 96 && epi == EPI_PROJ && proj_cg_env == 2)) ? 2 : 1;
  if (!cached_tmap(&ta, A, args.M, K, lda, 128)) return set_error(PKV_ERR_CUDA, "gemm: TMA encode A failed");
  if (!cached_tmap(&tb, B, args.N, K, ldb, bn / cg)) return set_error(PKV_ERR_CUDA, "gemm: TMA encode B failed");
  // cluster split-K for the narrow projection: correct, but clusters of 2..8 CTAs with
  // ~200 KB of shared memory each co-schedule poorly (GPC packing) -- measured +4 ms per
  // prefill, so opt-in (PKV_PROJ_CLUSTER=1)
  static const bool proj_cluster = getenv("PKV_PROJ_CLUSTER") && getenv("PKV_PROJ_CLUSTER")[0] == '1';
  if (cg == 1 && bn == 96 && epi == EPI_PROJ && proj_cluster && args.n_splits >= 2 && args.n_splits <= 8)
    return launch_proj_cluster(ta, tb, args, stream);
  // grouped raster when the A operand does not stay in L2 (Stage-II down: 188 MB): a wave of
  // ~P = SMs / cg tiles then covers ~sqrt(P) m-tiles x ~sqrt(P) n-tiles instead of every
  // m-tile x P / tiles_m n-tiles, so each wave re-reads ~8 A panels instead of all 26.
  // Opt-in (PKV_GEMM_RASTER=g, group size g): down 608 vs 568 us with g = 8 and 0, within
  // the run-to-run spread under the power cap (profiles/r02/ab_ttft_r02d.txt), Stage II 125.8
  // vs 125.6 ms -- the re-read A panels hit L2 often enough (ncu: 69 % hit rate on down).
  static const int raster_env = getenv("PKV_GEMM_RASTER") ? atoi(getenv("PKV_GEMM_RASTER")) : 0;
  if (epi != EPI_PROJ && args.raster_gm == 0) args.raster_gm = raster_env;
  args.sk_pairs = 0;
  if (cg == 2 && epi != EPI_PROJ && bn == 256 && args.n_splits == 1 && args.sk_part && args.sk_cnt) {
    int rem, maxp;
    args.sk_pairs = gemm_sk_plan(args.M, args.N, K, &rem, &maxp);
    args.sk_maxp = maxp;
  }
  if (cg == 2) {
    switch (epi) {
      case EPI_F32: return launch_one<256, EPI_F32, 2>(ta, tb, args, stream);
      case EPI_BF16: return launch_one<256, EPI_BF16, 2>(ta, tb, args, stream);
      case EPI_RESID: return launch_one<256, EPI_RESID, 2>(ta, tb, args, stream);
      case EPI_SILU: return launch_one<256, EPI_SILU, 2>(ta, tb, args, stream);
      case EPI_QKV: return launch_one<256, EPI_QKV, 2>(ta, tb, args, stream);
      case EPI_PROJ: return launch_one<96, EPI_PROJ, 2>(ta, tb, args, stream);
      default: return set_error(PKV_ERR_ARGUMENT, "gemm: unsupported pair epilogue %d", epi);
    }
  }
  switch (bn * 16 + epi) {
    case 256 * 16 + EPI_F32: return launch_one<256, EPI_F32>(ta, tb, args, stream);
    case 256 * 16 + EPI_BF16: return launch_one<256, EPI_BF16>(ta, tb, args, stream);
    case 256 * 16 + EPI_RESID: return launch_one<256, EPI_RESID>(ta, tb, args, stream);
    case 256 * 16 + EPI_SILU: return launch_one<256, EPI_SILU>(ta, tb, args, stream);
    case 256 * 16 + EPI_QKV: return launch_one<256, EPI_QKV>(ta, tb, args, stream);
    case 128 * 16 + EPI_F32: return launch_one<128, EPI_F32>(ta, tb, args, stream);
    case 128 * 16 + EPI_RESID: return launch_one<128, EPI_RESID>(ta, tb, args, stream);
    case 96 * 16 + EPI_F32: return launch_one<96, EPI_F32>(ta, tb, args, stream);
    case 96 * 16 + EPI_PROJ: return launch_one<96, EPI_PROJ>(ta, tb, args, stream);
    default: return set_error(PKV_ERR_ARGUMENT, "gemm: unsupported (BN=%d, epi=%d)", bn, epi);
  }
}

}  // namespace pkv

extern "C" int pkv_debug_gemm_trace(unsigned long long* host, int n_ctas) {
  if (pkv::g_trace == nullptr) return -1;
  const int n = n_ctas < pkv::kTraceCtas ? n_ctas : pkv::kTraceCtas;
  cudaDeviceSynchronize();
  cudaMemcpy(host, pkv::g_trace, (size_t)n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemset(pkv::g_trace, 0, pkv::kTraceCtas * 8 * sizeof(unsigned long long));
  return 0;
}
