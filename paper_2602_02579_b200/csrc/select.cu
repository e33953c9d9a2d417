// K4: layer fusion + budgeted top-k (reference selection.py:52-61, tensor.py:117-133).
//
// fused[t] = f32( sum_l f64(per_layer[l][t]) / L ), summed in ascending l exactly
// like numpy's axis-0 mean, so the fused vector is bit-identical to the oracle's
// on identical per-layer input.  Selection is a single-CTA MSB radix select over
// the 64-bit composite key (orderable f32 << 32 | ~index): "larger score first,
// then smaller index" -- numpy's stable argsort(-s) -- is exactly descending key
// order, so the k largest keys are the reference set, ties included.  Indices are
// emitted ascending by an ordered block compaction.
#include <mutex>
#include "kernels.cuh"

namespace pkv {

__global__ void fuse_layers_kernel(const float* per_layer, int L, int s, float* fused) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  double acc = 0.0;
  for (int l = 0; l < L; ++l) acc += (double)per_layer[(long)l * s + t];
  fused[t] = (float)(acc / (double)L);
}

__device__ __forceinline__ uint64_t topk_key(const float* v, int i) {
  float f = v[i];
  if (f == 0.f) f = 0.f;  // -0.0 ties with +0.0 (numpy compares them equal)
  uint32_t u = __float_as_uint(f);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)i);
}

constexpr int TOPK_THREADS = 1024;

__global__ void __launch_bounds__(TOPK_THREADS) topk_kernel(const float* v, int n, int k, int32_t* out,
                                                            int32_t* status) {
  pdl_entry();
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int s_remaining;
  __shared__ int s_bad;
  __shared__ int warp_cnt[TOPK_THREADS / 32];
  __shared__ int s_base;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_bad = 0;
    s_prefix = 0;
    s_remaining = k;
  }
  __syncthreads();
  for (int i = tid; i < n; i += TOPK_THREADS)
    if (!isfinite(v[i])) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) *status = PKV_ERR_NUMERICS;
    return;
  }
  if (k == 0) {
    if (tid == 0) *status = PKV_OK;
    return;
  }
  // MSB-first radix select of the k-th largest key
  uint64_t mask = 0;
  for (int pass = 7; pass >= 0; --pass) {
    const int shift = pass * 8;
    for (int b = tid; b < 256; b += TOPK_THREADS) hist[b] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int i = tid; i < n; i += TOPK_THREADS) {
      const uint64_t key = topk_key(v, i);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int need = s_remaining;
      int b = 255;
      for (; b > 0; --b) {
        if ((int)hist[b] >= need) break;
        need -= (int)hist[b];
      }
      s_prefix = prefix | ((uint64_t)b << shift);
      s_remaining = need;
    }
    mask |= (uint64_t)0xFF << shift;
    __syncthreads();
  }
  const uint64_t kth = s_prefix;  // exact key of the k-th largest element
  // ordered compaction of {i : key(i) >= kth}
  if (tid == 0) s_base = 0;
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < n; c0 += TOPK_THREADS) {
    const int i = c0 + tid;
    const bool take = i < n && topk_key(v, i) >= kth;
    const uint32_t bal = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int acc = s_base;
      for (int w = 0; w < TOPK_THREADS / 32; ++w) {
        int c = warp_cnt[w];
        warp_cnt[w] = acc;
        acc += c;
      }
      s_base = acc;
    }
    __syncthreads();
    if (take) out[warp_cnt[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
    __syncthreads();
  }
  if (tid == 0) *status = (s_base == k) ? PKV_OK : PKV_ERR_CUDA;
}

__global__ void mark_kernel(const int32_t* idx, int n, uint8_t* flags) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[idx[i]] = 1;
}

int mark_launch(const int32_t* idx, int n, uint8_t* flags, cudaStream_t st) {
  if (n <= 0) return PKV_OK;
  launch_k(mark_kernel, ceil_div(n, 256), 256, 0, st, idx, n, flags);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("mark_kernel");
  return PKV_OK;
}

int fuse_layers_launch(const float* per_layer, int L, int s, float* fused, cudaStream_t st) {
  if (s <= 0) return PKV_OK;
  launch_k(fuse_layers_kernel, ceil_div(s, 256), 256, 0, st, per_layer, L, s, fused);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("fuse_layers_kernel");
  return PKV_OK;
}

int topk_launch(const float* v, int n, int k, int32_t* out, int32_t* status, cudaStream_t st) {
  launch_k(topk_kernel, 1, TOPK_THREADS, 0, st, v, n, k, out, status);
  PKV_LAUNCHED();
  PKV_CHECK_LAUNCH("topk_kernel");
  return PKV_OK;
}

}  // namespace pkv
