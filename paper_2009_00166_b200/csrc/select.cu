// k-NN with k beyond the pruned path's PARIS_MAX_K (1 <= k <= n):
// when k is a large share of the collection, pruning cannot pay, so every series' exact
// squared distance is computed (warp per series, the refinement's own summation) and the
// (d^2 bits << 32 | id) keys are sorted -- ascending distance, ties to the lower id (R6),
// exactly the plain k-NN definition.  CUB radix sort: a library sort, as the
// index build uses; the distances are this file's kernel.
#include "runtime.cuh"

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

namespace paris {

namespace {

__global__ void __launch_bounds__(256) k_all_d2(const float* __restrict__ raw, int64_t n, int len,
                                                const float* __restrict__ q, uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int nf = len >> 2;
  const float4* qv = reinterpret_cast<const float4*>(q);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float4* row = reinterpret_cast<const float4*>(raw + (size_t)i * len);
    float acc = 0.f;
    for (int f = lane; f < nf; f += 32) {
      const float4 x = __ldcs(row + f), y = __ldg(qv + f);
      float d;
      d = x.x - y.x; acc = fmaf(d, d, acc);
      d = x.y - y.y; acc = fmaf(d, d, acc);
      d = x.z - y.z; acc = fmaf(d, d, acc);
      d = x.w - y.w; acc = fmaf(d, d, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) keys[i] = ((uint64_t)__float_as_uint(acc) << 32) | (uint32_t)i;
  }
}

__global__ void k_keys_out(const uint64_t* __restrict__ sorted, int k, int64_t* __restrict__ out_idx,
                           float* __restrict__ out_dist) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    const uint64_t key = sorted[i];
    out_idx[i] = (int64_t)(uint32_t)key;
    out_dist[i] = sqrtf(__uint_as_float((uint32_t)(key >> 32)));
  }
}

}  // namespace

// raw: device (or mapped host) pointer; queries / outputs: device pointers [nq][len], [nq][k].
int knn_large_k(const float* raw, int64_t n, int len, const float* queries, int nq, int k, int64_t* out_idx,
                float* out_dist, cudaStream_t st) {
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)n, 0, 64,
                                 st);
  const size_t kb = ((size_t)n * 8 + 255) & ~(size_t)255;
  void* wsh = nullptr;
  char* base = (char*)ws_acquire(2 * kb + temp_bytes, st, &wsh, nullptr);
  if (!base) return PARIS_ENOMEM;
  uint64_t* keys = (uint64_t*)base;
  uint64_t* sorted = (uint64_t*)(base + kb);
  void* temp = base + 2 * kb;
  const int grid = device_sms() * 8;
  int rc = PARIS_OK;
  for (int q = 0; q < nq && rc == PARIS_OK; ++q) {
    cudaError_t e = PARIS_LAUNCH("all_d2", k_all_d2, grid, 256, 0, st, raw, n, len, queries + (size_t)q * len, keys);
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys, sorted, (int)n, 0, 64, st);
    if (e == cudaSuccess)
      e = PARIS_LAUNCH("finalize", k_keys_out, std::min(1024, (k + 255) / 256), 256, 0, st, sorted, k,
                       out_idx + (size_t)q * k, out_dist + (size_t)q * k);
    if (e != cudaSuccess) rc = cuda_error(e, "paris_knn (k > PARIS_MAX_K)");
  }
  ws_release(wsh, st);
  return rc;
}

}  // namespace paris
