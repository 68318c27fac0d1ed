// Microbenchmark: random 1 KB row gathers on B200 -- LDG (warp per row, U rows in flight per warp)
// vs cp.async.bulk (TMA) 1 KB copies into a shared ring.  Prints GB/s of rows gathered.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) g_ldg(const float4* __restrict__ raw, const uint32_t* __restrict__ ids, int m, int nf, float* out) {
  int lane = threadIdx.x & 31;
  int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, GW = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int i0 = gw * U; i0 < m; i0 += GW * U) {
    float4 x[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int i = i0 + u;
      if (i < m) {
        const float4* r = raw + (size_t)ids[i] * nf;
#pragma unroll
        for (int c = 0; c < 2; ++c) x[u][c] = __ldg(r + lane + 32 * c);
      } else { x[u][0] = x[u][1] = make_float4(0,0,0,0); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc += x[u][c].x + x[u][c].y + x[u][c].z + x[u][c].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SLOTS>
__global__ void __launch_bounds__(128, 1) g_tma(const float* __restrict__ raw, const uint32_t* __restrict__ ids, int m, int len, float* out) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t full[SLOTS];
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < SLOTS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // single warp does everything: lanes issue copies for SLOTS rows, wait, sum, repeat
  if (tid >= 32) return;
  int lane = tid;
  float acc = 0.f;
  unsigned bytes = len * 4;
  int it = 0;
  for (int i0 = blockIdx.x * SLOTS; i0 < m; i0 += gridDim.x * SLOTS, ++it) {
    for (int s = lane; s < SLOTS; s += 32) {
      int i = i0 + s;
      if (i < m) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&full[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sa(dsm + (size_t)s * bytes)), "l"(raw + (size_t)ids[i] * len), "r"(bytes), "r"(sa(&full[s])) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(&full[s])) : "memory");
      }
    }
    for (int s = 0; s < SLOTS; ++s) {
      asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" :: "r"(sa(&full[s])), "r"(it & 1) : "memory");
      const float4* r = reinterpret_cast<const float4*>(dsm + (size_t)s * bytes);
      float4 v = r[lane];
      acc += v.x;
    }
    __syncwarp();
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const size_t n = 20000000; const int len = 256; const int m = 2000000;
  float* raw; uint32_t* ids; float* out;
  cudaMalloc(&raw, n * len * 4); cudaMemset(raw, 0, n * len * 4);
  cudaMalloc(&ids, m * 4); cudaMalloc(&out, 4);
  std::vector<uint32_t> h(m); std::mt19937 g(1); for (auto& x : h) x = g() % n;
  cudaMemcpy(ids, h.data(), m * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-28s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, (double)m * len * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  int sms = 148;
  run("ldg U=1 occ", [&] { g_ldg<1><<<sms * 8, 256>>>((const float4*)raw, ids, m, len / 4, out); });
  run("ldg U=2", [&] { g_ldg<2><<<sms * 8, 256>>>((const float4*)raw, ids, m, len / 4, out); });
  run("ldg U=4", [&] { g_ldg<4><<<sms * 8, 256>>>((const float4*)raw, ids, m, len / 4, out); });
  run("ldg U=8", [&] { g_ldg<8><<<sms * 4, 256>>>((const float4*)raw, ids, m, len / 4, out); });
  cudaFuncSetAttribute(g_tma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(g_tma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(g_tma<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
  run("tma 64 slots/SM", [&] { g_tma<64><<<sms, 128, 64 * 1024>>>(raw, ids, m, len, out); });
  run("tma 128 slots/SM", [&] { g_tma<128><<<sms, 128, 128 * 1024>>>(raw, ids, m, len, out); });
  run("tma 192 slots/SM", [&] { g_tma<192><<<sms, 128, 192 * 1024>>>(raw, ids, m, len, out); });
  run("tma 64 slots x2 CTA/SM", [&] { g_tma<64><<<sms * 2, 128, 64 * 1024>>>(raw, ids, m, len, out); });
  return 0;
}
