// K1 -- paris_summarize: PAA + iSAX quantization of a whole collection.
//
// Paper: ConvertToSAX in IndexBulkLoading (Alg2 line al2:cover, P:587-590;
// Alg5): PAA = segment means; symbol = region of the
// y-axis the mean falls in, N(0,1) breakpoints (R2), value on a
// cut -> upper region (R3).  SAX[p] holds series p; stored [w][n].
//
// B200 design: HBM-bound (4*len bytes in, w bytes out per
// series).  One warp per series, lane l loads float4 #(l + 32j) -- a warp reads
// 512 contiguous bytes per request.  A segment of seglen = 4G points spans G
// lanes; its sum is a G-lane xor-shuffle tree in fp32.  The symbol comes from a
// branchless binary search over the fp32 cuts in shared memory; whenever the
// fp32 PAA's rounding-error bound straddles a cut (~1e-3 of segments) the warp
// recomputes that series' sums in fp64 and the ambiguous lanes search the fp64
// cuts, so every symbol equals the one of the exact PAA.  Symbols of a 128-series
// tile are staged in shared memory and leave as 16-byte row stores.
#include "runtime.cuh"

namespace paris {
namespace {

constexpr int kTile = 128;       // series per CTA tile
constexpr int kThreads = 256;    // 8 warps
constexpr int kSeriesPerWarp = kTile / (kThreads / 32);  // 16
constexpr int kUnroll = 4;       // series loaded per warp step (bytes in flight)
constexpr int kMaxW = 64;

// #{c : cuts[c] <= v} over a table padded with +inf to 256 entries; `top` is
// the largest power of two <= card/2 (first step).
template <typename T>
__device__ __forceinline__ int upper_bound_pow2(const T* cuts, T v, int top) {
  int pos = 0;
  for (int step = top; step >= 1; step >>= 1)
    if (cuts[pos + step - 1] <= v) pos += step;
  return pos;
}

template <int NV>  // len = 128 * NV
__global__ void __launch_bounds__(kThreads)
k_summarize_fast(const float* __restrict__ raw, int64_t n, int w, int card, int G,
                 uint8_t* __restrict__ sax, const CardTables* __restrict__ tab) {
  __shared__ float s_cf[kMaxCard];
  __shared__ double s_cd[kMaxCard];
  __shared__ __align__(16) uint8_t s_tile[kMaxW * kTile];

  for (int i = threadIdx.x; i < kMaxCard; i += kThreads) {
    s_cf[i] = tab->cuts_f[i];
    s_cd[i] = tab->cuts_d[i];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int len = 128 * NV;
  const int seglen = 4 * G;
  const float inv_seglen = 1.0f / (float)seglen;  // exact: seglen is a power of two
  const int top = card >> 1;
  int depth = 2;  // pairwise depth of the fp32 segment sum: 2 in-lane + log2(G)
  for (int g = G; g > 1; g >>= 1) ++depth;
  // |fp32 sum - exact sum| <= depth * 2^-24 * sum|x| (pairwise summation bound, with slack)
  const float err_scale = (float)(depth + 1) * 5.9604645e-08f * inv_seglen * 1.001f;
  const bool aligned = (n % 16) == 0;

  for (int64_t base = (int64_t)blockIdx.x * kTile; base < n; base += (int64_t)gridDim.x * kTile) {
    const int cnt = (int)imin64(kTile, n - base);

#pragma unroll 1
    for (int u0 = 0; u0 < kSeriesPerWarp; u0 += kUnroll) {
      float4 v[kUnroll][NV];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int col = warp * kSeriesPerWarp + u0 + u;
        if (col < cnt) {
          const float4* row = reinterpret_cast<const float4*>(raw + (size_t)(base + col) * len);
#pragma unroll
          for (int j = 0; j < NV; ++j) v[u][j] = __ldcs(row + lane + 32 * j);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int col = warp * kSeriesPerWarp + u0 + u;
        if (col >= cnt) continue;  // warp-uniform
        float sum[NV], asum[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const float4 x = v[u][j];
          sum[j] = (x.x + x.y) + (x.z + x.w);
          asum[j] = (fabsf(x.x) + fabsf(x.y)) + (fabsf(x.z) + fabsf(x.w));
        }
        for (int o = 1; o < G; o <<= 1) {
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            sum[j] += __shfl_xor_sync(0xffffffffu, sum[j], o);
            asum[j] += __shfl_xor_sync(0xffffffffu, asum[j], o);
          }
        }
        // lane l owns slice j of its segment group iff (l % G) == (j % G)
        int sym[NV];
        bool amb_any = false;
        bool amb[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const bool mine = (lane % G) == (j % G);
          const float paa = sum[j] * inv_seglen;
          const int s = upper_bound_pow2(s_cf, paa, top);
          const float err = asum[j] * err_scale;
          bool a = false;
          if (s > 0) {
            const float c = s_cf[s - 1];
            a |= (paa - c) <= err + fabsf(c) * 1.2e-7f + 1e-30f;
          }
          if (s < card - 1) {
            const float c = s_cf[s];
            a |= (c - paa) <= err + fabsf(c) * 1.2e-7f + 1e-30f;
          }
          sym[j] = s;
          amb[j] = mine && a;
          amb_any |= amb[j];
        }
        if (__any_sync(0xffffffffu, amb_any)) {
          // exact path: fp64 sums (error ~1e-16, far inside the 1e-6 window), fp64 cuts
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const float4 x = v[u][j];
            double d = ((double)x.x + (double)x.y) + ((double)x.z + (double)x.w);
            for (int o = 1; o < G; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (amb[j]) sym[j] = upper_bound_pow2(s_cd, d / (double)seglen, top);
          }
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if ((lane % G) == (j % G)) {
            const int seg = (lane + 32 * j) / G;
            s_tile[seg * kTile + (warp * kSeriesPerWarp + u0 + u)] = (uint8_t)sym[j];
          }
        }
      }
    }
    __syncthreads();
    // write the tile: row s -> sax[s*n + base .. base+cnt)
    if (aligned && cnt == kTile) {
      for (int t = threadIdx.x; t < w * (kTile / 16); t += kThreads) {
        const int s = t / (kTile / 16), part = t % (kTile / 16);
        const uint4 val = *reinterpret_cast<const uint4*>(s_tile + s * kTile + part * 16);
        __stcs(reinterpret_cast<uint4*>(sax + (size_t)s * n + base) + part, val);
      }
    } else {
      for (int t = threadIdx.x; t < w * cnt; t += kThreads) {
        const int s = t / cnt, col = t % cnt;
        sax[(size_t)s * n + base + col] = s_tile[s * kTile + col];
      }
    }
    __syncthreads();
  }
}

// Generic fallback (any len % w == 0): one thread per series, fp64 segment sums
// (sequential), fp64 binary search.  Correct for every supported shape; used
// only when the fast path's shape conditions do not hold.
__global__ void __launch_bounds__(kThreads)
k_summarize_generic(const float* __restrict__ raw, int64_t n, int len, int w, int card,
                    uint8_t* __restrict__ sax, const CardTables* __restrict__ tab) {
  __shared__ double s_cd[kMaxCard];
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) s_cd[i] = tab->cuts_d[i];
  __syncthreads();
  const int seglen = len / w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float* x = raw + (size_t)i * len;
    for (int s = 0; s < w; ++s) {
      double acc = 0.0;
      for (int j = 0; j < seglen; ++j) acc += (double)x[s * seglen + j];
      sax[(size_t)s * n + i] = (uint8_t)upper_bound_pow2(s_cd, acc / (double)seglen, card >> 1);
    }
  }
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached = v > 0 ? v : 148;
  }
  return cached;
}

}  // namespace

int summarize_impl(const float* raw, int64_t n, int len, int w, int card, uint8_t* out_sax,
                   cudaStream_t st) {
  if (!raw || !out_sax) { set_error("paris_summarize: null pointer"); return PARIS_EINVAL; }
  if (n < 1 || n >= (int64_t(1) << 31)) { set_error("paris_summarize: n=%lld out of range", (long long)n); return PARIS_EINVAL; }
  if (len < 4 || len > 4096 || (len % 4) || w < 1 || w > kMaxW || (len % w)) {
    set_error("paris_summarize: unsupported (len=%d, w=%d)", len, w);
    return PARIS_ECONFIG;
  }
  const CardTables* tab = device_tables(card);
  if (!tab) return PARIS_ECONFIG;
  if ((reinterpret_cast<uintptr_t>(raw) & 15) != 0) {
    set_error("paris_summarize: raw must be 16-byte aligned");
    return PARIS_EINVAL;
  }
  const int seglen = len / w;
  const int G = seglen / 4;
  const bool fast = (len % 128 == 0) && (seglen % 4 == 0) && G >= 1 && G <= 32 && ((G & (G - 1)) == 0);
  const int sms = sm_count();
  if (fast) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    const int grid = (int)imin64(tiles, (int64_t)sms * 8);
    cudaError_t e;
    switch (len / 128) {
      case 1: e = PARIS_LAUNCH("summarize", k_summarize_fast<1>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, tab); break;
      case 2: e = PARIS_LAUNCH("summarize", k_summarize_fast<2>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, tab); break;
      case 4: e = PARIS_LAUNCH("summarize", k_summarize_fast<4>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, tab); break;
      case 8: e = PARIS_LAUNCH("summarize", k_summarize_fast<8>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, tab); break;
      default: {
        const int gg = (int)imin64((n + kThreads - 1) / kThreads, (int64_t)sms * 8);
        e = PARIS_LAUNCH("summarize_generic", k_summarize_generic, gg, kThreads, 0, st, raw, n, len, w, card, out_sax, tab);
      }
    }
    PARIS_CHECK_LAUNCH(e, "summarize launch");
  } else {
    const int gg = (int)imin64((n + kThreads - 1) / kThreads, (int64_t)sms * 8);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("summarize_generic", k_summarize_generic, gg, kThreads, 0, st,
                                    raw, n, len, w, card, out_sax, tab),
                       "summarize launch");
  }
  return PARIS_OK;
}

}  // namespace paris

extern "C" int paris_summarize(const float* raw, int64_t n, int32_t len, int32_t w, int32_t card,
                               uint8_t* out_sax, void* stream) {
  return paris::summarize_impl(raw, n, len, w, card, out_sax, (cudaStream_t)stream);
}
