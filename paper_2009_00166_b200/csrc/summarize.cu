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

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

namespace paris {
namespace {

constexpr int kTile = 128;       // series per CTA tile
constexpr int kThreads = 256;    // 8 warps
constexpr int kSeriesPerWarp = kTile / (kThreads / 32);  // 16
constexpr int kUnroll = 4;       // series loaded per warp step (bytes in flight)
constexpr int kMaxW = 64;
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
constexpr size_t kHostChunkBytes = (size_t)256 << 20;  // host-raw staging: 2 x 256 MB device buffers

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
                 uint8_t* __restrict__ sax, int64_t ld, const CardTables* __restrict__ tab) {
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
  const bool aligned = (ld % 16) == 0 && (reinterpret_cast<uintptr_t>(sax) & 15) == 0;

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
    // write the tile: row s -> sax[s*ld + base .. base+cnt)
    if (aligned && cnt == kTile) {
      for (int t = threadIdx.x; t < w * (kTile / 16); t += kThreads) {
        const int s = t / (kTile / 16), part = t % (kTile / 16);
        const uint4 val = *reinterpret_cast<const uint4*>(s_tile + s * kTile + part * 16);
        __stcs(reinterpret_cast<uint4*>(sax + (size_t)s * ld + base) + part, val);
      }
    } else {
      for (int t = threadIdx.x; t < w * cnt; t += kThreads) {
        const int s = t / cnt, col = t % cnt;
        sax[(size_t)s * ld + base + col] = s_tile[s * kTile + col];
      }
    }
    __syncthreads();
  }
}

// TMA-tiled variant (len in {128, 256, 512}, n % 4 == 0): a persistent CTA per SM
// streams 64 KB tiles of consecutive raw series (one contiguous range, one
// cp.async.bulk each) into a kSumStages-deep shared-memory ring (mbarrier
// completion), so HBM reads run ahead of the arithmetic.  Warp w owns SPW
// consecutive series of a tile; lane l takes float4 #(l + 32j) of a series from
// shared memory (conflict-free); segment sums by G-lane xor shuffles; the symbol
// comes from the bucket table (one 8-byte shared load per segment, no search).
// The owner lane of a segment packs the SPW symbols of its series into one store.
constexpr int kSumThreads = 1024;  // 32 warps: latency of the per-series shuffle chains is hidden by width
constexpr int kSumWarps = kSumThreads / 32;
constexpr int kSumStages = 3;
constexpr int kSumTileBytes = 65536;
constexpr size_t kSumSmem = (size_t)kSumStages * kSumTileBytes + kLutN * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase flips
// (or the hint elapses) instead of spinning on issue slots the working warps need
constexpr unsigned kMbarSuspendNs = 100000;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(kMbarSuspendNs)
      : "memory");
}

template <int NV>  // len = 128 * NV
__global__ void __launch_bounds__(kSumThreads, 1)
k_summarize_tma(const float* __restrict__ raw, int64_t n, int w, int card, int G,
                uint8_t* __restrict__ sax, int64_t ld, const CardTables* __restrict__ tab) {
  constexpr int len = 128 * NV;
  constexpr int TS = kSumTileBytes / (4 * len);  // series per tile
  constexpr int SPW = TS / kSumWarps;             // series per warp per tile (1, 2 or 4)
  static_assert(SPW >= 1 && SPW <= 4, "tile shape");
  extern __shared__ __align__(128) uint8_t dsm[];
  float* s_tiles = reinterpret_cast<float*>(dsm);
  uint2* s_lut = reinterpret_cast<uint2*>(dsm + (size_t)kSumStages * kSumTileBytes);
  __shared__ double s_cd[kMaxCard];
  __shared__ __align__(8) uint64_t s_full[kSumStages];
  __shared__ unsigned s_cnt[kSumStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + TS - 1) / TS;

  auto issue = [&](int64_t tile, int st) {
    const int64_t base = tile * TS;
    const unsigned bytes = (unsigned)(imin64(TS, n - base) * len * 4);
    mbar_expect_tx(&s_full[st], bytes);
    bulk_g2s(s_tiles + (size_t)st * (kSumTileBytes / 4), raw + (size_t)base * len, bytes, &s_full[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < kSumStages; ++st) {
      mbar_init(&s_full[st], 1);
      s_cnt[st] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int st = 0; st < kSumStages; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles) issue(tile, st);
    }
  }
  for (int i = tid; i < kLutN; i += kSumThreads) s_lut[i] = tab->lut[i];
  for (int i = tid; i < kMaxCard; i += kSumThreads) s_cd[i] = tab->cuts_d[i];
  __syncthreads();

  const int seglen = 4 * G;
  const float inv_seglen = 1.0f / (float)seglen;
  const int top = card >> 1;
  int depth = 2;
  for (int g = G; g > 1; g >>= 1) ++depth;
  const float err_scale = (float)(depth + 1) * 5.9604645e-08f * inv_seglen * 1.001f;

  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= ntiles) break;
    const int st = (int)(it % kSumStages);
    mbar_wait(&s_full[st], (unsigned)((it / kSumStages) & 1));
    const int64_t base = tile * TS + warp * SPW;
    const int cnt = (int)std::max<int64_t>(0, imin64(SPW, n - base));
    const float4* tl = reinterpret_cast<const float4*>(s_tiles + (size_t)st * (kSumTileBytes / 4)) +
                       (size_t)warp * SPW * (len / 4);
    float4 v[SPW][NV];
#pragma unroll
    for (int u = 0; u < SPW; ++u)
#pragma unroll
      for (int j = 0; j < NV; ++j) v[u][j] = (u < cnt) ? tl[u * (len / 4) + lane + 32 * j] : make_float4(0, 0, 0, 0);
    __syncwarp();
    if (lane == 0) {
      if (atomicAdd(&s_cnt[st], 1u) == kSumWarps - 1) {
        s_cnt[st] = 0;
        const int64_t next = tile + (int64_t)kSumStages * gridDim.x;
        if (next < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(next, st);
        }
      }
    }
    uint32_t packed[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) packed[j] = 0;
#pragma unroll
    for (int u = 0; u < SPW; ++u) {
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
      int sym[NV];
      bool amb_any = false, amb[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const float paa = sum[j] * inv_seglen;
        int k = __float2int_rd((paa + kLutLo) * kLutScale);
        k = min(max(k, 0), kLutN - 1);
        const uint2 e = s_lut[k];
        const float c = __uint_as_float(e.x);
        sym[j] = (int)e.y + (paa >= c ? 1 : 0);
        const float err = asum[j] * err_scale;
        amb[j] = ((lane % G) == (j % G)) && (fabsf(paa - c) <= err + fabsf(c) * 1.2e-7f + 1e-30f);
        amb_any |= amb[j];
      }
      if (__any_sync(0xffffffffu, amb_any)) {
        // exact path: fp64 sums and fp64 cuts (binary search), as in k_summarize_fast
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const float4 x = v[u][j];
          double d = ((double)x.x + (double)x.y) + ((double)x.z + (double)x.w);
          for (int o = 1; o < G; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (amb[j]) sym[j] = upper_bound_pow2(s_cd, d / (double)seglen, top);
        }
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) packed[j] |= (uint32_t)sym[j] << (8 * u);
    }
    // owner lane of segment (lane + 32 j) / G stores the SPW symbols of its series
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if ((lane % G) == (j % G) && cnt > 0) {
        const int seg = (lane + 32 * j) / G;
        uint8_t* dst = sax + (size_t)seg * ld + base;
        if (cnt == SPW) {
          if (SPW == 4) *reinterpret_cast<uint32_t*>(dst) = packed[j];
          else if (SPW == 2) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)packed[j];
          else *dst = (uint8_t)packed[j];
        } else {
          for (int u = 0; u < cnt; ++u) dst[u] = (uint8_t)(packed[j] >> (8 * u));
        }
      }
    }
  }
}

// Segment-per-lane variant of the TMA-tiled kernel (w = 16, len = 64 F): the
// same 64 KB tile ring, but a half-warp owns a series and lane l its segment l --
// the segment's 4F points are summed in registers (no shuffles; the same
// pairwise tree, depth 2 + log2 F, as the xor-shuffle form, so the same rounding
// bound), and each lane quantizes one segment (no lane repeats another's lookup).
// Lane l reads float4 #((c + l / (8/F)) mod F) of its segment at step c: the 8
// lanes of each shared-memory phase then cover all 32 banks (segments are 16F
// bytes apart).
template <int F>
__global__ void __launch_bounds__(kSumThreads, 1)
k_summarize_seg(const float* __restrict__ raw, int64_t n, int card, uint8_t* __restrict__ sax, int64_t ld,
                const CardTables* __restrict__ tab) {
  constexpr int w = 16, len = 64 * F, seglen = 4 * F;
  constexpr int TS = kSumTileBytes / (4 * len);  // series per tile
  constexpr int SPW = TS / kSumWarps;             // series per warp per tile (2 halves x SPW/2)
  static_assert(SPW % 2 == 0 && SPW >= 2 && SPW <= 4, "tile shape");
  constexpr int SPH = SPW / 2;                    // series per half-warp
  extern __shared__ __align__(128) uint8_t dsm[];
  float* s_tiles = reinterpret_cast<float*>(dsm);
  uint2* s_lut = reinterpret_cast<uint2*>(dsm + (size_t)kSumStages * kSumTileBytes);
  __shared__ double s_cd[kMaxCard];
  __shared__ __align__(8) uint64_t s_full[kSumStages];
  __shared__ unsigned s_cnt[kSumStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hf = lane >> 4, hl = lane & 15;
  const int64_t ntiles = (n + TS - 1) / TS;

  auto issue = [&](int64_t tile, int st) {
    const int64_t base = tile * TS;
    const unsigned bytes = (unsigned)(imin64(TS, n - base) * len * 4);
    mbar_expect_tx(&s_full[st], bytes);
    bulk_g2s(s_tiles + (size_t)st * (kSumTileBytes / 4), raw + (size_t)base * len, bytes, &s_full[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < kSumStages; ++st) {
      mbar_init(&s_full[st], 1);
      s_cnt[st] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int st = 0; st < kSumStages; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles) issue(tile, st);
    }
  }
  for (int i = tid; i < kLutN; i += kSumThreads) s_lut[i] = tab->lut[i];
  for (int i = tid; i < kMaxCard; i += kSumThreads) s_cd[i] = tab->cuts_d[i];
  __syncthreads();

  constexpr float inv_seglen = 1.0f / (float)seglen;
  const int top = card >> 1;
  constexpr int depth = 2 + (F == 1 ? 0 : F == 2 ? 1 : F == 4 ? 2 : 3);
  const float err_scale = (float)(depth + 1) * 5.9604645e-08f * inv_seglen * 1.001f;
  constexpr int rdiv = 8 / F;  // lanes per rotation step

  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= ntiles) break;
    const int st = (int)(it % kSumStages);
    mbar_wait(&s_full[st], (unsigned)((it / kSumStages) & 1));
    const int64_t base = tile * TS + warp * SPW;  // series base of this warp
    const int cnt = (int)std::max<int64_t>(0, imin64(SPW, n - base));
    const float4* tl = reinterpret_cast<const float4*>(s_tiles + (size_t)st * (kSumTileBytes / 4));
    float4 v[SPH][F];
#pragma unroll
    for (int u = 0; u < SPH; ++u) {
      const int sl = warp * SPW + 2 * u + hf;  // series within the tile: halves interleave
      const float4* sp = tl + (size_t)sl * (len / 4) + hl * F;
#pragma unroll
      for (int c = 0; c < F; ++c)  // register c holds float4 #r (the sum tree is order-free in its bound)
        v[u][c] = (2 * u + hf < cnt) ? sp[(c + hl / rdiv) & (F - 1)] : make_float4(0, 0, 0, 0);
    }
    __syncwarp();
    if (lane == 0) {
      if (atomicAdd(&s_cnt[st], 1u) == kSumWarps - 1) {
        s_cnt[st] = 0;
        const int64_t next = tile + (int64_t)kSumStages * gridDim.x;
        if (next < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(next, st);
        }
      }
    }
    uint32_t packed = 0;  // symbols of this lane's segment for the warp's SPW series (byte 2u + hf)
#pragma unroll
    for (int u = 0; u < SPH; ++u) {
      float part[F], apart[F];
#pragma unroll
      for (int c = 0; c < F; ++c) {
        const float4 x = v[u][c];
        part[c] = (x.x + x.y) + (x.z + x.w);
        apart[c] = (fabsf(x.x) + fabsf(x.y)) + (fabsf(x.z) + fabsf(x.w));
      }
#pragma unroll
      for (int o = 1; o < F; o <<= 1)
#pragma unroll
        for (int c = 0; c < F; c += 2 * o) {
          part[c] += part[c + o];
          apart[c] += apart[c + o];
        }
      const float paa = part[0] * inv_seglen;
      int k = __float2int_rd((paa + kLutLo) * kLutScale);
      k = min(max(k, 0), kLutN - 1);
      const uint2 e = s_lut[k];
      const float cut = __uint_as_float(e.x);
      int sym = (int)e.y + (paa >= cut ? 1 : 0);
      const bool amb = fabsf(paa - cut) <= apart[0] * err_scale + fabsf(cut) * 1.2e-7f + 1e-30f;
      if (__any_sync(0xffffffffu, amb) && amb) {
        // exact path: the fp64 segment sum and the fp64 cuts
        double d = 0.0;
#pragma unroll
        for (int c = 0; c < F; ++c) {
          const float4 x = v[u][c];
          d += ((double)x.x + (double)x.y) + ((double)x.z + (double)x.w);
        }
        sym = upper_bound_pow2(s_cd, d / (double)seglen, top);
      }
      packed |= (uint32_t)sym << (8 * (2 * u + hf));
    }
    // lane hl of the first half stores segment hl's SPW symbols (both halves' bytes)
    packed |= __shfl_down_sync(0xffffffffu, packed, 16);
    if (hf == 0 && cnt > 0) {
      uint8_t* dst = sax + (size_t)hl * ld + base;
      if (cnt == SPW) {
        if (SPW == 4) *reinterpret_cast<uint32_t*>(dst) = packed;
        else *reinterpret_cast<uint16_t*>(dst) = (uint16_t)packed;
      } else {
        for (int u = 0; u < cnt; ++u) dst[u] = (uint8_t)(packed >> (8 * u));
      }
    }
    (void)w;
  }
}

// Generic fallback (any len % w == 0): one thread per series, fp64 segment sums
// (sequential), fp64 binary search.  Correct for every supported shape; used
// only when the fast path's shape conditions do not hold.
__global__ void __launch_bounds__(kThreads)
k_summarize_generic(const float* __restrict__ raw, int64_t n, int len, int w, int card,
                    uint8_t* __restrict__ sax, int64_t ld, const CardTables* __restrict__ tab) {
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
      sax[(size_t)s * ld + i] = (uint8_t)upper_bound_pow2(s_cd, acc / (double)seglen, card >> 1);
    }
  }
}

int sm_count() { return device_sms(); }

}  // namespace

// Summarize n device-resident series into rows of stride ld (out_sax[s*ld + i]).
static int summarize_device(const float* raw, int64_t n, int len, int w, int card, uint8_t* out_sax, int64_t ld,
                            const CardTables* tab, cudaStream_t st) {
  const int seglen = len / w;
  const int G = seglen / 4;
  const bool fast = (len % 128 == 0) && (seglen % 4 == 0) && G >= 1 && G <= 32 && ((G & (G - 1)) == 0);
  const int sms = sm_count();
  const bool tma = fast && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(out_sax) & 3) == 0) &&
                   (n % 4 == 0) && (len == 128 || len == 256 || len == 512);
  if (tma) {
    const int64_t tiles = (n + (kSumTileBytes / (4 * len)) - 1) / (kSumTileBytes / (4 * len));
    const int grid = (int)imin64(tiles, (int64_t)sms);
    cudaError_t e;
    static int attr_key;
    e = once_per_device(&attr_key, [](int) {  // every variant's shared-memory limit, once per device
      cudaError_t r = cudaFuncSetAttribute(k_summarize_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k_summarize_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k_summarize_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k_summarize_seg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k_summarize_seg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSumSmem);
      return r;
    });
    PARIS_CHECK_LAUNCH(e, "summarize smem attribute");
    if (w == 16 && len <= 256 && !getenv("PARIS_SUMMARIZE_SHFL")) {  // segment per lane (env: A/B of the shuffle form)
      switch (len) {
        case 128: e = PARIS_LAUNCH("summarize", k_summarize_seg<2>, grid, kSumThreads, kSumSmem, st, raw, n, card, out_sax, ld, tab); break;
        default: e = PARIS_LAUNCH("summarize", k_summarize_seg<4>, grid, kSumThreads, kSumSmem, st, raw, n, card, out_sax, ld, tab); break;
      }
    } else {
      switch (len) {
        case 128: e = PARIS_LAUNCH("summarize", k_summarize_tma<1>, grid, kSumThreads, kSumSmem, st, raw, n, w, card, G, out_sax, ld, tab); break;
        case 256: e = PARIS_LAUNCH("summarize", k_summarize_tma<2>, grid, kSumThreads, kSumSmem, st, raw, n, w, card, G, out_sax, ld, tab); break;
        default: e = PARIS_LAUNCH("summarize", k_summarize_tma<4>, grid, kSumThreads, kSumSmem, st, raw, n, w, card, G, out_sax, ld, tab); break;
      }
    }
    PARIS_CHECK_LAUNCH(e, "summarize launch");
  } else if (fast) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    const int grid = (int)imin64(tiles, (int64_t)sms * 8);
    cudaError_t e;
    switch (len / 128) {
      case 1: e = PARIS_LAUNCH("summarize", k_summarize_fast<1>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, ld, tab); break;
      case 2: e = PARIS_LAUNCH("summarize", k_summarize_fast<2>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, ld, tab); break;
      case 4: e = PARIS_LAUNCH("summarize", k_summarize_fast<4>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, ld, tab); break;
      case 8: e = PARIS_LAUNCH("summarize", k_summarize_fast<8>, grid, kThreads, 0, st, raw, n, w, card, G, out_sax, ld, tab); break;
      default: {
        const int gg = (int)imin64((n + kThreads - 1) / kThreads, (int64_t)sms * 8);
        e = PARIS_LAUNCH("summarize_generic", k_summarize_generic, gg, kThreads, 0, st, raw, n, len, w, card, out_sax, ld, tab);
      }
    }
    PARIS_CHECK_LAUNCH(e, "summarize launch");
  } else {
    const int gg = (int)imin64((n + kThreads - 1) / kThreads, (int64_t)sms * 8);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("summarize_generic", k_summarize_generic, gg, kThreads, 0, st,
                                    raw, n, len, w, card, out_sax, ld, tab),
                       "summarize launch");
  }
  return PARIS_OK;
}



// Raw series in HOST memory (the paper's raw data stays on disk, P:52-56,
// 380-404): the Coordinator / IndexBulkLoading pipeline (Alg. Coordinator, P:477-483,
// 552) -- the Coordinator fills one half of the double-buffered raw data buffer
// while the workers summarize the other -- as stream-ordered
// H2D copies into two device staging buffers on a copy stream, overlapped with
// the summarize kernel on the caller's stream (truly asynchronous for pinned
// memory; pageable memory still works, the copies are then staged by the driver).
static int summarize_host(const float* raw, int64_t n, int len, int w, int card, uint8_t* out_sax,
                          const CardTables* tab, cudaStream_t st) {
  const size_t row = (size_t)len * 4;
  size_t cbytes = kHostChunkBytes;
  if (const char* ev = getenv("PARIS_HOST_CHUNK_BYTES")) {  // test hook: force many chunks
    const long long v = atoll(ev);
    if (v > 0) cbytes = (size_t)v;
  }
  int64_t chunk = std::max<int64_t>(16, ((int64_t)(cbytes / row)) / 16 * 16);
  chunk = std::min<int64_t>(chunk, (n + 15) / 16 * 16);
  float* buf[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  int rc = PARIS_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&buf[i], (size_t)chunk * row, st);
  }
  if (e == cudaSuccess) e = cudaEventRecord(consumed[0], st);  // buffers allocated on st
  if (e == cudaSuccess) e = cudaEventRecord(consumed[1], st);
  for (int64_t c0 = 0, c = 0; c0 < n && e == cudaSuccess && rc == PARIS_OK; c0 += chunk, ++c) {
    const int b = (int)(c & 1);
    const int64_t m = std::min<int64_t>(chunk, n - c0);
    e = cudaStreamWaitEvent(cs, consumed[b], 0);  // the summarize of chunk c-2 is done with buf[b]
    if (e == cudaSuccess) e = cudaMemcpyAsync(buf[b], raw + (size_t)c0 * len, (size_t)m * row, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, copied[b], 0);
    if (e == cudaSuccess) rc = summarize_device(buf[b], m, len, w, card, out_sax + c0, n, tab, st);
    if (e == cudaSuccess && rc == PARIS_OK) e = cudaEventRecord(consumed[b], st);
  }
  if (e != cudaSuccess && rc == PARIS_OK) rc = cuda_error(e, "paris_summarize (host raw)");
  for (int i = 0; i < 2; ++i) {
    if (buf[i]) cudaFreeAsync(buf[i], st);
    if (copied[i]) cudaEventDestroy(copied[i]);
    if (consumed[i]) cudaEventDestroy(consumed[i]);
  }
  if (cs) cudaStreamDestroy(cs);  // released once its queued copies complete
  return rc;
}

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
  retain_pool();
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, raw);
  if (e != cudaSuccess) cudaGetLastError();
  const bool host = (e != cudaSuccess) || at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
  if (host) return summarize_host(raw, n, len, w, card, out_sax, tab, st);
  return summarize_device(raw, n, len, w, card, out_sax, n, tab, st);
}

}  // namespace paris

namespace paris {
namespace {
// PAA with w2 segments (seglen = len / w2), each mean in fp64 then rounded to nearest fp16
// (through fp32: |x - fl16(x)| <= 2^-11 (1 + 2^-10) |fl16(x)| + 2^-24);
// a mean beyond the fp16 range is stored as NaN -- the refine then never prunes on it.
// Warp per series: lane l owns segments l, l + 32, ...
__global__ void __launch_bounds__(256) k_paa16(const float* __restrict__ raw, int64_t n, int len, int w2,
                                              __half* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int seglen = len / w2;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* x = raw + (size_t)i * len;
    for (int s = lane; s < w2; s += 32) {
      double acc = 0.0;
      for (int j = 0; j < seglen; ++j) acc += (double)__ldcs(x + (size_t)s * seglen + j);
      const double m = acc / (double)seglen;
      out[(size_t)i * w2 + s] = fabs(m) < 65000.0 ? __float2half_rn((float)m) : __ushort_as_half((unsigned short)0x7E00u);
    }
  }
}

// fp32 -> bf16 (round to nearest even), 8 values per thread-iteration
__global__ void __launch_bounds__(256) k_raw_bf16(const float4* __restrict__ raw, int64_t n8,
                                                  uint4* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = ld_stream_f4(raw + 2 * i), b = ld_stream_f4(raw + 2 * i + 1);
    uint4 o;
    o.x = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a.x)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a.y)) << 16);
    o.y = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a.z)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a.w)) << 16);
    o.z = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b.x)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b.y)) << 16);
    o.w = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b.z)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b.w)) << 16);
    out[i] = o;
  }
}
}  // namespace
}  // namespace paris

namespace paris {
int raw_bf16_launch(const float* raw, int64_t n, int len, uint16_t* out, cudaStream_t st) {
  const int64_t n8 = n * (int64_t)len / 8;
  const int grid = (int)std::min<int64_t>((n8 + 255) / 256, (int64_t)sm_count() * 16);
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("raw_bf16", k_raw_bf16, grid, 256, 0, st, reinterpret_cast<const float4*>(raw), n8,
                                  reinterpret_cast<uint4*>(out)),
                     "raw_bf16 launch");
  return PARIS_OK;
}
}  // namespace paris

extern "C" int paris_paa_f16(const float* raw, int64_t n, int32_t len, int32_t w2, uint16_t* out, void* stream) {
  if (!raw || !out || n < 1 || len < 4 || w2 < 1 || w2 > 256 || (len % w2) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      (w2 % 8)) {
    paris::set_error("paris_paa_f16: bad arguments (n=%lld len=%d w2=%d; w2 | len, w2 %% 8 == 0, w2 <= 256)",
                     (long long)n, len, w2);
    return PARIS_EINVAL;
  }
  const int grid = (int)std::min<int64_t>((n + 7) / 8, (int64_t)paris::sm_count() * 16);
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("paa_f16", paris::k_paa16, grid, 256, 0, (cudaStream_t)stream, raw, n, len, w2,
                                  reinterpret_cast<__half*>(out)),
                     "paa_f16 launch");
  return PARIS_OK;
}

extern "C" int paris_raw_bf16(const float* raw, int64_t n, int32_t len, uint16_t* out, void* stream) {
  if (!raw || !out || n < 1 || len < 8 || (len % 8) || (reinterpret_cast<uintptr_t>(raw) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15)) {
    paris::set_error("paris_raw_bf16: bad arguments (n=%lld len=%d; 16-byte aligned device pointers, len %% 8 == 0)",
                     (long long)n, len);
    return PARIS_EINVAL;
  }
  return paris::raw_bf16_launch(raw, n, len, out, (cudaStream_t)stream);
}

extern "C" int paris_summarize(const float* raw, int64_t n, int32_t len, int32_t w, int32_t card,
                               uint8_t* out_sax, void* stream) {
  return paris::summarize_impl(raw, n, len, w, card, out_sax, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- raw data in a file (f3)
// The paper's setting: the raw collection is a file on disk and index construction reads
// it sequentially (IndexBulkLoading's Coordinator fills one half of the double-buffered
// raw data buffer while the workers summarize the other).  Here a
// reader thread preads chunks into three pinned host buffers; the calling thread copies
// each chunk to a device staging buffer (copy stream) and summarizes it there (plus,
// optionally, its bf16 copy for paris_knn_index_x); a pinned buffer is re-read only once
// its copy completed.  O_DIRECT (page-cache bypass: the disk's own bandwidth) when the
// file system allows it, buffered reads otherwise.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <condition_variable>
#include <mutex>
#include <thread>

namespace paris {
int raw_bf16_launch(const float* raw, int64_t n, int len, uint16_t* out, cudaStream_t st);

static int summarize_file_impl(const char* path, int64_t offset, int64_t n, int len, int w, int card,
                               uint8_t* out_sax, uint16_t* out_bf16, int direct_io, cudaStream_t st) {
  const CardTables* tab = device_tables(card);
  if (!tab) return PARIS_ECONFIG;
  const size_t row = (size_t)len * 4;
  size_t cbytes = kHostChunkBytes;
  if (const char* ev = getenv("PARIS_HOST_CHUNK_BYTES")) {  // test hook: force many chunks
    const long long v = atoll(ev);
    if (v > 0) cbytes = (size_t)v;
  }
  int64_t chunk = std::max<int64_t>(16, ((int64_t)(cbytes / row)) / 16 * 16);
  chunk = std::min<int64_t>(chunk, (n + 15) / 16 * 16);
  const size_t cb = (size_t)chunk * row;
  int fd = -1;
  bool odirect = false;
  if (direct_io && (offset % 4096) == 0 && (cb % 4096) == 0) {
    fd = open(path, O_RDONLY | O_DIRECT);
    odirect = fd >= 0;
  }
  if (fd < 0) fd = open(path, O_RDONLY);
  if (fd < 0) {
    set_error("paris_summarize_file: cannot open %s", path);
    return PARIS_EINVAL;
  }
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (int64_t)sb.st_size < offset + n * (int64_t)row) {
    close(fd);
    set_error("paris_summarize_file: %s holds fewer than n=%lld rows of %d floats after offset %lld", path,
              (long long)n, len, (long long)offset);
    return PARIS_EINVAL;
  }
  if (!odirect) posix_fadvise(fd, offset, n * (int64_t)row, POSIX_FADV_SEQUENTIAL);
  constexpr int NB = 3;  // pinned read buffers: the reader runs up to two chunks ahead
  void* hb[NB] = {nullptr, nullptr, nullptr};
  float* db[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr;
  cudaEvent_t copied[NB] = {nullptr, nullptr, nullptr}, dcopied[2] = {nullptr, nullptr},
              consumed[2] = {nullptr, nullptr};
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  for (int i = 0; i < NB && e == cudaSuccess; ++i) {
    e = cudaHostAlloc(&hb[i], cb, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
  }
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dcopied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&db[i], cb, st);
  }
  if (e == cudaSuccess) e = cudaEventRecord(consumed[0], st);
  if (e == cudaSuccess) e = cudaEventRecord(consumed[1], st);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  // reader thread: chunk c into hb[c % NB] once the H2D copy of chunk c - NB is done
  std::mutex mu;
  std::condition_variable cv;
  int64_t ready = 0;       // chunks read
  bool failed = false;
  std::thread reader;
  if (e == cudaSuccess) {
    reader = std::thread([&]() {
      for (int64_t c = 0; c < nchunks; ++c) {
        {
          std::lock_guard<std::mutex> lk(mu);
          if (failed) return;  // the consumer gave up
        }
        if (c >= NB && cudaEventSynchronize(copied[c % NB]) != cudaSuccess) { std::lock_guard<std::mutex> lk(mu); failed = true; cv.notify_all(); return; }
        const size_t want = (size_t)std::min<int64_t>(chunk, n - c * chunk) * row;
        const size_t rd = odirect ? ((want + 4095) & ~(size_t)4095) : want;  // O_DIRECT: whole blocks
        size_t got = 0;
        while (got < want) {
          const ssize_t r = pread(fd, (char*)hb[c % NB] + got, rd - got, offset + (off_t)(c * chunk * row + got));
          if (r <= 0) { std::lock_guard<std::mutex> lk(mu); failed = true; cv.notify_all(); return; }
          got += (size_t)r;
        }
        std::lock_guard<std::mutex> lk(mu);
        ready = c + 1;
        cv.notify_all();
      }
    });
  }
  int rc = PARIS_OK;
  for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == PARIS_OK; ++c) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return ready > c || failed; });
      if (failed) { rc = PARIS_EINVAL; set_error("paris_summarize_file: read of %s failed", path); break; }
    }
    const int b = (int)(c & 1), h = (int)(c % NB);
    const int64_t c0 = c * chunk, m = std::min<int64_t>(chunk, n - c0);
    e = cudaStreamWaitEvent(cs, consumed[b], 0);  // the kernels of chunk c-2 are done with db[b]
    if (e == cudaSuccess) e = cudaMemcpyAsync(db[b], hb[h], (size_t)m * row, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(copied[h], cs);
    if (e == cudaSuccess) e = cudaEventRecord(dcopied[b], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, dcopied[b], 0);
    if (e == cudaSuccess) rc = summarize_device(db[b], m, len, w, card, out_sax + c0, n, tab, st);
    if (e == cudaSuccess && rc == PARIS_OK && out_bf16) rc = raw_bf16_launch(db[b], m, len, out_bf16 + (size_t)c0 * len, st);
    if (e == cudaSuccess && rc == PARIS_OK) e = cudaEventRecord(consumed[b], st);
  }
  if (reader.joinable()) {
    if (e != cudaSuccess || rc != PARIS_OK) {  // let the reader finish its waits, then stop it
      std::lock_guard<std::mutex> lk(mu);
      failed = true;
    }
    reader.join();
  }
  if (e != cudaSuccess && rc == PARIS_OK) rc = cuda_error(e, "paris_summarize_file");
  cudaStreamSynchronize(cs);  // the pinned buffers are freed below
  for (int i = 0; i < NB; ++i) {
    if (hb[i]) cudaFreeHost(hb[i]);
    if (copied[i]) cudaEventDestroy(copied[i]);
  }
  for (int i = 0; i < 2; ++i) {
    if (db[i]) cudaFreeAsync(db[i], st);
    if (consumed[i]) cudaEventDestroy(consumed[i]);
    if (dcopied[i]) cudaEventDestroy(dcopied[i]);
  }
  if (cs) cudaStreamDestroy(cs);
  close(fd);
  return rc;
}
}  // namespace paris

extern "C" int paris_summarize_file(const char* path, int64_t offset, int64_t n, int32_t len, int32_t w, int32_t card,
                                    uint8_t* out_sax, uint16_t* out_bf16, int32_t direct_io, void* stream) {
  if (!path || !out_sax || n < 1 || n >= (int64_t(1) << 31) || offset < 0) {
    paris::set_error("paris_summarize_file: bad arguments");
    return PARIS_EINVAL;
  }
  if (len < 4 || len > 4096 || (len % 4) || w < 1 || w > 64 || (len % w) || (out_bf16 && (len % 8))) {
    paris::set_error("paris_summarize_file: unsupported (len=%d, w=%d)", len, w);
    return PARIS_ECONFIG;
  }
  paris::retain_pool();
  return paris::summarize_file_impl(path, offset, n, len, w, card, out_sax, out_bf16, direct_io, (cudaStream_t)stream);
}

// A raw file mapped read-only and registered with CUDA (its pages pinned): the exact
// search then reads the candidates' rows straight from it (zero-copy over PCIe), the
// RDC workers' random reads of the raw file.  Needs the file in host RAM.
extern "C" int paris_map_raw_file(const char* path, int64_t offset, int64_t bytes, void** out_ptr) {
  if (!path || !out_ptr || bytes <= 0 || offset < 0 || (offset % 4096)) {
    paris::set_error("paris_map_raw_file: bad arguments (offset must be page aligned)");
    return PARIS_EINVAL;
  }
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    paris::set_error("paris_map_raw_file: cannot open %s", path);
    return PARIS_EINVAL;
  }
  // a read-only shared mapping registered read-only (the page cache's own pages); where the
  // driver refuses that, a private writable mapping (pinning copies each page once)
  void* p = mmap(nullptr, (size_t)bytes, PROT_READ, MAP_SHARED | MAP_POPULATE, fd, offset);
  cudaError_t e = cudaErrorInvalidValue;
  if (p != MAP_FAILED) {
    e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly);
    if (e != cudaSuccess) {
      cudaGetLastError();
      munmap(p, (size_t)bytes);
      p = MAP_FAILED;
    }
  }
  if (p == MAP_FAILED) {
    p = mmap(nullptr, (size_t)bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_POPULATE, fd, offset);
    if (p != MAP_FAILED) {
      e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterMapped);
      if (e != cudaSuccess) {
        munmap(p, (size_t)bytes);
        p = MAP_FAILED;
      }
    }
  }
  close(fd);
  if (p == MAP_FAILED) {
    if (e != cudaSuccess) return paris::cuda_error(e, "paris_map_raw_file: cudaHostRegister");
    paris::set_error("paris_map_raw_file: mmap of %lld bytes failed", (long long)bytes);
    return PARIS_ENOMEM;
  }
  *out_ptr = p;
  return PARIS_OK;
}

extern "C" int paris_unmap_raw_file(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return PARIS_EINVAL;
  cudaHostUnregister(ptr);
  munmap(ptr, (size_t)bytes);
  cudaGetLastError();
  return PARIS_OK;
}
