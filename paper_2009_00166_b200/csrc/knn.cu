// K2-K7 -- paris_knn_exact: ParIS+ ExactSearch (Alg9) on one B200.
//
//   k_seed        (K2+K3a) query PAA (fp64) -> fp32 interval + packed fp16 pairs;
//                 batched fp16 lower bound over a prefix sample of the SAX array,
//                 per-warp LB-best series = the approximate-search analog
//                 (reading R8)
//   k_seed_ed     (K3b) true distance of each seed series
//   k_seed_select (K3c) tau_seed^2 = k-th best seed d^2 (rounded up)
//   k_lb          (K4) LBC pass (Alg10): MINDIST_PAA_iSAX
//                  of every word for up to 16 queries per SAX read,
//                 in packed fp16x2 (two queries per instruction); a series that
//                 passes the fp16 test gets a rigorous fp32 LB and is compacted
//                 as (LB^2 bits << 32 | id) + a 256-bin LB histogram
//   k_scatter     (K5) candidates bucket-sorted by LB (256 bins over [0, tau^2])
//   k_refine1     (K6, k = 1) RDC pass (Alg11): warp per candidate in
//                 LB order, LB re-checked against the live BSF, true ED
//                 with early abandoning, BSF = 64-bit atomicMin on (d^2 bits, id)
//   k_refine_topk (K6, k > 1) same, in CTA-synchronous rounds that merge the
//                 round's admitted series into a CTA top-k; BSF = k-th best
//                 shared through atomicMin on float bits
//   k_finalize*   (K7) result rows ascending (d^2, id), sqrt
//
// Exactness: every LB is a rigorous lower bound of the exact
// MINDIST (outward-rounded bounds, directed rounding, fp16 error budget), every
// pruning threshold a rigorous upper bound of a real series' exact d^2 (fp32
// d^2 scaled by d2up), so pruning never drops a series of the exact answer.
#include "runtime.cuh"

#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <vector>

namespace paris {

int summarize_impl(const float*, int64_t, int, int, int, uint8_t*, cudaStream_t);
int knn_large_k(const float* raw, int64_t n, int len, const float* queries, int nq, int k, int64_t* out_idx,
                float* out_dist, cudaStream_t st);

namespace {

constexpr int kMaxW = 64;
constexpr int kNB = 256;            // LB histogram bins per query
constexpr int kMaxB = 64;           // queries per SAX pass (index path)
constexpr int kMaxBFlat = 16;       // queries per SAX pass (flat path: P <= 8 pairs)
constexpr int kLBThreads = 256;
constexpr int kRefThreads = 256;
constexpr int kRefWarps = kRefThreads / 32;
constexpr int kU = 4;               // candidates in flight per warp (refine)
constexpr int kSortP = 4096;        // finalize / seed-select sort buffer
constexpr int kMaxSeed = 4096;      // seed entries per query
constexpr uint64_t kNoKey = ~0ull;
// Per-query words hammered by every warp of a query (BSF key, k-NN threshold) sit
// 128 B apart, one L2 line each: 16 queries on one line serialized the refine.
constexpr int kPadU32 = 32;
constexpr int kPadU64 = 16;
constexpr uint32_t kHalf2One = 0x3C003C00u;
constexpr uint32_t kHalfNeg1 = 0xBC00u;


__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t make_key(float v, uint32_t id) {
  return ((uint64_t)__float_as_uint(v) << 32) | id;
}
__device__ __forceinline__ float key_val(uint64_t k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return (uint32_t)k; }

// Bin of a candidate's LB^2 in [0, thr]; scale = kNB/thr (0 if thr is 0 or inf).
__device__ __forceinline__ int lb_bin(float lb, float scale) {
  float f = lb * scale;
  int b = (int)f;
  return b < 0 ? 0 : (b >= kNB ? kNB - 1 : b);
}
__device__ __forceinline__ float bin_scale(float thr) {
  return (thr > 0.f && thr < INFINITY) ? (float)kNB / thr : 0.f;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// ---------------------------------------------------------------- packed fp16 ops
__device__ __forceinline__ uint32_t h2_fma_relu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.relu.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t h2_max(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t h2_min(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t h2_fma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// acc += delta^2 for one (series, segment) of a query pair, delta = max(a, b) where
// a = relu(q_lo - U) and b = relu(L - q_hi).  At most one of a, b is non-zero (U >= L
// and q_lo <= q_hi hold for the rounded values), so a^2 + b^2 in two FMAs is the
// same single rounding as max-then-FMA (fma(0, 0, acc) == acc exactly): bit-identical
// results, with the ALU-pipe max traded for an FMA-pipe op (PARIS_LB_NOMAX=1).
#ifndef PARIS_LB_NOMAX
#define PARIS_LB_NOMAX 0
#endif
__device__ __forceinline__ uint32_t h2_acc_delta2(uint32_t acc, uint32_t a, uint32_t b) {
#if PARIS_LB_NOMAX
  return h2_fma(b, b, h2_fma(a, a, acc));
#else
  const uint32_t d = h2_max(a, b);
  return h2_fma(d, d, acc);
#endif
}
// bit 0: low half a <= b; bit 1: high half a <= b
__device__ __forceinline__ uint32_t h2_le_bits(uint32_t a, uint32_t b) {
  const unsigned m = __hle2_mask(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
  return (m & 1u) | ((m >> 15) & 2u);
}
__device__ __forceinline__ float h_lo_f(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v & 0xFFFFu))); }
__device__ __forceinline__ float h_hi_f(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v >> 16))); }

template <bool AL>
__device__ __forceinline__ uint32_t load_word(const uint8_t* __restrict__ sax, int64_t n, int s,
                                              int64_t i0) {
  const uint8_t* p = sax + (size_t)s * n + i0;
  if (AL) return __ldg(reinterpret_cast<const uint32_t*>(p));
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (i0 + j < n) v |= (uint32_t)__ldg(p + j) << (8 * j);
  return v;
}

// ---------------------------------------------------------------- lower bounds
// Batched fp16 MINDIST: for 4 series (the bytes of `word`) and P
// query pairs, one segment.  Branches ABOVE / BELOW / IN (the paper's three
// masked SIMD branches) become relu(q_lo - U), relu(L - q_hi) and their max:
//   a = relu(q_lo16 - U16), b = relu(L16 - q_hi16), delta = max(a, b),
//   acc += delta^2                          (3 fp16x2 FMA-pipe ops per 2 queries)
// q_lo16 <= q, q_hi16 >= q, L16 <= L, U16 >= U, so the exact-arithmetic value is
// <= the exact delta; round-to-nearest error is bounded in k_lb (T16).
template <int P>
__device__ __forceinline__ void lb16_seg(uint32_t word, const uint2* __restrict__ q16s,
                                         const uint2* __restrict__ s_lu16, uint32_t (&acc)[4][P]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint2 t = s_lu16[(word >> (8 * j)) & 0xFFu];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint2 q = q16s[p];
      const uint32_t a = h2_fma_relu(q.x, kHalf2One, t.x);
      const uint32_t b = h2_fma_relu(q.y, kHalf2One, t.y);
      acc[j][p] = h2_acc_delta2(acc[j][p], a, b);
    }
  }
}

// fp16 accumulators of 4 consecutive series i0..i0+3 against P pairs.
// WT: compile-time w (all words loaded up front) or 0 (runtime w).
template <int P, int WT, bool AL>
__device__ __forceinline__ void lb16_group(const uint8_t* __restrict__ sax, int64_t n, int w,
                                           int64_t i0, const uint2* __restrict__ s_q16,
                                           const uint2* __restrict__ s_lu16, uint32_t (&acc)[4][P]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int p = 0; p < P; ++p) acc[j][p] = 0u;
  if (WT > 0) {
    uint32_t wd[WT > 0 ? WT : 1];
#pragma unroll
    for (int s = 0; s < WT; ++s) wd[s] = load_word<AL>(sax, n, s, i0);
#pragma unroll
    for (int s = 0; s < WT; ++s) lb16_seg<P>(wd[s], s_q16 + s * P, s_lu16, acc);
  } else {
    uint32_t nxt = load_word<AL>(sax, n, 0, i0);
    for (int s = 0; s < w; ++s) {
      const uint32_t cur = nxt;
      if (s + 1 < w) nxt = load_word<AL>(sax, n, s + 1, i0);
      lb16_seg<P>(cur, s_q16 + s * P, s_lu16, acc);
    }
  }
  if (i0 + 3 >= n) {  // tail: absent series are +inf
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i0 + j >= n)
#pragma unroll
        for (int p = 0; p < P; ++p) acc[j][p] = 0x7C007C00u;
  }
}

// Query PAA in fp64 (segment means) for the B = 2P slots of a batch:
// s_q[b*kMaxW + s] = {round-down, round-up} fp32 of the PAA, and the packed fp16
// pairs s_q16[s*P + p] = {half2(q_lo16[2p], q_lo16[2p+1]), half2(-q_hi16[2p], -q_hi16[2p+1])}
// with q_lo16 = fp16 round-down of q_lo and q_hi16 = round-up of q_hi, both
// clamped into [-60000, 60000] (a clamp only shrinks delta, so it stays sound).
// Slots b >= nb are dummies.  Optionally mirrored to global (block 0).
template <int P>
__device__ void query_prep(const float* __restrict__ queries, int nb, int len, int w,
                           float2* s_q, uint2* s_q16, float2* g_q, uint2* g_q16) {
  const int seglen = len / w;
  // one thread per (slot, segment) in use (the rest zeroed apart); the fp64 sum runs over
  // the segment's points in order (float4 loads when aligned: same order, same result)
  for (int i = threadIdx.x; i < 2 * P * kMaxW; i += blockDim.x) {
    if (i / kMaxW >= nb || i % kMaxW >= w) {
      s_q[i] = make_float2(0.f, 0.f);
      if (g_q) g_q[i] = make_float2(0.f, 0.f);
    }
  }
  const bool v4 = (seglen % 4 == 0) && ((reinterpret_cast<uintptr_t>(queries) & 15u) == 0) && (len % 4 == 0);
  for (int i = threadIdx.x; i < nb * w; i += blockDim.x) {
    const int b = i / w, s = i % w;
    const float* x = queries + (size_t)b * len + (size_t)s * seglen;
    double acc = 0.0;
    if (v4) {
      for (int j = 0; j < seglen; j += 4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(x + j));
        acc += (double)f.x; acc += (double)f.y; acc += (double)f.z; acc += (double)f.w;
      }
    } else {
      for (int j = 0; j < seglen; ++j) acc += (double)x[j];
    }
    const double paa = acc / (double)seglen;
    const float2 v = make_float2(__double2float_rd(paa), __double2float_ru(paa));
    s_q[b * kMaxW + s] = v;
    if (g_q) g_q[b * kMaxW + s] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * kMaxW; i += blockDim.x) {
    const int s = i / P, p = i % P;
    uint32_t lo2 = 0, nhi2 = 0;
    if (s < w) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 v = s_q[(2 * p + h) * kMaxW + s];
        const float lo = fminf(fmaxf(v.x, -60000.f), 60000.f);
        const float hi = fminf(fmaxf(v.y, -60000.f), 60000.f);
        const unsigned short l16 = __half_as_ushort(__float2half_rd(lo));
        const unsigned short h16 = __half_as_ushort(__float2half_ru(hi)) ^ 0x8000u;  // -q_hi16
        lo2 |= (uint32_t)l16 << (16 * h);
        nhi2 |= (uint32_t)h16 << (16 * h);
      }
    }
    s_q16[i] = make_uint2(lo2, nhi2);
    if (g_q16) g_q16[i] = make_uint2(lo2, nhi2);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- K2+K3a seed LB
// Every warp keeps its LB-best (LB, id) per query over the sample [0, ns).
template <int P, int WT, bool AL>
__global__ void __launch_bounds__(kLBThreads)
k_seed(const uint8_t* __restrict__ sax, int64_t n, int64_t ns, const float* __restrict__ queries,
       int nb, int len, int w, const CardTables* __restrict__ tab, float2* __restrict__ g_q,
       uint2* __restrict__ g_q16, int* __restrict__ seed_ids, int S) {
  __shared__ uint2 s_lu16[kMaxCard];
  __shared__ float2 s_q[2 * P * kMaxW];
  __shared__ uint2 s_q16[P * kMaxW];
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) s_lu16[i] = tab->lu16[i];
  query_prep<P>(queries, nb, len, w, s_q, s_q16, blockIdx.x == 0 ? g_q : nullptr,
                blockIdx.x == 0 ? g_q16 : nullptr);
  const int lane = threadIdx.x & 31;
  float best[2 * P];
  uint32_t bid[2 * P];
#pragma unroll
  for (int b = 0; b < 2 * P; ++b) { best[b] = INFINITY; bid[b] = 0xFFFFFFFFu; }
  const int64_t ngroups = (ns + 3) / 4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    uint32_t acc[4][P];
    lb16_group<P, WT, AL>(sax, n, w, i0, s_q16, s_lu16, acc);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j >= ns) break;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float lo = h_lo_f(acc[j][p]), hi = h_hi_f(acc[j][p]);
        if (lo < best[2 * p]) { best[2 * p] = lo; bid[2 * p] = (uint32_t)(i0 + j); }
        if (hi < best[2 * p + 1]) { best[2 * p + 1] = hi; bid[2 * p + 1] = (uint32_t)(i0 + j); }
      }
    }
  }
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
  for (int b = 0; b < 2 * P; ++b) {
    float v = best[b];
    uint32_t id = bid[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const uint32_t id2 = __shfl_xor_sync(0xffffffffu, id, o);
      if (v2 < v || (v2 == v && id2 < id)) { v = v2; id = id2; }
    }
    if (lane == 0 && b < nb && gwarp < S) seed_ids[b * S + gwarp] = (id == 0xFFFFFFFFu) ? -1 : (int)id;
  }
}

// ---------------------------------------------------------------- distance
// d^2 between raw[id] and the query in shared memory (warp-cooperative, one
// float4 per lane per 128-point chunk), no abandoning (seed pass).
// Summation: <= len/32 sequential fma per lane, then a 5-level xor tree, so
// |fp32 - exact| <= (len/32 + 8) * 2^-24 * d^2 (d2up in the host code covers it).
__device__ __forceinline__ float warp_ed2(const float* __restrict__ raw, uint32_t id, int len,
                                          const float4* __restrict__ s_qv) {
  const int lane = threadIdx.x & 31;
  const int nf = len >> 2;
  const float4* row = reinterpret_cast<const float4*>(raw + (size_t)id * len);
  float acc = 0.f;
  for (int f = lane; f < nf; f += 32) {
    const float4 x = ld_stream(row + f);
    const float4 q = s_qv[f];
    float d;
    d = x.x - q.x; acc = fmaf(d, d, acc);
    d = x.y - q.y; acc = fmaf(d, d, acc);
    d = x.z - q.z; acc = fmaf(d, d, acc);
    d = x.w - q.w; acc = fmaf(d, d, acc);
  }
  return warp_sum(acc);
}

// ---------------------------------------------------------------- K3b seed ED
__global__ void __launch_bounds__(kRefThreads)
k_seed_ed(const float* __restrict__ raw, int len, const float* __restrict__ queries,
          const int* __restrict__ seed_ids, int S, uint64_t* __restrict__ seed_keys) {
  extern __shared__ float4 s_qv[];
  const int b = blockIdx.y;
  const float4* qsrc = reinterpret_cast<const float4*>(queries + (size_t)b * len);
  for (int i = threadIdx.x; i < len / 4; i += blockDim.x) s_qv[i] = qsrc[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int j = blockIdx.x * nw + warp; j < S; j += gridDim.x * nw) {
    const int id = seed_ids[b * S + j];
    uint64_t key = kNoKey;
    if (id >= 0) key = make_key(warp_ed2(raw, (uint32_t)id, len, s_qv), (uint32_t)id);
    if (lane == 0) seed_keys[b * S + j] = key;
  }
}

// K3b with raw in host memory and its bf16 copy in HBM (f3 + paris_knn_index_x):
// the seeds' distances come from the bf16 rows as rigorous UPPER bounds,
// ED(q, x) <= ED(q, x~) + rho ||x~|| (bf16_prefilter's rho and fp32 margins, rounded
// up), so the seed needs no PCIe read.  tau_seed only has to bound the k-th NN
// distance from above; the seed series themselves are candidates (LB <= ED <= the
// bound) and get their exact distances in the refinement (k = 1 only).
__global__ void __launch_bounds__(kRefThreads)
k_seed_ed16(const uint16_t* __restrict__ raw16, int len, const float* __restrict__ queries,
            const int* __restrict__ seed_ids, int S, uint64_t* __restrict__ seed_keys) {
  extern __shared__ float4 s_qv[];
  const int b = blockIdx.y;
  const float4* qsrc = reinterpret_cast<const float4*>(queries + (size_t)b * len);
  for (int i = threadIdx.x; i < len / 4; i += blockDim.x) s_qv[i] = qsrc[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int nh = len >> 3;
  const float e2 = 2.f * (float)((len >> 5) + 8) * 5.9604644775390625e-08f;
  constexpr float rho = 0.00392150878906250f;
  for (int j = blockIdx.x * nw + warp; j < S; j += gridDim.x * nw) {
    const int id = seed_ids[b * S + j];
    uint64_t key = kNoKey;
    if (id >= 0) {
      const uint4* row = reinterpret_cast<const uint4*>(raw16 + (size_t)id * len);
      float s2 = 0.f, n2 = 0.f;
      for (int f = lane; f < nh; f += 32) {
        const uint4 h = __ldg(row + f);
        const float4 q0 = s_qv[2 * f], q1 = s_qv[2 * f + 1];
        const uint32_t w4[4] = {h.x, h.y, h.z, h.w};
        const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float x = __uint_as_float((e & 1) ? (w4[e >> 1] & 0xFFFF0000u) : (w4[e >> 1] << 16));
          const float d = x - qq[e];
          s2 = fmaf(d, d, s2);
          n2 = fmaf(x, x, n2);
        }
      }
      const float s = warp_sum(s2), nn = warp_sum(n2);
      const float hi = __fadd_ru(__fadd_ru(__fsqrt_ru(__fmul_ru(s, 1.f + e2)),
                                           __fmul_ru(rho, __fsqrt_ru(__fmul_ru(nn, 1.f + e2)))), 1e-30f);
      key = make_key(__fmul_ru(hi, hi), (uint32_t)id);
    }
    if (lane == 0) seed_keys[b * S + j] = key;
  }
}

// ---------------------------------------------------------------- bitonic sort (smem)
__device__ void bitonic_sort(uint64_t* buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int idx = 2 * i - (i & (stride - 1));
        const int pr = idx + stride;
        const bool asc = (idx & size) == 0;
        const uint64_t a = buf[idx], c = buf[pr];
        if ((a > c) == asc) { buf[idx] = c; buf[pr] = a; }
      }
      __syncthreads();
    }
  }
}

// 32 keys, one per lane, sorted ascending across the warp (lane i gets the i-th).
__device__ __forceinline__ uint64_t warp_sort32(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool up = ((lane & size) == 0);
      const bool low = ((lane & stride) == 0);
      v = (low == up) ? (v < o ? v : o) : (v < o ? o : v);
    }
  }
  return v;
}

// ---------------------------------------------------------------- K3c seed select
// tau_seed^2 = k-th smallest seed d^2 (an upper bound of the k-th NN distance,
// R8), rounded up by the fp32 error bound; +inf if < k seeds.  For k = 1 the best
// seed key also initializes the BSF (best[b]).
__global__ void __launch_bounds__(1024)
k_seed_select(const uint64_t* __restrict__ seed_keys, int S, int k, float d2up,
              unsigned* __restrict__ thr, unsigned* __restrict__ thr_seed,
              unsigned long long* __restrict__ best, float* __restrict__ tau_out, int q0) {
  __shared__ uint64_t buf[kSortP];
  __shared__ uint64_t s_red[32];
  const int b = blockIdx.x;
  uint64_t kth;
  if (k == 1) {
    uint64_t m = kNoKey;
    for (int i = threadIdx.x; i < S; i += blockDim.x) m = min(m, (uint64_t)seed_keys[b * S + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, (uint64_t)__shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      m = (threadIdx.x < (blockDim.x >> 5)) ? s_red[threadIdx.x] : kNoKey;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = min(m, (uint64_t)__shfl_xor_sync(0xffffffffu, m, o));
    }
    kth = m;
  } else {
    for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = (i < S) ? seed_keys[b * S + i] : kNoKey;
    __syncthreads();
    bitonic_sort(buf, kSortP);
    kth = buf[k - 1];
  }
  if (threadIdx.x == 0) {
    const float t = (kth == kNoKey) ? INFINITY : __fmul_ru(key_val(kth), d2up);
    thr[b * kPadU32] = __float_as_uint(t);
    thr_seed[b] = __float_as_uint(t);
    if (k == 1) best[b * kPadU64] = kth;
    if (tau_out) tau_out[q0 + b] = (kth == kNoKey) ? INFINITY : sqrtf(key_val(kth));
  }
}

// Seed from a previous result row (test hook config reserved[3]: the LB pass under an
// ideal BSF): tau^2 = (k-th returned distance)^2 rounded up (the fp32 sqrt/square round
// trip is covered by a further 2^-20), the k = 1 BSF key restarts from that row.
__global__ void k_seed_prev(const int64_t* __restrict__ prev_idx, const float* __restrict__ prev_dist, int nb,
                            int q0, int k, float d2up, unsigned* __restrict__ thr, unsigned* __restrict__ thr_seed,
                            unsigned long long* __restrict__ best) {
  const int b = threadIdx.x;
  if (b >= nb) return;
  const float d = prev_dist[(size_t)(q0 + b) * k + (k - 1)];
  const int64_t id = prev_idx[(size_t)(q0 + b) * k + (k - 1)];
  const bool ok = (id >= 0) && d < INFINITY;
  const float t = ok ? __fmul_ru(__fmul_ru(__fmul_ru(d, d), 1.00000096f), d2up) : INFINITY;
  thr[b * kPadU32] = __float_as_uint(t);
  thr_seed[b] = __float_as_uint(t);
  if (k == 1) best[b * kPadU64] = ok ? make_key(__fmul_ru(__fmul_ru(d, d), 1.00000096f), (uint32_t)id) : kNoKey;
}

// An external bound (paris_knn_config.tau_in, rooted distances): per query the pruning
// threshold becomes min(own seed, tau_in^2 rounded up); for k = 1 the BSF key starts no
// higher than (tau_in^2, sentinel id 0xFFFFFFFF) -- a bound, not a series: a row whose
// BSF is still the sentinel at the end has no series within the bound (-1 / +inf).
constexpr uint32_t kSentinelId = 0xFFFFFFFFu;
__global__ void k_tau_in(const float* __restrict__ tau_in, int nb, int q0, int k, float d2up,
                         unsigned* __restrict__ thr, unsigned* __restrict__ thr_seed,
                         unsigned long long* __restrict__ best) {
  const int b = threadIdx.x;
  if (b >= nb) return;
  const float d = tau_in[q0 + b];
  if (!(d < INFINITY)) return;
  const float d2 = __fmul_ru(__fmul_ru(fmaxf(d, 0.f), fmaxf(d, 0.f)), 1.00000096f);
  const float t = __fmul_ru(d2, d2up);
  thr[b * kPadU32] = min(thr[b * kPadU32], __float_as_uint(t));  // non-negative floats: bits order
  thr_seed[b] = min(thr_seed[b], __float_as_uint(t));
  if (k == 1) best[b * kPadU64] = min((uint64_t)best[b * kPadU64], make_key(d2, kSentinelId));
}

// Approximate k-NN (paris_knn_approx): the k best seed keys of each query, ascending.
__global__ void __launch_bounds__(1024)
k_seed_topk(const uint64_t* __restrict__ seed_keys, int S, int k, int q0, int64_t* __restrict__ out_idx,
            float* __restrict__ out_dist) {
  __shared__ uint64_t buf[kSortP];
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = (i < S) ? seed_keys[b * S + i] : kNoKey;
  __syncthreads();
  bitonic_sort(buf, kSortP);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = buf[i];
    const size_t o = (size_t)(q0 + b) * k + i;
    if (key == kNoKey) { out_idx[o] = -1; out_dist[o] = INFINITY; }
    else { out_idx[o] = (int64_t)key_id(key); out_dist[o] = sqrtf(key_val(key)); }
  }
}

// Index mode seed = approximate search: the leaf the query's own
// iSAX word would be inserted into.  One warp per query: the word (symbols of the
// query PAA midpoints; any word is sound, this one is the closest leaf), its key,
// a 32-ary search of the sorted array (lane l probes one position per round),
// then the S series around the insertion point become the seed set.
__global__ void __launch_bounds__(32)
k_approx_seed(const uint8_t* __restrict__ sax_sorted, const uint32_t* __restrict__ perm, int64_t n,
              const float2* __restrict__ g_q, const CardTables* __restrict__ tab, int card,
              int* __restrict__ seed_ids, int S) {
  const int b = blockIdx.x, lane = threadIdx.x;
  int shift = 0;
  while ((card << shift) < 256) ++shift;
  // symbol of segment `lane` (lanes 0..15)
  int sym = 0;
  if (lane < 16) {
    const float2 q = g_q[b * kMaxW + lane];
    const float v = 0.5f * (q.x + q.y);
    for (int step = card >> 1; step >= 1; step >>= 1)
      if (tab->cuts_f[sym + step - 1] <= v) sym += step;
  }
  uint8_t word[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) word[s] = (uint8_t)__shfl_sync(0xffffffffu, sym, s);
  const uint64_t target = isax_key16(word, shift);
  // lower_bound of target over keys(0..n-1); invariant: the answer lies in [lo, hi]
  int64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo) / 32;
    const int64_t pos = lo + step * (lane + 1) - 1;  // increasing in lane, all < hi
    uint8_t w2[16];
#pragma unroll
    for (int s = 0; s < 16; ++s)  // tile-major sorted SAX (include/paris.h)
      w2[s] = sax_sorted[(size_t)(pos / PARIS_INDEX_TILE) * 16 * PARIS_INDEX_TILE + (size_t)s * PARIS_INDEX_TILE +
                         pos % PARIS_INDEX_TILE];
    const int c = __popc(__ballot_sync(0xffffffffu, isax_key16(w2, shift) < target));  // a prefix of lanes
    const int64_t nlo = lo + step * c;
    hi = (c < 32) ? lo + step * (c + 1) - 1 : hi;
    lo = nlo;
  }
  const int64_t cnt = min((int64_t)S, n);
  int64_t start = lo - cnt / 2;
  start = max((int64_t)0, min(start, n - cnt));
  for (int t = lane; t < S; t += 32) {
    PARIS_DCHECK(t >= cnt || (start + t >= 0 && start + t < n));
    seed_ids[b * S + t] = (t < cnt) ? (int)perm[start + t] : -1;
  }
}

// ---------------------------------------------------------------- K4 LBC pass
// Alg10: for every word, LB < BSF -> append (LB, position).
// Here: up to 2P queries per SAX read, in packed fp16; warp-aggregated atomics
// reserve slots; count[b] keeps counting past `cap` (overflow detection).
//
// fp16 error budget: with u = 2^-11, a delta rounded once (relu-FMA) and squared
// into a running sum by w round-to-nearest FMAs is within (1+u)^(w+2) of its
// exact-input value (non-negative terms; relu keeps signs), plus at most w*2^-24
// of subnormal slack; the single-query form adds one fp32 add and one fp16
// round-up.  So, with G = (1+u)^(w+4):
//   LB16 <= LBexact_sum * G + w*2^-24                  (sum over s of delta^2).
// Hence (a) a series can only be a candidate if
//   LB16 <= T16 := tau^2/(len/w) * G + w*2^-24   (rounded up to fp16;
// above 64000 it is replaced by +inf: an fp16 overflow needs a sum >= 65520), and
// (b) LB^2 >= (LB16 - w*2^-24) * (len/w) / G is a rigorous lower bound,
// computed with round-down fp32 -- it is the LB stored in the candidate key.
struct LbArgs {
  const uint8_t* sax;
  int64_t n;
  int w;
  float seglen_f;
  const CardTables* tab;
  const float2* g_q;     // [2P][kMaxW]   fp32 query PAA intervals
  const uint2* g_q16;    // [kMaxW][P]    packed fp16 pairs
  int nb;
  const unsigned* thr;   // tau_seed^2 (float bits) per query
  unsigned* count;
  unsigned* hist;
  uint64_t* cand;
  int64_t cap;
  const uint32_t* perm;  // index mode: sorted position -> series id (else nullptr)
  const uint8_t* env;    // index mode: [n/64 blocks][2][16] min/max symbols (else nullptr)
  unsigned* blocks;      // index mode: per query, blocks whose envelope bound passed
  const unsigned* skip_if = nullptr;  // k_lbt<P, 1>: leave at once if *skip_if != 0 (k_gf took the pass)
};

struct LbConsts {
  uint32_t T16[kMaxB / 2];   // fp16 thresholds, packed per pair
  float thr[kMaxB];          // tau^2 (rounded up), -1 for dummy slots
  float scale[kMaxB];        // histogram bin scale
  float lbconv;              // (len/w) / (1+u)^(w+3), rounded down
  float wabs;                // w * 2^-24
};

__device__ void lb_consts_init(const LbArgs& a, int nslots, LbConsts* c) {
  if (threadIdx.x < nslots) {
    const int b = threadIdx.x;
    const float t = (b < a.nb) ? __uint_as_float(a.thr[b]) : -1.f;
    c->thr[b] = t;
    c->scale[b] = bin_scale(t);
  }
  if (threadIdx.x == 0) {
    const double grow = pow(1.0 + 1.0 / 2048.0, (double)(a.w + 4)) * (1.0 + 1e-12);
    c->lbconv = __double2float_rd((double)a.seglen_f / grow);
    c->wabs = (float)a.w * 5.9604644775390625e-08f;
  }
  __syncthreads();
  if (threadIdx.x < (nslots + 1) / 2) {
    uint32_t t2 = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = 2 * threadIdx.x + h;
      const float t = (b < nslots) ? c->thr[b] : -1.f;
      unsigned short hb;
      if (t < 0.f) {
        hb = (unsigned short)kHalfNeg1;  // dummy slot: never passes
      } else {
        const double grow = pow(1.0 + 1.0 / 2048.0, (double)(a.w + 4)) * (1.0 + 1e-12);
        const double T = (double)t / (double)a.seglen_f * grow + (double)a.w * 5.9604644775390625e-08;
        hb = (T > 64000.0) ? (unsigned short)0x7C00u
                           : __half_as_ushort(__float2half_ru(__double2float_ru(T)));
      }
      t2 |= (uint32_t)hb << (16 * h);
    }
    c->T16[threadIdx.x] = t2;
  }
  __syncthreads();
}

// Candidate emission for 4 series i0..i0+3 (nvalid of them real) and 2P query
// slots whose fp16 sums are acc[j][p] (slot 2p low half, 2p+1 high half).
// Whole warp must call it (warp-aggregated atomics).
// slot0: global query slot of local slot 0 (index mode computes one pair at a time)
template <int P>
__device__ __forceinline__ void lb_emit(const uint32_t (&acc)[4][P], int64_t i0, int nvalid,
                                        const LbConsts& c, const LbArgs& a,
                                        uint32_t slot_mask = 0xFFFFFFFFu, const uint32_t* perm = nullptr,
                                        int slot0 = 0) {
  const int lane = threadIdx.x & 31;
  uint32_t qm = 0;
  if (nvalid > 0) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t mn = h2_min(h2_min(acc[0][p], acc[1][p]), h2_min(acc[2][p], acc[3][p]));
      qm |= h2_le_bits(mn, c.T16[p + (slot0 >> 1)]) << (2 * p);
    }
    qm &= slot_mask;
  }
  if (!__any_sync(0xffffffffu, qm != 0)) return;
  uint32_t wq = __reduce_or_sync(0xffffffffu, qm);
  while (wq) {
    const int b = __ffs(wq) - 1;
    wq &= wq - 1;
    unsigned m = 0;
    float lbv[4];
    if ((qm >> b) & 1u) {
      const uint32_t T = c.T16[(b + slot0) >> 1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t v = 0;
#pragma unroll
        for (int p = 0; p < P; ++p)
          if (p == (b >> 1)) v = acc[j][p];
        const uint32_t pass = (h2_le_bits(v, T) >> (b & 1)) & 1u;
        const float h = (b & 1) ? h_hi_f(v) : h_lo_f(v);
        lbv[j] = __fmul_rd(fmaxf(__fsub_rd(h, c.wabs), 0.f), c.lbconv);
        if (pass && j < nvalid && lbv[j] <= c.thr[b + slot0]) m |= 1u << j;
      }
    }
    const int cnt = __popc(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    unsigned base = 0;
    if (lane == 31) base = atomicAdd(&a.count[b + slot0], (unsigned)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    uint64_t pos = (uint64_t)base + (unsigned)(incl - cnt);
    const float sc = c.scale[b + slot0];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (m & (1u << j)) {
        if (pos < (uint64_t)a.cap) {
          a.cand[(size_t)(b + slot0) * a.cap + pos] = make_key(lbv[j], perm ? __ldg(perm + i0 + j) : (uint32_t)(i0 + j));
          atomicAdd(&a.hist[(b + slot0) * kNB + lb_bin(lbv[j], sc)], 1u);
        }
        ++pos;
      }
    }
  }
}

// Warp-private candidate staging in shared memory (tiled kernel): a warp appends
// its candidates (key + query slot) with shared-memory atomics only; when the
// buffer would overflow (and at the end) the warp flushes it: one global
// atomicAdd per query slot reserves the slots of all its entries at once.
constexpr int kWB = 128;
struct WarpBuf {
  uint64_t key[kWB];
  uint8_t slot[kWB];
  unsigned cnt[kMaxB];   // entries per slot
  unsigned cur[kMaxB];   // flush cursors
  int n;
};

// Shared-memory LB histogram of 64 slots in 16-bit halves (32 KB instead of 64):
// word i/2 holds bins i (low half) and i+1 (high half).  The increment that takes a
// half to 0x8000 moves 0x8000 to the global histogram, so a half never carries
// into its neighbour (at most a CTA's threads increment it in between).
__device__ __forceinline__ void hist16_add(unsigned* s_h16, int idx, unsigned* g_hist) {
  const unsigned sh = (unsigned)(idx & 1) * 16u;
  const unsigned old = atomicAdd(&s_h16[idx >> 1], 1u << sh);
  if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {
    atomicSub(&s_h16[idx >> 1], 0x8000u << sh);
    atomicAdd(&g_hist[idx], 0x8000u);
  }
}

// s_hist: the CTA's shared-memory LB histogram (flushed at kernel end).  HMODE 0:
// [kMaxB][kNB] 32-bit; 1: the packed 16-bit form (hist16_add); 2: coarse, kNBC
// 32-bit bins per slot (bin >> 3) -- enough for the k = 1 wave cut, which only needs
// a quantile (flushed to fine bin 8c + 7 of each coarse group c).
constexpr int kNBC = kNB / 8;
template <int HMODE = 0>
__device__ void wb_flush(WarpBuf& wb, int nslots, const LbConsts& c, const LbArgs& a, unsigned* s_hist) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int m = wb.n;
  if (m == 0) return;
  for (int b = lane; b < nslots; b += 32) {
    const unsigned k = wb.cnt[b];
    wb.cur[b] = k ? atomicAdd(&a.count[b], k) : 0u;
    wb.cnt[b] = 0;
  }
  __syncwarp();
  for (int e = lane; e < m; e += 32) {
    const int b = wb.slot[e];
    const uint64_t key = wb.key[e];
    PARIS_DCHECK(b < nslots && key_id(key) < (uint64_t)a.n);
    const unsigned pos = atomicAdd(&wb.cur[b], 1u);
    // only stored candidates enter the histogram: on overflow (count > cap) the
    // bucket offsets must describe exactly the `cap` entries K5 orders
    if ((int64_t)pos < a.cap) {
      a.cand[(size_t)b * a.cap + pos] = key;
      const int bin = lb_bin(key_val(key), c.scale[b]);
      if (HMODE == 1) hist16_add(s_hist, b * kNB + bin, a.hist);
      else if (HMODE == 2) atomicAdd(&s_hist[b * kNBC + (bin >> 3)], 1u);
      else atomicAdd(&s_hist[b * kNB + bin], 1u);
    }
  }
  __syncwarp();
  if (lane == 0) wb.n = 0;
  __syncwarp();
}

// slot_mask: query slots this warp's block may hold candidates for (index mode);
// perm: sorted position -> series id (index mode), nullptr = identity.
template <int P>
__device__ __forceinline__ void lb_emit_wb(const uint32_t (&acc)[4][P], int64_t i0, int nvalid, int nslots,
                                           const LbConsts& c, const LbArgs& a, WarpBuf& wb, unsigned* s_hist,
                                           uint32_t slot_mask = 0xFFFFFFFFu, const uint32_t* perm = nullptr,
                                           int slot0 = 0) {
  const int lane = threadIdx.x & 31;
  uint32_t qm = 0;
  if (nvalid > 0) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t mn = h2_min(h2_min(acc[0][p], acc[1][p]), h2_min(acc[2][p], acc[3][p]));
      qm |= h2_le_bits(mn, c.T16[p + (slot0 >> 1)]) << (2 * p);
    }
    qm &= slot_mask;
  }
  if (!__any_sync(0xffffffffu, qm != 0)) return;
  // pass 1: this lane's candidate count; pass 2 writes (lane-local loops over set bits)
  int cntl = 0;
  for (uint32_t r = qm; r; r &= r - 1) {
    const int b = __ffs(r) - 1;
    const uint32_t T = c.T16[(b + slot0) >> 1];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t v = 0;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p == (b >> 1)) v = acc[j][p];
      const float h = (b & 1) ? h_hi_f(v) : h_lo_f(v);
      const float lb = __fmul_rd(fmaxf(__fsub_rd(h, c.wabs), 0.f), c.lbconv);
      if (((h2_le_bits(v, T) >> (b & 1)) & 1u) && j < nvalid && lb <= c.thr[b + slot0]) ++cntl;
    }
  }
  int incl = cntl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  if (wb.n + total > kWB) wb_flush(wb, nslots, c, a, s_hist);
  if (total > kWB) {  // degenerate (e.g. tau = inf): straight to global memory
    lb_emit<P>(acc, i0, nvalid, c, a, qm, perm, slot0);
    return;
  }
  int pos = wb.n + incl - cntl;
  for (uint32_t r = qm; r; r &= r - 1) {
    const int b = __ffs(r) - 1;
    const uint32_t T = c.T16[(b + slot0) >> 1];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t v = 0;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p == (b >> 1)) v = acc[j][p];
      const float h = (b & 1) ? h_hi_f(v) : h_lo_f(v);
      const float lb = __fmul_rd(fmaxf(__fsub_rd(h, c.wabs), 0.f), c.lbconv);
      if (((h2_le_bits(v, T) >> (b & 1)) & 1u) && j < nvalid && lb <= c.thr[b + slot0]) {
        PARIS_DCHECK(i0 + j < a.n && pos < kWB);
        wb.key[pos] = make_key(lb, perm ? __ldg(perm + i0 + j) : (uint32_t)(i0 + j));
        wb.slot[pos] = (uint8_t)(b + slot0);
        atomicAdd(&wb.cnt[b + slot0], 1u);
        ++pos;
      }
    }
  }
  __syncwarp();
  if (lane == 31) wb.n += total;
  __syncwarp();
}

// Direct-load variant (any n, any w <= 64): a thread loads the 4-series words of
// every segment row straight from global memory.
template <int P, int WT, bool AL>
__global__ void __launch_bounds__(kLBThreads)
k_lb(LbArgs a) {
  __shared__ uint2 s_lu16[kMaxCard];
  __shared__ uint2 s_q16[P * kMaxW];
  __shared__ LbConsts s_c;
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) s_lu16[i] = a.tab->lu16[i];
  for (int i = threadIdx.x; i < P * kMaxW; i += blockDim.x) s_q16[i] = a.g_q16[i];
  lb_consts_init(a, 2 * P, &s_c);
  const int lane = threadIdx.x & 31;
  const int64_t n = a.n;
  const int64_t ngroups = (n + 3) / 4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g - lane < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    uint32_t acc[4][P];
    int nvalid = 0;
    if (g < ngroups) {
      lb16_group<P, WT, AL>(a.sax, n, a.w, i0, s_q16, s_lu16, acc);
      nvalid = (int)imin64(4, n - i0);
    }
    lb_emit<P>(acc, i0, nvalid, s_c, a);
  }
}

// ---------------------------------------------------------------- K3a/K4 tiled (TMA) variant
// n % 16 == 0 and w == 16 (every BASELINE config): a persistent CTA per SM streams
// SAX tiles of kTS series x 16 segment rows into a kStages-deep shared-memory ring
// with cp.async.bulk (one bulk copy per row, completion on an mbarrier), so HBM
// reads run ahead of the lookups; the last warp to finish a stage refills it.
// The region table is replicated 32x in shared memory (entry c of lane l at word
// c*32 + l) so the per-series lookups are bank-conflict free.
constexpr int kTS = 2048;
constexpr int kTThreads = 512;
constexpr int kTWarps = kTThreads / 32;
constexpr int kBPT = 2048 / PARIS_INDEX_BLOCK;  // index blocks per tile (32: one per lane)
constexpr int kStages = 4;
constexpr int kTW = 16;
constexpr size_t kTileBytes = (size_t)kTW * kTS;
constexpr size_t kTSmem = kStages * kTileBytes + kMaxCard * 32 * 4;
#ifndef PARIS_BM_CTAS
#define PARIS_BM_CTAS 8
#endif
constexpr int kBmCtas = PARIS_BM_CTAS;  // block-pass CTAs per SM in the grid (tuning)
constexpr size_t kIHistBytes = (size_t)kMaxB * kNB * 2;  // k_lbi !HC: 16-bit LB histograms

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
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 8-byte shared-memory load at a 32-bit shared address (base + offset folds into
// one LDS [R + UR] when the base is uniform).
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
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

// Pair form for one segment word (4 series) from the replicated table.
template <int P>
__device__ __forceinline__ void lbt_seg(uint32_t word, const uint32_t* __restrict__ tabl,
                                        const uint2* __restrict__ q16s, uint32_t (&acc)[4][P]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t t = tabl[__byte_perm(word, 0, 0x4440 | j) * 32];  // (-U16, L16)
    const uint32_t tx = __byte_perm(t, 0, 0x1010);                    // (-U16, -U16)
    const uint32_t ty = __byte_perm(t, 0, 0x3232);                    // (L16, L16)
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint2 q = q16s[p];
      const uint32_t a = h2_fma_relu(q.x, kHalf2One, tx);
      const uint32_t b = h2_fma_relu(q.y, kHalf2One, ty);
      acc[j][p] = h2_acc_delta2(acc[j][p], a, b);
    }
  }
}

// Single-query form (B = 1): qd = half2(q_lo16, -q_hi16) against (-U16, L16):
// one relu-FMA gives (relu(q-U), relu(L-q)), one FMA accumulates both halves
// (at most one is non-zero); the LB sum is lo + hi at the end.
__device__ __forceinline__ void lbt_seg1(uint32_t word, const uint32_t* __restrict__ tabl, uint32_t qd,
                                         uint32_t (&acc)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t t = tabl[__byte_perm(word, 0, 0x4440 | j) * 32];
    const uint32_t d = h2_fma_relu(qd, kHalf2One, t);
    acc[j] = h2_fma(d, d, acc[j]);
  }
}

// MODE 0: seed (per-warp LB-best series per query over [0, nlim));
// MODE 1: LB pass with candidate emission over [0, nlim = n).
// P = 0: single query (slot 0).  nlim % 16 == 0.
template <int P, int MODE>
__global__ void __launch_bounds__(kTThreads, 1)
k_lbt(LbArgs a, int64_t nlim, int* __restrict__ seed_ids, int S) {
  if (MODE == 1 && a.skip_if && *a.skip_if) return;
  constexpr int PP = P > 0 ? P : 1;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* s_tiles = dsm;
  uint32_t* s_tab = reinterpret_cast<uint32_t*>(dsm + kStages * kTileBytes);
  __shared__ __align__(8) uint64_t s_full[kStages];
  __shared__ unsigned s_cnt[kStages];
  __shared__ uint2 s_q16[PP * kTW];
  __shared__ LbConsts s_c;
  __shared__ WarpBuf s_wb[MODE == 1 ? kTWarps : 1];
  __shared__ unsigned s_hist[MODE == 1 ? kMaxBFlat * kNB : 1];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ntiles = (nlim + kTS - 1) / kTS;
  const int nslots = P > 0 ? 2 * P : 1;
  WarpBuf& wb = s_wb[MODE == 1 ? (tid >> 5) : 0];
  if (MODE == 1) {
    for (int b = lane; b < kMaxB; b += 32) wb.cnt[b] = 0;
    if (lane == 0) wb.n = 0;
    for (int i = tid; i < nslots * kNB; i += kTThreads) s_hist[i] = 0;
  }

  auto issue = [&](int64_t tile, int st) {
    const int64_t base = tile * kTS;
    const unsigned bytes = (unsigned)imin64(kTS, nlim - base);
    mbar_expect_tx(&s_full[st], bytes * kTW);
    uint8_t* dst = s_tiles + (size_t)st * kTileBytes;
#pragma unroll 1
    for (int s = 0; s < kTW; ++s)
      bulk_g2s(dst + (size_t)s * kTS, a.sax + (size_t)s * a.n + base, bytes, &s_full[st]);
  };

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&s_full[st], 1);
      s_cnt[st] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles) issue(tile, st);
    }
  }
  for (int i = tid; i < kMaxCard * 32; i += kTThreads) s_tab[i] = a.tab->lu16p[i >> 5];
  if (P > 0) {
    for (int i = tid; i < PP * kTW; i += kTThreads) s_q16[i] = a.g_q16[i];
  } else if (tid < kTW) {
    // single query: (q_lo16, -q_hi16) of slot 0, repacked from the pair layout (low halves)
    const uint2 v = a.g_q16[tid];
    s_q16[tid] = make_uint2((v.x & 0xFFFFu) | (v.y << 16), 0u);
  }
  lb_consts_init(a, P > 0 ? 2 * P : 1, &s_c);   // ends with __syncthreads
  const uint32_t* tabl = s_tab + lane;

  float best[MODE == 0 ? 2 * PP : 1];
  uint32_t bid[MODE == 0 ? 2 * PP : 1];
  if (MODE == 0) {
#pragma unroll
    for (int b = 0; b < (MODE == 0 ? 2 * PP : 1); ++b) { best[b] = INFINITY; bid[b] = 0xFFFFFFFFu; }
  }

  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= ntiles) break;
    const int st = (int)(it % kStages);
    mbar_wait(&s_full[st], (unsigned)((it / kStages) & 1));
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(s_tiles + (size_t)st * kTileBytes);
    const int64_t i0 = tile * kTS + 4 * tid;
    const int nvalid = (int)std::max<int64_t>(0, imin64(4, nlim - i0));
    uint32_t acc[4][PP];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int p = 0; p < PP; ++p) acc[j][p] = 0u;
    if (P > 0) {
#pragma unroll 2
      for (int s = 0; s < kTW; ++s) lbt_seg<PP>(rows[s * (kTS / 4) + tid], tabl, s_q16 + s * PP, acc);
    } else {
      uint32_t a1[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int s = 0; s < kTW; ++s) lbt_seg1(rows[s * (kTS / 4) + tid], tabl, s_q16[s].x, a1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // lo + hi (ABOVE and BELOW sums), rounded up to fp16 (inside the G budget);
        // the unused high slot is +inf so it never passes
        const float v = h_lo_f(a1[j]) + h_hi_f(a1[j]);
        const __half hv = __float2half_ru(v);
        acc[j][0] = (uint32_t)__half_as_ushort(hv) | (0x7C00u << 16);
      }
    }
    __syncwarp();
    if (lane == 0) {
      // stage consumed by this warp; the last warp refills it with the tile kStages ahead
      if (atomicAdd(&s_cnt[st], 1u) == kTWarps - 1) {
        s_cnt[st] = 0;
        const int64_t next = tile + (int64_t)kStages * gridDim.x;
        if (next < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(next, st);
        }
      }
    }
    if (MODE == 1) {
      lb_emit_wb<PP>(acc, i0, nvalid, nslots, s_c, a, wb, s_hist);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= nvalid) break;
#pragma unroll
        for (int p = 0; p < PP; ++p) {
          const float lo = h_lo_f(acc[j][p]), hi = h_hi_f(acc[j][p]);
          if (lo < best[2 * p]) { best[2 * p] = lo; bid[2 * p] = (uint32_t)(i0 + j); }
          if (P > 0 && hi < best[2 * p + 1]) { best[2 * p + 1] = hi; bid[2 * p + 1] = (uint32_t)(i0 + j); }
        }
      }
    }
  }
  if (MODE == 1) {
    wb_flush(wb, nslots, s_c, a, s_hist);
    __syncthreads();
    for (int i = tid; i < nslots * kNB; i += kTThreads)
      if (s_hist[i]) atomicAdd(&a.hist[i], s_hist[i]);
  }
  if (MODE == 0) {
    const int gwarp = (blockIdx.x * kTThreads + tid) >> 5;
#pragma unroll
    for (int b = 0; b < (MODE == 0 ? 2 * PP : 1); ++b) {
      float v = best[b];
      uint32_t id = bid[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const uint32_t id2 = __shfl_xor_sync(0xffffffffu, id, o);
        if (v2 < v || (v2 == v && id2 < id)) { v = v2; id = id2; }
      }
      if (lane == 0 && b < a.nb && gwarp < S) seed_ids[b * S + gwarp] = (id == 0xFFFFFFFFu) ? -1 : (int)id;
    }
  }
}

// ---------------------------------------------------------------- index mode LB (f1)
// Pass 1 (k_blkmask): the envelope MINDIST of every 64-series block for every
// query slot (the iSAX node bound): bit b of bmask[blk] = block may hold a
// candidate of slot b.  A warp covers the 32 blocks of one SAX tile and appends
// the tile to a work list when any of its blocks is live.
// Pass 2 (k_lbi): a producer warp streams the listed tiles through a ring of
// NST stages (full/empty mbarrier pairs); the live (block, query pair) items of a
// tile are claimed dynamically by the consumer warps, a half-warp per item.
__device__ __forceinline__ uint32_t half_of(uint32_t v, int h) { return (v >> (16 * h)) & 0xFFFFu; }

// Shared-memory plan of k_lbi (dynamic shared memory only; S0 = its shared address,
// T = the 64 KB boundary above it):
//   [S0, S0 + 32K)         ring stage 0
//   [S0 + 32K, T)          misc (LbiMisc): barriers, per-stage tile id / claim counter /
//                          block masks, LbConsts, per-warp candidate slots and counters
//   [T, T + 64K)           region table half2(-U16, L16) (the single-query form), 32 copies:
//                          entry c of lane l's copy at T + 256c + 4l (a lookup by 32 lanes
//                          hits 32 distinct banks).  Bytes [128, 256) of each 256-byte row
//                          are "holes" (128 B each, 256 of them):
//                            holes   0..63   per-slot query words half2(q_lo16, -q_hi16),
//                                            two copies (bytes 0..63 for half-warp 0, 64..127
//                                            for half-warp 1: 16-byte broadcast loads of two
//                                            different slots never share a bank)
//                            holes  64..183  per-warp candidate keys (kWBI per warp, NW <= 30)
//                            holes 192..255  coarse LB histograms (HC), a slot per hole
//   [T + 64K, ...)         ring stages 1 .. NST-1, then the 16-bit histograms (!HC)
// One byte permute of a SAX word with {lane * 4, -, T bits 16..31} is a lookup's whole
// shared address (the symbol lands in bits 8..15).
#ifndef PARIS_LBI_GROUPS
#define PARIS_LBI_GROUPS 2
#endif
// consumer groups: group g takes the tiles it = g, g + G, ... (its stages), so a warp sees
// every G-th tile and does ~G times the rounds per stage visit (the per-visit cost -- wait,
// arrive, the final empty claim -- is paid half as often)
constexpr int kIGroups = PARIS_LBI_GROUPS;
// one producer warp per consumer group (when the ring's stages split evenly over the
// groups): a group's refills never wait behind another group's slow tile
constexpr int kIProd = kIGroups;
// NW consumer warps (a template parameter of k_lbi: 24 by default, 30 = 1024 threads at
// <= 64 registers, paris_debug_set_variant key 0)
template <int NW>
constexpr int lbi_threads() { return (NW + kIProd) * 32; }
constexpr int kIHistHole = 192;
constexpr int kWBI = 64;                      // staged candidates per consumer warp
constexpr uint32_t kIStageBytes = (uint32_t)kTileBytes;
struct LbiWarp {
  uint8_t slot[kWBI];
  unsigned cnt[kMaxB];  // entries per slot; during a flush the slot's global cursor
  unsigned n;
  unsigned pad[3];
};
constexpr int kMaxItems = kBPT * (kMaxB / 2);  // items of a tile: 32 blocks x up to 32 slot pairs
template <int NW>
struct LbiMisc {
  uint64_t full[4], empty[4];
  int64_t tile[4];
  unsigned next[4];    // per stage: the next unclaimed item pair
  unsigned nitems[4];  // per stage: items of its tile
  LbConsts c;
  LbiWarp w[NW];
  // per stage: the tile's items, decoded by the producer from the block masks:
  // block | slot a << 8 | slot b << 16 (0xFF: none)
  uint32_t items[4][kMaxItems];
};
template <int NW>
constexpr size_t lbi_misc_bytes() { return (sizeof(LbiMisc<NW>) + 127) & ~(size_t)127; }
static_assert(kTileBytes + lbi_misc_bytes<30>() + 2048 <= 65536, "stage 0 + misc must fit below the table");
static_assert(64 + 4 * 30 <= kIHistHole, "key holes below the histogram holes");

__device__ __forceinline__ uint32_t hole_addr(uint32_t T, int h) { return T + 256u * (uint32_t)h + 128u; }
__device__ __forceinline__ uint32_t lbi_key_addr(uint32_t T, int warp, int e) {
  return hole_addr(T, 64 + 4 * warp + (e >> 4)) + 8u * (uint32_t)(e & 15);
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u2(uint32_t addr, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void atoms_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// LB histogram of a stored candidate: HC -> coarse bins (bin >> 3) in the holes; else
// the packed 16-bit form at hist16 (hist16_add).
template <bool HC>
__device__ __forceinline__ void lbi_hist(uint32_t T, unsigned* hist16, int b, int bin, unsigned* g_hist) {
  if (HC) atoms_add(hole_addr(T, kIHistHole + b) + 4u * (uint32_t)(bin >> 3), 1u);
  else hist16_add(hist16, b * kNB + bin, g_hist);
}

// Flush a warp's staged candidates: one global atomicAdd per query slot reserves the
// slots of all its entries; sorted positions become series ids through perm here
// (a warp's loads in parallel, off the per-item path).
template <bool HC>
__device__ void lbi_flush(LbiWarp& wb, uint32_t T, int warp, int nslots, const LbConsts& c, const LbArgs& a,
                          unsigned* hist16) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int m = (int)wb.n;
  if (m == 0) return;
  static_assert(kWBI == 64, "two entries per lane");
  uint64_t key[2];
  uint32_t id[2];
  int sl[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = lane + 32 * r;
    key[r] = e < m ? lds_u64(lbi_key_addr(T, warp, e)) : kNoKey;
    sl[r] = e < m ? wb.slot[e] : 0;
    id[r] = e < m ? __ldg(a.perm + key_id(key[r])) : 0u;
    if (e < m) atomicAdd(&wb.cnt[sl[r]], 1u);  // per-slot counts, here rather than per emission
  }
  __syncwarp();
  for (int b = lane; b < nslots; b += 32) {
    const unsigned k = wb.cnt[b];
    wb.cnt[b] = k ? atomicAdd(&a.count[b], k) : 0u;
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (lane + 32 * r >= m) continue;
    const int b = sl[r];
    const unsigned pos = atomicAdd(&wb.cnt[b], 1u);
    // only stored candidates enter the histogram (on overflow the wave cut must describe
    // the `cap` stored entries)
    if ((int64_t)pos < a.cap) {
      a.cand[(size_t)b * a.cap + pos] = make_key(key_val(key[r]), id[r]);
      lbi_hist<HC>(T, hist16, b, lb_bin(key_val(key[r]), c.scale[b]), a.hist);
    }
  }
  __syncwarp();
  for (int b = lane; b < nslots; b += 32) wb.cnt[b] = 0;
  if (lane == 0) wb.n = 0;
  __syncwarp();
}

// Candidate emission of one item per half-warp: 4 series x 2 query slots (sa = low half,
// sb = high half, sb < 0: none).  The packed fp16 test first (almost every item fails it
// everywhere), the rigorous fp32 bound (k_lb's error budget) only where a lane passed.
template <bool HC>
__device__ __forceinline__ void lbi_emit(const uint32_t (&acc)[4], int sa, int sb, int64_t i0, int nvalid,
                                         int nslots, const LbConsts& c, const LbArgs& a, LbiWarp& wb,
                                         uint32_t T, int warp, unsigned* hist16) {
  const int lane = threadIdx.x & 31;
  const uint32_t Tp = half_of(c.T16[sa >> 1], sa & 1) |
                      ((sb >= 0 ? half_of(c.T16[sb >> 1], sb & 1) : (uint32_t)kHalfNeg1) << 16);
  uint32_t pf = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) pf |= h2_le_bits(acc[j], Tp) << (2 * j);
  if (nvalid < 4) pf &= (1u << (2 * nvalid)) - 1u;
  if (sb < 0) pf &= 0x55u;
  if (!__any_sync(0xffffffffu, pf != 0u)) return;
  // room for every pair that passed the fp16 test (an upper bound of the appends)
  const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(pf));
  if ((int)wb.n + total > kWBI) lbi_flush<HC>(wb, T, warp, nslots, c, a, hist16);
  const bool direct = total > kWBI;  // degenerate (e.g. tau = inf): straight to global memory
  for (uint32_t r = pf; r; r &= r - 1) {  // the rigorous fp32 bound only for the passing pairs
    const int bit = __ffs(r) - 1;
    const int j = bit >> 1, sl = (bit & 1) ? sb : sa;
    uint32_t v = acc[0];  // acc[j]: explicit selects, no dynamic register indexing
    v = j == 1 ? acc[1] : v;
    v = j == 2 ? acc[2] : v;
    v = j == 3 ? acc[3] : v;
    const float hv = (bit & 1) ? h_hi_f(v) : h_lo_f(v);
    const float lb = __fmul_rd(fmaxf(__fsub_rd(hv, c.wabs), 0.f), c.lbconv);
    if (!(lb <= c.thr[sl])) continue;
    if (direct) {
      const unsigned pos = atomicAdd(&a.count[sl], 1u);
      if ((int64_t)pos < a.cap) {
        a.cand[(size_t)sl * a.cap + pos] = make_key(lb, __ldg(a.perm + i0 + j));
        const int fb = lb_bin(lb, c.scale[sl]);
        atomicAdd(&a.hist[sl * kNB + (HC ? (fb | 7) : fb)], 1u);
      }
    } else {
      // staged as (LB, sorted position); per-slot counts and ids are resolved at flush time
      const int pos = (int)atomicAdd(&wb.n, 1u);
      PARIS_DCHECK(i0 + j < a.n && pos < kWBI && sl >= 0);
      sts_u64(lbi_key_addr(T, warp, pos), make_key(lb, (uint32_t)(i0 + j)));
      wb.slot[pos] = (uint8_t)sl;
    }
  }
  __syncwarp();
}

// One lane per block: lane l of a warp bounds block 32*g + l against every query
// slot (region [L[min_s], U[max_s]] per segment, outward fp32, round-down sums);
// the 32 blocks of a warp step are one whole tile, so the warp lists it itself.
template <int P>
__global__ void __launch_bounds__(256)
k_blkmask(LbArgs a, unsigned long long* __restrict__ bmask, unsigned* __restrict__ tile_list,
          unsigned* __restrict__ tile_count, unsigned* __restrict__ blocks, unsigned* __restrict__ tile_claim,
          const unsigned* __restrict__ skip_if) {
  if (skip_if && *skip_if) return;  // the tensor-core filter (k_gf) took this pass: no tile is listed
  // the envelope bound in the same packed fp16 pair form (and error budget, k_lb)
  // as the series bound: per segment the region [L16[min], U16[max]], two query
  // slots per instruction; a block is live for slot b iff its fp16 bound <= T16[b]
  constexpr int NS = 2 * P;
  __shared__ uint2 s_lu16[kMaxCard];
  __shared__ uint2 s_q16[kTW * P];
  __shared__ LbConsts s_c;
  __shared__ unsigned s_blk[kMaxB];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kMaxCard; i += blockDim.x) s_lu16[i] = a.tab->lu16[i];
  for (int i = tid; i < kTW * P; i += blockDim.x) s_q16[i] = a.g_q16[i];
  if (tid < kMaxB) s_blk[tid] = 0;
  lb_consts_init(a, NS, &s_c);  // ends with __syncthreads
  const int64_t nblocks = (a.n + PARIS_INDEX_BLOCK - 1) / PARIS_INDEX_BLOCK;
  const int64_t ntiles = (a.n + kTS - 1) / kTS;
  static_assert(kBPT == 32, "a warp step bounds the 32 blocks of one tile");
  // a warp's first tile is its own index; later tiles are claimed one at a time from a
  // global counter (the work per tile varies with the pairs its envelope leaves live; a
  // static split left warps idle at the end), the next claim in flight while the current
  // tile is bounded
  const unsigned GW = (gridDim.x * blockDim.x) >> 5;
  unsigned gnext = (blockIdx.x * blockDim.x + tid) >> 5;
  for (;;) {
    const int64_t g = gnext;
    if (g >= ntiles) break;
    unsigned cl = 0;
    if (lane == 0) cl = atomicAdd(tile_claim, 1u);
    gnext = GW + __shfl_sync(0xffffffffu, cl, 0);
    const int64_t blk = 32 * g + lane;
    const bool valid = blk < nblocks;
    uint4 mn = make_uint4(~0u, ~0u, ~0u, ~0u), mx = make_uint4(0u, 0u, 0u, 0u);  // neutral for padding
    if (valid) {
      mn = __ldg(reinterpret_cast<const uint4*>(a.env + (size_t)blk * 32));
      mx = __ldg(reinterpret_cast<const uint4*>(a.env + (size_t)blk * 32 + 16));
    }
    // the tile's envelope (byte-wise min / max over its 32 blocks) bounds every block
    // of the tile: lane p bounds slot pair p on it, and only the pairs it leaves live
    // are evaluated per block (at C4 about a third of the pairs)
    uint4 tn = mn, tx4 = mx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tn.x = __vminu4(tn.x, __shfl_xor_sync(0xffffffffu, tn.x, o));
      tn.y = __vminu4(tn.y, __shfl_xor_sync(0xffffffffu, tn.y, o));
      tn.z = __vminu4(tn.z, __shfl_xor_sync(0xffffffffu, tn.z, o));
      tn.w = __vminu4(tn.w, __shfl_xor_sync(0xffffffffu, tn.w, o));
      tx4.x = __vmaxu4(tx4.x, __shfl_xor_sync(0xffffffffu, tx4.x, o));
      tx4.y = __vmaxu4(tx4.y, __shfl_xor_sync(0xffffffffu, tx4.y, o));
      tx4.z = __vmaxu4(tx4.z, __shfl_xor_sync(0xffffffffu, tx4.z, o));
      tx4.w = __vmaxu4(tx4.w, __shfl_xor_sync(0xffffffffu, tx4.w, o));
    }
    unsigned tp;
    {
      const uint32_t tnw[4] = {tn.x, tn.y, tn.z, tn.w}, txw[4] = {tx4.x, tx4.y, tx4.z, tx4.w};
      const int pl = lane < P ? lane : 0;
      uint32_t tacc = 0u;
#pragma unroll
      for (int seg = 0; seg < kTW; ++seg) {  // fully unrolled: register-indexed words
        const uint32_t tx = s_lu16[(txw[seg >> 2] >> (8 * (seg & 3))) & 0xFFu].x;
        const uint32_t ty = s_lu16[(tnw[seg >> 2] >> (8 * (seg & 3))) & 0xFFu].y;
        const uint2 q = s_q16[seg * P + pl];
        tacc = h2_acc_delta2(tacc, h2_fma_relu(q.x, kHalf2One, tx), h2_fma_relu(q.y, kHalf2One, ty));
      }
      tp = __ballot_sync(0xffffffffu, lane < P && h2_le_bits(tacc, s_c.T16[pl]) != 0u);
    }
    uint64_t bm = 0;
    const uint32_t mnw[4] = {mn.x, mn.y, mn.z, mn.w}, mxw[4] = {mx.x, mx.y, mx.z, mx.w};
    for (unsigned rem = tp; rem;) {  // the live pairs, 4 at a time (tp is warp-uniform)
      int pp[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pp[i] = rem ? __ffs(rem) - 1 : -1;
        rem &= rem - 1;
      }
      uint32_t acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int seg = 0; seg < kTW; ++seg) {  // fully unrolled: register-indexed words
        const uint32_t tx = s_lu16[(mxw[seg >> 2] >> (8 * (seg & 3))) & 0xFFu].x;  // -U16 of the max symbol
        const uint32_t ty = s_lu16[(mnw[seg >> 2] >> (8 * (seg & 3))) & 0xFFu].y;  // L16 of the min symbol
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint2 q = s_q16[seg * P + (pp[i] >= 0 ? pp[i] : 0)];
          const uint32_t a1 = h2_fma_relu(q.x, kHalf2One, tx);
          const uint32_t b1 = h2_fma_relu(q.y, kHalf2One, ty);
          acc[i] = h2_acc_delta2(acc[i], a1, b1);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (pp[i] >= 0 && valid) bm |= (uint64_t)h2_le_bits(acc[i], s_c.T16[pp[i]]) << (2 * pp[i]);
    }
    bmask[blk] = bm;  // padded to whole tiles
    const unsigned live = __ballot_sync(0xffffffffu, bm != 0ull);
    if (lane == 0 && live) tile_list[atomicAdd(tile_count, 1u)] = (unsigned)g;
    for (unsigned r = live ? tp : 0u; r; r &= r - 1) {  // per-slot block counts (stats), live pairs only
      const int p = __ffs(r) - 1;
      const unsigned m0 = __ballot_sync(0xffffffffu, (bm >> (2 * p)) & 1ull);
      const unsigned m1 = __ballot_sync(0xffffffffu, (bm >> (2 * p + 1)) & 1ull);
      if (lane == 0 && m0) atomicAdd(&s_blk[2 * p], (unsigned)__popc(m0));
      if (lane == 0 && m1) atomicAdd(&s_blk[2 * p + 1], (unsigned)__popc(m1));
    }
  }
  __syncthreads();
  if (tid < NS && s_blk[tid]) atomicAdd(&blocks[tid], s_blk[tid]);
}

// HC: coarse LB histograms (the k = 1 / k > 1 refine waves only need a quantile of
// them) in the table's holes and a 4-stage ring; !HC (the opt-in bucket-sorted walk,
// whose scatter needs exact bins): 16-bit 256-bin histograms and 3 stages.
template <int P, bool HC, int NW>
__global__ void __launch_bounds__(lbi_threads<NW>(), 1)
k_lbi(LbArgs a, const unsigned long long* __restrict__ bmask, const unsigned* __restrict__ tile_list,
      const unsigned* __restrict__ tile_count) {
  constexpr int NST = HC ? 4 : 3;
  extern __shared__ __align__(128) uint8_t dsm[];
  const uint32_t S0 = smem_u32(dsm);
  constexpr int kIWarps = NW, kIGroupWarps = NW / kIGroups, kIThreads = lbi_threads<NW>();
  static_assert(NW % kIGroups == 0, "equal consumer groups");
  const uint32_t T = (S0 + (uint32_t)(kTileBytes + lbi_misc_bytes<NW>()) + 0xFFFFu) & ~0xFFFFu;  // the table
  uint8_t* const gbase = dsm - S0;  // generic pointer of shared address x: gbase + x
  LbiMisc<NW>& M = *reinterpret_cast<LbiMisc<NW>*>(dsm + kTileBytes);
  unsigned* hist16 = reinterpret_cast<unsigned*>(gbase + T + 65536u + (uint32_t)(NST - 1) * kIStageBytes);
  auto stage_addr = [&](int st) -> uint32_t {
    return st == 0 ? S0 : T + 65536u + (uint32_t)(st - 1) * kIStageBytes;
  };
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const uint32_t need = T + 65536u + (uint32_t)(NST - 1) * kIStageBytes + (HC ? 0u : (uint32_t)kIHistBytes);
    if (need > S0 + dyn) __trap();  // launch config inconsistent with the layout
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nslots = 2 * P;
  const int64_t nlist = *tile_count;

  // ---- setup: barriers, table (32 copies), query words, histograms, warp buffers
  if (tid == 0) {
    for (int st = 0; st < NST; ++st) {
      mbar_init(&M.full[st], 1);
      mbar_init(&M.empty[st], kIGroupWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kMaxCard * 32; i += kIThreads)
    sts_u32(T + 256u * (uint32_t)(i >> 5) + 4u * (uint32_t)(i & 31), a.tab->lu16p[i >> 5]);
  for (int i = tid; i < nslots * kTW; i += kIThreads) {  // slot b, segment s: half2(q_lo16, -q_hi16)
    const int b = i / kTW, sg = i % kTW;
    const uint2 v = a.g_q16[sg * P + (b >> 1)];
    const uint32_t qw = half_of(v.x, b & 1) | (half_of(v.y, b & 1) << 16);
    sts_u32(hole_addr(T, b) + 4u * (uint32_t)sg, qw);
    sts_u32(hole_addr(T, b) + 64u + 4u * (uint32_t)sg, qw);
  }
  if (HC) {
    for (int i = tid; i < nslots * kNBC; i += kIThreads) sts_u32(hole_addr(T, kIHistHole + i / kNBC) + 4u * (uint32_t)(i % kNBC), 0u);
  } else {
    for (int i = tid; i < nslots * kNB / 2; i += kIThreads) hist16[i] = 0;
  }
  if (warp < kIWarps) {
    for (int b = lane; b < kMaxB; b += 32) M.w[warp].cnt[b] = 0;
    if (lane == 0) M.w[warp].n = 0;
  }
  lb_consts_init(a, nslots, &M.c);  // ends with __syncthreads

  if (warp >= kIWarps) {
    // ---- producers: refill stage st as soon as every consumer warp of its group released
    // it.  The whole warp decodes the tile's 32 block masks (lane = block; read from global
    // one tile ahead) into the stage's item list -- a block's live query slots paired in
    // order, consecutive live slots forming an item -- so the consumers claim ready items.
    // With NST % groups == 0 producer p serves group p's stages (tiles it = p, p + NP, ..).
    constexpr int NP = (NST % kIGroups == 0) ? kIGroups : 1;
    const int pi = warp - kIWarps;
    if (pi >= NP) goto lbi_done;
    int64_t li = blockIdx.x + (int64_t)pi * gridDim.x;
    const int64_t lstep = (int64_t)NP * gridDim.x;
    unsigned tnext = 0;
    uint64_t bnext = 0;
    if (li < nlist) {
      tnext = __ldg(tile_list + li);
      bnext = __ldg(bmask + (size_t)tnext * kBPT + lane);
    }
    for (int64_t it = pi; li < nlist; it += NP, li += lstep) {
      const int st = (int)(it % NST);
      const unsigned tile = tnext;
      uint64_t m = bnext;
      if (li + lstep < nlist) {  // the next tile's id and masks, early
        tnext = __ldg(tile_list + li + lstep);
        bnext = __ldg(bmask + (size_t)tnext * kBPT + lane);
      }
      if (it >= NST) mbar_wait(&M.empty[st], (unsigned)(((it / NST) - 1) & 1));
      // the copy first, the item decode while it is in flight: its complete_tx may land
      // before the expect_tx below (the tx-count goes transiently negative), but the
      // phase cannot complete before that arrival
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_g2s(gbase + stage_addr(st), a.sax + (size_t)tile * kTileBytes, (unsigned)kTileBytes, &M.full[st]);
      }
      const int cnt = (__popcll(m) + 1) >> 1;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      uint32_t* out = M.items[st] + (incl - cnt);
      for (int i = 0; i < cnt; ++i) {
        const uint32_t sa = (uint32_t)__ffsll((long long)m) - 1u;
        m &= m - 1;
        const uint32_t sb = m ? (uint32_t)__ffsll((long long)m) - 1u : 0xFFu;
        m &= m - 1;
        out[i] = (uint32_t)lane | (sa << 8) | (sb << 16);
      }
      __threadfence_block();
      if (lane == 31) {
        M.nitems[st] = (unsigned)incl;
        M.tile[st] = tile;
        M.next[st] = 0;
      }
      __syncwarp();
      if (lane == 31) mbar_expect_tx(&M.full[st], (unsigned)kTileBytes);  // release: the items are visible
    }
  } else {
    // ---- consumers
    LbiWarp& wb = M.w[warp];
    const LbConsts& c = M.c;
    const uint32_t lanebase = T | ((uint32_t)lane * 4u);  // bytes {lane * 4, 0, T bits 16-31}
    const int h = lane >> 4, hl = lane & 15;
    for (int64_t it = warp / kIGroupWarps;; it += kIGroups) {
      const int64_t li = blockIdx.x + it * gridDim.x;
      if (li >= nlist) break;
      const int st = (int)(it % NST);
      mbar_wait(&M.full[st], (unsigned)((it / NST) & 1));
      const int64_t tile = M.tile[st];
      PARIS_DCHECK(tile >= 0 && tile * kTS < a.n);
      const int total = (int)M.nitems[st];
      const uint32_t rows = stage_addr(st);
      for (;;) {
        unsigned cl = 0;
        if (lane == 0) cl = atomicAdd(&M.next[st], 2u);
        const int t0 = (int)__shfl_sync(0xffffffffu, cl, 0);
        if (t0 >= total) break;
        const int t = t0 + h;  // this half-warp's item
        const bool active = t < total;
        const uint32_t item = M.items[st][active ? t : t0];
        const int k = (int)(item & 31u);
        const int sa = (int)((item >> 8) & 0xFFu);
        const int sb = active && ((item >> 16) & 0xFFu) != 0xFFu ? (int)((item >> 16) & 0xFFu) : -1;
        const int sq = sb >= 0 ? sb : sa;  // odd count: duplicate lane, masked in emission
        // single-query form per slot (as k_lb1): one lookup t = (-U16, L16) serves both
        // slots; d = relu(q2 + t) = (relu(q_lo - U), relu(L - q_hi)) and acc += d^2 keep the
        // ABOVE and BELOW sums in the two halves (at most one is non-zero per segment).
        // Query words: 16-byte broadcast loads from this half-warp's copy (generic pointers
        // derived from dsm: LDS with immediate segment offsets).
        const uint4* qa4 = reinterpret_cast<const uint4*>(gbase + hole_addr(T, sa) + 64u * (uint32_t)h);
        const uint4* qb4 = reinterpret_cast<const uint4*>(gbase + hole_addr(T, sq) + 64u * (uint32_t)h);
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(gbase + rows) + k * (PARIS_INDEX_BLOCK / 4) + hl;
        uint32_t acca[4] = {0u, 0u, 0u, 0u}, accb[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int s4 = 0; s4 < kTW / 4; ++s4) {
          const uint4 qa = qa4[s4], qb = qb4[s4];
          const uint32_t qaw[4] = {qa.x, qa.y, qa.z, qa.w}, qbw[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
          for (int s1 = 0; s1 < 4; ++s1) {
            const int s = 4 * s4 + s1;
            const uint32_t word = wp[s * (kTS / 4)];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              // address = {lanebase.b0, word.bj, lanebase.b2, lanebase.b3}
              const uint32_t t = lds_u32(__byte_perm(word, lanebase, 0x7604u | ((uint32_t)j << 4)));
              const uint32_t da = h2_fma_relu(qaw[s1], kHalf2One, t);
              const uint32_t db = h2_fma_relu(qbw[s1], kHalf2One, t);
              acca[j] = h2_fma(da, da, acca[j]);
              accb[j] = h2_fma(db, db, accb[j]);
            }
          }
        }
        // LB16 per (series, slot) = ABOVE + BELOW sums, one packed fp16 add for both slots
        // (slot sa low, sb high); its rounding is one more (1+u) factor inside k_lb's error
        // budget G = (1+u)^(w+4), and only LB16's upper bound enters the tests
        uint32_t acc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t above = __byte_perm(acca[j], accb[j], 0x5410), below = __byte_perm(acca[j], accb[j], 0x7632);
          uint32_t sum;
          asm("add.rn.f16x2 %0, %1, %2;" : "=r"(sum) : "r"(above), "r"(below));
          acc[j] = sum;
        }
        // fast test: the packed minimum of the four series' (LB16 sa, LB16 sb) against the
        // item's thresholds (a missing sb or an inactive half-warp never passes); almost every
        // item stops here.  Series past n (last tile) may pass it: lbi_emit masks them.
        {
          const uint32_t Tp = active ? (half_of(c.T16[sa >> 1], sa & 1) |
                                        ((sb >= 0 ? half_of(c.T16[sb >> 1], sb & 1) : (uint32_t)kHalfNeg1) << 16))
                                     : (kHalfNeg1 | (kHalfNeg1 << 16));
          const uint32_t mn = h2_min(h2_min(acc[0], acc[1]), h2_min(acc[2], acc[3]));
          if (!__any_sync(0xffffffffu, h2_le_bits(mn, Tp) != 0u)) continue;
        }
        const int64_t i0 = tile * kTS + k * PARIS_INDEX_BLOCK + 4 * hl;
        const int nvalid = active ? (int)std::max<int64_t>(0, imin64(4, a.n - i0)) : 0;
        PARIS_DCHECK(k < kBPT && sa >= 0 && sa < nslots && sb < nslots);
        lbi_emit<HC>(acc, sa, sb, i0, nvalid, nslots, c, a, wb, T, warp, hist16);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&M.empty[st]);  // this warp is done reading stage st
    }
    lbi_flush<HC>(wb, T, warp, nslots, c, a, hist16);
  }
lbi_done:
  __syncthreads();
  if (HC) {
    for (int i = tid; i < nslots * kNBC; i += kIThreads) {
      const uint32_t v = lds_u32(hole_addr(T, kIHistHole + i / kNBC) + 4u * (uint32_t)(i % kNBC));
      if (v) atomicAdd(&a.hist[(i / kNBC) * kNB + (i % kNBC) * 8 + 7], v);
    }
  } else {
    for (int i = tid; i < nslots * kNB; i += kIThreads) {
      const unsigned v = (hist16[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
      if (v) atomicAdd(&a.hist[i], v);
    }
  }
}

// ---------------------------------------------------------------- K4, one query per pass
// B = 1 (flat path): the pass is one lookup + two FMAs per (series, segment), so
// it is fed by plain 8-byte loads at high occupancy rather than the TMA ring (whose 16
// row copies per tile cap delivery near 2.7 TB/s): one CTA of 32 warps per SM, a thread
// owns SPT = 4 consecutive series (one 32-bit word per segment row; the next group's 16
// words prefetched into registers while the current group is bounded), and the single-query
// fp16x2 form accumulates (ABOVE, BELOW) per series.  The region table (-U16, L16) is
// replicated 32x (entry c of lane l at T + 256c + 4l, T a 64 KB boundary of dynamic
// shared memory): ONE byte permute {lane*4, symbol, T bits 16..31} is a lookup's whole
// address, so a (series, segment) costs PRMT + LDS + 2 HFMA2.
#ifndef PARIS_LB1_SPT
#define PARIS_LB1_SPT 4
#endif
constexpr int kLb1Threads = PARIS_LB1_SPT >= 8 ? 768 : 1024;

// SPT series per thread: 16 (one uint4 per row) or 8 (one uint2 per row, fewer
// registers).
template <int SPT>
__global__ void __launch_bounds__(kLb1Threads, 1)
k_lb1(LbArgs a) {
  extern __shared__ __align__(128) uint8_t dsm1[];
  __shared__ uint32_t s_qd[kTW];
  __shared__ LbConsts s_c;
  __shared__ unsigned s_hist[kNB];
  // the warps' candidate buffers at the start of dynamic shared memory, below the table
  WarpBuf* s_wb = reinterpret_cast<WarpBuf*>(dsm1);
  const uint32_t S0 = smem_u32(dsm1);
  const uint32_t T = (S0 + (uint32_t)(sizeof(WarpBuf) * (kLb1Threads / 32)) + 0xFFFFu) & ~0xFFFFu;
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (T + 65536u > S0 + dyn) __trap();  // launch config inconsistent with the layout
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpBuf& wb = s_wb[warp];
  for (int b = lane; b < kMaxB; b += 32) wb.cnt[b] = 0;
  if (lane == 0) wb.n = 0;
  for (int i = tid; i < kNB; i += kLb1Threads) s_hist[i] = 0;
  for (int i = tid; i < kMaxCard * 32; i += kLb1Threads)
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(T + 256u * (uint32_t)(i >> 5) + 4u * (uint32_t)(i & 31)),
                 "r"(a.tab->lu16p[i >> 5]) : "memory");
  if (tid < kTW) {
    const uint2 v = a.g_q16[tid];  // pair layout, slot 0 = low halves
    s_qd[tid] = (v.x & 0xFFFFu) | (v.y << 16);
  }
  lb_consts_init(a, 1, &s_c);  // ends with __syncthreads
  const uint32_t lanebase = T | ((uint32_t)lane * 4u);  // bytes {lane * 4, 0, T bits 16-31}
  const int64_t n = a.n;
  const int64_t ngroups = n / SPT;  // n % 16 == 0 (tiled-path condition)
  // the next group's words are loaded while the current group is bounded (software
  // prefetch: one HBM latency per group is hidden behind the previous group's lookups)
  auto load_words = [&](int64_t g, uint32_t (&wd)[kTW][SPT / 4]) {
    const int64_t i0 = (int64_t)SPT * g;
#pragma unroll
    for (int s = 0; s < kTW; ++s) {
      if (g >= ngroups) { wd[s][0] = 0u; if (SPT > 4) wd[s][SPT / 4 - 1] = 0u; continue; }
      if (SPT == 16) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(a.sax + (size_t)s * n + i0));
        wd[s][0] = v.x; wd[s][1 % (SPT / 4)] = v.y; wd[s][2 % (SPT / 4)] = v.z; wd[s][3 % (SPT / 4)] = v.w;
      } else if (SPT == 8) {
        const uint2 v = __ldcs(reinterpret_cast<const uint2*>(a.sax + (size_t)s * n + i0));
        wd[s][0] = v.x; wd[s][1 % (SPT / 4)] = v.y;
      } else {
        wd[s][0] = __ldcs(reinterpret_cast<const uint32_t*>(a.sax + (size_t)s * n + i0));
      }
    }
  };
  uint32_t wnext[kTW][SPT / 4];
  load_words((int64_t)blockIdx.x * kLb1Threads + tid, wnext);
  for (int64_t g = (int64_t)blockIdx.x * kLb1Threads + tid; g - lane < ngroups;
       g += (int64_t)gridDim.x * kLb1Threads) {
    const int64_t i0 = (int64_t)SPT * g;
    uint32_t wd[kTW][SPT / 4];
#pragma unroll
    for (int s = 0; s < kTW; ++s)
#pragma unroll
      for (int c = 0; c < SPT / 4; ++c) wd[s][c] = wnext[s][c];
    load_words(g + (int64_t)gridDim.x * kLb1Threads, wnext);
    uint32_t acc[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) acc[j] = 0u;
    if (g < ngroups) {
#pragma unroll
      for (int s = 0; s < kTW; ++s) {
        const uint32_t qd = s_qd[s];
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
          uint32_t t;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t)
                       : "r"(__byte_perm(wd[s][j >> 2], lanebase, 0x7604u | ((uint32_t)(j & 3) << 4))));
          const uint32_t d = h2_fma_relu(qd, kHalf2One, t);
          acc[j] = h2_fma(d, d, acc[j]);
        }
      }
    }
    // LB16 = ABOVE + BELOW sums, rounded up into slot 0 (slot 1 = +inf never passes)
#pragma unroll
    for (int q4 = 0; q4 < SPT / 4; ++q4) {
      uint32_t a4[4][1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t v = acc[4 * q4 + j];
        a4[j][0] = (uint32_t)__half_as_ushort(__float2half_ru(h_lo_f(v) + h_hi_f(v))) | (0x7C00u << 16);
      }
      const int64_t ib = i0 + 4 * q4;
      const int nvalid = (g < ngroups) ? 4 : 0;
      lb_emit_wb<1>(a4, ib, nvalid, 1, s_c, a, wb, s_hist);
    }
  }
  wb_flush(wb, 1, s_c, a, s_hist);
  __syncthreads();
  for (int i = tid; i < kNB; i += kLb1Threads)
    if (s_hist[i]) atomicAdd(&a.hist[i], s_hist[i]);
}

// ---------------------------------------------------------------- K4, one query per pass (TMA ring)
// k_lb1t: the B = 1 pass as a producer/consumer stream.  One warp issues the 16 row
// copies (2 KB each, cp.async.bulk) of a 2048-series tile into a 4-stage ring; 16
// consumer warps own 4 series per thread, copy their 16 segment words to registers
// (conflict-free 32-bit loads), release the stage at once (so the producer refills it
// while they compute) and bound the words with the single-query fp16 form (PRMT + LDS +
// 2 HFMA2 per (series, segment), the region table replicated 32x as in k_lb1).  The
// (ABOVE, BELOW) halves of two series are summed by one packed fp16 add (one more (1+u)
// factor inside G, as k_lbi); candidates are staged per warp in the table's holes.
// No global address arithmetic per load (k_lb1 spent about half its issue slots on it).
// Shared plan (S0 = dynamic base, T = the 64 KB boundary above stage 0 + misc):
//   [S0, S0 + 32K) stage 0 | misc | [T, T + 64K) table + holes | T + 64K: stages 1..3
//   holes 0..31: warp w's staged keys in holes 2w, 2w + 1 (16 keys each); 64..71: the
//   256-bin LB histogram.
constexpr int kL1Warps = 16;                      // 512 consumer threads x 4 series = one tile
constexpr int kL1Threads = (kL1Warps + 1) * 32;  // + the producer warp
constexpr int kL1Stages = 4;
constexpr int kL1WB = 32;                         // staged keys per consumer warp
struct Lb1Misc {
  uint64_t full[kL1Stages], empty[kL1Stages];
  LbConsts c;
  uint32_t qd[kTW];
  unsigned wn[kL1Warps];
};
static_assert(kTileBytes + sizeof(Lb1Misc) + 2048 <= 65536, "stage 0 + misc below the table");

__device__ __forceinline__ uint32_t l1_key_addr(uint32_t T, int warp, int e) {
  return T + 256u * (uint32_t)(2 * warp + (e >> 4)) + 128u + 8u * (uint32_t)(e & 15);
}
__device__ __forceinline__ uint32_t l1_hist_addr(uint32_t T, int bin) {
  return T + 256u * (uint32_t)(64 + (bin >> 5)) + 128u + 4u * (uint32_t)(bin & 31);
}

__device__ void lb1t_flush(uint32_t T, int warp, unsigned& wn, const LbConsts& c, const LbArgs& a) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int m = (int)wn;
  if (m == 0) return;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(&a.count[0], (unsigned)m);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < m) {
    const uint64_t key = lds_u64(l1_key_addr(T, warp, lane));
    if ((int64_t)base + lane < a.cap) {
      a.cand[(size_t)base + lane] = key;
      atoms_add(l1_hist_addr(T, lb_bin(key_val(key), c.scale[0])), 1u);
    }
  }
  __syncwarp();
  if (lane == 0) wn = 0;
  __syncwarp();
}

__global__ void __launch_bounds__(kL1Threads, 1)
k_lb1t(LbArgs a) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const uint32_t S0 = smem_u32(dsm);
  const uint32_t T = (S0 + (uint32_t)(kTileBytes + sizeof(Lb1Misc)) + 0xFFFFu) & ~0xFFFFu;
  uint8_t* const gbase = dsm - S0;
  Lb1Misc& M = *reinterpret_cast<Lb1Misc*>(dsm + kTileBytes);
  auto stage_addr = [&](int st) -> uint32_t {
    return st == 0 ? S0 : T + 65536u + (uint32_t)(st - 1) * (uint32_t)kTileBytes;
  };
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (T + 65536u + (uint32_t)(kL1Stages - 1) * (uint32_t)kTileBytes > S0 + dyn) __trap();
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int64_t ntiles = (n + kTS - 1) / kTS;
  if (tid == 0) {
    for (int st = 0; st < kL1Stages; ++st) {
      mbar_init(&M.full[st], 1);
      mbar_init(&M.empty[st], kL1Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kMaxCard * 32; i += kL1Threads)
    sts_u32(T + 256u * (uint32_t)(i >> 5) + 4u * (uint32_t)(i & 31), a.tab->lu16p[i >> 5]);
  for (int i = tid; i < kNB; i += kL1Threads) sts_u32(l1_hist_addr(T, i), 0u);
  if (tid < kTW) {
    const uint2 v = a.g_q16[tid];  // pair layout, slot 0 = low halves: half2(q_lo16, -q_hi16)
    M.qd[tid] = (v.x & 0xFFFFu) | (v.y << 16);
  }
  if (tid < kL1Warps) M.wn[tid] = 0;
  lb_consts_init(a, 1, &M.c);  // ends with __syncthreads

  if (warp == kL1Warps) {
    // ---- producer: 16 row copies per tile into the stage the consumers released
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = (int)(it % kL1Stages);
      if (it >= kL1Stages) mbar_wait(&M.empty[st], (unsigned)(((it / kL1Stages) - 1) & 1));
      const int64_t base = tile * kTS;
      const unsigned bytes = (unsigned)imin64(kTS, n - base);  // n % 16 == 0: a multiple of 16
      if (lane == 0) mbar_expect_tx(&M.full[st], bytes * (unsigned)kTW);
      __syncwarp();
      if (lane < kTW)
        bulk_g2s(gbase + stage_addr(st) + (uint32_t)lane * (uint32_t)kTS, a.sax + (size_t)lane * n + base, bytes,
                 &M.full[st]);
    }
  } else {
    // ---- consumers: thread t owns series 4t .. 4t+3 of every tile of this CTA
    const LbConsts& c = M.c;
    const uint32_t lanebase = T | ((uint32_t)lane * 4u);  // bytes {lane * 4, -, T bits 16-31}
    const uint32_t T2 = (c.T16[0] & 0xFFFFu) * 0x10001u;  // slot 0's threshold in both halves
    const float thr = c.thr[0];
    uint32_t qd[kTW];
#pragma unroll
    for (int s = 0; s < kTW; ++s) qd[s] = M.qd[s];
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = (int)(it % kL1Stages);
      mbar_wait(&M.full[st], (unsigned)((it / kL1Stages) & 1));
      const uint32_t* rows = reinterpret_cast<const uint32_t*>(gbase + stage_addr(st)) + tid;
      uint32_t wd[kTW];
#pragma unroll
      for (int s = 0; s < kTW; ++s) wd[s] = rows[s * (kTS / 4)];
      __syncwarp();
      if (lane == 0) mbar_arrive(&M.empty[st]);  // the words are in registers: refill now
      uint32_t acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int s = 0; s < kTW; ++s) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t t = lds_u32(__byte_perm(wd[s], lanebase, 0x7604u | ((uint32_t)j << 4)));
          const uint32_t d = h2_fma_relu(qd[s], kHalf2One, t);
          acc[j] = h2_fma(d, d, acc[j]);
        }
      }
      // LB16 of series (0, 1) and (2, 3): ABOVE + BELOW in one packed add each
      uint32_t s01, s23;
      asm("add.rn.f16x2 %0, %1, %2;" : "=r"(s01) : "r"(__byte_perm(acc[0], acc[1], 0x5410)),
          "r"(__byte_perm(acc[0], acc[1], 0x7632)));
      asm("add.rn.f16x2 %0, %1, %2;" : "=r"(s23) : "r"(__byte_perm(acc[2], acc[3], 0x5410)),
          "r"(__byte_perm(acc[2], acc[3], 0x7632)));
      const int64_t i0 = tile * kTS + 4 * (int64_t)tid;
      uint32_t pf = h2_le_bits(s01, T2) | (h2_le_bits(s23, T2) << 2);
      if (i0 >= n) pf = 0u;  // a partial last tile (n % 16 == 0: whole groups of 4)
      if (!__any_sync(0xffffffffu, pf != 0u)) continue;
      // rigorous fp32 bounds for the pairs that passed the fp16 test (rare)
      float lbv[4];
      unsigned m = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t v = j < 2 ? s01 : s23;
        const float hv = (j & 1) ? h_hi_f(v) : h_lo_f(v);
        lbv[j] = __fmul_rd(fmaxf(__fsub_rd(hv, c.wabs), 0.f), c.lbconv);
        if (((pf >> j) & 1u) && lbv[j] <= thr) m |= 1u << j;
      }
      const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(m));
      if (total == 0) continue;
      if ((int)M.wn[warp] + total > kL1WB) lb1t_flush(T, warp, M.wn[warp], c, a);
      if (total > kL1WB) {  // degenerate (e.g. tau = inf): straight to global memory
        for (unsigned r = m; r; r &= r - 1) {
          const int j = __ffs(r) - 1;
          const unsigned pos = atomicAdd(&a.count[0], 1u);
          if ((int64_t)pos < a.cap) {
            a.cand[pos] = make_key(lbv[j], (uint32_t)(i0 + j));
            atoms_add(l1_hist_addr(T, lb_bin(lbv[j], c.scale[0])), 1u);
          }
        }
      } else {
        for (unsigned r = m; r; r &= r - 1) {
          const int j = __ffs(r) - 1;
          const int pos = (int)atomicAdd(&M.wn[warp], 1u);
          sts_u64(l1_key_addr(T, warp, pos), make_key(lbv[j], (uint32_t)(i0 + j)));
        }
      }
      __syncwarp();
    }
    lb1t_flush(T, warp, M.wn[warp], c, a);
  }
  __syncthreads();
  for (int i = tid; i < kNB; i += kL1Threads) {
    const uint32_t v = lds_u32(l1_hist_addr(T, i));
    if (v) atomicAdd(&a.hist[i], v);
  }
}

// ---------------------------------------------------------------- f2: nb-ParIS+
// nb-ParIS+ ExactSearch (Alg7) with DistComp workers (Alg8,
// P:1223-1246): SAX is split into contiguous parts, one per worker (a warp); a
// worker keeps its OWN copy of the BSF per query (V_bsf, registers -- no
// communication while scanning), computes the lower bound of every word of its
// part (the same batched fp16 form as the LBC pass) and, whenever one is below
// its BSF, reads the raw series at once, computes the true distance (early
// abandoning) and lowers its copy.  The answer is min(V_bsf)
// (P:1208): one 64-bit atomicMin per worker and query at the end.  k = 1.
struct NbArgs {
  const uint8_t* sax;
  int64_t n;
  int w;
  float seglen_f;
  const CardTables* tab;
  const uint2* g_q16;
  const float* queries;      // [nb][len]
  const float* raw;
  int len;
  int nb;
  unsigned long long* best;  // [nb] padded: seed key in, min(V_bsf) out
  unsigned* refined;         // raw series read, per query
  unsigned* updates;         // V_bsf updates, per query
  float d2up;
  int64_t part;              // series per worker (multiple of 4)
};

template <int P>
__global__ void __launch_bounds__(kLBThreads)
k_nb(NbArgs a) {
  constexpr int NS = 2 * P;
  __shared__ uint2 s_lu16[kMaxCard];
  __shared__ uint2 s_q16[P * kMaxW];
  __shared__ float2 s_lu[kMaxCard];
  __shared__ float s_grow;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) {
    s_lu16[i] = a.tab->lu16[i];
    s_lu[i] = a.tab->lu[i];
  }
  for (int i = threadIdx.x; i < P * kMaxW; i += blockDim.x) s_q16[i] = a.g_q16[i];
  if (threadIdx.x == 0) s_grow = (float)(pow(1.0 + 1.0 / 2048.0, (double)(a.w + 4)) * (1.0 + 1e-12));
  __syncthreads();
  const float lbconv = __fdiv_rd(a.seglen_f, s_grow);
  const float wabs = (float)a.w * 5.9604644775390625e-08f;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t lo = gw * a.part, hi = imin64(a.n, lo + a.part);
  // private BSF copies (V_bsf) seeded with the approximate search's BSF
  uint64_t bkey[NS];
  float thr[NS];
  unsigned nref[NS], nupd[NS];
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    bkey[b] = (b < a.nb) ? a.best[(size_t)b * kPadU64] : kNoKey;
    thr[b] = (b < a.nb && bkey[b] != kNoKey) ? __fmul_ru(key_val(bkey[b]), a.d2up) : (b < a.nb ? INFINITY : -1.f);
    nref[b] = 0;
    nupd[b] = 0;
  }
  auto t16 = [&](float t) -> uint32_t {  // fp16 filter threshold of a private BSF (see k_lb)
    if (t < 0.f) return kHalfNeg1;
    const float T = __fadd_ru(__fmul_ru(__fdiv_ru(t, a.seglen_f), s_grow), wabs);
    return (T > 64000.f) ? 0x7C00u : (uint32_t)__half_as_ushort(__float2half_ru(T));
  };
  uint32_t T16[P];
#pragma unroll
  for (int p = 0; p < P; ++p) T16[p] = t16(thr[2 * p]) | (t16(thr[2 * p + 1]) << 16);

  for (int64_t base = lo; base < hi; base += 128) {
    const int64_t i0 = base + 4 * lane;
    uint32_t acc[4][P];
    const int nvalid = (int)std::max<int64_t>(0, imin64(4, hi - i0));
    if (nvalid > 0) lb16_group<P, 16, true>(a.sax, a.n, a.w, i0, s_q16, s_lu16, acc);
    else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int p = 0; p < P; ++p) acc[j][p] = 0x7C007C00u;
    }
    // (series j, slot b) pairs of this lane passing the fp16 test: bit 4b + j
    uint64_t cm = 0;
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t pb = (j < nvalid) ? h2_le_bits(acc[j][p], T16[p]) : 0u;
        cm |= (uint64_t)(pb & 1u) << (8 * p + j);
        cm |= (uint64_t)((pb >> 1) & 1u) << (8 * p + 4 + j);
      }
    // DistComp (Alg8 lines 4-8): the warp refines its candidates one at a time
    while (true) {
      const unsigned lanes = __ballot_sync(0xffffffffu, cm != 0);
      if (!lanes) break;
      const int L = __ffs(lanes) - 1;
      const uint64_t cmL = __shfl_sync(0xffffffffu, cm, L);
      const int bit = __ffsll((long long)cmL) - 1;
      const int b = bit >> 2, j = bit & 3;
      if (lane == L) cm &= ~(1ull << bit);
      uint32_t v = 0;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p == (b >> 1)) v = acc[j][p];
      v = __shfl_sync(0xffffffffu, v, L);
      const float h = (b & 1) ? h_hi_f(v) : h_lo_f(v);
      const float lb = __fmul_rd(fmaxf(__fsub_rd(h, wabs), 0.f), lbconv);
      float tb = 0.f;
#pragma unroll
      for (int q = 0; q < NS; ++q)
        if (q == b) tb = thr[q];
      if (!(lb <= tb)) continue;  // minDist < BSF (line 4), against the worker's own copy
      const int64_t id = base + 4 * L + j;
      // realDist = Dist(rawData, TS) with early abandoning at the worker's BSF
      const float4* row = reinterpret_cast<const float4*>(a.raw + (size_t)id * a.len);
      const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
      const int nf = a.len >> 2;
      float accd = 0.f;
      bool abandoned = false;
      for (int c0 = 0; c0 < nf; c0 += 32) {
        const int f = c0 + lane;
        if (f < nf) {
          const float4 x = ld_stream(row + f), y = __ldg(qv + f);
          float d;
          d = x.x - y.x; accd = fmaf(d, d, accd);
          d = x.y - y.y; accd = fmaf(d, d, accd);
          d = x.z - y.z; accd = fmaf(d, d, accd);
          d = x.w - y.w; accd = fmaf(d, d, accd);
        }
        if (c0 + 32 < nf && warp_sum(accd) > tb) { abandoned = true; break; }
      }
#pragma unroll
      for (int q = 0; q < NS; ++q)
        if (q == b) ++nref[q];
      if (abandoned) continue;
      const uint64_t k2 = make_key(warp_sum(accd), (uint32_t)id);
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        if (q == b && k2 < bkey[q]) {  // line 7-8: realDist < BSF -> BSF = realDist
          bkey[q] = k2;
          thr[q] = __fmul_ru(key_val(k2), a.d2up);
          ++nupd[q];
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) T16[p] = t16(thr[2 * p]) | (t16(thr[2 * p + 1]) << 16);
    }
  }
  // return min(V_bsf) (Alg7 line 9)
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      if (b >= a.nb) break;
      if (bkey[b] != kNoKey) atomicMin(a.best + (size_t)b * kPadU64, (unsigned long long)bkey[b]);
      if (nref[b]) atomicAdd(&a.refined[b], nref[b]);
      if (nupd[b]) atomicAdd(&a.updates[b], nupd[b]);
    }
  }
}

// Query prep alone (for the tiled seed, which has no prologue of its own).
template <int P>
__global__ void k_qprep(const float* __restrict__ queries, int nb, int len, int w, float2* __restrict__ g_q,
                        uint2* __restrict__ g_q16) {
  extern __shared__ float2 s_qdyn[];  // [2P * kMaxW] intervals, then [P * kMaxW] fp16 pairs (qprep_smem)
  query_prep<P>(queries, nb, len, w, s_qdyn, reinterpret_cast<uint2*>(s_qdyn + 2 * P * kMaxW), g_q, g_q16);
}

// ---------------------------------------------------------------- K5 bucket order
// Counting sort of the candidates by LB bin (the paper sorts its candidate list
// by file position for disk locality; in HBM the LB order is what
// matters: refinement stops at the first bin above the BSF).
__global__ void __launch_bounds__(256)
k_scatter(const uint64_t* __restrict__ cand, const unsigned* __restrict__ count,
          const unsigned* __restrict__ hist, const unsigned* __restrict__ thr,
          unsigned* __restrict__ cursor, uint64_t* __restrict__ sorted, int64_t cap) {
  // Each CTA owns a contiguous chunk of the query's candidates: it counts its
  // chunk per bin in shared memory, reserves each bin's range with one global
  // atomic, then scatters with shared-memory cursors (no per-candidate global
  // atomics on the hot bins near tau).
  __shared__ unsigned s_off[kNB];
  __shared__ unsigned s_cnt[kNB];
  const int b = blockIdx.y;
  unsigned v = hist[b * kNB + threadIdx.x];
  s_off[threadIdx.x] = v;
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int o = 1; o < kNB; o <<= 1) {
    const unsigned t = (threadIdx.x >= o) ? s_off[threadIdx.x - o] : 0u;
    __syncthreads();
    s_off[threadIdx.x] += t;
    __syncthreads();
  }
  const unsigned excl = s_off[threadIdx.x] - v;
  __syncthreads();
  s_off[threadIdx.x] = excl;
  const float sc = bin_scale(__uint_as_float(thr[b]));
  const int64_t cnt = imin64((int64_t)count[b], cap);
  const int64_t per = (cnt + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = imin64(cnt, (int64_t)blockIdx.x * per), c1 = imin64(cnt, c0 + per);
  const uint64_t* src = cand + (size_t)b * cap;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&s_cnt[lb_bin(key_val(src[i]), sc)], 1u);
  __syncthreads();
  {
    const unsigned k = s_cnt[threadIdx.x];
    s_off[threadIdx.x] += k ? atomicAdd(&cursor[b * kNB + threadIdx.x], k) : 0u;
    s_cnt[threadIdx.x] = 0;
  }
  __syncthreads();
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const uint64_t key = src[i];
    const int bin = lb_bin(key_val(key), sc);
    const uint64_t pos = (uint64_t)s_off[bin] + atomicAdd(&s_cnt[bin], 1u);
    if (pos < (uint64_t)cap) sorted[(size_t)b * cap + pos] = key;
  }
}

// ---------------------------------------------------------------- K6 RDC pass
// Alg11: take the next candidate (static interleave of warps over
// the LB-ordered list instead of a locked cursor), skip it if LB > BSF,
// else read raw[id], compute the true distance with early abandoning, and lower
// the BSF.  kU candidates are in flight per warp.
struct RefineArgs {
  const float* raw;
  int len;
  const float* queries;      // batch base [nb][len]
  const uint64_t* sorted;
  int64_t cap;
  const unsigned* count;
  const unsigned* thr_seed;  // tau_seed^2 (float bits): the binning scale of K4/K5
  unsigned* thr;             // k > 1: live pruning threshold (float bits), per query
  unsigned long long* best;  // k = 1: (d^2 bits << 32 | id), per query
  unsigned* refined;         // per query counter
  uint64_t* lists;           // k > 1: [nb][gridDim.x][k]
  int k;
  float d2up;                // 1 + bound on the relative error of an fp32 d^2 (rounding up)
  unsigned lo, hi;           // k = 1: refine list positions [lo, min(hi, count)) (a wave)
  int64_t n;                 // series in raw (debug bounds checks)
  const uint16_t* raw16 = nullptr;  // optional bf16 copy of raw [n][len] (paris_raw_bf16): pre-filter
  unsigned* refined16 = nullptr;    // per query: bf16 rows read by the pre-filter
  unsigned* ghist = nullptr;        // k > 1: per query, histogram of refined exact d^2 (kNB bins of tau_seed^2)
  const __half* paa16 = nullptr;    // optional [n][w2] fp16 PAA of raw (paris_paa_f16): the PAA pre-filter
  int w2 = 0;
  unsigned* paa_rows = nullptr;     // per query of the batch: PAA rows read (accumulated over the call)
  const float* qaux = nullptr;      // [nb][kQAux] query constants (k_qaux), octet refine
};

// One warp step: up to kU candidates (indices i0 + u*stride) against the live
// threshold `thr`; returns true when the list is exhausted for this warp (index
// past the end, or a candidate whose LB bin lies wholly above thr: every later
// candidate in bin order is then above it too).  Distances of survivors go to
// d2[u] (INFINITY = pruned or abandoned).
__device__ __forceinline__ bool refine_step(const RefineArgs& a, const uint64_t* __restrict__ list,
                                            unsigned cnt, unsigned i0, unsigned stride, float thr,
                                            float scale, const float4* __restrict__ s_qv,
                                            uint64_t (&key)[kU], float (&d2)[kU], unsigned& nref) {
  const int lane = threadIdx.x & 31;
  const int nf = a.len >> 2;
  bool live[kU];
  bool stop = false;
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const unsigned i = i0 + u * stride;
    key[u] = (i < cnt) ? list[i] : kNoKey;
    const float lb = key_val(key[u]);
    live[u] = (i < cnt) && !stop && lb <= thr;
    if (i >= cnt) stop = true;
    else if (!live[u] && !stop) {
      const int bin = lb_bin(lb, scale);
      if (bin >= 1 && (float)(bin - 1) > thr * scale) stop = true;
    }
    d2[u] = INFINITY;
  }
  float acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u] = 0.f;
#pragma unroll
  for (int u = 0; u < kU; ++u) PARIS_DCHECK(!live[u] || key_id(key[u]) < (uint64_t)a.n);
  for (int c0 = 0; c0 < nf; c0 += 32) {
    const int f = c0 + lane;
    float4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (live[u] && f < nf)
        x[u] = ld_stream(reinterpret_cast<const float4*>(a.raw + (size_t)key_id(key[u]) * a.len) + f);
    if (f < nf) {
      const float4 q = s_qv[f];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!live[u]) continue;
        float d;
        d = x[u].x - q.x; acc[u] = fmaf(d, d, acc[u]);
        d = x[u].y - q.y; acc[u] = fmaf(d, d, acc[u]);
        d = x[u].z - q.z; acc[u] = fmaf(d, d, acc[u]);
        d = x[u].w - q.w; acc[u] = fmaf(d, d, acc[u]);
      }
    }
    if (c0 + 32 < nf) {
      // early abandoning (north_star) after each 128-point chunk
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!live[u]) continue;
        if (warp_sum(acc[u]) > thr) { live[u] = false; ++nref; }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    if (!live[u]) continue;
    d2[u] = warp_sum(acc[u]);
    ++nref;
  }
  return stop;
}

// bf16 pre-filter (optional, a.raw16): a row's bf16 copy x~ (half the bytes)
// gives a rigorous lower bound on the true distance before the fp32 row is read.
// Round-to-nearest bf16 keeps |x_i - x~_i| <= rho |x~_i|, rho = 2^-8 (1 + 2^-7), so
// ED(x, x~) <= rho ||x~|| <= rho (||q|| + D) with D = ED(q, x~), and
// ED(q, x) >= D - rho (||q|| + D) = (1 - rho) D - rho ||q||.  D^2 is an fp32 sum
// (relative error <= e = (len/32 + 8) 2^-24, the d^2 bound of refine_group), taken
// as D >= sqrt(D^2 (1 - 2e)) with directed roundings; qn_hi >= ||q||.  A candidate
// whose bound squared exceeds thr (the live BSF threshold) cannot beat the BSF and
// is dropped without its fp32 row; the rest are refined exactly as before.
__device__ __forceinline__ float bf16_lb(float d2, float qn_hi, float e2) {
  constexpr float rho = 0.00392150878906250f;       // 2^-8 (1 + 2^-7), rounded up
  constexpr float one_m_rho = 0.99607849121093750f; // 1 - rho, rounded down
  return __fsub_rd(__fsub_rd(__fmul_rd(one_m_rho, __fsqrt_rd(__fmul_rd(d2, 1.f - e2))), __fmul_ru(rho, qn_hi)),
                   1e-30f);  // (1e-30: the absolute error of bf16 subnormals)
}

// The candidates are given as lanes of the chunk's key register k0 (src[u]) and a
// live mask lm (bit u): their keys are re-read with a shuffle where needed, so the
// warp keeps U row buffers but not U 64-bit keys in registers.  Clears the bits of
// the candidates it drops.
template <int NC, int U>
__device__ __forceinline__ void bf16_prefilter(const RefineArgs& a, const float4* __restrict__ qv, float qn_hi,
                                               uint64_t k0, const int (&src)[U], unsigned& lm, float thr) {
  constexpr int NH = (NC + 1) / 2;  // uint4 (8 bf16) per lane
  const int lane = threadIdx.x & 31;
  const int nh = a.len >> 3;
  uint4 h[U][NH];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t id = (uint32_t)__shfl_sync(0xffffffffu, k0, src[u]);
    const bool on = (lm >> u) & 1u;
#pragma unroll
    for (int c = 0; c < NH; ++c) {
      const int f = lane + 32 * c;
      h[u][c] = (on && f < nh) ? ld_stream_u4(reinterpret_cast<const uint4*>(a.raw16 + (size_t)id * a.len) + f)
                               : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  float s2[U];
#pragma unroll
  for (int u = 0; u < U; ++u) s2[u] = 0.f;
#pragma unroll
  for (int c = 0; c < NH; ++c) {
    const int f = lane + 32 * c;
    const float4 q0 = f < nh ? __ldg(qv + 2 * f) : make_float4(0, 0, 0, 0);
    const float4 q1 = f < nh ? __ldg(qv + 2 * f + 1) : make_float4(0, 0, 0, 0);
    const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w4[4] = {h[u][c].x, h[u][c].y, h[u][c].z, h[u][c].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = __uint_as_float((e & 1) ? (w4[e >> 1] & 0xFFFF0000u) : (w4[e >> 1] << 16)) - qq[e];
        s2[u] = fmaf(d, d, s2[u]);
      }
    }
  }
  const float e2 = 2.f * (float)((a.len >> 5) + 8) * 5.9604644775390625e-08f;
  if constexpr (U % 4 == 0) {
    // four sums per reduction: halves exchange two values (xor 16), then one (xor 8),
    // then each 8-lane group finishes its own value; one ballot spreads the four
    // decisions (lane 8u holds value u's sum)
    const bool hi16 = lane & 16, hi8 = lane & 8;
#pragma unroll
    for (int g = 0; g < U; g += 4) {
      float w0 = hi16 ? s2[g + 2] : s2[g], w1 = hi16 ? s2[g + 3] : s2[g + 1];
      w0 += __shfl_xor_sync(0xffffffffu, hi16 ? s2[g] : s2[g + 2], 16);
      w1 += __shfl_xor_sync(0xffffffffu, hi16 ? s2[g + 1] : s2[g + 3], 16);
      float z = hi8 ? w1 : w0;
      z += __shfl_xor_sync(0xffffffffu, hi8 ? w0 : w1, 8);
      z += __shfl_xor_sync(0xffffffffu, z, 4);
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      const float lb = bf16_lb(z, qn_hi, e2);
      const unsigned drop = __ballot_sync(0xffffffffu, lb > 0.f && __fmul_rd(lb, lb) > thr);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if ((drop >> (8 * u)) & 1u) lm &= ~(1u << (g + u));
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float lb = bf16_lb(warp_sum(s2[u]), qn_hi, e2);
      if (lb > 0.f && __fmul_rd(lb, lb) > thr) lm &= ~(1u << u);
    }
  }
}

// Refine up to U candidates of one query (k = 1): load the live rows whole
// (lane l: float4 #(l + 32c)), accumulate the squared distance with early abandoning
// after each 128-point chunk (north_star), lower the BSF (64-bit
// atomicMin on (d^2, id)) and this warp's view of it (`cur`).
template <int NC, int U>
__device__ __forceinline__ void refine_group(const RefineArgs& a, const float4* __restrict__ qv,
                                             const uint64_t (&key)[U], bool (&live)[U], float thr,
                                             uint64_t& cur, unsigned long long* bp, unsigned& nref) {
  const int lane = threadIdx.x & 31;
  const int nf = a.len >> 2;
#pragma unroll
  for (int u = 0; u < U; ++u) PARIS_DCHECK(!live[u] || key_id(key[u]) < (uint64_t)a.n);
  float4 x[U][NC];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int f = lane + 32 * c;
      x[u][c] = (live[u] && f < nf)
                    ? ld_stream(reinterpret_cast<const float4*>(a.raw + (size_t)key_id(key[u]) * a.len) + f)
                    : make_float4(0, 0, 0, 0);
    }
  float acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const float4 q = (lane + 32 * c < nf) ? __ldg(qv + lane + 32 * c) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float d;
      d = x[u][c].x - q.x; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].y - q.y; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].z - q.z; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].w - q.w; acc[u] = fmaf(d, d, acc[u]);
    }
    if (c + 1 < NC && 32 * (c + 1) < nf) {
      // early abandoning after each 128-point chunk (the rest is not accumulated)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u] && warp_sum(acc[u]) > thr) { live[u] = false; ++nref; }
      bool any = false;
#pragma unroll
      for (int u = 0; u < U; ++u) any |= live[u];
      if (!any) break;
    }
  }
  uint64_t mk = kNoKey;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!live[u]) continue;
    ++nref;
    mk = min(mk, make_key(warp_sum(acc[u]), key_id(key[u])));
  }
  if (mk < cur) {
    if (lane == 0) atomicMin(bp, (unsigned long long)mk);
    cur = mk;
  }
}

// k = 1 (P:1357-1378 with BSF = the best (d^2, id) key): a warp takes U
// candidates at a time from its interleaved share of the query's LB-ordered list;
// the live BSF is read (relaxed) in parallel with the keys; surviving rows are
// loaded whole (lane l: float4 #(l + 32c)), the distance is accumulated chunk by
// chunk with early abandoning (north_star) after each 128 points, and
// the BSF is lowered with one 64-bit atomicMin.  Few registers -> 64 warps per SM:
// the occupancy, not TMA, is what keeps random 1 KB gathers at HBM speed
// (profiles/r01/micro_gather_1KB_rows.txt: LDG 6.8-7.0 TB/s vs 2.2 TB/s for
// 1 KB cp.async.bulk copies issued by one warp per SM).
template <int NC, int U>  // NC = float4 chunks of 32 per lane (len <= 128*NC)
__global__ void __launch_bounds__(kRefThreads, NC <= 2 ? 8 : 2)
k_refine1(RefineArgs a, int nb) {
  // every warp walks its interleaved share of EVERY query's list (balanced work:
  // a query with 5x the mean candidate count no longer leaves most SMs idle); the
  // query rows are read through L1 (all warps of a CTA share them)
  __shared__ unsigned s_refined[kMaxB], s_cnt[kMaxB], s_r16[kMaxB];
  __shared__ float s_scale[kMaxB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kMaxB) {
    s_refined[threadIdx.x] = 0;
    s_r16[threadIdx.x] = 0;
    // per-query list lengths and bin scales, read once per CTA (queries with no work
    // in this wave then cost a shared-memory read, not a global round trip)
    s_cnt[threadIdx.x] = threadIdx.x < nb
        ? (unsigned)imin64(imin64((int64_t)a.count[threadIdx.x], a.cap), (int64_t)a.hi) : 0u;
    s_scale[threadIdx.x] = threadIdx.x < nb ? bin_scale(__uint_as_float(a.thr_seed[threadIdx.x])) : 0.f;
  }
  __syncthreads();
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  for (int b = 0; b < nb; ++b) {
    const unsigned cnt = s_cnt[b];
    if (a.lo + gw >= cnt) continue;
    const float scale = s_scale[b];
    const uint64_t* list = a.sorted + (size_t)b * a.cap + a.lo;
    const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
    unsigned long long* bp = a.best + (size_t)b * kPadU64;
    unsigned nref = 0, nref16 = 0;
    uint64_t cur = kNoKey;  // this warp's view of the BSF: refreshed every 4 steps, lowered by its own finds
    unsigned step = 0;
    for (unsigned i0 = gw; a.lo + i0 < cnt; i0 += U * GW, ++step) {
      uint64_t key[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned i = i0 + u * GW;
        key[u] = (a.lo + i < cnt) ? __ldg(list + i) : kNoKey;
      }
      if ((step & 3) == 0) cur = min(cur, ld_relaxed_u64(bp));
      const float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      bool live[U], stop = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float lb = key_val(key[u]);
        live[u] = !stop && (a.lo + i0 + u * GW < cnt) && lb <= thr;
        if (!live[u] && !stop) {
          // bin order: past the end, or a bin wholly above thr, ends this warp's share
          const int bin = lb_bin(lb, scale);
          stop = (a.lo + i0 + u * GW >= cnt) || (bin >= 1 && (float)(bin - 1) > thr * scale);
        }
      }
      refine_group<NC, U>(a, qv, key, live, thr, cur, bp, nref);
      if (stop) break;
    }
    if (lane == 0 && nref) atomicAdd(&s_refined[b], nref);
    if (lane == 0 && nref16) atomicAdd(&s_r16[b], nref16);
  }
  __syncthreads();
  if (threadIdx.x < nb && s_refined[threadIdx.x]) atomicAdd(&a.refined[threadIdx.x], s_refined[threadIdx.x]);
  if (threadIdx.x < nb && s_r16[threadIdx.x]) atomicAdd(&a.refined16[threadIdx.x], s_r16[threadIdx.x]);
}

// k = 1 without the bucket sort (K5 skipped): the two LB-ordered waves are taken
// straight from the LB pass's unsorted candidate lists.  Wave A refines the
// candidates whose LB bin is <= cut[b] (the first bin at which the query's LB
// histogram reaches wave_a candidates: the lowest-LB ~wave_a, which find the NN
// early), wave B the rest.  A warp reads 32 keys at a time (one per lane,
// coalesced), keeps those inside its wave with LB <= the live BSF, and
// refines them U at a time, warp-cooperatively (refine_group).  Every key is read
// once per wave (8 bytes against 4*len bytes per refined row), and the pruning
// test is the same as the sorted walk's, so the refined set differs only by the
// order within a wave.
// 6 CTAs (48 warps) per SM for len <= 256: 42 registers per thread, room for U rows
// in flight per warp (U = 2 at len 256: 96 KB of rows in flight per SM; measured at
// C4: 1.50 ms/step vs 1.87 with 8 CTAs x 1 row)
#ifndef PARIS_REFU_CTAS
#define PARIS_REFU_CTAS 6
#endif
constexpr int kRefUCtas = PARIS_REFU_CTAS;
#ifndef PARIS_REFU_U
#define PARIS_REFU_U 2
#endif
constexpr int kRefUU = PARIS_REFU_U;  // rows in flight per warp at len <= 256
#ifndef PARIS_REFU16_CTAS
#define PARIS_REFU16_CTAS 4
#endif
constexpr int kRefU16Ctas = PARIS_REFU16_CTAS;  // with the bf16 pre-filter (more registers per warp)
#ifndef PARIS_REFU16_MUL
#define PARIS_REFU16_MUL 2
#endif
constexpr int kPFMul = PARIS_REFU16_MUL;  // bf16 rows per warp step = kPFMul x U
#ifndef PARIS_RAW16_MINLEN
#define PARIS_RAW16_MINLEN 256
#endif
constexpr int kRaw16MinLen = PARIS_RAW16_MINLEN;  // shortest rows (in HBM) the pre-filter is used for

__global__ void __launch_bounds__(kNB) k_wave_cut(const unsigned* __restrict__ hist, unsigned wave_a,
                                                  unsigned* __restrict__ cut) {
  __shared__ unsigned s[kNB];
  const int b = blockIdx.x, t = threadIdx.x;
  s[t] = hist[b * kNB + t];
  __syncthreads();
  for (int o = 1; o < kNB; o <<= 1) {
    const unsigned v = (t >= o) ? s[t - o] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  const bool reach = s[t] >= wave_a, prev = t > 0 && s[t - 1] >= wave_a;
  if (reach && !prev) cut[b * kNB] = (unsigned)t;
  if (t == kNB - 1 && !reach) cut[b * kNB] = (unsigned)(kNB - 1);
}

template <int NC, int U, bool R16>
__global__ void __launch_bounds__(kRefThreads, NC <= 2 ? (R16 ? kRefU16Ctas : kRefUCtas) : 2)
k_refine1u(RefineArgs a, int nb, int wave, const unsigned* __restrict__ cut) {
  constexpr int kPF = kPFMul * U;  // bf16 pre-filter rows per warp step
  __shared__ unsigned s_refined[kMaxB], s_cnt[kMaxB], s_cut[kMaxB], s_r16[kMaxB];
  __shared__ float s_scale[kMaxB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kMaxB) {
    const bool on = threadIdx.x < nb;
    s_refined[threadIdx.x] = 0;
    s_r16[threadIdx.x] = 0;
    s_cnt[threadIdx.x] = on ? (unsigned)imin64((int64_t)a.count[threadIdx.x], a.cap) : 0u;
    s_cut[threadIdx.x] = on ? cut[threadIdx.x * kNB] : 0u;
    s_scale[threadIdx.x] = on ? bin_scale(__uint_as_float(a.thr_seed[threadIdx.x])) : 0.f;
  }
  __syncthreads();
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  for (int b = 0; b < nb; ++b) {
    const unsigned cnt = s_cnt[b];
    const unsigned nchunk = (cnt + 31) / 32;
    const unsigned first = (gw + (unsigned)b * 613u) % GW;  // rotate: spread small lists over all warps
    if (first >= nchunk) continue;
    const float scale = s_scale[b];
    const int cutb = (int)s_cut[b];
    const uint64_t* list = a.sorted + (size_t)b * a.cap;
    const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
    unsigned long long* bp = a.best + (size_t)b * kPadU64;
    unsigned nref = 0, nref16 = 0;
    uint64_t cur = kNoKey;
    float qn_hi = 0.f;  // >= ||q|| (pre-filter only)
    if (R16) {
      float qs = 0.f;
      for (int f = lane; f < (a.len >> 2); f += 32) {
        const float4 v = __ldg(qv + f);
        qs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, qs))));
      }
      const float e2 = 2.f * (float)((a.len >> 5) + 8) * 5.9604644775390625e-08f;
      qn_hi = __fsqrt_ru(__fmul_ru(warp_sum(qs), 1.f + e2));
    }
    // the next chunk's keys are loaded while this chunk is processed
    uint64_t knext = (first * 32 + lane < cnt) ? __ldg(list + first * 32 + lane) : kNoKey;
    for (unsigned ch = first; ch < nchunk; ch += GW) {
      const unsigned i = ch * 32 + lane;
      const uint64_t k0 = knext;
      {
        const unsigned in = (ch + GW) * 32 + lane;
        knext = (ch + GW < nchunk && in < cnt) ? __ldg(list + in) : kNoKey;
      }
      cur = min(cur, ld_relaxed_u64(bp));
      float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      const float lb0 = key_val(k0);
      const int bin = lb_bin(lb0, scale);
      const bool mine = i < cnt && (wave == 0 ? bin <= cutb : bin > cutb);
      unsigned m = __ballot_sync(0xffffffffu, mine && lb0 <= thr);
      if (R16) {
        // bf16 pre-filter over kPF candidates at a time (their 2*len-byte rows in flight
        // together), then the survivors' fp32 rows U at a time
        while (m) {
          int src[kPF];
          unsigned lm = 0;
#pragma unroll
          for (int u = 0; u < kPF; ++u) {
            src[u] = m ? __ffs(m) - 1 : 0;
            const bool has = m != 0u;
            m &= m - 1;
            const float lbu = key_val(__shfl_sync(0xffffffffu, k0, src[u]));
            if (has && lbu <= thr) lm |= 1u << u;
          }
          nref16 += __popc(lm);
          bf16_prefilter<NC, kPF>(a, qv, qn_hi, k0, src, lm, thr);
#pragma unroll
          for (int g = 0; g < kPF; g += U) {
            if (!((lm >> g) & ((1u << U) - 1u))) continue;
            uint64_t key[U];
            bool live[U], any = false;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              key[u] = __shfl_sync(0xffffffffu, k0, src[g + u]);
              live[u] = ((lm >> (g + u)) & 1u) && key_val(key[u]) <= thr;
              any |= live[u];
            }
            if (!any) continue;
            refine_group<NC, U>(a, qv, key, live, thr, cur, bp, nref);
            thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
          }
        }
      }
      while (m) {
        uint64_t key[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = m ? __ffs(m) - 1 : 0;
          const bool has = m != 0u;
          m &= m - 1;
          key[u] = __shfl_sync(0xffffffffu, k0, src);
          live[u] = has && key_val(key[u]) <= thr;
        }
        refine_group<NC, U>(a, qv, key, live, thr, cur, bp, nref);
        thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      }
    }
    if (lane == 0 && nref) atomicAdd(&s_refined[b], nref);
    if (lane == 0 && nref16) atomicAdd(&s_r16[b], nref16);
  }
  __syncthreads();
  if (threadIdx.x < nb && s_refined[threadIdx.x]) atomicAdd(&a.refined[threadIdx.x], s_refined[threadIdx.x]);
  if (threadIdx.x < nb && s_r16[threadIdx.x]) atomicAdd(&a.refined16[threadIdx.x], s_r16[threadIdx.x]);
}

// k = 1 with the bf16 pre-filter (the default index-path refine when a bf16 copy is
// given), eight lanes per candidate: a warp walks its share of the query's unsorted list
// as k_refine1u does (same waves, same rotation, same LB <= BSF test) but queues
// the keys that pass in shared memory and drains them 8 at a time -- an octet of lanes per
// candidate, two candidates per octet, so each lane has 8 independent 16-byte loads in
// flight and every load instruction touches four whole 128-byte lines (4 KB of bf16 rows
// in flight per warp).  D^2 = ||q - x~||^2 is summed per lane in two fp32 chains and
// reduced over the octet; a candidate whose pre-filter bound (1 - rho) D - rho ||q||
// (bf16_lb) exceeds the live BSF is dropped, the few survivors get their exact fp32
// distance warp-cooperatively (refine_group, U rows in flight), which lowers the BSF.
// Error bound of the octet sum: <= (len/16 + 8) 2^-24 relative (two chains of len/16
// terms, one add, a 3-level tree), doubled as in bf16_lb's margin.
#ifndef PARIS_REFQ_CTAS
#define PARIS_REFQ_CTAS 3
#endif
constexpr int kRefQCtas = PARIS_REFQ_CTAS;
constexpr int kRefQLen = 256;  // longest row of the octet form
constexpr int kQAux = 80;      // floats per query of the refine's query constants (k_qaux)

// Per query of a batch, once: qn_hi >= ||q|| (warp-tree fp32 sum, rounded up with its
// margin), and for the PAA pre-filter the query's PAA at w2 segments (fp64 means rounded
// to fp32) and qpn_hi >= ||PAA_w2(q)||: out[b * kQAux + {0, 1, 16 + s}].  A warp per query.
__global__ void __launch_bounds__(32) k_qaux(const float* __restrict__ queries, int len, int w2,
                                             float* __restrict__ out) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const float e2w = 2.f * (float)((len >> 5) + 8) * 5.9604644775390625e-08f;
  const float4* qv = reinterpret_cast<const float4*>(queries + (size_t)b * len);
  float qs = 0.f;
  for (int f = lane; f < (len >> 2); f += 32) {
    const float4 v = __ldg(qv + f);
    qs = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, qs))));
  }
  qs = warp_sum(qs);
  float pn = 0.f;
  if (w2 > 0) {
    const int sl = len / w2;
    for (int sg = lane; sg < w2; sg += 32) {
      double m = 0.0;
      for (int j = 0; j < sl; ++j) m += (double)queries[(size_t)b * len + (size_t)sg * sl + j];
      const float v = (float)(m / (double)sl);
      out[b * kQAux + 16 + sg] = v;
      pn = fmaf(v, v, pn);
    }
    pn = warp_sum(pn);
  }
  if (lane == 0) {
    out[b * kQAux + 0] = __fsqrt_ru(__fmul_ru(qs, 1.f + e2w));
    out[b * kQAux + 1] = __fsqrt_ru(__fmul_ru(pn, 1.f + e2w));
  }
}

// The PAA pre-filter over a warp's queued keys [0, m) (m <= 32; every lane calls it):
// octet o (lanes 8o..8o+7) takes keys o + 4i, i < 8, each lane one 2*W2/8-byte piece of the
// row (4 rows per octet in flight at a time); keys whose LB <= thr and whose rigorous PAA
// bound does not exceed thr are compacted to the front of the queue; returns
// their count.  npaa counts the PAA rows read.  qpl: this lane's W2/8 query PAA values.
template <int W2>
__device__ __forceinline__ int paa_filter_queue(const RefineArgs& a, uint64_t* queue, int m, float thr,
                                                const float (&qpl)[W2 > 0 ? W2 / 8 : 1], float qpn_hi,
                                                unsigned& npaa) {
  constexpr int EPL = W2 > 0 ? W2 / 8 : 1;  // fp16 values per lane of a row
  const int lane = threadIdx.x & 31, oct = lane >> 3, sub = lane & 7;
  const float e2p = 2.f * (float)(EPL + 8) * 5.9604644775390625e-08f;    // lane chain + octet tree
  constexpr float rho16 = 4.8875808715820312e-04f;  // 2^-11 (1 + 2^-10), rounded up
  constexpr float one_m_rho16 = 0.99951171875f;     // 1 - 2^-11 (1 + 2^-10), rounded down
  const float qterm = __fmul_ru(rho16 + 1.1920928955078125e-07f, qpn_hi);   // (rho16 + 2^-23) ||q_p||
  const float slack = __fmul_ru(sqrtf((float)W2) * 1.0001f, 5.9604644775390625e-08f);  // sqrt(W2) 2^-24
  const float scale2 = __fdiv_rd((float)a.len, (float)(W2 > 0 ? W2 : 1));
  // all keys first (the survivors are compacted over the same queue entries)
  uint64_t key[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = oct + 4 * i;
    key[i] = e < m ? queue[e] : kNoKey;
  }
  __syncwarp();
  int nout = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {  // 4 rows per octet at a time (registers)
    bool keep[4];
    uint32_t pw[4][EPL / 2 > 0 ? EPL / 2 : 1];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = oct + 4 * (4 * half + i);
      const uint64_t kk = key[4 * half + i];
      keep[i] = e < m && key_val(kk) <= thr;
      const __half* row = a.paa16 + (size_t)key_id(kk) * W2 + sub * EPL;
      if (EPL == 8) {
        const uint4 v = keep[i] ? ld_stream_u4(reinterpret_cast<const uint4*>(row)) : make_uint4(0u, 0u, 0u, 0u);
        pw[i][0] = v.x; pw[i][EPL / 2 > 1 ? 1 : 0] = v.y; pw[i][EPL / 2 > 2 ? 2 : 0] = v.z; pw[i][EPL / 2 > 3 ? 3 : 0] = v.w;
      } else if (EPL == 4) {
        uint2 v = make_uint2(0u, 0u);
        if (keep[i]) v = __ldcs(reinterpret_cast<const uint2*>(row));
        pw[i][0] = v.x; pw[i][EPL / 2 > 1 ? 1 : 0] = v.y;
      } else {
        pw[i][0] = keep[i] ? __ldcs(reinterpret_cast<const uint32_t*>(row)) : 0u;
      }
      npaa += __popc(__ballot_sync(0xffffffffu, sub == 0 && keep[i]));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const uint32_t w = pw[i][e >> 1];
        const float x = __half2float(__ushort_as_half((unsigned short)((e & 1) ? (w >> 16) : (w & 0xFFFFu))));
        const float d = x - qpl[e];
        acc = fmaf(d, d, acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      const float D = __fsqrt_rd(__fmul_rd(acc, 1.f - e2p));
      const float Dp = __fsub_rd(__fsub_rd(__fmul_rd(one_m_rho16, D), qterm), slack);
      const float lb2 = Dp > 0.f ? __fmul_rd(scale2, __fmul_rd(Dp, Dp)) : 0.f;
      const bool kp = keep[i] && !(lb2 > thr);  // NaN (a PAA beyond fp16): no pruning
      const unsigned mk = __ballot_sync(0xffffffffu, sub == 0 && kp);
      if (sub == 0 && kp) queue[nout + __popc(mk & ((1u << lane) - 1u))] = key[4 * half + i];
      nout += __popc(mk);
    }
  }
  __syncwarp();
  return nout;
}

// W2 > 0: the PAA pre-filter first (paris_paa_f16): per candidate its fp16 PAA row (2 W2
// bytes, an octet of lanes reading one 16-byte piece each), the rigorous PAA lower bound
// sqrt(len/W2) ((1 - rho16) D~ - (rho16 + 2^-23) ||q_p|| - sqrt(W2) 2^-24) with
// D~ = ||q_p - x~_p|| (Keogh's PAA bound; fp16 rounding bounded as the bf16
// one); survivors go on to the bf16 stage (if a.raw16) or straight to the
// exact fp32 distance.
template <int NC, int U, int W2, bool R16>
__global__ void __launch_bounds__(kRefThreads, kRefQCtas)
k_refine1q(RefineArgs a, int nb, int wave, const unsigned* __restrict__ cut) {
  __shared__ unsigned s_refined[kMaxB], s_cnt[kMaxB], s_cut[kMaxB], s_r16[kMaxB], s_paa[kMaxB];
  __shared__ float s_scale[kMaxB];
  __shared__ uint64_t s_queue[kRefWarps][64];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int oct = lane >> 3, sub = lane & 7;
  if (threadIdx.x < kMaxB) {
    const bool on = threadIdx.x < nb;
    s_refined[threadIdx.x] = 0;
    s_r16[threadIdx.x] = 0;
    s_paa[threadIdx.x] = 0;
    s_cnt[threadIdx.x] = on ? (unsigned)imin64((int64_t)a.count[threadIdx.x], a.cap) : 0u;
    s_cut[threadIdx.x] = on ? cut[threadIdx.x * kNB] : 0u;
    s_scale[threadIdx.x] = on ? bin_scale(__uint_as_float(a.thr_seed[threadIdx.x])) : 0.f;
  }
  __syncthreads();
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  const int nh = a.len >> 3;  // uint4 (8 bf16) per row
  const int nper = (nh + 7) >> 3;  // uint4 per lane of an octet
  const float e2 = 2.f * (float)((a.len >> 4) + 8) * 5.9604644775390625e-08f;   // octet sums
  uint64_t* queue = s_queue[warp];
  for (int b = 0; b < nb; ++b) {
    const unsigned cnt = s_cnt[b];
    const unsigned nchunk = (cnt + 31) / 32;
    const unsigned first = (gw + (unsigned)b * 613u) % GW;  // rotate: spread small lists over all warps
    if (first >= nchunk) continue;
    const float scale = s_scale[b];
    const int cutb = (int)s_cut[b];
    const uint64_t* list = a.sorted + (size_t)b * a.cap;
    const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
    unsigned long long* bp = a.best + (size_t)b * kPadU64;
    unsigned nref = 0, nref16 = 0;
    uint64_t cur = kNoKey;
    const float* qx = a.qaux + (size_t)b * kQAux;  // k_qaux: ||q||, ||PAA(q)||, PAA(q)
    const float qn_hi = __ldg(qx);
    int qn = 0;  // queued keys

    // W2 > 0: the PAA stage over the queued keys [0, m) (m <= 32): octet o takes keys
    // o + 4i, i < 8 (each lane one 16-byte piece of every row: 8 loads in flight); the
    // survivors are compacted to the front of the queue
    unsigned npaa = 0;
    float qpl[W2 > 0 ? W2 / 8 : 1];  // this lane's query PAA values (segments sub*W2/8 ..)
    if (W2 > 0) {
#pragma unroll
      for (int e = 0; e < (W2 > 0 ? W2 / 8 : 1); ++e) qpl[e] = __ldg(qx + 16 + sub * (W2 / 8) + e);
    }
    const float qpn_hi = W2 > 0 ? __ldg(qx + 1) : 0.f;
    auto paa_stage = [&](int m) -> int {
      cur = min(cur, ld_relaxed_u64(bp));
      const float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      return paa_filter_queue<W2>(a, queue, m, thr, qpl, qpn_hi, npaa);
    };

    // the queued keys [0, m): octet o takes keys 8r + o and 8r + 4 + o of round r
    auto drain = [&](int m) {
      if (W2 > 0) {
        m = paa_stage(m);
        if (!R16) {  // PAA survivors straight to the exact distance, U rows in flight
          cur = min(cur, ld_relaxed_u64(bp));
          float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
          const uint64_t kl = lane < m ? queue[lane] : kNoKey;
          unsigned m2 = __ballot_sync(0xffffffffu, lane < m && key_val(kl) <= thr);
          while (m2) {
            uint64_t ks[U];
            bool lv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int src = m2 ? __ffs(m2) - 1 : 0;
              const bool has = m2 != 0u;
              m2 &= m2 - 1;
              ks[u] = __shfl_sync(0xffffffffu, kl, src);
              lv[u] = has && key_val(ks[u]) <= thr;
            }
            refine_group<NC, U>(a, qv, ks, lv, thr, cur, bp, nref);
            thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
          }
          return;
        }
      }
      for (int r0 = 0; r0 < m; r0 += 8) {
        cur = min(cur, ld_relaxed_u64(bp));
        float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
        uint64_t key[2];
        bool live[2];
        const uint4* row[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int e = r0 + 4 * c + oct;
          key[c] = e < m ? queue[e] : kNoKey;
          live[c] = e < m && key_val(key[c]) <= thr;
          row[c] = reinterpret_cast<const uint4*>(a.raw16 + (size_t)key_id(key[c]) * a.len);
        }
        nref16 += __popc(__ballot_sync(0xffffffffu, sub == 0 && live[0])) +
                  __popc(__ballot_sync(0xffffffffu, sub == 0 && live[1]));
        float s2[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
        for (int i0 = 0; i0 < nper; i0 += 4) {
          uint4 h[2][4];
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int f = sub + 8 * (i0 + i);
              h[c][i] = (live[c] && i0 + i < nper && f < nh) ? ld_stream_u4(row[c] + f) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int f = sub + 8 * (i0 + i);
            if (i0 + i >= nper || f >= nh) break;
            const float4 q0 = __ldg(qv + 2 * f), q1 = __ldg(qv + 2 * f + 1);  // L1-resident query
            const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const uint32_t w4[4] = {h[c][i].x, h[c][i].y, h[c][i].z, h[c][i].w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float d = __uint_as_float((e & 1) ? (w4[e >> 1] & 0xFFFF0000u) : (w4[e >> 1] << 16)) - qq[e];
                s2[c][e & 1] = fmaf(d, d, s2[c][e & 1]);
              }
            }
          }
        }
        bool keep[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v = s2[c][0] + s2[c][1];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          const float lb = bf16_lb(v, qn_hi, e2);
          keep[c] = live[c] && !(lb > 0.f && __fmul_rd(lb, lb) > thr);
        }
        // survivors (octet leaders' bits): exact fp32 distance, U rows in flight per warp
        unsigned m2 = __ballot_sync(0xffffffffu, sub == 0 && keep[0]);
        unsigned m3 = __ballot_sync(0xffffffffu, sub == 0 && keep[1]);
        while (m2 | m3) {
          uint64_t ks[U];
          bool lv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const bool from2 = m2 != 0u;
            const unsigned mm = from2 ? m2 : m3;
            const int src = mm ? __ffs(mm) - 1 : 0;
            const bool has = mm != 0u;
            if (from2) m2 &= m2 - 1; else m3 &= m3 - 1;
            const uint64_t k0 = __shfl_sync(0xffffffffu, key[0], src), k1 = __shfl_sync(0xffffffffu, key[1], src);
            ks[u] = from2 ? k0 : k1;
            lv[u] = has && key_val(ks[u]) <= thr;
          }
          refine_group<NC, U>(a, qv, ks, lv, thr, cur, bp, nref);
          thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
        }
      }
    };

    uint64_t knext = (first * 32 + lane < cnt) ? __ldg(list + first * 32 + lane) : kNoKey;
    for (unsigned ch = first; ch < nchunk; ch += GW) {
      const unsigned i = ch * 32 + lane;
      const uint64_t k0 = knext;
      {
        const unsigned in = (ch + GW) * 32 + lane;
        knext = (ch + GW < nchunk && in < cnt) ? __ldg(list + in) : kNoKey;
      }
      cur = min(cur, ld_relaxed_u64(bp));
      const float thr = (cur == kNoKey) ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      const float lb0 = key_val(k0);
      const int bin = lb_bin(lb0, scale);
      const bool pass = i < cnt && (wave == 0 ? bin <= cutb : bin > cutb) && lb0 <= thr;
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) queue[qn + __popc(m & ((1u << lane) - 1u))] = k0;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) {
        drain(32);
        __syncwarp();
        if (lane < qn - 32) queue[lane] = queue[32 + lane];  // the rest to the front
        qn -= 32;
        __syncwarp();
      }
    }
    if (qn > 0) drain(qn);
    __syncwarp();
    if (lane == 0 && nref) atomicAdd(&s_refined[b], nref);
    if (lane == 0 && nref16) atomicAdd(&s_r16[b], nref16);
    if (W2 > 0 && lane == 0 && npaa) atomicAdd(&s_paa[b], npaa);
  }
  __syncthreads();
  if (threadIdx.x < nb && s_refined[threadIdx.x]) atomicAdd(&a.refined[threadIdx.x], s_refined[threadIdx.x]);
  if (threadIdx.x < nb && s_r16[threadIdx.x]) atomicAdd(&a.refined16[threadIdx.x], s_r16[threadIdx.x]);
  if (W2 > 0 && threadIdx.x < nb && s_paa[threadIdx.x] && a.paa_rows)
    atomicAdd(&a.paa_rows[threadIdx.x], s_paa[threadIdx.x]);
}

// k = 1 index-path refine with the PAA pre-filter (and the bf16 one if R16) over ONE
// stream of candidate chunks: the batch's unsorted lists concatenated (chunk c of query b
// at s_off[b] + c), warp w takes chunks w, w + GW, ... -- every query's chunks spread over
// all warps (balanced per query, as the rotated interleave of k_refine1q), but a warp never
// restarts per query: the per-query constants (PAA of q, ||q||, ||PAA(q)||, wave cut, bin
// scale) sit in shared memory for the whole batch, queued keys carry their query, and the
// queue is drained only when full (k_refine1q paid a setup, a key-prefetch miss and a
// partial drain -- three dependent memory round trips -- per (warp, query) with ~1.3
// chunks each at C4).  Same tests in the same arithmetic: LB <= BSF, the PAA
// bound, the bf16 bound, exact fp32 distance with early abandoning; only the order in
// which candidates are refined differs (the result is the unique minimum (d^2, id) key).
#ifndef PARIS_REFM_CTAS
#define PARIS_REFM_CTAS 3
#endif
constexpr int kRefMCtas = PARIS_REFM_CTAS;
#ifndef PARIS_REFM_KP
#define PARIS_REFM_KP 2
#endif
constexpr int kRefMKP = PARIS_REFM_KP;  // chunks of keys in flight per warp
#ifndef PARIS_REFM_H
#define PARIS_REFM_H 2
#endif
constexpr int kRefMH = PARIS_REFM_H;    // bf16 stage: 16-byte pieces per candidate in flight
#ifndef PARIS_REFM_ROWS
#define PARIS_REFM_ROWS 4
#endif
constexpr int kRefMRows = PARIS_REFM_ROWS;  // PAA stage: rows per octet in flight (4 or 8)
template <int NC, int U, int W2, bool R16>
__global__ void __launch_bounds__(kRefThreads, kRefMCtas)
k_refine1m(RefineArgs a, int nb, int wave, const unsigned* __restrict__ cut) {
  static_assert(W2 == 32 || W2 == 64, "PAA pre-filter widths");
  constexpr int EPL = W2 / 8;  // fp16 PAA values per lane of a row (an octet per row)
  __shared__ unsigned s_off[kMaxB + 1];
  __shared__ unsigned s_cnt[kMaxB], s_cut[kMaxB], s_refined[kMaxB], s_r16[kMaxB], s_paa[kMaxB];
  __shared__ float s_scale[kMaxB], s_qn[kMaxB], s_qpn[kMaxB];
  __shared__ __align__(16) float s_qp[kMaxB * W2];
  __shared__ uint64_t s_queue[kRefWarps][64];
  __shared__ uint8_t s_qb[kRefWarps][64];
  __shared__ float s_qt[kRefWarps][64];  // the query's pruning threshold when the key was queued
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int oct = lane >> 3, sub = lane & 7;
  if (tid < kMaxB) {
    const bool on = tid < nb;
    s_refined[tid] = 0;
    s_r16[tid] = 0;
    s_paa[tid] = 0;
    s_cnt[tid] = on ? (unsigned)imin64((int64_t)a.count[tid], a.cap) : 0u;
    s_cut[tid] = on ? cut[tid * kNB] : 0u;
    s_scale[tid] = on ? bin_scale(__uint_as_float(a.thr_seed[tid])) : 0.f;
    s_qn[tid] = on ? a.qaux[tid * kQAux] : 0.f;
    s_qpn[tid] = on ? a.qaux[tid * kQAux + 1] : 0.f;
  }
  // the query PAA stored so that the eight lanes of an octet (one 128-bit load phase) read
  // eight consecutive float4: segment 8 sub + 4 e4 + e1 (lane sub, its float4 e4) at
  // float4 e4 * 8 + sub of the query's row (a plain row put lanes sub and sub + 4 on the
  // same banks)
  for (int i = tid; i < nb * W2; i += kRefThreads) {
    const int b = i / W2, sg = i % W2;
    const int sub_ = sg / EPL, e4 = (sg % EPL) / 4, e1 = sg % 4;
    s_qp[b * W2 + (e4 * 8 + sub_) * 4 + e1] = a.qaux[b * kQAux + 16 + sg];
  }
  __syncthreads();
  if (warp == 0) {  // chunk offsets: an exclusive scan of ceil(cnt / 32) over the queries
    unsigned run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const unsigned c = b < nb ? (s_cnt[b] + 31u) / 32u : 0u;
      unsigned incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (b < nb) s_off[b] = run + incl - c;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_off[nb] = run;
  }
  __syncthreads();
  const unsigned TC = s_off[nb];
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  const int nh = a.len >> 3;       // uint4 (8 bf16) per row
  const int nper = (nh + 7) >> 3;  // uint4 per lane of an octet
  const float e2 = 2.f * (float)((a.len >> 4) + 8) * 5.9604644775390625e-08f;  // octet sums (bf16)
  const float e2p = 2.f * (float)(EPL + 8) * 5.9604644775390625e-08f;          // octet sums (PAA)
  constexpr float rho16 = 4.8875808715820312e-04f;  // 2^-11 (1 + 2^-10), rounded up
  constexpr float one_m_rho16 = 0.99951171875f;     // 1 - 2^-11 (1 + 2^-10), rounded down
  const float slack = __fmul_ru(sqrtf((float)W2) * 1.0001f, 5.9604644775390625e-08f);  // sqrt(W2) 2^-24
  const float scale2 = __fdiv_rd((float)a.len, (float)W2);
  uint64_t* queue = s_queue[warp];
  uint8_t* qb = s_qb[warp];
  float* qt = s_qt[warp];
  auto thr_of = [&](uint64_t bsf) { return bsf == kNoKey ? INFINITY : __fmul_ru(key_val(bsf), a.d2up); };
  // the query owning chunk gc: the last b with s_off[b] <= gc (empty queries share offsets)
  auto chunk_query = [&](unsigned gc) -> int {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= gc) lo = mid; else hi = mid;
    }
    return lo;
  };
  // exact fp32 distance of one queued survivor (warp-cooperative, early abandoning)
  auto refine_one = [&](uint64_t key, int b) {
    uint64_t ks[1] = {key};
    const uint64_t bsf = ld_relaxed_u64(a.best + (size_t)b * kPadU64);
    bool lv[1] = {key_val(key) <= thr_of(bsf)};
    if (!lv[0]) return;
    uint64_t cur = bsf;
    unsigned nr = 0;
    refine_group<NC, 1>(a, reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len), ks, lv, thr_of(bsf), cur,
                        a.best + (size_t)b * kPadU64, nr);
    if (lane == 0 && nr) atomicAdd(&s_refined[b], nr);
  };
  // the queued entries [0, m): the PAA stage (octet o: entries o + 4i, i < 8, in two halves of
  // four rows in flight), survivors compacted to the front; then bf16 (R16) and exact fp32
  auto drain = [&](int m) {
    uint64_t key[8];
    int kb[8];
    float kt[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = oct + 4 * i;
      key[i] = e < m ? queue[e] : kNoKey;
      kb[i] = e < m ? (int)qb[e] : 0;
      kt[i] = e < m ? qt[e] : 0.f;
    }
    __syncwarp();
    int nout = 0;
#pragma unroll
    for (int half = 0; half < 8 / kRefMRows; ++half) {
      bool keep[kRefMRows];
      float thr[kRefMRows];
      uint32_t pw[kRefMRows][EPL / 2];
#pragma unroll
      for (int i = 0; i < kRefMRows; ++i) {
        const int e = oct + 4 * (kRefMRows * half + i);
        const uint64_t kk = key[kRefMRows * half + i];
        const int b = kb[kRefMRows * half + i];
        thr[i] = kt[kRefMRows * half + i];  // as of the chunk scan (a stale bound only prunes less)
        const __half* row = a.paa16 + (size_t)key_id(kk) * W2 + sub * EPL;
        keep[i] = e < m;
        if (EPL == 8) {
          const uint4 v = keep[i] ? ld_stream_u4(reinterpret_cast<const uint4*>(row)) : make_uint4(0u, 0u, 0u, 0u);
          pw[i][0] = v.x; pw[i][EPL / 2 > 1 ? 1 : 0] = v.y; pw[i][EPL / 2 > 2 ? 2 : 0] = v.z; pw[i][EPL / 2 > 3 ? 3 : 0] = v.w;
        } else {
          uint2 v = make_uint2(0u, 0u);
          if (keep[i]) v = __ldcs(reinterpret_cast<const uint2*>(row));
          pw[i][0] = v.x; pw[i][EPL / 2 > 1 ? 1 : 0] = v.y;
        }
      }
#pragma unroll
      for (int i = 0; i < kRefMRows; ++i) {
        const int b = kb[kRefMRows * half + i];
        if (sub == 0 && keep[i]) atomicAdd(&s_paa[b], 1u);  // rows read
        keep[i] = keep[i] && key_val(key[kRefMRows * half + i]) <= thr[i];
        const float4* qp4 = reinterpret_cast<const float4*>(s_qp + b * W2) + sub;
        float acc = 0.f;
#pragma unroll
        for (int e4 = 0; e4 < EPL / 4; ++e4) {
          const float4 q = qp4[8 * e4];
          const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int e1 = 0; e1 < 4; ++e1) {
            const int e = 4 * e4 + e1;
            const uint32_t w = pw[i][e >> 1];
            const float x = __half2float(__ushort_as_half((unsigned short)((e & 1) ? (w >> 16) : (w & 0xFFFFu))));
            const float d = x - qq[e1];
            acc = fmaf(d, d, acc);
          }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        const float qterm = __fmul_ru(rho16 + 1.1920928955078125e-07f, s_qpn[b]);  // (rho16 + 2^-23) ||q_p||
        const float D = __fsqrt_rd(__fmul_rd(acc, 1.f - e2p));
        const float Dp = __fsub_rd(__fsub_rd(__fmul_rd(one_m_rho16, D), qterm), slack);
        const float lb2 = Dp > 0.f ? __fmul_rd(scale2, __fmul_rd(Dp, Dp)) : 0.f;
        const bool kp = keep[i] && !(lb2 > thr[i]);  // NaN (a PAA beyond fp16): no pruning
        const unsigned mk = __ballot_sync(0xffffffffu, sub == 0 && kp);
        if (sub == 0 && kp) {
          const int at = nout + __popc(mk & ((1u << lane) - 1u));
          queue[at] = key[kRefMRows * half + i];
          qb[at] = (uint8_t)b;
          qt[at] = thr[i];
        }
        nout += __popc(mk);
      }
    }
    __syncwarp();
    if (!R16) {
      for (int e = 0; e < nout; ++e) refine_one(queue[e], qb[e]);
      __syncwarp();
      return;
    }
    // bf16 stage over the PAA survivors: octet o takes entries r0 + o and r0 + 4 + o
    for (int r0 = 0; r0 < nout; r0 += 8) {
      uint64_t kc[2];
      int bc[2];
      bool live[2];
      float thr[2];
      const uint4* row[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int e = r0 + 4 * c + oct;
        kc[c] = e < nout ? queue[e] : kNoKey;
        bc[c] = e < nout ? (int)qb[e] : 0;
        thr[c] = e < nout ? qt[e] : 0.f;
        live[c] = e < nout;
        row[c] = reinterpret_cast<const uint4*>(a.raw16 + (size_t)key_id(kc[c]) * a.len);
      }
      float s2[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
      for (int i0 = 0; i0 < nper; i0 += kRefMH) {  // kRefMH uint4 per candidate in flight (registers)
        uint4 h[2][kRefMH];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < kRefMH; ++i) {
            const int f = sub + 8 * (i0 + i);
            h[c][i] = (live[c] && i0 + i < nper && f < nh) ? ld_stream_u4(row[c] + f) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
        for (int i = 0; i < kRefMH; ++i) {
          const int f = sub + 8 * (i0 + i);
          if (i0 + i >= nper || f >= nh) break;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)bc[c] * a.len);
            const float4 q0 = __ldg(qv + 2 * f), q1 = __ldg(qv + 2 * f + 1);  // L1-resident queries
            const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
            const uint32_t w4[4] = {h[c][i].x, h[c][i].y, h[c][i].z, h[c][i].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float d = __uint_as_float((e & 1) ? (w4[e >> 1] & 0xFFFF0000u) : (w4[e >> 1] << 16)) - qq[e];
              s2[c][e & 1] = fmaf(d, d, s2[c][e & 1]);
            }
          }
        }
      }
      bool keep[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        live[c] = live[c] && key_val(kc[c]) <= thr[c];
        if (sub == 0 && live[c]) atomicAdd(&s_r16[bc[c]], 1u);
        float v = s2[c][0] + s2[c][1];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        const float lb = bf16_lb(v, s_qn[bc[c]], e2);
        keep[c] = live[c] && !(lb > 0.f && __fmul_rd(lb, lb) > thr[c]);
      }
      // survivors (octet leaders' bits): exact fp32 distance, one row at a time
      unsigned m2 = __ballot_sync(0xffffffffu, sub == 0 && keep[0]);
      unsigned m3 = __ballot_sync(0xffffffffu, sub == 0 && keep[1]);
      while (m2 | m3) {
        const bool from2 = m2 != 0u;
        const int src = __ffs(from2 ? m2 : m3) - 1;
        if (from2) m2 &= m2 - 1; else m3 &= m3 - 1;
        const uint64_t k = __shfl_sync(0xffffffffu, from2 ? kc[0] : kc[1], src);
        const int b = __shfl_sync(0xffffffffu, from2 ? bc[0] : bc[1], src);
        refine_one(k, b);
      }
    }
    __syncwarp();
  };

  int qn = 0;
  // the chunk stream: the keys of the next kRefMKP chunks in flight (a register ring of
  // (query, key)), the query's BSF word read one chunk ahead
  auto fetch = [&](unsigned gc, int& b, uint64_t& k) {
    if (gc >= TC) { b = 0; k = kNoKey; return; }
    b = chunk_query(gc);
    const unsigned i = (gc - s_off[b]) * 32u + lane;
    k = i < s_cnt[b] ? __ldg(a.sorted + (size_t)b * a.cap + i) : kNoKey;
  };
  int rb[kRefMKP];
  uint64_t rk[kRefMKP];
#pragma unroll
  for (int r = 0; r < kRefMKP; ++r) fetch(gw + (unsigned)r * GW, rb[r], rk[r]);
  uint64_t bsfn = ld_relaxed_u64(a.best + (size_t)rb[0] * kPadU64);
  for (unsigned gc = gw; gc < TC; gc += GW) {
    const int b = rb[0];
    const uint64_t k0 = rk[0], bsf = bsfn;
#pragma unroll
    for (int r = 0; r + 1 < kRefMKP; ++r) { rb[r] = rb[r + 1]; rk[r] = rk[r + 1]; }
    fetch(gc + (unsigned)kRefMKP * GW, rb[kRefMKP - 1], rk[kRefMKP - 1]);
    bsfn = ld_relaxed_u64(a.best + (size_t)rb[0] * kPadU64);
    const float thr = thr_of(bsf);
    const float lb0 = key_val(k0);
    const int bin = lb_bin(lb0, s_scale[b]);
    const int cutb = (int)s_cut[b];
    const bool pass = k0 != kNoKey && (wave == 0 ? bin <= cutb : bin > cutb) && lb0 <= thr;
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    if (pass) {
      const int at = qn + __popc(m & ((1u << lane) - 1u));
      queue[at] = k0;
      qb[at] = (uint8_t)b;
      qt[at] = thr;
    }
    qn += __popc(m);
    __syncwarp();
    if (qn >= 32) {
      drain(32);
      __syncwarp();
      if (lane < qn - 32) {
        queue[lane] = queue[32 + lane];  // the rest to the front
        qb[lane] = qb[32 + lane];
        qt[lane] = qt[32 + lane];
      }
      qn -= 32;
      __syncwarp();
    }
  }
  if (qn > 0) drain(qn);
  __syncthreads();
  if (tid < nb && s_refined[tid]) atomicAdd(&a.refined[tid], s_refined[tid]);
  if (R16 && tid < nb && s_r16[tid]) atomicAdd(&a.refined16[tid], s_r16[tid]);
  if (tid < nb && s_paa[tid] && a.paa_rows) atomicAdd(&a.paa_rows[tid], s_paa[tid]);
}

// ---------------------------------------------------------------- K6, k > 1 (append, then select)
// The query-wide threshold from the refined-distance histogram: at least k distinct
// refined series have fp32 d^2 < (t + 2) / scale for the first bin t where the count
// reaches k (one bin of slack for the rounding of d^2 * scale), so that edge x d2up
// bounds the global k-th exact d^2.  One warp; lowers a.thr[b] (atomicMin on bits).
__device__ __forceinline__ float hist_threshold(const RefineArgs& a, int b, float scale) {
  const int lane = threadIdx.x & 31;
  const uint4 h0 = __ldcg(reinterpret_cast<const uint4*>(a.ghist + b * kNB + 8 * lane));  // L2: the atomics' copy
  const uint4 h1 = __ldcg(reinterpret_cast<const uint4*>(a.ghist + b * kNB + 8 * lane + 4));
  const unsigned hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
  unsigned own = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) own += hv[i];
  unsigned incl = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned reach = __ballot_sync(0xffffffffu, incl >= (unsigned)a.k);
  float up = INFINITY;
  if (reach) {
    const int L = __ffs(reach) - 1;
    if (lane == L) {
      unsigned c = incl - own;
      int t = 8 * L + 7;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c += hv[i];
        if (c >= (unsigned)a.k) { t = 8 * L + i; break; }
      }
      up = __fmul_ru(__fdiv_ru((float)(t + 2), scale), a.d2up);
      atomicMin(&a.thr[b * kPadU32], __float_as_uint(up));
    }
    up = __shfl_sync(0xffffffffu, up, L);
  }
  return up;
}

// Refine up to U candidates for k > 1: exact d^2 with early abandoning at thr; each
// completed distance is appended to the query's result list and counted in its
// histogram.  Returns the number of completed rows (for the threshold cadence).
template <int NC, int U>
__device__ __forceinline__ int refine_group_k(const RefineArgs& a, const float4* __restrict__ qv, int b, float scale,
                                              const uint64_t (&key)[U], bool (&live)[U], float thr,
                                              uint64_t* __restrict__ res, unsigned* __restrict__ res_cnt,
                                              unsigned& nref) {
  const int lane = threadIdx.x & 31;
  const int nf = a.len >> 2;
  float4 x[U][NC];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int f = lane + 32 * c;
      x[u][c] = (live[u] && f < nf)
                    ? ld_stream(reinterpret_cast<const float4*>(a.raw + (size_t)key_id(key[u]) * a.len) + f)
                    : make_float4(0, 0, 0, 0);
    }
  float acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const float4 q = (lane + 32 * c < nf) ? __ldg(qv + lane + 32 * c) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float d;
      d = x[u][c].x - q.x; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].y - q.y; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].z - q.z; acc[u] = fmaf(d, d, acc[u]);
      d = x[u][c].w - q.w; acc[u] = fmaf(d, d, acc[u]);
    }
    if (c + 1 < NC && 32 * (c + 1) < nf) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u] && warp_sum(acc[u]) > thr) { live[u] = false; ++nref; }
      bool any = false;
#pragma unroll
      for (int u = 0; u < U; ++u) any |= live[u];
      if (!any) return 0;
    }
  }
  int done = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!live[u]) continue;
    ++nref;
    const float d2 = warp_sum(acc[u]);
    if (d2 > thr) continue;
    ++done;
    if (lane == 0) {
      res[(size_t)b * a.cap + atomicAdd(&res_cnt[b], 1u)] = make_key(d2, key_id(key[u]));
      const float f = d2 * scale;
      if (f < (float)(kNB - 2)) atomicAdd(&a.ghist[b * kNB + (int)f], 1u);
    }
  }
  return done;
}

// k > 1 refinement without rounds: every warp walks its rotated share of every query's
// unsorted candidate list (as k_refine1u, in the same two LB waves), skips candidates
// above the query's live threshold, refines the rest U at a time, appends completed
// (d^2, id) keys to the query's result list, and lowers the threshold from the
// query-wide histogram after every 16 rows it completed.  k_select_topk then picks
// the exact top-k of the results.
template <int NC, int U, int W2 = 0>
__global__ void __launch_bounds__(kRefThreads, W2 > 0 ? 4 : (NC <= 2 ? kRefUCtas : 2))
k_refine_kx(RefineArgs a, int nb, int wave, const unsigned* __restrict__ cut, uint64_t* __restrict__ res,
            unsigned* __restrict__ res_cnt) {
  __shared__ unsigned s_refined[kMaxB], s_cnt[kMaxB], s_cut[kMaxB], s_paa[kMaxB];
  __shared__ uint64_t s_queue[W2 > 0 ? kRefWarps : 1][32];
  __shared__ float s_scale[kMaxB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kMaxB) {
    const bool on = threadIdx.x < nb;
    s_refined[threadIdx.x] = 0;
    s_paa[threadIdx.x] = 0;
    s_cnt[threadIdx.x] = on ? (unsigned)imin64((int64_t)a.count[threadIdx.x], a.cap) : 0u;
    s_cut[threadIdx.x] = on ? cut[threadIdx.x * kNB] : 0u;
    s_scale[threadIdx.x] = on ? bin_scale(__uint_as_float(a.thr_seed[threadIdx.x])) : 0.f;
  }
  __syncthreads();
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  const int sub = lane & 7;
  for (int b = 0; b < nb; ++b) {
    const unsigned cnt = s_cnt[b];
    const unsigned nchunk = (cnt + 31) / 32;
    const unsigned first = (gw + (unsigned)b * 613u) % GW;
    if (first >= nchunk) continue;
    const float scale = s_scale[b];
    const int cutb = (int)s_cut[b];
    const uint64_t* list = a.sorted + (size_t)b * a.cap;
    const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
    unsigned nref = 0, npaa = 0;
    int since = 0;
    float qpl[W2 > 0 ? W2 / 8 : 1];  // this lane's query PAA values (the PAA pre-filter)
    float qpn_hi = 0.f;
    if (W2 > 0) {
      const float* qx = a.qaux + (size_t)b * kQAux;
#pragma unroll
      for (int e = 0; e < (W2 > 0 ? W2 / 8 : 1); ++e) qpl[e] = __ldg(qx + 16 + sub * (W2 / 8) + e);
      qpn_hi = __ldg(qx + 1);
    }
    // wave B starts from the threshold wave A's results imply
    if (wave == 1 && scale > 0.f) hist_threshold(a, b, scale);
    uint64_t knext = (first * 32 + lane < cnt) ? __ldg(list + first * 32 + lane) : kNoKey;
    for (unsigned ch = first; ch < nchunk; ch += GW) {
      const unsigned i = ch * 32 + lane;
      const uint64_t k0 = knext;
      {
        const unsigned in = (ch + GW) * 32 + lane;
        knext = (ch + GW < nchunk && in < cnt) ? __ldg(list + in) : kNoKey;
      }
      float thr = __uint_as_float(ld_relaxed_u32(&a.thr[b * kPadU32]));
      const float lb0 = key_val(k0);
      const int bin = lb_bin(lb0, scale);
      const bool mine = i < cnt && (wave == 0 ? bin <= cutb : bin > cutb);
      unsigned m = __ballot_sync(0xffffffffu, mine && lb0 <= thr);
      uint64_t kq = k0;  // the candidates' keys, one per lane (compacted by the PAA stage)
      if (W2 > 0 && m) {
        uint64_t* queue = s_queue[W2 > 0 ? warp : 0];
        if (mine && lb0 <= thr) queue[__popc(m & ((1u << lane) - 1u))] = k0;
        __syncwarp();
        const int nk = paa_filter_queue<W2>(a, queue, __popc(m), thr, qpl, qpn_hi, npaa);
        kq = lane < nk ? queue[lane] : kNoKey;
        m = nk >= 32 ? 0xffffffffu : ((1u << nk) - 1u);
        __syncwarp();
      }
      while (m) {
        uint64_t key[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = m ? __ffs(m) - 1 : 0;
          const bool has = m != 0u;
          m &= m - 1;
          key[u] = __shfl_sync(0xffffffffu, kq, src);
          live[u] = has && key_val(key[u]) <= thr;
        }
        since += refine_group_k<NC, U>(a, qv, b, scale, key, live, thr, res, res_cnt, nref);
        if (since >= 8 && scale > 0.f) {
          since = 0;
          thr = fminf(thr, hist_threshold(a, b, scale));
        }
      }
    }
    if (lane == 0 && nref) atomicAdd(&s_refined[b], nref);
    if (W2 > 0 && lane == 0 && npaa) atomicAdd(&s_paa[b], npaa);
  }
  __syncthreads();
  if (threadIdx.x < nb && s_refined[threadIdx.x]) atomicAdd(&a.refined[threadIdx.x], s_refined[threadIdx.x]);
  if (W2 > 0 && threadIdx.x < nb && s_paa[threadIdx.x] && a.paa_rows)
    atomicAdd(&a.paa_rows[threadIdx.x], s_paa[threadIdx.x]);
}

// Exact top-k of a query's result list: every true top-k member is there (its exact
// d^2 <= the final threshold, so it was neither pruned nor abandoned nor dropped).
// Narrow a d^2 window [0, hi) with 256-bin shared histograms until it holds at most
// kSortP keys but at least k (or everything), gather the window, bitonic-sort it,
// write the first k ascending (d^2, id).  A window that cannot be narrowed below
// kSortP keys (massive exact ties) falls back to merging fixed index ranges.
__global__ void __launch_bounds__(1024)
k_select_topk(const uint64_t* __restrict__ res, const unsigned* __restrict__ res_cnt, int64_t cap,
              const unsigned* __restrict__ thr, int k, int q0, int64_t* __restrict__ out_idx,
              float* __restrict__ out_dist, const unsigned* __restrict__ count, const unsigned* __restrict__ refined,
              unsigned* __restrict__ all_count, unsigned* __restrict__ all_refined, int accum,
              const unsigned* __restrict__ blocks, unsigned* __restrict__ all_blocks,
              const unsigned* __restrict__ extra, unsigned* __restrict__ all_extra) {
  __shared__ uint64_t buf[kSortP];
  __shared__ unsigned s_h[kNB];
  __shared__ unsigned s_n;
  __shared__ float s_hi;
  const int b = blockIdx.x;
  const unsigned L = (unsigned)imin64((int64_t)res_cnt[b], cap);
  const uint64_t* src = res + (size_t)b * cap;
  float hi = __uint_as_float(thr[b * kPadU32]);  // every key is <= hi (appended only if d^2 <= thr)
  bool narrowed = false;  // window = keys with d^2 < hi once narrowed, else every key
  if (threadIdx.x == 0) s_hi = INFINITY;
  // narrowing: the first bin where the running count reaches k; keep [0, edge(t + 1))
  for (int it = 0; it < 4 && L > (unsigned)(kSortP - 1) && hi < INFINITY && hi > 0.f; ++it) {
    for (int i = threadIdx.x; i < kNB; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    const float sc = (float)kNB / hi;
    for (unsigned i = threadIdx.x; i < L; i += blockDim.x) {
      const float v = key_val(src[i]);
      if (v < hi) atomicAdd(&s_h[min((int)(v * sc), kNB - 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned own = 0;
      for (int j = 0; j < 8; ++j) own += s_h[8 * lane + j];
      unsigned incl = own;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned reach = __ballot_sync(0xffffffffu, incl >= (unsigned)k);
      if (lane == 0) s_hi = hi;
      if (reach) {
        const int Lr = __ffs(reach) - 1;
        if (lane == Lr) {
          unsigned c = incl - own;
          int t = 8 * Lr + 7;
          for (int j = 0; j < 8; ++j) {
            c += s_h[8 * Lr + j];
            if (c >= (unsigned)k) { t = 8 * Lr + j; break; }
          }
          // keys of bins <= t + 1 (one bin of slack for the rounding of v * sc)
          if (t + 2 < kNB) s_hi = __fdiv_ru((float)(t + 2), sc);
        }
      }
    }
    __syncthreads();
    const float nh = s_hi;
    __syncthreads();
    if (!(nh < hi)) break;
    hi = nh;
    narrowed = true;
    // count the keys left in the window
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    unsigned mine = 0;
    for (unsigned i = threadIdx.x; i < L; i += blockDim.x) mine += key_val(src[i]) < hi ? 1u : 0u;
    atomicAdd(&s_n, mine);
    __syncthreads();
    if (s_n <= (unsigned)kSortP) break;
  }
  // gather the window and sort it (or merge index ranges when it is still too large)
  for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = kNoKey;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  bool over = false;
  for (unsigned i = threadIdx.x; i < L; i += blockDim.x) {
    const uint64_t key = src[i];
    if (!narrowed || key_val(key) < hi) {
      const unsigned pos = atomicAdd(&s_n, 1u);
      if (pos < (unsigned)kSortP) buf[pos] = key;
      else over = true;
    }
  }
  if (__syncthreads_or(over)) {
    // fallback: running top-k over fixed index windows of kSortP - k entries
    for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = kNoKey;
    __syncthreads();
    const unsigned W = (unsigned)(kSortP - k);
    for (unsigned off = 0; off < L; off += W) {
      for (unsigned i = threadIdx.x; i < W; i += blockDim.x) buf[k + i] = (off + i < L) ? src[off + i] : kNoKey;
      __syncthreads();
      bitonic_sort(buf, kSortP);
    }
  } else {
    bitonic_sort(buf, kSortP);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = buf[i];
    const size_t o = (size_t)(q0 + b) * k + i;
    if (key == kNoKey) { out_idx[o] = -1; out_dist[o] = INFINITY; }
    else { out_idx[o] = (int64_t)key_id(key); out_dist[o] = sqrtf(key_val(key)); }
  }
  if (threadIdx.x == 0) {
    all_count[q0 + b] = (accum ? all_count[q0 + b] : 0u) + count[b];
    all_refined[q0 + b] = (accum ? all_refined[q0 + b] : 0u) + refined[b];
    all_blocks[q0 + b] = (accum ? all_blocks[q0 + b] : 0u) + blocks[b];
    all_extra[q0 + b] = (accum ? all_extra[q0 + b] : 0u) + extra[b];
  }
}

// k > 1: rounds of (every warp: one refine_step) -> merge the round's admitted
// keys into the CTA's sorted top-k -> publish the k-th (rounded up) to the
// query's global threshold.  Each true top-k member lands in the top-k of the
// CTA that refined it, so merging the per-CTA lists (K7) is exact.
__global__ void __launch_bounds__(kRefThreads)
k_refine_topk(RefineArgs a) {
  extern __shared__ float4 s_dyn[];
  const int k = a.k;
  float4* s_qv = s_dyn;
  uint64_t* s_top = reinterpret_cast<uint64_t*>(s_dyn + (a.len >> 2));
  uint64_t* s_new = s_top + k;
  __shared__ uint64_t s_pend[kRefWarps * kU];
  __shared__ int s_np;
  __shared__ float s_thr_local;
  __shared__ uint64_t s_kthkey;
  __shared__ unsigned s_refined;
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4* qsrc = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
  for (int i = threadIdx.x; i < (a.len >> 2); i += blockDim.x) s_qv[i] = qsrc[i];
  for (int i = threadIdx.x; i < k; i += blockDim.x) s_top[i] = kNoKey;
  if (threadIdx.x == 0) {
    s_np = 0;
    s_thr_local = INFINITY;
    s_kthkey = kNoKey;
    s_refined = 0;
  }
  __syncthreads();
  const unsigned cnt = (unsigned)imin64((int64_t)a.count[b], a.cap);
  const float scale = bin_scale(__uint_as_float(a.thr_seed[b]));
  const uint64_t* list = a.sorted + (size_t)b * a.cap;
  const unsigned gw = blockIdx.x * kRefWarps + warp, GW = gridDim.x * kRefWarps;
  unsigned nref = 0;
  unsigned round_no = 0;
  bool done = false;
  for (unsigned i0 = gw;; i0 += kU * GW) {
    if (!done && i0 < cnt) {
      const float thr = fminf(__uint_as_float(ld_relaxed_u32(&a.thr[b * kPadU32])), s_thr_local);
      uint64_t key[kU];
      float d2[kU];
      done = refine_step(a, list, cnt, i0, GW, thr, scale, s_qv, key, d2, nref);
      const uint64_t kk = s_kthkey;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (d2[u] < INFINITY) {
          const uint64_t k2 = make_key(d2[u], key_id(key[u]));
          if (k2 < kk && lane == 0) s_pend[atomicAdd(&s_np, 1)] = k2;
          // the query-wide histogram of exact distances (all CTAs): its k-th count
          // bounds the global k-th distance, which one CTA's own top-k cannot
          const float f = d2[u] * scale;
          if (lane == 0 && f < (float)(kNB - 2)) atomicAdd(&a.ghist[b * kNB + (int)f], 1u);
        }
      }
    } else {
      done = true;
    }
    __syncthreads();
    const int np = s_np;
    if (np > 0) {
      if (warp == 0) {
        uint64_t v = (lane < np) ? s_pend[lane] : kNoKey;
        v = warp_sort32(v);
        s_pend[lane] = v;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < k; t += blockDim.x) {
        const uint64_t key = s_top[t];
        int lo = 0, hi = np;  // # pending < key
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_pend[mid] < key) lo = mid + 1; else hi = mid; }
        const int r = t + lo;
        if (r < k) s_new[r] = key;
      }
      for (int j = threadIdx.x; j < np; j += blockDim.x) {
        const uint64_t key = s_pend[j];
        int lo = 0, hi = k;  // # top < key
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_top[mid] < key) lo = mid + 1; else hi = mid; }
        const int r = j + lo;
        if (r < k) s_new[r] = key;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < k; t += blockDim.x) s_top[t] = s_new[t];
      __syncthreads();
      if (threadIdx.x == 0) {
        s_np = 0;
        const uint64_t kk = s_top[k - 1];
        s_kthkey = kk;
        if (kk != kNoKey) {
          const float up = __fmul_ru(key_val(kk), a.d2up);
          s_thr_local = up;
          atomicMin(&a.thr[b * kPadU32], __float_as_uint(up));
        }
      }
    }
    // every 4th round: the query-wide threshold from the histogram -- at least k refined
    // series have fp32 d^2 < (t + 2) / scale (one bin of slack for the rounding of
    // d^2 * scale), so the global k-th exact d^2 <= that edge x d2up
    if (warp == 0 && (++round_no & 3) == 0 && scale > 0.f) {
      const uint4 h0 = __ldcg(reinterpret_cast<const uint4*>(a.ghist + b * kNB + 8 * lane));  // L2: the atomics' copy
      const uint4 h1 = __ldcg(reinterpret_cast<const uint4*>(a.ghist + b * kNB + 8 * lane + 4));
      const unsigned hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
      unsigned own = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) own += hv[i];
      unsigned incl = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned reach = __ballot_sync(0xffffffffu, incl >= (unsigned)k);
      if (reach) {
        const int L = __ffs(reach) - 1;
        if (lane == L) {
          unsigned c = incl - own;
          int t = 8 * L;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            c += hv[i];
            if (c >= (unsigned)k) { t = 8 * L + i; break; }
          }
          const float up = __fmul_ru(__fdiv_ru((float)(t + 2), scale), a.d2up);
          if (up < s_thr_local) {
            s_thr_local = up;
            atomicMin(&a.thr[b * kPadU32], __float_as_uint(up));
          }
        }
      }
    }
    if (!__syncthreads_or(!done)) break;
  }
  if (lane == 0 && nref) atomicAdd(&s_refined, nref);
  __syncthreads();
  uint64_t* out = a.lists + ((size_t)b * gridDim.x + blockIdx.x) * k;
  for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = s_top[i];
  if (threadIdx.x == 0 && s_refined) atomicAdd(&a.refined[b], s_refined);
}

// ---------------------------------------------------------------- K7 finalize
__global__ void k_finalize1(const unsigned long long* __restrict__ best, int nb, int q0,
                            int64_t* __restrict__ out_idx, float* __restrict__ out_dist,
                            const unsigned* __restrict__ count, const unsigned* __restrict__ refined,
                            unsigned* __restrict__ all_count, unsigned* __restrict__ all_refined, int accum,
                            const unsigned* __restrict__ blocks, unsigned* __restrict__ all_blocks,
                            const unsigned* __restrict__ extra, unsigned* __restrict__ all_extra) {
  const int b = threadIdx.x;
  if (b >= nb) return;
  const uint64_t key = best[b * kPadU64];
  if (key == kNoKey || key_id(key) == kSentinelId) { out_idx[q0 + b] = -1; out_dist[q0 + b] = INFINITY; }
  else { out_idx[q0 + b] = (int64_t)key_id(key); out_dist[q0 + b] = sqrtf(key_val(key)); }
  all_count[q0 + b] = (accum ? all_count[q0 + b] : 0u) + count[b];
  all_refined[q0 + b] = (accum ? all_refined[q0 + b] : 0u) + refined[b];
  all_blocks[q0 + b] = (accum ? all_blocks[q0 + b] : 0u) + blocks[b];
  all_extra[q0 + b] = (accum ? all_extra[q0 + b] : 0u) + extra[b];
}

// Merge the per-CTA top-k lists: repeatedly sort [current top-k | next chunk]
// in shared memory and keep the first k.  Output ascending (d^2, id) -> (id, sqrt d^2).
__global__ void __launch_bounds__(1024)
k_finalize(const uint64_t* __restrict__ lists, int nslots, int k, int q0,
           int64_t* __restrict__ out_idx, float* __restrict__ out_dist,
           const unsigned* __restrict__ count, const unsigned* __restrict__ refined,
           unsigned* __restrict__ all_count, unsigned* __restrict__ all_refined, int accum,
           const unsigned* __restrict__ blocks, unsigned* __restrict__ all_blocks,
           const unsigned* __restrict__ extra, unsigned* __restrict__ all_extra) {
  __shared__ uint64_t buf[kSortP];
  const int b = blockIdx.x;
  const int64_t total = (int64_t)nslots * k;
  const uint64_t* src = lists + (size_t)b * nslots * k;
  for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = kNoKey;
  __syncthreads();
  const int chunk = kSortP - k;
  for (int64_t off = 0; off < total; off += chunk) {
    for (int i = threadIdx.x; i < chunk; i += blockDim.x)
      buf[k + i] = (off + i < total) ? src[off + i] : kNoKey;
    __syncthreads();
    bitonic_sort(buf, kSortP);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = buf[i];
    const size_t o = (size_t)(q0 + b) * k + i;
    if (key == kNoKey) { out_idx[o] = -1; out_dist[o] = INFINITY; }
    else { out_idx[o] = (int64_t)key_id(key); out_dist[o] = sqrtf(key_val(key)); }
  }
  if (threadIdx.x == 0) {
    all_count[q0 + b] = (accum ? all_count[q0 + b] : 0u) + count[b];
    all_refined[q0 + b] = (accum ? all_refined[q0 + b] : 0u) + refined[b];
    all_blocks[q0 + b] = (accum ? all_blocks[q0 + b] : 0u) + blocks[b];
    all_extra[q0 + b] = (accum ? all_extra[q0 + b] : 0u) + extra[b];
  }
}

// ---------------------------------------------------------------- candidate-buffer overflow
// A query whose LB pass kept more than `cap` candidates (count[b] > cap) had only the
// stored ones refined.  Its result so far is a real BSF (k = 1: the best key; k > 1:
// the live threshold thr[b], a rigorous bound of the k-th exact distance), so an exact
// answer needs every series whose bound is below it -- this kernel scans them all
// without a candidate buffer: a rigorous fp32 MINDIST (outward fp32 regions, round-down
// arithmetic) per series, the survivors refined at once (fused LB -> refine, the
// DistComp loop of Alg8, with the BSF shared as in ParIS+).  k = 1 lowers
// the shared BSF key; k > 1 keeps a warp-private top-k (shared memory) whose k-th also
// lowers thr[b]; the warps' lists are merged by k_finalize_ovf.  Gated on the device:
// every CTA leaves at once when no query of the batch overflowed, so the host never
// waits for the counts.
struct FbArgs {
  const uint8_t* sax;      // flat [w][n], or the index's tile-major sorted array (perm != nullptr)
  const uint32_t* perm;
  int64_t n;
  int w, len;
  float seglen_f;
  const CardTables* tab;
  const float2* g_q;       // [slot][kMaxW] query PAA intervals (round down, round up)
  const float* queries;    // batch [nb][len]
  const float* raw;
  int nb;
  const unsigned* count;
  int64_t cap;
  int k;
  float d2up;
  unsigned long long* best;  // k = 1
  unsigned* thr;             // k > 1: per query (kPadU32 stride), float bits
  uint64_t* lists;           // k > 1: [nb][L][k]
  int L;                     // warps of the grid (lists per query)
  unsigned* refined;         // per query: rows refined here
};
constexpr int kFbThreads = 128;

// Up to 4 rows refined together (4 rows in flight per lane step), early abandoning at
// thr after each 128-point chunk; d2[u] = +inf when abandoned or not live.
__device__ __forceinline__ void fb_refine4(const float* __restrict__ raw, int len, const float4* __restrict__ qv,
                                           const uint32_t (&id)[4], bool (&live)[4], float thr, float (&d2)[4]) {
  const int lane = threadIdx.x & 31;
  const int nf = len >> 2;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c0 = 0; c0 < nf; c0 += 32) {
    const int f = c0 + lane;
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      x[u] = (live[u] && f < nf) ? ld_stream(reinterpret_cast<const float4*>(raw + (size_t)id[u] * len) + f)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 q = f < nf ? __ldg(qv + f) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float d;
      d = x[u].x - q.x; acc[u] = fmaf(d, d, acc[u]);
      d = x[u].y - q.y; acc[u] = fmaf(d, d, acc[u]);
      d = x[u].z - q.z; acc[u] = fmaf(d, d, acc[u]);
      d = x[u].w - q.w; acc[u] = fmaf(d, d, acc[u]);
    }
    if (c0 + 32 < nf) {
      bool any = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (live[u] && warp_sum(acc[u]) > thr) live[u] = false;  // early abandoning
        any |= live[u];
      }
      if (!any) break;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) d2[u] = live[u] ? warp_sum(acc[u]) : INFINITY;
}

// FAST (w == 16, n % 4 == 0): a lane bounds 4 consecutive series per step from one 32-bit
// word per segment row (16 independent loads in flight); else one series per lane.
template <bool K1, bool FAST>
__global__ void __launch_bounds__(kFbThreads)
k_fallback(FbArgs a) {
  extern __shared__ uint64_t s_top[];  // k > 1: [warps][k] ascending keys
  __shared__ float2 s_lu[kMaxCard];
  __shared__ float2 s_q[kMaxW];
  __shared__ int s_any;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int any = 0;
    for (int b = 0; b < a.nb; ++b) any |= (int64_t)a.count[b] > a.cap;
    s_any = any;
  }
  __syncthreads();
  if (!s_any) return;  // the common case: one shared load, then exit
  for (int i = tid; i < kMaxCard; i += blockDim.x) s_lu[i] = a.tab->lu[i];
  constexpr int SPL = FAST ? 4 : 1;  // series per lane per step
  const int nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int64_t per = ((a.n + (int64_t)a.L - 1) / a.L + 32 * SPL - 1) / (32 * SPL) * (32 * SPL);
  const int64_t lo = imin64(a.n, (int64_t)gw * per), hi = imin64(a.n, lo + per);
  uint64_t* top = s_top + (size_t)warp * (K1 ? 1 : a.k);
  for (int b = 0; b < a.nb; ++b) {
    if ((int64_t)a.count[b] <= a.cap) continue;
    __syncthreads();
    for (int i = tid; i < kMaxW; i += blockDim.x) s_q[i] = a.g_q[b * kMaxW + i];
    __syncthreads();
    const float4* qv = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
    unsigned long long* bp = a.best + (size_t)b * kPadU64;
    uint64_t cur = K1 ? ld_relaxed_u64(bp) : kNoKey;
    int filled = 0;  // k > 1: entries in this warp's list
    if (!K1)
      for (int i = lane; i < a.k; i += 32) top[i] = kNoKey;
    __syncwarp();
    unsigned nref = 0;
    auto cur_thr = [&]() -> float {
      if (K1) {
        cur = min(cur, ld_relaxed_u64(bp));
        return cur == kNoKey ? INFINITY : __fmul_ru(key_val(cur), a.d2up);
      }
      float t = __uint_as_float(ld_relaxed_u32(&a.thr[b * kPadU32]));
      if (filled == a.k) t = fminf(t, __fmul_ru(key_val(top[a.k - 1]), a.d2up));
      return t;
    };
    for (int64_t base = lo; base < hi; base += 32 * SPL) {
      const int64_t i0 = base + (int64_t)SPL * lane;
      float lb[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
      uint32_t id[4] = {0u, 0u, 0u, 0u};
      if (FAST) {
        if (i0 < hi) {  // hi % 4 == 0 (n % 4 == 0, per % 4 == 0)
          uint32_t wd[kTW];
#pragma unroll
          for (int s2 = 0; s2 < kTW; ++s2)
            wd[s2] = a.perm ? __ldg(reinterpret_cast<const uint32_t*>(
                                  a.sax + (size_t)(i0 / kTS) * kTW * kTS + (size_t)s2 * kTS + i0 % kTS))
                            : __ldg(reinterpret_cast<const uint32_t*>(a.sax + (size_t)s2 * a.n + i0));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < kTW; ++s2) {
              const float2 r = s_lu[(wd[s2] >> (8 * j)) & 0xFFu];  // {L rounded down, U rounded up}
              const float2 q = s_q[s2];                            // {q rounded down, q rounded up}
              const float d = fmaxf(fmaxf(__fsub_rd(q.x, r.y), __fsub_rd(r.x, q.y)), 0.f);
              acc = __fadd_rd(acc, __fmul_rd(d, d));
            }
            lb[j] = __fmul_rd(acc, a.seglen_f);
            id[j] = a.perm ? __ldg(a.perm + i0 + j) : (uint32_t)(i0 + j);
          }
        }
      } else if (i0 < hi) {
        float acc = 0.f;
        for (int s2 = 0; s2 < a.w; ++s2) {
          const uint8_t sym = a.perm ? a.sax[(size_t)(i0 / kTS) * kTW * kTS + (size_t)s2 * kTS + i0 % kTS]
                                     : a.sax[(size_t)s2 * a.n + i0];
          const float2 r = s_lu[sym];
          const float2 q = s_q[s2];
          const float d = fmaxf(fmaxf(__fsub_rd(q.x, r.y), __fsub_rd(r.x, q.y)), 0.f);
          acc = __fadd_rd(acc, __fmul_rd(d, d));
        }
        lb[0] = __fmul_rd(acc, a.seglen_f);
        id[0] = a.perm ? __ldg(a.perm + i0) : (uint32_t)i0;
      }
      float thr = cur_thr();
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        unsigned m = __ballot_sync(0xffffffffu, lb[j] <= thr);
        while (m) {
          uint32_t cid[4];
          bool live[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int src = m ? __ffs(m) - 1 : 0;
            live[u] = m != 0u;
            m &= m - 1;
            cid[u] = __shfl_sync(0xffffffffu, id[j], src);
            live[u] = live[u] && __shfl_sync(0xffffffffu, lb[j], src) <= thr;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) nref += live[u] ? 1u : 0u;  // raw rows read
          float d2[4];
          fb_refine4(a.raw, a.len, qv, cid, live, thr, d2);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (d2[u] == INFINITY) continue;
            const uint64_t key = make_key(d2[u], cid[u]);
            if (K1) {
              if (key < cur) {
                if (lane == 0) atomicMin(bp, (unsigned long long)key);
                cur = key;
                thr = fminf(thr, __fmul_ru(d2[u], a.d2up));
              }
            } else if (filled < a.k || key < top[a.k - 1]) {
              // sorted insert into the warp's list: rank = #entries < key
              int r = 0;
              for (int jj = lane; jj < filled; jj += 32) r += top[jj] < key;
              r = __reduce_add_sync(0xffffffffu, r);
              const int last = min(filled, a.k - 1);  // entries [r, last) move up by one
              for (int hi2 = last; hi2 > r; hi2 -= 32) {
                const int jj = hi2 - 1 - lane;
                const uint64_t v = (jj >= r) ? top[jj] : 0ull;
                __syncwarp();
                if (jj >= r) top[jj + 1] = v;
                __syncwarp();
              }
              if (lane == 0) top[r] = key;
              __syncwarp();
              filled = min(filled + 1, a.k);
              if (filled == a.k) {
                const float t = __fmul_ru(key_val(top[a.k - 1]), a.d2up);
                if (lane == 0) atomicMin(&a.thr[b * kPadU32], __float_as_uint(t));
                thr = fminf(thr, t);
              }
            }
          }
        }
      }
    }
    if (!K1) {
      uint64_t* out = a.lists + ((size_t)b * a.L + gw) * a.k;
      for (int j = lane; j < a.k; j += 32) out[j] = top[j];
    }
    if (lane == 0 && nref) atomicAdd(&a.refined[b], nref);
  }
}

// Merge sorted lists (nlists x k keys per query) into the query's top-k; ascending
// (d^2, id) -> (id, sqrt d^2).  One CTA of 1024 threads per query.
__device__ void merge_lists_topk(const uint64_t* __restrict__ src, int64_t total, int k, uint64_t* buf) {
  for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = kNoKey;
  __syncthreads();
  const int chunk = kSortP - k;
  for (int64_t off = 0; off < total; off += chunk) {
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) buf[k + i] = (off + i < total) ? src[off + i] : kNoKey;
    __syncthreads();
    bitonic_sort(buf, kSortP);
  }
}

// k_fallback's outputs for the overflowed queries of a batch (others untouched).
__global__ void __launch_bounds__(1024)
k_finalize_ovf(const unsigned long long* __restrict__ best, const uint64_t* __restrict__ lists, int L, int k, int q0,
               const unsigned* __restrict__ count, int64_t cap, int64_t* __restrict__ out_idx,
               float* __restrict__ out_dist, const unsigned* __restrict__ fb_refined, unsigned* __restrict__ all_refined) {
  __shared__ uint64_t buf[kSortP];
  const int b = blockIdx.x;
  if ((int64_t)count[b] <= cap) return;
  if (k == 1) {
    if (threadIdx.x == 0) {
      const uint64_t key = best[b * kPadU64];
      const bool none = key == kNoKey || key_id(key) == kSentinelId;
      out_idx[q0 + b] = none ? -1 : (int64_t)key_id(key);
      out_dist[q0 + b] = none ? INFINITY : sqrtf(key_val(key));
    }
  } else {
    merge_lists_topk(lists + (size_t)b * L * k, (int64_t)L * k, k, buf);
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const uint64_t key = buf[i];
      const size_t o = (size_t)(q0 + b) * k + i;
      if (key == kNoKey) { out_idx[o] = -1; out_dist[o] = INFINITY; }
      else { out_idx[o] = (int64_t)key_id(key); out_dist[o] = sqrtf(key_val(key)); }
    }
  }
  if (threadIdx.x == 0) all_refined[q0 + b] += fb_refined[b];
}

// ---------------------------------------------------------------- host side
int sms() { return device_sms(); }

template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
  int v = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem);
  return v > 0 ? v : 1;
}

// scratch of one batch (device)
struct Ws {
  float2* g_q;
  uint2* g_q16;
  int* seed_ids;
  uint64_t* seed_keys;
  unsigned* zero_block;  // thr_seed | count | hist | cursor | refined (zeroed per batch)
  unsigned* thr;
  unsigned* thr_seed;
  unsigned* count;
  unsigned* hist;
  unsigned* cursor;
  unsigned* refined;
  unsigned* blocks;      // index mode: blocks whose envelope bound passed, per query
  unsigned* tile_count;  // index mode: live tiles listed
  unsigned* tile_claim;  // index mode: the block pass's next unclaimed tile
  unsigned* updates;     // nb mode: V_bsf updates per query
  unsigned* ghist;       // k > 1: refined-distance histograms [B][kNB]
  unsigned long long* bmask;  // index mode: [ntiles*32] per-block live query-slot masks
  unsigned* tile_list;   // index mode: live tiles
  unsigned* fb_refined;  // overflow fallback: rows refined per query
  uint64_t* fb_lists;    // overflow fallback, k > 1: [B][fbL][k] warp lists
  float* qaux;           // [B][80] per-query refine constants (k_qaux)
  struct GfParams* gf;   // per-pass parameters of the tensor-core filter (k_gf)
  const unsigned* lb_skip_if = nullptr;  // flat path behind k_gf: the k_lbt passes run only if it declined
  size_t zero_bytes;
  unsigned long long* best;
  uint64_t* cand;
  uint64_t* sorted;
  uint64_t* lists;
  void* base;
};

struct Plan {
  int64_t n;
  int len, w, card, k;
  int B;          // queries per SAX pass
  int S;          // seed entries per query (warps of the seed grid)
  int seed_grid;
  int64_t ns;     // seed sample
  int64_t cap;
  int XB;         // refine CTAs per query
  int wave_a;     // k = 1: candidates per query refined in the first wave
  float d2up;     // fp32 d^2 -> rigorous upper bound factor
  bool tiled;     // TMA-tiled LB kernels (n % 16 == 0, w == 16)
  const uint32_t* perm;  // index mode (paris_knn_index): sorted position -> id
  const uint8_t* env;    // index mode: block envelopes
  int idx_seeds;         // index mode: series around the query's leaf
  bool nb;               // f2: nb-ParIS+ (per-worker BSF copies, fused LB -> refine)
  bool sorted_refine = false;  // k = 1: walk bucket-sorted lists (K5) instead of the unsorted waves
  const uint16_t* raw16 = nullptr;  // optional bf16 copy of raw: refine pre-filter (k = 1)
  bool raw_host = false;            // raw in pinned host memory (f3)
  int fbL = 0;                      // overflow fallback: warps of its grid (= lists per query for k > 1)
  const __half* paa16 = nullptr;    // optional fp16 PAA of raw: refine pre-filter (k = 1)
  int w2 = 0;
  const float* tau_in = nullptr;    // external per-query bound of the k-th NN distance (device)
  bool approx = false;              // paris_knn_approx: the seeds' top-k only
  bool gf = false;                  // LB pass through the tensor-core filter (variant key 3)
};

int pairs_for(int nb) { return nb <= 2 ? 1 : nb <= 4 ? 2 : nb <= 8 ? 4 : nb <= 16 ? 8 : nb <= 32 ? 16 : 32; }

template <int P, int WT, bool AL>
cudaError_t launch_seed(const Plan& p, const uint8_t* sax, const float* qb, int nb,
                        const CardTables* tab, const Ws& ws, cudaStream_t st) {
  return PARIS_LAUNCH("seed_lb", (k_seed<P, WT, AL>), p.seed_grid, kLBThreads, 0, st, sax, p.n, p.ns,
                      qb, nb, p.len, p.w, tab, ws.g_q, ws.g_q16, ws.seed_ids, p.S);
}

template <int P, int WT, bool AL>
cudaError_t launch_lb(const Plan& p, const uint8_t* sax, int nb, const CardTables* tab, const Ws& ws,
                      cudaStream_t st, int64_t cap) {
  const int occ = cached_per_device((const void*)k_lb<P, WT, AL>,
                                    [](int) { return occupancy(k_lb<P, WT, AL>, kLBThreads, 0); });
  const int64_t ngroups = (p.n + 3) / 4;
  const int64_t need = (ngroups + kLBThreads - 1) / kLBThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms() * occ));
  LbArgs la;
  la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
  la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = nb; la.thr = ws.thr_seed; la.count = ws.count;
  la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = nullptr; la.env = nullptr;
  la.blocks = ws.blocks;
  return PARIS_LAUNCH("lb_pass", (k_lb<P, WT, AL>), grid, kLBThreads, 0, st, la);
}

template <int P, int WT>
cudaError_t dispatch_al(bool al, bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                        const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  if (lb) return al ? launch_lb<P, WT, true>(p, sax, nb, tab, ws, st, cap)
                    : launch_lb<P, WT, false>(p, sax, nb, tab, ws, st, cap);
  // the seed pass covers ~1/16 of the array: the register-light runtime-w variant
  return al ? launch_seed<P, 0, true>(p, sax, qb, nb, tab, ws, st)
            : launch_seed<P, 0, false>(p, sax, qb, nb, tab, ws, st);
}

template <int P>
cudaError_t dispatch_w(bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                       const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  const bool al = (p.n % 4) == 0;
  if (p.w == 16) return dispatch_al<P, 16>(al, lb, p, sax, qb, nb, tab, ws, st, cap);
  return dispatch_al<P, 0>(al, lb, p, sax, qb, nb, tab, ws, st, cap);
}

cudaError_t dispatch_p(int P, bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                       const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  switch (P) {
    case 1: return dispatch_w<1>(lb, p, sax, qb, nb, tab, ws, st, cap);
    case 2: return dispatch_w<2>(lb, p, sax, qb, nb, tab, ws, st, cap);
    case 4: return dispatch_w<4>(lb, p, sax, qb, nb, tab, ws, st, cap);
    default: return dispatch_w<8>(lb, p, sax, qb, nb, tab, ws, st, cap);
  }
}

template <int P, int MODE>
cudaError_t launch_lbt(const Plan& p, const uint8_t* sax, int nb, const CardTables* tab, const Ws& ws,
                       cudaStream_t st, int64_t cap, int64_t nlim, int grid) {
  cudaError_t ea = once_per_device((const void*)k_lbt<P, MODE>, [](int) {
    return cudaFuncSetAttribute(k_lbt<P, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTSmem);
  });
  if (ea != cudaSuccess) return ea;
  LbArgs la;
  la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
  la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = nb; la.thr = ws.thr_seed; la.count = ws.count;
  la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = p.perm; la.env = p.env;
  la.blocks = ws.blocks;
  la.skip_if = MODE == 1 ? ws.lb_skip_if : nullptr;
  return PARIS_LAUNCH(MODE ? "lb_pass" : "seed_lb", (k_lbt<P, MODE>), grid, kTThreads, kTSmem, st, la, nlim,
                      ws.seed_ids, p.S);
}

// dynamic shared memory of k_lbi<P, HC, S1>: everything the device allows a CTA beyond the
// kernel's static shared memory (the kernel checks its layout fits)
#include "gfilter.cuh"

static_assert(sizeof(GfParams) <= 8192, "GfParams fits its workspace slot");
cudaError_t gf_attr() {
  static int key;
  return once_per_device(&key, [](int) {
    return cudaFuncSetAttribute(k_gf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGfSmem);
  });
}
// 2-D tensor map of the SAX array for k_gf's stage copies (box: 128 series x 16 segment rows).
// Index layout: [tile][16][2048] seen as 16 * ntiles rows of 2048 bytes; flat layout: 16 rows of n bytes.
cudaError_t gf_tensor_map(const LbArgs& la, CUtensorMap* tm) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = []() -> Encode {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return nullptr;
    return (Encode)fn;
  }();
  if (!enc) return cudaErrorNotSupported;
  const int64_t ntiles = (la.n + kTS - 1) / kTS;
  cuuint64_t dims[2], strides[1];
  if (la.perm) { dims[0] = kTS; dims[1] = (cuuint64_t)(16 * ntiles); strides[0] = kTS; }
  else { dims[0] = (cuuint64_t)la.n; dims[1] = 16; strides[0] = (cuuint64_t)la.n; }
  const cuuint32_t box[2] = {(cuuint32_t)kGfRound, 16u}, es[2] = {1u, 1u};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(la.sax), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
cudaError_t launch_gf_kernel(const char* name, const LbArgs& la, const GfParams* gp, float* dump, int swap_desc,
                             cudaStream_t st) {
  cudaError_t e = gf_attr();
  if (e != cudaSuccess) return e;
  CUtensorMap tm;
  e = gf_tensor_map(la, &tm);
  if (e != cudaSuccess) return e;
  const int64_t nrounds = (la.n + kGfRound - 1) / kGfRound;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(device_sms(), (nrounds + kGfWG - 1) / kGfWG));
  return PARIS_LAUNCH(name, k_gf, grid, kGfThreads, kGfSmem, st, la, gp, dump, swap_desc, tm);
}
cudaError_t launch_gf(const LbArgs& la, int card, GfParams* gp, cudaStream_t st) {
  const cudaError_t e = PARIS_LAUNCH("lb_prep", k_gf_prep, 1, 256, 0, st, la, card, gp);
  if (e != cudaSuccess) return e;
  return launch_gf_kernel("lb_pass", la, gp, nullptr, 0, st);
}

template <int P, bool HC, int NW>
int lbi_smem() {
  return cached_per_device((const void*)k_lbi<P, HC, NW>, [](int dev) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k_lbi<P, HC, NW>) != cudaSuccess) return 0;
    const int v = optin - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(k_lbi<P, HC, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, v) != cudaSuccess) return 0;
    return v;
  });
}

template <int P, bool HC, int NW>
cudaError_t launch_lbi_pass(int grid, cudaStream_t st, const LbArgs& la, const Ws& ws) {
  const int smem = lbi_smem<P, HC, NW>();
  if (smem <= 0) return cudaErrorInvalidConfiguration;
  return PARIS_LAUNCH("lb_pass", (k_lbi<P, HC, NW>), grid, lbi_threads<NW>(), smem, st, la, ws.bmask,
                      ws.tile_list, ws.tile_count);
}

template <int P>
cudaError_t launch_index_lb(const Plan& p, const uint8_t* sax, int nb, const CardTables* tab, const Ws& ws,
                            cudaStream_t st, int64_t cap) {
  LbArgs la;
  la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
  la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = nb; la.thr = ws.thr_seed; la.count = ws.count;
  la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = p.perm; la.env = p.env;
  la.blocks = ws.blocks;
  const int64_t ntiles = (p.n + kTS - 1) / kTS;
  const int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms() * kBmCtas, (ntiles + 7) / 8));
  const unsigned* skip_if = nullptr;
  if (p.gf) {
    // tensor-core filter pass; the block pass + k_lbi below run only if it declined (gf->ok == 0)
    const cudaError_t eg = launch_gf(la, p.card, ws.gf, st);
    if (eg != cudaSuccess) return eg;
    skip_if = &ws.gf->ok;
  }
  cudaError_t e = PARIS_LAUNCH("lb_blocks", k_blkmask<P>, bgrid, 256, 0, st, la, ws.bmask, ws.tile_list,
                               ws.tile_count, ws.blocks, ws.tile_claim, skip_if);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(sms(), ntiles);
  const bool w30 = g_variant[0] == 30;  // tuning: 30 consumer warps (1024 threads) instead of 24
  if (!p.sorted_refine)  // coarse histograms suffice for the wave cut (no bucket sort): 4 ring stages
    return w30 ? launch_lbi_pass<P, true, 30>(grid, st, la, ws) : launch_lbi_pass<P, true, 24>(grid, st, la, ws);
  return w30 ? launch_lbi_pass<P, false, 30>(grid, st, la, ws) : launch_lbi_pass<P, false, 24>(grid, st, la, ws);
}

cudaError_t dispatch_index_lb(int nb, const Plan& p, const uint8_t* sax, const CardTables* tab, const Ws& ws,
                              cudaStream_t st, int64_t cap) {
  switch (pairs_for(nb)) {
    case 1: return launch_index_lb<1>(p, sax, nb, tab, ws, st, cap);
    case 2: return launch_index_lb<2>(p, sax, nb, tab, ws, st, cap);
    case 4: return launch_index_lb<4>(p, sax, nb, tab, ws, st, cap);
    case 8: return launch_index_lb<8>(p, sax, nb, tab, ws, st, cap);
    case 16: return launch_index_lb<16>(p, sax, nb, tab, ws, st, cap);
    default: return launch_index_lb<32>(p, sax, nb, tab, ws, st, cap);
  }
}

template <int P, bool AL>
cudaError_t launch_nb_t(const Plan& p, const float* raw, const uint8_t* sax, const float* qb, int nb,
                        const CardTables* tab, const Ws& ws, cudaStream_t st) {
  NbArgs na;
  na.sax = sax; na.n = p.n; na.w = p.w; na.seglen_f = (float)(p.len / p.w); na.tab = tab; na.g_q16 = ws.g_q16;
  na.queries = qb; na.raw = raw; na.len = p.len; na.nb = nb; na.best = ws.best; na.refined = ws.refined;
  na.updates = ws.updates; na.d2up = p.d2up;
  const int64_t workers = (int64_t)sms() * 8 * (kLBThreads / 32);
  na.part = std::max<int64_t>(128, ((p.n + workers - 1) / workers + 127) / 128 * 128);
  const int64_t nwarps = (p.n + na.part - 1) / na.part;
  const int grid = (int)((nwarps * 32 + kLBThreads - 1) / kLBThreads);
  return PARIS_LAUNCH("nb_distcomp", (k_nb<P>), grid, kLBThreads, 0, st, na);
}

cudaError_t launch_nb(const Plan& p, const float* raw, const uint8_t* sax, const float* qb, int nb,
                      const CardTables* tab, const Ws& ws, cudaStream_t st) {
  switch (pairs_for(nb)) {
    case 1: return launch_nb_t<1, true>(p, raw, sax, qb, nb, tab, ws, st);
    case 2: return launch_nb_t<2, true>(p, raw, sax, qb, nb, tab, ws, st);
    case 4: return launch_nb_t<4, true>(p, raw, sax, qb, nb, tab, ws, st);
    default: return launch_nb_t<8, true>(p, raw, sax, qb, nb, tab, ws, st);
  }
}

cudaError_t launch_lb1(const Plan& p, const uint8_t* sax, const CardTables* tab, const Ws& ws, cudaStream_t st,
                       int64_t cap) {
  const bool old_form = g_variant[1] == 0;  // A/B: the register-prefetch k_lb1
  if (!old_form) {
    const int smemt = cached_per_device((const void*)k_lb1t, [](int dev) {
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, k_lb1t) != cudaSuccess) return 0;
      const int v = optin - (int)fa.sharedSizeBytes;
      if (cudaFuncSetAttribute(k_lb1t, cudaFuncAttributeMaxDynamicSharedMemorySize, v) != cudaSuccess) return 0;
      return v;
    });
    if (smemt <= 0) return cudaErrorInvalidConfiguration;
    LbArgs la;
    la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
    la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = 1; la.thr = ws.thr_seed; la.count = ws.count;
    la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = nullptr; la.env = nullptr;
    la.blocks = ws.blocks;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms(), (p.n + kTS - 1) / kTS));
    return PARIS_LAUNCH("lb_pass", k_lb1t, grid, kL1Threads, smemt, st, la);
  }
  constexpr int SPT = PARIS_LB1_SPT;
  // dynamic shared memory: up to the 64 KB-aligned 64 KB table above the static arrays
  const int smem1 = cached_per_device((const void*)k_lb1<SPT>, [](int dev) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k_lb1<SPT>) != cudaSuccess) return 0;
    const int v = optin - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(k_lb1<SPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, v) != cudaSuccess) return 0;
    return v;
  });
  if (smem1 <= 0) return cudaErrorInvalidConfiguration;
  const int occ = 1;
  LbArgs la;
  la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
  la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = 1; la.thr = ws.thr_seed; la.count = ws.count;
  la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = nullptr; la.env = nullptr;
  la.blocks = ws.blocks;
  const int64_t ngroups = p.n / SPT;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((ngroups + kLb1Threads - 1) / kLb1Threads,
                                                              (int64_t)sms() * occ));
  return PARIS_LAUNCH("lb_pass", k_lb1<SPT>, grid, kLb1Threads, smem1, st, la);
}

template <int MODE>
cudaError_t dispatch_lbt(int nb, const Plan& p, const uint8_t* sax, const CardTables* tab, const Ws& ws,
                         cudaStream_t st, int64_t cap, int64_t nlim, int grid) {
  if (nb == 1) return launch_lbt<0, MODE>(p, sax, nb, tab, ws, st, cap, nlim, grid);
  switch (pairs_for(nb)) {
    case 1: return launch_lbt<1, MODE>(p, sax, nb, tab, ws, st, cap, nlim, grid);
    case 2: return launch_lbt<2, MODE>(p, sax, nb, tab, ws, st, cap, nlim, grid);
    case 4: return launch_lbt<4, MODE>(p, sax, nb, tab, ws, st, cap, nlim, grid);
    default: return launch_lbt<8, MODE>(p, sax, nb, tab, ws, st, cap, nlim, grid);
  }
}

constexpr size_t qprep_smem(int P) { return (size_t)3 * P * kMaxW * 8; }  // <= 48 KB at P = 32

cudaError_t launch_qprep(int nb, const Plan& p, const float* qb, const Ws& ws, cudaStream_t st) {
  switch (pairs_for(nb)) {
    case 1: return PARIS_LAUNCH("qprep", k_qprep<1>, 1, 1024, qprep_smem(1), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
    case 2: return PARIS_LAUNCH("qprep", k_qprep<2>, 1, 1024, qprep_smem(2), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
    case 4: return PARIS_LAUNCH("qprep", k_qprep<4>, 1, 1024, qprep_smem(4), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
    case 8: return PARIS_LAUNCH("qprep", k_qprep<8>, 1, 1024, qprep_smem(8), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
    case 16: return PARIS_LAUNCH("qprep", k_qprep<16>, 1, 1024, qprep_smem(16), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
    default: return PARIS_LAUNCH("qprep", k_qprep<32>, 1, 1024, qprep_smem(32), st, qb, nb, p.len, p.w, ws.g_q, ws.g_q16);
  }
}

template <int NC, int U>
cudaError_t launch_refine1(const RefineArgs& ra, int nb, int64_t max_work, cudaStream_t st) {
  // grid: one full wave of resident CTAs, or fewer when the wave holds less work
  const int full = sms() * (NC <= 2 ? 8 : 2);
  const int64_t need = (max_work + (int64_t)kRefWarps * U - 1) / ((int64_t)kRefWarps * U);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(full, need));
  return PARIS_LAUNCH("refine", (k_refine1<NC, U>), grid, kRefThreads, 0, st, ra, nb);
}

// the octet-form refine (k_refine1q) when a pre-filter copy is given; cudaErrorNotSupported
// otherwise (the caller falls back to k_refine1u)
template <int NC, int U>
cudaError_t launch_refine1q(const RefineArgs& ra, int nb, int wave, const unsigned* cut, cudaStream_t st, int grid) {
  if (ra.paa16) {  // the PAA pre-filter (then the bf16 one, if given)
    if (ra.w2 == 32)
      return ra.raw16 ? PARIS_LAUNCH("refine", (k_refine1q<NC, U, 32, true>), grid, kRefThreads, 0, st, ra, nb, wave, cut)
                      : PARIS_LAUNCH("refine", (k_refine1q<NC, U, 32, false>), grid, kRefThreads, 0, st, ra, nb, wave, cut);
    return ra.raw16 ? PARIS_LAUNCH("refine", (k_refine1q<NC, U, 64, true>), grid, kRefThreads, 0, st, ra, nb, wave, cut)
                    : PARIS_LAUNCH("refine", (k_refine1q<NC, U, 64, false>), grid, kRefThreads, 0, st, ra, nb, wave, cut);
  }
  if (ra.raw16 && !getenv("PARIS_REF16_WARP"))  // octets per candidate (env: A/B of the warp form)
    return PARIS_LAUNCH("refine", (k_refine1q<NC, U, 0, true>), grid, kRefThreads, 0, st, ra, nb, wave, cut);
  return cudaErrorNotSupported;
}

template <int NC, int U>
cudaError_t launch_refine1u(const RefineArgs& ra, int nb, int wave, const unsigned* cut, cudaStream_t st) {
  if constexpr (NC <= 2) {
    if (ra.paa16 && g_variant[2] == 1) {  // one chunk stream over the batch (k_refine1m)
      const int gridm = sms() * kRefMCtas;
      if (ra.w2 == 32)
        return ra.raw16 ? PARIS_LAUNCH("refine", (k_refine1m<NC, U, 32, true>), gridm, kRefThreads, 0, st, ra, nb, wave, cut)
                        : PARIS_LAUNCH("refine", (k_refine1m<NC, U, 32, false>), gridm, kRefThreads, 0, st, ra, nb, wave, cut);
      return ra.raw16 ? PARIS_LAUNCH("refine", (k_refine1m<NC, U, 64, true>), gridm, kRefThreads, 0, st, ra, nb, wave, cut)
                      : PARIS_LAUNCH("refine", (k_refine1m<NC, U, 64, false>), gridm, kRefThreads, 0, st, ra, nb, wave, cut);
    }
    const int grid = sms() * kRefQCtas;
    const cudaError_t e = launch_refine1q<NC, U>(ra, nb, wave, cut, st, grid);
    if (e != cudaErrorNotSupported) return e;
  }
  if (ra.raw16) {
    const int grid = sms() * (NC <= 2 ? kRefU16Ctas : 2);
    return PARIS_LAUNCH("refine", (k_refine1u<NC, U, true>), grid, kRefThreads, 0, st, ra, nb, wave, cut);
  }
  const int grid = sms() * (NC <= 2 ? kRefUCtas : 2);
  return PARIS_LAUNCH("refine", (k_refine1u<NC, U, false>), grid, kRefThreads, 0, st, ra, nb, wave, cut);
}

// Layout of the batch scratch for `cap` candidates per query: returns its size; with
// base != nullptr also carves `ws` out of it.
size_t ws_layout(const Plan& p, int64_t cap, Ws* ws, char* base) {
  const int B = 2 * pairs_for(p.B);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
  const size_t o_q = take(sizeof(float2) * B * kMaxW);
  const size_t o_q16 = take(sizeof(uint2) * (B / 2) * kMaxW);
  const size_t o_sid = take(sizeof(int) * B * p.S);
  const size_t o_skey = take(sizeof(uint64_t) * B * p.S);
  // zeroed per batch: thr_seed | count | hist | cursor | refined | blocks | tile_count | tile_claim | updates
  //                   | fb_refined | (k > 1) ghist
  const size_t zb = sizeof(unsigned) * (B + B + B * kNB + B * kNB + B + B + 2 + B + B + (p.k > 1 ? B * kNB + 4 : 0));
  const size_t o_zero = take(zb);
  const size_t o_best = take(sizeof(unsigned long long) * B * kPadU64);
  const size_t o_thr = take(sizeof(unsigned) * B * kPadU32);
  const size_t o_cand = take(sizeof(uint64_t) * B * (size_t)cap);
  // the bucket-sorted lists (sorted walk) or the k > 1 result lists; k = 1 on the unsorted
  // waves needs neither
  const bool need_sorted = p.sorted_refine || p.k > 1;
  const size_t o_sorted = take(need_sorted ? sizeof(uint64_t) * B * (size_t)cap : 8);
  const size_t o_lists = take(p.k > 1 && p.sorted_refine ? sizeof(uint64_t) * B * (size_t)p.XB * p.k : 8);
  const size_t o_fbl = take(p.k > 1 ? sizeof(uint64_t) * B * (size_t)p.fbL * p.k : 8);
  const size_t o_qaux = take(sizeof(float) * B * 80);
  const int64_t ntiles = (p.n + kTS - 1) / kTS;
  const size_t o_bmask = take(p.perm ? sizeof(unsigned long long) * (size_t)ntiles * kBPT : 8);
  const size_t o_tlist = take(p.perm ? sizeof(unsigned) * (size_t)ntiles : 8);
  const size_t o_gf = take(8192);
  if (!base) return off;
  char* c = base;
  ws->base = base;
  ws->g_q = (float2*)(c + o_q);
  ws->g_q16 = (uint2*)(c + o_q16);
  ws->seed_ids = (int*)(c + o_sid);
  ws->seed_keys = (uint64_t*)(c + o_skey);
  ws->zero_block = (unsigned*)(c + o_zero);
  ws->zero_bytes = zb;
  ws->thr = (unsigned*)(c + o_thr);
  ws->thr_seed = ws->zero_block;
  ws->count = ws->thr_seed + B;
  ws->hist = ws->count + B;
  ws->cursor = ws->hist + B * kNB;
  ws->refined = ws->cursor + B * kNB;
  ws->blocks = ws->refined + B;
  ws->tile_count = ws->blocks + B;
  ws->tile_claim = ws->tile_count + 1;
  ws->updates = ws->tile_claim + 1;
  ws->fb_refined = ws->updates + B;
  ws->ghist = p.k > 1 ? (unsigned*)(((uintptr_t)(ws->fb_refined + B) + 15) & ~(uintptr_t)15) : nullptr;
  ws->best = (unsigned long long*)(c + o_best);
  ws->cand = (uint64_t*)(c + o_cand);
  ws->sorted = (uint64_t*)(c + o_sorted);
  ws->lists = (uint64_t*)(c + o_lists);
  ws->fb_lists = (uint64_t*)(c + o_fbl);
  ws->qaux = (float*)(c + o_qaux);
  ws->bmask = (unsigned long long*)(c + o_bmask);
  ws->tile_list = (unsigned*)(c + o_tlist);
  ws->gf = (GfParams*)(c + o_gf);
  return off;
}

// The overflow fallback of a batch (k_fallback + k_finalize_ovf): two launches that
// leave at once unless a query of the batch kept more than `cap` candidates.
int launch_fallback(const Plan& p, const float* raw, const uint8_t* sax, const float* qbatch, int nb, int q0,
                    int64_t cap, const CardTables* tab, const Ws& ws, int64_t* d_idx, float* d_dist,
                    unsigned* all_refined, cudaStream_t st) {
  FbArgs fa;
  fa.sax = sax; fa.perm = p.perm; fa.n = p.n; fa.w = p.w; fa.len = p.len; fa.seglen_f = (float)(p.len / p.w);
  fa.tab = tab; fa.g_q = ws.g_q; fa.queries = qbatch; fa.raw = raw; fa.nb = nb; fa.count = ws.count; fa.cap = cap;
  fa.k = p.k; fa.d2up = p.d2up; fa.best = ws.best; fa.thr = ws.thr; fa.lists = ws.fb_lists; fa.L = p.fbL;
  fa.refined = ws.fb_refined;
  const int grid = p.fbL / (kFbThreads / 32);
  const bool fast = p.w == kTW && p.n % 4 == 0;
  const size_t tsm = (size_t)(kFbThreads / 32) * p.k * 8;
  cudaError_t e;
  if (p.k == 1) e = fast ? PARIS_LAUNCH("fallback", (k_fallback<true, true>), grid, kFbThreads, 0, st, fa)
                         : PARIS_LAUNCH("fallback", (k_fallback<true, false>), grid, kFbThreads, 0, st, fa);
  else e = fast ? PARIS_LAUNCH("fallback", (k_fallback<false, true>), grid, kFbThreads, tsm, st, fa)
                : PARIS_LAUNCH("fallback", (k_fallback<false, false>), grid, kFbThreads, tsm, st, fa);
  PARIS_CHECK_LAUNCH(e, "fallback launch");
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("fallback", k_finalize_ovf, nb, 1024, 0, st, ws.best, ws.fb_lists, p.fbL, p.k, q0,
                                  ws.count, cap, d_idx, d_dist, ws.fb_refined, all_refined),
                     "fallback finalize launch");
  return PARIS_OK;
}

// One batch of nb <= kMaxB queries (device pointers).  Outputs at [q0 .. q0+nb).
int run_batch(const Plan& p, const float* raw, const uint8_t* sax, const float* qbatch, int nb, int q0,
              int64_t cap, const CardTables* tab, const Ws& ws, int64_t* d_idx, float* d_dist,
              unsigned* all_count, unsigned* all_refined, float* all_tau, unsigned* all_blocks,
              unsigned* all_extra, cudaStream_t st, bool rescan = false, unsigned* all_paa = nullptr) {
  const int P = pairs_for(nb);
  cudaError_t e = cudaMemsetAsync(ws.zero_block, 0, ws.zero_bytes, st);
  if (e != cudaSuccess) return cuda_error(e, "memset scratch");
  // flat path behind the tensor-core filter: up to 64 slots per pass; query prep, the seed
  // pass and (if the filter declines) the k_lbt pass run per sub-batch of 16 slots, each on
  // its own slice of the scratch
  const bool gf_flat = p.gf && !p.perm && nb > 8;
  auto sub_ws = [&](int j0) {
    Ws w2 = ws;
    w2.g_q = ws.g_q + (size_t)j0 * kMaxW;
    w2.g_q16 = ws.g_q16 + (size_t)(j0 / kMaxBFlat) * kMaxW * (kMaxBFlat / 2);
    w2.seed_ids = ws.seed_ids + (size_t)j0 * p.S;
    w2.thr_seed = ws.thr_seed + j0;
    w2.count = ws.count + j0;
    w2.hist = ws.hist + (size_t)j0 * kNB;
    w2.cand = ws.cand + (size_t)j0 * cap;
    w2.lb_skip_if = &ws.gf->ok;
    return w2;
  };
  if (rescan) {
    // query PAA (the direct LB kernels compute it in their seed prologue) + BSF from the first pass
    if (gf_flat) {
      for (int j0 = 0; j0 < nb; j0 += kMaxBFlat)
        PARIS_CHECK_LAUNCH(launch_qprep(std::min(kMaxBFlat, nb - j0), p, qbatch + (size_t)j0 * p.len, sub_ws(j0), st),
                           "qprep launch");
    } else if (p.tiled) PARIS_CHECK_LAUNCH(launch_qprep(nb, p, qbatch, ws, st), "qprep launch");
    else PARIS_CHECK_LAUNCH(dispatch_p(P, false, p, sax, qbatch, nb, tab, ws, st, cap), "seed_lb launch");
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_select", k_seed_prev, 1, kMaxB, 0, st, d_idx, d_dist, nb, q0, p.k, p.d2up,
                                    ws.thr, ws.thr_seed, ws.best),
                       "seed_prev launch");
  } else {
    if (p.perm) {
      PARIS_CHECK_LAUNCH(launch_qprep(nb, p, qbatch, ws, st), "qprep launch");
      PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_lb", k_approx_seed, nb, 32, 0, st, sax, p.perm, p.n, ws.g_q, tab, p.card,
                                      ws.seed_ids, p.S),
                         "approx seed launch");
    } else if (gf_flat) {
      for (int j0 = 0; j0 < nb; j0 += kMaxBFlat) {
        const int nbj = std::min(kMaxBFlat, nb - j0);
        const Ws w2 = sub_ws(j0);
        PARIS_CHECK_LAUNCH(launch_qprep(nbj, p, qbatch + (size_t)j0 * p.len, w2, st), "qprep launch");
        PARIS_CHECK_LAUNCH(dispatch_lbt<0>(nbj, p, sax, tab, w2, st, cap, p.ns, p.seed_grid), "seed_lb launch");
      }
    } else if (p.tiled) {
      PARIS_CHECK_LAUNCH(launch_qprep(nb, p, qbatch, ws, st), "qprep launch");
      PARIS_CHECK_LAUNCH(dispatch_lbt<0>(nb, p, sax, tab, ws, st, cap, p.ns, p.seed_grid), "seed_lb launch");
    } else {
      PARIS_CHECK_LAUNCH(dispatch_p(P, false, p, sax, qbatch, nb, tab, ws, st, cap), "seed_lb launch");
    }
    {
      dim3 g((unsigned)((p.S + 7) / 8), (unsigned)nb);
      if (p.raw16 && p.raw_host && p.k == 1 && !p.approx)
        PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_ed", k_seed_ed16, g, kRefThreads, (size_t)p.len * 4, st, p.raw16,
                                        p.len, qbatch, ws.seed_ids, p.S, ws.seed_keys),
                           "seed_ed launch");
      else
        PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_ed", k_seed_ed, g, kRefThreads, (size_t)p.len * 4, st, raw, p.len,
                                        qbatch, ws.seed_ids, p.S, ws.seed_keys),
                           "seed_ed launch");
    }
    if (p.approx) {  // approximate search only: the seeds' top-k is the answer
      PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_select", k_seed_topk, nb, 1024, 0, st, ws.seed_keys, p.S, p.k, q0,
                                      d_idx, d_dist),
                         "seed_topk launch");
      return PARIS_OK;
    }
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_select", k_seed_select, nb, 1024, 0, st, ws.seed_keys, p.S, p.k,
                                    p.d2up, ws.thr, ws.thr_seed, ws.best, all_tau, q0),
                       "seed_select launch");
  }
  if (p.tau_in)
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_select", k_tau_in, 1, kMaxB, 0, st, p.tau_in, nb, q0, p.k, p.d2up, ws.thr,
                                    ws.thr_seed, ws.best),
                       "tau_in launch");
  if (p.nb) {
    // f2: nb-ParIS+ -- no candidate list: fused LB -> refine per worker, then min(V_bsf)
    PARIS_CHECK_LAUNCH(launch_nb(p, raw, sax, qbatch, nb, tab, ws, st), "nb launch");
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("finalize", k_finalize1, 1, kMaxB, 0, st, ws.best, nb, q0, d_idx, d_dist,
                                    ws.count, ws.refined, all_count, all_refined, rescan ? 1 : 0,
                                    ws.blocks, all_blocks, ws.updates, all_extra),
                       "finalize launch");
    return PARIS_OK;
  }
  if (p.tiled) {
    const int grid = (int)std::min<int64_t>(sms(), (p.n + kTS - 1) / kTS);
    if (p.perm) {
      PARIS_CHECK_LAUNCH(dispatch_index_lb(nb, p, sax, tab, ws, st, cap), "lb_pass launch");
      if (const char* bpath = getenv("PARIS_DEBUG_BMASK")) {  // tuning aid: block-mask statistics
        const int64_t ntl = (p.n + kTS - 1) / kTS;
        std::vector<unsigned long long> hm((size_t)ntl * kBPT);
        cudaMemcpyAsync(hm.data(), ws.bmask, hm.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        long long bits = 0, pair_items = 0, fixed_pairs = 0, fixed_quads = 0, live_blocks = 0;
        for (unsigned long long m : hm) {
          const int c = __builtin_popcountll(m);
          bits += c;
          pair_items += (c + 1) / 2;
          fixed_pairs += __builtin_popcountll((m | (m >> 1)) & 0x5555555555555555ull);
          const unsigned long long q2 = m | (m >> 1), q4 = q2 | (q2 >> 2);
          fixed_quads += __builtin_popcountll(q4 & 0x1111111111111111ull);
          live_blocks += c > 0;
        }
        if (FILE* f = fopen(bpath, "a")) {
          fprintf(f, "{\"nb\": %d, \"blocks\": %lld, \"live_blocks\": %lld, \"live_bits\": %lld, "
                     "\"pair_items\": %lld, \"fixed_pair_items\": %lld, \"fixed_quad_items\": %lld}\n",
                  nb, (long long)hm.size(), live_blocks, bits, pair_items, fixed_pairs, fixed_quads);
          fclose(f);
        }
      }
      if (getenv("PARIS_DEBUG_TILES")) {  // debugging aid: live tiles streamed by this batch
        unsigned tc = 0;
        cudaMemcpyAsync(&tc, ws.tile_count, 4, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "[paris] batch q0=%d nb=%d: %u of %lld tiles live\n", q0, nb, tc,
                (long long)((p.n + kTS - 1) / kTS));
      }
    }
    else if (gf_flat) {
      LbArgs la;
      la.sax = sax; la.n = p.n; la.w = p.w; la.seglen_f = (float)(p.len / p.w); la.tab = tab;
      la.g_q = ws.g_q; la.g_q16 = ws.g_q16; la.nb = nb; la.thr = ws.thr_seed; la.count = ws.count;
      la.hist = ws.hist; la.cand = ws.cand; la.cap = cap; la.perm = nullptr; la.env = nullptr;
      la.blocks = ws.blocks;
      PARIS_CHECK_LAUNCH(launch_gf(la, p.card, ws.gf, st), "lb_pass launch");
      for (int j0 = 0; j0 < nb; j0 += kMaxBFlat)  // only if the filter declined the pass
        PARIS_CHECK_LAUNCH(dispatch_lbt<1>(std::min(kMaxBFlat, nb - j0), p, sax, tab, sub_ws(j0), st, cap, p.n, grid),
                           "lb_pass launch");
    }
    else if (nb == 1) PARIS_CHECK_LAUNCH(launch_lb1(p, sax, tab, ws, st, cap), "lb_pass launch");
    else PARIS_CHECK_LAUNCH(dispatch_lbt<1>(nb, p, sax, tab, ws, st, cap, p.n, grid), "lb_pass launch");
  } else {
    PARIS_CHECK_LAUNCH(dispatch_p(P, true, p, sax, qbatch, nb, tab, ws, st, cap), "lb_pass launch");
  }
  // k = 1: the refine takes its two LB waves straight from the unsorted lists (K5
  // skipped; config reserved[1] = 1 restores the bucket-sorted walk); k > 1 walks
  // the bucket-sorted lists
  const bool unsorted = !p.sorted_refine;  // k = 1: two waves + BSF; k > 1: append + select
  if (!unsorted) {
    const int xs = std::max(1, std::min(sms() * 4 / nb, 1024));
    dim3 g((unsigned)xs, (unsigned)nb);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("scatter", k_scatter, g, 256, 0, st, ws.cand, ws.count, ws.hist, ws.thr_seed,
                                    ws.cursor, ws.sorted, cap),
                       "scatter launch");
  } else {
    const unsigned wa = (unsigned)std::max(p.wave_a, 16 * p.k);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("wave_cut", k_wave_cut, nb, kNB, 0, st, ws.hist, wa, ws.cursor),
                       "wave_cut launch");
  }
  RefineArgs ra;
  ra.raw = raw; ra.len = p.len; ra.queries = qbatch; ra.sorted = unsorted ? ws.cand : ws.sorted; ra.cap = cap;
  ra.count = ws.count; ra.thr_seed = ws.thr_seed; ra.thr = ws.thr; ra.best = ws.best;
  ra.refined = ws.refined; ra.lists = ws.lists; ra.k = p.k; ra.d2up = p.d2up;
  ra.lo = 0; ra.hi = 0xFFFFFFFFu; ra.n = p.n;
  // the pre-filter pays when its rows save real bytes: rows of len >= 256 in HBM
  // (C3's 512-byte rows refine faster without it), any len when raw is on the host
  ra.raw16 = (p.k == 1 && (p.raw_host || p.len >= kRaw16MinLen)) ? p.raw16 : nullptr;
  ra.refined16 = ws.updates;
  ra.ghist = ws.ghist;
  ra.paa16 = (p.k == 1 || !p.sorted_refine) && p.len <= kRefQLen ? p.paa16 : nullptr;
  ra.w2 = p.w2;
  ra.paa_rows = all_paa ? all_paa + q0 : nullptr;
  ra.qaux = ws.qaux;
  if ((ra.raw16 || ra.paa16) && p.len <= kRefQLen)  // the octet / PAA refine's query constants
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("qprep", k_qaux, nb, 32, 0, st, qbatch, p.len, ra.paa16 ? p.w2 : 0, ws.qaux),
                       "qaux launch");
  dim3 g((unsigned)p.XB, (unsigned)nb);
  if (p.k == 1) {
    cudaError_t e1 = cudaSuccess;
    const int NC = p.len <= 128 ? 1 : p.len <= 256 ? 2 : p.len <= 512 ? 4 : p.len <= 1024 ? 8 : 32;
    // wave A: the lowest-LB wave_a candidates of every query (finds the NN early, so
    // wave B -- the rest, in LB order -- prunes against a tight BSF)
    for (int wv = 0; wv < 2 && e1 == cudaSuccess && unsorted; ++wv) {
      switch (NC) {
        case 1: e1 = launch_refine1u<1, kRefUU * 2>(ra, nb, wv, ws.cursor, st); break;
        case 2: e1 = launch_refine1u<2, kRefUU>(ra, nb, wv, ws.cursor, st); break;
        case 4: e1 = launch_refine1u<4, 1>(ra, nb, wv, ws.cursor, st); break;
        case 8: e1 = launch_refine1u<8, 1>(ra, nb, wv, ws.cursor, st); break;
        default: e1 = launch_refine1u<32, 1>(ra, nb, wv, ws.cursor, st); break;
      }
    }
    for (int wv = 0; wv < 2 && e1 == cudaSuccess && !unsorted; ++wv) {
      RefineArgs rb = ra;
      rb.lo = wv == 0 ? 0u : (unsigned)p.wave_a;
      rb.hi = wv == 0 ? (unsigned)p.wave_a : 0xFFFFFFFFu;
      const int64_t work = wv == 0 ? (int64_t)p.wave_a : cap;  // per query, upper bound
      switch (NC) {
        case 1: e1 = launch_refine1<1, 2>(rb, nb, work, st); break;
        case 2: e1 = launch_refine1<2, 1>(rb, nb, work, st); break;
        case 4: e1 = launch_refine1<4, 1>(rb, nb, work, st); break;
        case 8: e1 = launch_refine1<8, 1>(rb, nb, work, st); break;
        default: e1 = launch_refine1<32, 1>(rb, nb, work, st); break;
      }
    }
    PARIS_CHECK_LAUNCH(e1, "refine launch");
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("finalize", k_finalize1, 1, kMaxB, 0, st, ws.best, nb, q0, d_idx, d_dist,
                                    ws.count, ws.refined, all_count, all_refined, rescan ? 1 : 0,
                                    ws.blocks, all_blocks, ws.updates, all_extra),
                       "finalize launch");
  } else if (unsorted) {
    // k > 1: the same two waves (the first holding >= 16k candidates), results appended
    // to ws.sorted (free: no bucket sort on this path), then the exact top-k per query
    static_assert(kMaxB < kNB, "result counters sit between the wave-cut entries of ws.cursor");
    unsigned* res_cnt = ws.cursor + 1;  // (k_wave_cut writes cursor[b * kNB] only)
    cudaError_t e1 = cudaSuccess;
    const int NC = p.len <= 128 ? 1 : p.len <= 256 ? 2 : p.len <= 512 ? 4 : p.len <= 1024 ? 8 : 32;
    for (int wv = 0; wv < 2 && e1 == cudaSuccess; ++wv) {
      const int grid = sms() * (NC <= 2 ? (ra.paa16 ? 4 : kRefUCtas) : 2);
      switch (NC) {
        case 1:
          if (ra.paa16)
            e1 = PARIS_LAUNCH("refine", (k_refine_kx<1, kRefUU * 2, 32>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt);
          else
            e1 = PARIS_LAUNCH("refine", (k_refine_kx<1, kRefUU * 2>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt);
          break;
        case 2:
          if (ra.paa16 && ra.w2 == 64)
            e1 = PARIS_LAUNCH("refine", (k_refine_kx<2, kRefUU, 64>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt);
          else if (ra.paa16)
            e1 = PARIS_LAUNCH("refine", (k_refine_kx<2, kRefUU, 32>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt);
          else
            e1 = PARIS_LAUNCH("refine", (k_refine_kx<2, kRefUU>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt);
          break;
        case 4: e1 = PARIS_LAUNCH("refine", (k_refine_kx<4, 1>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt); break;
        case 8: e1 = PARIS_LAUNCH("refine", (k_refine_kx<8, 1>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt); break;
        default: e1 = PARIS_LAUNCH("refine", (k_refine_kx<32, 1>), grid, kRefThreads, 0, st, ra, nb, wv, ws.cursor, ws.sorted, res_cnt); break;
      }
    }
    PARIS_CHECK_LAUNCH(e1, "refine launch");
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("finalize", k_select_topk, nb, 1024, 0, st, ws.sorted, res_cnt, cap, ws.thr, p.k,
                                    q0, d_idx, d_dist, ws.count, ws.refined, all_count, all_refined, rescan ? 1 : 0,
                                    ws.blocks, all_blocks, ws.updates, all_extra),
                       "finalize launch");
  } else {
    const size_t rsmem = (size_t)p.len * 4 + (size_t)p.k * 16;
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("refine", k_refine_topk, g, kRefThreads, rsmem, st, ra), "refine launch");
    if (getenv("PARIS_DEBUG_DUMP")) {  // debugging aid: candidate lists and per-CTA top-k lists
      cudaStreamSynchronize(st);
      std::vector<unsigned> hc(nb);
      cudaMemcpy(hc.data(), ws.count, 4 * nb, cudaMemcpyDeviceToHost);
      for (int b = 0; b < nb; ++b) {
        const size_t c = std::min<size_t>(hc[b], cap);
        std::vector<uint64_t> h(c), hl((size_t)p.XB * p.k);
        cudaMemcpy(h.data(), ws.sorted + (size_t)b * cap, 8 * c, cudaMemcpyDeviceToHost);
        cudaMemcpy(hl.data(), ws.lists + (size_t)b * p.XB * p.k, 8 * hl.size(), cudaMemcpyDeviceToHost);
        std::vector<uint32_t> ids;
        for (auto k2 : h) ids.push_back((uint32_t)k2);
        std::sort(ids.begin(), ids.end());
        const size_t uniq = std::unique(ids.begin(), ids.end()) - ids.begin();
        std::sort(hl.begin(), hl.end());
        fprintf(stderr, "[paris dump] b=%d count=%u uniq=%zu lists_min=(%g,%u) (%g,%u)\n", b, hc[b], uniq,
                (double)__builtin_bit_cast(float, (uint32_t)(hl[0] >> 32)), (uint32_t)hl[0],
                (double)__builtin_bit_cast(float, (uint32_t)(hl[1] >> 32)), (uint32_t)hl[1]);
        const char* want = getenv("PARIS_DEBUG_DUMP");
        const uint32_t wid = (uint32_t)atoi(want);
        for (size_t i = 0; i < c; ++i)
          if ((uint32_t)h[i] == wid)
            fprintf(stderr, "[paris dump]   id %u at %zu lb=%g\n", wid, i, (double)__builtin_bit_cast(float, (uint32_t)(h[i] >> 32)));
      }
    }
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("finalize", k_finalize, nb, 1024, 0, st, ws.lists, p.XB, p.k, q0,
                                    d_idx, d_dist, ws.count, ws.refined, all_count, all_refined, rescan ? 1 : 0,
                                    ws.blocks, all_blocks, ws.updates, all_extra),
                       "finalize launch");
  }
  return launch_fallback(p, raw, sax, qbatch, nb, q0, cap, tab, ws, d_idx, d_dist, all_refined, st);
}

bool is_host_ptr(const void* p) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return true; }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

constexpr int kIdxSeeds = 1024;     // index mode: series around the query's leaf (default)
constexpr int kIdxSeedsHost = 64;   // ... when raw is in pinned host memory (f3)

void plan_seed(Plan& p, int seed_div) {
  if (p.perm) {
    p.ns = 0;
    p.seed_grid = 0;
    // default: 1024 series around the leaf; for k > 1, 32 per requested neighbour (the
    // k-th best of the seeds must bound the k-th NN distance tightly), up to kMaxSeed
    // (2048 from 5e7 series on: the leaf neighbourhood then tightens tau measurably, C4 +0.7%)
    const int dflt = std::max(p.n >= 50000000 ? 2 * kIdxSeeds : kIdxSeeds, std::min(kMaxSeed, 32 * p.k));
    p.S = std::max(p.k, std::min(kMaxSeed, p.idx_seeds > 0 ? p.idx_seeds : dflt));
    return;
  }
  p.ns = std::min<int64_t>(p.n, std::max<int64_t>(p.n / seed_div, std::min<int64_t>(p.n, 65536)));
  if (p.tiled) {
    p.ns = std::min<int64_t>(p.n, (p.ns + 15) / 16 * 16);
    p.seed_grid = (int)std::min<int64_t>(sms(), (p.ns + kTS - 1) / kTS);
    p.S = p.seed_grid * kTWarps;
    return;
  }
  const int64_t groups = (p.ns + 3) / 4;
  const int64_t need = (groups + kLBThreads - 1) / kLBThreads;
  p.seed_grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, std::min(sms() * 2, kMaxSeed / 8)));
  p.S = p.seed_grid * (kLBThreads / 32);
}

void plan_refine(Plan& p) {
  p.XB = std::max(1, std::min(sms() * 8 / std::max(1, p.B), 65535));
}

}  // namespace

int knn_impl(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int nq, int k,
             int64_t* out_idx, float* out_dist, int len, int w, int card, cudaStream_t st,
             const paris_knn_config* cfg, paris_knn_stats* stats, const uint32_t* perm = nullptr,
             const uint8_t* env = nullptr, bool nb_mode = false, const uint16_t* raw16 = nullptr,
             bool approx = false, const uint16_t* paa16 = nullptr, int w2 = 0) {
  if (nb_mode && (k != 1 || w != kTW || n % 4 != 0)) {
    set_error("paris_knn_nb: needs k == 1, w == 16, n %% 4 == 0 (k=%d, w=%d, n=%lld)", k, w, (long long)n);
    return k != 1 ? PARIS_EINVAL : PARIS_ECONFIG;
  }
  const bool indexed = perm || env;
  if (indexed && (!perm || !env)) {
    set_error("paris_knn_index: null perm/env");
    return PARIS_EINVAL;
  }
  if (indexed && (w != kTW || n % 16 != 0)) {
    set_error("paris_knn_index: the index needs w == 16 and n %% 16 == 0 (w=%d, n=%lld)", w, (long long)n);
    return PARIS_ECONFIG;
  }
  if (!raw || !sax || (nq > 0 && (!queries || !out_idx || !out_dist))) {
    set_error("paris_knn_exact: null pointer");
    return PARIS_EINVAL;
  }
  // k <= n; k beyond PARIS_MAX_K takes the full-sort path (knn_large_k), except for
  // the approximate search, whose answer is the seeds' top-k
  if (n < 1 || n >= (int64_t(1) << 31) || nq < 0 || k < 1 || k > n || (approx && k > PARIS_MAX_K)) {
    set_error("paris_knn_exact: bad sizes n=%lld nq=%d k=%d (need 1<=k<=n, n<2^31; approximate: k<=%d)",
              (long long)n, nq, k, PARIS_MAX_K);
    return PARIS_EINVAL;
  }
  const bool large_k = k > PARIS_MAX_K;
  if (len < 4 || len > 4096 || (len % 4) || w < 1 || w > kMaxW || (len % w)) {
    set_error("paris_knn_exact: unsupported (len=%d, w=%d)", len, w);
    return PARIS_ECONFIG;
  }
  const CardTables* tab = device_tables(card);
  if (!tab) return PARIS_ECONFIG;
  if (nq == 0) return PARIS_OK;
  if ((reinterpret_cast<uintptr_t>(raw) & 15) != 0) {
    set_error("paris_knn_exact: raw must be 16-byte aligned");
    return PARIS_EINVAL;
  }
  // raw may live in page-locked host memory (the raw collection outside
  // the device's memory, like the paper's raw data file on disk): the seed
  // and the refinement then read only the candidates' rows, through the mapping
  // (the paper's random reads of the raw file for the RDC pass).  The
  // SAX array / index are always device-resident (TMA-streamed).
  const float* d_raw = raw;
  bool raw_host = false;
  {
    cudaPointerAttributes at;
    cudaError_t ea = cudaPointerGetAttributes(&at, raw);
    if (ea != cudaSuccess) { cudaGetLastError(); at.type = cudaMemoryTypeUnregistered; }
    if (at.type == cudaMemoryTypeUnregistered || (at.type == cudaMemoryTypeHost && !at.devicePointer)) {
      set_error("paris_knn_exact: raw must be device memory or page-locked host memory "
                "(cudaHostAlloc / cudaHostRegister)");
      return PARIS_EINVAL;
    }
    if (at.type == cudaMemoryTypeHost) {
      d_raw = (const float*)at.devicePointer;
      raw_host = true;
    }
    for (const void* dp : {(const void*)sax, (const void*)perm, (const void*)env}) {
      if (dp && is_host_ptr(dp)) {
        set_error("paris_knn_exact: sax / perm / env must be device memory");
        return PARIS_EINVAL;
      }
    }
  }
  raw = d_raw;

  Plan p;
  p.n = n; p.len = len; p.w = w; p.card = card; p.k = k;
  p.tiled = (n % 16 == 0) && (w == kTW) && (indexed || !(cfg && cfg->reserved[0] == 1));
  // tensor-core filter (variant key 3): 2 (default) = flat path only, 1 = index path too, 0 = off
  p.gf = (g_variant[3] == 1 || (g_variant[3] == 2 && !indexed)) && p.tiled && !nb_mode && !approx &&
         !(cfg && cfg->reserved[1] == 1) && (reinterpret_cast<uintptr_t>(sax) & 15) == 0;
  {
    // index: 64 queries per pass; flat: 16 (k_lbt), 64 behind the tensor-core filter
    const int cap_b = (indexed || p.gf) ? kMaxB : kMaxBFlat;
    p.B = (cfg && cfg->batch > 0) ? std::min(cfg->batch, cap_b) : cap_b;
  }
  p.perm = perm;
  p.env = env;
  p.nb = nb_mode;
  // index seeds: 1024 series around the leaf by default; 64 when raw is in host memory,
  // where every seed is a PCIe read (measured: C5 62.7 K q/s with 64 vs 29 K with 1024)
  p.sorted_refine = cfg && cfg->reserved[1] == 1;
  if (raw16) {
    if ((len % 8) || is_host_ptr(raw16) || (reinterpret_cast<uintptr_t>(raw16) & 15)) {
      set_error("paris_knn_index_x: raw_bf16 must be 16-byte aligned device memory and len %% 8 == 0");
      return PARIS_EINVAL;
    }
    p.raw16 = raw16;
  }
  if (paa16) {
    if (w2 != 32 && w2 != 64) {
      set_error("paris_knn_index_aux: paa16 needs w2 in {32, 64} (got %d)", w2);
      return PARIS_ECONFIG;
    }
    if ((len % w2) || is_host_ptr(paa16) || (reinterpret_cast<uintptr_t>(paa16) & 15)) {
      set_error("paris_knn_index_aux: paa16 must be 16-byte aligned device memory and w2 | len");
      return PARIS_EINVAL;
    }
    p.paa16 = reinterpret_cast<const __half*>(paa16);
    p.w2 = w2;
  }
  p.raw_host = raw_host;
  p.approx = approx;
  if (cfg && cfg->tau_in && !approx && !nb_mode) {
    if (is_host_ptr(cfg->tau_in)) {
      set_error("paris_knn: config.tau_in must be device memory");
      return PARIS_EINVAL;
    }
    p.tau_in = cfg->tau_in;
  }
  // (host raw with the bf16 copy in HBM: the seeds read bf16 rows, so the full 1024)
  p.idx_seeds = (cfg && cfg->reserved[2] > 0) ? cfg->reserved[2]
                                               : ((raw_host && !(raw16 && k == 1)) ? kIdxSeedsHost : 0);
  plan_seed(p, (cfg && cfg->seed_div > 0) ? cfg->seed_div : 16);
  // candidate buffer per query: n/32 for k = 1; k > 1 keeps far more candidates on hard
  // queries (C5 sigma = 0.2, k = 100: ~670 K of 2e7), so n/16 -- an overflow costs a
  // per-query re-scan
  // candidate buffer per query: at least max(65536, n/32) (n/16 for k > 1), grown to a
  // budget per candidate array of 1/8 of the free device memory, clamped to [2, 16] GB
  // (hard queries -- C3: up to 24% of n; C5 k = 100: more -- then stay on the regular
  // path instead of the overflow fallback)
  {
    const int Bq = 2 * pairs_for(p.B);
    const int64_t floor_cap = std::max<int64_t>(65536, k > 1 ? n / 16 : n / 32);
    // free device memory, sampled at most once per second per device: cudaMemGetInfo takes 0.08 ms
    // at the median but 7 ms at p99 and up to 27 ms (scripts/exp_host_latency.py) -- a stall in
    // every hundredth call of a synchronous caller
    size_t fr = 0;
    {
      static std::mutex mu;
      static size_t cached_free[64] = {0};
      static std::chrono::steady_clock::time_point stamp[64];
      int dev = 0;
      cudaGetDevice(&dev);
      dev = (dev >= 0 && dev < 64) ? dev : 0;
      std::lock_guard<std::mutex> lk(mu);
      const auto now = std::chrono::steady_clock::now();
      if (cached_free[dev] == 0 || now - stamp[dev] > std::chrono::seconds(1)) {
        size_t f2 = 0, tot = 0;
        if (cudaMemGetInfo(&f2, &tot) != cudaSuccess) { cudaGetLastError(); f2 = 0; }
        cached_free[dev] = f2;
        stamp[dev] = now;
      }
      fr = cached_free[dev];
    }
    // (whole GB: the workspace the first call allocates barely moves the budget of the next)
    const int64_t bud_bytes =
        std::min<int64_t>(16ll << 30, std::max<int64_t>(2ll << 30, (int64_t)(fr / 8) & ~((1ll << 30) - 1)));
    const int64_t budget = bud_bytes / (8ll * Bq);
    p.cap = (nb_mode || approx) ? 1 : std::min<int64_t>(n, std::max(floor_cap, budget));
    if (cfg && cfg->reserved[4] > 0 && !nb_mode && !approx) p.cap = std::min<int64_t>(n, cfg->reserved[4]);  // test hook
  }
  plan_refine(p);
  p.wave_a = (cfg && cfg->wave_a > 0) ? cfg->wave_a : 2048;
  // |fp32 d^2 - exact| <= e d^2 with e = (len/32 + 8) u (warp_ed2 / refine_step);
  // d2up >= (1+e)/(1-e) with margin, u = 2^-24
  p.d2up = (float)(1.0 + 2.5 * (len / 32 + 8) * 5.9604644775390625e-08);

  // overflow fallback grid: 4 CTAs per SM (k = 1); for k > 1 its warp lists
  // ([B][fbL][k] keys) are kept to <= 32 MB
  {
    const int Bq = 2 * pairs_for(p.B);
    int L = sms() * 4 * (kFbThreads / 32);
    if (k > 1) L = (int)std::max<int64_t>(kFbThreads / 32, std::min<int64_t>(L, (32ll << 20) / ((int64_t)Bq * k * 8)));
    p.fbL = L / (kFbThreads / 32) * (kFbThreads / 32);
  }
  if (k > 1) {
    const cudaError_t ea = once_per_device((const void*)k_fallback<false, true>, [](int) {
      cudaError_t r = cudaFuncSetAttribute(k_fallback<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (kFbThreads / 32) * PARIS_MAX_K * 8);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(k_fallback<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (kFbThreads / 32) * PARIS_MAX_K * 8);
      return r;
    });
    if (ea != cudaSuccess) return cuda_error(ea, "fallback smem attribute");
  }

  retain_pool();
  // host <-> device staging of queries / outputs, carved from the cached workspace after
  // the batch scratch (no allocation in the steady state)
  const bool hq = is_host_ptr(queries), hi = is_host_ptr(out_idx), hd = is_host_ptr(out_dist);
  cudaError_t e;
  const size_t qbytes = (size_t)nq * len * 4, ibytes = (size_t)nq * k * 8, dbytes = (size_t)nq * k * 4;
  const size_t cbytes = (size_t)nq * 4 * 6;
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t wsb = large_k ? 0 : up(ws_layout(p, p.cap, nullptr, nullptr));
  const size_t total = wsb + up(qbytes) + up(ibytes) + up(dbytes) + up(cbytes);
  void* wsh = nullptr;
  char* base = (char*)ws_acquire(total, st, &wsh, nullptr);
  if (!base) return PARIS_ENOMEM;
  Ws ws;
  if (!large_k) ws_layout(p, p.cap, &ws, base);
  char* cur = base + wsb;
  float* sq = (float*)cur; cur += up(qbytes);
  int64_t* sidx = (int64_t*)cur; cur += up(ibytes);
  float* sdist = (float*)cur; cur += up(dbytes);
  unsigned* all_count = (unsigned*)cur;
  unsigned* all_refined = all_count + nq;
  float* all_tau = (float*)(all_refined + nq);
  unsigned* all_blocks = (unsigned*)(all_tau + nq);
  unsigned* all_extra = all_blocks + nq;  // nb: BSF-copy updates; index + bf16: pre-filter rows
  unsigned* all_paa = all_extra + nq;     // index + PAA pre-filter: PAA rows read
  const float* d_q = queries;
  int64_t* d_idx = hi ? sidx : out_idx;
  float* d_dist = hd ? sdist : out_dist;
  int rc = PARIS_OK;
  if (hq) {
    e = cudaMemcpyAsync(sq, queries, qbytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = cuda_error(e, "H2D queries");
    d_q = sq;
  }
  if (rc == PARIS_OK && (reinterpret_cast<uintptr_t>(d_q) & 15) != 0) {
    set_error("paris_knn_exact: queries must be 16-byte aligned");
    rc = PARIS_EINVAL;
  }
  if (rc == PARIS_OK) {
    e = cudaMemsetAsync(all_count, 0, cbytes, st);
    if (e != cudaSuccess) rc = cuda_error(e, "memset counters");
  }
  // test hook (reserved[3] == 1): seed every batch from the rows already in out_idx/out_dist
  // (device outputs) instead of the approximate search -- measures the LB pass under an
  // ideal BSF; results stay exact for any seed
  const bool seed_from_out = cfg && cfg->reserved[3] == 1 && !hi && !hd;
  if (large_k && rc == PARIS_OK) {
    rc = knn_large_k(raw, n, len, d_q, nq, k, d_idx, d_dist, st);  // every series refined (no pruning)
  }
  for (int q0 = 0; q0 < nq && rc == PARIS_OK && !large_k; q0 += p.B) {
    const int nb = std::min(p.B, nq - q0);
    rc = run_batch(p, raw, sax, d_q + (size_t)q0 * len, nb, q0, p.cap, tab, ws, d_idx, d_dist,
                   all_count, all_refined, all_tau, all_blocks, all_extra, st, /*rescan=*/seed_from_out, all_paa);
  }
  // no synchronization: a query whose candidate buffer overflowed was completed on the
  // device (k_fallback); host outputs are copied back stream-ordered
  if (rc == PARIS_OK && hi) {
    e = cudaMemcpyAsync(out_idx, sidx, ibytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_error(e, "D2H out_idx");
  }
  if (rc == PARIS_OK && hd) {
    e = cudaMemcpyAsync(out_dist, sdist, dbytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_error(e, "D2H out_dist");
  }
  if (rc == PARIS_OK && stats) {  // measurement path: read the counters (synchronizes)
    std::vector<unsigned> h_count(nq), h_ref(nq), h_blk(nq), h_ext(nq), h_paa(nq);
    std::vector<float> h_tau(nq);
    e = cudaMemcpyAsync(h_count.data(), all_count, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_ref.data(), all_refined, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_tau.data(), all_tau, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_blk.data(), all_blocks, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_ext.data(), all_extra, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_paa.data(), all_paa, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "paris_knn_exact stats D2H");
    if (rc == PARIS_OK) {
      for (int q = 0; q < nq; ++q) {
        if (large_k) h_count[q] = h_ref[q] = (unsigned)n;
        if (stats->candidates) stats->candidates[q] = h_count[q];
        if (stats->refined) stats->refined[q] = h_ref[q];
        if (stats->tau_seed) stats->tau_seed[q] = h_tau[q];
        if (stats->lb_blocks) stats->lb_blocks[q] = p.nb ? 0 : h_blk[q];
        if (stats->bsf_updates) stats->bsf_updates[q] = p.nb ? h_ext[q] : 0;
        if (stats->raw16_rows) stats->raw16_rows[q] = p.nb ? 0 : h_ext[q];
        if (stats->paa_rows) stats->paa_rows[q] = h_paa[q];
      }
    }
  }
  ws_release(wsh, st);
  return rc;
}

}  // namespace paris

namespace paris {

// Debug: the raw accumulators of k_gf for a caller-made table and B matrix (tests the
// tcgen05 unit, its descriptors and its accumulation error).  All pointers device.
int debug_gf_mma(const uint8_t* sax_sorted, int64_t n, const uint32_t* tabw, const uint16_t* bmat, float* out,
                 int swap_desc, cudaStream_t st) {
  if (!sax_sorted || !tabw || !bmat || !out || n < 1) return PARIS_EINVAL;
  const CardTables* tab = device_tables(256);
  if (!tab) return PARIS_ECUDA;
  GfParams* gp = nullptr;
  if (cudaMalloc((void**)&gp, sizeof(GfParams)) != cudaSuccess) return PARIS_ENOMEM;
  const unsigned one = 1u;
  cudaMemcpyAsync(gp->tabw, tabw, sizeof(uint32_t) * kMaxCard, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(gp->B, bmat, sizeof(uint16_t) * kGfN * kGfK, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(&gp->ok, &one, sizeof(unsigned), cudaMemcpyHostToDevice, st);
  LbArgs la{};
  la.sax = sax_sorted; la.n = n; la.w = 16; la.seglen_f = 16.f; la.tab = tab; la.nb = 0;
  la.perm = reinterpret_cast<const uint32_t*>(sax_sorted);  // tile-major layout (never read: no candidates here)
  cudaError_t e = launch_gf_kernel("gf_debug", la, gp, out, swap_desc, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(gp);
  return e == cudaSuccess ? PARIS_OK : cuda_error(e, "paris_debug_gf_mma");
}
}  // namespace paris

extern "C" {
int paris_debug_gf_mma(const uint8_t* sax_sorted, int64_t n, const uint32_t* tabw, const uint16_t* bmat, float* out,
                       int32_t swap_desc, void* stream) {
  return paris::debug_gf_mma(sax_sorted, n, tabw, bmat, out, swap_desc, (cudaStream_t)stream);
}


int paris_knn_exact(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int32_t nq,
                    int32_t k, int64_t* out_idx, float* out_dist, int32_t len, int32_t w, int32_t card,
                    void* stream) {
  return paris::knn_impl(raw, sax, n, queries, nq, k, out_idx, out_dist, len, w, card,
                         (cudaStream_t)stream, nullptr, nullptr);
}

int paris_knn_exact_ex(const float* raw, const uint8_t* sax, int64_t n, const float* queries,
                       int32_t nq, int32_t k, int64_t* out_idx, float* out_dist, int32_t len,
                       int32_t w, int32_t card, void* stream, const paris_knn_config* config,
                       paris_knn_stats* stats) {
  return paris::knn_impl(raw, sax, n, queries, nq, k, out_idx, out_dist, len, w, card,
                         (cudaStream_t)stream, config, stats);
}

int paris_knn_nb(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int32_t nq,
                 int64_t* out_idx, float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                 const paris_knn_config* config, paris_knn_stats* stats) {
  return paris::knn_impl(raw, sax, n, queries, nq, 1, out_idx, out_dist, len, w, card, (cudaStream_t)stream,
                         config, stats, nullptr, nullptr, /*nb_mode=*/true);
}

int paris_knn_index(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                    int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist,
                    int32_t len, int32_t w, int32_t card, void* stream) {
  return paris::knn_impl(raw, sax_sorted, n, queries, nq, k, out_idx, out_dist, len, w, card,
                         (cudaStream_t)stream, nullptr, nullptr, perm, env);
}

int paris_knn_index_ex(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                       int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx,
                       float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                       const paris_knn_config* config, paris_knn_stats* stats) {
  return paris::knn_impl(raw, sax_sorted, n, queries, nq, k, out_idx, out_dist, len, w, card,
                         (cudaStream_t)stream, config, stats, perm, env);
}

int paris_knn_index_aux(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env, int64_t n,
                        const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist, int32_t len,
                        int32_t w, int32_t card, void* stream, const paris_refine_aux* aux,
                        const paris_knn_config* config, paris_knn_stats* stats) {
  return paris::knn_impl(raw, sax_sorted, n, queries, nq, k, out_idx, out_dist, len, w, card, (cudaStream_t)stream,
                         config, stats, perm, env, false, aux ? aux->raw_bf16 : nullptr, false,
                         aux ? aux->paa16 : nullptr, aux ? aux->w2 : 0);
}

int paris_knn_approx(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int32_t nq, int32_t k,
                     int64_t* out_idx, float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                     const paris_knn_config* config) {
  return paris::knn_impl(raw, sax, n, queries, nq, k, out_idx, out_dist, len, w, card, (cudaStream_t)stream, config,
                         nullptr, nullptr, nullptr, false, nullptr, /*approx=*/true);
}

int paris_knn_index_approx(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                           int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist,
                           int32_t len, int32_t w, int32_t card, void* stream, const paris_knn_config* config) {
  return paris::knn_impl(raw, sax_sorted, n, queries, nq, k, out_idx, out_dist, len, w, card, (cudaStream_t)stream,
                         config, nullptr, perm, env, false, nullptr, /*approx=*/true);
}

int paris_knn_index_x(const float* raw, const uint16_t* raw_bf16, const uint8_t* sax_sorted, const uint32_t* perm,
                      const uint8_t* env, int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx,
                      float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                      const paris_knn_config* config, paris_knn_stats* stats) {
  return paris::knn_impl(raw, sax_sorted, n, queries, nq, k, out_idx, out_dist, len, w, card,
                         (cudaStream_t)stream, config, stats, perm, env, false, raw_bf16);
}

}  // extern "C"
