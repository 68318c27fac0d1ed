// K2-K7 -- paris_knn_exact: ParIS+ ExactSearch (Alg9) on one B200.
//
//   k_seed        (K2+K3a) query PAA (fp64) -> outward-rounded fp32 pair per
//                 segment; lower bound over a SAX sample, per-warp best (LB,id)
//                 = the approximate-search analog (reading R8)
//   k_seed_ed     (K3b) true distance of each seed series
//   k_seed_select (K3c) tau_seed^2 = k-th best seed d^2, rounded up
//   k_lb          (K4) LBC pass (Alg10): MINDIST_PAA_iSAX
//                  of every word for B queries at once; candidates
//                 (LB^2 bits << 32 | id) compacted per query + LB histogram
//   k_scatter     (K5) candidates bucket-sorted by LB (256 bins over [0, tau^2])
//   k_refine      (K6) RDC pass (Alg11): warp per candidate in LB
//                 order, LB re-checked against the live BSF, true ED
//                 with early abandoning, BSF = k-th best shared via atomicMin
//   k_finalize    (K7) merge per-CTA top-k lists -> ascending (d^2, id), sqrt
//
// Exactness: every LB is a rigorous lower bound of the
// exact MINDIST (outward-rounded region bounds, round-down arithmetic), every
// pruning threshold a rigorous upper bound of a real series' distance (fp32 d^2
// scaled by 1 + 2^-19 > its summation error bound), so pruning never drops a
// series that belongs in the exact answer; ranking among refined series uses
// fp32 d^2 with the lower id breaking exact ties.
#include "runtime.cuh"

#include <algorithm>
#include <vector>

namespace paris {

int summarize_impl(const float*, int64_t, int, int, int, uint8_t*, cudaStream_t);

namespace {

constexpr int kMaxW = 64;
constexpr int kNB = 256;            // LB histogram bins per query
constexpr int kMaxB = 8;            // queries per SAX pass
constexpr int kLBThreads = 256;
constexpr int kRefThreads = 256;
constexpr int kRefAThreads = 1024;
constexpr int kSortP = 4096;        // finalize / seed-select sort buffer
constexpr int kMaxSeed = 4096;      // seed entries per query
constexpr uint64_t kNoKey = ~0ull;

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

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

__device__ __forceinline__ float ld_volatile_f(const unsigned* p) {
  return __uint_as_float(*(const volatile unsigned*)p);
}

// ---------------------------------------------------------------- lower bound
// One SAX word row (4 consecutive series' symbols of segment s) against B
// queries.  MINDIST branches: ABOVE q-U, BELOW L-q, IN 0 -- the
// paper's 3 masked SIMD branches become one 3-input max.  All arithmetic rounds
// toward -inf on outward-rounded bounds, so acc <= exact sum of delta^2.
template <int B>
__device__ __forceinline__ void lb_row(uint32_t word, const float2* __restrict__ q,
                                       const float2* __restrict__ s_lu, float (&acc)[4][B]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 lu = s_lu[(word >> (8 * j)) & 0xFFu];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float above = __fsub_rd(q[b].x, lu.y);  // q_lo - U_up  <= q - U
      const float below = __fsub_rd(lu.x, q[b].y);  // L_dn - q_hi  <= L - q
      const float delta = fmax3(above, below, 0.f);
      acc[j][b] = __fmaf_rd(delta, delta, acc[j][b]);
    }
  }
}

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

// acc[j][b] = sum_s delta^2 for series i0+j (4 consecutive series) and query b.
// WT = compile-time w (words preloaded for memory-level parallelism) or 0 (runtime w).
template <int B, int WT, bool AL>
__device__ __forceinline__ void lb_group(const uint8_t* __restrict__ sax, int64_t n, int w,
                                         int64_t i0, const float2* __restrict__ s_q,
                                         const float2* __restrict__ s_lu, float (&acc)[4][B]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int b = 0; b < B; ++b) acc[j][b] = 0.f;
  if (WT > 0) {
    uint32_t wd[WT > 0 ? WT : 1];
#pragma unroll
    for (int s = 0; s < WT; ++s) wd[s] = load_word<AL>(sax, n, s, i0);
#pragma unroll
    for (int s = 0; s < WT; ++s) {
      float2 q[B];
#pragma unroll
      for (int b = 0; b < B; ++b) q[b] = s_q[b * kMaxW + s];
      lb_row<B>(wd[s], q, s_lu, acc);
    }
  } else {
    uint32_t nxt = load_word<AL>(sax, n, 0, i0);
    for (int s = 0; s < w; ++s) {
      const uint32_t cur = nxt;
      if (s + 1 < w) nxt = load_word<AL>(sax, n, s + 1, i0);
      float2 q[B];
#pragma unroll
      for (int b = 0; b < B; ++b) q[b] = s_q[b * kMaxW + s];
      lb_row<B>(cur, q, s_lu, acc);
    }
  }
}

// Shared prologue: region bounds for the card, query pairs for the batch.
template <int B>
__device__ __forceinline__ void load_lu_q(const CardTables* __restrict__ tab,
                                          const float2* __restrict__ qlh, int w, float2* s_lu,
                                          float2* s_q) {
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) s_lu[i] = tab->lu[i];
  for (int i = threadIdx.x; i < B * kMaxW; i += blockDim.x) s_q[i] = qlh[i];
}

// ---------------------------------------------------------------- K2+K3a seed LB
// Query PAA in fp64 (segment means), stored as {round-down,
// round-up} fp32 -> qlh[b][s].  Then the LB over the sample [0, ns): every warp
// keeps its best (LB^2, id) per query -> seed_ids[b][warp].
template <int B, int WT, bool AL>
__global__ void __launch_bounds__(kLBThreads)
k_seed(const uint8_t* __restrict__ sax, int64_t n, int64_t ns, const float* __restrict__ queries,
       int nb, int len, int w, const CardTables* __restrict__ tab, float2* __restrict__ qlh,
       int* __restrict__ seed_ids, int S) {
  __shared__ float2 s_lu[kMaxCard];
  __shared__ float2 s_q[B * kMaxW];
  const int seglen = len / w;
  for (int i = threadIdx.x; i < kMaxCard; i += blockDim.x) s_lu[i] = tab->lu[i];
  for (int i = threadIdx.x; i < B * kMaxW; i += blockDim.x) {
    const int b = i / kMaxW, s = i % kMaxW;
    float2 v = make_float2(0.f, 0.f);
    if (b < nb && s < w) {
      const float* x = queries + (size_t)b * len + (size_t)s * seglen;
      double acc = 0.0;
      for (int j = 0; j < seglen; ++j) acc += (double)x[j];
      const double paa = acc / (double)seglen;
      v = make_float2(__double2float_rd(paa), __double2float_ru(paa));
    }
    s_q[i] = v;
    if (blockIdx.x == 0) qlh[i] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float best[B];
  uint32_t bid[B];
#pragma unroll
  for (int b = 0; b < B; ++b) { best[b] = INFINITY; bid[b] = 0xFFFFFFFFu; }
  const int64_t ngroups = (ns + 3) / 4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    float acc[4][B];
    lb_group<B, WT, AL>(sax, n, w, i0, s_q, s_lu, acc);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j >= ns) break;
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (acc[j][b] < best[b]) { best[b] = acc[j][b]; bid[b] = (uint32_t)(i0 + j); }
    }
  }
  // warp argmin of (LB, id) per query
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
  for (int b = 0; b < B; ++b) {
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
// d^2 between raw[id] and the query held in shared memory (warp-cooperative,
// one float4 per lane per 128-point chunk).  Early abandoning (north_star;
// S:159-167): after each chunk but the last, if the partial sum already exceeds
// `limit` the rest is not read and +inf is returned (*abandoned = true).
// Summation: <= len/128 sequential fma per lane, then a 5-level xor tree, so
// |fp32 - exact| <= (len/32 + 8) * 2^-24 * d^2 (d2up in the host code covers it).
__device__ __forceinline__ float warp_ed2(const float* __restrict__ raw, uint32_t id, int len,
                                          const float4* __restrict__ s_qv, float limit,
                                          bool* abandoned) {
  const int lane = threadIdx.x & 31;
  const int nf = len >> 2;
  const float4* row = reinterpret_cast<const float4*>(raw + (size_t)id * len);
  float acc = 0.f;
  for (int c0 = 0; c0 < nf; c0 += 32) {
    const int f = c0 + lane;
    if (f < nf) {
      const float4 x = __ldg(row + f);
      const float4 q = s_qv[f];
      float d;
      d = x.x - q.x; acc = fmaf(d, d, acc);
      d = x.y - q.y; acc = fmaf(d, d, acc);
      d = x.z - q.z; acc = fmaf(d, d, acc);
      d = x.w - q.w; acc = fmaf(d, d, acc);
    }
    if (c0 + 32 < nf && limit < INFINITY) {
      const float part = warp_sum(acc);
      if (part > limit) { *abandoned = true; return INFINITY; }
    }
  }
  *abandoned = false;
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
    if (id >= 0) {
      bool ab;
      const float d2 = warp_ed2(raw, (uint32_t)id, len, s_qv, INFINITY, &ab);
      key = make_key(d2, (uint32_t)id);
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

// ---------------------------------------------------------------- K3c seed select
// tau_seed^2 = k-th smallest seed d^2 (upper bound of the k-th NN distance,
// R8), rounded up by the fp32 summation error bound; +inf if < k seeds.
__global__ void __launch_bounds__(1024)
k_seed_select(const uint64_t* __restrict__ seed_keys, int S, int k, float d2up,
              unsigned* __restrict__ thr, unsigned* __restrict__ thr_seed, float* __restrict__ tau_out,
              int q0) {
  __shared__ uint64_t buf[kSortP];
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < kSortP; i += blockDim.x) buf[i] = (i < S) ? seed_keys[b * S + i] : kNoKey;
  __syncthreads();
  bitonic_sort(buf, kSortP);
  if (threadIdx.x == 0) {
    const uint64_t kth = buf[k - 1];
    const float t = (kth == kNoKey) ? INFINITY : __fmul_ru(key_val(kth), d2up);
    thr[b] = __float_as_uint(t);
    thr_seed[b] = __float_as_uint(t);
    if (tau_out) tau_out[q0 + b] = (kth == kNoKey) ? INFINITY : sqrtf(key_val(kth));
  }
}

// ---------------------------------------------------------------- K4 LBC pass
// Alg10: for every word, LB^2 < BSF^2 -> append (LB, position).
// Here: LB^2 <= tau_seed^2 (rigorous bounds on both sides), B queries per SAX
// read; warp-aggregated atomics reserve slots; a 256-bin LB histogram per
// query drives the ordering (K5).  count[b] keeps counting past `cap` so an
// overflow is detected exactly.
template <int B, int WT, bool AL>
__global__ void __launch_bounds__(kLBThreads)
k_lb(const uint8_t* __restrict__ sax, int64_t n, int w, float seglen_f,
     const CardTables* __restrict__ tab, const float2* __restrict__ qlh, int nb,
     const unsigned* __restrict__ thr, unsigned* __restrict__ count, unsigned* __restrict__ hist,
     uint64_t* __restrict__ cand, int64_t cap) {
  __shared__ float2 s_lu[kMaxCard];
  __shared__ float2 s_q[B * kMaxW];
  __shared__ float s_thr[B], s_scale[B];
  load_lu_q<B>(tab, qlh, w, s_lu, s_q);
  if (threadIdx.x < B) {
    const float t = (threadIdx.x < nb) ? __uint_as_float(thr[threadIdx.x]) : -1.f;
    s_thr[threadIdx.x] = t;
    s_scale[threadIdx.x] = bin_scale(t);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (n + 3) / 4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g - lane < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    float acc[4][B];
    if (g < ngroups) {
      lb_group<B, WT, AL>(sax, n, w, i0, s_q, s_lu, acc);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int b = 0; b < B; ++b) acc[j][b] = INFINITY;
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float t = s_thr[b];
      float lb[4];
      unsigned m = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lb[j] = __fmul_rd(acc[j][b], seglen_f);
        if (i0 + j < n && lb[j] <= t) m |= 1u << j;
      }
      if (__any_sync(0xffffffffu, m != 0)) {
        const int c = __popc(m);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        unsigned base = 0;
        if (lane == 31) base = atomicAdd(&count[b], (unsigned)incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint64_t pos = (uint64_t)base + (unsigned)(incl - c);
        const float sc = s_scale[b];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (m & (1u << j)) {
            if (pos < (uint64_t)cap) cand[(size_t)b * cap + pos] = make_key(lb[j], (uint32_t)(i0 + j));
            atomicAdd(&hist[b * kNB + lb_bin(lb[j], sc)], 1u);
            ++pos;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K5 bucket order
// Counting sort of the candidates by LB bin (the paper sorts its candidate list
// by file position for disk locality; in HBM the LB order is what
// matters: refinement stops at the first bin above the BSF).
__global__ void __launch_bounds__(256)
k_scatter(const uint64_t* __restrict__ cand, const unsigned* __restrict__ count,
          const unsigned* __restrict__ hist, const unsigned* __restrict__ thr,
          unsigned* __restrict__ cursor, uint64_t* __restrict__ sorted, int64_t cap) {
  __shared__ unsigned s_off[kNB];
  const int b = blockIdx.y;
  // exclusive prefix of the histogram (Hillis-Steele over 256 bins)
  unsigned v = hist[b * kNB + threadIdx.x];
  s_off[threadIdx.x] = v;
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
  __syncthreads();
  const float sc = bin_scale(__uint_as_float(thr[b]));
  const int64_t cnt = imin64((int64_t)count[b], cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = cand[(size_t)b * cap + i];
    const int bin = lb_bin(key_val(key), sc);
    const uint64_t pos = (uint64_t)s_off[bin] + atomicAdd(&cursor[b * kNB + bin], 1u);
    if (pos < (uint64_t)cap) sorted[(size_t)b * cap + pos] = key;
  }
}

// ---------------------------------------------------------------- K6 RDC pass
// Alg11: take the next candidate (static interleave over the
// LB-ordered list instead of a locked cursor), skip it if LB > BSF,
// else read raw[id] and compute the true distance (early abandoning), and
// update the BSF.  BSF for k-NN = k-th best: each CTA keeps a
// top-k list in shared memory; when full, its k-th d^2 (rounded up) is pushed to
// the query's global threshold with atomicMin on the float bits, which every
// warp re-reads before each candidate.
//   wave 0 (k > 1 only): one CTA refines the lowest-LB ~max(M, 2k) candidates so
//                       that its list fills and tightens the BSF early;
//   wave 1: all other candidates, many CTAs per query.
struct RefineArgs {
  const float* raw;
  int len;
  const float* queries;  // batch base [nb][len]
  const uint64_t* sorted;
  int64_t cap;
  const unsigned* count;
  const unsigned* hist;
  unsigned* thr;         // live pruning threshold (float bits), per query
  const unsigned* thr_seed;  // tau_seed^2 (float bits): the binning scale of K4/K5
  unsigned* wave_end;    // per query: end of wave 0 in the sorted list
  unsigned* refined;     // per query counter
  uint64_t* lists;       // [nb][nslots][k]
  int nslots;
  int k;
  int wave;
  int wave_m;            // wave-0 size target
  float d2up;            // 1 + bound on the relative error of an fp32 d^2 (rounding up)
};

__global__ void __launch_bounds__(1024)
k_refine(RefineArgs a) {
  extern __shared__ float4 s_dyn[];
  float4* s_qv = s_dyn;                                            // len/4 float4
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(s_dyn + (a.len >> 2));  // k keys
  __shared__ int s_lock, s_size, s_maxpos;
  __shared__ uint64_t s_maxkey;
  __shared__ float s_kth;          // local k-th d^2 (unscaled) when full, else inf
  __shared__ float s_thr_local;    // local k-th d^2 rounded up, else inf
  __shared__ unsigned s_begin, s_end, s_refined;
  __shared__ float s_scale;

  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float4* qsrc = reinterpret_cast<const float4*>(a.queries + (size_t)b * a.len);
  for (int i = threadIdx.x; i < (a.len >> 2); i += blockDim.x) s_qv[i] = qsrc[i];
  for (int i = threadIdx.x; i < a.k; i += blockDim.x) s_keys[i] = kNoKey;
  if (threadIdx.x == 0) {
    s_lock = 0; s_size = 0; s_maxpos = 0; s_maxkey = kNoKey;
    s_kth = INFINITY; s_thr_local = INFINITY; s_refined = 0;
    s_scale = bin_scale(__uint_as_float(a.thr_seed[b]));
    const unsigned cnt = (unsigned)imin64((int64_t)a.count[b], a.cap);
    if (a.wave == 0) {
      // wave 0 = all bins up to the first whose cumulative count reaches wave_m
      unsigned cum = 0;
      int bin = 0;
      for (; bin < kNB; ++bin) {
        cum += a.hist[b * kNB + bin];
        if (cum >= (unsigned)a.wave_m) break;
      }
      const unsigned e = min(cum, cnt);
      s_begin = 0; s_end = e;
      a.wave_end[b] = e;
    } else {
      s_begin = min(a.wave_end[b], cnt); s_end = cnt;
    }
  }
  __syncthreads();
  const unsigned begin = s_begin, end = s_end;
  const float scale = s_scale;
  unsigned my_refined = 0;
  const uint64_t* list = a.sorted + (size_t)b * a.cap;

  for (unsigned i = begin + blockIdx.x * nw + warp; i < end; i += gridDim.x * nw) {
    const uint64_t key = list[i];
    const float lb = key_val(key);
    const float thr_live = fminf(ld_volatile_f(&a.thr[b]), *(volatile float*)&s_thr_local);
    if (lb > thr_live) {
      // sorted by bin: once this bin's lower edge is above the BSF, so is every later one
      const int bin = lb_bin(lb, scale);
      if (bin >= 1 && (float)(bin - 1) > thr_live * scale) break;
      continue;
    }
    const float limit = fminf(thr_live, *(volatile float*)&s_kth);
    bool ab;
    const float d2 = warp_ed2(a.raw, key_id(key), a.len, s_qv, limit, &ab);
    ++my_refined;
    if (ab) continue;
    const uint64_t k2 = make_key(d2, key_id(key));
    if (*(volatile int*)&s_size >= a.k && k2 >= *(volatile uint64_t*)&s_maxkey) continue;
    // insert under the CTA lock (warp-cooperative max recomputation)
    if (lane == 0) {
      while (atomicCAS(&s_lock, 0, 1) != 0) { }
    }
    __syncwarp();
    __threadfence_block();
    volatile uint64_t* vk = s_keys;
    const int size = *(volatile int*)&s_size;
    bool changed = false;
    if (size < a.k) {
      if (lane == 0) { vk[size] = k2; *(volatile int*)&s_size = size + 1; }
      changed = (size + 1 == a.k);
    } else if (k2 < *(volatile uint64_t*)&s_maxkey) {
      if (lane == 0) vk[*(volatile int*)&s_maxpos] = k2;
      changed = true;
    }
    __syncwarp();
    __threadfence_block();
    if (changed) {
      uint64_t mk = 0;
      int mp = 0;
      for (int t = lane; t < a.k; t += 32) {
        const uint64_t v = vk[t];
        if (v >= mk) { mk = v; mp = t; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t v2 = __shfl_xor_sync(0xffffffffu, mk, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, mp, o);
        if (v2 > mk || (v2 == mk && p2 > mp)) { mk = v2; mp = p2; }
      }
      if (lane == 0) {
        *(volatile uint64_t*)&s_maxkey = mk;
        *(volatile int*)&s_maxpos = mp;
        const float kth = key_val(mk);
        *(volatile float*)&s_kth = kth;
        const float up = __fmul_ru(kth, a.d2up);
        *(volatile float*)&s_thr_local = up;
        atomicMin(&a.thr[b], __float_as_uint(up));
      }
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) atomicExch(&s_lock, 0);
  }
  if (lane == 0 && my_refined) atomicAdd(&s_refined, my_refined);
  __syncthreads();
  uint64_t* out = a.lists + ((size_t)b * a.nslots + (a.wave == 0 ? 0 : 1 + blockIdx.x)) * a.k;
  for (int i = threadIdx.x; i < a.k; i += blockDim.x) out[i] = s_keys[i];
  if (threadIdx.x == 0 && s_refined) atomicAdd(&a.refined[b], s_refined);
}

// ---------------------------------------------------------------- K7 finalize
// Merge the per-CTA top-k lists: repeatedly sort [current top-k | next chunk]
// in shared memory and keep the first k.  Output ascending (d^2, id) -> (id, sqrt d^2).
__global__ void __launch_bounds__(1024)
k_finalize(const uint64_t* __restrict__ lists, int nslots, int first_slot, int k, int q0,
           int64_t* __restrict__ out_idx, float* __restrict__ out_dist,
           const unsigned* __restrict__ count, const unsigned* __restrict__ refined,
           unsigned* __restrict__ all_count, unsigned* __restrict__ all_refined) {
  __shared__ uint64_t buf[kSortP];
  const int b = blockIdx.x;
  const int64_t total = (int64_t)(nslots - first_slot) * k;
  const uint64_t* src = lists + ((size_t)b * nslots + first_slot) * k;
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
    all_count[q0 + b] = count[b];
    all_refined[q0 + b] = refined[b];
  }
}

// ---------------------------------------------------------------- host side
int g_sms = 0;
int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
  int v = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem);
  return v > 0 ? v : 1;
}

// scratch of one batch (device)
struct Ws {
  float2* qlh;
  int* seed_ids;
  uint64_t* seed_keys;
  unsigned* zero_block;  // thr | count | hist | cursor | refined | wave_end (zeroed per batch)
  unsigned* thr;
  unsigned* thr_seed;
  unsigned* count;
  unsigned* hist;
  unsigned* cursor;
  unsigned* refined;
  unsigned* wave_end;
  size_t zero_bytes;
  uint64_t* cand;
  uint64_t* sorted;
  uint64_t* lists;
  void* base;
};

struct Plan {
  int64_t n;
  int len, w, card, k;
  int B;          // batch
  int S;          // seed entries per query (warps of the seed grid)
  int seed_grid;
  int64_t ns;     // seed sample
  int64_t cap;
  int XB;         // wave-1 CTAs per query
  int nslots;
  int wave_m;
  float d2up;     // fp32 d^2 -> rigorous upper bound factor
};

template <int B, int WT, bool AL>
cudaError_t launch_seed_lb(const Plan& p, const uint8_t* sax, const float* qb, int nb,
                           const CardTables* tab, const Ws& ws, cudaStream_t st) {
  return PARIS_LAUNCH("seed_lb", (k_seed<B, WT, AL>), p.seed_grid, kLBThreads, 0, st, sax, p.n, p.ns,
                      qb, nb, p.len, p.w, tab, ws.qlh, ws.seed_ids, p.S);
}

template <int B, int WT, bool AL>
cudaError_t launch_lb(const Plan& p, const uint8_t* sax, int nb, const CardTables* tab, const Ws& ws,
                      cudaStream_t st, int64_t cap) {
  static int occ = 0;
  if (!occ) occ = occupancy(k_lb<B, WT, AL>, kLBThreads, 0);
  const int64_t ngroups = (p.n + 3) / 4;
  const int64_t need = (ngroups + kLBThreads - 1) / kLBThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms() * occ));
  return PARIS_LAUNCH("lb_pass", (k_lb<B, WT, AL>), grid, kLBThreads, 0, st, sax, p.n, p.w,
                      (float)(p.len / p.w), tab, ws.qlh, nb, ws.thr_seed, ws.count, ws.hist, ws.cand, cap);
}

template <int B, int WT>
cudaError_t dispatch_al(bool al, bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                        const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  if (lb) return al ? launch_lb<B, WT, true>(p, sax, nb, tab, ws, st, cap)
                    : launch_lb<B, WT, false>(p, sax, nb, tab, ws, st, cap);
  // the seed pass covers ~1/16 of the array: the register-light runtime-w variant suffices
  return al ? launch_seed_lb<B, 0, true>(p, sax, qb, nb, tab, ws, st)
            : launch_seed_lb<B, 0, false>(p, sax, qb, nb, tab, ws, st);
}

template <int B>
cudaError_t dispatch_w(bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                       const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  const bool al = (p.n % 4) == 0;
  if (p.w == 16) return dispatch_al<B, 16>(al, lb, p, sax, qb, nb, tab, ws, st, cap);
  return dispatch_al<B, 0>(al, lb, p, sax, qb, nb, tab, ws, st, cap);
}

cudaError_t dispatch_b(int Bt, bool lb, const Plan& p, const uint8_t* sax, const float* qb, int nb,
                       const CardTables* tab, const Ws& ws, cudaStream_t st, int64_t cap) {
  switch (Bt) {
    case 1: return dispatch_w<1>(lb, p, sax, qb, nb, tab, ws, st, cap);
    case 2: return dispatch_w<2>(lb, p, sax, qb, nb, tab, ws, st, cap);
    case 4: return dispatch_w<4>(lb, p, sax, qb, nb, tab, ws, st, cap);
    default: return dispatch_w<8>(lb, p, sax, qb, nb, tab, ws, st, cap);
  }
}

int pow2_batch(int nb) { return nb <= 1 ? 1 : nb <= 2 ? 2 : nb <= 4 ? 4 : 8; }

// Allocate the batch scratch for `cap` candidates per query.
int alloc_ws(const Plan& p, int64_t cap, Ws& ws, cudaStream_t st) {
  const int B = pow2_batch(p.B);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
  const size_t o_qlh = take(sizeof(float2) * B * kMaxW);
  const size_t o_sid = take(sizeof(int) * B * p.S);
  const size_t o_skey = take(sizeof(uint64_t) * B * p.S);
  const size_t zb = sizeof(unsigned) * (B + B + B + B * kNB + B * kNB + B + B);
  const size_t o_zero = take(zb);
  const size_t o_cand = take(sizeof(uint64_t) * B * (size_t)cap);
  const size_t o_sorted = take(sizeof(uint64_t) * B * (size_t)cap);
  const size_t o_lists = take(sizeof(uint64_t) * B * (size_t)p.nslots * p.k);
  void* base = nullptr;
  cudaError_t e = cudaMallocAsync(&base, off, st);
  if (e != cudaSuccess) {
    set_error("paris_knn_exact: scratch allocation of %zu bytes failed (%s)", off, cudaGetErrorString(e));
    cudaGetLastError();
    return PARIS_ENOMEM;
  }
  char* c = (char*)base;
  ws.base = base;
  ws.qlh = (float2*)(c + o_qlh);
  ws.seed_ids = (int*)(c + o_sid);
  ws.seed_keys = (uint64_t*)(c + o_skey);
  ws.zero_block = (unsigned*)(c + o_zero);
  ws.zero_bytes = zb;
  ws.thr = ws.zero_block;
  ws.thr_seed = ws.thr + B;
  ws.count = ws.thr_seed + B;
  ws.hist = ws.count + B;
  ws.cursor = ws.hist + B * kNB;
  ws.refined = ws.cursor + B * kNB;
  ws.wave_end = ws.refined + B;
  ws.cand = (uint64_t*)(c + o_cand);
  ws.sorted = (uint64_t*)(c + o_sorted);
  ws.lists = (uint64_t*)(c + o_lists);
  return PARIS_OK;
}

// One batch of nb <= 8 queries (device pointers).  Outputs at [q0 .. q0+nb).
int run_batch(const Plan& p, const float* raw, const uint8_t* sax, const float* qbatch, int nb, int q0,
              int64_t cap, const CardTables* tab, const Ws& ws, int64_t* d_idx, float* d_dist,
              unsigned* all_count, unsigned* all_refined, float* all_tau, cudaStream_t st) {
  const int Bt = pow2_batch(nb);
  cudaError_t e = cudaMemsetAsync(ws.zero_block, 0, ws.zero_bytes, st);
  if (e != cudaSuccess) return cuda_error(e, "memset scratch");
  PARIS_CHECK_LAUNCH(dispatch_b(Bt, false, p, sax, qbatch, nb, tab, ws, st, cap), "seed_lb launch");
  {
    dim3 g((unsigned)((p.S + 7) / 8), (unsigned)nb);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_ed", k_seed_ed, g, kRefThreads, (size_t)p.len * 4, st, raw, p.len,
                                    qbatch, ws.seed_ids, p.S, ws.seed_keys),
                       "seed_ed launch");
  }
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("seed_select", k_seed_select, nb, 1024, 0, st, ws.seed_keys, p.S, p.k,
                                  p.d2up, ws.thr, ws.thr_seed, all_tau, q0),
                     "seed_select launch");
  PARIS_CHECK_LAUNCH(dispatch_b(Bt, true, p, sax, qbatch, nb, tab, ws, st, cap), "lb_pass launch");
  {
    const int xs = std::max(1, std::min(sms() * 4 / nb, 1024));
    dim3 g((unsigned)xs, (unsigned)nb);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("scatter", k_scatter, g, 256, 0, st, ws.cand, ws.count, ws.hist, ws.thr_seed,
                                    ws.cursor, ws.sorted, cap),
                       "scatter launch");
  }
  RefineArgs ra;
  ra.raw = raw; ra.len = p.len; ra.queries = qbatch; ra.sorted = ws.sorted; ra.cap = cap;
  ra.count = ws.count; ra.hist = ws.hist; ra.thr = ws.thr; ra.thr_seed = ws.thr_seed; ra.wave_end = ws.wave_end;
  ra.refined = ws.refined; ra.lists = ws.lists; ra.nslots = p.nslots; ra.k = p.k; ra.wave_m = p.wave_m;
  ra.d2up = p.d2up;
  const size_t rsmem = (size_t)p.len * 4 + (size_t)p.k * 8;
  if (p.k > 1) {
    ra.wave = 0;
    dim3 g(1u, (unsigned)nb);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("refine_wave0", k_refine, g, kRefAThreads, rsmem, st, ra), "refine0 launch");
  }
  {
    ra.wave = 1;
    dim3 g((unsigned)p.XB, (unsigned)nb);
    PARIS_CHECK_LAUNCH(PARIS_LAUNCH("refine", k_refine, g, kRefThreads, rsmem, st, ra), "refine launch");
  }
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("finalize", k_finalize, nb, 1024, 0, st, ws.lists, p.nslots,
                                  p.k > 1 ? 0 : 1, p.k, q0,
                                  d_idx, d_dist, ws.count, ws.refined, all_count, all_refined),
                     "finalize launch");
  return PARIS_OK;
}

bool is_host_ptr(const void* p) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return true; }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

}  // namespace

int knn_impl(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int nq, int k,
             int64_t* out_idx, float* out_dist, int len, int w, int card, cudaStream_t st,
             const paris_knn_config* cfg, paris_knn_stats* stats) {
  if (!raw || !sax || (nq > 0 && (!queries || !out_idx || !out_dist))) {
    set_error("paris_knn_exact: null pointer");
    return PARIS_EINVAL;
  }
  if (n < 1 || n >= (int64_t(1) << 31) || nq < 0 || k < 1 || k > n || k > PARIS_MAX_K) {
    set_error("paris_knn_exact: bad sizes n=%lld nq=%d k=%d (need 1<=k<=min(n,%d), n<2^31)",
              (long long)n, nq, k, PARIS_MAX_K);
    return PARIS_EINVAL;
  }
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

  Plan p;
  p.n = n; p.len = len; p.w = w; p.card = card; p.k = k;
  p.B = (cfg && cfg->batch > 0) ? std::min(cfg->batch, kMaxB) : kMaxB;
  const int seed_div = (cfg && cfg->seed_div > 0) ? cfg->seed_div : 16;
  p.ns = std::min<int64_t>(n, std::max<int64_t>(n / seed_div, std::min<int64_t>(n, 65536)));
  {
    const int64_t groups = (p.ns + 3) / 4;
    const int64_t need = (groups + kLBThreads - 1) / kLBThreads;
    p.seed_grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, std::min(sms() * 2, kMaxSeed / 8)));
    p.S = p.seed_grid * (kLBThreads / 32);
  }
  p.cap = std::min<int64_t>(n, std::max<int64_t>(65536, n / 32));
  p.XB = std::max(1, std::min(sms() * 4 / std::max(1, p.B), 65535));
  p.nslots = 1 + p.XB;
  p.wave_m = std::max((cfg && cfg->wave_a > 0) ? cfg->wave_a : 256, 2 * k);
  // |fp32 d^2 - exact| <= (len/32 + 8) u d^2 (warp_ed2); doubled for slack, u = 2^-24
  p.d2up = (float)(1.0 + 2.0 * (len / 32 + 8) * 5.9604644775390625e-08);

  // host <-> device staging of queries / outputs
  const bool hq = is_host_ptr(queries), hi = is_host_ptr(out_idx), hd = is_host_ptr(out_dist);
  cudaError_t e;
  char* stage = nullptr;
  const size_t qbytes = (size_t)nq * len * 4, ibytes = (size_t)nq * k * 8, dbytes = (size_t)nq * k * 4;
  const size_t cbytes = (size_t)nq * 4 * 3;
  e = cudaMallocAsync((void**)&stage, qbytes + ibytes + dbytes + cbytes + 1024, st);
  if (e != cudaSuccess) { cudaGetLastError(); set_error("paris_knn_exact: staging alloc failed"); return PARIS_ENOMEM; }
  const float* d_q = queries;
  int64_t* d_idx = out_idx;
  float* d_dist = out_dist;
  char* cur = stage;
  float* sq = (float*)cur; cur += (qbytes + 255) & ~255ull;
  int64_t* sidx = (int64_t*)cur; cur += (ibytes + 255) & ~255ull;
  float* sdist = (float*)cur; cur += (dbytes + 255) & ~255ull;
  unsigned* all_count = (unsigned*)cur;
  unsigned* all_refined = all_count + nq;
  float* all_tau = (float*)(all_refined + nq);
  if (hq) {
    e = cudaMemcpyAsync(sq, queries, qbytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { cudaFreeAsync(stage, st); return cuda_error(e, "H2D queries"); }
    d_q = sq;
  }
  if (hi) d_idx = sidx;
  if (hd) d_dist = sdist;
  if ((reinterpret_cast<uintptr_t>(d_q) & 15) != 0) {
    cudaFreeAsync(stage, st);
    set_error("paris_knn_exact: queries must be 16-byte aligned");
    return PARIS_EINVAL;
  }

  Ws ws;
  int rc = alloc_ws(p, p.cap, ws, st);
  if (rc) { cudaFreeAsync(stage, st); return rc; }
  for (int q0 = 0; q0 < nq && rc == PARIS_OK; q0 += p.B) {
    const int nb = std::min(p.B, nq - q0);
    rc = run_batch(p, raw, sax, d_q + (size_t)q0 * len, nb, q0, p.cap, tab, ws, d_idx, d_dist,
                   all_count, all_refined, all_tau, st);
  }
  // overflow check: one synchronization per call
  std::vector<unsigned> h_count(nq), h_ref(nq);
  std::vector<float> h_tau(nq);
  if (rc == PARIS_OK) {
    e = cudaMemcpyAsync(h_count.data(), all_count, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "paris_knn_exact execution");
  }
  if (rc == PARIS_OK) {
    for (int q = 0; q < nq && rc == PARIS_OK; ++q) {
      if ((int64_t)h_count[q] <= p.cap) continue;
      // re-scan this query alone with an exact-size candidate buffer
      Plan p1 = p;
      p1.B = 1;
      p1.XB = std::max(1, std::min(sms() * 4, 65535));
      p1.nslots = 1 + p1.XB;
      p1.cap = std::min<int64_t>(n, (int64_t)h_count[q]);
      Ws ws1;
      rc = alloc_ws(p1, p1.cap, ws1, st);
      if (rc) break;
      rc = run_batch(p1, raw, sax, d_q + (size_t)q * len, 1, q, p1.cap, tab, ws1, d_idx, d_dist,
                     all_count, all_refined, all_tau, st);
      cudaFreeAsync(ws1.base, st);
    }
  }
  if (rc == PARIS_OK && (hi || hd || stats)) {
    e = cudaSuccess;
    if (hi) e = cudaMemcpyAsync(out_idx, sidx, ibytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && hd) e = cudaMemcpyAsync(out_dist, sdist, dbytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && stats) {
      e = cudaMemcpyAsync(h_count.data(), all_count, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h_ref.data(), all_refined, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h_tau.data(), all_tau, (size_t)nq * 4, cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "paris_knn_exact D2H");
    if (rc == PARIS_OK && stats) {
      for (int q = 0; q < nq; ++q) {
        if (stats->candidates) stats->candidates[q] = h_count[q];
        if (stats->refined) stats->refined[q] = h_ref[q];
        if (stats->tau_seed) stats->tau_seed[q] = h_tau[q];
      }
    }
  }
  cudaFreeAsync(ws.base, st);
  cudaFreeAsync(stage, st);
  return rc;
}

}  // namespace paris

extern "C" {

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

}  // extern "C"
