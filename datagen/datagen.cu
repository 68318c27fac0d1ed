// Harness-side synthetic data generator (NOT part of libparis, NOT method arithmetic).
//
// Same counter-based generator as datagen/__init__.py: Philox4x32-10 with
// counter (id lo, id hi, point/4, stream) and key (seed lo, seed hi), Box-Muller
// in double, random walk x0 ~ N(0,1), x_t = x_{t-1} + N(0,1) (PAPER.md
// P:1436-1442), z-normalization in double with population std (SURVEY §8(c)
// reading 9), stored fp32.  One warp per series: lane l owns a contiguous run of
// points, the cumulative sum is a warp scan in double.
//
// Built as datagen/libparis_datagen.so (see __graft_entry__.build()).
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
constexpr int kMaxPerLane = 32;  // len <= 1024

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(kM0, c.x), lo0 = kM0 * c.x;
    uint32_t hi1 = __umulhi(kM1, c.z), lo1 = kM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += kW0;
    k1 += kW1;
  }
  return c;
}

__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, double& z0, double& z1) {
  const double scale = 2.3283064365386963e-10;  // 2^-32
  double u1 = ((double)a + 0.5) * scale;
  double u2 = ((double)b + 0.5) * scale;
  double rad = sqrt(-2.0 * log(u1));
  double ang = 2.0 * 3.141592653589793 * u2;
  z0 = rad * cos(ang);
  z1 = rad * sin(ang);
}

// Normals of points [4*blk, 4*blk+4) of series `id`.
__device__ __forceinline__ void normals4(uint64_t id, uint32_t blk, uint32_t stream,
                                         uint64_t seed, double z[4]) {
  uint4 r = philox(make_uint4((uint32_t)id, (uint32_t)(id >> 32), blk, stream),
                   (uint32_t)seed, (uint32_t)(seed >> 32));
  box_muller(r.x, r.y, z[0], z[1]);
  box_muller(r.z, r.w, z[2], z[3]);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// mode 0: random walk of series id (first_id + s).
// mode 1: noisy member: base = data[src[s]] (fp32) + fp32(sigma * z), z from stream 1 with id s.
__global__ void k_gen(float* __restrict__ out, int64_t n, int len, uint64_t seed, int64_t first_id,
                      int mode, const float* __restrict__ data, const int64_t* __restrict__ src,
                      double sigma) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nblk = len >> 2;
  const int bpl = (nblk + 31) / 32;  // Philox blocks per lane (contiguous run)
  for (int64_t s = warp; s < n; s += nwarps) {
    double x[kMaxPerLane];
    int cnt = 0;
    const int b0 = lane * bpl;
#pragma unroll 1
    for (int b = 0; b < bpl; ++b) {
      int blk = b0 + b;
      double z[4];
      if (blk < nblk) {
        if (mode == 0) {
          normals4((uint64_t)(first_id + s), (uint32_t)blk, 0u, seed, z);
        } else {
          normals4((uint64_t)s, (uint32_t)blk, 1u, seed, z);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) x[b * 4 + j] = (blk < nblk) ? z[j] : 0.0;
      cnt += (blk < nblk) ? 4 : 0;
    }
    double mean, sd;
    if (mode == 0) {
      // lane-local inclusive prefix, then warp exclusive scan of lane totals
      double run = 0.0;
      for (int i = 0; i < bpl * 4; ++i) { run += x[i]; x[i] = run; }
      double incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      double off = incl - run;
      for (int i = 0; i < bpl * 4; ++i) x[i] += off;
    } else {
      const float* base = data + (size_t)src[s] * len;
      for (int i = 0; i < bpl * 4; ++i) {
        int p = b0 * 4 + i;
        if (p < len) {
          float v = base[p] + (float)(sigma * x[i]);
          x[i] = (double)v;
        } else {
          x[i] = 0.0;
        }
      }
    }
    double ls = 0.0;
    for (int i = 0; i < cnt; ++i) ls += x[i];
    mean = warp_sum(ls) / (double)len;
    double lv = 0.0;
    for (int i = 0; i < cnt; ++i) { double d = x[i] - mean; lv += d * d; }
    sd = sqrt(warp_sum(lv) / (double)len);
    float* o = out + (size_t)s * len;
    for (int i = 0; i < cnt; ++i) {
      int p = b0 * 4 + i;
      o[p] = (sd < 1e-8) ? 0.0f : (float)((x[i] - mean) / sd);
    }
  }
}

int launch(float* out, int64_t n, int len, uint64_t seed, int64_t first_id, int mode,
           const float* data, const int64_t* src, double sigma, cudaStream_t st) {
  if (!out || n < 0 || len < 4 || (len & 3) || len > 4 * 32 * (kMaxPerLane / 4)) return -1;
  if (n == 0) return 0;
  int64_t warps = n;
  int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_gen<<<(unsigned)blocks, 256, 0, st>>>(out, n, len, seed, first_id, mode, data, src, sigma);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace

extern "C" {

// out: device [n][len] fp32. Random walks for ids first_id .. first_id+n-1, z-normalized.
int paris_datagen_walks(float* out, int64_t n, int32_t len, uint64_t seed, int64_t first_id,
                        void* stream) {
  return launch(out, n, len, seed, first_id, 0, nullptr, nullptr, 0.0, (cudaStream_t)stream);
}

// out: device [nq][len]; data: device [*][len]; src: device int64 [nq] source ids.
int paris_datagen_noisy(const float* data, const int64_t* src, int32_t nq, int32_t len,
                        double sigma, uint64_t seed, float* out, void* stream) {
  if (!data || !src) return -1;
  return launch(out, nq, len, seed, 0, 1, data, src, sigma, (cudaStream_t)stream);
}

}  // extern "C"
