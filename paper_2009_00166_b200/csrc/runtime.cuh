// libparis internal runtime: error reporting, launch accounting/profiling,
// breakpoint tables.  Product code (sm_100a); shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>

#include "../../include/paris.h"

namespace paris {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kMaxCard = 256;
constexpr int kNumCards = 8;  // 2, 4, ..., 256

// Per-cardinality breakpoint tables (device resident, built once per device).
//   cuts_f[c]  fp32 round-to-nearest of cut_{c+1} = Phi^-1((c+1)/card), c < card-1;
//              +inf for c >= card-1 (pads the binary search to 256 entries)
//   cuts_d[c]  same in fp64
//   lu[c]      region bounds of symbol c as fp32 {L rounded down, U rounded up}:
//              L = cut_c (-inf for c = 0), U = cut_{c+1} (+inf for c = card-1);
//              outward rounding makes the fp32 region contain the exact one, so
//              the fp32 lower bound never exceeds the exact one.
//   lu16[c]    the same region as packed fp16 pairs for the batched lower bound:
//              .x = half2(-U16, -U16), .y = half2(L16, L16) with L16 = L rounded
//              down and U16 = U rounded up to fp16 (so [L16, U16] contains the
//              exact region; +-inf stay infinite)
//   lu16p[c]   half2(-U16, L16) (low half -U16): the single-query form
//   lut[k]     quantization shortcut over kLutN buckets of width 1/kLutScale on
//              [-kLutLo, kLutLo): {fp32 bits of the single cut lying within
//              kLutMargin of bucket k (3e38 if none), #cuts <= left edge - margin}
//              so that symbol = lut.y + (v >= cut) for every v whose computed
//              bucket is k (the cut gap, >= 0.0097 at card 256, exceeds the
//              window 1/kLutScale + 2*kLutMargin = 0.0059)
constexpr int kLutN = 2048;
constexpr float kLutLo = 4.0f;
constexpr float kLutScale = 256.0f;
constexpr double kLutMargin = 1e-3;
struct CardTables {
  float cuts_f[kMaxCard];
  double cuts_d[kMaxCard];
  float2 lu[kMaxCard];
  uint2 lu16[kMaxCard];
  uint32_t lu16p[kMaxCard];
  uint2 lut[kLutN];
};

// Index sort key (f1): 8-bit-normalized symbols (card < 256 shifted up), bits
// interleaved most significant first -- bit 7 of segments 0..15, then bit 6, ...
// down to bit 4: the iSAX tree's split order at uniform cardinality.
__device__ __forceinline__ uint64_t isax_key16(const uint8_t* sym, int shift) {
  uint64_t key = 0;
#pragma unroll
  for (int b = 7; b >= 4; --b)
#pragma unroll
    for (int s = 0; s < 16; ++s) key = (key << 1) | (uint64_t)(((sym[s] << shift) >> b) & 1u);
  return key;
}

// Returns the device table for `card` (power of two in [2,256]) on the current
// device, building all eight on first use.  nullptr + error set on failure.
const CardTables* device_tables(int card);

// Host copy (for tests/debug): fills cuts (card-1 doubles).
void host_cuts(int card, double* cuts);

// fp16 bits of v rounded toward -inf (dir < 0) or +inf (dir > 0); +-inf map to +-inf.
uint16_t half_bits_dir(double v, int dir);

// Keep freed stream-ordered scratch mapped in the current device's default
// memory pool (release threshold = max) so repeated calls do not remap it.
void retain_pool();

// SM count of the current device (cached per device; thread-safe).
int device_sms();
// tuning variants (paris_debug_set_variant): [0] index LB item form, [1] batch-1 LB kernel
extern int g_variant[4];

// Per-(key, device) one-time setup -- e.g. cudaFuncSetAttribute of a kernel -- run under
// a lock, so a concurrent first caller waits until it is done; cached only on success.
cudaError_t once_per_device(const void* key, const std::function<cudaError_t(int dev)>& f);

// Per-(key, device) integer (an occupancy or a shared-memory size), computed once
// under a lock by f (thread-safe).
int cached_per_device(const void* key, const std::function<int(int dev)>& f);

// Cached device scratch (the boundary's workspace): `bytes` of device memory usable by
// work on stream st.  A grow-only entry per device is reused across calls; every reuse
// is ordered after the previous user's work on the device (an event recorded at
// release), so a call never allocates or synchronizes in the steady state.  Distinct
// host threads get distinct entries.  *gen changes whenever the entry's memory is
// reallocated.  nullptr (+ error set) on failure.
void* ws_acquire(size_t bytes, cudaStream_t st, void** handle, uint64_t* gen);
void ws_release(void* handle, cudaStream_t st);
// Free every idle cached entry (synchronizes the device).
void ws_free_all();

// ---- errors
void set_error(const char* fmt, ...);
int cuda_error(cudaError_t e, const char* what);

// ---- launch accounting
struct LaunchScope {
  LaunchScope(const char* name, cudaStream_t st);
  ~LaunchScope();
  const char* name_;
  cudaStream_t st_;
  int slot_;
};

}  // namespace paris

// Device-side bounds checks for debug builds (PARIS_DEBUG=1 at build time):
// a violated check traps the kernel (cudaErrorLaunchFailure) instead of reading
// or writing out of bounds.  Compiled out otherwise.
#ifdef PARIS_DEBUG_CHECKS
#define PARIS_DCHECK(cond)                                                             \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("PARIS_DCHECK failed: %s at %s:%d\n", #cond, __FILE__, __LINE__);         \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define PARIS_DCHECK(cond) \
  do {                     \
  } while (0)
#endif

// Launch a kernel with accounting; evaluates to the cudaError_t of the launch.
#define PARIS_LAUNCH(name, kernel, grid, block, smem, stream, ...)            \
  ([&]() -> cudaError_t {                                                     \
    ::paris::LaunchScope _scope(name, stream);                                \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);               \
    return cudaGetLastError();                                                \
  }())

#define PARIS_CHECK_LAUNCH(call, what)                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::paris::cuda_error(_e, what); \
  } while (0)
