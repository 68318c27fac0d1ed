// libparis runtime: errors, launch accounting / per-kernel device time, and the
// N(0,1) breakpoint tables (reading R2: cut_k = Phi^-1(k/card)).
#include "runtime.cuh"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

namespace paris {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err = "no error";

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

int cuda_error(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return PARIS_ECUDA;
}

// ------------------------------------------------------------------ launch accounting
static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_profile_on{0};

struct ProfRec {
  std::string name;
  cudaEvent_t ev0, ev1;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;          // pending (unread) launches
static std::vector<cudaEvent_t> g_ev_pool;   // recycled events
struct ProfAgg {
  std::string name;
  int64_t launches;
  double ms;
};
static std::vector<ProfAgg> g_agg;

static cudaEvent_t get_event() {
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

LaunchScope::LaunchScope(const char* name, cudaStream_t st) : name_(name), st_(st), slot_(-1) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_profile_on.load(std::memory_order_relaxed)) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r{name, get_event(), get_event()};
    cudaEventRecord(r.ev0, st);
    g_prof.push_back(r);
    slot_ = (int)g_prof.size() - 1;
  }
}

static int sync_debug() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PARIS_SYNC_DEBUG");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v;
}

LaunchScope::~LaunchScope() {
  if (slot_ >= 0) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (slot_ < (int)g_prof.size()) cudaEventRecord(g_prof[slot_].ev1, st_);
  }
  if (sync_debug()) {  // debugging aid: name each launch, wait for it
    fprintf(stderr, "[paris] launch %s\n", name_);
    fflush(stderr);
    cudaError_t e = cudaStreamSynchronize(st_);
    fprintf(stderr, "[paris] done %s: %s\n", name_, cudaGetErrorString(e));
    fflush(stderr);
  }
}

static void drain_locked() {
  for (auto& r : g_prof) {
    float ms = 0.f;
    cudaEventSynchronize(r.ev1);
    cudaEventElapsedTime(&ms, r.ev0, r.ev1);
    bool found = false;
    for (auto& a : g_agg)
      if (a.name == r.name) { a.launches++; a.ms += ms; found = true; break; }
    if (!found) g_agg.push_back({r.name, 1, (double)ms});
    g_ev_pool.push_back(r.ev0);
    g_ev_pool.push_back(r.ev1);
  }
  g_prof.clear();
}

// ------------------------------------------------------------------ breakpoints
// Phi^-1 by Acklam's rational approximation (relative error < 1.2e-9) refined
// by two Halley steps on the lower-tail CDF 0.5*erfc(-x/sqrt2); the upper half
// uses the symmetry Phi^-1(p) = -Phi^-1(1-p) (1-p is exact for p = k/card).
static double inv_phi_lower(double p) {  // p in (0, 0.5]
  static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                              -2.759285104469687e+02, 1.383577518672690e+02,
                              -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                              -1.556989798598866e+02, 6.680131188771972e+01,
                              -1.328068155288572e+01};
  static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                              -2.400758277161838e+00, -2.549732539343734e+00,
                              4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                              2.445134137142996e+00, 3.754408661907416e+00};
  double x;
  if (p < 0.02425) {
    double q = sqrt(-2.0 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else {
    double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  }
  if (p == 0.5) return 0.0;
  for (int it = 0; it < 2; ++it) {
    double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
    double u = e * sqrt(2.0 * M_PI) * exp(0.5 * x * x);
    x = x - u / (1.0 + 0.5 * x * u);
  }
  return x;
}

void host_cuts(int card, double* cuts) {
  for (int k = 1; k < card; ++k) {
    if (2 * k <= card)
      cuts[k - 1] = inv_phi_lower((double)k / card);
    else
      cuts[k - 1] = -inv_phi_lower((double)(card - k) / card);
  }
}

static float round_down_f(double v) {
  float f = (float)v;
  if ((double)f > v) f = nextafterf(f, -INFINITY);
  return f;
}
static float round_up_f(double v) {
  float f = (float)v;
  if ((double)f < v) f = nextafterf(f, INFINITY);
  return f;
}

// fp16 with directed rounding, by hand (host): normal numbers have 10 stored
// mantissa bits and exponents -14..15, subnormals are multiples of 2^-24.
uint16_t half_bits_dir(double v, int dir) {
  if (isnan(v)) return 0x7E00;
  if (isinf(v)) return v > 0 ? 0x7C00 : 0xFC00;
  const uint16_t sign = v < 0 ? 0x8000 : 0;
  const double a = fabs(v);
  // magnitude rounded toward zero (trunc) or away from zero (up), per dir and sign
  const bool away = (dir > 0) != (v < 0);
  if (a == 0.0) return sign;  // exact
  int e;
  frexp(a, &e);  // a = f * 2^e, f in [0.5, 1)
  int ex = e - 1;  // a in [2^ex, 2^(ex+1))
  if (ex < -14) ex = -14;
  const double quantum = ldexp(1.0, ex - 10);
  double m = a / quantum;  // exact (power-of-two scaling)
  double mi = away ? ceil(m) : floor(m);
  if (ex == -14 && mi < 1024.0) {  // subnormal (or the top of it rounding into 2^-14)
    return (uint16_t)(sign | (uint16_t)mi);
  }
  if (mi >= 2048.0) { mi = 1024.0; ex += 1; }  // mantissa overflow
  if (ex > 15) return away ? (uint16_t)(sign | 0x7C00) : (uint16_t)(sign | 0x7BFF);
  const uint16_t bits = (uint16_t)(((ex + 15) << 10) | ((int)mi - 1024));
  return (uint16_t)(sign | bits);
}

static int retain_pool_key;
void retain_pool() {
  once_per_device(&retain_pool_key, [](int dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    return cudaSuccess;
  });
}

// ------------------------------------------------------------------ per-device caches
static std::mutex g_once_mu;
static std::set<std::pair<const void*, int>> g_once_done;
static std::map<std::pair<const void*, int>, int> g_cached_int;

cudaError_t once_per_device(const void* key, const std::function<cudaError_t(int)>& f) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_once_mu);
  if (g_once_done.count({key, dev})) return cudaSuccess;
  e = f(dev);
  if (e == cudaSuccess) g_once_done.insert({key, dev});
  return e;
}

int cached_per_device(const void* key, const std::function<int(int)>& f) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_once_mu);
  auto it = g_cached_int.find({key, dev});
  if (it != g_cached_int.end()) return it->second;
  const int v = f(dev);
  g_cached_int[{key, dev}] = v;
  return v;
}

static int sms_key;
int device_sms() {
  return cached_per_device(&sms_key, [](int dev) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  });
}

// ------------------------------------------------------------------ workspace cache
struct WsEntry {
  int dev = 0;
  void* base = nullptr;
  size_t bytes = 0;
  cudaEvent_t done = nullptr;  // recorded when the last user released it
  bool busy = false;
  uint64_t gen = 0;
};
static std::mutex g_ws_mu;
static std::vector<WsEntry*> g_ws;
static std::atomic<uint64_t> g_ws_gen{1};

void* ws_acquire(size_t bytes, cudaStream_t st, void** handle, uint64_t* gen) {
  int dev = 0;
  cudaGetDevice(&dev);
  WsEntry* e = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (WsEntry* w : g_ws) {
      if (w->dev != dev || w->busy) continue;
      // prefer the smallest entry that is large enough, else the largest one (grown below)
      if (!e) e = w;
      else if (w->bytes >= bytes) { if (e->bytes < bytes || w->bytes < e->bytes) e = w; }
      else if (e->bytes < bytes && w->bytes > e->bytes) e = w;
    }
    if (!e) {
      e = new WsEntry;
      e->dev = dev;
      g_ws.push_back(e);
    }
    e->busy = true;
  }
  cudaError_t err = cudaSuccess;
  if (!e->done) err = cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming);
  else err = cudaStreamWaitEvent(st, e->done, 0);  // after the previous user's work
  if (err == cudaSuccess && e->bytes < bytes) {
    if (e->base) cudaFreeAsync(e->base, st);
    e->base = nullptr;
    e->bytes = 0;
    size_t want = bytes + bytes / 8;  // headroom: fewer regrowths across calls
    err = cudaMallocAsync(&e->base, want, st);
    if (err != cudaSuccess) {
      cudaGetLastError();
      want = bytes;
      err = cudaMallocAsync(&e->base, want, st);
    }
    if (err == cudaSuccess) {
      e->bytes = want;
      e->gen = g_ws_gen.fetch_add(1);
    } else {
      e->base = nullptr;
    }
  }
  if (err != cudaSuccess) {
    cudaGetLastError();
    set_error("workspace allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(err));
    std::lock_guard<std::mutex> lk(g_ws_mu);
    e->busy = false;
    return nullptr;
  }
  *handle = e;
  if (gen) *gen = e->gen;
  return e->base;
}

void ws_release(void* handle, cudaStream_t st) {
  WsEntry* e = static_cast<WsEntry*>(handle);
  if (!e) return;
  cudaEventRecord(e->done, st);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  e->busy = false;
}

void ws_free_all() {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_ws_mu);
  std::vector<WsEntry*> keep;
  for (WsEntry* w : g_ws) {
    if (w->busy) { keep.push_back(w); continue; }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(w->dev);
    if (w->base) cudaFree(w->base);
    if (w->done) cudaEventDestroy(w->done);
    cudaSetDevice(cur);
    delete w;
  }
  g_ws = keep;
  cudaGetLastError();
}

static std::mutex g_tab_mu;
static CardTables* g_tables[64] = {nullptr};  // per device

const CardTables* device_tables(int card) {
  if (card < 2 || card > 256 || (card & (card - 1))) {
    set_error("card must be a power of two in [2, 256] (got %d)", card);
    return nullptr;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64) {
    cuda_error(e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (!g_tables[dev]) {
    std::vector<CardTables> h(kNumCards);
    for (int ci = 0; ci < kNumCards; ++ci) {
      int cd = 2 << ci;
      double cuts[kMaxCard];
      host_cuts(cd, cuts);
      CardTables& t = h[ci];
      for (int c = 0; c < kMaxCard; ++c) {
        t.cuts_d[c] = (c < cd - 1) ? cuts[c] : INFINITY;
        t.cuts_f[c] = (c < cd - 1) ? (float)cuts[c] : INFINITY;
        float lo = (c == 0) ? -INFINITY : (c < cd ? round_down_f(cuts[c - 1]) : INFINITY);
        float hi = (c >= cd - 1) ? INFINITY : round_up_f(cuts[c]);
        t.lu[c] = make_float2(lo, hi);
        // fp16 region pair: L rounded down, U rounded up (from the fp64 cuts)
        const double Ld = (c == 0) ? -INFINITY : (c < cd ? cuts[c - 1] : INFINITY);
        const double Ud = (c >= cd - 1) ? INFINITY : cuts[c];
        const uint32_t nU = (uint32_t)(half_bits_dir(Ud, +1) ^ 0x8000u);  // -U16 (exact negation)
        const uint32_t L16 = half_bits_dir(Ld, -1);
        t.lu16[c] = make_uint2(nU | (nU << 16), L16 | (L16 << 16));
        t.lu16p[c] = nU | (L16 << 16);
      }
      for (int k = 0; k < kLutN; ++k) {
        const double x0 = -(double)kLutLo + (double)k / kLutScale;
        const double lo_edge = x0 - kLutMargin, hi_edge = x0 + 1.0 / kLutScale + kLutMargin;
        uint32_t lo = 0;
        float cut = 3.0e38f;  // "no cut in this bucket": finite, so |v - cut| never looks ambiguous
        for (int c = 0; c < cd - 1; ++c) {
          if (cuts[c] <= lo_edge) ++lo;
          else if (cuts[c] <= hi_edge) cut = (float)cuts[c];
        }
        uint32_t cb;
        memcpy(&cb, &cut, 4);
        t.lut[k] = make_uint2(cb, lo);
      }
    }
    CardTables* d = nullptr;
    e = cudaMalloc(&d, sizeof(CardTables) * kNumCards);
    if (e != cudaSuccess) {
      cuda_error(e, "cudaMalloc(tables)");
      return nullptr;
    }
    e = cudaMemcpy(d, h.data(), sizeof(CardTables) * kNumCards, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d);
      cuda_error(e, "cudaMemcpy(tables)");
      return nullptr;
    }
    g_tables[dev] = d;
  }
  int ci = 0;
  while ((2 << ci) != card) ++ci;
  return g_tables[dev] + ci;
}

}  // namespace paris

// ------------------------------------------------------------------ C ABI (misc)
namespace paris {
namespace {
// Read-only streaming probe (the read peak beside the copy peak):
// grid-stride 16-byte non-allocating loads folded into one word per thread.
__global__ void __launch_bounds__(512) k_read_probe(const uint4* __restrict__ p, int64_t n16, unsigned* out) {
  uint32_t x = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x9E3779B9u) out[0] = x;  // keeps the loads live; practically never taken
}

// fp16x2 FMA-pipe probe (the measured peak behind the batched LB's "alu" roofline):
// every thread runs 8 independent chains of fma.rn.f16x2; one instruction = 2 fp16 FMAs.
__global__ void __launch_bounds__(512) k_hfma2_probe(int iters, unsigned* out) {
  uint32_t a[8], b = 0x3C003C00u ^ (threadIdx.x & 1u), c = 0x00010001u;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0x3C003C00u + j + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
  }
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) x ^= a[j];
  if (x == 0x9E3779B9u) out[0] = x;  // keeps the chains live; practically never taken
}
}  // namespace
int g_variant[4] = {24, 1, 1, 2};
// PARIS_VARIANT="key=value,key=value" sets tuning variants at load time (profiling runs
// of unmodified scripts); paris_debug_set_variant overrides them later
static struct VariantEnv {
  VariantEnv() {
    const char* e = getenv("PARIS_VARIANT");
    while (e && *e) {
      int k = -1, v = 0, used = 0;
      if (sscanf(e, "%d=%d%n", &k, &v, &used) != 2) break;
      if (k >= 0 && k < 4) g_variant[k] = v;
      e += used;
      if (*e == ',') ++e;
    }
  }
} g_variant_env;
}  // namespace paris

extern "C" {

int32_t paris_debug_set_variant(int32_t key, int32_t value) {
  if (key < 0 || key >= 4) return -1;
  const int old = paris::g_variant[key];
  paris::g_variant[key] = value;
  return old;
}

int paris_debug_hfma2_probe(int32_t iters, int32_t blocks_per_sm, void* stream) {
  if (iters < 1 || blocks_per_sm < 1) return PARIS_EINVAL;
  static int sink_key;
  static unsigned* sinks[64] = {nullptr};
  const cudaError_t ea = paris::once_per_device(&sink_key, [](int dev) {
    return dev < 64 ? cudaMalloc(&sinks[dev], 4) : cudaErrorInvalidDevice;
  });
  if (ea != cudaSuccess) return paris::cuda_error(ea, "hfma2 probe sink");
  int dev = 0;
  cudaGetDevice(&dev);
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("hfma2_probe", paris::k_hfma2_probe, paris::device_sms() * blocks_per_sm, 512, 0,
                                  (cudaStream_t)stream, iters, sinks[dev]),
                     "hfma2 probe launch");
  return 0;
}

int paris_debug_read_probe(const void* p, int64_t bytes, void* stream) {
  if (!p || bytes < 16 || (reinterpret_cast<uintptr_t>(p) & 15)) return PARIS_EINVAL;
  const int sms = paris::device_sms();
  static int sink_key;
  static unsigned* sinks[64] = {nullptr};  // per device, allocated once
  const cudaError_t ea = paris::once_per_device(&sink_key, [](int dev) {
    return dev < 64 ? cudaMalloc(&sinks[dev], 4) : cudaErrorInvalidDevice;
  });
  if (ea != cudaSuccess) return paris::cuda_error(ea, "read probe sink");
  int dev = 0;
  cudaGetDevice(&dev);
  unsigned* sink = sinks[dev];
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("read_probe", paris::k_read_probe, sms * 4, 512, 0, (cudaStream_t)stream,
                                  reinterpret_cast<const uint4*>(p), bytes / 16, sink),
                     "read probe launch");
  return 0;
}


const char* paris_last_error(void) { return paris::g_err.c_str(); }

int32_t paris_version(void) { return 108; }

void paris_release_workspace(void) { paris::ws_free_all(); }

void paris_profile_enable(int32_t on) { paris::g_profile_on.store(on ? 1 : 0); }

void paris_profile_reset(void) {
  std::lock_guard<std::mutex> lk(paris::g_prof_mu);
  paris::drain_locked();
  paris::g_agg.clear();
}

int32_t paris_profile_read(paris_kernel_profile* out, int32_t max_entries) {
  std::lock_guard<std::mutex> lk(paris::g_prof_mu);
  paris::drain_locked();
  int32_t n = 0;
  for (auto& a : paris::g_agg) {
    if (out && n < max_entries) {
      memset(out[n].name, 0, sizeof out[n].name);
      strncpy(out[n].name, a.name.c_str(), sizeof out[n].name - 1);
      out[n].launches = a.launches;
      out[n].total_ms = a.ms;
    }
    ++n;
  }
  return n;
}

int64_t paris_launch_count(void) { return paris::g_launches.load(); }

// Test hook: fp16 bits of v rounded down (dir < 0) / up (dir > 0).
uint16_t paris_debug_half_dir(double v, int32_t dir) { return paris::half_bits_dir(v, dir); }

// Test hook: the library's own breakpoints (fp64), card-1 values.
int paris_debug_cuts(int32_t card, double* out) {
  if (card < 2 || card > 256 || (card & (card - 1)) || !out) return PARIS_ECONFIG;
  paris::host_cuts(card, out);
  return 0;
}

}  // extern "C"
