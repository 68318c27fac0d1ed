// Index LB pass as a tensor-core filter (k_gf; tcgen05 / TMEM, sm_100a only).
// Included by knn.cu inside its anonymous namespace (uses LbArgs, LbConsts, WarpBuf).
//
// MINDIST of a query PAA q against a SAX word is the distance from q to
// the box of the word's regions [L_j, U_j].  With a centre c_j and a half-width h_j per
// symbol ([L_j, U_j] inside [c_j - h_j, c_j + h_j]), x = q16 - c (q16 the fp16-rounded
// query PAA, |q - q16| <= eps) and any theta in (0, 1):
//     sqrt(sum_j d_j^2) + eps >= |x| - |h|           (triangle inequality)
//     (|x| - |h|)^2 >= (1 - theta) |x|^2 - (1/theta - 1) |h|^2
// so a series can only have MINDIST^2 <= tau if
//     F = sum_j [ c_j * (-2 q16_j) + (c_j^2 - h_j^2 / theta) ] + |q16|^2 - T / (1 - theta) <= 0,
//     T = (sqrt(tau / (len/w)) + eps)^2.
// F is bilinear in a per-series vector A = (c_j, g_j = c_j^2 - h_j^2/theta)_j -- a pure
// function of the symbols, one 4-byte table word per symbol -- and a per-query vector
// B = (-2 q16_j, 1)_j plus a per-query constant Q (a third k-step against a constant tile
// of ones).  So the 64 query slots of a pass are bounded against 128 series by THREE
// tcgen05.mma (M = 128, N = 64, K = 16, fp16 inputs, fp32 accumulators in TMEM) and the
// pass only needs the SIGN of each accumulator: survivors (about 2 per thousand) get the
// rigorous fp32 MINDIST from their symbols and are staged like k_lbi's candidates.
// Conservative by construction: c is exact in fp16, g and Q are rounded down, every
// product of two fp16 is exact, and Q carries the accumulation error bound kGfAccRel *
// (sum of |products|) (tests/test_gpu_gf.py measures the actual error of the unit).
// The filter decides nothing by itself: a candidate still needs its fp32 LB <= tau.
#pragma once

constexpr int kGfN = 64;            // query columns per MMA (= kMaxB)
constexpr int kGfK = 48;            // K: 16 x (c, g) + 16 for the per-query constant
constexpr int kGfRound = 128;       // series per warpgroup round (one 128-row MMA tile)
constexpr int kGfWG = 4;            // warpgroups per CTA, each an independent pipeline
constexpr int kGfWorkers = 128 * kGfWG;
constexpr int kGfThreads = kGfWorkers + 32 * kGfWG;  // + an issuing warp per warpgroup (MMAs, SAX copies)
constexpr int kGfStages = 8;        // SAX stages per warpgroup (queued survivors read their symbols later)
constexpr int kGfAhead = 3;         // rounds whose SAX copy is in flight
constexpr int kGfKeep = 3;          // a survivor waits at most this many rounds in its warp's queue
constexpr int kGfQ = 128;           // survivor queue entries per warp (ring)
static_assert(kGfAhead + kGfKeep + 2 <= kGfStages, "a stage is refilled only after its queued survivors are done");
constexpr uint32_t kGfStageBytes = 16 * kGfRound;
constexpr uint32_t kGfASbo = 528;   // 8-row group stride of an A tile (conflict-free row stores)
constexpr uint32_t kGfATile = 16 * kGfASbo;
constexpr uint32_t kGfBSbo = 6 * 128;
constexpr uint32_t kGfBBytes = (kGfN / 8) * kGfBSbo;
constexpr uint32_t kGfA2Sbo = 256;
constexpr uint32_t kGfA2Bytes = 16 * kGfA2Sbo;
constexpr double kGfAccRel = 1.0 / 131072.0;  // 2^-17 of sum |products| (measured: test_gpu_gf.py)

struct GfParams {
  uint32_t tabw[kMaxCard];          // half2(c, g) per symbol
  unsigned short B[kGfN * kGfK];    // fp16 bits, row per query slot
  unsigned ok;                      // 1: the filter applies to this pass; 0: fall back
  float theta, qmax, cmax, gabs;    // diagnostics
};

// ---- tcgen05 / TMEM wrappers (PTX ISA: tcgen05.*)
__device__ __forceinline__ void tc_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void wg_bar(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
// Shared-memory matrix descriptor, K-major, no swizzle: 8-row x 16-byte core matrices,
// lbo = bytes between the two K chunks of a k-step, sbo = bytes between 8-row groups.
__device__ __forceinline__ uint64_t gf_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46);
}
// 64 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld64(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]),
        "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]),
        "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]),
        "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
        "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
      : "r"(taddr)
      : "memory");
}
// non-blocking phase test of an mbarrier
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0u;
}
// one 2-D tile (box of the tensor map) global -> shared, completing on an mbarrier
__device__ __forceinline__ void tma_tile_2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sts_u4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// ---------------------------------------------------------------- per-pass parameters
// One CTA: the symbol table (c, g) and the B rows of the pass's query slots.
__global__ void __launch_bounds__(256)
k_gf_prep(LbArgs a, int card, GfParams* __restrict__ gp) {
  __shared__ double s_red[256];
  __shared__ double s_qmax, s_rbar, s_theta, s_cmax, s_gabs;
  __shared__ int s_nvalid;
  const int tid = threadIdx.x;
  const double seglen = (double)a.seglen_f;
  // (a) largest |query PAA| of the pass; mean PAA-space radius of the finite thresholds
  double qm = 0.0, rs = 0.0;
  int nv = 0;
  for (int i = tid; i < a.nb * a.w; i += 256) {
    const float2 q = a.g_q[(i / a.w) * kMaxW + (i % a.w)];
    qm = fmax(qm, fmax(fabs((double)q.x), fabs((double)q.y)));
  }
  for (int b = tid; b < a.nb; b += 256) {
    const float t = __uint_as_float(a.thr[b]);
    if (t >= 0.f && t < INFINITY) { rs += sqrt((double)t / seglen); ++nv; }
  }
  s_red[tid] = qm;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) { if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]); __syncthreads(); }
  if (tid == 0) s_qmax = s_red[0];
  __syncthreads();
  s_red[tid] = rs;
  if (tid == 0) s_nvalid = 0;
  __syncthreads();
  if (nv) atomicAdd(&s_nvalid, nv);
  for (int o = 128; o > 0; o >>= 1) { if (tid < o) s_red[tid] += s_red[tid + o]; __syncthreads(); }
  if (tid == 0) {
    s_rbar = s_nvalid > 0 ? s_red[0] / s_nvalid : 1.0;
    // theta = H0 / (R + H0), H0 a typical |h|: sqrt(w) x the half-width of a central region
    const float2 mid = a.tab->lu[card / 2];
    const double h0 = (card > 2 ? 0.75 * ((double)mid.y - (double)mid.x) : 0.5) * sqrt((double)a.w);
    double th = h0 / (s_rbar + h0);
    s_theta = fmin(fmax(th, 1e-3), 0.5);
  }
  __syncthreads();
  const double theta = s_theta, qmax = s_qmax;
  // (b) the table: centre (exact in fp16), half-width (outward), g rounded down
  double cabs = 0.0, gab = 0.0;
  if (tid < card) {
    const float2 lu = a.tab->lu[tid];
    double lo = (double)lu.x, hi = (double)lu.y;
    const double qedge = qmax * (1.0 + 1e-6) + 1e-6;  // every query PAA lies in [-qedge, qedge]
    const double hmin = card > 2 ? 4.0 * ((double)a.tab->lu[card / 2].y - (double)a.tab->lu[card / 2].x) : 0.25;
    if (tid == 0) lo = fmin(hi - 2.0 * hmin, -qedge);            // (-inf, U]: the part a query can be nearest to
    if (tid == card - 1) hi = fmax(lo + 2.0 * hmin, qedge);      // [L, +inf)
    const __half c16 = __double2half(0.5 * (lo + hi));
    const double c = (double)__half2float(c16);
    const double h = fmax(hi - c, c - lo) * (1.0 + 1e-12);
    const double g = c * c - h * h / theta * (1.0 + 1e-12);
    const __half g16 = __float2half_rd(__double2float_rd(g));
    gp->tabw[tid] = (uint32_t)__half_as_ushort(c16) | ((uint32_t)__half_as_ushort(g16) << 16);
    cabs = fabs(c);
    gab = fabs((double)__half2float(g16));
  } else {
    gp->tabw[tid] = 0u;
  }
  s_red[tid] = cabs;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) { if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]); __syncthreads(); }
  if (tid == 0) s_cmax = s_red[0];
  __syncthreads();
  s_red[tid] = gab;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) { if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]); __syncthreads(); }
  if (tid == 0) s_gabs = s_red[0];
  __syncthreads();
  // (c) B rows
  if (tid < kGfN) {
    const int b = tid;
    unsigned short* row = gp->B + b * kGfK;
    for (int k = 0; k < kGfK; ++k) row[k] = 0;
    const float t = b < a.nb ? __uint_as_float(a.thr[b]) : -1.f;
    double Q;
    if (t < 0.f) {
      Q = 60000.0;  // dummy slot: never passes
    } else {
      double qq = 0.0, q1 = 0.0, e2 = 0.0;
      for (int j = 0; j < a.w; ++j) {
        const float2 q = a.g_q[b * kMaxW + j];
        const __half q16 = __double2half(0.5 * ((double)q.x + (double)q.y));
        const double qh = (double)__half2float(q16);
        const double e = fmax(fabs((double)q.x - qh), fabs((double)q.y - qh));
        e2 += e * e;
        qq += qh * qh;
        q1 += fabs(qh);
        row[2 * j] = __half_as_ushort(__double2half(-2.0 * qh));  // exact
        row[2 * j + 1] = 0x3C00u;                                 // 1.0
      }
      if (t < INFINITY) {
        const double eps = sqrt(e2) * (1.0 + 1e-9);
        const double r = sqrt((double)t / seglen) * (1.0 + 1e-12) + eps;
        const double T = r * r / (1.0 - theta) * (1.0 + 1e-12);
        const double S = 2.0 * s_cmax * q1 + (double)a.w * s_gabs + fabs(qq - T);
        Q = qq - T - kGfAccRel * S - 1e-6;
      } else {
        Q = -60000.0;
      }
      Q = fmin(fmax(Q, -60000.0), 60000.0);
    }
    const __half qhi = __float2half_rd(__double2float_rd(Q));
    const double rem = Q - (double)__half2float(qhi);
    const __half qlo = __float2half_rd(__double2float_rd(rem));
    row[32] = __half_as_ushort(qhi);
    row[33] = __half_as_ushort(qlo);
  }
  if (tid == 0) {
    gp->ok = (qmax <= 16.0 && a.w == 16) ? 1u : 0u;
    gp->theta = (float)theta;
    gp->qmax = (float)qmax;
    gp->cmax = (float)s_cmax;
    gp->gabs = (float)s_gabs;
  }
}

struct GfShared {
  uint64_t full[kGfWG][kGfStages];
  uint64_t mma[kGfWG][2];
  uint64_t ready[kGfWG][2];
  uint32_t tmem_base;
  LbConsts c;
  float2 lu[kMaxCard];
  float2 q[kGfN * 17];  // row stride 17: lanes bounding different slots read different banks
  unsigned hist[kGfN * kNBC];
  uint32_t hq[kGfWorkers / 32][kGfQ];
  WarpBuf wb[kGfWorkers / 32];
};
constexpr size_t kGfSmem = 1024 /* alignment */ + kMaxCard * 128 /* table */ + kGfWG * kGfStages * kGfStageBytes +
                           kGfWG * 2 * kGfATile + kGfA2Bytes + kGfBBytes + sizeof(GfShared);
static_assert(kGfSmem <= 227 * 1024, "k_gf shared memory");

// Flush of a warp's staged candidates (keys hold sorted positions; ids through perm here).
__device__ void gf_flush(WarpBuf& wb, int nslots, const LbConsts& c, const LbArgs& a, unsigned* s_hist) {
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
    const unsigned pos = atomicAdd(&wb.cur[b], 1u);
    if ((int64_t)pos < a.cap) {
      const uint32_t id = a.perm ? __ldg(a.perm + key_id(key)) : key_id(key);
      a.cand[(size_t)b * a.cap + pos] = make_key(key_val(key), id);
      atomicAdd(&s_hist[b * kNBC + (lb_bin(key_val(key), c.scale[b]) >> 3)], 1u);
    }
  }
  __syncwarp();
  if (lane == 0) wb.n = 0;
  __syncwarp();
}

// a: LbArgs of the index path (a.perm set, a.sax = tile-major sorted SAX) or of the flat path (a.perm null,
// a.sax = [16][n], n % 16 == 0).  dump != nullptr (debug): the raw
// accumulators, dump[pos * 64 + slot], and no candidate work.
//
// Four warpgroups per CTA, each its own pipeline over 128-series rounds: iteration i builds
// the A tile of round i (a thread per series: 16 symbol bytes -> 16 table words -> 4 row
// stores), one warpgroup barrier, one thread issues the three MMAs of round i into TMEM
// buffer i & 1 and the SAX copy of round i + kGfAhead, and then the warpgroup reads the
// accumulators of round i - 1 (its MMA was issued a whole iteration earlier): 64 sign bits
// per series.  Survivors go to a per-warp queue (round, row, slot) and are bounded 32 at a
// time (a lane each), at most kGfKeep rounds later -- their symbols are still in the ring.
__global__ void __launch_bounds__(kGfThreads, 1)
k_gf(LbArgs a, const GfParams* __restrict__ gp, float* __restrict__ dump, int swap_desc,
     const __grid_constant__ CUtensorMap tmap) {
  if (gp->ok == 0u) return;
  extern __shared__ uint8_t dsm_raw[];
  const uint32_t S0 = (smem_u32(dsm_raw) + 1023u) & ~1023u;
  uint8_t* const gbase = dsm_raw - smem_u32(dsm_raw);  // generic pointer of shared address x: gbase + x
  const uint32_t s_tab = S0;
  const uint32_t s_stage = s_tab + kMaxCard * 128;
  const uint32_t s_A = s_stage + kGfWG * kGfStages * kGfStageBytes;
  const uint32_t s_A2 = s_A + kGfWG * 2 * kGfATile;
  const uint32_t s_B = s_A2 + kGfA2Bytes;
  GfShared& M = *reinterpret_cast<GfShared*>(gbase + ((s_B + kGfBBytes + 15u) & ~15u));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid >> 7, wt = tid & 127;
  const int nslots = kGfN;

  // ---- setup
  if (tid == 0) {
    for (int i = 0; i < kGfWG; ++i) {
      for (int s = 0; s < kGfStages; ++s) mbar_init(&M.full[i][s], 1);
      mbar_init(&M.mma[i][0], 1);
      mbar_init(&M.mma[i][1], 1);
      mbar_init(&M.ready[i][0], 4);
      mbar_init(&M.ready[i][1], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc_alloc(&M.tmem_base, 512);
  for (int i = tid; i < kMaxCard * 32; i += kGfThreads) sts_u32(s_tab + 4u * (uint32_t)i, gp->tabw[i >> 5]);
  for (int i = tid; i < kGfN * kGfK / 2; i += kGfThreads) {  // B: two halves (k even, k + 1) per word
    const int n = i / (kGfK / 2), k = 2 * (i % (kGfK / 2));
    const uint32_t v = (uint32_t)gp->B[n * kGfK + k] | ((uint32_t)gp->B[n * kGfK + k + 1] << 16);
    sts_u32(s_B + (uint32_t)(n >> 3) * kGfBSbo + (uint32_t)(k >> 3) * 128u + (uint32_t)(n & 7) * 16u + 2u * (uint32_t)(k & 7), v);
  }
  for (int i = tid; i < 128 * 8; i += kGfThreads) {  // A2: row r = (1, 1, 0, ...), 32 bytes
    const int r = i >> 3, wd = i & 7;
    sts_u32(s_A2 + (uint32_t)(r >> 3) * kGfA2Sbo + (uint32_t)(wd >> 2) * 128u + (uint32_t)(r & 7) * 16u + 4u * (uint32_t)(wd & 3),
            wd == 0 ? kHalf2One : 0u);
  }
  for (int i = tid; i < kMaxCard; i += kGfThreads) M.lu[i] = a.tab->lu[i];
  for (int i = tid; i < kGfN * 16; i += kGfThreads)
    M.q[(i >> 4) * 17 + (i & 15)] = (i >> 4) < a.nb ? a.g_q[(i >> 4) * kMaxW + (i & 15)] : make_float2(0.f, 0.f);
  for (int i = tid; i < kGfN * kNBC; i += kGfThreads) M.hist[i] = 0;
  if (warp < kGfWorkers / 32) {
    WarpBuf& wb0 = M.wb[warp];
    for (int b = lane; b < kMaxB; b += 32) wb0.cnt[b] = 0;
    if (lane == 0) wb0.n = 0;
  }
  lb_consts_init(a, nslots, &M.c);  // ends with __syncthreads
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A2, B visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = M.tmem_base;
  const int64_t nrounds = (a.n + kGfRound - 1) / kGfRound;
  const int64_t gstride = (int64_t)gridDim.x * kGfWG;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(kGfN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  constexpr int kRPT = kTS / kGfRound;  // rounds per index tile

  if (warp >= kGfWorkers / 32) {
    // ---- the issuing warp of warpgroup gg: once the group's four warps have written the A tile
    // of round i (and read the accumulators of round i - 2), the three MMAs of round i and the
    // SAX copy of round i + kGfAhead (into the stage of round i + kGfAhead - kGfStages: no warp
    // holds a survivor that old).  One 2-D tensor-map copy per stage: 16 rows x 128 bytes.  (One
    // warp serving all four groups was the bottleneck: ~580 cycles per round served.)
    const int gg = warp - kGfWorkers / 32;
    const int64_t gw2 = (int64_t)blockIdx.x * kGfWG + gg;
    const int cnt2 = gw2 < nrounds ? (int)((nrounds - gw2 + gstride - 1) / gstride) : 0;
    auto load = [&](int i) {
      const int64_t round = gw2 + (int64_t)i * gstride;
      const int st = i % kGfStages;
      // index: rows of [tile][16][2048] (whole tiles allocated); flat: [16][n], columns past n zero-filled
      const int c0 = a.perm ? (int)(round % kRPT) * kGfRound : (int)(round * kGfRound);
      const int c1 = a.perm ? (int)(round / kRPT) * 16 : 0;
      mbar_expect_tx(&M.full[gg][st], kGfStageBytes);
      tma_tile_2d(s_stage + (uint32_t)(gg * kGfStages + st) * kGfStageBytes, &tmap, c0, c1, &M.full[gg][st]);
    };
    const uint32_t la = swap_desc ? kGfASbo : 128u, sa = swap_desc ? 128u : kGfASbo;
    const uint32_t lb = swap_desc ? kGfBSbo : 128u, sb = swap_desc ? 128u : kGfBSbo;
    const uint32_t l2 = swap_desc ? kGfA2Sbo : 128u, s2 = swap_desc ? 128u : kGfA2Sbo;
    const uint64_t dB0 = gf_desc(s_B, lb, sb), dB1 = gf_desc(s_B + 256u, lb, sb), dB2 = gf_desc(s_B + 512u, lb, sb);
    const uint64_t dA2 = gf_desc(s_A2, l2, s2);
    if (lane == 0)
      for (int i = 0; i < kGfAhead && i < cnt2; ++i) load(i);
    for (int i = 0; i < cnt2; ++i) {
      mbar_wait(&M.ready[gg][i & 1], (unsigned)(i >> 1) & 1u);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t At = s_A + (uint32_t)(gg * 2 + (i & 1)) * kGfATile;
        const uint32_t d = tmem + (uint32_t)gg * 128u + (uint32_t)(i & 1) * kGfN;
        tc_mma_f16(d, gf_desc(At, la, sa), dB0, idesc, 0u);
        tc_mma_f16(d, gf_desc(At + 256u, la, sa), dB1, idesc, 1u);
        tc_mma_f16(d, dA2, dB2, idesc, 1u);
        tc_commit(&M.mma[gg][i & 1]);
        if (i + kGfAhead < cnt2) load(i + kGfAhead);
      }
      __syncwarp();
    }
  } else {
  WarpBuf& wb = M.wb[warp];
  uint32_t* const hq = M.hq[warp];
  const LbConsts& c = M.c;
  const int64_t gw = (int64_t)blockIdx.x * kGfWG + g;
  const int cnt = gw < nrounds ? (int)((nrounds - gw + gstride - 1) / gstride) : 0;  // this warpgroup's rounds
  const uint32_t my_stage0 = s_stage + (uint32_t)g * kGfStages * kGfStageBytes;
  const uint32_t my_A = s_A + (uint32_t)g * 2 * kGfATile;
  const uint32_t my_tmem = tmem + (uint32_t)g * 128u + ((uint32_t)(32 * (warp & 3)) << 16);

  // survivor queue (ring of kGfQ entries): entry = round index << 11 | lane << 6 | slot
  unsigned qhead = 0, qcount = 0;  // warp-uniform registers
  auto drain = [&](unsigned take) {  // bound `take` <= 32 queued survivors, a lane each
    const bool have = (unsigned)lane < take;
    const uint32_t e = have ? hq[(qhead + (unsigned)lane) % kGfQ] : 0u;
    const int b = (int)(e & 63u), ln = (int)((e >> 6) & 31u), ri = (int)(e >> 11);
    const uint32_t stage = my_stage0 + (uint32_t)(ri % kGfStages) * kGfStageBytes + (uint32_t)(32 * (warp & 3) + ln);
    float lbv = 0.f;
    bool cand = false;
    if (have) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t sym = lds_u8(stage + (uint32_t)j * kGfRound);
        const float2 lu = M.lu[sym];
        const float2 q = M.q[b * 17 + j];
        const float d = fmaxf(fmaxf(__fsub_rd(lu.x, q.y), __fsub_rd(q.x, lu.y)), 0.f);
        acc = __fmaf_rd(d, d, acc);
      }
      lbv = __fmul_rd(acc, a.seglen_f);
      cand = lbv <= c.thr[b];
    }
    const unsigned bal = __ballot_sync(0xffffffffu, cand);
    if (bal) {
      const int total = __popc(bal);
      if (wb.n + total > kWB) gf_flush(wb, nslots, c, a, M.hist);
      if (cand) {
        const int64_t pos = (gw + (int64_t)ri * gstride) * kGfRound + 32 * (warp & 3) + ln;
        const int e2 = wb.n + __popc(bal & ((1u << lane) - 1u));
        wb.key[e2] = make_key(lbv, (uint32_t)pos);
        wb.slot[e2] = (uint8_t)b;
        atomicAdd(&wb.cnt[b], 1u);
      }
      __syncwarp();
      if (lane == 0) wb.n += total;
      __syncwarp();
    }
    qhead = (qhead + take) % kGfQ;
    qcount -= take;
  };

  for (int i = 0; i <= cnt; ++i) {
    if (i < cnt) {
      const int st = i % kGfStages;
      const uint32_t stage = my_stage0 + (uint32_t)st * kGfStageBytes + (uint32_t)wt;
      mbar_wait(&M.full[g][st], (unsigned)(i / kGfStages) & 1u);
      // ---- A row of series wt of the round: the table words of its symbols
      const uint32_t tl = s_tab + 4u * (uint32_t)lane;
      const uint32_t rowa = my_A + (uint32_t)(i & 1) * kGfATile + (uint32_t)(wt >> 3) * kGfASbo + (uint32_t)(wt & 7) * 16u;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        uint32_t w0[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) w0[e] = lds_u32(tl + (lds_u8(stage + (uint32_t)(4 * kc + e) * kGfRound) << 7));
        sts_u4(rowa + (uint32_t)kc * 128u, w0[0], w0[1], w0[2], w0[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&M.ready[g][i & 1]);  // this warp: A(i) rows written, accumulators of round i - 2 read
    }
    if (i == 0) continue;
    // ---- epilogue of round i - 1: the sign of each accumulator
    const int ri = i - 1;
    mbar_wait(&M.mma[g][ri & 1], (unsigned)(ri >> 1) & 1u);
    tc_fence_after();
    uint32_t v[64];
    tc_ld64(my_tmem + (uint32_t)(ri & 1) * kGfN, v);
    const int64_t pos = (gw + (int64_t)ri * gstride) * kGfRound + 32 * (warp & 3) + lane;
    if (dump) {
      if (pos < a.n) {
#pragma unroll
        for (int k = 0; k < 64; ++k) dump[(size_t)pos * 64 + k] = __uint_as_float(v[k]);
      }
      continue;
    }
    uint32_t m0, m1;
    {
      uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // four independent chains of 16 sign bits
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        c0 = __funnelshift_l(v[k], c0, 1);
        c1 = __funnelshift_l(v[16 + k], c1, 1);
        c2 = __funnelshift_l(v[32 + k], c2, 1);
        c3 = __funnelshift_l(v[48 + k], c3, 1);
      }
      m0 = __brev((c0 << 16) | c1);  // bit k: slot k
      m1 = __brev((c2 << 16) | c3);  // bit k: slot 32 + k
    }
    if (pos >= a.n) { m0 = 0; m1 = 0; }
    // ---- queue the survivors, one per lane per turn
    while (__any_sync(0xffffffffu, (m0 | m1) != 0u)) {
      if (qcount + 32u > (unsigned)kGfQ) drain(32u);
      const bool have = (m0 | m1) != 0u;
      int b = 0;
      if (m0) { b = __ffs(m0) - 1; m0 &= m0 - 1; }
      else if (m1) { b = 32 + __ffs(m1) - 1; m1 &= m1 - 1; }
      const bool keep = have && b < a.nb;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) hq[(qhead + qcount + (unsigned)__popc(bal & ((1u << lane) - 1u))) % kGfQ] = ((uint32_t)ri << 11) | ((uint32_t)lane << 6) | (uint32_t)b;
      qcount += (unsigned)__popc(bal);
      __syncwarp();
    }
    // every warp bounds its queued survivors in the same rounds (every kGfKeep-th): a warp that
    // drained alone held up its warpgroup's next MMA while the other three waited
    if (ri % kGfKeep == kGfKeep - 1)
      while (qcount) drain(qcount < 32u ? qcount : 32u);
  }
  if (!dump) {
    while (qcount) drain(qcount < 32u ? qcount : 32u);
    gf_flush(wb, nslots, c, a, M.hist);
  }
  }  // worker warps
  tc_fence_before();
  __syncthreads();
  if (!dump)
    for (int i = tid; i < nslots * kNBC; i += kGfThreads) {
      const unsigned hv = M.hist[i];
      if (hv) atomicAdd(&a.hist[(i / kNBC) * kNB + (i % kNBC) * 8 + 7], hv);
    }
  if (warp == 0) {
    tc_fence_after();
    tc_dealloc(tmem, 512);
  }
}
