// f4 -- paris_merge_topk: exact merge of per-shard k-NN rows.
//
// A collection sharded by series-id range across R GPUs is searched shard by
// shard; every rank's rows are ascending (distance, global id) and hold that
// shard's k best.  The global k best are among the R*k gathered entries (each
// true member is in the top-k of its own shard), so one merge per query is exact.
// One CTA per query: the R*k entries are sorted in shared memory by (distance,
// id) -- a bitonic sort over index pairs -- in chunks when R*k exceeds the buffer.
#include "runtime.cuh"

namespace paris {
namespace {

constexpr int kMergeBuf = 2048;  // 32 KB of (distance, id) entries; k <= 1024 leaves >= 1024 per chunk
constexpr int kMergeThreads = 512;

struct Ent {
  float d;
  int64_t id;
};

__device__ __forceinline__ bool ent_less(const Ent& a, const Ent& b) {
  // NaN never occurs (finite inputs); +inf marks an empty slot and sorts last
  return a.d < b.d || (a.d == b.d && (uint64_t)a.id < (uint64_t)b.id);
}

__device__ void bitonic_ent(Ent* buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int idx = 2 * i - (i & (stride - 1));
        const int pr = idx + stride;
        const bool asc = (idx & size) == 0;
        const Ent a = buf[idx], c = buf[pr];
        if (ent_less(c, a) == asc) {
          buf[idx] = c;
          buf[pr] = a;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kMergeThreads)
k_merge_topk(const float* __restrict__ dist, const int64_t* __restrict__ idx, int R, int nq, int k,
             int64_t* __restrict__ out_idx, float* __restrict__ out_dist) {
  __shared__ Ent buf[kMergeBuf];
  const int q = blockIdx.x;
  const int64_t total = (int64_t)R * k;
  const Ent empty = {INFINITY, -1};
  for (int i = threadIdx.x; i < kMergeBuf; i += blockDim.x) buf[i] = empty;
  __syncthreads();
  const int chunk = kMergeBuf - k;
  for (int64_t off = 0; off < total; off += chunk) {
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) {
      Ent e = empty;
      const int64_t t = off + i;
      if (t < total) {
        const int r = (int)(t / k), j = (int)(t % k);
        const size_t at = ((size_t)r * nq + q) * k + j;  // gathered [R][nq][k]
        e.id = idx[at];
        e.d = (e.id >= 0) ? dist[at] : INFINITY;
        if (e.id < 0) e.id = -1;
      }
      buf[k + i] = e;
    }
    __syncthreads();
    bitonic_ent(buf, kMergeBuf);
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    out_idx[(size_t)q * k + j] = buf[j].id;
    out_dist[(size_t)q * k + j] = buf[j].d;
  }
}

}  // namespace
}  // namespace paris

extern "C" int paris_merge_topk(const float* dist, const int64_t* idx, int32_t R, int32_t nq, int32_t k,
                                int64_t* out_idx, float* out_dist, void* stream) {
  if (nq == 0) return PARIS_OK;
  if (!dist || !idx || !out_idx || !out_dist || R < 1 || nq < 0 || k < 1 || k > PARIS_MAX_K) {
    paris::set_error("paris_merge_topk: bad arguments (R=%d nq=%d k=%d)", R, nq, k);
    return PARIS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  PARIS_CHECK_LAUNCH(PARIS_LAUNCH("merge_topk", paris::k_merge_topk, nq, paris::kMergeThreads, 0, st, dist, idx,
                                  R, nq, k, out_idx, out_dist),
                     "merge launch");
  return PARIS_OK;
}
