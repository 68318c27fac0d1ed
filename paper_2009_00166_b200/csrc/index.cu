// f1 -- paris_index_build: GPU-native iSAX organization of the SAX array
// (SURVEY §8(f) f1), the data-parallel analog of ParIS+'s index construction
// (Stage 3): series are grouped the way the iSAX tree groups them --
// the root splits on the first bit of every segment, deeper
// nodes on further bits -- here at uniform cardinality, by sorting on
// the bit-interleaved symbol key (bit 7 of segments 0..w-1, then bit 6, ...).
// Consecutive sorted series then share symbol prefixes, so the per-segment
// [min, max] symbol envelope of each block of kIdxBlock series is tight and the
// block's MINDIST (the iSAX node lower bound) prunes whole blocks (knn.cu,
// k_lbt MODE 2).  The leaf that would hold the query word (binary search on the
// key) is the approximate-search seed.
//
//   k_idx_aos    SoA [w][n] -> AoS [n][16] words + 64-bit keys + ids (smem transpose)
//   (CUB radix sort of (key, id) pairs -- a library sort, off the query path)
//   k_idx_gather sorted ids -> tile-major sorted SAX + block envelopes (smem transpose)
//
// Layout of the sorted array: tile-major SoA, [ceil(n/PARIS_INDEX_TILE)][16][PARIS_INDEX_TILE]:
// the 16 segment rows of 2048 consecutive sorted series are one contiguous 32 KB
// range, so the query kernel streams a tile with ONE bulk copy (16 row copies of
// 2 KB each capped the [w][n] layout's TMA ring near 2.7 TB/s).
#include "runtime.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace paris {

namespace {

constexpr int kIdxW = 16;
constexpr int kIdxTile = 256;

__global__ void __launch_bounds__(kIdxTile)
k_idx_aos(const uint8_t* __restrict__ sax, int64_t n, int shift, uint4* __restrict__ aos,
          uint64_t* __restrict__ keys, uint32_t* __restrict__ ids) {
  __shared__ __align__(16) uint8_t tile[kIdxW][kIdxTile];
  for (int64_t base = (int64_t)blockIdx.x * kIdxTile; base < n; base += (int64_t)gridDim.x * kIdxTile) {
    // rows: 16 x 256 bytes, 64 uint32 per row
    for (int t = threadIdx.x; t < kIdxW * (kIdxTile / 4); t += kIdxTile) {
      const int s = t / (kIdxTile / 4), c = t % (kIdxTile / 4);
      const int64_t i = base + 4 * c;
      uint32_t v = 0;
      if (i + 3 < n) v = *reinterpret_cast<const uint32_t*>(sax + (size_t)s * n + i);
      else
        for (int j = 0; j < 4; ++j)
          if (i + j < n) v |= (uint32_t)sax[(size_t)s * n + i + j] << (8 * j);
      reinterpret_cast<uint32_t*>(tile[s])[c] = v;
    }
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      uint8_t sym[kIdxW];
#pragma unroll
      for (int s = 0; s < kIdxW; ++s) sym[s] = tile[s][threadIdx.x];
      uint32_t wd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        wd[q] = sym[4 * q] | (sym[4 * q + 1] << 8) | (sym[4 * q + 2] << 16) | ((uint32_t)sym[4 * q + 3] << 24);
      aos[i] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
      keys[i] = isax_key16(sym, shift);
      ids[i] = (uint32_t)i;
    }
    __syncthreads();
  }
}

// sorted position j <- series perm[j]: SoA rows of the sorted array + envelopes
// of every kIdxBlock-series block ([blk][0][s] = min symbol, [blk][1][s] = max).
__global__ void __launch_bounds__(kIdxTile)
k_idx_gather(const uint4* __restrict__ aos, const uint32_t* __restrict__ perm, int64_t n,
             uint8_t* __restrict__ sax_sorted, uint8_t* __restrict__ env) {
  static_assert(kIdxTile % PARIS_INDEX_BLOCK == 0, "tile holds whole blocks");
  __shared__ __align__(16) uint8_t tile[kIdxW][kIdxTile];
  for (int64_t base = (int64_t)blockIdx.x * kIdxTile; base < n; base += (int64_t)gridDim.x * kIdxTile) {
    const int64_t j = base + threadIdx.x;
    if (j < n) {
      const uint4 v = aos[perm[j]];
      const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int s = 0; s < kIdxW; ++s) tile[s][threadIdx.x] = (uint8_t)(wd[s >> 2] >> (8 * (s & 3)));
    }
    __syncthreads();
    const int cnt = (int)imin64(kIdxTile, n - base);
    for (int t = threadIdx.x; t < kIdxW * (kIdxTile / 4); t += kIdxTile) {
      const int s = t / (kIdxTile / 4), c = t % (kIdxTile / 4);
      const int64_t i = base + 4 * c;  // whole uint32 stays inside one index tile (2048 % 4 == 0)
      const uint32_t v = reinterpret_cast<const uint32_t*>(tile[s])[c];
      const int64_t T = i / PARIS_INDEX_TILE, r = i % PARIS_INDEX_TILE;
      if (i < n)  // padding past n is left as is (never a candidate)
        *reinterpret_cast<uint32_t*>(sax_sorted + (size_t)T * kIdxW * PARIS_INDEX_TILE + (size_t)s * PARIS_INDEX_TILE + r) = v;
    }
    // envelopes: one thread per (block in tile, segment)
    constexpr int kBlocks = kIdxTile / PARIS_INDEX_BLOCK;
    if (threadIdx.x < kBlocks * kIdxW) {
      const int bl = threadIdx.x / kIdxW, s = threadIdx.x % kIdxW;
      const int j0 = bl * PARIS_INDEX_BLOCK;
      if (j0 < cnt) {
        const int j1 = min(cnt, j0 + PARIS_INDEX_BLOCK);
        unsigned mn = 255, mx = 0;
        for (int jj = j0; jj < j1; ++jj) {
          const unsigned c = tile[s][jj];
          mn = min(mn, c);
          mx = max(mx, c);
        }
        const int64_t blk = (base + j0) / PARIS_INDEX_BLOCK;
        env[(size_t)blk * 2 * kIdxW + s] = (uint8_t)mn;
        env[(size_t)blk * 2 * kIdxW + kIdxW + s] = (uint8_t)mx;
      }
    }
    __syncthreads();
  }
}

int sm_count_idx() { return device_sms(); }

}  // namespace

int index_build_impl(const uint8_t* sax, int64_t n, int w, int card, uint8_t* out_sax_sorted, uint32_t* out_perm,
                     uint8_t* out_env, cudaStream_t st) {
  if (!sax || !out_sax_sorted || !out_perm || !out_env) {
    set_error("paris_index_build: null pointer");
    return PARIS_EINVAL;
  }
  if (n < 1 || n >= (int64_t(1) << 31)) {
    set_error("paris_index_build: n=%lld out of range", (long long)n);
    return PARIS_EINVAL;
  }
  if (w != kIdxW || card < 2 || card > 256 || (card & (card - 1)) || (n % 16) != 0) {
    set_error("paris_index_build: unsupported (n=%lld, w=%d, card=%d); the index needs w == 16, n %% 16 == 0",
              (long long)n, w, card);
    return PARIS_ECONFIG;
  }
  int shift = 0;
  while ((card << shift) < 256) ++shift;
  retain_pool();
  // scratch: AoS words, keys in/out, ids in (ids out = out_perm), CUB temp
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, st);
  const size_t a_aos = 16 * (size_t)n, a_keys = 8 * (size_t)n, a_ids = 4 * (size_t)n;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  char* scratch = nullptr;
  const size_t total = al(a_aos) + 2 * al(a_keys) + al(a_ids) + al(temp_bytes);
  cudaError_t e = cudaMallocAsync((void**)&scratch, total, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("paris_index_build: scratch allocation of %zu bytes failed", total);
    return PARIS_ENOMEM;
  }
  uint4* aos = (uint4*)scratch;
  uint64_t* keys_in = (uint64_t*)(scratch + al(a_aos));
  uint64_t* keys_out = (uint64_t*)(scratch + al(a_aos) + al(a_keys));
  uint32_t* ids_in = (uint32_t*)(scratch + al(a_aos) + 2 * al(a_keys));
  void* temp = scratch + al(a_aos) + 2 * al(a_keys) + al(a_ids);
  const int grid = (int)imin64((n + kIdxTile - 1) / kIdxTile, (int64_t)sm_count_idx() * 8);
  int rc = PARIS_OK;
  e = PARIS_LAUNCH("index_aos", k_idx_aos, grid, kIdxTile, 0, st, sax, n, shift, aos, keys_in, ids_in);
  if (e == cudaSuccess) {
    ::paris::LaunchScope scope("index_sort", st);
    e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, ids_in, out_perm, (int)n, 0, 64, st);
  }
  if (e == cudaSuccess)
    e = PARIS_LAUNCH("index_gather", k_idx_gather, grid, kIdxTile, 0, st, aos, out_perm, n, out_sax_sorted, out_env);
  if (e != cudaSuccess) rc = cuda_error(e, "paris_index_build");
  cudaFreeAsync(scratch, st);
  return rc;
}

}  // namespace paris

extern "C" int paris_index_build(const uint8_t* sax, int64_t n, int32_t w, int32_t card, uint8_t* out_sax_sorted,
                                 uint32_t* out_perm, uint8_t* out_env, void* stream) {
  return paris::index_build_impl(sax, n, w, card, out_sax_sorted, out_perm, out_env, (cudaStream_t)stream);
}
