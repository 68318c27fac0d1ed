/*
 * paris.h -- C ABI of libparis: the B200 (sm_100a) hot path of ParIS+ exact
 * whole-series k-NN search over an in-HBM iSAX summary array.
 *
 * Paper: Peng, Fatourou, Palpanas, "ParIS+: Data Series Indexing on Multi-Core
 * Architectures" (arXiv 2009.00166).  "P:N" cites line N of its LaTeX source
 * (PAPER.md); "S:N" a line of SPEC.md; readings (R#) are listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   - raw / queries: fp32, row-major [count][len], 16-byte aligned, finite values
 *     (non-finite input is the caller's responsibility).
 *   - sax: uint8 structure-of-arrays [w][n]: the symbol of segment s of series i
 *     is sax[s*n + i], in [0, card).  (The paper's SAX[p] array holds the word of
 *     series p at position p; it is stored segment-major here so a
 *     warp reads one segment of 128 consecutive series with one 128-byte request.)
 *   - Unless stated otherwise pointers are DEVICE pointers owned by the caller
 *     (e.g. torch tensors); the library never frees or retains them.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is ordered
 *     on it; see each call for when results are valid.
 *   - Return 0 on success or a negative PARIS_E* code; paris_last_error() gives a
 *     thread-local message.  On error nothing is promised about the outputs.
 *   - Supported: 1 <= n < 2^31 series, len % 4 == 0, 4 <= len <= 4096, w | len,
 *     1 <= w <= 64, card a power of two in [2, 256] (8-bit symbols P:294).
 *     Fast paths: len % 128 == 0 with (len/w) % 4 == 0 and len/w <= 128 for
 *     summarize; n % 16 == 0 for the SAX scans (other n run a byte-granular tail).
 */
#ifndef PARIS_H_
#define PARIS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARIS_OK 0
#define PARIS_EINVAL (-1)  /* null pointer, n < 1, nq < 0, k < 1, k > n (approximate search: k > PARIS_MAX_K) */
#define PARIS_ECONFIG (-2) /* unsupported (len, w, card) -- see the list above */
#define PARIS_ECUDA (-3)   /* a CUDA launch/runtime error; details in paris_last_error() */
#define PARIS_ENOMEM (-4)  /* scratch allocation failed */

#define PARIS_MAX_K 1024  /* largest k of the pruned search; 1024 < k <= n: every series' distance
                              is computed and the keys sorted (no pruning can pay there) */
#define PARIS_INDEX_BLOCK 64  /* series per envelope block of the index (paris_index_build) */
#define PARIS_INDEX_TILE 2048 /* series per tile of the index's tile-major sorted SAX array   */

/*
 * paris_summarize -- ConvertToSAX over a whole collection (IndexBulkLoading,
 * Alg2 line al2:cover): for every series i,
 *   PAA  paa[s] = mean of points [s*len/w, (s+1)*len/w)
 *   iSAX out_sax[s*n + i] = #{k in 1..card-1 : cut_k <= paa[s]},
 *        cut_k = Phi^-1(k/card) (N(0,1) equiprobable breakpoints, R2;
 *        a value on a cut goes to the upper region, R3).
 * The symbol is decided as if PAA were computed exactly: an fp32 PAA whose
 * rounding-error bound straddles a cut is recomputed in fp64.
 *   raw      [n][len] fp32, device OR host memory (pinned or pageable; 16-byte aligned)
 *   out_sax  device [w][n] uint8 (caller-allocated, n*w bytes)
 * Host raw (the paper's raw data is not in memory): rows are
 * streamed in 256 MB chunks through two device staging buffers, the copy of chunk
 * c+1 overlapping the summarize of chunk c (the Coordinator's double buffer,
 * P:459-465, 477-483); pinned memory makes the copies asynchronous.  The host
 * buffer must stay valid until `stream` completes.
 * Asynchronous: returns after enqueueing; results valid once `stream` completes.
 */
int paris_summarize(const float* raw, int64_t n, int32_t len, int32_t w, int32_t card,
                    uint8_t* out_sax, void* stream);

/*
 * paris_summarize_file -- paris_summarize of a raw collection stored in a FILE (the paper's
 * setting: raw data on disk, index construction reading it sequentially):
 * n rows of len fp32 starting at byte `offset` of `path`.  A reader thread preads 256 MB
 * chunks into three pinned host buffers while the calling thread copies each chunk to a
 * device staging buffer and summarizes it (the Coordinator's double buffer); direct_io != 0
 * asks for O_DIRECT (the disk's own bandwidth, no page cache; needs offset % 4096 == 0,
 * else buffered reads).  out_bf16 (optional, device [n][len] bf16 bits, len % 8 == 0): the
 * bf16 copy of paris_raw_bf16 built from the same staged chunks.  Returns once the whole
 * file has been read (results valid when `stream` completes).  PARIS_EINVAL for an
 * unreadable or short file.
 */
int paris_summarize_file(const char* path, int64_t offset, int64_t n, int32_t len, int32_t w, int32_t card,
                         uint8_t* out_sax, uint16_t* out_bf16, int32_t direct_io, void* stream);

/*
 * paris_map_raw_file / paris_unmap_raw_file -- map `bytes` of a raw file (from a page-aligned
 * `offset`) read-only and register the mapping with CUDA (cudaHostRegisterReadOnly; its
 * pages are pinned, so the file must fit in host RAM): *out_ptr is then a host raw pointer
 * the k-NN calls accept -- the candidates' rows are read straight from the
 * file's pages over PCIe (the RDC workers' random reads of the raw file).
 */
int paris_map_raw_file(const char* path, int64_t offset, int64_t bytes, void** out_ptr);
int paris_unmap_raw_file(void* ptr, int64_t bytes);

/*
 * paris_knn_exact -- exact k-NN under Euclidean distance (k-NN per
 * S:406-414) following ParIS+ ExactSearch (Alg9):
 *   1. BSF seed (approximate search analog, R8): the lower bound over
 *      a sample of the SAX array ranks seed series; their true distances give an
 *      upper bound tau_seed on the k-th NN distance.
 *   2. LBC pass (Alg10): MINDIST_PAA_iSAX (R1) for every
 *      series' word, up to 16 queries per read of the SAX array (packed fp16 with
 *      a rigorous error budget as a filter); a series is a candidate iff its
 *      rigorous (round-down fp32) LB^2 <= tau_seed^2 (rounded up).  Candidates
 *      are compacted per query.
 *   3. RDC pass (Alg11): candidates are refined in LB order, each
 *      re-checked against the live BSF before its raw series is read; true squared
 *      ED with early abandoning; the BSF (k-th best) is shared through atomics.
 *   4. Result: ascending (distance, id); ties go to the lower id (R6).
 *   raw       [n][len] fp32: device memory, or page-locked host memory (cudaHostAlloc /
 *             cudaHostRegister) -- then only the seeds' and candidates' rows
 *             cross PCIe; pageable host raw -> PARIS_EINVAL
 *   sax       device [w][n] uint8 (paris_summarize); host sax -> PARIS_EINVAL
 *   queries   [nq][len] fp32                 -- device OR host memory
 *   out_idx   [nq][k] int64 series ids       -- device OR host memory
 *   out_dist  [nq][k] fp32 Euclidean (rooted) distance -- device OR host memory
 * queries/out_idx/out_dist may be host pointers (pageable or pinned): the library
 * then stages them through device memory on `stream`.
 * Asynchronous: the call enqueues its work on `stream` and returns without waiting;
 * outputs are final once `stream` completes (host outputs: pinned ones are copied back
 * stream-ordered; pageable ones block the call until the copy is done, as
 * cudaMemcpyAsync does).  The host never reads device state: a query whose candidate
 * list outgrew its buffer (more than max(65536, n/32) candidates, n/16 for k > 1) is
 * completed on the device by a fused LB -> refine scan seeded with its first-pass
 * result (gated kernels that exit at once when no query overflowed).
 * Scratch (candidate lists, up to B * 8 * max(65536, n/32) bytes, with B = 16 queries
 * per pass on the flat path, 64 on the index path) comes from a workspace cached per
 * device (grown on demand, reused across calls, each reuse ordered after the previous
 * call's work by an event): no allocation and no synchronization in the steady state.
 * paris_release_workspace() frees it.  With `stats` (paris_knn_exact_ex) the call
 * synchronizes to read the counters.  nq == 0 is a no-op.
 */
int paris_knn_exact(const float* raw, const uint8_t* sax, int64_t n, const float* queries,
                    int32_t nq, int32_t k, int64_t* out_idx, float* out_dist, int32_t len,
                    int32_t w, int32_t card, void* stream);

/*
 * paris_index_build -- GPU-native iSAX organization of a SAX array (SURVEY §8(f)
 * f1; the data-parallel analog of ParIS+'s index construction, Stage 3,
 * P:396-402).  Series are ordered the way the iSAX tree groups them (root split
 * on the first bit of every segment; deeper nodes on further
 * bits) at uniform cardinality: by the key interleaving bits 7..4 of
 * the 16 symbols (card < 256: symbols scaled to 8 bits), ties by id.
 *   sax            device [w][n] uint8 (paris_summarize)
 *   out_sax_sorted device [ceil(n/PARIS_INDEX_TILE)][w][PARIS_INDEX_TILE] uint8 (tile-major
 *                  SoA; the last tile padded): the symbol of segment s of sorted series j
 *                  is out_sax_sorted[(j/T)*w*T + s*T + j%T] = sax[s*n + perm[j]], T = PARIS_INDEX_TILE
 *   out_perm       device [n] uint32: series id at sorted position j
 *   out_env        device [ceil(n/PARIS_INDEX_BLOCK)][2][w] uint8: per block of
 *                  PARIS_INDEX_BLOCK consecutive sorted series, the min ([blk][0][s])
 *                  and max ([blk][1][s]) symbol of segment s (the node envelope)
 * Requires w == 16, n % 16 == 0 (PARIS_ECONFIG otherwise).  Asynchronous on
 * `stream`; scratch (~36 bytes per series) is stream-ordered.
 */
int paris_index_build(const uint8_t* sax, int64_t n, int32_t w, int32_t card, uint8_t* out_sax_sorted,
                      uint32_t* out_perm, uint8_t* out_env, void* stream);

/* Tunables for paris_knn_exact_ex (0 = library default). */
typedef struct paris_knn_config {
  int32_t batch;        /* queries per SAX pass: 1..16 (flat, default 16), 1..64 (index, default 64) */
  int32_t seed_div;     /* seed sample = n / seed_div series (default 16) */
  int32_t wave_a;       /* k = 1: candidates per query refined in the first (lowest-LB) wave; default 2048 */
  int32_t reserved[5];  /* tuning/test hooks: [0] = 1 forces the direct-load LB kernels;
                           [1] = 1: the k = 1 refine walks bucket-sorted lists (K5 scatter)
                           instead of taking its two LB waves from the unsorted lists;
                           [2] index mode: seed series around the leaf (0 = max(1024 (2048 from 5e7 series), 32k) up to 4096; 64 when
                           raw is host memory);
                           [3] = 1 seeds every batch from the rows already in out_idx/out_dist
                           (device outputs; experiments with an ideal BSF);
                           [4] > 0: candidate-buffer capacity per query (test hook: forces the
                           overflow fallback; default max(65536, n/32 | n/16 for k > 1) grown
                           to a budget per candidate array of 1/8 of the free device memory,
                           clamped to [2, 16] GB) */
  const float* tau_in;  /* optional DEVICE [nq]: per query, an upper bound of its k-th NN
                           distance from outside the call (+inf = none) -- e.g. the minimum
                           over the shards of a sharded collection of their approximate
                           answers' k-th distances (paris_knn_approx); the
                           search then prunes against min(its own seed, tau_in) and rows
                           with no series within the bound come back as id -1 / +inf.
                           NULL = none. */
} paris_knn_config;

/* Per-query counters (host memory, arrays of nq), filled by paris_knn_exact_ex. */
typedef struct paris_knn_stats {
  int64_t* candidates;  /* series whose LB passed tau_seed (Alg10 list length)       */
  int64_t* refined;     /* raw series read and distance computed (Alg11 line al9:rcal) */
  float* tau_seed;      /* seed BSF distance (rooted)                                 */
  int64_t* lb_blocks;   /* index mode: PARIS_INDEX_BLOCK-series blocks whose envelope
                           bound passed (their series' LBs were computed); 0 otherwise */
  int64_t* bsf_updates; /* paris_knn_nb: updates of the workers' private BSF copies   */
  int64_t* raw16_rows;  /* paris_knn_index_x: bf16 rows read by the refinement pre-filter
                           (refined = the fp32 rows read after it)                     */
  int64_t* paa_rows;    /* paris_knn_index_aux: fp16 PAA rows read by the PAA pre-filter */
} paris_knn_stats;

/* Same as paris_knn_exact with tunables and optional stats (either may be NULL). */
int paris_knn_exact_ex(const float* raw, const uint8_t* sax, int64_t n, const float* queries,
                       int32_t nq, int32_t k, int64_t* out_idx, float* out_dist, int32_t len,
                       int32_t w, int32_t card, void* stream, const paris_knn_config* config,
                       paris_knn_stats* stats);

/*
 * paris_knn_index -- exact k-NN like paris_knn_exact, over an index built by
 * paris_index_build (same results; raw stays in its original order):
 *   1. approximate search: the query's own word is located in the
 *      sorted array (the leaf it would be inserted into); the true distances of
 *      the 1024 series around it (configurable) give tau_seed;
 *   2. LBC pass over the sorted SAX array: each block's envelope MINDIST (the
 *      iSAX node bound) is computed first and only the queries the block can hold
 *      candidates for are evaluated on its series;
 *   3-4. as paris_knn_exact (candidate ids are the original series ids).
 * Requires w == 16 and n % 16 == 0.
 */
int paris_knn_index(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                    int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist,
                    int32_t len, int32_t w, int32_t card, void* stream);

int paris_knn_index_ex(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                       int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx,
                       float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                       const paris_knn_config* config, paris_knn_stats* stats);

/*
 * paris_knn_approx / paris_knn_index_approx -- approximate k-NN (ParIS+ approximate
 * search): only step 1 of paris_knn_exact / paris_knn_index -- for every
 * query the k best of the seed series (flat: the LB-best series of a prefix sample;
 * index: the series around the leaf the query's word would be inserted into), with
 * their true fp32 distances, ascending (distance, id); -1 / +inf pads a row when fewer
 * than k seeds exist.  The k-th distance bounds the exact k-th NN distance from above,
 * which is what a sharded search exchanges (paris_knn_config.tau_in).  Same arguments,
 * conventions and asynchrony as the exact calls (config: batch / seed_div /
 * reserved[2] apply).
 */
int paris_knn_approx(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int32_t nq, int32_t k,
                     int64_t* out_idx, float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                     const paris_knn_config* config);
int paris_knn_index_approx(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env,
                           int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist,
                           int32_t len, int32_t w, int32_t card, void* stream, const paris_knn_config* config);

/*
 * paris_raw_bf16 -- a bf16 copy of the raw collection for the refinement pre-filter
 * of paris_knn_index_x (a B200 addition, not in the paper):
 *   raw  device [n][len] fp32, out device [n][len] bf16 bits (round to nearest even),
 *   caller-allocated (2*n*len bytes); both 16-byte aligned, len % 8 == 0.
 * Asynchronous on `stream`.
 */
int paris_raw_bf16(const float* raw, int64_t n, int32_t len, uint16_t* out, void* stream);

/*
 * paris_knn_index_x -- paris_knn_index_ex with the bf16 pre-filter: for k = 1 the
 * refinement first bounds each candidate's true distance from below with its bf16
 * row (half the bytes): ED(q, x) >= ED(q, x~) - rho ||x~||, rho = 2^-8 (1 + 2^-7),
 * with fp32 error margins and directed roundings; a candidate whose bound exceeds
 * the live BSF is dropped without reading its fp32 row (same exact results).
 *   raw_bf16  device [n][len] bf16 (paris_raw_bf16 of `raw`), 16-byte aligned,
 *             len % 8 == 0; NULL = paris_knn_index_ex.  k > 1 ignores it, and so
 *             does raw in device memory with len < 256 (no gain on short rows).
 */
int paris_knn_index_x(const float* raw, const uint16_t* raw_bf16, const uint8_t* sax_sorted, const uint32_t* perm,
                      const uint8_t* env, int64_t n, const float* queries, int32_t nq, int32_t k, int64_t* out_idx,
                      float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                      const paris_knn_config* config, paris_knn_stats* stats);

/*
 * paris_paa_f16 -- the PAA of every raw series at w2 segments (w2 | len, w2 % 8 == 0,
 * w2 <= 256), each mean computed in fp64 and rounded to nearest fp16 (|mean| >= 65000 -> NaN,
 * which disables the filter for that series): out device [n][w2] fp16 bits, 16-byte aligned
 * (a B200 addition, not in the paper: 2 w2 bytes per series -- 128 B at w2 = 64 against 1 KB of
 * raw -- for the PAA pre-filter of paris_knn_index_aux).  Asynchronous on `stream`.
 */
int paris_paa_f16(const float* raw, int64_t n, int32_t len, int32_t w2, uint16_t* out, void* stream);

/* Refinement pre-filters for paris_knn_index_aux (NULL members = off). */
typedef struct paris_refine_aux {
  const uint16_t* raw_bf16; /* [n][len] bf16 copy of raw (paris_raw_bf16), or NULL                */
  const uint16_t* paa16;    /* [n][w2] fp16 PAA of raw (paris_paa_f16), or NULL                     */
  int32_t w2;               /* segments of paa16: 32 or 64 (w2 | len)                              */
  int32_t reserved;
} paris_refine_aux;

/*
 * paris_knn_index_aux -- paris_knn_index_ex with refinement pre-filters (k = 1, len <= 256):
 * a candidate that passes the LB test against the live BSF first meets the PAA lower bound
 * ED(q, x) >= sqrt(len/w2) ||PAA_w2(q) - PAA_w2(x)|| (Keogh's PAA bound; the fp16 rounding of
 * the stored PAA bounded rigorously) -- the w2 > w resolution prunes most of the
 * candidates the iSAX bound let through, reading 2 w2 bytes instead of the raw row -- then, if
 * given, the bf16 bound of paris_knn_index_x, then the exact fp32 distance.  Same exact
 * results as paris_knn_index; k > 1 ignores the filters.  Stats: paa_rows.
 */
int paris_knn_index_aux(const float* raw, const uint8_t* sax_sorted, const uint32_t* perm, const uint8_t* env, int64_t n,
                        const float* queries, int32_t nq, int32_t k, int64_t* out_idx, float* out_dist, int32_t len,
                        int32_t w, int32_t card, void* stream, const paris_refine_aux* aux,
                        const paris_knn_config* config, paris_knn_stats* stats);

/*
 * paris_knn_nb -- exact 1-NN with nb-ParIS+ (Alg7-Alg8,
 * P:1158-1246): the same seed as paris_knn_exact (approximate search analog),
 * then SAX is split into contiguous parts, one per DistComp worker (a warp);
 * each worker keeps its own copy of the BSF per query (no communication while
 * scanning), computes the lower bound of every word of its part and refines a
 * series at once when its bound is below that copy; the answer is the minimum
 * over the copies.  The ablation of ParIS+'s shared candidate list: stats report
 * raw series read (refined) and BSF-copy updates (bsf_updates) -- the quantities
 * of the paper's fig:notpruned.  k = 1 (out rows [nq][1]);
 * w == 16, n % 4 == 0.  Same pointer/stream conventions as paris_knn_exact.
 */
int paris_knn_nb(const float* raw, const uint8_t* sax, int64_t n, const float* queries, int32_t nq,
                 int64_t* out_idx, float* out_dist, int32_t len, int32_t w, int32_t card, void* stream,
                 const paris_knn_config* config, paris_knn_stats* stats);

/*
 * paris_merge_topk -- exact merge of per-shard k-NN rows: a
 * collection sharded by series-id range over R GPUs is searched per shard; the
 * gathered rows dist/idx [R][nq][k] (each ascending by (distance, global id);
 * id < 0 = empty) hold the global k best of every query, which are written to
 * out_idx/out_dist [nq][k] ascending by (distance, id).  Device pointers,
 * asynchronous on `stream`.  R >= 1, 1 <= k <= PARIS_MAX_K.
 */
int paris_merge_topk(const float* dist, const int64_t* idx, int32_t R, int32_t nq, int32_t k, int64_t* out_idx,
                     float* out_dist, void* stream);

/* Free the cached device workspace of the k-NN calls (all devices; synchronizes the
 * device).  The next call allocates it again. */
void paris_release_workspace(void);

/* Thread-local text of the last failure (never NULL). */
const char* paris_last_error(void);

/* ABI version (major*100 + minor). */
int32_t paris_version(void);  /* 108: paris_debug_set_variant (tuning A/B hook);
                                 107: paris_paa_f16, paris_knn_index_aux (PAA pre-filter);
                                 106: asynchronous k-NN calls, device-side overflow, paris_release_workspace,
                                 paris_knn_approx / paris_knn_index_approx, paris_knn_config.tau_in */

/* Test hook: the library's own fp64 breakpoints cut_1..cut_{card-1} (R2) into
 * out[0..card-2] (host memory).  PARIS_ECONFIG for a bad card. */
int paris_debug_cuts(int32_t card, double* out);

/* Measurement hook: stream `bytes` of device memory at p with read-only 16-byte
 * loads (no writes) -- the read-only HBM peak beside MEASURED_PEAKS.json's copy
 * peak (bench.py times it).  Asynchronous on `stream`. */
int paris_debug_read_probe(const void* p, int64_t bytes, void* stream);

/* Measurement hook: the fp16x2 FMA-pipe peak -- device_sms * blocks_per_sm CTAs of 512
 * threads, each thread `iters` x 8 independent fma.rn.f16x2 (2 fp16 FMAs each); bench.py
 * times it for the batched LB's "alu" roofline denominator.  Asynchronous on `stream`. */
int paris_debug_hfma2_probe(int32_t iters, int32_t blocks_per_sm, void* stream);

/* Tuning hook (A/B of kernel variants inside one process; results are identical, only
 * the speed differs): key 0 = consumer warps of the index LB pass (24 (default) or 30),
 * key 1 = batch-1 flat LB (0: register-prefetch k_lb1,
 * 1 (default): TMA ring k_lb1t), key 2 = pre-filtered k = 1 refine (0: k_refine1q, a warp per
 * (query, chunk run); 1 (default): k_refine1m, one chunk stream over the batch), key 3 = the LB pass as a
 * tensor-core filter (k_gf: 64 query slots per pass, tcgen05.mma + the sign of the accumulators, fp32 MINDIST for
 * the survivors; a pass falls back to the fp16 kernels when a query PAA exceeds 16 in magnitude): 2 (default) = on
 * the flat path (paris_knn_exact; 2.6x at 1e8 x 256), 1 = on the index path too (slower there than the block pass +
 * k_lbi), 0 = off.  Returns the previous value, -1 for an unknown key.
 * Process-global; not synchronized with calls in flight on other host threads. */
int32_t paris_debug_set_variant(int32_t key, int32_t value);

/* Test hook for the tensor-core filter of the index LB pass (key 3 below; k_gf, DESIGN.md f1):
 * the raw fp32 accumulators out[pos * 64 + slot] of the three tcgen05.mma per 128 series,
 *   sum_j half(tabw[sym_j]).lo * B[slot][2j] + half(tabw[sym_j]).hi * B[slot][2j+1] + B[slot][32] + B[slot][33],
 * for a caller-made symbol table tabw (256 words, half2) and B matrix (64 rows x 48 fp16,
 * columns 34..47 zero) over the tile-major sorted SAX array of n series (w = 16).  All
 * pointers device; out holds n * 64 floats.  swap_desc != 0 swaps the descriptor's leading /
 * stride byte offsets (diagnosis).  Synchronizes `stream`. */
int paris_debug_gf_mma(const uint8_t* sax_sorted, int64_t n, const uint32_t* tabw, const uint16_t* bmat, float* out,
                       int32_t swap_desc, void* stream);

/* Test hook: IEEE binary16 bits of v rounded toward -inf (dir < 0) or +inf
 * (dir > 0) -- the directed rounding behind the batched fp16 lower bound. */
uint16_t paris_debug_half_dir(double v, int32_t dir);

/*
 * Launch accounting / per-kernel device time (for benchmarks).
 *   paris_profile_enable(1): every kernel launch is bracketed by CUDA events on its
 *   stream; paris_profile_read() synchronizes on those events and returns, per
 *   kernel name, the launch count and the summed device milliseconds.
 *   paris_launch_count() counts every kernel launched by the library (always on).
 */
typedef struct paris_kernel_profile {
  char name[48];
  int64_t launches;
  double total_ms;
} paris_kernel_profile;

void paris_profile_enable(int32_t on);
void paris_profile_reset(void);
int32_t paris_profile_read(paris_kernel_profile* out, int32_t max_entries);
int64_t paris_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* PARIS_H_ */
