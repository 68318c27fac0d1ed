/*
 * ParIS+ exact k-NN hot path -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * Plain, slow, single-threaded, double precision.  Written from the paper
 * (/root/reference/PAPER.md, "P:N" = line N; SPEC.md "S:N" only for the readings
 * SURVEY.md §8(c) adopts).  It shares no code, header, table or constant with
 * the CUDA path (paper_2009_00166_b200/csrc); only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Functions, each following one passage:
 *   oracle_cuts            breakpoints Phi^-1(k/card)            P:290-297 (+ reading 2)
 *   oracle_paa             PAA segment means
 *   oracle_sax             iSAX symbol of each PAA value          P:290-297, 563-565 (+ reading 3)
 *   oracle_summarize       ConvertToSAX over a collection -> SAX[p]  Alg2 P:577-599 line al2:cover
 *   oracle_lb_table        MINDIST_PAA_iSAX dictionaries          P:1107-1123 (+ reading 1)
 *   oracle_lb2             lower bound of one (query, word) pair
 *   oracle_ed2             squared Euclidean distance             P:219 (+ reading 4)
 *   oracle_ed2_abandon     ED with early abandoning               north_star
 *   oracle_knn_bruteforce  plain k-NN definition (ground truth)
 *   oracle_knn_pruned      LB-pruned exact search (Alg8 logic,
 *                          one worker, BSF = k-th best)
 *
 * Every function is pinned by tests/test_oracle_*.py against closed forms,
 * library routines, brute force and invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- breakpoints
 * "divides the (y-axis) space in different regions".  Reading 2 (SURVEY
 * §8(c)): N(0,1) equiprobable quantiles, cut_k = Phi^-1(k/card), k = 1..card-1.
 * Solved by plain bisection until the bracket stops shrinking (1 ulp), on the
 * form of the CDF that is accurate in double there (all three are the same
 * function Phi in exact arithmetic):
 *   centre (1/4 <= p <= 3/4):  Phi(x) - 1/2 = 0.5*erf(x/sqrt2)  vs  p - 1/2
 *   lower tail (p < 1/4):      Phi(x) = 0.5*erfc(-x/sqrt2)       vs  p
 *   upper tail (p > 3/4):      1 - Phi(x) = 0.5*erfc(x/sqrt2)    vs  1 - p
 * (p - 1/2 and 1 - p are exact for p = k/card).  cuts[k-1] = cut_k.
 */
/* g(x) = signed CDF residual at x for p = k/card, increasing in x, zero at the quantile. */
static double residual(double x, int k, int card) {
  if (4 * k < card) return 0.5 * erfc(-x / sqrt(2.0)) - (double)k / (double)card;
  if (4 * k > 3 * card) return (double)(card - k) / (double)card - 0.5 * erfc(x / sqrt(2.0));
  return 0.5 * erf(x / sqrt(2.0)) - (double)(2 * k - card) / (double)(2 * card);
}

int oracle_cuts(int card, double* cuts) {
  if (card < 2 || card > 256 || (card & (card - 1))) return -1;
  for (int k = 1; k < card; ++k) {
    double lo = -40.0, hi = 40.0;
    for (int it = 0; it < 4000; ++it) {
      double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi || hi - lo < 1e-300) break; /* 1 ulp (or below any cut's scale) */
      if (residual(mid, k, card) < 0.0) lo = mid; else hi = mid;
    }
    /* the bracket endpoint with the smaller residual */
    cuts[k - 1] = (fabs(residual(lo, k, card)) < fabs(residual(hi, k, card))) ? lo : hi;
  }
  return 0;
}

/* ---------------------------------------------------------------- PAA
 * "divides the data series in segments of equal length, and uses the
 * mean value of the points in each segment".  paa[s] = (1/seglen) * sum of the
 * seglen points of segment s, summed in order in double.
 */
void oracle_paa(const float* x, int len, int w, double* paa) {
  int seglen = len / w;
  for (int s = 0; s < w; ++s) {
    double acc = 0.0;
    for (int j = 0; j < seglen; ++j) acc += (double)x[s * seglen + j];
    paa[s] = acc / (double)seglen;
  }
}

/* ---------------------------------------------------------------- SAX symbol
 * "represents each segment of the series with the symbol of the region
 * the PAA falls into".  Region c = [cut_c, cut_{c+1}) with cut_0 = -inf,
 * cut_card = +inf; symbol = number of cuts <= v (a value on a cut goes to the
 * upper region, reading 3).  Linear count, no search.
 */
int oracle_sax_symbol(double v, const double* cuts, int card) {
  int c = 0;
  for (int k = 0; k < card - 1; ++k)
    if (cuts[k] <= v) ++c;
  return c;
}

/* ---------------------------------------------------------------- summarize
 * Alg2 line al2:cover: SAX[p+i] = ConvertToSAX(TS[i]); the word of
 * series p is stored at position p.  Output row-major [n][w].
 */
int oracle_summarize(const float* raw, int64_t n, int len, int w, int card, uint8_t* sax) {
  if (len % w) return -2;
  double* cuts = (double*)malloc(sizeof(double) * 256);
  double* paa = (double*)malloc(sizeof(double) * (size_t)w);
  if (!cuts || !paa) { free(cuts); free(paa); return -4; }
  if (oracle_cuts(card, cuts)) { free(cuts); free(paa); return -2; }
  for (int64_t i = 0; i < n; ++i) {
    oracle_paa(raw + (size_t)i * len, len, w, paa);
    for (int s = 0; s < w; ++s) sax[(size_t)i * w + s] = (uint8_t)oracle_sax_symbol(paa[s], cuts, card);
  }
  free(cuts);
  free(paa);
  return 0;
}

/* ---------------------------------------------------------------- LB table
 * the lower bound between the query PAA and an iSAX word has three
 * branches per segment -- the PAA lies ABOVE, BELOW or IN the symbol's interval
 * -- each taking its value from its own "dictionary".  Reading 1 (standard
 * MINDIST_PAA_iSAX): LB^2 = (len/w) * sum_s delta_s^2 with
 *   ABOVE (q > U[c]):  delta = q - U[c]
 *   BELOW (q < L[c]):  delta = L[c] - q
 *   IN:                delta = 0
 * L[c] = cut_c, U[c] = cut_{c+1}.  T[s*card + c] = (len/w) * delta^2.
 */
int oracle_lb_table(const double* qpaa, int len, int w, int card, double* T) {
  double cuts[256];
  if (oracle_cuts(card, cuts)) return -2;
  double seglen = (double)(len / w);
  for (int s = 0; s < w; ++s) {
    double q = qpaa[s];
    for (int c = 0; c < card; ++c) {
      double lower = (c == 0) ? -INFINITY : cuts[c - 1];
      double upper = (c == card - 1) ? INFINITY : cuts[c];
      double delta;
      if (q > upper) delta = q - upper;        /* ABOVE */
      else if (q < lower) delta = lower - q;   /* BELOW */
      else delta = 0.0;                        /* IN */
      T[s * card + c] = seglen * delta * delta;
    }
  }
  return 0;
}

/* LB^2 of one word (symbols word[0..w-1]) from the table: sum of w dictionary values. */
double oracle_lb2(const double* T, const uint8_t* word, int w, int card) {
  double acc = 0.0;
  for (int s = 0; s < w; ++s) acc += T[s * card + word[s]];
  return acc;
}

/* ---------------------------------------------------------------- distances
 * P:219 (reading 4): ED = sqrt(sum_t (a_t - b_t)^2); ranking uses the square.
 */
double oracle_ed2(const float* a, const float* b, int len) {
  double acc = 0.0;
  for (int t = 0; t < len; ++t) {
    double d = (double)a[t] - (double)b[t];
    acc += d * d;
  }
  return acc;
}

/* Early abandoning (north_star): stop as soon as the running sum is
 * strictly greater than `limit` and return it (any value > limit); otherwise the
 * exact sum.  Strict, so a series tying the current k-th distance is still
 * computed exactly and the id tie-break can decide. */
double oracle_ed2_abandon(const float* a, const float* b, int len, double limit) {
  double acc = 0.0;
  for (int t = 0; t < len; ++t) {
    double d = (double)a[t] - (double)b[t];
    acc += d * d;
    if (acc > limit) return acc;
  }
  return acc;
}

/* ---------------------------------------------------------------- k-NN
 * Result order: ascending by (d^2, id) -- ties go to the lower id (reading 6).
 */
typedef struct { double d2; int64_t id; } entry_t;

static int entry_less(entry_t a, entry_t b) {
  return (a.d2 < b.d2) || (a.d2 == b.d2 && a.id < b.id);
}

/* max-heap of (d2, id) under entry_less, size <= k */
static void heap_sift_down(entry_t* h, int size, int i) {
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < size && entry_less(h[m], h[l])) m = l;
    if (r < size && entry_less(h[m], h[r])) m = r;
    if (m == i) return;
    entry_t t = h[i]; h[i] = h[m]; h[m] = t;
    i = m;
  }
}
static void heap_sift_up(entry_t* h, int i) {
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!entry_less(h[p], h[i])) return;
    entry_t t = h[i]; h[i] = h[p]; h[p] = t;
    i = p;
  }
}
static int cmp_entry(const void* x, const void* y) {
  entry_t a = *(const entry_t*)x, b = *(const entry_t*)y;
  return entry_less(a, b) ? -1 : (entry_less(b, a) ? 1 : 0);
}
/* heap -> ascending output */
static void heap_emit(entry_t* h, int size, int64_t* out_idx, double* out_d2) {
  qsort(h, (size_t)size, sizeof(entry_t), cmp_entry);
  for (int j = 0; j < size; ++j) { out_idx[j] = h[j].id; out_d2[j] = h[j].d2; }
}

/* Plain definition (generalized to k per S:406-414): for every query,
 * d^2 to every series, keep the k smallest (d^2, id).  Ground truth. */
int oracle_knn_bruteforce(const float* raw, int64_t n, int len, const float* queries, int nq,
                          int k, int64_t* out_idx, double* out_d2) {
  if (k < 1 || k > n) return -1;
  entry_t* h = (entry_t*)malloc(sizeof(entry_t) * (size_t)k);
  if (!h) return -4;
  for (int q = 0; q < nq; ++q) {
    const float* qs = queries + (size_t)q * len;
    int size = 0;
    for (int64_t i = 0; i < n; ++i) {
      entry_t e = {oracle_ed2(raw + (size_t)i * len, qs, len), i};
      if (size < k) { h[size] = e; heap_sift_up(h, size); ++size; }
      else if (entry_less(e, h[0])) { h[0] = e; heap_sift_down(h, size, 0); }
    }
    heap_emit(h, size, out_idx + (size_t)q * k, out_d2 + (size_t)q * k);
  }
  free(h);
  return 0;
}

/* LB-pruned exact search: the nb-ParIS+ DistComp logic (Alg8) run by
 * one worker over the whole SAX array, with the RDC-Worker checks (Alg11,
 * P:1364-1371) and BSF generalized to the k-th best:
 *   BSF = +inf until k results exist, then the k-th best d^2;
 *   for i = 0..n-1:  minDist = LB^2(q, SAX[i]);  if minDist < BSF ...
 *     realDist = Dist(raw[i], q) with early abandoning at BSF;
 *     if (realDist, i) < k-th best: insert.
 * Scanning i in increasing order makes "LB >= BSF => prune" and "abandon once
 * the partial sum exceeds BSF" consistent with the lower-id tie rule: a later id
 * can never win a tie.  The pruning test keeps LB == BSF (a tie may exist only
 * if d^2 == BSF, which needs LB <= d^2 == BSF).  sax is row-major [n][w].
 * stats (may be NULL): [0] LB computations, [1] raw series read (refined),
 * [2] BSF updates, summed over queries.
 */
int oracle_knn_pruned(const float* raw, const uint8_t* sax, int64_t n, int len, int w, int card,
                      const float* queries, int nq, int k, int64_t* out_idx, double* out_d2,
                      int64_t* stats) {
  if (k < 1 || k > n || len % w) return -1;
  entry_t* h = (entry_t*)malloc(sizeof(entry_t) * (size_t)k);
  double* T = (double*)malloc(sizeof(double) * (size_t)w * card);
  double* qpaa = (double*)malloc(sizeof(double) * (size_t)w);
  if (!h || !T || !qpaa) { free(h); free(T); free(qpaa); return -4; }
  int64_t n_lb = 0, n_read = 0, n_upd = 0;
  for (int q = 0; q < nq; ++q) {
    const float* qs = queries + (size_t)q * len;
    oracle_paa(qs, len, w, qpaa);
    if (oracle_lb_table(qpaa, len, w, card, T)) { free(h); free(T); free(qpaa); return -2; }
    int size = 0;
    for (int64_t i = 0; i < n; ++i) {
      double bsf = (size < k) ? INFINITY : h[0].d2;
      double lb2 = oracle_lb2(T, sax + (size_t)i * w, w, card);
      ++n_lb;
      if (lb2 > bsf) continue; /* pruned: LB > BSF */
      ++n_read;
      double d2 = oracle_ed2_abandon(raw + (size_t)i * len, qs, len, bsf);
      entry_t e = {d2, i};
      if (size < k) { h[size] = e; heap_sift_up(h, size); ++size; ++n_upd; }
      else if (entry_less(e, h[0])) { h[0] = e; heap_sift_down(h, size, 0); ++n_upd; }
    }
    heap_emit(h, size, out_idx + (size_t)q * k, out_d2 + (size_t)q * k);
  }
  if (stats) { stats[0] += n_lb; stats[1] += n_read; stats[2] += n_upd; }
  free(h);
  free(T);
  free(qpaa);
  return 0;
}
