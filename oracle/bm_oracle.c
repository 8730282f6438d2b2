/*
 * bm_oracle.c — plain, slow, obviously-correct CPU oracle for the Ball Mapper
 * cover construction (arxiv 2601.01405).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product path
 * (paper_2601_01405_b200/) never links, imports or executes it; the two share
 * no code, headers, helpers, tables or constants.
 *
 * What it computes, in the paper's order and notation:
 *   1. Greedy eps-net (§2.2): walk the points in index order
 *      (reading A2 in DESIGN.md); a point not yet covered becomes a landmark
 *      ("Add x to N") and every point within distance < eps of
 *      it is marked covered ("Mark all points within distance eps of x as
 *      covered").  "Within" is the open ball of PAPER.md:69
 *      (strict <, reading A1).
 *   2. Ball membership: one naive linear range query per landmark over ALL
 *      points (§3) — B(c_i, eps) ∩ X, including
 *      points before the landmark and the landmark itself (reading A3).
 *   3. Nerve 1-skeleton (Def 2.2): landmarks i<j are joined
 *      iff some data point lies in both balls (∩ X ≠ ∅; reading
 *      A4), enumerated per point over its covering landmarks, sorted and
 *      de-duplicated (reading A5).
 *
 * Distances (reading A6-A10), no Gram trick, no blocking, no reordering:
 *   L2  ints:  d2 = Σ_j (x_j - y_j)^2 in int64;    in iff (double)d2 < eps*eps
 *   L2  f32:   d2 = Σ_j ((double)x_j - (double)y_j)^2, j ascending, fp64,
 *              compiled with -ffp-contract=off;    in iff d2 < eps*eps
 *   L1  ints:  s = Σ_j |x_j - y_j| in int64;       in iff (double)s < eps
 *   L1  f32:   s = Σ_j |(double)x_j - (double)y_j| in fp64; in iff s < eps
 *   COS f32:   1 - dot/(sqrt(xx)*sqrt(yy)) < eps, all fp64 (PAPER.md:253
 *              names cosine; reading A7 for the zero vector: two zero vectors
 *              are at distance 0, a zero and a non-zero vector at distance 1).
 *              Parity unpinned for zero vectors (no config contains one).
 *   u8 data is used as-is (integers 0..255); i8 as-is.
 *
 * Overrides (tie protocol): an optional list of (point p,
 * landmark point i, value) triples replaces the in-ball decision for that
 * pair; the comparator uses it only for pairs whose fp64 distance lies within
 * the 1e-6*eps tolerance band stated in BASELINE.json `north_star`.
 *
 * Parallelism: each range query is an OpenMP parallel-for over p; every p
 * writes only its own slot, so the result is deterministic.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_F32 = 0, OR_I8 = 1, OR_U8 = 2 };
enum { OR_L2 = 0, OR_L1 = 1, OR_COS = 2 };

typedef struct {
  int64_t L;            /* number of landmarks                                  */
  int64_t *landmarks;   /* [L] point indices, ascending                         */
  int64_t M;            /* total memberships Σ_j |B_j|                          */
  int64_t *ball_ptr;    /* [L+1] landmark-major CSR                             */
  int64_t *ball_idx;    /* [M] point indices ascending within a ball           */
  int64_t *pt_ptr;      /* [n+1] point-major transpose                          */
  int64_t *pt_lm;       /* [M] landmark positions ascending within a point     */
  int64_t E;            /* number of edges                                      */
  int64_t *edges;       /* [E][2] (i, j) landmark positions, i < j, lexicographic */
  int64_t pairs_evaluated; /* L * n range-query evaluations                    */
} oracle_cover_t;

/* ---- distance predicates: one function per (dtype, metric), plain loops --- */

static double coord(const void *X, int dtype, int64_t p, int d, int j) {
  if (dtype == OR_F32) return (double)((const float *)X)[p * (int64_t)d + j];
  if (dtype == OR_I8) return (double)((const int8_t *)X)[p * (int64_t)d + j];
  return (double)((const uint8_t *)X)[p * (int64_t)d + j];
}

static int64_t icoord(const void *X, int dtype, int64_t p, int d, int j) {
  if (dtype == OR_I8) return (int64_t)((const int8_t *)X)[p * (int64_t)d + j];
  return (int64_t)((const uint8_t *)X)[p * (int64_t)d + j];
}

/* fp64 / int64 distance between rows p and q, exactly as documented above.
 * For L2 the value returned is the SQUARED distance. */
double oracle_distance(const void *X, int dtype, int d, int metric, int64_t p, int64_t q) {
  if (metric == OR_L2) {
    if (dtype == OR_F32) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) {
        double t = coord(X, dtype, p, d, j) - coord(X, dtype, q, d, j);
        double sq = t * t;
        s = s + sq;
      }
      return s;
    } else {
      int64_t s = 0;
      for (int j = 0; j < d; ++j) {
        int64_t t = icoord(X, dtype, p, d, j) - icoord(X, dtype, q, d, j);
        s += t * t;
      }
      return (double)s;
    }
  }
  if (metric == OR_L1) {
    if (dtype == OR_F32) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) {
        double t = coord(X, dtype, p, d, j) - coord(X, dtype, q, d, j);
        s = s + fabs(t);
      }
      return s;
    } else {
      int64_t s = 0;
      for (int j = 0; j < d; ++j) {
        int64_t t = icoord(X, dtype, p, d, j) - icoord(X, dtype, q, d, j);
        s += t < 0 ? -t : t;
      }
      return (double)s;
    }
  }
  /* cosine distance 1 - x.y / (|x| |y|) */
  double dot = 0.0, xx = 0.0, yy = 0.0;
  for (int j = 0; j < d; ++j) {
    double a = coord(X, dtype, p, d, j), b = coord(X, dtype, q, d, j);
    double ab = a * b, aa = a * a, bb = b * b;
    dot = dot + ab;
    xx = xx + aa;
    yy = yy + bb;
  }
  if (xx == 0.0 && yy == 0.0) return 0.0;
  if (xx == 0.0 || yy == 0.0) return 1.0;
  double nx = sqrt(xx), ny = sqrt(yy);
  double den = nx * ny;
  return 1.0 - dot / den;
}

/* in-ball predicate d(p, q) < eps (open ball) */
static int in_ball(const void *X, int dtype, int d, int metric, double eps, int64_t p, int64_t q) {
  double v = oracle_distance(X, dtype, d, metric, p, q);
  if (metric == OR_L2) return v < eps * eps;
  return v < eps;
}

/* ---- override lookup: keys p*n + q, sorted ascending ---------------------- */
typedef struct { int64_t key; int val; } ov_t;
static int ov_cmp(const void *a, const void *b) {
  int64_t x = ((const ov_t *)a)->key, y = ((const ov_t *)b)->key;
  return (x > y) - (x < y);
}
static int ov_find(const ov_t *ov, int64_t n_ov, int64_t key) {
  int64_t lo = 0, hi = n_ov;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (ov[mid].key < key) lo = mid + 1; else hi = mid;
  }
  if (lo < n_ov && ov[lo].key == key) return ov[lo].val;
  return -1;
}

static int i64_cmp(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

void oracle_free(oracle_cover_t *c) {
  if (!c) return;
  free(c->landmarks); free(c->ball_ptr); free(c->ball_idx);
  free(c->pt_ptr); free(c->pt_lm); free(c->edges);
  memset(c, 0, sizeof(*c));
}

int oracle_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
  return omp_get_max_threads();
#else
  (void)t;
  return 1;
#endif
}

/*
 * oracle_cover: returns 0 on success, 1 on invalid input, 3 on allocation
 * failure.  ov_p / ov_q / ov_val: n_ov override triples (point p, landmark
 * point q, decision) — may be NULL when n_ov == 0.
 */
/*
 * Farthest point sampling eps-net (§2.2), NEXT-2 in SURVEY
 * §8(f): start from x_0 = `start`; repeatedly take x* = argmax_x min_{l in L}
 * d(x, l) (ties: lowest index, reading F2) and add it while that maximum is
 * >= eps (reading F1: the paper's step 4 says "> eps", which would leave a
 * point at distance exactly eps uncovered by the open balls; SPEC S:311 takes
 * ">=").  d is oracle_distance (for L2 the fp64 squared distance, compared
 * with eps*eps).  Writes the selection order into seq (capacity n), returns L.
 */
int64_t oracle_fps(const void *X, int dtype, int64_t n, int d, int metric, double eps,
                   int64_t start, int64_t *seq) {
  if (!X || n < 1 || d < 1 || start < 0 || start >= n || !seq) return -1;
  const double thr = metric == OR_L2 ? eps * eps : eps;
  double *mind = (double *)malloc(sizeof(double) * (size_t)n);
  if (!mind) return -1;
  int64_t L = 0;
  int64_t cur = start;                       /* step 1: initial landmark x_0 */
  for (int64_t p = 0; p < n; ++p) mind[p] = INFINITY;
  for (;;) {
    seq[L++] = cur;                          /* add x* to L */
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {        /* min over the landmark set */
      double v = oracle_distance(X, dtype, d, metric, p, cur);
      if (v < mind[p]) mind[p] = v;
    }
    int64_t best = 0;                        /* step 3: argmax, lowest index on ties */
    for (int64_t p = 1; p < n; ++p)
      if (mind[p] > mind[best]) best = p;
    if (!(mind[best] >= thr)) break;         /* step 4 (reading F1), step 5 */
    cur = best;
  }
  free(mind);
  return L;
}

int oracle_cover_given(const void *X, int dtype, int64_t n, int d, int metric, double eps,
                       const int64_t *given, int64_t n_given, const int64_t *ov_p,
                       const int64_t *ov_q, const int8_t *ov_val, int64_t n_ov,
                       oracle_cover_t *out);

int oracle_cover(const void *X, int dtype, int64_t n, int d, int metric, double eps,
                 const int64_t *ov_p, const int64_t *ov_q, const int8_t *ov_val, int64_t n_ov,
                 oracle_cover_t *out) {
  return oracle_cover_given(X, dtype, n, d, metric, eps, NULL, 0, ov_p, ov_q, ov_val, n_ov, out);
}

/* The cover of a landmark set: the greedy's (given == NULL) or a given
 * ascending list (e.g. the FPS landmarks, sorted) — one linear range query per
 * landmark either way. */
int oracle_cover_given(const void *X, int dtype, int64_t n, int d, int metric, double eps,
                       const int64_t *given, int64_t n_given, const int64_t *ov_p,
                       const int64_t *ov_q, const int8_t *ov_val, int64_t n_ov,
                       oracle_cover_t *out) {
  memset(out, 0, sizeof(*out));
  if (!X || n < 1 || d < 1 || !(eps > 0.0) || !isfinite(eps)) return 1;
  if (dtype < 0 || dtype > 2 || metric < 0 || metric > 2) return 1;

  ov_t *ov = NULL;
  if (n_ov > 0) {
    ov = (ov_t *)malloc(sizeof(ov_t) * (size_t)n_ov);
    if (!ov) return 3;
    for (int64_t k = 0; k < n_ov; ++k) { ov[k].key = ov_p[k] * n + ov_q[k]; ov[k].val = ov_val[k] ? 1 : 0; }
    qsort(ov, (size_t)n_ov, sizeof(ov_t), ov_cmp);
  }

  uint8_t *covered = (uint8_t *)calloc((size_t)n, 1);
  uint8_t *hit = (uint8_t *)malloc((size_t)n);
  int64_t cap_l = 1024, cap_m = 1 << 16;
  int64_t *lm = (int64_t *)malloc(sizeof(int64_t) * cap_l);
  int64_t *bptr = (int64_t *)malloc(sizeof(int64_t) * (cap_l + 1));
  int64_t *bidx = (int64_t *)malloc(sizeof(int64_t) * cap_m);
  if (!covered || !hit || !lm || !bptr || !bidx) goto nomem;
  int64_t L = 0, M = 0;
  bptr[0] = 0;

  /* 1+2: greedy eps-net with one linear range query per landmark */
  for (int64_t gi = 0; gi < (given ? n_given : n); ++gi) {
    const int64_t i = given ? given[gi] : gi;
    if (!given && covered[i]) continue;       /* "Select an uncovered point x" */
    if (L == cap_l) {                         /* "Add x to N"                  */
      cap_l *= 2;
      int64_t *a = (int64_t *)realloc(lm, sizeof(int64_t) * cap_l);
      int64_t *b = (int64_t *)realloc(bptr, sizeof(int64_t) * (cap_l + 1));
      if (!a || !b) { lm = a ? a : lm; bptr = b ? b : bptr; goto nomem; }
      lm = a; bptr = b;
    }
    lm[L] = i;
    /* range query B(x_i, eps) ∩ X over all points */
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
      int v = -1;
      if (ov) v = ov_find(ov, n_ov, p * n + i);
      if (v < 0) v = in_ball(X, dtype, d, metric, eps, p, i);
      hit[p] = (uint8_t)v;
    }
    int64_t cnt = 0;
    for (int64_t p = 0; p < n; ++p) cnt += hit[p];
    if (M + cnt > cap_m) {
      while (M + cnt > cap_m) cap_m *= 2;
      int64_t *a = (int64_t *)realloc(bidx, sizeof(int64_t) * cap_m);
      if (!a) goto nomem;
      bidx = a;
    }
    for (int64_t p = 0; p < n; ++p)
      if (hit[p]) { bidx[M++] = p; covered[p] = 1; }  /* "Mark ... as covered" */
    ++L;
    bptr[L] = M;
  }

  /* point-major transpose pt_lm (landmark positions ascending per point) */
  int64_t *pptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *plm = (int64_t *)malloc(sizeof(int64_t) * (M > 0 ? M : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!pptr || !plm || !fill) { free(pptr); free(plm); free(fill); goto nomem; }
  for (int64_t k = 0; k < M; ++k) pptr[bidx[k] + 1]++;
  for (int64_t p = 0; p < n; ++p) pptr[p + 1] += pptr[p];
  for (int64_t p = 0; p < n; ++p) fill[p] = pptr[p];
  for (int64_t j = 0; j < L; ++j)
    for (int64_t k = bptr[j]; k < bptr[j + 1]; ++k) plm[fill[bidx[k]]++] = j;
  free(fill);

  /* 3: 1-skeleton — every point with t covering landmarks witnesses C(t,2) pairs */
  int64_t P = 0;
  for (int64_t p = 0; p < n; ++p) { int64_t t = pptr[p + 1] - pptr[p]; P += t * (t - 1) / 2; }
  int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * (P > 0 ? P : 1));
  if (!keys) { free(pptr); free(plm); goto nomem; }
  int64_t q = 0;
  for (int64_t p = 0; p < n; ++p)
    for (int64_t a = pptr[p]; a < pptr[p + 1]; ++a)
      for (int64_t b = a + 1; b < pptr[p + 1]; ++b) keys[q++] = plm[a] * L + plm[b];
  qsort(keys, (size_t)P, sizeof(int64_t), i64_cmp);
  int64_t E = 0;
  for (int64_t k = 0; k < P; ++k)
    if (k == 0 || keys[k] != keys[k - 1]) keys[E++] = keys[k];
  int64_t *edges = (int64_t *)malloc(sizeof(int64_t) * 2 * (E > 0 ? E : 1));
  if (!edges) { free(keys); free(pptr); free(plm); goto nomem; }
  for (int64_t k = 0; k < E; ++k) { edges[2 * k] = keys[k] / L; edges[2 * k + 1] = keys[k] % L; }
  free(keys);

  free(covered); free(hit); free(ov);
  out->L = L; out->landmarks = lm; out->M = M; out->ball_ptr = bptr; out->ball_idx = bidx;
  out->pt_ptr = pptr; out->pt_lm = plm; out->E = E; out->edges = edges;
  out->pairs_evaluated = L * n;
  return 0;

nomem:
  free(covered); free(hit); free(lm); free(bptr); free(bidx); free(ov);
  return 3;
}

/* Plain range query: out[p] = (d(p, q) < eps) for all p. */
int oracle_range_query(const void *X, int dtype, int64_t n, int d, int metric, double eps,
                       int64_t q, uint8_t *out) {
  if (!X || n < 1 || d < 1 || q < 0 || q >= n || !(eps > 0.0)) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < n; ++p) out[p] = (uint8_t)in_ball(X, dtype, d, metric, eps, p, q);
  return 0;
}

/* fp64 distances between given pairs (used by the tie comparator and by the
 * sampled full-size parity checks): out[k] = distance(pp[k], qq[k]) where for
 * L2 the value is the Euclidean distance sqrt(d2) (d2 for the test itself is
 * oracle_distance). */
void oracle_pair_distances(const void *X, int dtype, int d, int metric, const int64_t *pp,
                           const int64_t *qq, int64_t k, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < k; ++t) {
    double v = oracle_distance(X, dtype, d, metric, pp[t], qq[t]);
    out[t] = metric == OR_L2 ? sqrt(v) : v;
  }
}

/* in-ball decisions for given pairs, exactly the oracle's predicate */
void oracle_pair_inball(const void *X, int dtype, int d, int metric, double eps,
                        const int64_t *pp, const int64_t *qq, int64_t k, uint8_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < k; ++t) out[t] = (uint8_t)in_ball(X, dtype, d, metric, eps, pp[t], qq[t]);
}
