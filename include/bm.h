/*
 * bm.h — C ABI of the B200-native Ball Mapper cover-construction library
 * (libbm_b200.so), arxiv 2601.01405.
 *
 * The library computes, on one sm_100a GPU, the three steps of the paper's
 * cover construction:
 *
 *   1. the greedy eps-net in point order (§2.2): point i is a
 *      landmark iff no earlier landmark l has d(x_i, x_l) < eps;
 *   2. ball membership B(c, eps) ∩ X = {p : d(c, x_p) < eps} of every point in
 *      every landmark ball (open balls; the range queries of
 *      §3);
 *   3. the nerve 1-skeleton (Def 2.2): an edge (i, j), i < j
 *      landmark positions, iff some data point lies in both balls (∩ X ≠ ∅,
 *      PAPER.md:88).
 *
 * Distances (BASELINE.json north_star):
 *   BM_L2      Euclidean  (Gram form PAPER.md:245 on the tensor path)
 *   BM_L1      Manhattan  sum_j |x_j - y_j|
 *   BM_COSINE  1 - x.y / (|x| |y|)                (a zero vector is at
 *              distance 0 from another zero vector and 1 from any other vector)
 *
 * Exactness: integer inputs are decided exactly (int32 arithmetic).  Float
 * inputs are decided in fp32 (CUDA cores) or tf32 (tensor cores) with a
 * rigorous error band; every pair inside the band is re-decided with the
 * fp64 formula  sum_j ((double)x_j - (double)y_j)^2 < eps*eps  (L1 / cosine
 * analogously), evaluated in ascending j without FMA contraction.  Pairs
 * whose fp64 distance lies within 1e-6*eps of eps ("near ties") are counted
 * and reported in bm_cover.near_tie_pairs.
 *
 * Threading: calls on different streams may run concurrently; the only
 * global state is the thread-local error string.
 */
#ifndef BM_B200_H
#define BM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_VERSION_MAJOR 0
#define BM_VERSION_MINOR 1

typedef enum bm_status {
  BM_OK = 0,
  BM_EINVAL = 1,        /* n < 1, d < 1, eps <= 0 or non-finite, non-finite coordinate, NULL pointer */
  BM_EUNSUPPORTED = 2,  /* dtype x metric combination not supported (e.g. integer cosine)            */
  BM_ENOMEM = 3,        /* device or host allocation failed                                          */
  BM_ECUDA = 4,         /* a CUDA runtime/driver error; text in bm_last_error()                       */
  BM_EOVERFLOW = 5      /* n > INT32_MAX, or a count exceeds an index type                           */
} bm_status;

typedef enum bm_metric { BM_L2 = 0, BM_L1 = 1, BM_COSINE = 2 } bm_metric;

typedef enum bm_dtype {
  BM_F32 = 0,  /* IEEE binary32 coordinates                                 */
  BM_I8 = 1,   /* int8 coordinates   (exact integer path: L2, L1)          */
  BM_U8 = 2,   /* uint8 coordinates  (exact integer path: L2, L1)          */
  BM_I32 = 3   /* int32 values: labels for bm_color (not a coordinate type) */
} bm_dtype;

/* Coloring aggregators (PAPER.md:125-133, 167, 187 [§2.3]). */
typedef enum bm_agg {
  BM_AGG_MEAN = 0,      /* (1/|X_i|) sum f                                        */
  BM_AGG_MEDIAN = 1,    /* even |X_i|: mean of the two central order statistics  */
  BM_AGG_TRIMMED = 2,   /* mean after dropping floor(alpha |X_i|) at each end     */
  BM_AGG_MIN = 3,
  BM_AGG_MAX = 4,
  BM_AGG_MODE = 5,      /* most frequent value, ties -> smallest value            */
  BM_AGG_VARIANCE = 6,  /* population variance                                    */
  BM_AGG_RANGE = 7      /* max - min                                              */
} bm_agg;

/* Per-step device timings, indices into bm_cover.step_ms. */
enum {
  BM_STEP_PREP = 0,     /* A0: packing, norms, finite check                      */
  BM_STEP_GREEDY = 1,   /* A1-A4 + B, B': blocked greedy eps-net; each tile's new   */
                        /* balls are filled over all points in the same loop      */
  BM_STEP_MEMBER = 2,   /* B fallback: exact-capacity membership recount (normally ~0) */
  BM_STEP_CSR = 3,      /* C: compaction into both CSRs                           */
  BM_STEP_EDGES = 4,    /* D1-D3: pair emission, radix sort, unique               */
  BM_STEP_TOTAL = 5,
  BM_STEP_MEMBER_KERNEL = 6,  /* membership contraction kernels alone, summed over tiles */
  BM_STEP_SELECT = 7,   /* BM_SELECT_FPS: the farthest point sampling kernel alone    */
  BM_NUM_STEPS = 8
};

/* Execution path for the membership / coverage contraction. */
typedef enum bm_path {
  BM_PATH_AUTO = 0,     /* tensor cores for L2 / cosine with d >= 32 or n >= 32768 and for
                           fp32 L1 with d <= 16 and n >= 65536, else CUDA cores */
  BM_PATH_CUDA_CORE = 1,
  BM_PATH_TENSOR = 2    /* tcgen05: L2, cosine, and fp32 L1 with d <= 16 (thermometer-code
                           contraction); BM_EUNSUPPORTED otherwise */
} bm_path;

/* Optional knobs.  Zero-initialise, set struct_size = sizeof(bm_options). */
typedef struct bm_options {
  int32_t struct_size;
  int32_t tile;          /* greedy candidate tile T: 0 = default (8192 on pruned tensor-core
                            launches, else 1024); 32..8192, multiple of 32                  */
  int32_t path;          /* bm_path                                                             */
  int32_t timing;        /* 1 = record per-step CUDA events into step_ms                        */
  int64_t near_tie_cap;  /* max near-tie pairs stored (0 = default 65536); all are counted      */
  int32_t key_cap;       /* initial membership key capacity (0 = default 16 n); a smaller M
                            fits, a larger one costs one exact-capacity recount             */
  int32_t reserved0;     /* must be 0 (layout slot)                                           */
  int32_t flags;         /* BM_FLAG_* (diagnostics)                                           */
  int32_t select;        /* bm_select: landmark selection (default greedy in point order)     */
  int32_t fps_start;     /* BM_SELECT_FPS: index of the initial landmark x_0 (default 0)      */
  int32_t reserved[3];
} bm_options;

/* Landmark selection (PAPER.md:98-119 [§2.2]). */
typedef enum bm_select {
  BM_SELECT_GREEDY = 0,  /* greedy eps-net in point order (the north-star path)           */
  BM_SELECT_FPS = 1      /* farthest point sampling: x* = argmax min d, added while >= eps
                            (ties: lowest index); landmarks are returned ascending        */
} bm_select;

/* bm_options.flags */
#define BM_FLAG_NO_L1_PREFILTER 1   /* L1: score every pair in fp32 (no 8-bit SAD prefilter) */
#define BM_FLAG_EDGE_POINT_PAIRS 2  /* L > 4096: D1 emits every witnessed pair per point (C(t_p, 2)),
                                       not the row-union keys deduplicated per ball row item;
                                       then the same sort + unique           */
#define BM_FLAG_NO_EDGE_TRIANGLE BM_FLAG_EDGE_POINT_PAIRS   /* (former name)                 */
#define BM_FLAG_NO_PRUNE 4          /* tensor path: no tile-level pruning of the membership contraction */
#define BM_FLAG_FORCE_PRUNE 8       /* tensor path: prune even below the size where it pays (tests) */
#define BM_FLAG_DENSE_RESOLVE 16    /* tiles > 1024: resolve from the dense words, not the sparse list (tests) */
#define BM_FLAG_EDGE_TRIANGLE 32    /* L > 4096: edges from a strictly-upper L x L bit triangle (no
                                       sort) when it fits in a quarter of free HBM (<= 8 GiB);
                                       default only while it is <= 256 MiB                    */
#define BM_FLAG_EDGE_ROWS 64        /* L > 4096: D1 always by row union (default: only when the
                                       witnessed pairs are >= 512 per landmark)                */

/*
 * Result of one cover construction.  All arrays are owned by the library and
 * released by bm_free().  For bm_cover_build / bm_cover_build_ex they are
 * DEVICE pointers (valid on the device of the call); for bm_cover_build_host
 * they are HOST pointers.  on_host says which.
 */
typedef struct bm_cover {
  int64_t n;                 /* number of points                                         */
  int32_t d;                 /* dimension                                                */
  int32_t dtype;             /* bm_dtype                                                 */
  int32_t metric;            /* bm_metric                                                */
  int32_t on_host;           /* 0: device arrays, 1: host arrays                         */
  double eps;

  int64_t n_landmarks;       /* L                                                        */
  int32_t *landmarks;        /* [L] point indices, strictly ascending                    */

  int64_t n_members;         /* M = sum_j |B_j|                                           */
  int64_t *ball_ptr;         /* [L+1] landmark-major CSR row pointer                     */
  int32_t *ball_idx;         /* [M] point indices, ascending within each ball            */
  int64_t *pt_ptr;           /* [n+1] point-major CSR row pointer                        */
  int32_t *pt_lm;            /* [M] landmark POSITIONS, ascending within each point      */

  int64_t n_edges;           /* E                                                        */
  int32_t *edges;            /* [E][2] landmark positions (i, j), i < j, lexicographic   */

  int64_t n_witness_pairs;   /* P = sum_p C(t_p, 2): landmark pairs witnessed by points  */
  int64_t n_pair_evals;      /* n * L: point-landmark distance evaluations of step B     */
  int64_t n_greedy_evals;    /* extra evaluations inside the greedy (tiles + coverage)   */
  int64_t n_band_pairs;      /* float paths: pairs re-decided in fp64                    */
  int64_t n_near_ties;       /* pairs with |d_fp64 - eps| <= 1e-6 eps (all counted)      */
  int64_t n_near_ties_stored;/* min(n_near_ties, near_tie_cap)                           */
  int64_t *near_tie_pairs;   /* [n_near_ties_stored][3] (point, landmark point, decision); HOST */
  int64_t n_greedy_tiles;    /* candidate tiles resolved                                 */
  int64_t n_launches;        /* library kernels launched by this call                    */
  int64_t n_member_launches; /* membership-contraction launches (one per greedy tile)    */
  int32_t path_used;         /* bm_path actually used for the contraction                */
  int32_t tile_used;         /* greedy tile T                                            */
  float step_ms[BM_NUM_STEPS];/* per-step device time (ms) when options.timing = 1       */
  /* tensor path, fused greedy membership: 128 x 256 tiles contracted / skipped by
   * the tile-level pruning, 128 x 32 accumulator chunks read from TMEM / skipped */
  int64_t n_tc_tiles_run, n_tc_tiles_skipped, n_tc_chunks_run, n_tc_chunks_skipped;
  void *priv;                /* library-private                                          */
} bm_cover;

/*
 * bm_cover_build — build the cover of `points` on the caller's CUDA stream.
 *
 *   points  DEVICE pointer to n*d elements of `dtype`, row-major (point p is
 *           points[p*d .. p*d+d)), read-only, any alignment.
 *   n, d    number of points (1 <= n <= INT32_MAX) and dimension (d >= 1).
 *   metric  bm_metric; eps > 0 and finite.  The integer L2 path takes
 *           eps = sqrt(eps^2) and decides (double)d2 < eps*eps exactly.
 *   stream  cudaStream_t (may be NULL = legacy default stream).  All device
 *           work is ordered on it; the call returns after the final count
 *           read-back, i.e. synchronously with respect to the host.
 *   out     receives a newly allocated bm_cover on BM_OK, NULL otherwise.
 *
 * Errors are returned, never thrown; on error nothing is leaked and
 * bm_last_error() holds a message.
 */
bm_status bm_cover_build(const void *points, bm_dtype dtype, int64_t n, int32_t d,
                         bm_metric metric, double eps, void *stream, bm_cover **out);

/* As bm_cover_build with options (NULL = defaults). */
bm_status bm_cover_build_ex(const void *points, bm_dtype dtype, int64_t n, int32_t d,
                            bm_metric metric, double eps, void *stream,
                            const bm_options *opts, bm_cover **out);

/*
 * bm_cover_build_host — same computation from a HOST buffer: the points are
 * copied to the device inside the call (pinned host memory gives the best
 * copy rate) and every output array is copied back into library-owned HOST
 * memory (on_host = 1): one pinned block per cover, recycled by bm_free and
 * released by bm_trim_memory.  Used for end-to-end timing.
 */
bm_status bm_cover_build_host(const void *host_points, bm_dtype dtype, int64_t n, int32_t d,
                              bm_metric metric, double eps, void *stream,
                              const bm_options *opts, bm_cover **out);

/*
 * bm_color — colour every landmark of a cover (PAPER.md:125-133 [§2.3]):
 * out[j] = agg of values over the ball X_j = X ∩ B(l_j, eps) (landmark-major
 * CSR of `c`).
 *   c       a DEVICE cover (from bm_cover_build / _ex) on the current device.
 *   values  DEVICE pointer to n values f(x_p): BM_F32 (finite) or BM_I32 (labels).
 *   agg     bm_agg; alpha in [0, 0.5) for BM_AGG_TRIMMED (ignored otherwise).
 *   out     DEVICE pointer to L doubles (labels are returned as exact doubles).
 * Ordered on `stream`; returns after the work is queued and checked.
 * Errors: BM_EINVAL (NULL pointer, host cover, bad alpha), BM_EUNSUPPORTED
 * (value type / aggregator), BM_ENOMEM, BM_ECUDA.
 */
bm_status bm_color(const bm_cover *c, const void *values, bm_dtype vtype, bm_agg agg,
                   double alpha, double *out, void *stream);

/*
 * bm_skeleton — the k-simplices of the nerve (Def 2.2): the
 * sets of k+1 landmark positions whose balls share a data point, each
 * ascending, in lexicographic order.  k >= 1 (k = 1 gives the edge list).
 *   out       DEVICE pointer to capacity*(k+1) int32 (may be NULL with capacity 0);
 *             receives the first min(count, capacity) simplices.
 *   count     HOST, receives the number of k-simplices.
 *   max_emit  cap on the witnessed (k+1)-subsets enumerated (sum_p C(t_p, k+1));
 *             0 = default 2^31.  Exceeding it returns BM_EOVERFLOW.
 * Requires (k+1) * bits(L-1) <= 64 (BM_EUNSUPPORTED otherwise).  Synchronous.
 */
bm_status bm_skeleton(const bm_cover *c, int32_t k, int32_t *out, int64_t capacity,
                      int64_t *count, int64_t max_emit, void *stream);

/* Release a cover and every array it owns.  NULL-safe. */
void bm_free(bm_cover *c);

/* Return the device memory the library keeps cached between calls (its
 * stream-ordered pool on the current device) to the system.  Memory still
 * owned by live covers is unaffected. */
bm_status bm_trim_memory(void);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char *bm_last_error(void);

/* Library version: (major << 16) | minor. */
int32_t bm_version(void);

/* ----------------------------------------------------------------------------
 * Diagnostic entry points (used by the kernel unit tests; same conventions).
 * -------------------------------------------------------------------------- */

/* Sort n uint64 keys in place on the device (LSD radix over the low `bits`
 * bits, stable); keys is a DEVICE pointer.  The library's own D2 sort. */
bm_status bm_debug_radix_sort_u64(uint64_t *keys, int64_t n, int32_t bits, void *stream);

/* Exclusive prefix sum of n int64 values (DEVICE pointers); *total (HOST)
 * receives the sum.  The library's own scan. */
bm_status bm_debug_exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n,
                                      int64_t *total, void *stream);

/* In-order LFMIS resolve of one candidate tile (step A3) from a dense
 * lower-triangular adjacency: adj is a HOST array of nc*ceil(nc/32) uint32
 * words, row a word w bit b = [candidate a adjacent to candidate 32w+b],
 * only bits with 32w+b < a are read.  lm_out (HOST, nc bytes) receives 1 for
 * selected candidates.  nc <= 1024. */
bm_status bm_debug_resolve_tile(const uint32_t *adj, int32_t nc, uint8_t *lm_out, void *stream);

/* Raw tcgen05 Gram accumulators of the membership contraction (step B):
 * out[p*L + j] = bits of sum_k x_p[k] * x_{lm[j]}[k] as accumulated by the
 * tensor core (fp32 bits of the tf32 products for BM_F32, int32 for
 * BM_U8 / BM_I8).  points, lm and out are DEVICE pointers; d*elem <= 4096
 * bytes. */
bm_status bm_debug_tc_gram(const void *points, bm_dtype dtype, int64_t n, int32_t d,
                           const int32_t *lm, int64_t L, uint32_t *out, void *stream);

/* Timing probe of the tcgen05 contraction (step B) for fp32 data with d <= 64:
 * n points (DEVICE pointer, row-major) against the first L of them, with an
 * epilogue that classifies (mode 0: the membership epilogue, every pair out),
 * only reads the accumulators (mode 2) or releases them unread (mode 3).
 * *ms_out (HOST) receives the mean launch time over `iters` launches. */
bm_status bm_debug_tc_probe(const float *points, int64_t n, int32_t d, int64_t L, int32_t mode,
                            int32_t iters, float *ms_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BM_B200_H */
