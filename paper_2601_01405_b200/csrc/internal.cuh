// internal.cuh — shared declarations of the CUDA implementation behind include/bm.h.
//
// Layout in HBM:
//   rows   : prepped point rows, NU 8-byte units per row (fp32: 2 coords/unit,
//            int8: 8 coords/unit), zero padded, 16-B aligned base.  For fp32
//            these are the input values bit-for-bit, so they also serve the
//            fp64 recheck.
//   xhat   : cosine only — rows normalised by their fp64 norm, rounded to fp32
//            (a zero row holds NaN in unit 0 so every pair with it is sent to the
//            fp64 recheck, which applies the zero-vector rule).
//   inorm  : integer L2 only — exact int32 squared norms.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/bm.h"

namespace bm {

// ------------------------------------------------- programmatic dependent launch
// Kernels of the dependent chains (greedy tile loop, sorts, CSR, edges) are
// launched with programmatic stream serialization: the next kernel's launch
// overlaps the current one's tail, and every such kernel begins with
// pdl_wait() (griddepcontrol.wait: full completion and memory visibility of
// the previous grid) before touching its inputs.  pdl_trigger() lets the next
// kernel start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Decoupled look-back over per-tile descriptors (tag << 34 | flag << 32 |
// 32-bit value; flag 1 = aggregate, 2 = inclusive prefix), run by one full
// warp: lanes read 32 predecessors at once, the nearest inclusive prefix ends
// the walk.  Publishes this tile's aggregate first and its inclusive prefix
// last; returns the exclusive prefix.  Descriptors are never reset: a word
// with another launch's tag counts as not ready.
__device__ __forceinline__ uint32_t warp_lookback(unsigned long long* state, int64_t tile,
                                                  uint32_t tag, uint32_t agg) {
  volatile unsigned long long* st = state;
  const int lane = threadIdx.x & 31;
  const unsigned long long hdr = (unsigned long long)tag << 34;
  if (tile == 0) {
    if (lane == 0) st[0] = hdr | (2ull << 32) | agg;
    return 0u;
  }
  if (lane == 0) st[tile] = hdr | (1ull << 32) | agg;
  uint32_t excl = 0u;
  for (int64_t base = tile - 1;; base -= 32) {
    const int64_t j = base - lane;
    unsigned long long v = 2ull << 32;   // below tile 0: an inclusive prefix of 0
    if (j >= 0) {
      do {
        v = st[j];
      } while ((uint32_t)(v >> 34) != tag || ((v >> 32) & 3ull) == 0ull);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, ((v >> 32) & 3ull) == 2ull);
    const int first = inc ? __ffs(inc) - 1 : 32;   // nearest predecessor with a prefix
    uint32_t val = lane <= first ? (uint32_t)v : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    if (inc) break;
  }
  if (lane == 0) st[tile] = hdr | (2ull << 32) | (uint32_t)(excl + agg);
  return excl;
}

// BM_NO_PDL=1 (diagnostics): launch the dependent chains with plain stream
// ordering (griddepcontrol.wait then returns at once)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// ---------------------------------------------------------------- kinds
enum Kind : int { K_L2F = 0, K_L1F = 1, K_COSF = 2, K_L2I = 3, K_L1I = 4 };

enum PairMode : int { MODE_ADJ = 0, MODE_MEMBER = 2 };

// Thresholds for the classification "score < lo -> in, score >= hi -> out,
// else band (fp64 recheck)".  Score = d^2 (L2F), L1 sum (L1F), -cos (COSF),
// exact integer d^2 / L1 (int kinds; lo == hi, no band).
struct Thresh {
  float lo_f, hi_f;
  int32_t lo_i;          // in iff score <= lo_i - 1 (i.e. score < lo_i)
  double eps, eps2;      // fp64 truth: L2 d2 < eps2, L1 s < eps, cos 1-c < eps
  double tie_rel;        // near-tie band (1e-6)
  int cosine;            // metric is cosine (for kernels shared with L2)
};

struct Dev;   // per-call device workspace (api.cu)

// Statistics counters living in device memory (one struct per call).
struct DevStats {
  unsigned long long key_count;      // membership pairs emitted
  unsigned long long band_pairs;     // fp64 rechecks (all modes)
  unsigned long long near_ties;      // near ties found in MODE_MEMBER
  unsigned long long greedy_evals;   // in-tile + coverage evaluations
  unsigned long long tiles;          // greedy tiles with nc > 0
  unsigned long long tc_tiles_run;   // tensor path: 128 x 256 tiles contracted
  unsigned long long tc_tiles_skip;  //   ... skipped by the tile-level pruning
  unsigned long long tc_chunks_run;  //   128 x 32 accumulator chunks read from TMEM
  unsigned long long tc_chunks_skip; //   ... skipped
  int nonfinite;                     // prep: a NaN/Inf coordinate was seen
  int overflow;                      // fused greedy: a tile's band queue overflowed
};

// A2's non-zero adjacency words as a list (the in-tile graph is sparse on the
// BASELINE workloads: k_resolve_big decides the tile from it).  Entry k =
// {a << 16 | v, word}: word v of candidate a; *count may exceed cap (then
// the list is incomplete and the resolve falls back to the dense words).
struct AdjList {
  uint2* e;
  uint32_t* count;
  uint32_t cap;
};
__device__ __forceinline__ void adj_list_push(const AdjList& L, int64_t a, int64_t v,
                                              uint32_t word) {
  if (word == 0u || L.e == nullptr) return;
  const uint32_t k = atomicAdd(L.count, 1u);
  if (k < L.cap) L.e[k] = make_uint2(((uint32_t)a << 16) | (uint32_t)v, word);
}

struct PairArgs {
  const uint2* rows;        // [n][nu] scoring rows (xhat for cosine)
  const uint2* xrows;       // [n][nu] fp32 rows for the fp64 recheck (== rows except cosine)
  const int32_t* inorm;     // [n] exact int L2 norms (K_L2I)
  int64_t n;
  int nu;                   // units per row (runtime copy of the template NU)
  int d;                    // true dimension (recheck loop bound)
  Thresh th;
  // queries: contiguous [q_begin, q_end) or list qidx[q_begin .. q_end)
  const int32_t* qidx;
  int64_t q_begin, q_end;
  const int32_t* q_end_dev;   // if non-null: q_end = min(q_end, *q_end_dev)
  const int32_t* q_begin_dev; // if non-null: q_begin = min(q_begin, *q_begin_dev)
  // landmarks: point indices lidx[l_begin .. l_end); positions are l_begin-relative + lpos0
  const int32_t* lidx;
  int64_t l_begin, l_end;
  const int32_t* l_end_dev;   // if non-null: l_end = min(l_end, *l_end_dev)
  int64_t lpos0;
  const int32_t* l_total_dev; // if non-null: lpos0 = *l_total_dev - (l_end - l_begin)
                              // (fused greedy tile: the new landmarks are the last ones)
  // outputs
  uint32_t* adj; int adj_words;                 // MODE_ADJ: word v of candidate a at
                                                //   adj[v * (32 * adj_words) + a]
  AdjList nz;                                   // MODE_ADJ: list of the non-zero words
  uint8_t* covered;                             // MODE_MEMBER: covered[p] = 1 for in-ball pairs
  // L1 prefilter (K_L1F, MODE_MEMBER): 8-bit quantised rows, nq 32-bit words
  // per row; qparam = {min, max} of all coordinates (device, fp64)
  const uint32_t* qrows; int nq; const double* qparam;
  unsigned long long* keys; int64_t key_cap; int lbits;   // MODE_MEMBER: (p << lbits) | j
  int64_t* ties; int64_t tie_cap;               // MODE_MEMBER near-tie triples (host-mapped)
  DevStats* stats;
};

// ------------------------------------------------------------ launchers
// All return cudaError_t of the launch; `launches` is incremented per kernel.
cudaError_t launch_prep(const void* X, int dtype, int64_t n, int d, int kind, int nu,
                        uint2* rows, uint2* xhat, int32_t* inorm, DevStats* stats,
                        cudaStream_t s, int64_t* launches);

cudaError_t launch_pairs(int kind, int mode, const PairArgs& a, int64_t q_rows_max,
                         cudaStream_t s, int64_t* launches);

// L1 prefilter: coordinate range -> qparam[0..1],
// then 8-bit rows q = rint((x - min) / s), s = (max - min) / 255, nq words per row.
int l1q_words(int d);   // 0 if the prefilter does not apply (d > 64)
cudaError_t launch_l1_quantize(const float* X, int64_t n, int d, int nq, double* qparam,
                               uint32_t* qrows, cudaStream_t s, int64_t* launches);

// L1 prefilter threshold: with q = rint((x - min)/s)
// every coordinate is within s (1/2 + 1e-6) of min + s q, so
// L1(x, y) >= s (SAD(q_x, q_y) - d (1 + 2e-6)); SAD >= thr proves
// L1 >= eps (1 + 1.001e-6): out, and not a near tie.
__device__ __forceinline__ double l1q_scale(const double* qp) {
  const double r = qp[1] - qp[0];
  return r > 0.0 ? r / 255.0 : 1.0;
}
__device__ __forceinline__ uint32_t l1q_threshold(const double* qp, double eps, int d) {
  const double t = ceil(eps * (1.0 + 1.001e-6) / l1q_scale(qp) + d * (1.0 + 2e-6)) + 1.0;
  return t > 4.0e9 ? 0xffffffffu : (uint32_t)t;
}
__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// L1 on tensor cores ("coarse L1 as a Hamming Gram"): every
// coordinate is binned into B + 1 levels (s_t = (max - min) / (B + 1)) and
// written as a B-byte thermometer code, so the squared L2 distance of two codes
// is the sum of the absolute level differences SADq; since every coordinate
// lies within its bin (1e-9 s_t of slack for the fp64 binning),
// L1(x, y) >= s_t (SADq - d (1 + 2e-9)), and SADq >= cut proves
// L1 >= eps (1 + 4e-6): out, and not a near tie.  Bytes per coordinate B
// (0: the path does not apply): the row (d B bytes + 6 bytes of folded
// constants, tc.cu k_l1t_prep) fills at most three 128-byte K atoms (C5,
// d = 16: B = 19, 20 levels, 310 bytes = ten 32-byte K steps; measured on
// C5, 24 levels leave ~0.26% of the pairs as candidates for the 8-bit bound,
// 20 levels ~0.5%, 16 levels ~1.2%; the contraction took 836 / 810 / 855 ms
// at B = 23 / 19 / 17, same box).
__host__ __device__ __forceinline__ int l1t_bytes_per_coord(int d) {
  // (d <= 16: the 8-bit rows of the candidate filter are <= 4 words, staged
  // for a whole greedy tile in shared memory)
  if (d < 1 || d > 16) return 0;
#ifndef BM_L1T_KB
#define BM_L1T_KB 314   // thermometer + fold bytes per row (<= 3 K atoms)
#endif
  int b = (BM_L1T_KB) / d;
  if (b > 32) b = 32;
  return b;
}
__device__ __forceinline__ int32_t l1t_cut(const double* qp, double eps, int d, int B) {
  const double r = qp[1] - qp[0];
  const double st = r > 0.0 ? r / (double)(B + 1) : 1.0;
  const double c = ceil(eps * (1.0 + 4e-6) / st + (double)d * (1.0 + 2e-9)) + 1.0;
  const double cmax = (double)d * B + 1.0;   // every pair a candidate
  return (int32_t)(c < cmax ? c : cmax);
}

// A3; also resets the per-tile device counters (*ticket = 0, *band_count = 0).
// pruning outputs of A3 (cells.cu): the tile's landmarks sorted by cell rank
// and the chunk / tile cell masks (all null: no pruning)
struct PruneTile {
  const int32_t* cell;
  const int32_t* rank;
  int32_t* col_pt;
  int32_t* col_pos;
  uint32_t* cmask;
  uint32_t* tmask;
};
cudaError_t launch_resolve(const uint32_t* adj, int adj_words, const int32_t* unc,
                           const int32_t* n_unc, int T, int32_t* lm_out, int32_t* L_dev,
                           int32_t* new_lm, int32_t* dL_dev, DevStats* stats,
                           int32_t* ticket, unsigned long long* band_count,
                           cudaStream_t s, int64_t* launches, PruneTile pt_out = PruneTile{});

// A3 for 1024 < T <= kBigT (greedy.cu k_resolve_big): decides the tile from
// A2's non-zero word list when it is complete (sparse rounds), otherwise (or
// with force_dense) from the dense words in sub-tiles of 1024; resets
// *nz.count for the next tile.  pt_out arrays hold T entries (col_pt,
// col_pos), T/32 x 8 (cmask) and T/256 x 8 (tmask) words.
constexpr int kBigT = 8192;
constexpr int64_t kBigNzCap = 8192;   // list entries (= the resolve's shared-memory stage)
cudaError_t launch_resolve_big(const uint32_t* adj, AdjList nz, const int32_t* unc,
                               const int32_t* n_unc, int T, int32_t* lm_out, int32_t* L_dev,
                               int32_t* new_lm, int32_t* dL_dev, DevStats* stats,
                               int32_t* ticket, unsigned long long* band_count, cudaStream_t s,
                               int64_t* launches, PruneTile pt_out, int force_dense);

// Order-preserving compaction of the uncovered list after a tile: keeps
// unc[i], nc <= i < n_unc, with covered[unc[i]] == 0 (single pass, decoupled
// look-back; `state` holds compact_state_words(n) zero-initialised words,
// `ticket` is reset by the resolve kernel of the same tile, `tag` is unique
// per launch within a call and non-zero).
int64_t compact_state_words(int64_t n);
cudaError_t launch_compact_unc(const uint8_t* covered, const int32_t* unc, const int32_t* n_unc,
                               int T, int32_t* unc_next, int32_t* n_unc_next,
                               unsigned long long* state, int32_t* ticket, uint32_t tag,
                               int64_t n, cudaStream_t s, int64_t* launches);

// scan / sort (sort.cu)
size_t scan_temp_bytes(int64_t n);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp,
                               int64_t* total_dev, cudaStream_t s, int64_t* launches);
size_t radix_temp_bytes(int64_t n);
// Stable LSD sort of keys on the concatenation of bit ranges (ranges[0] least
// significant, at most 64 bits in total); result in *keys (may swap with alt).
struct BitRange {
  int lo, hi;  // bits [lo, hi)
};
cudaError_t radix_sort_u64(unsigned long long** keys, unsigned long long** alt, int64_t n,
                           const BitRange* ranges, int nranges, void* temp, cudaStream_t s,
                           int64_t* launches);

// csr / edges (csr.cu)
cudaError_t launch_segment_ptr(const unsigned long long* keys, int64_t m, int shift,
                               unsigned long long mask, int64_t nseg, int64_t* ptr,
                               cudaStream_t s, int64_t* launches);
cudaError_t launch_unpack_low(const unsigned long long* keys, int64_t m,
                              unsigned long long mask, int32_t* out, cudaStream_t s,
                              int64_t* launches);
cudaError_t launch_unpack_high(const unsigned long long* keys, int64_t m, int32_t* out,
                               cudaStream_t s, int64_t* launches);
cudaError_t launch_rekey_landmark_major(const unsigned long long* pm_keys, int64_t m, int lbits,
                                        int pbits, unsigned long long* out, cudaStream_t s,
                                        int64_t* launches);
// D1 row-union emission (edges.cu): items of <= 512 members per landmark row
size_t row_items_temp_bytes(int64_t L);
cudaError_t launch_row_items(const int64_t* ball_ptr, int64_t L, int64_t* cnt, cudaStream_t s,
                             int64_t* launches);
cudaError_t launch_item_rows(const int64_t* item_off, const int64_t* cnt, int64_t L,
                             int32_t* item_row, cudaStream_t s, int64_t* launches);
cudaError_t launch_row_pairs(const int64_t* ball_ptr, const int32_t* ball_idx,
                             const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                             const int64_t* item_off, const int32_t* item_row, int64_t n_items,
                             int lbits, unsigned long long* keys, int64_t cap,
                             unsigned long long* kcount, unsigned long long* npairs,
                             cudaStream_t s, int64_t* launches);
cudaError_t launch_pair_counts(const int64_t* pt_ptr, int64_t n, int64_t* cnt, cudaStream_t s,
                               int64_t* launches);
cudaError_t launch_pair_emit(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n,
                             const int64_t* off, int lbits, unsigned long long* keys,
                             cudaStream_t s, int64_t* launches);
cudaError_t launch_unique_flags(const unsigned long long* keys, int64_t m, int64_t* flags,
                                cudaStream_t s, int64_t* launches);
cudaError_t launch_unique_scatter(const unsigned long long* keys, int64_t m,
                                  const int64_t* pos, int lbits, int32_t* edges,
                                  cudaStream_t s, int64_t* launches);
// cells.cu: tile-level pruning of the tensor-core membership contraction
constexpr int kPruneCells = 256;
constexpr int kPruneSplit = 32;  // slices per cell in the centre / radius passes
struct PruneState {
  int32_t* cell;        // [n] cell of each point
  int32_t* rank;        // [K] position of each cell in the pivot chain
  float* pdist;         // [K*K] pivot distances (scratch)
  int32_t* perm;        // [n] permuted row r -> point
  int64_t* seg;         // [K+1] rank segments of perm
  double* center;       // [K*d]
  double* radius;       // [K] (-1: empty cell)
  double* part;         // [K][kPruneSplit][128] per-slice coordinate sums (scratch)
  unsigned long long* rad2;   // [K] bits of the max squared distance to the centre
  uint32_t* near;       // [K][K/32]
  uint32_t* bmask;      // [ceil(n/128)][K/32] cells near some row of the block
  uint8_t* xop_perm;    // [n][row_bytes] the A operand in permuted order
  double* nrm_perm;     // [n] norms in permuted order
  int32_t* col_pt;      // [1024] the tile's landmarks sorted by cell rank
  int32_t* col_pos;     // [1024] their positions in the tile (key positions)
  uint32_t* cmask;      // [32 chunks][K/32] cells of each 32-column chunk
  uint32_t* tmask;      // [4 tiles][K/32] cells of each 256-column tile
  uint32_t* act;        // [ceil(n/128)] per row block: bit 8 t + c = chunk c of tile t may
                        // hold an in-ball pair (from bmask and cmask, per greedy tile,
                        // folded by the landmark-operand launch, tc.cu)
};
cudaError_t cell_order(const float* xrows, int xstride, int d, int64_t n, int32_t* cell,
                       int32_t* rank, float* pdist, unsigned long long** keys,
                       unsigned long long** alt, void* sort_temp, int32_t* perm, cudaStream_t s,
                       int64_t* launches);
cudaError_t prune_prepare(const float* xrows, int xstride, int d, int64_t n, double eps,
                          const uint8_t* xop, int64_t row_bytes, const double* nrm, PruneState& ps,
                          void* sort_temp, unsigned long long* keys, unsigned long long* alt,
                          cudaStream_t s, int64_t* launches);

// fps.cu (NEXT-2)
int fps_max_candidates();
// perm (may be null): the points in spatial (cell) order; each warp then owns
// a contiguous run of it and skips a landmark whose distance to the run's
// bounding ball proves no running minimum can change (float L2 / L1, d <= 128)
cudaError_t launch_fps(const uint2* rows, const int32_t* inorm, int nu, int d, int kind, int64_t n,
                       double thr, int64_t start, double* mind, int32_t* seq, int32_t* L_out,
                       double* cval, int64_t* cidx, const int32_t* perm, cudaStream_t s);
cudaError_t launch_fps_keys(const int32_t* seq, int64_t L, unsigned long long* keys,
                            cudaStream_t s, int64_t* launches);

// color.cu (NEXT-1)
cudaError_t launch_color_reduce(const int64_t* ball_ptr, const int32_t* ball_idx, int64_t L,
                                const void* values, int is_int, int agg, double* out,
                                cudaStream_t s);
cudaError_t launch_color_keys(const int64_t* ball_ptr, const int32_t* ball_idx, int64_t L,
                              const void* values, int is_int, unsigned long long* keys,
                              cudaStream_t s);
cudaError_t launch_color_order(const int64_t* ball_ptr, int64_t L, const unsigned long long* keys,
                               int is_int, int agg, double alpha, double* out, cudaStream_t s);
// skeleton.cu (NEXT-3)
cudaError_t launch_simplex_counts(const int64_t* pt_ptr, int64_t n, int r, int64_t* cnt,
                                  cudaStream_t s);
cudaError_t launch_simplex_emit(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int r,
                                int lbits, const int64_t* off, unsigned long long* keys,
                                cudaStream_t s);
size_t simplex_unique_temp_bytes(int64_t m);
cudaError_t launch_simplex_unique(const unsigned long long* keys, int64_t m, int r, int lbits,
                                  int32_t* out, int64_t cap, int64_t* total, void* temp,
                                  cudaStream_t s);

// edges.cu, step C for n * L <= kCsrBitmapMaxBits: both CSRs from bit matrices
constexpr int64_t kCsrBitmapMaxBits = (int64_t)1 << 30;
int64_t csr_bitmap_words(int64_t n, int64_t L);
size_t csr_bitmap_temp_bytes(int64_t n, int64_t L);
cudaError_t csr_from_keys_bitmap(const unsigned long long* keys, int64_t m, int64_t n, int64_t L,
                                 uint32_t* bits, void* temp, int64_t* pt_ptr, int32_t* pt_lm,
                                 int64_t* ball_ptr, int32_t* ball_idx, cudaStream_t s,
                                 int64_t* launches);
// edges.cu: bitmap path for L <= kEdgeBitmapMaxL, keys path (sort + unique) above
constexpr int64_t kEdgeBitmapMaxL = 4096;
int64_t edge_bitmap_words(int64_t L);
// triangular bit matrix for 4096 < L (bytes = 4 * tri_bitmap_words(L))
int64_t tri_bitmap_words(int64_t L);
cudaError_t launch_tri_bits(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                            uint32_t* bits, unsigned long long* npairs, cudaStream_t s,
                            int64_t* launches);
cudaError_t launch_tri_rowcount(const uint32_t* bits, int64_t L, int64_t* cnt, cudaStream_t s,
                                int64_t* launches);
cudaError_t launch_tri_emit(const uint32_t* bits, int64_t L, const int64_t* off, int32_t* edges,
                            cudaStream_t s, int64_t* launches);
size_t edge_lb_temp_bytes(int64_t items);
cudaError_t launch_edge_bits(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                             uint32_t* bits, unsigned long long* npairs, cudaStream_t s,
                             int64_t* launches);
cudaError_t launch_bits_compact(const uint32_t* bits, int64_t L, int32_t* edges, int64_t cap,
                                int64_t* total, void* temp, cudaStream_t s, int64_t* launches);
cudaError_t launch_unique_compact(const unsigned long long* keys, int64_t m, int lbits,
                                  int32_t* edges, int64_t* total, void* temp, cudaStream_t s,
                                  int64_t* launches);
cudaError_t launch_copy_i32(const int32_t* src, int32_t* dst, int64_t n, cudaStream_t s,
                            int64_t* launches);

// resolve-only diagnostic kernel
cudaError_t launch_resolve_debug(const uint32_t* adj, int adj_words, int nc, uint8_t* lm,
                                 cudaStream_t s, int64_t* launches);

}  // namespace bm

namespace bm {
// Instantiated register-row widths of the CUDA-core pair kernel (8-byte units);
// 0 = wide variant (rows re-read from L1/global).
// Index of the current device for per-device caches of launch settings
// (function attributes and occupancy are per context, so a process driving
// several GPUs must not reuse one device's values on another).
constexpr int kMaxDevices = 64;
inline int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

inline int pick_nu(int nu_needed) {
  static const int widths[] = {1, 2, 4, 5, 8, 12, 16, 24, 32};
  for (int w : widths)
    if (nu_needed <= w) return w;
  return 0;
}
}  // namespace bm
