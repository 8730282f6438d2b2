// tc.cuh — interface of the tcgen05 membership contraction (tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace bm {
namespace tc {

enum TcKind : int { TC_TF32 = 0, TC_U8 = 1, TC_S8 = 2 };
enum TcMode : int {
  TC_MODE_MEMBER = 0,
  TC_MODE_GRAM = 1,
  TC_MODE_PROBE_LDONLY = 2,   // diagnostics: epilogue reads TMEM, no classification
  TC_MODE_PROBE_NOLD = 3,     // diagnostics: epilogue releases buffers without reading
  TC_MODE_ADJ = 4,            // A2: candidate x candidate adjacency bits of a greedy tile
  TC_MODE_L1T = 5             // B for L1 (TC_S8): thermometer-code Gram, sign of the folded
                              //   accumulator = "not proven out"; 8-bit SAD, then fp64 (B')
};

// Per-row thresholds of the contraction, shared by the point
// rows and the greedy tile's candidate rows.
struct RowParams {
  int tf32, cosine;
  double C2, eps, eps2, tau, m;
  int32_t lo_i;
};

// Operand geometry (host side).
struct TcPlan {
  int kind;            // TcKind
  const void* xop;     // [n][row_bytes] point operand (tf32-rounded fp32 or int8 bytes)
  void* lop;           // [l_rows][row_bytes] landmark operand (gathered rows, zero padded)
  int64_t n_rows;      // n (TMA zero-fills rows beyond)
  int64_t n_pad;       // row-constant array length (multiple of the CTA row block)
  int64_t l_rows;      // padded landmark count (multiple of BN)
  int64_t row_bytes;   // bytes per operand row (multiple of 16)
  int64_t k_elems;     // row_bytes / element size
  int katoms;          // ceil(row_bytes / 128)
  int num_sms;
  const float* ones;   // tf32: [128][8] constant A tile {1,1,1,0,0,0,0,0} (column-constant fold)
  int cosine;          // tf32: operands are x / |x| and the contraction scores cosine similarity
};

struct TcArgs {
  int64_t n, L;                              // L: landmark columns (host value)
  const int32_t* l_count_dev;                // if non-null: columns = *l_count_dev (fused tile)
  const int32_t* l_total_dev;                // fused tile: position base = *l_total_dev - columns
  int64_t n_mblk;                            // filled by the launcher
  int ksteps;                                // 32-byte K steps to issue
  int lbits;                                 // key = point << lbits | landmark position
  // per-row / per-column constants
  const float* row_lo;
  const float* row_hi;
  const int32_t* row_r;
  const float* col_a;    // tf32: in-test offset d_j (acc' - d_j > row_hi proves "in")
  const float* col_b;    // tf32: column constant cb_j folded into the MMA (diagnostics)
  const float* colk;     // tf32: [l_rows][8] {-cb_hi, -cb_mid, -cb_lo, 0...}: B operand of
                         //       the fold MMA, so the accumulator is acc' = x.l - cb_j
  const int32_t* col_c;
  // outputs
  unsigned long long* keys;
  unsigned long long* key_count;
  int64_t key_cap;
  // B' (tf32): band pairs are re-decided inside the epilogue with the oracle's
  // fp64 formula on the original fp32 rows
  const float* xrows;  // [rows][xstride] fp32 coordinates (first d used)
  int xstride;
  int d;
  double eps, eps2, tie_rel;
  double tie_abs;          // tie_rel * eps (precomputed: no fp64 multiply in the epilogue)
  const int32_t* lm_idx;   // landmark column -> point index
  int cosine;              // recheck with the cosine formula (else Euclidean; L1T: Manhattan)
  // L1 on tensor cores (TC_MODE_L1T, l1t != 0): candidates (SADq < cut, the
  // sign of the folded accumulator) pass the 8-bit SAD filter of the
  // CUDA-core path (qrows: nq words per point, qparam: coordinate range)
  // before the fp64 decision
  int l1t;
  const uint32_t* qrows;
  int nq;
  const double* qparam;
  int64_t* ties;           // near-tie triples (point, landmark point, decision)
  int64_t tie_cap;
  DevStats* stats;         // band_pairs / near_ties counters
  uint32_t* gram;      // debug: raw accumulators [n][L]
  uint32_t* adj;       // TC_MODE_ADJ: word-major adjacency, word v of candidate a at adj[v*adj_T + a]
  int adj_T;
  AdjList nz;          // TC_MODE_ADJ: the non-zero words as a list (internal.cuh)
  uint8_t* covered;    // fused greedy: covered[p] = 1 for every in-ball pair (may be null)
  unsigned long long* trace;   // diagnostics: [grid][16] %globaltimer stamps (null: off)
  unsigned long long* wtrace;  // diagnostics: [grid][16] wait cycles per role (null: off)
  unsigned long long* tline;   // diagnostics: CTA 0's per-tile clock64 stamps [512][5] (null: off)
  // tile-level pruning (cells.cu; all null when off): A rows are permuted
  // (row r is point row_pt[r]); columns are the tile's landmarks sorted by
  // cell (key position lpos0 + col_pos[j]); a 256-column tile / 32-column
  // chunk whose cell mask meets no cell of the row block's near mask is
  // skipped (no MMA / no TMEM read)
  const int32_t* row_pt;
  const int32_t* col_pos;
  const uint32_t* act;     // [row block][1 + act_words]: word 0 bit t = tile t is live; then
                           //   bit 8 t + c of the chunk words = chunk c of tile t is live
  int act_words;           // chunk words per row block (tiles / 4 rounded up, <= 8)
  const uint32_t* act_bmask;   // its inputs (cells.cu), folded by the landmark-operand
  const uint32_t* act_cmask;   //   launch of each greedy tile
  const uint32_t* act_tmask;
};

int tc_bn_for(int kind, int katoms);
int tc_rows_for(int kind, int katoms);
bool tc_supported(int kind, int katoms);

// fill the [128][8] constant A tile of the column-constant fold ({1,1,1,0,...})
cudaError_t launch_tc_prep(const void* X, int dtype, int64_t n, int d, const TcPlan& P,
                           void* nrm, DevStats* stats, cudaStream_t s, int64_t* launches);
cudaError_t launch_tc_rows(const TcPlan& P, const void* nrm, int64_t n, double C2, double eps2,
                           double tau, int32_t lo_i, TcArgs& a, cudaStream_t s,
                           int64_t* launches);
// cosine: uniform row thresholds around 1 - eps with margin m (zero rows: every pair rechecked)
cudaError_t launch_tc_rows_cos(const TcPlan& P, const void* nrm, int64_t n, double eps, double m,
                               TcArgs& a, cudaStream_t s, int64_t* launches);
cudaError_t launch_tc_landmarks(const TcPlan& P, const void* nrm, const int32_t* lm, int64_t L,
                                double C2, TcArgs& a, cudaStream_t s, int64_t* launches);
// Fused greedy tile: gather the *l_count_dev new landmarks' operand rows into
// P.lop (rows up to P.l_rows zero-filled) and their column constants.
cudaError_t launch_tc_tile_landmarks(const TcPlan& P, const void* nrm, const int32_t* new_lm,
                                     const int32_t* l_count_dev, double C2, TcArgs& a,
                                     cudaStream_t s, int64_t* launches);
cudaError_t launch_tc(const TcPlan& P, const TcArgs& a, cudaStream_t s, int64_t* launches);
// A2 on tensor cores: gather the tile's candidates (first min(T, *n_unc) of unc)
// into Pc.xop (= Pc.lop) with their row and column constants, then one
// contraction candidates x candidates with the adjacency epilogue.
cudaError_t launch_tc_tile_cand(const TcPlan& P, const TcPlan& Pc, const void* nrm,
                                const int32_t* unc, const int32_t* n_unc_dev, int T, double C2,
                                const RowParams& rp, TcArgs& ac, cudaStream_t s,
                                int64_t* launches);
// L1 on tensor cores (internal.cuh l1t_bytes_per_coord): point operand rows
// (-2 x thermometer bits, then the folded constants 1,1,1 and n_p - cut in
// three bytes) and n_p = sum of the levels; qparam from launch_l1_quantize.
cudaError_t launch_l1t_prep(const float* X, int64_t n, int d, const TcPlan& P,
                            const double* qparam, double eps, int32_t* nrm, cudaStream_t s,
                            int64_t* launches);
// ... and the greedy tile's landmark operand (thermometer bits, n_l in three
// bytes, then 1,1,1), rows >= *l_count_dev zero
cudaError_t launch_l1t_tile_landmarks(const TcPlan& P, const int32_t* nrm, const int32_t* new_lm,
                                      const int32_t* l_count_dev, int d, cudaStream_t s,
                                      int64_t* launches);
cudaError_t launch_tc_adj(const TcPlan& Pc, const TcArgs& ac, cudaStream_t s, int64_t* launches);
// diagnostics: the contraction with a probe epilogue (TC_MODE_PROBE_*), tf32 K <= 64 only
cudaError_t launch_tc_probe(const TcPlan& P, const TcArgs& a, int mode, cudaStream_t s);

}  // namespace tc
}  // namespace bm
