// greedy.cu — steps A1/A3 of the blocked greedy eps-net.
//
// The paper's greedy walks the points in order and makes the
// next uncovered point a landmark.  Blocked form: the list `unc` holds the
// still-uncovered point indices in ascending order; its first nc = min(T, |unc|)
// entries are the tile's candidates (A1 is a pointer offset).  A2 (MODE_ADJ in
// pairs_impl.cuh) produced the strictly-lower adjacency bits among them.  A3
// (k_resolve) decides them in order — candidate a is a landmark iff no earlier
// candidate landmark b < a is adjacent to it — which is exactly the greedy
// restricted to the tile, because every landmark from earlier tiles has
// already removed its ball from `unc`.  The result is independent of T
// (lexicographically-first maximal independent set).  A4 (MODE_COVER) marks
// the remaining unc[nc..) against the new landmarks and k_scan_blocks /
// k_compact keep the survivors in order.
#include "internal.cuh"

namespace bm {

constexpr unsigned FULLMASK = 0xffffffffu;

// One CTA, warp w owns candidates 32w .. 32w+31.  Warp w folds in the landmark
// words of earlier warps as they become ready (a wavefront through shared
// memory flags), then resolves its own 32 candidates by a ballot fixed point.
__device__ __forceinline__ uint32_t resolve_tile_core(const uint32_t* __restrict__ adj,
                                                      int adj_words, int nc,
                                                      volatile uint32_t* lmw,
                                                      volatile int* ready) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nb = (nc + 31) >> 5;
  if (w >= nb) return 0u;
  const int a = tid;
  const bool valid = a < nc;
  uint32_t wv[32];
#pragma unroll
  for (int v = 0; v < 32; ++v) wv[v] = (valid && v < w) ? adj[(int64_t)a * adj_words + v] : 0u;
  uint32_t inrow = valid ? (adj[(int64_t)a * adj_words + w] & ((1u << lane) - 1u)) : 0u;
  bool conflict = false;
#pragma unroll
  for (int v = 0; v < 32; ++v) {
    if (v < w) {
      while (ready[v] == 0) {
      }
      conflict = conflict || ((wv[v] & lmw[v]) != 0u);
    }
  }
  unsigned undecided = __ballot_sync(FULLMASK, valid && !conflict);
  unsigned S = 0u;
  while (undecided) {
    const bool me = (undecided >> lane) & 1u;
    const bool is_lm = me && !(inrow & S) && !(inrow & undecided);
    const bool not_lm = me && (inrow & S);
    const unsigned ns = __ballot_sync(FULLMASK, is_lm);
    const unsigned nn = __ballot_sync(FULLMASK, not_lm);
    S |= ns;
    undecided &= ~(ns | nn);
  }
  if (lane == 0) {
    lmw[w] = S;
    __threadfence_block();
    ready[w] = 1;
  }
  return S;
}

__global__ void __launch_bounds__(1024) k_resolve(const uint32_t* __restrict__ adj, int adj_words,
                                                  const int32_t* __restrict__ unc,
                                                  const int32_t* __restrict__ n_unc_dev, int T,
                                                  int32_t* __restrict__ lm_out,
                                                  int32_t* __restrict__ L_dev,
                                                  int32_t* __restrict__ new_lm,
                                                  int32_t* __restrict__ dL_dev, DevStats* stats) {
  __shared__ volatile uint32_t lmw[32];
  __shared__ volatile int ready[32];
  __shared__ int wpre[33];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int n_unc = *n_unc_dev;
  const int nc = min(T, n_unc);
  if (nc == 0) {
    if (tid == 0) *dL_dev = 0;
    return;
  }
  if (tid < 32) ready[tid] = 0;
  __syncthreads();
  resolve_tile_core(adj, adj_words, nc, lmw, ready);
  __syncthreads();
  const int nb = (nc + 31) >> 5;
  if (tid < 32) {
    int c = tid < nb ? __popc(lmw[tid]) : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += v;
    }
    wpre[tid + 1] = incl;
    if (tid == 0) wpre[0] = 0;
  }
  __syncthreads();
  const int L0 = *L_dev;
  if (w < nb && tid < nc) {
    const uint32_t S = lmw[w];
    if ((S >> lane) & 1u) {
      const int pos = wpre[w] + __popc(S & ((1u << lane) - 1u));
      const int32_t pt = unc[tid];
      new_lm[pos] = pt;
      lm_out[L0 + pos] = pt;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int dL = wpre[nb];
    *dL_dev = dL;
    *L_dev = L0 + dL;
    stats->greedy_evals += (unsigned long long)nc * (unsigned long long)(nc - 1) / 2ull +
                           (unsigned long long)(n_unc - nc) * (unsigned long long)dL;
    stats->tiles += 1ull;
  }
}

cudaError_t launch_resolve(const uint32_t* adj, int adj_words, const int32_t* unc,
                           const int32_t* n_unc, int T, int32_t* lm_out, int32_t* L_dev,
                           int32_t* new_lm, int32_t* dL_dev, DevStats* stats, cudaStream_t s,
                           int64_t* launches) {
  ++*launches;
  k_resolve<<<1, 1024, 0, s>>>(adj, adj_words, unc, n_unc, T, lm_out, L_dev, new_lm, dL_dev,
                               stats);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(1024) k_resolve_debug(const uint32_t* __restrict__ adj,
                                                        int adj_words, int nc, uint8_t* lm) {
  __shared__ volatile uint32_t lmw[32];
  __shared__ volatile int ready[32];
  const int tid = threadIdx.x;
  if (tid < 32) ready[tid] = 0;
  __syncthreads();
  resolve_tile_core(adj, adj_words, nc, lmw, ready);
  __syncthreads();
  if (tid < nc) lm[tid] = (lmw[tid >> 5] >> (tid & 31)) & 1u;
}

cudaError_t launch_resolve_debug(const uint32_t* adj, int adj_words, int nc, uint8_t* lm,
                                 cudaStream_t s, int64_t* launches) {
  ++*launches;
  k_resolve_debug<<<1, 1024, 0, s>>>(adj, adj_words, nc, lm);
  return cudaGetLastError();
}

// Exclusive scan of the per-CTA kept counts of the coverage pass (one CTA).
__global__ void __launch_bounds__(1024) k_scan_blocks(const int32_t* __restrict__ cnt, int nblk,
                                                      int32_t* __restrict__ off,
                                                      int32_t* __restrict__ total) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblk; base += 1024) {
    const int i = base + tid;
    const int v = i < nblk ? cnt[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int s = wsum[lane];
      int si = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULLMASK, si, o);
        if (lane >= o) si += t;
      }
      wsum[lane] = si - s;
    }
    __syncthreads();
    const int excl = carry + wsum[w] + incl - v;
    if (i < nblk) off[i] = excl;
    __syncthreads();
    if (tid == 1023) carry = excl + v;
    __syncthreads();
  }
  if (tid == 0) *total = carry;
}

// Order-preserving scatter of the survivors: unc_next[off[b] + rank] = unc[nc + i].
__global__ void __launch_bounds__(256) k_compact(const uint8_t* __restrict__ keep,
                                                 const int32_t* __restrict__ off, int blk_rows,
                                                 const int32_t* __restrict__ unc,
                                                 const int32_t* __restrict__ n_unc_dev, int T,
                                                 int32_t* __restrict__ unc_next) {
  __shared__ int wsum[8];
  const int n_unc = *n_unc_dev;
  const int nc = min(T, n_unc);
  const int64_t m = n_unc - nc;
  const int64_t b0 = (int64_t)blockIdx.x * blk_rows;
  if (b0 >= m) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = blk_rows / 256;     // consecutive items per thread
  const int64_t i0 = b0 + (int64_t)tid * per;
  int c = 0;
  for (int k = 0; k < per; ++k) {
    const int64_t i = i0 + k;
    if (i < m) c += keep[i];
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(FULLMASK, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int wpre = 0;
  for (int k = 0; k < w; ++k) wpre += wsum[k];
  int pos = off[blockIdx.x] + wpre + incl - c;
  for (int k = 0; k < per; ++k) {
    const int64_t i = i0 + k;
    if (i < m && keep[i]) unc_next[pos++] = unc[nc + i];
  }
}

cudaError_t launch_compact_unc(const uint8_t* keep, const int32_t* blk_count, int nblk,
                               int blk_rows, const int32_t* unc, const int32_t* n_unc, int T,
                               int32_t* blk_off, int32_t* unc_next, int32_t* n_unc_next,
                               cudaStream_t s, int64_t* launches) {
  k_scan_blocks<<<1, 1024, 0, s>>>(blk_count, nblk, blk_off, n_unc_next);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_compact<<<nblk, 256, 0, s>>>(keep, blk_off, blk_rows, unc, n_unc, T, unc_next);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace bm
