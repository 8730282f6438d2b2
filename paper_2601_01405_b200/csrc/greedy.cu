// greedy.cu — steps A1/A3/A4 of the blocked greedy eps-net.
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
// (lexicographically-first maximal independent set).  The tile's membership
// pass (step B for the new landmarks, over all points) sets covered[p] for
// every point in a new ball; k_compact keeps the survivors unc[nc..) with
// covered == 0, in order (A4), in one pass with a decoupled look-back.
#include "internal.cuh"

namespace bm {

constexpr unsigned FULLMASK = 0xffffffffu;

// The tile's adjacency words are staged in shared memory by the whole CTA
// (coalesced), then ONE warp resolves the 32 blocks of 32 candidates in order:
// lane l holds candidate 32w + l of block w; it folds in the landmark words of
// the earlier blocks (lane v keeps block v's word, read by shuffles), then the
// block's own 32 candidates are decided by a ballot fixed point.  (Measured:
// a 32-warp wavefront that handed each block's word to the next warp through
// shared-memory flags or mbarriers took ~20 us per 1024-candidate tile, almost
// all of it cross-warp hand-off latency.)
// adj: word v of candidate a at adj[v * gstride + a] (global); sadj: the
// staged lower triangle, word v of candidate a at sadj[v * sstride + a];
// preb (optional, shared): bit a set = candidate a is already dominated by a
// landmark outside this block of <= 1024 candidates (k_resolve_big's sub-tiles).
__device__ __forceinline__ void resolve_core(const uint32_t* __restrict__ adj, int64_t gstride,
                                             int nc, volatile uint32_t* lmw, uint32_t* sadj,
                                             int sstride, const uint32_t* preb) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nb = (nc + 31) >> 5;
  // stage the lower triangle (word v of candidate a is needed for v <= a / 32):
  // thread a issues its (up to 32) independent loads before any store
  if (tid < nc) {
    const int wa = tid >> 5;
    uint32_t x[32];
#pragma unroll
    for (int v = 0; v < 32; ++v) x[v] = v <= wa ? __ldcg(adj + (int64_t)v * gstride + tid) : 0u;
#pragma unroll
    for (int v = 0; v < 32; ++v)
      if (v <= wa) sadj[v * sstride + tid] = x[v];
  }
  __syncthreads();
  if (tid < 32) {
    for (int w = 0; w < nb; ++w) {
      const int a = 32 * w + lane;
      const bool valid = a < nc;
      // fold in the earlier blocks' landmark words (independent loads, 8 in flight)
      uint32_t conf = 0u;
      if (valid) {
        if (preb) conf = (preb[w] >> lane) & 1u;
        for (int v0 = 0; v0 < w; v0 += 8) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int v = v0 + k;
            if (v < w) conf |= sadj[v * sstride + a] & lmw[v];
          }
        }
      }
      const uint32_t inrow = valid ? (sadj[w * sstride + a] & ((1u << lane) - 1u)) : 0u;
      unsigned undecided = __ballot_sync(FULLMASK, valid && conf == 0u);
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
      if (lane == 0) lmw[w] = S;
      __syncwarp();
    }
  }
}

// sadj: [nb][T] words, T = 32 * adj_words.
__device__ __forceinline__ void resolve_tile_core(const uint32_t* __restrict__ adj,
                                                  int adj_words, int nc, volatile uint32_t* lmw,
                                                  uint32_t* sadj) {
  resolve_core(adj, 32 * adj_words, nc, lmw, sadj, 32 * adj_words, nullptr);
}

__global__ void __launch_bounds__(1024) k_resolve(const uint32_t* __restrict__ adj, int adj_words,
                                                  const int32_t* __restrict__ unc,
                                                  const int32_t* __restrict__ n_unc_dev, int T,
                                                  int32_t* __restrict__ lm_out,
                                                  int32_t* __restrict__ L_dev,
                                                  int32_t* __restrict__ new_lm,
                                                  int32_t* __restrict__ dL_dev, DevStats* stats,
                                                  int32_t* __restrict__ ticket,
                                                  unsigned long long* __restrict__ band_count,
                                                  PruneTile pt_out) {
  __shared__ volatile uint32_t lmw[32];
  __shared__ int wpre[33];
  __shared__ uint32_t skey[1024];      // pruning: positions in cell-rank order
  __shared__ uint32_t scm[32 * 8];     // pruning: cell masks of the 32-column chunks
  __shared__ int shist[256];           // pruning: landmarks per cell rank, then slots
  extern __shared__ uint32_t sadj[];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  pdl_wait();
  pdl_trigger();   // a single CTA
  const int n_unc = *n_unc_dev;
  const int nc = min(T, n_unc);
  if (tid == 0) {
    if (ticket) *ticket = 0;
    if (band_count) *band_count = 0ull;
  }
  if (nc == 0) {
    if (tid == 0) *dL_dev = 0;
    return;
  }
  resolve_tile_core(adj, adj_words, nc, lmw, sadj);
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
  const bool prune = pt_out.cell != nullptr;
  if (prune) {
    if (tid < 256) shist[tid] = 0;
    if (tid < 32 * 8) scm[tid] = 0u;
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
  if (prune) {
    // the new landmarks grouped by cell rank (counting sort; the order inside
    // a cell only affects which chunk a landmark lands in, never a result:
    // keys carry the original positions) and the cell masks of every
    // 32-column chunk / 256-column tile
    int my_rank = -1, my_pos = -1;
    if (w < nb && tid < nc) {
      const uint32_t S = lmw[w];
      if ((S >> lane) & 1u) {
        my_pos = wpre[w] + __popc(S & ((1u << lane) - 1u));
        my_rank = pt_out.rank[pt_out.cell[unc[tid]]];
        atomicAdd(&shist[my_rank], 1);
      }
    }
    __syncthreads();
    if (tid < 32) {   // exclusive scan of the 256 counts (8 per lane)
      int v[8], t = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = shist[tid * 8 + i];
        t += v[i];
      }
      int incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(FULLMASK, incl, o);
        if (lane >= o) incl += u;
      }
      int run = incl - t;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        shist[tid * 8 + i] = run;
        run += v[i];
      }
    }
    __syncthreads();
    if (my_rank >= 0) skey[atomicAdd(&shist[my_rank], 1)] = (uint32_t)my_pos;
    __syncthreads();
    const int dL = wpre[nb];
    if (tid < dL) {
      const int src = (int)skey[tid];
      const int32_t p = new_lm[src];   // written above by this CTA
      pt_out.col_pt[tid] = p;
      pt_out.col_pos[tid] = src;
      const int c = pt_out.cell[p];
      atomicOr(&scm[(tid >> 5) * 8 + (c >> 5)], 1u << (c & 31));
    }
    __syncthreads();
    // (only the tile's chunks: the masks are allocated for T rounded up to
    // 256 columns, api.cu; a T = 256 tile has 8 chunks and one 256-column
    // tile, and writing all 32 / 4 of them overran into the next buffer)
    const int tq = ((T + 255) / 256) * 256;
    if (tid < (tq / 32) * 8) pt_out.cmask[tid] = scm[tid];
    if (tid < (tq / 256) * 8) {
      const int t = tid >> 3, wd = tid & 7;
      uint32_t v = 0u;
      for (int c = 0; c < 8; ++c) v |= scm[(t * 8 + c) * 8 + wd];
      pt_out.tmask[tid] = v;
    }
  }
  if (tid == 0) {
    const int dL = wpre[nb];
    *dL_dev = dL;
    *L_dev = L0 + dL;
    stats->greedy_evals += (unsigned long long)nc * (unsigned long long)(nc - 1) / 2ull;
    stats->tiles += 1ull;
  }
}

__global__ void __launch_bounds__(1024) k_resolve_debug(const uint32_t* __restrict__ adj,
                                                        int adj_words, int nc, uint8_t* lm) {
  __shared__ volatile uint32_t lmw[32];
  extern __shared__ uint32_t sadj[];
  const int tid = threadIdx.x;
  resolve_tile_core(adj, adj_words, nc, lmw, sadj);
  __syncthreads();
  if (tid < nc) lm[tid] = (lmw[tid >> 5] >> (tid & 31)) & 1u;
}

// ---------------------------------------------------------------------------
// A3 for tiles of 1024 < T <= kBigT candidates (k_resolve_big, one CTA).
//
// Sparse path (the BASELINE workloads: a candidate has an earlier in-tile
// neighbour with probability ~T x ball size / n): A2 also listed its non-zero
// lower-triangle words (AdjList).  A candidate with no listed word has no
// earlier neighbour and is a landmark; the "contested" rest are decided by
// rounds: an undecided candidate with a landmark neighbour is covered, one
// whose earlier neighbours are all decided non-landmarks is a landmark.  The
// smallest undecided candidate is decided in every round (its neighbours are
// all earlier), so the rounds reproduce the in-order greedy exactly; they stop
// when every candidate is decided (usually 1-3 rounds).
// Dense path (list overflow, or more than kBigRounds rounds): the tile is
// resolved in sub-tiles of 1024 candidates in order, each first folding in
// its rows' words against the landmarks of the earlier sub-tiles (coalesced
// loads of the word-major matrix), then the in-order core above.
// Output as k_resolve: landmarks appended in order, new_lm / counts, and with
// pruning the landmarks sorted by cell rank with chunk / tile cell masks.
constexpr int kBigW = kBigT / 32;
constexpr uint32_t kBigNz = (uint32_t)kBigNzCap;   // list entries staged in shared memory
constexpr int kBigRounds = 48;
struct BigSmem {
  static constexpr int BITS = 0;                               // 5 x kBigW words
  static constexpr int WPRE = BITS + 5 * kBigW * 4;            // kBigW + 1 ints
  static constexpr int REG = (WPRE + (kBigW + 1) * 4 + 15) & ~15;
  static constexpr int REG_BYTES = 32 * 1024 * 4;              // sadj (dense) / entries (sparse)
  static constexpr int SKEY = REG + REG_BYTES;                 // kBigT words
  static constexpr int SPT = SKEY + kBigT * 4;                 // kBigT points
  static constexpr int SCM = SPT + kBigT * 4;                  // (kBigT / 32) x 8 words
  static constexpr int SHIST = SCM + kBigW * 8 * 4;            // 256 ints
  static constexpr int MISC = SHIST + 256 * 4;                 // 64 words
  static constexpr int TOTAL = MISC + 64 * 4;
};
static_assert(kBigNz * 8 <= BigSmem::REG_BYTES, "sparse entries fit the shared region");

__global__ void __launch_bounds__(1024) k_resolve_big(
    const uint32_t* __restrict__ adj, AdjList nz, const int32_t* __restrict__ unc,
    const int32_t* __restrict__ n_unc_dev, int T, int32_t* __restrict__ lm_out,
    int32_t* __restrict__ L_dev, int32_t* __restrict__ new_lm, int32_t* __restrict__ dL_dev,
    DevStats* stats, int32_t* __restrict__ ticket, unsigned long long* __restrict__ band_count,
    PruneTile pt_out, int force_dense) {
  extern __shared__ __align__(16) uint8_t bsm[];
  uint32_t* lmb = reinterpret_cast<uint32_t*>(bsm + BigSmem::BITS);   // landmark bits
  uint32_t* decb = lmb + kBigW;                                        // decided bits
  uint32_t* killb = decb + kBigW;                                      // round: has landmark nb
  uint32_t* blkb = killb + kBigW;                                      // round: undecided nb
  uint32_t* conb = blkb + kBigW;                                       // contested
  int* wpre = reinterpret_cast<int*>(bsm + BigSmem::WPRE);
  uint2* ent = reinterpret_cast<uint2*>(bsm + BigSmem::REG);
  uint32_t* sadj = reinterpret_cast<uint32_t*>(bsm + BigSmem::REG);
  uint32_t* skey = reinterpret_cast<uint32_t*>(bsm + BigSmem::SKEY);
  uint32_t* scm = reinterpret_cast<uint32_t*>(bsm + BigSmem::SCM);
  int32_t* spt = reinterpret_cast<int32_t*>(bsm + BigSmem::SPT);
  int* shist = reinterpret_cast<int*>(bsm + BigSmem::SHIST);
  uint32_t* misc = reinterpret_cast<uint32_t*>(bsm + BigSmem::MISC);
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  pdl_wait();
  pdl_trigger();   // a single CTA
  const int n_unc = *n_unc_dev;
  const int nc = min(T, n_unc);
  const uint32_t cnt = *nz.count;
  if (tid == 0) {
    if (ticket) *ticket = 0;
    if (band_count) *band_count = 0ull;
    *nz.count = 0u;   // the next tile's A2 starts a fresh list (stream order)
  }
  if (nc == 0) {
    if (tid == 0) *dL_dev = 0;
    return;
  }
  const int W = (nc + 31) >> 5;
  bool dense = force_dense || cnt > kBigNz || cnt > nz.cap;
  // ---- sparse path
  if (!dense) {
    for (uint32_t k = tid; k < cnt; k += blockDim.x) ent[k] = __ldcg(nz.e + k);
    for (int i = tid; i < W; i += blockDim.x) conb[i] = 0u;
    __syncthreads();
    for (uint32_t k = tid; k < cnt; k += blockDim.x) {
      const uint32_t a = ent[k].x >> 16;
      atomicOr(&conb[a >> 5], 1u << (a & 31));
    }
    __syncthreads();
    for (int i = tid; i < W; i += blockDim.x) {
      const uint32_t valid = (32 * i + 32 <= nc) ? 0xffffffffu : ((1u << (nc - 32 * i)) - 1u);
      lmb[i] = valid & ~conb[i];
      decb[i] = ~conb[i];          // contested candidates start undecided
    }
    __syncthreads();
    int rounds = 0;
    while (true) {
      for (int i = tid; i < W; i += blockDim.x) {
        killb[i] = 0u;
        blkb[i] = 0u;
      }
      __syncthreads();
      for (uint32_t k = tid; k < cnt; k += blockDim.x) {
        const uint2 e = ent[k];
        const uint32_t a = e.x >> 16, v = e.x & 0xffffu;
        if ((decb[a >> 5] >> (a & 31)) & 1u) continue;
        if (e.y & lmb[v]) atomicOr(&killb[a >> 5], 1u << (a & 31));
        if (e.y & ~decb[v]) atomicOr(&blkb[a >> 5], 1u << (a & 31));
      }
      __syncthreads();
      int still = 0;
      for (int i = tid; i < W; i += blockDim.x) {
        const uint32_t und = ~decb[i];
        const uint32_t nn = und & killb[i];
        const uint32_t nl = und & ~killb[i] & ~blkb[i];
        lmb[i] |= nl;
        decb[i] |= nn | nl;
        still |= (und & ~(nn | nl)) != 0u;
      }
      ++rounds;
      if (!__syncthreads_or(still)) break;
      if (rounds >= kBigRounds) {
        dense = true;   // a long in-tile dependency chain: the dense in-order path
        break;
      }
    }
  }
  // ---- dense path: sub-tiles of 1024 in order
  if (dense) {
    for (int i = tid; i < W; i += blockDim.x) lmb[i] = 0u;
    __syncthreads();
    for (int base = 0; base < nc; base += 1024) {
      const int ncs = min(1024, nc - base);
      const int a = base + tid;
      uint32_t pre = 0u;
      if (tid < ncs) {
        const int wb = base >> 5;
        for (int v = 0; v < wb && !pre; ++v)
          pre |= __ldcg(adj + (int64_t)v * T + a) & lmb[v];
      }
      const unsigned bal = __ballot_sync(FULLMASK, pre != 0u);
      if (lane == 0) misc[wp] = bal;   // preb: 32 words, one per warp of the sub-tile
      __syncthreads();
      resolve_core(adj + (int64_t)(base >> 5) * T + base, T, ncs, lmb + (base >> 5), sadj, 1024,
                   misc);
      __syncthreads();
    }
  }
  // ---- output: landmarks in order
  if (tid < 32) {   // exclusive scan of the per-word counts (8 words per lane)
    int v[8], t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int wd = tid * 8 + i;
      v[i] = wd < W ? __popc(lmb[wd]) : 0;
      t += v[i];
    }
    int incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += u;
    }
    int run = incl - t;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wpre[tid * 8 + i] = run;
      run += v[i];
    }
    if (tid == 31) wpre[kBigW] = run;
  }
  const bool prune = pt_out.cell != nullptr;
  if (prune) {
    for (int i = tid; i < 256; i += blockDim.x) shist[i] = 0;
    for (int i = tid; i < ((nc + 255) >> 8) * 64; i += blockDim.x) scm[i] = 0u;
  }
  __syncthreads();
  const int L0 = *L_dev;
  const int dL = wpre[kBigW];
  // each thread's (up to kBigT / 1024) candidates: point and cell rank loaded
  // once, all loads of a level in flight together (three memory latencies
  // per tile instead of three per candidate)
  constexpr int PER = kBigT / 1024;
  int32_t cpt[PER];
  int crk[PER], ccl[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int a = tid + 1024 * k;
    cpt[k] = a < nc && ((lmb[a >> 5] >> (a & 31)) & 1u) ? __ldcg(unc + a) : -1;
  }
  if (prune) {
#pragma unroll
    for (int k = 0; k < PER; ++k) ccl[k] = cpt[k] >= 0 ? __ldg(pt_out.cell + cpt[k]) : 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) crk[k] = cpt[k] >= 0 ? __ldg(pt_out.rank + ccl[k]) : -1;
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int a = tid + 1024 * k;
    if (cpt[k] >= 0) {
      const uint32_t S = lmb[a >> 5];
      const int pos = wpre[a >> 5] + __popc(S & ((1u << (a & 31)) - 1u));
      new_lm[pos] = cpt[k];
      lm_out[L0 + pos] = cpt[k];
      if (prune) atomicAdd(&shist[crk[k]], 1);
    }
  }
  __syncthreads();
  if (prune) {
    // landmarks grouped by cell rank (counting sort; positions kept in keys)
    if (tid < 32) {
      int v[8], t = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = shist[tid * 8 + i];
        t += v[i];
      }
      int incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(FULLMASK, incl, o);
        if (lane >= o) incl += u;
      }
      int run = incl - t;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        shist[tid * 8 + i] = run;
        run += v[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int a = tid + 1024 * k;
      if (cpt[k] >= 0) {
        const uint32_t S = lmb[a >> 5];
        const int pos = wpre[a >> 5] + __popc(S & ((1u << (a & 31)) - 1u));
        const int slot = atomicAdd(&shist[crk[k]], 1);
        skey[slot] = (uint32_t)pos | ((uint32_t)ccl[k] << 16);   // pos < 2^13, cell < 256
        spt[slot] = cpt[k];
      }
    }
    __syncthreads();
    for (int k = tid; k < dL; k += blockDim.x) {
      const uint32_t v = skey[k];
      const int c = (int)(v >> 16);
      pt_out.col_pt[k] = spt[k];
      pt_out.col_pos[k] = (int32_t)(v & 0xffffu);
      atomicOr(&scm[(k >> 5) * 8 + (c >> 5)], 1u << (c & 31));
    }
    __syncthreads();
    const int nch = (dL + 31) >> 5, ntl = (dL + 255) >> 8;
    for (int i = tid; i < ntl * 64; i += blockDim.x) pt_out.cmask[i] = scm[i];   // whole tiles
    for (int i = tid; i < ntl * 8; i += blockDim.x) {
      const int t = i >> 3, wd = i & 7;
      uint32_t v = 0u;
      for (int c = 0; c < 8; ++c)
        if (t * 8 + c < nch) v |= scm[(t * 8 + c) * 8 + wd];
      pt_out.tmask[i] = v;
    }
  }
  if (tid == 0) {
    *dL_dev = dL;
    *L_dev = L0 + dL;
    stats->greedy_evals += (unsigned long long)nc * (unsigned long long)(nc - 1) / 2ull;
    stats->tiles += 1ull;
  }
}

cudaError_t launch_resolve_big(const uint32_t* adj, AdjList nz, const int32_t* unc,
                               const int32_t* n_unc, int T, int32_t* lm_out, int32_t* L_dev,
                               int32_t* new_lm, int32_t* dL_dev, DevStats* stats,
                               int32_t* ticket, unsigned long long* band_count, cudaStream_t s,
                               int64_t* launches, PruneTile pt_out, int force_dense) {
  ++*launches;
  if (T > kBigT || (T % 32) != 0) return cudaErrorInvalidValue;
  static bool attr_set[kMaxDevices] = {};
  bool& attr = attr_set[cur_device()];
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_resolve_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         BigSmem::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_resolve_big, dim3(1), dim3(1024), (size_t)BigSmem::TOTAL, s, adj, nz, unc,
                    n_unc, T, lm_out, L_dev, new_lm, dL_dev, stats, ticket, band_count, pt_out,
                    force_dense);
}

cudaError_t launch_resolve(const uint32_t* adj, int adj_words, const int32_t* unc,
                           const int32_t* n_unc, int T, int32_t* lm_out, int32_t* L_dev,
                           int32_t* new_lm, int32_t* dL_dev, DevStats* stats, int32_t* ticket,
                           unsigned long long* band_count, cudaStream_t s, int64_t* launches,
                           PruneTile pt_out) {
  ++*launches;
  const size_t smem = sizeof(uint32_t) * 32 * (size_t)adj_words * adj_words;
  static bool attr_set[kMaxDevices] = {};   // per device (attributes are per context)
  bool& attr = attr_set[cur_device()];
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(uint32_t) * 32 * 32 * 32));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_resolve_debug, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(uint32_t) * 32 * 32 * 32));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_resolve, dim3(1), dim3(1024), smem, s, adj, adj_words, unc, n_unc, T,
                    lm_out, L_dev, new_lm, dL_dev, stats, ticket, band_count, pt_out);
}

cudaError_t launch_resolve_debug(const uint32_t* adj, int adj_words, int nc, uint8_t* lm,
                                 cudaStream_t s, int64_t* launches) {
  ++*launches;
  const size_t smem = sizeof(uint32_t) * 32 * (size_t)adj_words * adj_words;
  cudaError_t e = cudaFuncSetAttribute(k_resolve_debug, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(uint32_t) * 32 * 32 * 32));
  if (e != cudaSuccess) return e;
  k_resolve_debug<<<1, 1024, smem, s>>>(adj, adj_words, nc, lm);
  return cudaGetLastError();
}

// A4 compaction: unc_next = [unc[i] for nc <= i < n_unc if !covered[unc[i]]],
// in order.  Each CTA takes the next CP_TILE items by ticket (so a CTA only
// ever waits on CTAs that already started), ranks its survivors with ballots,
// publishes its count, and derives its output offset by looking back over the
// predecessors' published (aggregate | inclusive prefix) words.  Words carry the
// launch tag, so the state array never needs clearing between tiles.
constexpr int CP_NT = 256, CP_ROUNDS = 8, CP_TILE = CP_NT * CP_ROUNDS;

__global__ void __launch_bounds__(CP_NT) k_compact(const uint8_t* __restrict__ covered,
                                                   const int32_t* __restrict__ unc,
                                                   const int32_t* __restrict__ n_unc_dev, int T,
                                                   int32_t* __restrict__ unc_next,
                                                   int32_t* __restrict__ n_unc_next,
                                                   unsigned long long* state,
                                                   int32_t* ticket, uint32_t tag,
                                                   int one_wave) {
  __shared__ int s_bid;
  __shared__ int s_wcnt[CP_ROUNDS][CP_NT / 32];
  __shared__ int s_excl;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pdl_wait();
  // a grid that fits in one wave lets the next kernel launch early; a
  // multi-wave grid must not (waiting dependents could hold the SMs its
  // remaining CTAs need)
  if (one_wave) pdl_trigger();
  if (tid == 0) s_bid = atomicAdd(ticket, 1);
  __syncthreads();
  const int bid = s_bid;
  const int n_unc = *n_unc_dev;
  const int nc = min(T, n_unc);
  const int64_t m = (int64_t)n_unc - nc;
  const int64_t i0 = (int64_t)bid * CP_TILE;
  if (i0 >= m) {
    if (bid == 0 && tid == 0) *n_unc_next = 0;   // nothing left after this tile
    return;
  }
  // survivors of this CTA's items, round r covers [i0 + r*NT, i0 + (r+1)*NT)
  int32_t pt[CP_ROUNDS];
  unsigned keepm = 0u;
#pragma unroll
  for (int r = 0; r < CP_ROUNDS; ++r) {
    const int64_t i = i0 + r * CP_NT + tid;
    pt[r] = i < m ? unc[nc + i] : 0;
    const bool keep = i < m && covered[pt[r]] == 0;
    keepm |= (keep ? 1u : 0u) << r;
    const unsigned b = __ballot_sync(FULLMASK, keep);
    if (lane == 0) s_wcnt[r][w] = __popc(b);
  }
  __syncthreads();
  if (tid < 32) {
    // CTA aggregate, then the warp-wide look-back
    int agg = 0;
    for (int k = lane; k < CP_ROUNDS * (CP_NT / 32); k += 32) agg += (&s_wcnt[0][0])[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(FULLMASK, agg, o);
    const int excl = (int)warp_lookback(state, bid, tag, (uint32_t)agg);
    if (lane == 0) {
      s_excl = excl;
      if (i0 + CP_TILE >= m) *n_unc_next = excl + agg;   // the last CTA holds the total
    }
  }
  __syncthreads();
  // scatter in item order: offset = excl + all earlier rounds + earlier warps + lane rank
  int base = s_excl;
#pragma unroll
  for (int r = 0; r < CP_ROUNDS; ++r) {
    const bool keep = (keepm >> r) & 1u;
    const unsigned b = __ballot_sync(FULLMASK, keep);
    int pre = 0;
    for (int k = 0; k < w; ++k) pre += s_wcnt[r][k];
    if (keep) unc_next[base + pre + __popc(b & ((1u << lane) - 1u))] = pt[r];
    int tot = 0;
#pragma unroll
    for (int k = 0; k < CP_NT / 32; ++k) tot += s_wcnt[r][k];
    base += tot;
  }
}

int64_t compact_state_words(int64_t n) { return (n + CP_TILE - 1) / CP_TILE + 1; }

cudaError_t launch_compact_unc(const uint8_t* covered, const int32_t* unc, const int32_t* n_unc,
                               int T, int32_t* unc_next, int32_t* n_unc_next,
                               unsigned long long* state, int32_t* ticket, uint32_t tag,
                               int64_t n, cudaStream_t s, int64_t* launches) {
  const int64_t nblk = (n + CP_TILE - 1) / CP_TILE;
  ++*launches;
  static int cap_of[kMaxDevices] = {};   // CTAs resident at once, per device
  int& cap = cap_of[cur_device()];
  if (cap == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_compact, CP_NT, 0);
    cap = sms * (per > 0 ? per : 1);
  }
  const int one_wave = nblk <= cap ? 1 : 0;
  return launch_pdl(k_compact, dim3((unsigned)(nblk > 0 ? nblk : 1)), dim3(CP_NT), 0, s, covered,
                    unc, n_unc, T, unc_next, n_unc_next, state, ticket, tag, one_wave);
}

}  // namespace bm
