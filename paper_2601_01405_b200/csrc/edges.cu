// edges.cu — steps D1-D3 (the nerve's 1-skeleton, Def 2.2 / PAPER.md:84-92):
// landmarks i < j are joined iff some data point lies in both balls, i.e. iff
// (i, j) is a pair of some point's ascending landmark row pt_lm[p] (the
// "∩ X ≠ ∅" witness).
//
// Two device paths, both producing edges[E][2] in lexicographic order:
//   bitmap (L <= BM_EDGE_BITMAP_MAX_L): every witnessed pair sets bit (i, j)
//     of an L x L bit matrix (atomicOr), and one look-back compaction walks
//     the words in row-major order writing (i, j) for every set bit — no sort;
//   keys (large L): pair keys i << lbits | j are radix sorted (sort.cu) and
//     one look-back compaction keeps the first of each run of equal keys.
#include "internal.cuh"

namespace bm {

constexpr unsigned FME = 0xffffffffu;
constexpr unsigned long long LB_AGG = 1ull, LB_INC = 2ull;

__device__ __forceinline__ unsigned long long lb_pack(uint32_t tag, unsigned long long flag,
                                                      uint32_t v) {
  return ((unsigned long long)tag << 34) | (flag << 32) | (unsigned long long)v;
}

// ---------------------------------------------------------------- bitmap path
// One thread per point: set bit (i, j) for every pair a < c of its row
// (rows are short: t_p ~ 2-40 on the BASELINE configs); the warp adds its C(t,2).
__global__ void k_edge_bits(const int64_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_lm,
                            int64_t n, int W, uint32_t* __restrict__ bits,
                            unsigned long long* __restrict__ npairs) {
  pdl_wait();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long mine = 0ull;
  if (p < n) {
    const int64_t b = pt_ptr[p], t = pt_ptr[p + 1] - b;
    if (t >= 2) {
      mine = (unsigned long long)(t * (t - 1) / 2);
      for (int64_t a = 0; a + 1 < t; ++a) {
        uint32_t* row = bits + (int64_t)pt_lm[b + a] * W;
        for (int64_t c = a + 1; c < t; ++c) {
          const int32_t j = pt_lm[b + c];
          atomicOr(row + (j >> 5), 1u << (j & 31));
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FME, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(npairs, mine);
}

// Row-major walk of the bit matrix: CTA tile = 256 threads x 4 consecutive
// words each; edges written in (i, j) order.
constexpr int EB_NT = 256, EB_WPT = 16, EB_TILE = EB_NT * EB_WPT;

__global__ void __launch_bounds__(EB_NT) k_bits_compact(const uint32_t* __restrict__ bits,
                                                       int64_t nwords, int W,
                                                       int32_t* __restrict__ edges,
                                                       int64_t cap, int64_t* __restrict__ total,
                                                       unsigned long long* state,
                                                       int32_t* ticket, uint32_t tag) {
  __shared__ int s_tile;
  __shared__ uint32_t s_warp[EB_NT / 32];
  __shared__ uint32_t s_excl;
  pdl_wait();
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t w0 = tile * EB_TILE + (int64_t)threadIdx.x * EB_WPT;
  uint32_t wv[EB_WPT];
  uint32_t cnt = 0;
  if (w0 + EB_WPT <= nwords) {   // 16-byte loads (w0 is a multiple of 16 words)
#pragma unroll
    for (int k = 0; k < EB_WPT; k += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(bits + w0 + k);
      wv[k] = q.x;
      wv[k + 1] = q.y;
      wv[k + 2] = q.z;
      wv[k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < EB_WPT; ++k) wv[k] = w0 + k < nwords ? bits[w0 + k] : 0u;
  }
#pragma unroll
  for (int k = 0; k < EB_WPT; ++k) cnt += __popc(wv[k]);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FME, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t agg = 0;
    for (int k = 0; k < EB_NT / 32; ++k) agg += s_warp[k];
    const uint32_t ex = warp_lookback(state, tile, tag, agg);
    if (threadIdx.x == 0) {
      s_excl = ex;
      if ((tile + 1) * EB_TILE >= nwords) *total = (int64_t)ex + agg;
    }
  }
  __syncthreads();
  int64_t pos = s_excl + incl - cnt;
  for (int k = 0; k < w; ++k) pos += s_warp[k];
#pragma unroll
  for (int k = 0; k < EB_WPT; ++k) {
    uint32_t v = wv[k];
    const int64_t word = w0 + k;
    const int32_t i = (int32_t)(word / W);
    const int32_t jb = (int32_t)(word % W) * 32;
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1u;
      if (pos < cap) {
        edges[2 * pos] = i;
        edges[2 * pos + 1] = jb + b;
      }
      ++pos;
    }
  }
}

// ---------------------------------------------------------------- keys path
// Sorted keys i << lbits | j: keep the first of every run, in order.
constexpr int UQ_NT = 256, UQ_IPT = 8, UQ_TILE = UQ_NT * UQ_IPT;

__global__ void __launch_bounds__(UQ_NT) k_unique_compact(const unsigned long long* __restrict__ keys,
                                                         int64_t m, int lbits,
                                                         int32_t* __restrict__ edges,
                                                         int64_t* __restrict__ total,
                                                         unsigned long long* state,
                                                         int32_t* ticket, uint32_t tag) {
  __shared__ int s_tile;
  __shared__ uint32_t s_warp[UQ_NT / 32];
  __shared__ uint32_t s_excl;
  pdl_wait();
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t i0 = tile * UQ_TILE + (int64_t)threadIdx.x * UQ_IPT;
  unsigned long long kv[UQ_IPT];
  uint32_t keep = 0u, cnt = 0u;
  const bool whole = i0 + UQ_IPT <= m;   // the thread's 64 bytes in four 16-byte loads
  if (whole) {
    const ulonglong2* kp = reinterpret_cast<const ulonglong2*>(keys + i0);
#pragma unroll
    for (int k = 0; k < UQ_IPT / 2; ++k) {
      const ulonglong2 v = kp[k];
      kv[2 * k] = v.x;
      kv[2 * k + 1] = v.y;
    }
  }
  const unsigned long long kprev = i0 > 0 && i0 < m ? keys[i0 - 1] : 0ull;
#pragma unroll
  for (int k = 0; k < UQ_IPT; ++k) {
    const int64_t i = i0 + k;
    if (!whole) kv[k] = i < m ? keys[i] : 0ull;
    const bool f = i < m && (i == 0 || kv[k] != (k > 0 ? kv[k - 1] : kprev));
    keep |= (f ? 1u : 0u) << k;
    cnt += f ? 1u : 0u;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FME, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t agg = 0;
    for (int k = 0; k < UQ_NT / 32; ++k) agg += s_warp[k];
    const uint32_t ex = warp_lookback(state, tile, tag, agg);
    if (threadIdx.x == 0) {
      s_excl = ex;
      if ((tile + 1) * UQ_TILE >= m) *total = (int64_t)ex + agg;
    }
  }
  __syncthreads();
  int64_t pos = s_excl + incl - cnt;
  for (int k = 0; k < w; ++k) pos += s_warp[k];
  const unsigned long long lm = (1ull << lbits) - 1ull;
#pragma unroll
  for (int k = 0; k < UQ_IPT; ++k) {
    if ((keep >> k) & 1u) {
      edges[2 * pos] = (int32_t)(kv[k] >> lbits);
      edges[2 * pos + 1] = (int32_t)(kv[k] & lm);
      ++pos;
    }
  }
}

// ---------------------------------------------------------------- row-union emission
// D1 for large L (the default above 4096 landmarks): the pairs (i, j), j > i,
// are emitted landmark row by landmark row — row i's pairs are the entries
// j > i of pt_lm[p] over the members p of ball i (each pair of a point's row
// is met exactly once, at its smaller landmark) — and deduplicated in a
// per-warp shared-memory hash set before they reach HBM.  A point's C(t_p, 2)
// pairs repeat across the points two balls share (C3 eps=8: P = 1.4e8 pairs
// for E = 1.8e7 edges), so the radix sort (D2) and the unique pass (D3) then
// run on a few keys per edge instead of every witnessed pair.  A row is cut
// into items of RP_CH members (a ball of 5e6 points is spread over ~1e4
// warps); pairs an item repeats from another item of the same row are removed
// by D3, like every other duplicate.
constexpr int RP_CH = 512;                 // members per item
#ifndef BM_RP_H
#define BM_RP_H 1024
#endif
constexpr int RP_H = BM_RP_H;              // hash slots per warp
constexpr int kRpBits = RP_H == 2048 ? 11 : 10;
static_assert(RP_H == (1 << kRpBits), "RP_H: 1024 or 2048 slots");
constexpr int RP_U = 4;                    // row entries per lane per step (128 per warp)
constexpr uint32_t RP_EMPTY = 0xffffffffu;
constexpr int RP_NT = 128, RP_NW = RP_NT / 32;

__global__ void k_row_items(const int64_t* __restrict__ ball_ptr, int64_t L,
                            int64_t* __restrict__ cnt) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < L) cnt[i] = (ball_ptr[i + 1] - ball_ptr[i] + RP_CH - 1) / RP_CH;
}

// item -> landmark row (item_row[item_off[i] + k] = i)
__global__ void k_item_rows(const int64_t* __restrict__ item_off, const int64_t* __restrict__ cnt,
                            int64_t L, int32_t* __restrict__ item_row) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int64_t o = item_off[i], c = cnt[i];
  for (int64_t k = 0; k < c; ++k) item_row[o + k] = (int32_t)i;
}

// the warp writes the keys (i << lbits | j) of its set (slots listed in the
// insertion log) and empties those slots
__device__ __forceinline__ void rp_flush(uint32_t* tab, const uint16_t* log, int fill, int64_t i,
                                         int lbits, unsigned long long* __restrict__ keys,
                                         int64_t cap, unsigned long long* kcount, int lane) {
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(kcount, (unsigned long long)fill);
  base = __shfl_sync(FME, base, 0);
  const unsigned long long hi = (unsigned long long)i << lbits;
  for (int k = lane; k < fill; k += 32) {
    const uint32_t h = log[k];
    const uint32_t v = tab[h];
    if ((int64_t)(base + k) < cap) keys[base + k] = hi | v;
    tab[h] = RP_EMPTY;
  }
  __syncwarp();
}

// One warp per item.  The item's members are taken 32 at a time; their rows
// (pt_lm[p], t_p entries each) are walked as one flattened run of entries,
// 128 per step over all 32 lanes (lane-parallel whatever the row lengths, and
// consecutive entries of a row are consecutive loads).  Entries j > i go into
// the warp's open-addressing set; every new key's slot is appended to an
// insertion log, so a flush visits only the occupied slots.  The set is
// flushed before a step could fill it (the probe always finds a free slot).
__global__ void __launch_bounds__(RP_NT) k_row_pairs(
    const int64_t* __restrict__ ball_ptr, const int32_t* __restrict__ ball_idx,
    const int64_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_lm, int64_t n, int64_t L,
    const int64_t* __restrict__ item_off, const int32_t* __restrict__ item_row, int64_t n_items,
    int lbits, unsigned long long* __restrict__ keys, int64_t cap, unsigned long long* kcount,
    unsigned long long* npairs) {
  __shared__ uint32_t s_tab[RP_NW][RP_H];
  __shared__ uint16_t s_log[RP_NW][RP_H];
  pdl_wait();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* tab = s_tab[w];
  uint16_t* log = s_log[w];
  for (int k = lane; k < RP_H; k += 32) tab[k] = RP_EMPTY;
  __syncwarp();
  unsigned long long mine = 0ull;
  const int64_t nwarps = (int64_t)gridDim.x * RP_NW;
  for (int64_t it = (int64_t)blockIdx.x * RP_NW + w; it < n_items; it += nwarps) {
    const int64_t i = item_row[it];
    const int64_t m0 = ball_ptr[i] + (it - item_off[i]) * RP_CH;
    const int64_t m1 = min(ball_ptr[i + 1], m0 + RP_CH);
    int fill = 0;   // keys in the set (warp-uniform)
    for (int64_t mb = m0; mb < m1; mb += 32) {
      const int64_t m = mb + lane;
      int64_t b = 0;
      int t = 0;
      if (m < m1) {
        const int64_t p = ball_idx[m];
        b = pt_ptr[p];
        t = (int)(pt_ptr[p + 1] - b);
      }
      // exclusive prefix of the row lengths over the lanes, and the total
      int pre = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FME, pre, o);
        if (lane >= o) pre += v;
      }
      const int T = __shfl_sync(FME, pre, 31);
      pre -= t;
      for (int g0 = 0; g0 < T; g0 += 32 * RP_U) {
        if (fill > RP_H - 32 * RP_U - 1) {
          rp_flush(tab, log, fill, i, lbits, keys, cap, kcount, lane);
          fill = 0;
        }
        uint32_t jv[RP_U];
#pragma unroll
        for (int u = 0; u < RP_U; ++u) {
          const int g = g0 + u * 32 + lane;
          // member k of entry g: the last lane with pre_k <= g
          int k = 0;
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) {
            const int pk = __shfl_sync(FME, pre, (k + st) & 31);
            if (k + st < 32 && pk <= g) k += st;
          }
          const int64_t bk = __shfl_sync(FME, b, k);
          const int pk = __shfl_sync(FME, pre, k);
          jv[u] = g < T ? (uint32_t)pt_lm[bk + (g - pk)] : 0xffffffffu;
        }
        int cnt = 0;
        uint32_t slot[RP_U];
#pragma unroll
        for (int u = 0; u < RP_U; ++u) {
          slot[u] = 0xffffffffu;
          const uint32_t j = jv[u];
          if (j == 0xffffffffu || (int64_t)j <= i) continue;
          ++mine;
          uint32_t h = (j * 2654435761u) >> (32 - kRpBits);
          uint32_t old;
          while ((old = atomicCAS(&tab[h], RP_EMPTY, j)) != RP_EMPTY && old != j)
            h = (h + 1) & (RP_H - 1);
          if (old == RP_EMPTY) {
            slot[u] = h;
            ++cnt;
          }
        }
        // log positions: exclusive prefix of the per-lane counts (0..RP_U)
        const unsigned b0 = __ballot_sync(FME, cnt & 1), b1 = __ballot_sync(FME, cnt & 2),
                       b2 = __ballot_sync(FME, cnt & 4);
        int pos = fill + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
#pragma unroll
        for (int u = 0; u < RP_U; ++u)
          if (slot[u] != 0xffffffffu) log[pos++] = (uint16_t)slot[u];
        fill += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
      }
    }
    if (fill > 0) rp_flush(tab, log, fill, i, lbits, keys, cap, kcount, lane);
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FME, mine, o);
  if (lane == 0 && mine) atomicAdd(npairs, mine);
}

size_t row_items_temp_bytes(int64_t L) { return sizeof(int64_t) * (size_t)(2 * L + 2); }

cudaError_t launch_row_items(const int64_t* ball_ptr, int64_t L, int64_t* cnt, cudaStream_t s,
                             int64_t* launches) {
  ++*launches;
  const int64_t g = (L + 255) / 256;
  return launch_pdl(k_row_items, dim3((unsigned)(g > 0 ? g : 1)), dim3(256), 0, s, ball_ptr, L,
                    cnt);
}

cudaError_t launch_item_rows(const int64_t* item_off, const int64_t* cnt, int64_t L,
                             int32_t* item_row, cudaStream_t s, int64_t* launches) {
  ++*launches;
  const int64_t g = (L + 255) / 256;
  return launch_pdl(k_item_rows, dim3((unsigned)(g > 0 ? g : 1)), dim3(256), 0, s, item_off, cnt,
                    L, item_row);
}

cudaError_t launch_row_pairs(const int64_t* ball_ptr, const int32_t* ball_idx,
                             const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                             const int64_t* item_off, const int32_t* item_row, int64_t n_items,
                             int lbits, unsigned long long* keys, int64_t cap,
                             unsigned long long* kcount, unsigned long long* npairs,
                             cudaStream_t s, int64_t* launches) {
  ++*launches;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (n_items + RP_NW - 1) / RP_NW;
  const int64_t per_sm = (int64_t)(200 * 1024) / (RP_NW * RP_H * 6);   // sets + logs per SM
  if (g > (int64_t)sms * per_sm) g = (int64_t)sms * per_sm;
  return launch_pdl(k_row_pairs, dim3((unsigned)(g > 0 ? g : 1)), dim3(RP_NT), 0, s, ball_ptr,
                    ball_idx, pt_ptr, pt_lm, n, L, item_off, item_row, n_items, lbits, keys, cap,
                    kcount, npairs);
}

// ---------------------------------------------------------------- bitmap CSR
// Step C for moderate n * L: the membership keys (point << 32 | position) set
// bit (p, j) of a point-major [n][Wp] and bit (j, p) of a landmark-major [L][Wl]
// bit matrix; one look-back pass per matrix then writes the column index of
// every set bit in row-major order — i.e. a CSR already sorted both ways.
__global__ void k_keys_to_bits(const unsigned long long* __restrict__ keys, int64_t m, int Wp,
                               int Wl, uint32_t* __restrict__ pbits, uint32_t* __restrict__ lbits) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const int64_t p = (int64_t)(k >> 32), j = (int64_t)(k & 0xffffffffull);
    atomicOr(pbits + p * Wp + (j >> 5), 1u << (j & 31));
    atomicOr(lbits + j * Wl + (p >> 5), 1u << (p & 31));
  }
}

__global__ void __launch_bounds__(EB_NT) k_bits_csr(const uint32_t* __restrict__ bits, int64_t rows,
                                                   int W, int64_t* __restrict__ ptr,
                                                   int32_t* __restrict__ idx,
                                                   unsigned long long* state, int32_t* ticket,
                                                   uint32_t tag) {
  __shared__ int s_tile;
  __shared__ uint32_t s_warp[EB_NT / 32];
  __shared__ uint32_t s_excl;
  pdl_wait();
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t nwords = rows * (int64_t)W;
  const int64_t tile = s_tile;
  const int64_t w0 = tile * EB_TILE + (int64_t)threadIdx.x * EB_WPT;
  uint32_t wv[EB_WPT];
  uint32_t cnt = 0;
  if (w0 + EB_WPT <= nwords) {   // 16-byte loads (w0 is a multiple of 16 words)
#pragma unroll
    for (int k = 0; k < EB_WPT; k += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(bits + w0 + k);
      wv[k] = q.x;
      wv[k + 1] = q.y;
      wv[k + 2] = q.z;
      wv[k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < EB_WPT; ++k) wv[k] = w0 + k < nwords ? bits[w0 + k] : 0u;
  }
#pragma unroll
  for (int k = 0; k < EB_WPT; ++k) cnt += __popc(wv[k]);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FME, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t agg = 0;
    for (int k = 0; k < EB_NT / 32; ++k) agg += s_warp[k];
    const uint32_t ex = warp_lookback(state, tile, tag, agg);
    if (threadIdx.x == 0) {
      s_excl = ex;
      if ((tile + 1) * EB_TILE >= nwords) ptr[rows] = (int64_t)ex + agg;
    }
  }
  __syncthreads();
  int64_t pos = s_excl + incl - cnt;
  for (int k = 0; k < w; ++k) pos += s_warp[k];
#pragma unroll
  for (int k = 0; k < EB_WPT; ++k) {
    const int64_t word = w0 + k;
    if (word >= nwords) break;
    const int64_t row = word / W;
    const int64_t cb = (word - row * W) * 32;
    if (cb == 0) ptr[row] = pos;   // first word of a row: its CSR start
    uint32_t v = wv[k];
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1u;
      idx[pos++] = (int32_t)(cb + b);
    }
  }
}

// ---------------------------------------------------------------- host side
// the landmark-major matrix starts 16-byte aligned (the compaction loads 4 words at a time)
static int64_t csr_pm_words(int64_t n, int64_t L) { return (n * ((L + 31) / 32) + 3) & ~int64_t(3); }
int64_t csr_bitmap_words(int64_t n, int64_t L) {
  return csr_pm_words(n, L) + L * ((n + 31) / 32);
}

cudaError_t csr_from_keys_bitmap(const unsigned long long* keys, int64_t m, int64_t n, int64_t L,
                                 uint32_t* bits, void* temp, int64_t* pt_ptr, int32_t* pt_lm,
                                 int64_t* ball_ptr, int32_t* ball_idx, cudaStream_t s,
                                 int64_t* launches) {
  const int Wp = (int)((L + 31) / 32), Wl = (int)((n + 31) / 32);
  uint32_t* pb = bits;
  uint32_t* lb = bits + csr_pm_words(n, L);
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(uint32_t) * csr_bitmap_words(n, L), s);
  if (e != cudaSuccess) return e;
  int64_t g = (m + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  e = launch_pdl(k_keys_to_bits, dim3((unsigned)g), dim3(256), 0, s, keys, m, Wp, Wl, pb, lb);
  if (e != cudaSuccess) return e;
  // two look-back passes; state: [ticket x2 | pad][tiles_p + 1][tiles_l + 1]
  const int64_t tp = (n * (int64_t)Wp + EB_TILE - 1) / EB_TILE;
  const int64_t tl = (L * (int64_t)Wl + EB_TILE - 1) / EB_TILE;
  int32_t* tickets = (int32_t*)temp;
  unsigned long long* sp = (unsigned long long*)((char*)temp + 64);
  unsigned long long* sl = sp + tp + 1;
  e = cudaMemsetAsync(temp, 0, 64 + sizeof(unsigned long long) * (tp + tl + 2), s);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_bits_csr, dim3((unsigned)(tp > 0 ? tp : 1)), dim3(EB_NT), 0, s,
                 (const uint32_t*)pb, n, Wp, pt_ptr, pt_lm, sp, tickets, 1u);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_bits_csr, dim3((unsigned)(tl > 0 ? tl : 1)), dim3(EB_NT), 0, s,
                 (const uint32_t*)lb, L, Wl, ball_ptr, ball_idx, sl, tickets + 1, 1u);
  *launches += 3;
  return e;
}

size_t csr_bitmap_temp_bytes(int64_t n, int64_t L) {
  const int64_t Wp = (L + 31) / 32, Wl = (n + 31) / 32;
  const int64_t tp = (n * Wp + EB_TILE - 1) / EB_TILE, tl = (L * Wl + EB_TILE - 1) / EB_TILE;
  return 64 + sizeof(unsigned long long) * (size_t)(tp + tl + 2);
}

int64_t edge_bitmap_words(int64_t L) { return L * ((L + 31) / 32); }

size_t edge_lb_temp_bytes(int64_t items) {
  const int64_t t = (items + 1023) / 1024 + 2;
  return (size_t)t * 8 + 64;
}

cudaError_t launch_edge_bits(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                             uint32_t* bits, unsigned long long* npairs, cudaStream_t s,
                             int64_t* launches) {
  const int W = (int)((L + 31) / 32);
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(uint32_t) * edge_bitmap_words(L), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(npairs, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  int64_t g = (n + 255) / 256;
  return launch_pdl(k_edge_bits, dim3((unsigned)(g > 0 ? g : 1)), dim3(256), 0, s, pt_ptr, pt_lm,
                    n, W, bits, npairs);
}

cudaError_t launch_bits_compact(const uint32_t* bits, int64_t L, int32_t* edges, int64_t cap,
                                int64_t* total, void* temp, cudaStream_t s, int64_t* launches) {
  const int W = (int)((L + 31) / 32);
  const int64_t nwords = edge_bitmap_words(L);
  const int64_t t = (nwords + EB_TILE - 1) / EB_TILE;
  int32_t* ticket = (int32_t*)temp;
  unsigned long long* state = (unsigned long long*)((char*)temp + 64);
  cudaError_t e = cudaMemsetAsync(temp, 0, 64 + sizeof(unsigned long long) * (t + 1), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  return launch_pdl(k_bits_compact, dim3((unsigned)(t > 0 ? t : 1)), dim3(EB_NT), 0, s, bits,
                    nwords, W, edges, cap, total, state, ticket, 1u);
}

cudaError_t launch_unique_compact(const unsigned long long* keys, int64_t m, int lbits,
                                  int32_t* edges, int64_t* total, void* temp, cudaStream_t s,
                                  int64_t* launches) {
  const int64_t t = (m + UQ_TILE - 1) / UQ_TILE;
  int32_t* ticket = (int32_t*)temp;
  unsigned long long* state = (unsigned long long*)((char*)temp + 64);
  cudaError_t e = cudaMemsetAsync(temp, 0, 64 + sizeof(unsigned long long) * (t + 1), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  return launch_pdl(k_unique_compact, dim3((unsigned)(t > 0 ? t : 1)), dim3(UQ_NT), 0, s, keys,
                    m, lbits, edges, total, state, ticket, 1u);
}

// ------------------------------------------------- triangular bitmap path
// 4096 < L with the strictly-upper L x L bit triangle affordable (C5: L ~ 1e5
// to 3e5 -> 1-6 GB of HBM): pair (a, b), a < b, is bit b of row a; row a
// stores only the words from (a + 1) / 32 on, so the rows need no pair
// buffer, no sort and no dedupe, and a row-major walk emits the edges already
// in (a, b) order.  Word offset of row a: a W - sum_{x=1..a} floor(x / 32).
__host__ __device__ __forceinline__ int64_t tri_offset(int64_t a, int64_t W) {
  const int64_t q = a >> 5, r = a & 31;
  return a * W - (32 * q * (q - 1) / 2 + q * (r + 1));
}

int64_t tri_bitmap_words(int64_t L) { return tri_offset(L, (L + 31) / 32); }

// warp per point (lanes over the partner landmarks), as the keys path's pair
// emission: a point in many balls does not serialise on one thread
__global__ void k_tri_bits(const int64_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_lm,
                           int64_t n, int64_t W, uint32_t* __restrict__ bits,
                           unsigned long long* __restrict__ npairs) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long mine = 0ull;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nwarps) {
    const int64_t b = pt_ptr[p], t = pt_ptr[p + 1] - b;
    if (t < 2) continue;
    if (lane == 0) mine += (unsigned long long)(t * (t - 1) / 2);
    for (int64_t i = 0; i + 1 < t; ++i) {
      const int64_t a = pt_lm[b + i];
      uint32_t* row = bits + tri_offset(a, W) - ((a + 1) >> 5);
      for (int64_t c = i + 1 + lane; c < t; c += 32) {
        const int32_t j = pt_lm[b + c];
        atomicOr(row + (j >> 5), 1u << (j & 31));
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FME, mine, o);
  if (lane == 0 && mine) atomicAdd(npairs, mine);
}

// warp per row: number of set bits (edges leaving landmark a)
__global__ void k_tri_rowcount(const uint32_t* __restrict__ bits, int64_t L, int64_t W,
                               int64_t* __restrict__ cnt) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < L; a += nwarps) {
    const uint32_t* row = bits + tri_offset(a, W);
    const int64_t nw = W - ((a + 1) >> 5);
    int64_t c = 0;
    for (int64_t k = lane; k < nw; k += 32) c += __popc(__ldcs(row + k));
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FME, c, o);
    if (lane == 0) cnt[a] = c;
  }
}

// warp per row: edges (a, b) at off[a] onwards, b ascending
__global__ void k_tri_emit(const uint32_t* __restrict__ bits, int64_t L, int64_t W,
                           const int64_t* __restrict__ off, int32_t* __restrict__ edges) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < L; a += nwarps) {
    const int64_t c0 = (a + 1) >> 5;
    const uint32_t* row = bits + tri_offset(a, W);
    const int64_t nw = W - c0;
    int64_t pos = off[a];
    for (int64_t k0 = 0; k0 < nw; k0 += 32) {
      const int64_t k = k0 + lane;
      uint32_t v = k < nw ? __ldcs(row + k) : 0u;
      const uint32_t c = __popc(v);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FME, incl, o);
        if (lane >= o) incl += t;
      }
      int64_t q = pos + incl - c;
      const int32_t jb = (int32_t)((c0 + k) * 32);
      while (v) {
        const int bit = __ffs(v) - 1;
        v &= v - 1u;
        edges[2 * q] = (int32_t)a;
        edges[2 * q + 1] = jb + bit;
        ++q;
      }
      pos += __shfl_sync(FME, incl, 31);
    }
  }
}

static int64_t warp_grid(int64_t rows) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (rows + 7) / 8;   // 8 warps per 256-thread CTA
  const int64_t cap = (int64_t)sms * 8;
  return want < cap ? (want > 0 ? want : 1) : cap;
}

cudaError_t launch_tri_bits(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int64_t L,
                            uint32_t* bits, unsigned long long* npairs, cudaStream_t s,
                            int64_t* launches) {
  const int64_t W = (L + 31) / 32;
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(uint32_t) * tri_bitmap_words(L), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(npairs, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (n + 7) / 8;
  if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
  return launch_pdl(k_tri_bits, dim3((unsigned)(g > 0 ? g : 1)), dim3(256), 0, s, pt_ptr, pt_lm,
                    n, W, bits, npairs);
}

cudaError_t launch_tri_rowcount(const uint32_t* bits, int64_t L, int64_t* cnt, cudaStream_t s,
                                int64_t* launches) {
  ++*launches;
  return launch_pdl(k_tri_rowcount, dim3((unsigned)warp_grid(L)), dim3(256), 0, s, bits, L,
                    (L + 31) / 32, cnt);
}

cudaError_t launch_tri_emit(const uint32_t* bits, int64_t L, const int64_t* off, int32_t* edges,
                            cudaStream_t s, int64_t* launches) {
  ++*launches;
  return launch_pdl(k_tri_emit, dim3((unsigned)warp_grid(L)), dim3(256), 0, s, bits, L,
                    (L + 31) / 32, off, edges);
}

}  // namespace bm
