// sort.cu — device-wide exclusive scan and stable LSD radix sort (steps C, D2).
//
// Both are single-pass-per-level designs with decoupled look-back:
//
// Scan: one kernel.  Each CTA takes the next 4096-element tile by ticket
// (a CTA only ever waits on tiles whose owners already started), publishes
// its tile aggregate, walks back over its predecessors' (aggregate |
// inclusive-prefix) descriptors to find its exclusive offset, publishes its
// inclusive prefix, and writes its outputs.
//
// Radix sort ("onesweep" structure): 8-bit digits over a list of bit ranges.
// (1) one histogram kernel reads the keys once and counts every pass's
// digits; (2) one CTA turns them into global digit offsets; (3) one scatter
// kernel per pass: a CTA takes a 1024- or 4096-key tile by ticket, loads all
// its keys at once, ranks them (peers of equal digit within a warp round from
// a shared-memory OR mask, plus per-warp running digit counts), publishes its
// per-digit counts, places the keys in shared memory in (digit, input) order,
// then looks back per digit (thread d walks digit d, four earlier tiles per
// memory round trip) for the count of equal digits in earlier tiles and
// writes each digit's run out contiguously; equal digits keep their input
// order — LSD stability.  (Measured on 1.4e8 40-bit keys, 5 passes: 10.4 ms
// with match.any ranking and a one-tile look-back, 5.9 ms now.)
//
// Descriptor words carry a per-launch tag and the state arrays are cleared
// once per sort / scan call, so no per-pass reset is needed.
#include <stdlib.h>

#include "internal.cuh"

namespace bm {

constexpr unsigned FM = 0xffffffffu;

// ------------------------------------------------------------------ scan
constexpr int SC_NT = 512, SC_IPT = 8, SC_TILE = SC_NT * SC_IPT;
constexpr uint32_t ST_AGG = 1u, ST_INC = 2u;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(FM, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// block exclusive scan of one value per thread (NT multiple of 32, <= 1024)
template <int NT>
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
  __shared__ int64_t ws[32];
  __shared__ int64_t wtot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int64_t incl = warp_incl_scan(v, lane);
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < NT / 32 ? ws[lane] : 0;
    int64_t si = warp_incl_scan(s, lane);
    ws[lane] = si - s;
    if (lane == 31) wtot = si;
  }
  __syncthreads();
  int64_t r = ws[w] + incl - v;
  if (total) *total = wtot;
  __syncthreads();
  return r;
}

struct ScanState {       // per tile: flag word (tag << 2 | ST_*), aggregate, inclusive prefix
  uint32_t* flag;
  int64_t* agg;
  int64_t* inc;
  int32_t* ticket;
};

__global__ void __launch_bounds__(SC_NT) k_scan_lb(const int64_t* __restrict__ in, int64_t n,
                                                  int64_t* __restrict__ out,
                                                  int64_t* __restrict__ total, ScanState st,
                                                  uint32_t tag) {
  __shared__ int s_tile;
  __shared__ int64_t s_excl;
  pdl_wait();   // (multi-wave, ticketed: the next kernel launches as CTAs exit)
  if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
  int64_t v[SC_IPT];
  int64_t sum = 0;
#pragma unroll
  for (int k = 0; k < SC_IPT; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    sum += v[k];
  }
  int64_t agg;
  int64_t ex = block_excl_scan<SC_NT>(sum, &agg);
  if (threadIdx.x == 0) {
    volatile uint32_t* fl = st.flag;
    volatile int64_t* va = st.agg;
    volatile int64_t* vi = st.inc;
    int64_t excl = 0;
    if (tile == 0) {
      vi[0] = agg;
      __threadfence();
      fl[0] = (tag << 2) | ST_INC;
    } else {
      va[tile] = agg;
      __threadfence();
      fl[tile] = (tag << 2) | ST_AGG;
      for (int64_t j = tile - 1; j >= 0; --j) {
        uint32_t f;
        do {
          f = fl[j];
        } while ((f >> 2) != tag);
        __threadfence();
        if ((f & 3u) == ST_INC) {
          excl += vi[j];
          break;
        }
        excl += va[j];
      }
      vi[tile] = excl + agg;
      __threadfence();
      fl[tile] = (tag << 2) | ST_INC;
    }
    s_excl = excl;
    if ((tile + 1) * SC_TILE >= n && total) *total = excl + agg;
  }
  __syncthreads();
  ex += s_excl;
#pragma unroll
  for (int k = 0; k < SC_IPT; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
}

static int64_t scan_tiles(int64_t n) { return (n + SC_TILE - 1) / SC_TILE; }

size_t scan_temp_bytes(int64_t n) {
  const int64_t t = scan_tiles(n) + 1;
  return (size_t)t * (4 + 8 + 8) + 64;
}

cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp,
                               int64_t* total_dev, cudaStream_t s, int64_t* launches) {
  if (n <= 0) {
    if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(int64_t), s);
    return cudaSuccess;
  }
  const int64_t t = scan_tiles(n);
  ScanState st;
  st.agg = (int64_t*)temp;
  st.inc = st.agg + (t + 1);
  st.flag = (uint32_t*)(st.inc + (t + 1));
  st.ticket = (int32_t*)(st.flag + (t + 1));
  cudaError_t e = cudaMemsetAsync(st.flag, 0, sizeof(uint32_t) * (t + 2), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  return launch_pdl(k_scan_lb, dim3((unsigned)t), dim3(SC_NT), 0, s, in, n, out, total_dev, st,
                    1u);
}

// ------------------------------------------------------------------ radix sort
// Tiles of RS_NT x ROUNDS keys: 1024 for inputs below 2^22 keys (more CTAs,
// shorter per-CTA chains), 4096 above (fewer look-back descriptors).
constexpr int RS_NT = 256, RS_BINS = 256;
constexpr int RS_MAXP = 8;   // 64 bits / 8
constexpr int64_t RS_SMALL = (int64_t)1 << 22;
static inline int rs_rounds(int64_t n) {
  static const int ov = getenv("BM_RS_ROUNDS") ? atoi(getenv("BM_RS_ROUNDS")) : 0;   // A/B diagnostics
  if (ov == 4 || ov == 8 || ov == 16) return ov;
  return n < RS_SMALL ? 4 : 16;
}

struct RsPasses {
  int np;
  int shift[RS_MAXP];
  int bits[RS_MAXP];
};

__global__ void __launch_bounds__(RS_NT) k_rs_hist(const unsigned long long* __restrict__ keys,
                                                  int64_t n, RsPasses P,
                                                  unsigned long long* __restrict__ hist) {
  __shared__ unsigned h[RS_MAXP][RS_BINS];
  pdl_wait();
  pdl_trigger();   // one wave
  for (int p = 0; p < P.np; ++p) h[p][threadIdx.x] = 0u;
  __syncthreads();
  // eight keys per thread in flight (four 16-byte loads) before the counting:
  // with one key per iteration the pass was load-latency-bound (17% of DRAM peak)
  constexpr int KPT = 8;
  const bool aligned = ((uintptr_t)keys & 15u) == 0u;
  const int64_t stride = (int64_t)gridDim.x * RS_NT * KPT;
  int64_t i0 = ((int64_t)blockIdx.x * RS_NT + threadIdx.x) * 2;
  for (; i0 < n; i0 += stride) {
    unsigned long long k[KPT];
#pragma unroll
    for (int v = 0; v < KPT / 2; ++v) {
      const int64_t i = i0 + (int64_t)v * (RS_NT * 2) * gridDim.x;
      if (i + 1 < n && aligned) {
        const ulonglong2 kk = __ldcs(reinterpret_cast<const ulonglong2*>(keys + i));
        k[2 * v] = kk.x;
        k[2 * v + 1] = kk.y;
      } else {
        k[2 * v] = i < n ? keys[i] : 0ull;
        k[2 * v + 1] = i + 1 < n ? keys[i + 1] : 0ull;
      }
    }
#pragma unroll
    for (int v = 0; v < KPT; ++v) {
      const int64_t i = i0 + (int64_t)(v >> 1) * (RS_NT * 2) * gridDim.x + (v & 1);
      if (i < n)
        for (int p = 0; p < P.np; ++p)
          atomicAdd(&h[p][(unsigned)(k[v] >> P.shift[p]) & ((1u << P.bits[p]) - 1u)], 1u);
    }
  }
  __syncthreads();
  for (int p = 0; p < P.np; ++p)
    if (h[p][threadIdx.x]) atomicAdd(&hist[p * RS_BINS + threadIdx.x], (unsigned long long)h[p][threadIdx.x]);
}

// digit offsets: off[p][d] = number of keys with a smaller digit in pass p
__global__ void __launch_bounds__(RS_BINS) k_rs_offsets(const unsigned long long* __restrict__ hist,
                                                       int np, int64_t* __restrict__ off) {
  pdl_wait();
  pdl_trigger();
  for (int p = 0; p < np; ++p) {
    int64_t tot;
    const int64_t ex = block_excl_scan<RS_BINS>((int64_t)hist[p * RS_BINS + threadIdx.x], &tot);
    off[p * RS_BINS + threadIdx.x] = ex;
  }
}

__device__ __forceinline__ unsigned long long rs_pack(uint32_t tag, uint32_t flag, uint32_t v) {
  return ((unsigned long long)tag << 34) | ((unsigned long long)flag << 32) | v;
}

// One pass of the LSD sort over a tile of RS_NT * RS_ROUNDS keys.  Warp w owns
// the contiguous keys [w * 32 * RS_ROUNDS, (w + 1) * 32 * RS_ROUNDS) of the
// tile (round r: 32 consecutive keys), so input order = (warp, round, lane):
//   1. per-warp digit counts with __match_any_sync (no block barriers): each
//      key's rank among equal digits of its warp = the warp's running count +
//      its rank among its round's peers;
//   2. tile histogram -> tile-local digit offsets; per-digit look-back over the
//      earlier tiles -> the digit's global base;
//   3. keys are placed in shared memory in (digit, input order) order, then
//      written out by consecutive threads: each digit's run is a contiguous,
//      coalesced range of the output.  Equal digits keep their input order.
template <int RS_ROUNDS>
__global__ void __launch_bounds__(RS_NT, RS_ROUNDS >= 16 ? 3 : 4) k_rs_scatter(const unsigned long long* __restrict__ in,
                                                     unsigned long long* __restrict__ out,
                                                     int64_t n, int shift, int bits,
                                                     const int64_t* __restrict__ off,
                                                     unsigned long long* state, int32_t* ticket,
                                                     uint32_t tag) {
  constexpr int NW = RS_NT / 32, RS_TILE = RS_NT * RS_ROUNDS;
  __shared__ int s_tile;
  __shared__ int whist[NW][RS_BINS];    // per-warp counts, then per-warp bases
  __shared__ int64_t gbase[RS_BINS];     // global position of the tile's first key of digit d
  __shared__ unsigned long long skey[RS_TILE];
#ifndef BM_RS_MATCH
  // per-warp peer masks of one ranking round (kept zero between rounds); they
  // live in the key staging area, which is filled only after the ranking
  static_assert(NW * RS_BINS * 4 <= RS_TILE * 8, "mask area");
  unsigned(*wmask)[RS_BINS] = reinterpret_cast<unsigned(*)[RS_BINS]>(skey);
#endif
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pdl_wait();   // (multi-wave, ticketed: the next kernel launches as CTAs exit)
  if (tid == 0) s_tile = atomicAdd(ticket, 1);
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) whist[ww][tid] = 0;
#ifndef BM_RS_MATCH
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) wmask[ww][tid] = 0u;
#endif
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t t0 = tile * RS_TILE;
  const int64_t wbeg = t0 + (int64_t)w * 32 * RS_ROUNDS;
  const unsigned mask = (1u << bits) - 1u;
  unsigned long long key[RS_ROUNDS];
  int dig[RS_ROUNDS];
  int wrank[RS_ROUNDS];   // rank among equal digits within the warp
#pragma unroll
  // all of the thread's keys in flight at once (the ranking below has shared
  // memory atomics and warp barriers the compiler will not hoist loads across)
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = wbeg + r * 32 + lane;
    key[r] = i < n ? __ldcs(in + i) : 0ull;
  }
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = wbeg + r * 32 + lane;
    const bool valid = i < n;
    dig[r] = valid ? (int)((unsigned)(key[r] >> shift) & mask) : -1;
#ifdef BM_RS_MATCH
    const unsigned peers = __match_any_sync(FM, dig[r]);
#else
    // peers by a shared-memory OR (match.any is the scatter's longest
    // dependency: ~40% of its stall samples on B200)
    unsigned peers = 0u;
    if (valid) atomicOr(&wmask[w][dig[r]], 1u << lane);
    __syncwarp();
    if (valid) peers = wmask[w][dig[r]];
    __syncwarp();
    if (valid) wmask[w][dig[r]] = 0u;
#endif
    // every peer reads the digit's running count, then the highest peer
    // (no later lane shares its digit: no bit-scan, no shuffle) advances it
    const int before = valid ? whist[w][dig[r]] : 0;
    __syncwarp();
    if (valid && (peers >> lane) == 1u) whist[w][dig[r]] = before + __popc(peers);
    wrank[r] = before + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
  }
  __syncthreads();
  // tile histogram of digit tid, tile-local offsets, per-warp bases
  int c = 0;
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) {
    const int t = whist[ww][tid];
    whist[ww][tid] = c;   // exclusive prefix over the warps
    c += t;
  }
  int64_t tot;
  const int64_t toff = block_excl_scan<RS_NT>((int64_t)c, &tot);
  // per-warp local bases of digit tid: tile offset + the earlier warps' counts
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) whist[ww][tid] += (int)toff;
  // publish this tile's count of digit tid first (successors can look past
  // this tile while it works) ...
  volatile unsigned long long* st = state;
  if (tile == 0) st[tid] = rs_pack(tag, ST_INC, (uint32_t)c);
  else st[tile * RS_BINS + tid] = rs_pack(tag, ST_AGG, (uint32_t)c);
  __syncthreads();
  // ... place the keys in shared memory in (digit, input) order ...
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r)
    if (dig[r] >= 0) skey[whist[w][dig[r]] + wrank[r]] = key[r];
  // ... and only then look back over the earlier tiles for digit tid's global
  // base (four predecessors per memory round trip)
  {
    int64_t excl = 0;
    if (tile > 0) {
      for (int64_t j = tile - 1; j >= 0; j -= 4) {
        unsigned long long v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = j - k >= 0 ? st[(j - k) * RS_BINS + tid] : 0ull;
        bool done = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (done || j - k < 0) continue;
          while ((uint32_t)(v[k] >> 34) != tag || ((v[k] >> 32) & 3ull) == 0ull)
            v[k] = st[(j - k) * RS_BINS + tid];
          excl += (uint32_t)v[k];
          done = ((v[k] >> 32) & 3ull) == ST_INC;
        }
        if (done) break;
      }
      st[tile * RS_BINS + tid] = rs_pack(tag, ST_INC, (uint32_t)(excl + c));
    }
    gbase[tid] = off[tid] + excl - toff;
  }
  __syncthreads();
  // coalesced write-out: consecutive local positions of one digit are consecutive outputs
  const int nloc = (int)min((int64_t)RS_TILE, n - t0);
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int li = r * RS_NT + tid;
    if (li < nloc) {
      const unsigned long long k = skey[li];
      out[gbase[(unsigned)(k >> shift) & mask] + li] = k;
    }
  }
}

static int64_t rs_tiles(int64_t n) {
  const int64_t tile = (int64_t)RS_NT * rs_rounds(n);
  return (n + tile - 1) / tile;
}

// temp layout: off [MAXP][BINS] | hist [MAXP][BINS] | tickets [64] | state [tiles][BINS]
// (hist .. state is one contiguous region cleared by one memset)
size_t radix_temp_bytes(int64_t n) {
  const int64_t t = rs_tiles(n) > 0 ? rs_tiles(n) : 1;
  return (size_t)RS_MAXP * RS_BINS * (8 + 8)      // off, hist
         + 64 * sizeof(int32_t)                     // tickets
         + (size_t)t * RS_BINS * 8 + 256;           // look-back descriptors
}

cudaError_t radix_sort_u64(unsigned long long** keys, unsigned long long** alt, int64_t n,
                           const BitRange* ranges, int nranges, void* temp, cudaStream_t s,
                           int64_t* launches) {
  if (n <= 1) return cudaSuccess;
  RsPasses P{};
  for (int r = 0; r < nranges; ++r)
    for (int sh = ranges[r].lo; sh < ranges[r].hi; sh += 8) {
      if (P.np == RS_MAXP) return cudaErrorInvalidValue;
      P.shift[P.np] = sh;
      P.bits[P.np] = ranges[r].hi - sh < 8 ? ranges[r].hi - sh : 8;
      ++P.np;
    }
  if (P.np == 0) return cudaSuccess;
  const int64_t t = rs_tiles(n);
  int64_t* off = (int64_t*)temp;
  unsigned long long* hist = (unsigned long long*)(off + RS_MAXP * RS_BINS);
  int32_t* tickets = (int32_t*)(hist + RS_MAXP * RS_BINS);
  unsigned long long* state = (unsigned long long*)(tickets + 64);
  cudaError_t e = cudaMemsetAsync(hist, 0,
                                  sizeof(unsigned long long) * RS_MAXP * RS_BINS +
                                      64 * sizeof(int32_t) +
                                      sizeof(unsigned long long) * t * RS_BINS,
                                  s);
  if (e != cudaSuccess) return e;
  int64_t hg = t < 148 * 4 ? t : 148 * 4;
  e = launch_pdl(k_rs_hist, dim3((unsigned)hg), dim3(RS_NT), 0, s, *keys, n, P, hist);
  if (e == cudaSuccess) e = launch_pdl(k_rs_offsets, dim3(1), dim3(RS_BINS), 0, s, hist, P.np, off);
  if (e != cudaSuccess) return e;
  *launches += 2;
  for (int p = 0; p < P.np; ++p) {
    if (rs_rounds(n) == 4)
      e = launch_pdl(k_rs_scatter<4>, dim3((unsigned)t), dim3(RS_NT), 0, s, *keys, *alt, n,
                     P.shift[p], P.bits[p], (const int64_t*)(off + p * RS_BINS), state,
                     tickets + p, (uint32_t)(p + 1));
    else if (rs_rounds(n) == 8)
      e = launch_pdl(k_rs_scatter<8>, dim3((unsigned)t), dim3(RS_NT), 0, s, *keys, *alt, n,
                     P.shift[p], P.bits[p], (const int64_t*)(off + p * RS_BINS), state,
                     tickets + p, (uint32_t)(p + 1));
    else
      e = launch_pdl(k_rs_scatter<16>, dim3((unsigned)t), dim3(RS_NT), 0, s, *keys, *alt, n,
                     P.shift[p], P.bits[p], (const int64_t*)(off + p * RS_BINS), state,
                     tickets + p, (uint32_t)(p + 1));
    ++*launches;
    if (e != cudaSuccess) return e;
    unsigned long long* tmp = *keys;
    *keys = *alt;
    *alt = tmp;
  }
  return cudaSuccess;
}

}  // namespace bm
