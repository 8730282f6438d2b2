// skeleton.cu — NEXT-3: the k-skeleton of the nerve.  A set of
// k+1 landmarks is a k-simplex iff some data point lies in all of their balls
// (Def 2.2: the common intersection ∩ B ∩ X is non-empty), i.e.
// iff it is a (k+1)-subset of some point's landmark row pt_lm[p].  Same
// structure as the 1-skeleton (edges.cu, keys path): per point, every
// (k+1)-subset of its ascending row is packed into one key
// (a_0 << k*lbits | ... | a_k), keys are radix sorted, and one look-back pass
// keeps the first key of every run and unpacks it into [count][k+1].
#include "internal.cuh"

namespace bm {

__device__ __forceinline__ int64_t binom(int64_t t, int r) {
  if (t < r) return 0;
  int64_t c = 1;
  for (int i = 0; i < r; ++i) c = c * (t - i) / (i + 1);
  return c;
}

__global__ void k_simplex_counts(const int64_t* __restrict__ pt_ptr, int64_t n, int r,
                                 int64_t* __restrict__ cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) cnt[p] = binom(pt_ptr[p + 1] - pt_ptr[p], r);
}

// one thread per point: the r-subsets of its row in lexicographic order
__global__ void k_simplex_emit(const int64_t* __restrict__ pt_ptr,
                               const int32_t* __restrict__ pt_lm, int64_t n, int r, int lbits,
                               const int64_t* __restrict__ off,
                               unsigned long long* __restrict__ keys) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t b = pt_ptr[p], t = pt_ptr[p + 1] - b;
  if (t < r) return;
  int idx[8];
  for (int i = 0; i < r; ++i) idx[i] = i;
  int64_t o = off[p];
  for (;;) {
    unsigned long long key = 0ull;
    for (int i = 0; i < r; ++i) key = (key << lbits) | (unsigned long long)pt_lm[b + idx[i]];
    keys[o++] = key;
    int i = r - 1;   // next combination
    while (i >= 0 && idx[i] == (int)(t - r + i)) --i;
    if (i < 0) break;
    ++idx[i];
    for (int q = i + 1; q < r; ++q) idx[q] = idx[q - 1] + 1;
  }
}

// sorted keys -> unique simplices [count][r] (look-back compaction, 2048 keys per CTA)
constexpr int SX_NT = 256, SX_IPT = 8, SX_TILE = SX_NT * SX_IPT;

__global__ void __launch_bounds__(SX_NT) k_simplex_unique(const unsigned long long* __restrict__ keys,
                                                         int64_t m, int r, int lbits,
                                                         int32_t* __restrict__ out, int64_t cap,
                                                         int64_t* __restrict__ total,
                                                         unsigned long long* state,
                                                         int32_t* ticket) {
  __shared__ int s_tile;
  __shared__ uint32_t s_warp[SX_NT / 32];
  __shared__ uint32_t s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t i0 = tile * SX_TILE + (int64_t)threadIdx.x * SX_IPT;
  unsigned long long kv[SX_IPT];
  uint32_t keep = 0u, cnt = 0u;
#pragma unroll
  for (int k = 0; k < SX_IPT; ++k) {
    const int64_t i = i0 + k;
    kv[k] = i < m ? keys[i] : 0ull;
    const bool f = i < m && (i == 0 || kv[k] != (k > 0 ? kv[k - 1] : keys[i - 1]));
    keep |= (f ? 1u : 0u) << k;
    cnt += f ? 1u : 0u;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t agg = 0;
    for (int k = 0; k < SX_NT / 32; ++k) agg += s_warp[k];
    const uint32_t ex = warp_lookback(state, tile, 1u, agg);
    if (threadIdx.x == 0) {
      s_excl = ex;
      if ((tile + 1) * SX_TILE >= m) *total = (int64_t)ex + agg;
    }
  }
  __syncthreads();
  int64_t pos = s_excl + incl - cnt;
  for (int k = 0; k < w; ++k) pos += s_warp[k];
  const unsigned long long lm = (1ull << lbits) - 1ull;
#pragma unroll
  for (int k = 0; k < SX_IPT; ++k) {
    if ((keep >> k) & 1u) {
      if (pos < cap)
        for (int q = 0; q < r; ++q)
          out[pos * r + q] = (int32_t)((kv[k] >> ((r - 1 - q) * lbits)) & lm);
      ++pos;
    }
  }
}

cudaError_t launch_simplex_counts(const int64_t* pt_ptr, int64_t n, int r, int64_t* cnt,
                                  cudaStream_t s) {
  k_simplex_counts<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pt_ptr, n, r, cnt);
  return cudaGetLastError();
}

cudaError_t launch_simplex_emit(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n, int r,
                                int lbits, const int64_t* off, unsigned long long* keys,
                                cudaStream_t s) {
  k_simplex_emit<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(pt_ptr, pt_lm, n, r, lbits, off,
                                                             keys);
  return cudaGetLastError();
}

size_t simplex_unique_temp_bytes(int64_t m) {
  return 64 + sizeof(unsigned long long) * (size_t)((m + SX_TILE - 1) / SX_TILE + 2);
}

cudaError_t launch_simplex_unique(const unsigned long long* keys, int64_t m, int r, int lbits,
                                  int32_t* out, int64_t cap, int64_t* total, void* temp,
                                  cudaStream_t s) {
  const int64_t t = (m + SX_TILE - 1) / SX_TILE;
  int32_t* ticket = (int32_t*)temp;
  unsigned long long* state = (unsigned long long*)((char*)temp + 64);
  cudaError_t e = cudaMemsetAsync(temp, 0, simplex_unique_temp_bytes(m), s);
  if (e != cudaSuccess) return e;
  k_simplex_unique<<<(unsigned)(t > 0 ? t : 1), SX_NT, 0, s>>>(keys, m, r, lbits, out, cap, total,
                                                                state, ticket);
  return cudaGetLastError();
}

}  // namespace bm
