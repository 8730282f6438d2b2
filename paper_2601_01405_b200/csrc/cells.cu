// cells.cu — tile-level pruning of the membership contraction (the paper's
// ball-tree idea, §3.1, moved from single points to 128-row blocks
// and 32-landmark chunks of the tensor-core tiles).
//
// Once per build: the points are assigned to K = 256 cells (nearest of 256
// pivot points, fp32 — only a grouping, no decision depends on it), the cells
// are ordered along a nearest-neighbour chain of the pivots, and the points
// are permuted by (cell rank, index) for the contraction's A operand, so a
// 128-row block covers one or two neighbouring cells.  Every cell gets an
// fp64 centre and a radius rounded up; cells a and b are "near" unless
//   |c_a - c_b| (1 - 1e-12) >= r_a + r_b + eps (1 + 4e-6),
// and if they are not near every pair (p in a, l in b) has
//   d(p, l) >= |c_a - c_b| - r_a - r_b >= eps (1 + 4e-6):
// out, and outside the 1e-6 eps near-tie band, so it may be skipped.
// Per greedy tile the new landmarks are sorted by cell rank (stable; in the
// resolve CTA, greedy.cu) and each 32-column chunk gets the bit set of its
// landmarks' cells; the contraction
// skips a chunk whose cells are near none of the row block's cells (no TMEM
// read) and a whole 256-column tile whose chunks are all skipped (no MMA).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"

namespace bm {

constexpr int KC = kPruneCells;          // 256 cells
constexpr int KW = kPruneCells / 32;     // mask words

// nearest pivot (pivot i = point i * (n / K)); fp32 rows, first d coordinates.
// The point's row lives in registers (DMAX >= d, zero padded), the pivots in
// shared memory read as float4 broadcasts (one LDS.128 per four FMAs).
template <int DMAX>
__global__ void __launch_bounds__(256) k_cell_assign(const float* __restrict__ xrows, int xstride,
                                                     int d, int64_t n,
                                                     int32_t* __restrict__ cell) {
  extern __shared__ float4 spiv4[];   // [KC][DMAX / 4]
  constexpr int DQ = DMAX / 4;
  const int64_t step = n / KC;
  for (int t = threadIdx.x; t < KC * DQ; t += blockDim.x) {
    const int k = t / DQ, q = t - k * DQ;
    const float* c = xrows + (int64_t)k * step * xstride;
    float4 v;
    v.x = 4 * q + 0 < d ? c[4 * q + 0] : 0.f;
    v.y = 4 * q + 1 < d ? c[4 * q + 1] : 0.f;
    v.z = 4 * q + 2 < d ? c[4 * q + 2] : 0.f;
    v.w = 4 * q + 3 < d ? c[4 * q + 3] : 0.f;
    spiv4[t] = v;
  }
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const float* x = xrows + p * xstride;
    float xr[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) xr[j] = j < d ? x[j] : 0.f;
    float best = INFINITY;
    int bk = 0;
    for (int k = 0; k < KC; ++k) {
      const float4* c = spiv4 + k * DQ;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int q = 0; q < DQ; ++q) {
        const float4 v = c[q];
        const float t0 = xr[4 * q] - v.x, t1 = xr[4 * q + 1] - v.y;
        const float t2 = xr[4 * q + 2] - v.z, t3 = xr[4 * q + 3] - v.w;
        s0 = fmaf(t0, t0, s0);
        s1 = fmaf(t1, t1, s1);
        s0 = fmaf(t2, t2, s0);
        s1 = fmaf(t3, t3, s1);
      }
      const float sv = s0 + s1;
      if (sv < best) {
        best = sv;
        bk = k;
      }
    }
    cell[p] = bk;
  }
}

// pivot distances: CTA a, thread b (squared, fp32)
__global__ void k_pivot_dist(const float* __restrict__ xrows, int xstride, int d, int64_t n,
                             float* __restrict__ dist) {
  const int64_t step = n / KC;
  const int a = blockIdx.x, b = threadIdx.x;
  const float* x = xrows + (int64_t)a * step * xstride;
  const float* y = xrows + (int64_t)b * step * xstride;
  float s = 0.f;
  for (int j = 0; j < d; ++j) {
    const float u = x[j] - y[j];
    s = fmaf(u, u, s);
  }
  dist[a * KC + b] = s;
}

// nearest-neighbour chain over the pivots from pivot 0 (one warp): rank[k]
__global__ void k_pivot_chain(const float* __restrict__ dist /* [KC][KC] */,
                              int32_t* __restrict__ rank) {
  const int lane = threadIdx.x;
  __shared__ uint32_t svis[KW];
  if (lane < KW) svis[lane] = 0u;
  __syncwarp();
  int cur = 0;
  for (int r = 0; r < KC; ++r) {
    if (lane == 0) {
      rank[cur] = r;
      svis[cur >> 5] |= 1u << (cur & 31);
    }
    __syncwarp();
    float bv = INFINITY;
    int bi = KC;
#pragma unroll
    for (int i = 0; i < KC / 32; ++i) {
      const int k = lane + 32 * i;
      const bool seen = (svis[k >> 5] >> (k & 31)) & 1u;
      const float v = __ldcg(dist + cur * KC + k);
      if (!seen && (v < bv || (v == bv && k < bi))) {
        bv = v;
        bi = k;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (bi < KC) cur = bi;
    __syncwarp();
  }
}

__global__ void k_cell_keys(const int32_t* __restrict__ cell, const int32_t* __restrict__ rank,
                            int64_t n, unsigned long long* __restrict__ keys) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) keys[p] = ((unsigned long long)(uint32_t)rank[cell[p]] << 32) | (uint64_t)p;
}

// one CTA per cell rank r: the segment of the sorted points with that rank.
// Warps stride over the points, lanes over the coordinates (coalesced rows).
__global__ void __launch_bounds__(512) k_cell_stats(const float* __restrict__ xrows, int xstride,
                                                    int d, const int32_t* __restrict__ perm,
                                                    const int64_t* __restrict__ seg,
                                                    const int32_t* __restrict__ rank,
                                                    double* __restrict__ center,
                                                    double* __restrict__ radius) {
  constexpr int NW = 16;   // warps
  constexpr int UN = 4;    // rows in flight per warp
  __shared__ double sacc[NW][128];
  __shared__ double sc[128];
  __shared__ double sred[NW];
  __shared__ int s_cell;
  const int r = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = seg[r], e = seg[r + 1];
  if (threadIdx.x == 0) s_cell = -1;
  __syncthreads();
  for (int k = threadIdx.x; k < KC; k += blockDim.x)
    if (rank[k] == r) s_cell = k;
  __syncthreads();
  const int c = s_cell;
  if (c < 0) return;
  if (e <= b) {   // empty cell: never near anything
    if (threadIdx.x == 0) radius[c] = -1.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) center[(int64_t)c * d + j] = 0.0;
    return;
  }
  // centre: per-warp partial sums (lane j: coordinates j, j + 32, ...), then across warps
  double part[4] = {0.0, 0.0, 0.0, 0.0};   // d <= 128
  for (int64_t i0 = b + w; i0 < e; i0 += NW * UN) {
    float v[UN][4];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t i = i0 + (int64_t)u * NW;
      const float* x = i < e ? xrows + (int64_t)__ldg(perm + i) * xstride : nullptr;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = (x && lane + 32 * q < d) ? __ldg(x + lane + 32 * q) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) part[q] += (double)v[u][q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (lane + 32 * q < 128) sacc[w][lane + 32 * q] = part[q];
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double sum = 0.0;
    for (int k = 0; k < NW; ++k) sum += sacc[k][j];
    const double m = sum / (double)(e - b);
    center[(int64_t)c * d + j] = m;
    sc[j] = m;
  }
  __syncthreads();
  // radius: per point the squared distance (lanes over coordinates), max over points
  double mx = 0.0;
  for (int64_t i0 = b + w; i0 < e; i0 += NW * UN) {
    float v[UN][4];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t i = i0 + (int64_t)u * NW;
      const float* x = i < e ? xrows + (int64_t)__ldg(perm + i) * xstride : nullptr;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = (x && lane + 32 * q < d) ? __ldg(x + lane + 32 * q) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      if (i0 + (int64_t)u * NW >= e) break;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < d) {
          const double t = (double)v[u][q] - sc[lane + 32 * q];
          s += t * t;
        }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      mx = fmax(mx, s);
    }
  }
  if (lane == 0) sred[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < NW; ++k) m = fmax(m, sred[k]);
    // the fp64 sums above carry relative errors far below 1e-12
    radius[c] = sqrt(m) * (1.0 + 1e-12) + 1e-300;
  }
}

// near[a][w]: bit b of word w set iff cells a and b may hold an in-ball pair
__global__ void k_cell_near(const double* __restrict__ center, const double* __restrict__ radius,
                            int d, double eps, uint32_t* __restrict__ near) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;   // KC * KC threads
  const int a = t / KC, b = t - a * KC;
  bool nr = false;
  if (a < KC) {
    const double ra = radius[a], rb = radius[b];
    if (ra >= 0.0 && rb >= 0.0) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) {
        const double u = center[(int64_t)a * d + j] - center[(int64_t)b * d + j];
        s += u * u;
      }
      const double dcc = sqrt(s) * (1.0 - 1e-12);
      nr = !(dcc >= ra + rb + eps * (1.0 + 4e-6));
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, nr);
  if ((threadIdx.x & 31) == 0 && a < KC) near[a * KW + (b >> 5)] = m;
}

// bmask[blk][w]: OR of near rows over the cells present in row block blk
// (rows 128 blk .. 128 blk + 127 of the permuted order; padding rows none)
__global__ void k_block_masks(const int32_t* __restrict__ perm, const int32_t* __restrict__ cell,
                              int64_t n, int64_t nblk, const uint32_t* __restrict__ near,
                              uint32_t* __restrict__ bmask) {
  const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blk >= nblk) return;
  uint32_t acc[KW];
#pragma unroll
  for (int w = 0; w < KW; ++w) acc[w] = 0u;
  for (int i = lane; i < 128; i += 32) {
    const int64_t r = blk * 128 + i;
    if (r < n) {
      const int c = cell[perm[r]];
#pragma unroll
      for (int w = 0; w < KW; ++w) acc[w] |= near[c * KW + w];
    }
  }
#pragma unroll
  for (int w = 0; w < KW; ++w) {
    uint32_t v = acc[w];
    for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) bmask[blk * KW + w] = v;
  }
}

__global__ void k_gather_rows(const uint8_t* __restrict__ src, int64_t row_bytes,
                              const int32_t* __restrict__ perm, int64_t n,
                              uint8_t* __restrict__ dst) {
  const int64_t r = blockIdx.x;
  if (r >= n) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)perm[r] * row_bytes);
  uint4* t = reinterpret_cast<uint4*>(dst + r * row_bytes);
  for (int i = threadIdx.x; i < (int)(row_bytes / 16); i += blockDim.x) t[i] = s[i];
}

__global__ void k_gather_f64(const double* __restrict__ src, const int32_t* __restrict__ perm,
                             int64_t n, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[perm[r]];
}

// The spatial order alone (also used by the FPS kernel): cells, pivot chain,
// points sorted by (cell rank, index) into perm; keys hold the sorted keys.
cudaError_t cell_order(const float* xrows, int xstride, int d, int64_t n, int32_t* cell,
                       int32_t* rank, float* pdist, unsigned long long** keys,
                       unsigned long long** alt, void* sort_temp, int32_t* perm, cudaStream_t s,
                       int64_t* launches) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int dmax = d <= 32 ? 32 : (d <= 64 ? 64 : 128);
  const size_t smem = sizeof(float) * KC * dmax;
  auto kern = d <= 32 ? k_cell_assign<32> : (d <= 64 ? k_cell_assign<64> : k_cell_assign<128>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<sms * 2, 256, smem, s>>>(xrows, xstride, d, n, cell);
  k_pivot_dist<<<KC, KC, 0, s>>>(xrows, xstride, d, n, pdist);
  k_pivot_chain<<<1, 32, 0, s>>>(pdist, rank);
  k_cell_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cell, rank, n, *keys);
  *launches += 4;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const BitRange br[2] = {{0, 32}, {32, 40}};
  e = radix_sort_u64(keys, alt, n, br, 2, sort_temp, s, launches);
  if (e != cudaSuccess) return e;
  return launch_unpack_low(*keys, n, 0xffffffffull, perm, s, launches);
}

cudaError_t prune_prepare(const float* xrows, int xstride, int d, int64_t n, double eps,
                          const uint8_t* xop, int64_t row_bytes, const double* nrm, PruneState& ps,
                          void* sort_temp, unsigned long long* keys, unsigned long long* alt,
                          cudaStream_t s, int64_t* launches) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const bool ptr = getenv("BM_PRUNE_TRACE") != nullptr;   // diagnostics
  cudaEvent_t pe[12];
  int npe = 0;
  auto pmark = [&]() {
    if (ptr && npe < 12) {
      cudaEventCreate(&pe[npe]);
      cudaEventRecord(pe[npe++], s);
    }
  };
  pmark();
  const int dmax = d <= 32 ? 32 : (d <= 64 ? 64 : 128);
  const size_t smem = sizeof(float) * KC * dmax;
  auto kern = d <= 32 ? k_cell_assign<32> : (d <= 64 ? k_cell_assign<64> : k_cell_assign<128>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<sms * 2, 256, smem, s>>>(xrows, xstride, d, n, ps.cell);
  pmark();
  k_pivot_dist<<<KC, KC, 0, s>>>(xrows, xstride, d, n, ps.pdist);
  k_pivot_chain<<<1, 32, 0, s>>>(ps.pdist, ps.rank);
  pmark();
  k_cell_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ps.cell, ps.rank, n, keys);
  *launches += 3;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const BitRange br[2] = {{0, 32}, {32, 40}};
  unsigned long long* k = keys;
  unsigned long long* a = alt;
  e = radix_sort_u64(&k, &a, n, br, 2, sort_temp, s, launches);
  if (e != cudaSuccess) return e;
  e = launch_unpack_low(k, n, 0xffffffffull, ps.perm, s, launches);
  if (e != cudaSuccess) return e;
  e = launch_segment_ptr(k, n, 32, 0xffull, KC, ps.seg, s, launches);
  if (e != cudaSuccess) return e;
  pmark();
  k_cell_stats<<<KC, 512, 0, s>>>(xrows, xstride, d, ps.perm, ps.seg, ps.rank, ps.center,
                                  ps.radius);
  pmark();
  k_cell_near<<<KC * KC / 256, 256, 0, s>>>(ps.center, ps.radius, d, eps, ps.near);
  const int64_t nblk = (n + 127) / 128;
  k_block_masks<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, s>>>(ps.perm, ps.cell, n, nblk,
                                                                   ps.near, ps.bmask);
  pmark();
  k_gather_rows<<<(unsigned)n, 64, 0, s>>>(xop, row_bytes, ps.perm, n, ps.xop_perm);
  k_gather_f64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nrm, ps.perm, n, ps.nrm_perm);
  pmark();
  *launches += 5;
  if (ptr) {
    cudaEventSynchronize(pe[npe - 1]);
    static const char* nm[] = {"assign", "chain", "keys+sort+seg", "stats", "near+masks",
                               "gathers"};
    for (int i = 0; i + 1 < npe; ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, pe[i], pe[i + 1]);
      fprintf(stderr, "prune %-14s %8.3f ms\n", nm[i], t);
    }
    for (int i = 0; i < npe; ++i) cudaEventDestroy(pe[i]);
  }
  return cudaGetLastError();
}

}  // namespace bm
