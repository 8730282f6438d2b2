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
// Gram form: argmin_k |x - c_k|^2 = argmin_k (|c_k|^2 / 2 - x . c_k), one FMA
// per coordinate.  Two points per thread live in registers (DMAX >= d, zero
// padded), the pivots in shared memory read as float4 broadcasts (one LDS.128
// per eight FMAs).  fp32 rounding may pick another pivot on a near tie: the
// cells are only a grouping (centre and radius are exact enough in fp64,
// k_cell_*), no decision depends on which cell a point falls in.
template <int DMAX>
__global__ void __launch_bounds__(256) k_cell_assign(const float* __restrict__ xrows, int xstride,
                                                     int d, int64_t n,
                                                     int32_t* __restrict__ cell) {
  extern __shared__ float4 spiv4[];   // [KC][DMAX / 4], then half norms [KC]
  constexpr int DQ = DMAX / 4;
  float* shalf = reinterpret_cast<float*>(spiv4 + KC * DQ);
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
  for (int k = threadIdx.x; k < KC; k += blockDim.x) {
    float h = 0.f;
    for (int q = 0; q < DQ; ++q) {
      const float4 v = spiv4[k * DQ + q];
      h = fmaf(v.x, v.x, h);
      h = fmaf(v.y, v.y, h);
      h = fmaf(v.z, v.z, h);
      h = fmaf(v.w, v.w, h);
    }
    shalf[k] = 0.5f * h;
  }
  __syncthreads();
  constexpr bool TWO = DMAX <= 64;   // (two 128-coordinate rows do not fit the registers)
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n;
       p0 += (TWO ? 2 : 1) * nthr) {
    const int64_t p1 = TWO ? p0 + nthr : n;
    const float* x0 = xrows + p0 * xstride;
    const float* x1 = xrows + (p1 < n ? p1 : p0) * xstride;
    float xa[DMAX], xb[TWO ? DMAX : 1];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) {
      xa[j] = j < d ? x0[j] : 0.f;
      if constexpr (TWO) xb[j] = j < d ? x1[j] : 0.f;
    }
    float besta = INFINITY, bestb = INFINITY;
    int ka = 0, kb = 0;
    for (int k = 0; k < KC; ++k) {
      const float4* c = spiv4 + k * DQ;
      const float h = shalf[k];
      float a0 = h, a1 = 0.f, b0 = h, b1 = 0.f;
#pragma unroll
      for (int q = 0; q < DQ; ++q) {
        const float4 v = c[q];
        a0 = fmaf(-xa[4 * q], v.x, a0);
        a1 = fmaf(-xa[4 * q + 1], v.y, a1);
        a0 = fmaf(-xa[4 * q + 2], v.z, a0);
        a1 = fmaf(-xa[4 * q + 3], v.w, a1);
        if constexpr (TWO) {
          b0 = fmaf(-xb[4 * q], v.x, b0);
          b1 = fmaf(-xb[4 * q + 1], v.y, b1);
          b0 = fmaf(-xb[4 * q + 2], v.z, b0);
          b1 = fmaf(-xb[4 * q + 3], v.w, b1);
        }
      }
      const float sa = a0 + a1, sb = b0 + b1;
      if (sa < besta) {
        besta = sa;
        ka = k;
      }
      if (sb < bestb) {
        bestb = sb;
        kb = k;
      }
    }
    cell[p0] = ka;
    if (TWO && p1 < n) cell[p1] = kb;
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

// nearest-neighbour chain over the pivots from pivot 0: rank[k].  The chain is
// serial (256 steps, each an argmin over one row of the distance matrix), so
// the whole CTA first stages the matrix's upper triangle in shared memory
// (128 KB) and one warp then walks it without a global round trip per step.
constexpr int kTriWords = KC * (KC - 1) / 2;
__device__ __forceinline__ int tri_index(int a, int b) {   // a < b
  return a * (2 * KC - a - 1) / 2 + (b - a - 1);
}
__global__ void __launch_bounds__(1024) k_pivot_chain(const float* __restrict__ dist /* [KC][KC] */,
                                                      int32_t* __restrict__ rank) {
  extern __shared__ float stri[];   // [kTriWords]
  __shared__ uint32_t svis[KW];
  for (int t = threadIdx.x; t < KC * KC; t += blockDim.x) {
    const int a = t / KC, b = t - a * KC;
    if (a < b) stri[tri_index(a, b)] = dist[t];
  }
  if (threadIdx.x < KW) svis[threadIdx.x] = 0u;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
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
      const bool seen = (svis[k >> 5] >> (k & 31)) & 1u;   // (cur itself is seen)
      if (!seen) {
        // dist[cur][k] and dist[k][cur] are the same fp32 sum (k_pivot_dist adds
        // the squared differences in the same coordinate order)
        const float v = cur < k ? stri[tri_index(cur, k)] : stri[tri_index(k, cur)];
        if (v < bv || (v == bv && k < bi)) {
          bv = v;
          bi = k;
        }
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

// Cell centre and radius (fp64).  The segment of rank r in the sorted order is
// cut into CS_SPLIT slices, one CTA each (KC * CS_SPLIT CTAs keep every SM
// busy whatever the cell sizes); warps stride over the slice's points with
// CS_UN rows in flight, lanes over the coordinates (coalesced rows).
//   k_cell_sum:    per-slice coordinate sums -> part[r][slice][128]
//   k_cell_center: centre = sum of the slices in order / count; rad2 = 0
//   k_cell_rad:    per slice the max squared distance to the centre ->
//                  atomicMax on the bits of the non-negative double rad2[c]
//                  (order-independent: the result is deterministic)
//   k_cell_finish: radius = sqrt(rad2) rounded up; -1 for an empty cell
constexpr int CS_SPLIT = kPruneSplit;
constexpr int CS_NW = 8;   // warps per CTA
constexpr int CS_UN = 8;   // rows in flight per warp

__device__ __forceinline__ void cs_slice(const int64_t* __restrict__ seg, int r, int sp,
                                         int64_t& b, int64_t& e) {
  const int64_t sb = seg[r], len = seg[r + 1] - sb;
  b = sb + len * sp / CS_SPLIT;
  e = sb + len * (sp + 1) / CS_SPLIT;
}

__global__ void __launch_bounds__(CS_NW * 32) k_cell_sum(const float* __restrict__ xrows,
                                                         int xstride, int d,
                                                         const int32_t* __restrict__ perm,
                                                         const int64_t* __restrict__ seg,
                                                         double* __restrict__ part) {
  __shared__ double sacc[CS_NW][128];
  const int r = blockIdx.x / CS_SPLIT, sp = blockIdx.x % CS_SPLIT;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t b, e;
  cs_slice(seg, r, sp, b, e);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};   // d <= 128: lane j holds coordinates j + 32 q
  for (int64_t i0 = b + w; i0 < e; i0 += CS_NW * CS_UN) {
    float v[CS_UN][4];
#pragma unroll
    for (int u = 0; u < CS_UN; ++u) {
      const int64_t i = i0 + (int64_t)u * CS_NW;
      const float* x = i < e ? xrows + (int64_t)__ldg(perm + i) * xstride : nullptr;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = (x && lane + 32 * q < d) ? __ldg(x + lane + 32 * q) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < CS_UN; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += (double)v[u][q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) sacc[w][lane + 32 * q] = acc[q];
  __syncthreads();
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    double sum = 0.0;
    for (int k = 0; k < CS_NW; ++k) sum += sacc[k][j];
    part[((int64_t)r * CS_SPLIT + sp) * 128 + j] = sum;
  }
}

// one CTA per cell c (128 threads over the coordinates)
__global__ void k_cell_center(int d, const int64_t* __restrict__ seg,
                              const int32_t* __restrict__ rank, const double* __restrict__ part,
                              double* __restrict__ center, unsigned long long* __restrict__ rad2) {
  const int c = blockIdx.x, r = rank[c], j = threadIdx.x;
  const int64_t cnt = seg[r + 1] - seg[r];
  if (j < d) {
    double sum = 0.0;
    for (int sp = 0; sp < CS_SPLIT; ++sp) sum += part[((int64_t)r * CS_SPLIT + sp) * 128 + j];
    center[(int64_t)c * d + j] = cnt > 0 ? sum / (double)cnt : 0.0;
  }
  if (j == 0) rad2[c] = 0ull;
}

__global__ void __launch_bounds__(CS_NW * 32) k_cell_rad(const float* __restrict__ xrows,
                                                         int xstride, int d,
                                                         const int32_t* __restrict__ perm,
                                                         const int64_t* __restrict__ seg,
                                                         const int32_t* __restrict__ rank,
                                                         const double* __restrict__ center,
                                                         unsigned long long* __restrict__ rad2) {
  __shared__ double sc[128];
  __shared__ double sred[CS_NW];
  __shared__ int s_cell;
  const int r = blockIdx.x / CS_SPLIT, sp = blockIdx.x % CS_SPLIT;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t b, e;
  cs_slice(seg, r, sp, b, e);
  if (e <= b) return;
  for (int k = threadIdx.x; k < KC; k += blockDim.x)
    if (rank[k] == r) s_cell = k;   // (rank is a permutation: exactly one writer)
  __syncthreads();
  const int c = s_cell;
  for (int j = threadIdx.x; j < 128; j += blockDim.x) sc[j] = j < d ? center[(int64_t)c * d + j] : 0.0;
  __syncthreads();
  double cq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) cq[q] = sc[lane + 32 * q];
  // per point the squared distance (lanes over coordinates), max over points
  double mx = 0.0;
  for (int64_t i0 = b + w; i0 < e; i0 += CS_NW * CS_UN) {
    float v[CS_UN][4];
#pragma unroll
    for (int u = 0; u < CS_UN; ++u) {
      const int64_t i = i0 + (int64_t)u * CS_NW;
      const float* x = i < e ? xrows + (int64_t)__ldg(perm + i) * xstride : nullptr;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = (x && lane + 32 * q < d) ? __ldg(x + lane + 32 * q) : 0.f;
    }
    // each lane's partial squared distances of the 8 rows, then a transposing
    // butterfly (4 + 2 + 1 + 1 + 1 exchanges instead of 5 per row): lane l
    // ends with the whole sum of row 4 l[4] + 2 l[3] + l[2]
    double s2[CS_UN];
#pragma unroll
    for (int u = 0; u < CS_UN; ++u) {
      s2[u] = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < d) {
          const double t = (double)v[u][q] - cq[q];
          s2[u] += t * t;
        }
    }
    static_assert(CS_UN == 8, "the butterfly below folds eight rows");
#pragma unroll
    for (int h = 4, o = 16; h >= 1; h >>= 1, o >>= 1) {
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const double send = hi ? s2[k] : s2[k + h];
        const double keep = hi ? s2[k + h] : s2[k];
        s2[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 2);
    s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 1);
    const int urow = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    // (a row past the slice holds zeros: excluded)
    if (i0 + (int64_t)urow * CS_NW < e) mx = fmax(mx, s2[0]);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) sred[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < CS_NW; ++k) m = fmax(m, sred[k]);
    // non-negative doubles order like their bit patterns
    atomicMax(rad2 + c, (unsigned long long)__double_as_longlong(m));
  }
}

__global__ void k_cell_finish(const int64_t* __restrict__ seg, const int32_t* __restrict__ rank,
                              const unsigned long long* __restrict__ rad2,
                              double* __restrict__ radius) {
  const int c = threadIdx.x;
  const int r = rank[c];
  // the fp64 sums above carry relative errors far below 1e-12; an empty cell
  // is never near anything
  radius[c] = seg[r + 1] > seg[r]
                  ? sqrt(__longlong_as_double((long long)rad2[c])) * (1.0 + 1e-12) + 1e-300
                  : -1.0;
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
  // 16 lanes per row (a 256-byte row is one 16-byte load per lane), 16 rows per CTA
  const int64_t r = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);
  if (r >= n) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)perm[r] * row_bytes);
  uint4* t = reinterpret_cast<uint4*>(dst + r * row_bytes);
  for (int i = threadIdx.x & 15; i < (int)(row_bytes / 16); i += 16) t[i] = s[i];
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
  const size_t smem = sizeof(float) * KC * (dmax + 1);
  auto kern = d <= 32 ? k_cell_assign<32> : (d <= 64 ? k_cell_assign<64> : k_cell_assign<128>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<sms * 2, 256, smem, s>>>(xrows, xstride, d, n, cell);
  k_pivot_dist<<<KC, KC, 0, s>>>(xrows, xstride, d, n, pdist);
  e = cudaFuncSetAttribute(k_pivot_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kTriWords * sizeof(float)));
  if (e != cudaSuccess) return e;
  k_pivot_chain<<<1, 1024, kTriWords * sizeof(float), s>>>(pdist, rank);
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
  const size_t smem = sizeof(float) * KC * (dmax + 1);
  auto kern = d <= 32 ? k_cell_assign<32> : (d <= 64 ? k_cell_assign<64> : k_cell_assign<128>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<sms * 2, 256, smem, s>>>(xrows, xstride, d, n, ps.cell);
  pmark();
  k_pivot_dist<<<KC, KC, 0, s>>>(xrows, xstride, d, n, ps.pdist);
  e = cudaFuncSetAttribute(k_pivot_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kTriWords * sizeof(float)));
  if (e != cudaSuccess) return e;
  k_pivot_chain<<<1, 1024, kTriWords * sizeof(float), s>>>(ps.pdist, ps.rank);
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
  k_cell_sum<<<KC * CS_SPLIT, CS_NW * 32, 0, s>>>(xrows, xstride, d, ps.perm, ps.seg, ps.part);
  k_cell_center<<<KC, 128, 0, s>>>(d, ps.seg, ps.rank, ps.part, ps.center, ps.rad2);
  k_cell_rad<<<KC * CS_SPLIT, CS_NW * 32, 0, s>>>(xrows, xstride, d, ps.perm, ps.seg, ps.rank,
                                                  ps.center, ps.rad2);
  k_cell_finish<<<1, KC, 0, s>>>(ps.seg, ps.rank, ps.rad2, ps.radius);
  pmark();
  k_cell_near<<<KC * KC / 256, 256, 0, s>>>(ps.center, ps.radius, d, eps, ps.near);
  const int64_t nblk = (n + 127) / 128;
  k_block_masks<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, s>>>(ps.perm, ps.cell, n, nblk,
                                                                   ps.near, ps.bmask);
  pmark();
  k_gather_rows<<<(unsigned)((n + 15) / 16), 256, 0, s>>>(xop, row_bytes, ps.perm, n, ps.xop_perm);
  k_gather_f64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nrm, ps.perm, n, ps.nrm_perm);
  pmark();
  *launches += 8;
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
