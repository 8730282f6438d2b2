// color.cu — NEXT-1: coloring of the Ball Mapper graph,
// c(l_i) = aggregate of f over X_i = X ∩ B(l_i, eps) (PAPER.md:125-133 [§2.3]).
//
// Aggregators (readings C1-C4 in DESIGN.md): mean,
// min, max, variance (population), range — one warp per ball, fp64
// accumulation over the ball's members from the landmark-major CSR; median
// (even size: mean of the two central values), trimmed mean (drop
// floor(alpha m) at each end) and mode (ties: smallest value) — the members'
// values are sorted per ball first: keys (ball << 32 | order-preserving value
// bits) through the library's radix sort, then one warp per ball reads the
// order statistics.
#include <math.h>

#include "internal.cuh"

namespace bm {

// order-preserving 32-bit code of a value (fp32 or int32) and back to double
__device__ __forceinline__ uint32_t ord_code(uint32_t bits, int is_int) {
  if (is_int) return bits ^ 0x80000000u;
  return (bits & 0x80000000u) ? ~bits : (bits ^ 0x80000000u);
}
__device__ __forceinline__ double ord_value(uint32_t code, int is_int) {
  if (is_int) return (double)(int32_t)(code ^ 0x80000000u);
  const uint32_t bits = (code & 0x80000000u) ? (code ^ 0x80000000u) : ~code;
  return (double)__uint_as_float(bits);
}
__device__ __forceinline__ double load_value(const void* v, int is_int, int64_t i) {
  return is_int ? (double)((const int32_t*)v)[i] : (double)((const float*)v)[i];
}

__device__ __forceinline__ double warp_sum(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// mean, min, max, variance, range: one warp per ball
__global__ void k_color_reduce(const int64_t* __restrict__ ball_ptr,
                               const int32_t* __restrict__ ball_idx, int64_t L,
                               const void* __restrict__ values, int is_int, int agg,
                               double* __restrict__ out) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= L) return;
  const int64_t b = ball_ptr[j], e = ball_ptr[j + 1], m = e - b;
  double s = 0.0, lo = INFINITY, hi = -INFINITY;
  for (int64_t k = b + lane; k < e; k += 32) {
    const double v = load_value(values, is_int, ball_idx[k]);
    s += v;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  s = warp_sum(s);
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  double r;
  if (agg == BM_AGG_MEAN) {
    r = s / (double)m;
  } else if (agg == BM_AGG_MIN) {
    r = lo;
  } else if (agg == BM_AGG_MAX) {
    r = hi;
  } else if (agg == BM_AGG_RANGE) {
    r = hi - lo;
  } else {   // variance, two passes
    const double mu = s / (double)m;
    double q = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) {
      const double t = load_value(values, is_int, ball_idx[k]) - mu;
      q += t * t;
    }
    r = warp_sum(q) / (double)m;
  }
  if (lane == 0) out[j] = m > 0 ? r : NAN;
}

// keys (ball << 32 | order code of the member's value), one warp per ball
__global__ void k_color_keys(const int64_t* __restrict__ ball_ptr,
                             const int32_t* __restrict__ ball_idx, int64_t L,
                             const void* __restrict__ values, int is_int,
                             unsigned long long* __restrict__ keys) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= L) return;
  const int64_t b = ball_ptr[j], e = ball_ptr[j + 1];
  const uint32_t* v = (const uint32_t*)values;
  for (int64_t k = b + lane; k < e; k += 32)
    keys[k] = ((unsigned long long)j << 32) | ord_code(v[ball_idx[k]], is_int);
}

// median, trimmed mean, mode from the per-ball sorted codes
__global__ void k_color_order(const int64_t* __restrict__ ball_ptr, int64_t L,
                              const unsigned long long* __restrict__ keys, int is_int, int agg,
                              double alpha, double* __restrict__ out) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= L) return;
  const int64_t b = ball_ptr[j], m = ball_ptr[j + 1] - b;
  if (m == 0) {
    if (lane == 0) out[j] = NAN;
    return;
  }
  auto val = [&](int64_t k) { return ord_value((uint32_t)keys[b + k], is_int); };
  if (agg == BM_AGG_MEDIAN) {
    if (lane == 0)
      out[j] = (m & 1) ? val((m - 1) / 2) : (val(m / 2 - 1) + val(m / 2)) / 2.0;
  } else if (agg == BM_AGG_TRIMMED) {
    const int64_t t = (int64_t)floor(alpha * (double)m);
    double s = 0.0;
    for (int64_t k = t + lane; k < m - t; k += 32) s += val(k);
    s = warp_sum(s);
    if (lane == 0) out[j] = s / (double)(m - 2 * t);
  } else if (lane == 0) {   // mode: the longest run of equal codes, first (smallest) on ties
    uint32_t best = (uint32_t)keys[b], cur = best;
    int64_t best_n = 0, cur_n = 0;
    for (int64_t k = 0; k < m; ++k) {
      const uint32_t c = (uint32_t)keys[b + k];
      if (c == cur) {
        ++cur_n;
      } else {
        cur = c;
        cur_n = 1;
      }
      if (cur_n > best_n) {
        best_n = cur_n;
        best = cur;
      }
    }
    out[j] = ord_value(best, is_int);
  }
}

cudaError_t launch_color_reduce(const int64_t* ball_ptr, const int32_t* ball_idx, int64_t L,
                                const void* values, int is_int, int agg, double* out,
                                cudaStream_t s) {
  const int64_t g = (L * 32 + 255) / 256;
  k_color_reduce<<<(unsigned)(g > 0 ? g : 1), 256, 0, s>>>(ball_ptr, ball_idx, L, values, is_int,
                                                          agg, out);
  return cudaGetLastError();
}

cudaError_t launch_color_keys(const int64_t* ball_ptr, const int32_t* ball_idx, int64_t L,
                              const void* values, int is_int, unsigned long long* keys,
                              cudaStream_t s) {
  const int64_t g = (L * 32 + 255) / 256;
  k_color_keys<<<(unsigned)(g > 0 ? g : 1), 256, 0, s>>>(ball_ptr, ball_idx, L, values, is_int,
                                                        keys);
  return cudaGetLastError();
}

cudaError_t launch_color_order(const int64_t* ball_ptr, int64_t L, const unsigned long long* keys,
                               int is_int, int agg, double alpha, double* out, cudaStream_t s) {
  const int64_t g = (L * 32 + 255) / 256;
  k_color_order<<<(unsigned)(g > 0 ? g : 1), 256, 0, s>>>(ball_ptr, L, keys, is_int, agg, alpha,
                                                         out);
  return cudaGetLastError();
}

}  // namespace bm
