#include <stdlib.h>
// prep.cu — step A0: pack rows into 8-byte units, norms, finite check.
//
// fp32 rows are copied bit-for-bit (zero padded to NU units): the CUDA-core
// kernels score them in fp32 and the fp64 recheck reads the same values.  For
// cosine, xhat = x / ||x|| (norm in fp64) rounded to fp32; a
// zero row gets NaN so that every pair touching it lands in the fp64 band.
// Integer rows are packed as int8 (uint8 shifted by -128: exact, distances are
// translation invariant) with exact int32 squared norms for the Gram form
// d^2 = |x|^2 + |y|^2 - 2 x.y.
#include <math.h>

#include "internal.cuh"

namespace bm {

// G lanes per row (G = 1..8, the smallest power of two >= the row's float
// count, capped at 8): lanes stride over the row, coalesced for wide rows.
__global__ void k_prep_f32(const float* __restrict__ X, int64_t n, int d, int nu, int cosine,
                           int G, uint2* __restrict__ rows, uint2* __restrict__ xhat,
                           DevStats* stats) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = gt / G;
  const int lane = (int)(gt % G);
  const bool live = p < n;
  const float* x = X + p * (int64_t)d;
  float* r = reinterpret_cast<float*>(rows) + p * (int64_t)(2 * nu);
  double ss = 0.0;
  bool finite = true;
  for (int j = lane; live && j < 2 * nu; j += G) {
    const float a = j < d ? x[j] : 0.f;
    finite = finite && isfinite(a);
    r[j] = a;
    ss = __dadd_rn(ss, __dmul_rn((double)a, (double)a));
  }
  for (int o = G / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (!finite) atomicExch(&stats->nonfinite, 1);
  if (cosine && live) {
    float* h = reinterpret_cast<float*>(xhat) + p * (int64_t)(2 * nu);
    const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
    for (int j = lane; j < 2 * nu; j += G) {
      const float a = j < d ? x[j] : 0.f;
      // a zero row gets NaN in unit 0 so every pair with it goes to the fp64 rule
      h[j] = ss == 0.0 ? (j < 2 ? __int_as_float(0x7fc00000) : 0.f) : (float)((double)a * inv);
    }
  }
}

__global__ void k_prep_int(const uint8_t* __restrict__ X, int64_t n, int d, int nu, int is_u8,
                           uint2* __restrict__ rows, int32_t* __restrict__ inorm) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const uint8_t* x = X + p * (int64_t)d;
  uint32_t* r = reinterpret_cast<uint32_t*>(rows + p * (int64_t)nu);
  int32_t ss = 0;
  for (int w = lane; w < 2 * nu; w += 32) {   // 4 coordinates per 32-bit word
    uint32_t word = 0u;
    for (int k = 0; k < 4; ++k) {
      const int j = 4 * w + k;
      int v = 0;
      if (j < d) v = is_u8 ? (int)x[j] - 128 : (int)(int8_t)x[j];
      ss += v * v;
      word |= ((uint32_t)(uint8_t)(int8_t)v) << (8 * k);
    }
    r[w] = word;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (inorm && lane == 0) inorm[p] = ss;
}

// ---- L1 prefilter rows
// float -> int with the same order (for atomicMin / atomicMax)
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__global__ void k_minmax(const float* __restrict__ X, int64_t m, int* __restrict__ mm) {
  float lo = INFINITY, hi = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = X[i];
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], f2ord(lo));
    atomicMax(&mm[1], f2ord(hi));
  }
}

// q = rint((x - min) / s), s = (max - min) / 255, 4 coordinates per word, zero padded
__global__ void k_l1_quantize(const float* __restrict__ X, int64_t n, int d, int nq,
                              const int* __restrict__ mm, double* __restrict__ qparam,
                              uint32_t* __restrict__ qrows) {
  const double mn = (double)ord2f(mm[0]), mx = (double)ord2f(mm[1]);
  const double sc = mx > mn ? (mx - mn) / 255.0 : 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    qparam[0] = mn;
    qparam[1] = mx;
  }
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float* x = X + p * (int64_t)d;
  for (int w = 0; w < nq; ++w) {
    uint32_t word = 0u;
    for (int k = 0; k < 4; ++k) {
      const int j = 4 * w + k;
      uint32_t q = 0u;
      if (j < d) {
        double t = rint(((double)x[j] - mn) / sc);
        t = t < 0.0 ? 0.0 : (t > 255.0 ? 255.0 : t);
        q = (uint32_t)t;
      }
      word |= q << (8 * k);
    }
    qrows[p * nq + w] = word;
  }
}

bool pdl_enabled() {
  static const bool on = getenv("BM_NO_PDL") == nullptr;
  return on;
}

int l1q_words(int d) {
  if (d > 64) return 0;
  int w = 1;
  while (4 * w < d) w *= 2;
  return w;
}

cudaError_t launch_l1_quantize(const float* X, int64_t n, int d, int nq, double* qparam,
                               uint32_t* qrows, cudaStream_t s, int64_t* launches) {
  int* mm = reinterpret_cast<int*>(qparam + 2);   // scratch after the two doubles
  const int init[2] = {0x7fffffff, (int)0x80000000};
  cudaError_t e = cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  const int64_t m = n * (int64_t)d;
  int64_t g = (m + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  k_minmax<<<(unsigned)g, 256, 0, s>>>(X, m, mm);
  k_l1_quantize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(X, n, d, nq, mm, qparam, qrows);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_prep(const void* X, int dtype, int64_t n, int d, int kind, int nu,
                        uint2* rows, uint2* xhat, int32_t* inorm, DevStats* stats,
                        cudaStream_t s, int64_t* launches) {
  int bs = 256;
  if (dtype == BM_F32) {
    int G = 1;   // lanes per row (each strides over the row's 2 nu floats)
    while (G < 8 && G < 2 * nu) G *= 2;
    const int64_t g = (n * G + bs - 1) / bs;
    k_prep_f32<<<(unsigned)g, bs, 0, s>>>((const float*)X, n, d, nu, kind == K_COSF, G, rows,
                                          xhat, stats);
  } else {
    const int64_t g = (n * 32 + bs - 1) / bs;   // integer rows: one warp per row
    k_prep_int<<<(unsigned)g, bs, 0, s>>>((const uint8_t*)X, n, d, nu, dtype == BM_U8, rows,
                                          inorm);
  }
  ++*launches;
  return cudaGetLastError();
}

}  // namespace bm
