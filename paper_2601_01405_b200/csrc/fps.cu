// fps.cu — NEXT-2: the farthest point sampling eps-net
// (PAPER.md:108-119 [§2.2]).  Start from x_0; repeatedly take
// x* = argmax_x min_{l in L} d(x, l) and add it while that maximum is >= eps
// (reading F1: the paper's "> eps" would leave a point at distance exactly eps
// uncovered by the open balls); ties go to the lowest index (reading F2).
//
// One persistent cooperative kernel: every thread owns a fixed strided set of
// points and their running min distance; per step the CTAs fold in the newest
// landmark, reduce their (max, lowest index) candidate, one grid barrier, and
// every CTA reduces all candidates identically (double-buffered, so one
// barrier per landmark suffices).  Distances are the oracle's fp64 formulas
// operation for operation (ascending coordinates, no contraction; L2 compares
// squared distances with eps^2), so the argmax — an integer decision — is
// taken in the same precision as the oracle's (F3).
#include <cooperative_groups.h>
#include <math.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace bm {

struct FpsArgs {
  const uint2* rows;   // prepped rows (fp32 bits, or int8 with u8 shifted by -128)
  int nu, d, kind;     // Kind (K_L2F, K_L1F, K_COSF, K_L2I, K_L1I)
  int64_t n;
  double thr;          // eps^2 for L2, eps otherwise
  int64_t start;
  double* mind;        // [n]
  int32_t* seq;        // [n] selection order
  int32_t* L_out;
  double* cval;        // [2][grid] candidate values
  int64_t* cidx;       // [2][grid] candidate indices
};

__device__ __forceinline__ double fps_dist(const FpsArgs& a, int64_t p, const float* lf,
                                           const int8_t* li) {
  if (a.kind == K_L2F || a.kind == K_L1F || a.kind == K_COSF) {
    const float* x = reinterpret_cast<const float*>(a.rows + p * (int64_t)a.nu);
    if (a.kind == K_L2F) {
      double s = 0.0;
      for (int j = 0; j < a.d; ++j) {
        const double t = __dsub_rn((double)x[j], (double)lf[j]);
        s = __dadd_rn(s, __dmul_rn(t, t));
      }
      return s;
    }
    if (a.kind == K_L1F) {
      double s = 0.0;
      for (int j = 0; j < a.d; ++j) s = __dadd_rn(s, fabs(__dsub_rn((double)x[j], (double)lf[j])));
      return s;
    }
    double dot = 0.0, xx = 0.0, yy = 0.0;
    for (int j = 0; j < a.d; ++j) {
      const double u = (double)x[j], v = (double)lf[j];
      dot = __dadd_rn(dot, __dmul_rn(u, v));
      xx = __dadd_rn(xx, __dmul_rn(u, u));
      yy = __dadd_rn(yy, __dmul_rn(v, v));
    }
    if (xx == 0.0 && yy == 0.0) return 0.0;
    if (xx == 0.0 || yy == 0.0) return 1.0;
    return __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(xx), __dsqrt_rn(yy))));
  }
  const int8_t* x = reinterpret_cast<const int8_t*>(a.rows + p * (int64_t)a.nu);
  int64_t s = 0;
  for (int j = 0; j < a.d; ++j) {
    const int64_t t = (int64_t)x[j] - (int64_t)li[j];
    s += a.kind == K_L2I ? t * t : (t < 0 ? -t : t);
  }
  return (double)s;
}

// (value, index) order of the argmax: larger value first, then lower index
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

constexpr int FPS_NT = 256;

__global__ void __launch_bounds__(FPS_NT) k_fps(FpsArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float slm[];   // the current landmark's coordinates (fp32 or int8)
  __shared__ double sv[FPS_NT / 32];
  __shared__ int64_t si[FPS_NT / 32];
  __shared__ int64_t s_next;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t gt = (int64_t)blockIdx.x * FPS_NT + tid, gs = (int64_t)gridDim.x * FPS_NT;
  const bool is_float = a.kind == K_L2F || a.kind == K_L1F || a.kind == K_COSF;
  int64_t cur = a.start;
  int64_t L = 0;
  for (int step = 0;; ++step) {
    if (blockIdx.x == 0 && tid == 0) a.seq[L] = (int32_t)cur;
    ++L;
    // the landmark's coordinates
    for (int j = tid; j < a.d; j += FPS_NT) {
      if (is_float) slm[j] = reinterpret_cast<const float*>(a.rows + cur * (int64_t)a.nu)[j];
      else reinterpret_cast<int8_t*>(slm)[j] =
          reinterpret_cast<const int8_t*>(a.rows + cur * (int64_t)a.nu)[j];
    }
    __syncthreads();
    double bv = -INFINITY;
    int64_t bi = a.n;
    for (int64_t p = gt; p < a.n; p += gs) {
      const double v = fps_dist(a, p, slm, reinterpret_cast<const int8_t*>(slm));
      const double m = step == 0 ? v : fmin(a.mind[p], v);
      a.mind[p] = m;
      if (better(m, p, bv, bi)) {
        bv = m;
        bi = p;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sv[w] = bv;
      si[w] = bi;
    }
    __syncthreads();
    const int buf = step & 1;
    if (tid == 0) {
      double v = sv[0];
      int64_t i = si[0];
      for (int k = 1; k < FPS_NT / 32; ++k)
        if (better(sv[k], si[k], v, i)) {
          v = sv[k];
          i = si[k];
        }
      a.cval[buf * gridDim.x + blockIdx.x] = v;
      a.cidx[buf * gridDim.x + blockIdx.x] = i;
    }
    grid.sync();
    // every CTA reduces all candidates the same way
    if (w == 0) {
      double v = -INFINITY;
      int64_t i = a.n;
      for (int k = lane; k < (int)gridDim.x; k += 32) {
        const double cv = a.cval[buf * gridDim.x + k];
        const int64_t ci = a.cidx[buf * gridDim.x + k];
        if (better(cv, ci, v, i)) {
          v = cv;
          i = ci;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (better(ov, oi, v, i)) {
          v = ov;
          i = oi;
        }
      }
      if (lane == 0) s_next = (i < a.n && v >= a.thr) ? i : -1;   // reading F1: >= eps
    }
    __syncthreads();
    cur = s_next;
    if (cur < 0) break;
    __syncthreads();   // slm is rewritten next step
  }
  if (blockIdx.x == 0 && tid == 0) *a.L_out = (int32_t)L;
}

cudaError_t launch_fps(const uint2* rows, int nu, int d, int kind, int64_t n, double thr,
                       int64_t start, double* mind, int32_t* seq, int32_t* L_out, double* cval,
                       int64_t* cidx, int grid, cudaStream_t s) {
  FpsArgs a{rows, nu, d, kind, n, thr, start, mind, seq, L_out, cval, cidx};
  void* args[] = {&a};
  const size_t smem = (size_t)d * sizeof(float);
  return cudaLaunchCooperativeKernel((void*)k_fps, dim3(grid), dim3(FPS_NT), args, smem, s);
}

__global__ void k_fps_keys(const int32_t* __restrict__ seq, int64_t L,
                           unsigned long long* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < L) keys[i] = (unsigned long long)(uint32_t)seq[i];
}

// the selection order -> sort keys (the cover lists landmarks ascending)
cudaError_t launch_fps_keys(const int32_t* seq, int64_t L, unsigned long long* keys,
                            cudaStream_t s, int64_t* launches) {
  k_fps_keys<<<(unsigned)((L + 255) / 256), 256, 0, s>>>(seq, L, keys);
  ++*launches;
  return cudaGetLastError();
}

int fps_grid(int d) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fps, FPS_NT, (size_t)d * sizeof(float));
  if (per < 1) per = 1;
  if (per > 4) per = 4;
  return sms * per;
}

}  // namespace bm
