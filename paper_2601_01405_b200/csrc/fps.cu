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
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace bm {

struct FpsArgs {
  const uint2* rows;   // prepped rows: nu 8-byte units (fp32 pairs, or 8 int8 with u8 shifted by -128)
  const int32_t* inorm;   // K_L2I: sum of squares of the prepped row
  int nu, nue, d;      // row stride in units; units holding the d coordinates
  int64_t n;
  double thr;          // eps^2 for L2, eps otherwise
  int64_t start;
  double* mind;        // [n] running minimum (only when the points do not fit in registers)
  int32_t* seq;        // [n] selection order
  int32_t* L_out;
  double* cval;        // [2][grid] candidate values
  int64_t* cidx;       // [2][grid] candidate indices
  const int32_t* perm; // spatial order (null: strided ownership, no pruning)
  unsigned long long* dbg;   // diagnostics (BM_FPS_DEBUG): [0] warp-steps, [1] skipped
};

// d(x_p, l) with l's units in shared memory.  Float kinds: the oracle's fp64
// formula operation for operation (coordinates ascending, no contraction; the
// zero padding of the last unit adds an exact +0).  Integer kinds: exact
// integer arithmetic, so any order gives the oracle's value — L2 as
// |x|^2 + |l|^2 - 2 x.l with 4-way int8 dot products, L1 as byte SADs
// (signed bytes re-biased by 0x80, which keeps every difference).
template <int KIND>
__device__ __forceinline__ double fps_dist(const FpsArgs& a, int64_t p, const uint2* __restrict__ l,
                                           int32_t lnorm) {
  const uint2* x = a.rows + p * (int64_t)a.nu;
  if constexpr (KIND == K_L2F || KIND == K_L1F) {
    double s = 0.0;
    for (int u = 0; u < a.nue; ++u) {
      const uint2 w = __ldg(x + u), v = l[u];
      const double t0 = __dsub_rn((double)__uint_as_float(w.x), (double)__uint_as_float(v.x));
      const double t1 = __dsub_rn((double)__uint_as_float(w.y), (double)__uint_as_float(v.y));
      if constexpr (KIND == K_L2F) {
        s = __dadd_rn(s, __dmul_rn(t0, t0));
        s = __dadd_rn(s, __dmul_rn(t1, t1));
      } else {
        s = __dadd_rn(s, fabs(t0));
        s = __dadd_rn(s, fabs(t1));
      }
    }
    return s;
  } else if constexpr (KIND == K_COSF) {
    double dot = 0.0, xx = 0.0, yy = 0.0;
    for (int u = 0; u < a.nue; ++u) {
      const uint2 w = __ldg(x + u), v = l[u];
      const double u0 = (double)__uint_as_float(w.x), v0 = (double)__uint_as_float(v.x);
      const double u1 = (double)__uint_as_float(w.y), v1 = (double)__uint_as_float(v.y);
      dot = __dadd_rn(dot, __dmul_rn(u0, v0));
      xx = __dadd_rn(xx, __dmul_rn(u0, u0));
      yy = __dadd_rn(yy, __dmul_rn(v0, v0));
      dot = __dadd_rn(dot, __dmul_rn(u1, v1));
      xx = __dadd_rn(xx, __dmul_rn(u1, u1));
      yy = __dadd_rn(yy, __dmul_rn(v1, v1));
    }
    if (xx == 0.0 && yy == 0.0) return 0.0;
    if (xx == 0.0 || yy == 0.0) return 1.0;
    return __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(xx), __dsqrt_rn(yy))));
  } else if constexpr (KIND == K_L2I) {
    int dot = 0;
    for (int u = 0; u < a.nue; ++u) {
      const uint2 w = __ldg(x + u), v = l[u];
      dot = __dp4a((int)w.x, (int)v.x, dot);
      dot = __dp4a((int)w.y, (int)v.y, dot);
    }
    return (double)((int64_t)__ldg(a.inorm + p) + lnorm - 2 * (int64_t)dot);
  } else {
    unsigned s = 0u;
    for (int u = 0; u < a.nue; ++u) {
      const uint2 w = __ldg(x + u), v = l[u];
      s += __vsadu4(w.x ^ 0x80808080u, v.x ^ 0x80808080u);
      s += __vsadu4(w.y ^ 0x80808080u, v.y ^ 0x80808080u);
    }
    return (double)s;
  }
}

// (value, index) order of the argmax: larger value first, then lower index
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

constexpr int FPS_NT = 256;
constexpr int FPS_MAX_CAND = 1024;   // grid size bound

// PPT > 0: each thread owns points gt + k * gs (k < PPT) with their running
// minimum in registers; PPT == 0: any n, running minimum in a.mind.
__device__ __forceinline__ double warp_sum_d(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_max_d(double x) {
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// CL: the whole grid is one thread-block cluster (small n): candidates are
// exchanged through distributed shared memory and the per-landmark barrier is
// the cluster barrier instead of a grid-wide one.
template <int KIND, int PPT, bool CL>
__global__ void __launch_bounds__(FPS_NT) k_fps(FpsArgs a) {
  extern __shared__ uint2 slm[];   // the current landmark's units
  __shared__ double sv[FPS_NT / 32];
  __shared__ int64_t si[FPS_NT / 32];
  __shared__ int64_t s_next;
  __shared__ double ccv[2];    // CL: this CTA's candidate per buffer
  __shared__ int64_t cci[2];
  // pruning (a.perm): the bounding ball of each warp's points (centre, radius)
  constexpr bool FLT = KIND == K_L2F || KIND == K_L1F;
  __shared__ double scen[FLT ? FPS_NT / 32 : 1][FLT ? 128 : 1];
  __shared__ double srad[FPS_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t gt = (int64_t)blockIdx.x * FPS_NT + tid, gs = (int64_t)gridDim.x * FPS_NT;
  double mr[PPT > 0 ? PPT : 1];
  int32_t pidx[PPT > 0 ? PPT : 1];   // owned points (original indices; >= n: none)
#pragma unroll
  for (int k = 0; k < (PPT > 0 ? PPT : 1); ++k) mr[k] = INFINITY;
  const bool prune = FLT && PPT > 0 && a.perm != nullptr && a.d <= 128;
  if constexpr (PPT > 0) {
    // this warp's run of the spatial order: neighbouring runs go to different
    // CTAs (run = warp * grid + CTA), so the few warps near a landmark — the
    // ones that cannot skip it — are spread over the SMs instead of sharing one
    const int64_t wbase = ((int64_t)w * gridDim.x + blockIdx.x) * 32 * PPT;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (prune) {
        const int64_t r = wbase + lane + 32 * k;
        pidx[k] = r < a.n ? __ldg(a.perm + r) : (int32_t)a.n;
      } else {
        const int64_t p = gt + k * gs;
        pidx[k] = p < a.n ? (int32_t)p : (int32_t)a.n;
      }
    }
    if (prune) {
      // centre: mean of the warp's points; radius: max distance, fp64, rounded up
      double cnt = 0.0;
#pragma unroll
      for (int k = 0; k < PPT; ++k) cnt += pidx[k] < a.n ? 1.0 : 0.0;
      cnt = warp_sum_d(cnt);
      for (int j = 0; j < a.d; ++j) {
        double sj = 0.0;
#pragma unroll
        for (int k = 0; k < PPT; ++k)
          if (pidx[k] < a.n)
            sj += (double)reinterpret_cast<const float*>(a.rows + pidx[k] * (int64_t)a.nu)[j];
        sj = warp_sum_d(sj);
        if (lane == 0) scen[w][j] = cnt > 0.0 ? sj / cnt : 0.0;
      }
      __syncwarp();
      double rmax = 0.0;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        if (pidx[k] >= a.n) continue;
        const float* x = reinterpret_cast<const float*>(a.rows + pidx[k] * (int64_t)a.nu);
        double t2 = 0.0;
        for (int j = 0; j < a.d; ++j) {
          const double t = (double)x[j] - scen[w][j];
          t2 += KIND == K_L2F ? t * t : fabs(t);
        }
        rmax = fmax(rmax, KIND == K_L2F ? sqrt(t2) : t2);
      }
      rmax = warp_max_d(rmax);
      if (lane == 0) srad[w] = rmax * (1.0 + 1e-12) + 1e-300;
      __syncwarp();
    }
  }
  double bv = -INFINITY;   // this lane's (max running minimum, index): kept while skipped
  int64_t bi = a.n;
  int64_t cur = a.start;
  int64_t L = 0;
  for (int step = 0;; ++step) {
    if (blockIdx.x == 0 && tid == 0) a.seq[L] = (int32_t)cur;
    ++L;
    const uint2* lrow = a.rows + cur * (int64_t)a.nu;
    for (int u = tid; u < a.nue; u += FPS_NT) slm[u] = lrow[u];
    const int32_t lnorm = KIND == K_L2I ? __ldg(a.inorm + cur) : 0;
    __syncthreads();
    if constexpr (PPT > 0) {
      // pruning: d(p, l) >= |l - c| - r for every p of the warp; if that bound
      // is at least the warp's largest running minimum no minimum can change
      // (margins cover the fp64 rounding of the centre, the radius and the
      // oracle-formula distance, all relative 1e-13 or less), so the warp
      // keeps its minima and its argmax candidate
      bool skip = false;
      if (prune && step > 0) {
        const float* lf = reinterpret_cast<const float*>(slm);
        double part = 0.0;
        for (int j = lane; j < a.d; j += 32) {
          const double t = (double)lf[j] - scen[w][j];
          part += KIND == K_L2F ? t * t : fabs(t);
        }
        double dc = warp_sum_d(part);
        if (KIND == K_L2F) dc = sqrt(dc);
        const double lb = dc * (1.0 - 1e-12) - srad[w] * (1.0 + 1e-12);
        const double mx = warp_max_d(bv);
        skip = lb > 0.0 && (KIND == K_L2F ? lb * lb * (1.0 - 1e-12) >= mx : lb * (1.0 - 1e-12) >= mx);
        if (a.dbg && lane == 0) {
          atomicAdd(&a.dbg[0], 1ull);
          if (skip) atomicAdd(&a.dbg[1], 1ull);
        }
      }
      if (!skip) {
        bv = -INFINITY;
        bi = a.n;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const int64_t p = pidx[k];
          if (p < a.n) {
            const double v = fps_dist<KIND>(a, p, slm, lnorm);
            if (v < mr[k]) mr[k] = v;
            if (better(mr[k], p, bv, bi)) {
              bv = mr[k];
              bi = p;
            }
          }
        }
      }
    } else {
      bv = -INFINITY;
      bi = a.n;
      for (int64_t p = gt; p < a.n; p += gs) {
        const double v = fps_dist<KIND>(a, p, slm, lnorm);
        const double m = step == 0 ? v : fmin(a.mind[p], v);
        a.mind[p] = m;
        if (better(m, p, bv, bi)) {
          bv = m;
          bi = p;
        }
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
#pragma unroll
      for (int k = 1; k < FPS_NT / 32; ++k)
        if (better(sv[k], si[k], v, i)) {
          v = sv[k];
          i = si[k];
        }
      if constexpr (CL) {
        ccv[buf] = v;
        cci[buf] = i;
      } else {
        a.cval[buf * gridDim.x + blockIdx.x] = v;
        a.cidx[buf * gridDim.x + blockIdx.x] = i;
      }
    }
    if constexpr (CL) cg::this_cluster().sync();
    else cg::this_grid().sync();
    // every CTA reduces all candidates the same way (loads issued before the compares)
    if (w == 0 && CL) {
      cg::cluster_group cl = cg::this_cluster();
      double v = -INFINITY;
      int64_t i = a.n;
      if (lane < (int)gridDim.x) {
        v = *cl.map_shared_rank(&ccv[buf], (unsigned)lane);
        i = *cl.map_shared_rank(&cci[buf], (unsigned)lane);
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
    } else if (w == 0) {
      double v = -INFINITY;
      int64_t i = a.n;
      for (int base = 0; base < (int)gridDim.x; base += 256) {
        double cv[8];
        int64_t ci[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int k = base + lane + 32 * r;
          const bool ok = k < (int)gridDim.x;
          cv[r] = ok ? __ldcg(a.cval + buf * gridDim.x + k) : -INFINITY;
          ci[r] = ok ? __ldcg(a.cidx + buf * gridDim.x + k) : a.n;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (better(cv[r], ci[r], v, i)) {
            v = cv[r];
            i = ci[r];
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
  }
  // CL: no CTA leaves while another may still read its candidates
  if constexpr (CL) cg::this_cluster().sync();
  if (blockIdx.x == 0 && tid == 0) *a.L_out = (int32_t)L;
}

template <int KIND, int PPT>
static cudaError_t fps_go(const FpsArgs& a0, int grid, cudaStream_t s) {
  FpsArgs a = a0;
  void* args[] = {&a};
  const size_t smem = (size_t)a.nue * sizeof(uint2);
  return cudaLaunchCooperativeKernel((void*)k_fps<KIND, PPT, false>, dim3(grid), dim3(FPS_NT),
                                     args, smem, s);
}

// one cluster of FPS_CL CTAs (non-portable size 16): small problems
constexpr int FPS_CL = 16;
template <int KIND, int PPT>
static cudaError_t fps_go_cluster(const FpsArgs& a, cudaStream_t s) {
  auto kern = k_fps<KIND, PPT, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(FPS_CL);
  cfg.blockDim = dim3(FPS_NT);
  cfg.dynamicSmemBytes = (size_t)a.nue * sizeof(uint2);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = FPS_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// Grid: CTAs co-resident for every instance of the kind (cooperative launch),
// at most FPS_MAX_CAND, and no more than one CTA per 256 points (a small
// problem pays a smaller barrier).
// co-resident CTAs of one instance (cooperative launch), capped at
// FPS_MAX_CAND and at one CTA per 256 points (a small problem pays a smaller
// barrier)
template <int KIND, int PPT>
static int fps_grid_of(int64_t n, int nue) {
  int dev = 0, sms = 0, q = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_fps<KIND, PPT, false>, FPS_NT,
                                                (size_t)nue * sizeof(uint2));
  int64_t g = (int64_t)sms * (q > 0 ? q : 1);
  if (g > FPS_MAX_CAND) g = FPS_MAX_CAND;
  const int64_t want = (n + FPS_NT - 1) / FPS_NT;
  if (g > want) g = want;
  return (int)(g > 0 ? g : 1);
}

// the smallest register-resident PPT whose own grid covers n; else global minima
template <int KIND, int PPT>
static cudaError_t fps_try(const FpsArgs& a, cudaStream_t s, bool* done) {
  const int g = fps_grid_of<KIND, PPT>(a.n, a.nue);
  if ((int64_t)g * FPS_NT * PPT < a.n) return cudaSuccess;
  *done = true;
  return fps_go<KIND, PPT>(a, g, s);
}

template <int KIND>
static cudaError_t fps_kind(const FpsArgs& a, cudaStream_t s) {
  // small problems: one cluster, register-resident minima (the cluster barrier
  // costs a fraction of a grid barrier); falls through when it cannot launch
  static const bool no_cl = getenv("BM_FPS_NO_CLUSTER") != nullptr;   // diagnostics
  const int64_t cl_cap = (int64_t)FPS_CL * FPS_NT;
  // (measured: C1, n = 2000, 3.35 -> 2.36 us per landmark; at C2's n = 1e5
  // the 16 SMs are too few — 22 vs 5.6 us — so only up to 4 points per thread)
  if (!no_cl && a.n <= cl_cap * 4) {
    const cudaError_t e = fps_go_cluster<KIND, 4>(a, s);
    if (e == cudaSuccess) return e;
    cudaGetLastError();   // no cluster of this size: the cooperative path below
  }
  bool done = false;
  cudaError_t e = fps_try<KIND, 1>(a, s, &done);
  if (!done && e == cudaSuccess) e = fps_try<KIND, 2>(a, s, &done);
  if (!done && e == cudaSuccess) e = fps_try<KIND, 4>(a, s, &done);
  if (!done && e == cudaSuccess) e = fps_try<KIND, 8>(a, s, &done);
  if (!done && e == cudaSuccess) e = fps_try<KIND, 16>(a, s, &done);
  if (!done && e == cudaSuccess) e = fps_try<KIND, 32>(a, s, &done);
  if (!done && e == cudaSuccess) return fps_go<KIND, 0>(a, fps_grid_of<KIND, 0>(a.n, a.nue), s);
  return e;
}

cudaError_t launch_fps(const uint2* rows, const int32_t* inorm, int nu, int d, int kind, int64_t n,
                       double thr, int64_t start, double* mind, int32_t* seq, int32_t* L_out,
                       double* cval, int64_t* cidx, const int32_t* perm, cudaStream_t s) {
  const int nue = (kind == K_L2I || kind == K_L1I) ? (d + 7) / 8 : (d + 1) / 2;
  static unsigned long long* dbg = nullptr;
  if (getenv("BM_FPS_DEBUG") && !dbg) {
    cudaMallocManaged(&dbg, 16);
  }
  if (dbg) dbg[0] = dbg[1] = 0ull;
  FpsArgs a{rows, inorm, nu, nue, d, n, thr, start, mind, seq, L_out, cval, cidx, perm, dbg};
  switch (kind) {
    case K_L2F: {
      cudaError_t e = fps_kind<K_L2F>(a, s);
      if (dbg) {
        cudaStreamSynchronize(s);
        fprintf(stderr, "fps debug: warp-steps %llu skipped %llu (%.3f)\n", dbg[0], dbg[1],
                dbg[0] ? (double)dbg[1] / dbg[0] : 0.0);
      }
      return e;
    }
    case K_L1F: return fps_kind<K_L1F>(a, s);
    case K_COSF: return fps_kind<K_COSF>(a, s);
    case K_L2I: return fps_kind<K_L2I>(a, s);
    default: return fps_kind<K_L1I>(a, s);
  }
}

int fps_max_candidates() { return FPS_MAX_CAND; }

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

}  // namespace bm
