// pairs_impl.cuh — CUDA-core point x landmark predicate kernel (steps A2, A4, B).
//
// One kernel template serves the two places the method evaluates the ball
// predicate d(x_p, l) < eps (open ball):
//   MODE_ADJ    A2: candidate x candidate bits of the greedy tile (b < a)
//   MODE_MEMBER B (+A4): ball membership of every point in the balls of a
//               block of landmarks (the range queries), emitting
//               packed (point << lbits | landmark position) keys with
//               warp-aggregated atomics and, in the fused greedy, setting
//               covered[p] ("mark all points within eps of x as covered",
//               PAPER.md:104) for every in-ball pair
//
// Layout: each thread keeps R query rows in registers (NU 8-byte units each);
// LC landmark rows at a time are staged in shared memory and read as warp
// broadcasts.  Float kinds are scored in fp32 (direct difference form for L2
// and L1, normalised dot for cosine) and classified against a rigorous band
// (DESIGN.md "Float exactness"): score < lo -> in, score >= hi -> out, else the
// pair is re-decided with the fp64 formula of the oracle (same operation order,
// no FMA contraction), which is bit-identical to the CPU oracle's decision.
// Integer kinds are exact: int32 Gram form via dp4a for L2,
// byte |x-y| via vabsdiffs4 + dp4a for L1.
#pragma once
#include <math.h>

#include "internal.cuh"

namespace bm {

constexpr unsigned FULL = 0xffffffffu;

template <int KIND>
struct KindTraits;
template <> struct KindTraits<K_L2F> { using acc_t = float; static constexpr bool is_float = true; };
template <> struct KindTraits<K_L1F> { using acc_t = float; static constexpr bool is_float = true; };
template <> struct KindTraits<K_COSF> { using acc_t = float; static constexpr bool is_float = true; };
template <> struct KindTraits<K_L2I> { using acc_t = int; static constexpr bool is_float = false; };
template <> struct KindTraits<K_L1I> { using acc_t = int; static constexpr bool is_float = false; };

template <int KIND>
__device__ __forceinline__ void acc_unit(typename KindTraits<KIND>::acc_t& a, uint2 q, uint2 l) {
  if constexpr (KIND == K_L2F) {
    float t0 = __uint_as_float(q.x) - __uint_as_float(l.x);
    float t1 = __uint_as_float(q.y) - __uint_as_float(l.y);
    a = fmaf(t0, t0, a);
    a = fmaf(t1, t1, a);
  } else if constexpr (KIND == K_L1F) {
    a += fabsf(__uint_as_float(q.x) - __uint_as_float(l.x));
    a += fabsf(__uint_as_float(q.y) - __uint_as_float(l.y));
  } else if constexpr (KIND == K_COSF) {
    a = fmaf(__uint_as_float(q.x), __uint_as_float(l.x), a);
    a = fmaf(__uint_as_float(q.y), __uint_as_float(l.y), a);
  } else if constexpr (KIND == K_L2I) {
    a = __dp4a((int)q.x, (int)l.x, a);
    a = __dp4a((int)q.y, (int)l.y, a);
  } else {
    a = (int)__dp4a(__vabsdiffs4(q.x, l.x), 0x01010101u, (unsigned)a);
    a = (int)__dp4a(__vabsdiffs4(q.y, l.y), 0x01010101u, (unsigned)a);
  }
}

// fp64 re-decision, operation-for-operation the oracle's formula
// (oracle/bm_oracle.c oracle_distance; reading A6/A7).
// Returns in-ball; *dist = fp64 distance (Euclidean, not squared, for L2).
template <int KIND>
__device__ __noinline__ bool recheck64(const uint2* __restrict__ xrows, int nu, int d,
                                       double eps, double eps2, int64_t p, int64_t q,
                                       double* dist) {
  const float* x = reinterpret_cast<const float*>(xrows + p * (int64_t)nu);
  const float* y = reinterpret_cast<const float*>(xrows + q * (int64_t)nu);
  // coordinates loaded 16 at a time (one memory latency per 16 dimensions);
  // the fp64 sums still run in ascending coordinate order
  constexpr int G = 16;
  double s = 0.0, xx = 0.0, yy = 0.0;
  for (int j0 = 0; j0 < d; j0 += G) {
    float xa[G], ya[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      xa[i] = j0 + i < d ? __ldg(x + j0 + i) : 0.f;
      ya[i] = j0 + i < d ? __ldg(y + j0 + i) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      if (j0 + i < d) {
        const double a = (double)xa[i], b = (double)ya[i];
        if constexpr (KIND == K_L2F) {
          const double t = __dsub_rn(a, b);
          s = __dadd_rn(s, __dmul_rn(t, t));
        } else if constexpr (KIND == K_L1F) {
          s = __dadd_rn(s, fabs(__dsub_rn(a, b)));
        } else {
          s = __dadd_rn(s, __dmul_rn(a, b));
          xx = __dadd_rn(xx, __dmul_rn(a, a));
          yy = __dadd_rn(yy, __dmul_rn(b, b));
        }
      }
    }
  }
  if constexpr (KIND == K_L2F) {
    *dist = __dsqrt_rn(s);
    return s < eps2;
  } else if constexpr (KIND == K_L1F) {
    *dist = s;
    return s < eps;
  } else {
    double v;
    if (xx == 0.0 && yy == 0.0) v = 0.0;
    else if (xx == 0.0 || yy == 0.0) v = 1.0;
    else v = __dsub_rn(1.0, __ddiv_rn(s, __dmul_rn(__dsqrt_rn(xx), __dsqrt_rn(yy))));
    *dist = v;
    return v < eps;
  }
}

// Classification of a score: 1 = in, 0 = out, 2 = band.
template <int KIND>
__device__ __forceinline__ int classify(typename KindTraits<KIND>::acc_t acc, int32_t nq,
                                        int32_t nl, const Thresh& th) {
  if constexpr (KIND == K_L2I) {
    int s = nq + nl - 2 * acc;
    return s < th.lo_i ? 1 : 0;
  } else if constexpr (KIND == K_L1I) {
    return acc < th.lo_i ? 1 : 0;
  } else {
    float s = (KIND == K_COSF) ? -acc : acc;
    // NaN (cosine zero row) fails both comparisons -> band
    return s < th.lo_f ? 1 : (s >= th.hi_f ? 0 : 2);
  }
}

// NU > 0: query rows live in registers (NU units).  NU == 0 ("wide"): rows of
// any length; the query row is re-read from global/L1 for every landmark.
// NQ > 0 (K_L1F, MODE_MEMBER): the 8-bit quantised rows (NQ words) score a
// sum of absolute differences first; only pairs it cannot prove "out" are
// scored exactly in fp32 (and, in the band, fp64).
// One call = one block of NT*R query rows [blk_q0, ..) against landmarks
// lidx[l0 .. l1) (positions lpos0 + (l - l_begin)).
template <int KIND, int NU, int R, int MODE, int LC, int NQ>
__device__ __forceinline__ void pairs_block(const PairArgs& A, uint2* sl, int32_t* sln,
                                            int32_t* slp, int64_t blk_q0, int64_t q_end,
                                            int64_t l0, int64_t l1, int64_t lpos0) {
  constexpr int NT = 256;
  constexpr bool QF = NQ > 0;
  constexpr int QU = (NU > 0 && !QF) ? NU : 1;   // register units per query row
  using acc_t = typename KindTraits<KIND>::acc_t;
  const int nu = NU > 0 ? NU : A.nu;
  const int tid = threadIdx.x, lane = tid & 31;
  // prefilter: shared memory holds only the quantised landmark rows (the rare
  // exact check reads the landmark's fp32 row from global memory), so a whole
  // 1024-landmark tile is staged at once; otherwise the fp32 rows
  uint32_t* sq = reinterpret_cast<uint32_t*>(sl);
  // bias 2^15 - thr (thr > 2^15: the filter cannot prove anything, bias 0
  // makes every pair a candidate: SADs stay below 2^14 for d <= 64)
  uint32_t qbase = 0u;
  if constexpr (QF) {
    const uint32_t thrq = l1q_threshold(A.qparam, A.th.eps, A.d);
    qbase = thrq <= 0x8000u ? 0x8000u - thrq : 0u;
  }
  uint32_t qq[R][QF ? NQ : 1];

  // ---- query rows into registers
  uint2 q[R][QU];
  int64_t qp[R];
  int64_t qi[R];
  int32_t qn[R];
  bool act[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    qi[r] = blk_q0 + r * NT + tid;
    act[r] = qi[r] < q_end;
    qp[r] = act[r] ? (A.qidx ? (int64_t)A.qidx[qi[r]] : qi[r]) : 0;
    const uint2* src = A.rows + qp[r] * (int64_t)nu;
#pragma unroll
    for (int u = 0; u < QU; ++u)
      q[r][u] = (act[r] && NU > 0 && !QF) ? src[u] : make_uint2(0u, 0u);
    if constexpr (QF) {
#pragma unroll
      for (int w = 0; w < NQ; ++w) qq[r][w] = act[r] ? A.qrows[qp[r] * NQ + w] : 0u;
    }
    qn[r] = (KIND == K_L2I && act[r]) ? A.inorm[qp[r]] : 0;
  }

  uint32_t word[R];
#pragma unroll
  for (int r = 0; r < R; ++r) word[r] = 0u;

  for (int64_t lb = l0; lb < l1; lb += LC) {
    const int nl = (int)min((int64_t)LC, l1 - lb);
    __syncthreads();
    for (int t = tid; t < nl * nu && !QF; t += NT) {
      int jj = t / nu, u = t - jj * nu;
      int32_t pt = A.lidx[lb + jj];
      sl[jj * nu + u] = A.rows[(int64_t)pt * nu + u];
    }
    for (int t = tid; t < nl; t += NT) {
      int32_t pt = A.lidx[lb + t];
      slp[t] = pt;
      sln[t] = (KIND == K_L2I) ? A.inorm[pt] : 0;
    }
    if constexpr (QF) {
      // (rows nl .. up to the next multiple of 8 repeat the last landmark, so
      // the group screen below needs no tail clamp; those columns are never
      // classified)
      const int nl8 = (nl + 7) & ~7;
      for (int t = tid; t < nl8 * NQ; t += NT) {
        const int jj = min(t / NQ, nl - 1), w = t % NQ;
        sq[t] = A.qrows[(int64_t)A.lidx[lb + jj] * NQ + w];
      }
    }
    __syncthreads();

    // the prefilter screens UG landmarks at a time (one vote per group)
    constexpr int UG = QF ? 8 : 1;
    for (int jg = 0; jg < nl; jg += UG) {
    uint32_t gsad[UG][R];
    if constexpr (QF) {
      // quantised SAD (4 coordinates per instruction), accumulated on top of
      // 2^15 - thr: bit 15 of the sum is clear iff SAD < thr, so one AND over
      // the group tells whether any pair needs the exact check (cls 3)
      uint32_t all_out = 0xffffffffu;
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        const int jq = jg + u;   // (the staged rows are padded to a multiple of 8)
        uint32_t lq[NQ];
        if constexpr (NQ % 4 == 0) {   // 16-byte shared loads
#pragma unroll
          for (int w = 0; w < NQ; w += 4) {
            const uint4 v4 = *reinterpret_cast<const uint4*>(sq + jq * NQ + w);
            lq[w] = v4.x;
            lq[w + 1] = v4.y;
            lq[w + 2] = v4.z;
            lq[w + 3] = v4.w;
          }
        } else {
#pragma unroll
          for (int w = 0; w < NQ; ++w) lq[w] = sq[jq * NQ + w];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          uint32_t acc = qbase;
#pragma unroll
          for (int w = 0; w < NQ; ++w) acc = vsad4(qq[r][w], lq[w], acc);
          gsad[u][r] = acc;
          all_out &= acc;
        }
      }
      if (__all_sync(FULL, (all_out & 0x8000u) != 0u)) continue;
    }
#pragma unroll
    for (int ug = 0; ug < UG; ++ug) {
      const int jj = jg + ug;
      if (jj >= nl) break;
      int cls[R];
      bool special = false;
      if constexpr (QF) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          cls[r] = (act[r] && (gsad[ug][r] & 0x8000u) == 0u) ? 3 : 0;
          special = special || (cls[r] != 0);
        }
        if (!__any_sync(FULL, special)) continue;
        // exact fp32 score of the candidates (rows from global, landmark from smem)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (cls[r] == 3) {
            acc_t a = 0;
            const uint2* src = A.rows + qp[r] * (int64_t)nu;
            const uint2* lrow = A.rows + (int64_t)slp[jj] * nu;
            for (int u = 0; u < nu; ++u) acc_unit<KIND>(a, __ldg(src + u), __ldg(lrow + u));
            cls[r] = classify<KIND>(a, qn[r], sln[jj], A.th);
          }
        }
      }
      uint2 l[QU];
#pragma unroll
      for (int u = 0; u < QU; ++u)
        l[u] = (NU > 0 && !QF) ? sl[jj * nu + u] : make_uint2(0u, 0u);
#pragma unroll
      for (int r = 0; r < R && !QF; ++r) {
        acc_t a = 0;
        if constexpr (NU > 0) {
#pragma unroll
          for (int u = 0; u < NU; ++u) acc_unit<KIND>(a, q[r][u], l[u]);
        } else {
          const uint2* src = A.rows + qp[r] * (int64_t)nu;
          const uint2* ls = sl + jj * nu;
          for (int u = 0; u < nu; ++u) acc_unit<KIND>(a, __ldg(src + u), ls[u]);
        }
        int c = classify<KIND>(a, qn[r], sln[jj], A.th);
        c = act[r] ? c : 0;
        if (MODE == MODE_ADJ) {
          int64_t b = lb + jj;
          if (b >= qi[r]) c = 0;               // strictly lower triangle
        }
        cls[r] = c;
        if (MODE == MODE_MEMBER) special = special || (c != 0);
        else special = special || (c == 2);
        if (MODE == MODE_ADJ) word[r] |= (c == 1 ? 1u : 0u) << (int)(lb + jj - l0);
      }
      const unsigned ball = __ballot_sync(FULL, special);
      if (ball) {                               // rare, warp-uniform slow path
        const int64_t lpt = slp[jj];
        int nemit = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (KindTraits<KIND>::is_float && cls[r] == 2) {
            double dist;
            bool in = recheck64<KIND>(A.xrows, A.nu, A.d, A.th.eps, A.th.eps2, qp[r], lpt, &dist);
            atomicAdd(&A.stats->band_pairs, 1ull);
            cls[r] = in ? 1 : 0;
            if (MODE == MODE_MEMBER && fabs(dist - A.th.eps) <= A.th.tie_rel * A.th.eps) {
              unsigned long long k = atomicAdd(&A.stats->near_ties, 1ull);
              if ((int64_t)k < A.tie_cap && A.ties) {
                A.ties[3 * k + 0] = qp[r];
                A.ties[3 * k + 1] = lpt;
                A.ties[3 * k + 2] = in ? 1 : 0;
              }
            }
            if (MODE == MODE_ADJ) word[r] |= (in ? 1u : 0u) << (int)(lb + jj - l0);
          }
          if (MODE == MODE_MEMBER) nemit += (cls[r] == 1);
          if (MODE == MODE_MEMBER && A.covered && cls[r] == 1) A.covered[qp[r]] = 1;
        }
        if (MODE == MODE_MEMBER) {
          int incl = nemit;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
          }
          const int wtot = __shfl_sync(FULL, incl, 31);
          unsigned long long base = 0;
          if (wtot > 0) {
            if (lane == 31) base = atomicAdd(&A.stats->key_count, (unsigned long long)wtot);
            base = __shfl_sync(FULL, base, 31);
            unsigned long long k = base + (unsigned long long)(incl - nemit);
            const unsigned long long jpos =
                (unsigned long long)(lpos0 + (lb + jj - A.l_begin));
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (cls[r] == 1) {
                if ((int64_t)k < A.key_cap)
                  A.keys[k] = ((unsigned long long)qp[r] << A.lbits) | jpos;
                ++k;
              }
            }
          }
        }
      }
    }
    }
  }

  if (MODE == MODE_ADJ) {
    const int64_t wcol = l0 / 32;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (act[r]) {
        A.adj[wcol * (int64_t)A.adj_words * 32 + qi[r]] = word[r];   // word-major
        adj_list_push(A.nz, qi[r], wcol, word[r]);
      }
  }
}

// Device-side decomposition of MODE_MEMBER work into (query block, landmark
// chunk) items; the landmark count may live on the device (fused greedy tile).
struct MemberSched {
  int64_t nrb, nch, chunk;
};
__device__ __forceinline__ MemberSched member_sched(int64_t nq, int64_t nl, int rows_per_blk,
                                                    int64_t grid) {
  MemberSched m;
  m.nrb = (nq + rows_per_blk - 1) / rows_per_blk;
  const int64_t n32 = (nl + 31) / 32;
  int64_t merge = (m.nrb * n32 + 8 * grid - 1) / (8 * grid);
  if (merge < 1) merge = 1;
  m.chunk = 32 * merge;
  m.nch = nl > 0 ? (nl + m.chunk - 1) / m.chunk : 0;
  return m;
}

template <int KIND, int NU, int R, int MODE, int LC, int NQ>
__global__ void __launch_bounds__(256) k_pairs(PairArgs A) {
  constexpr int NT = 256;
  extern __shared__ uint2 sl[];          // [LC][nu]
  __shared__ int32_t sln[LC];
  __shared__ int32_t slp[LC];
  pdl_wait();
  pdl_trigger();   // one wave (ADJ) or persistent (MEMBER)
  // device-resident counts act as caps on the host bounds: actual = min(host, *dev)
  int64_t q_end = A.q_end_dev ? min(A.q_end, (int64_t)*A.q_end_dev) : A.q_end;
  int64_t q_begin = A.q_begin_dev ? min(A.q_begin, (int64_t)*A.q_begin_dev) : A.q_begin;
  q_begin = min(q_begin, q_end);
  const int64_t l_end = A.l_end_dev ? min(A.l_end, (int64_t)*A.l_end_dev) : A.l_end;
  if (MODE == MODE_ADJ) {
    const int64_t blk_q0 = q_begin + (int64_t)blockIdx.x * (NT * R);
    const int64_t l0 = A.l_begin + (int64_t)blockIdx.y * 32;
    const int64_t l1 = min(l_end, l0 + 32);
    if (blk_q0 >= q_end || l0 >= l1) return;
    if (l0 >= min(q_end, blk_q0 + NT * R)) return;   // only b < a is needed
    pairs_block<KIND, NU, R, MODE, LC, NQ>(A, sl, sln, slp, blk_q0, q_end, l0, l1, A.lpos0);
  } else {
    const int64_t nl = l_end - A.l_begin;
    const int64_t lpos0 = A.l_total_dev ? (int64_t)*A.l_total_dev - nl : A.lpos0;
    const MemberSched m = member_sched(q_end - q_begin, nl, NT * R, gridDim.x);
    const int64_t items = m.nrb * m.nch;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int64_t rb = it % m.nrb, ch = it / m.nrb;
      const int64_t l0 = A.l_begin + ch * m.chunk;
      const int64_t l1 = min(l_end, l0 + m.chunk);
      pairs_block<KIND, NU, R, MODE, LC, NQ>(A, sl, sln, slp, q_begin + rb * (NT * R), q_end, l0,
                                         l1, lpos0);
      __syncthreads();   // the next item restages the landmark rows
    }
  }
}

template <int KIND, int NU, int MODE, int NQ = 0>
cudaError_t launch_pairs_nu(const PairArgs& a, int64_t q_rows_max, cudaStream_t s) {
  constexpr int R = (MODE == MODE_ADJ || NU == 0) ? 1 : (NU <= 8 ? 4 : (NU <= 16 ? 2 : 1));
  // prefilter: a whole 1024-landmark tile of 8-bit rows per staging round
  constexpr int LC = NQ > 0 ? 1024 : (NU == 0 ? 32 : 64);
  constexpr int NT = 256;
  size_t smem = NQ > 0 ? (size_t)LC * NQ * sizeof(uint32_t) : (size_t)LC * a.nu * sizeof(uint2);
  auto kern = k_pairs<KIND, NU, R, MODE, LC, NQ>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t gx = (q_rows_max + NT * R - 1) / (NT * R);
  if (gx < 1) gx = 1;
  int64_t gy = 1;
  if (MODE == MODE_ADJ) {
    gy = (a.l_end - a.l_begin + 31) / 32;
    if (gy < 1) gy = 1;
  } else {
    // persistent: as many CTAs as fit on the GPU at once (or fewer if there
    // is less work than that); the kernel strides over the work items
    static int per_sm_of[kMaxDevices] = {}, sms_of[kMaxDevices] = {};   // per device
    const int dv = cur_device();
    int& per_sm = per_sm_of[dv];
    int& sms = sms_of[dv];
    if (per_sm == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
      if (per_sm < 1) per_sm = 1;
    }
    const int64_t items = gx * ((a.l_end - a.l_begin + 31) / 32);
    gx = (int64_t)per_sm * sms;
    if (items < gx) gx = items;
    if (gx < 1) gx = 1;
  }
  if (gx > 0x7fffffffLL || gy > 65535) return cudaErrorInvalidConfiguration;
  return launch_pdl(kern, dim3((unsigned)gx, (unsigned)gy), dim3(NT), smem, s, a);
}

template <int KIND, int NU>
cudaError_t launch_pairs_mode(int mode, const PairArgs& a, int64_t q_rows_max, cudaStream_t s) {
  if (mode == MODE_ADJ) return launch_pairs_nu<KIND, NU, MODE_ADJ>(a, q_rows_max, s);
  if constexpr (KIND == K_L1F && NU > 0 && NU <= 32) {
    if (a.qrows) {   // quantised prefilter: NQ = words per 8-bit row (power of two)
      switch (a.nq) {
        case 1: return launch_pairs_nu<KIND, NU, MODE_MEMBER, 1>(a, q_rows_max, s);
        case 2: return launch_pairs_nu<KIND, NU, MODE_MEMBER, 2>(a, q_rows_max, s);
        case 4: return launch_pairs_nu<KIND, NU, MODE_MEMBER, 4>(a, q_rows_max, s);
        case 8: return launch_pairs_nu<KIND, NU, MODE_MEMBER, 8>(a, q_rows_max, s);
        case 16: return launch_pairs_nu<KIND, NU, MODE_MEMBER, 16>(a, q_rows_max, s);
        default: break;
      }
    }
  }
  return launch_pairs_nu<KIND, NU, MODE_MEMBER>(a, q_rows_max, s);
}

// Runtime NU dispatch for one kind (NU must be one of the instantiated widths,
// see pick_nu in internal.cuh; 0 = wide).
template <int KIND>
cudaError_t launch_pairs_kind(int mode, const PairArgs& a, int64_t q_rows_max, cudaStream_t s) {
  switch (a.nu) {
    case 1: return launch_pairs_mode<KIND, 1>(mode, a, q_rows_max, s);
    case 2: return launch_pairs_mode<KIND, 2>(mode, a, q_rows_max, s);
    case 4: return launch_pairs_mode<KIND, 4>(mode, a, q_rows_max, s);
    case 5: return launch_pairs_mode<KIND, 5>(mode, a, q_rows_max, s);
    case 8: return launch_pairs_mode<KIND, 8>(mode, a, q_rows_max, s);
    case 12: return launch_pairs_mode<KIND, 12>(mode, a, q_rows_max, s);
    case 16: return launch_pairs_mode<KIND, 16>(mode, a, q_rows_max, s);
    case 24: return launch_pairs_mode<KIND, 24>(mode, a, q_rows_max, s);
    case 32: return launch_pairs_mode<KIND, 32>(mode, a, q_rows_max, s);
    default: return launch_pairs_mode<KIND, 0>(mode, a, q_rows_max, s);
  }
}

#define BM_INSTANTIATE_PAIRS(KIND)                                                       \
  template cudaError_t launch_pairs_kind<KIND>(int, const PairArgs&, int64_t, cudaStream_t);

}  // namespace bm
