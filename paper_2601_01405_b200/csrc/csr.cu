// csr.cu — steps C (CSR compaction) and D1/D3 (edge emission, unique).
//
// C : the sorted membership keys (point << lbits | landmark position) give the
//     point-major CSR directly (pt_ptr by segment boundaries, pt_lm = low bits);
//     re-keyed to (landmark << pbits | point) and stably sorted on the landmark
//     bits only they give the landmark-major CSR (ball_ptr, ball_idx) with the
//     points of each ball still ascending.
// D1: every point covered by t balls witnesses the C(t,2) landmark pairs of its
//     (ascending) pt_lm row — Def 2.2's "∩ X ≠ ∅" for 1-simplices
//     (PAPER.md:88-90); keys (i << lbits | j), i < j.
// D3: after the radix sort, adjacent-difference flags + scan + scatter keep one
//     copy of each key -> edges [E][2], lexicographic.
#include "internal.cuh"

namespace bm {

static inline unsigned grid_for(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (unsigned)g;
}

__global__ void k_segment_ptr(const unsigned long long* __restrict__ keys, int64_t m, int shift,
                              unsigned long long mask, int64_t nseg, int64_t* __restrict__ ptr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > m) return;
  int64_t prev = i > 0 ? (int64_t)((keys[i - 1] >> shift) & mask) : -1;
  int64_t cur = i < m ? (int64_t)((keys[i] >> shift) & mask) : nseg;
  for (int64_t s = prev + 1; s <= cur; ++s) ptr[s] = i;
}

cudaError_t launch_segment_ptr(const unsigned long long* keys, int64_t m, int shift,
                               unsigned long long mask, int64_t nseg, int64_t* ptr,
                               cudaStream_t s, int64_t* launches) {
  ++*launches;
  k_segment_ptr<<<grid_for(m + 1, 256), 256, 0, s>>>(keys, m, shift, mask, nseg, ptr);
  return cudaGetLastError();
}

__global__ void k_unpack_low(const unsigned long long* __restrict__ keys, int64_t m,
                             unsigned long long mask, int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = (int32_t)(keys[i] & mask);
}

cudaError_t launch_unpack_low(const unsigned long long* keys, int64_t m, unsigned long long mask,
                              int32_t* out, cudaStream_t s, int64_t* launches) {
  if (m <= 0) return cudaSuccess;
  ++*launches;
  k_unpack_low<<<grid_for(m, 256), 256, 0, s>>>(keys, m, mask, out);
  return cudaGetLastError();
}

__global__ void k_unpack_high(const unsigned long long* __restrict__ keys, int64_t m,
                              int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = (int32_t)(keys[i] >> 32);
}

cudaError_t launch_unpack_high(const unsigned long long* keys, int64_t m, int32_t* out,
                               cudaStream_t s, int64_t* launches) {
  if (m <= 0) return cudaSuccess;
  ++*launches;
  k_unpack_high<<<grid_for(m, 256), 256, 0, s>>>(keys, m, out);
  return cudaGetLastError();
}

__global__ void k_rekey(const unsigned long long* __restrict__ pm, int64_t m, int lbits, int pbits,
                        unsigned long long* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  unsigned long long k = pm[i];
  unsigned long long p = k >> lbits, j = k & ((1ull << lbits) - 1ull);
  out[i] = (j << pbits) | p;
}

cudaError_t launch_rekey_landmark_major(const unsigned long long* pm_keys, int64_t m, int lbits,
                                        int pbits, unsigned long long* out, cudaStream_t s,
                                        int64_t* launches) {
  if (m <= 0) return cudaSuccess;
  ++*launches;
  k_rekey<<<grid_for(m, 256), 256, 0, s>>>(pm_keys, m, lbits, pbits, out);
  return cudaGetLastError();
}

__global__ void k_pair_counts(const int64_t* __restrict__ pt_ptr, int64_t n,
                              int64_t* __restrict__ cnt) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int64_t t = pt_ptr[p + 1] - pt_ptr[p];
  cnt[p] = t * (t - 1) / 2;
}

cudaError_t launch_pair_counts(const int64_t* pt_ptr, int64_t n, int64_t* cnt, cudaStream_t s,
                               int64_t* launches) {
  ++*launches;
  k_pair_counts<<<grid_for(n, 256), 256, 0, s>>>(pt_ptr, n, cnt);
  return cudaGetLastError();
}

// One warp per point: the C(t,2) pairs (a, c), a < c, of the point's row in
// row-major order over the strict upper triangle; the warp walks the rows and
// its lanes stride over the columns of each row (O(1) per pair).
__global__ void k_pair_emit(const int64_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_lm,
                            int64_t n, const int64_t* __restrict__ off, int lbits,
                            unsigned long long* __restrict__ keys) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const int64_t b = pt_ptr[p], t = pt_ptr[p + 1] - b;
  if (t < 2) return;
  int64_t o = off[p];
  for (int64_t a = 0; a + 1 < t; ++a) {
    const unsigned long long hi = (unsigned long long)pt_lm[b + a] << lbits;
    for (int64_t c = a + 1 + lane; c < t; c += 32)
      keys[o + (c - a - 1)] = hi | (unsigned long long)pt_lm[b + c];
    o += t - 1 - a;
  }
}

cudaError_t launch_pair_emit(const int64_t* pt_ptr, const int32_t* pt_lm, int64_t n,
                             const int64_t* off, int lbits, unsigned long long* keys,
                             cudaStream_t s, int64_t* launches) {
  ++*launches;
  k_pair_emit<<<grid_for(n * 32, 256), 256, 0, s>>>(pt_ptr, pt_lm, n, off, lbits, keys);
  return cudaGetLastError();
}

__global__ void k_unique_flags(const unsigned long long* __restrict__ keys, int64_t m,
                               int64_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

cudaError_t launch_unique_flags(const unsigned long long* keys, int64_t m, int64_t* flags,
                                cudaStream_t s, int64_t* launches) {
  if (m <= 0) return cudaSuccess;
  ++*launches;
  k_unique_flags<<<grid_for(m, 256), 256, 0, s>>>(keys, m, flags);
  return cudaGetLastError();
}

__global__ void k_unique_scatter(const unsigned long long* __restrict__ keys, int64_t m,
                                 const int64_t* __restrict__ pos, int lbits,
                                 int32_t* __restrict__ edges) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (i > 0 && keys[i] == keys[i - 1]) return;
  const unsigned long long k = keys[i];
  const int64_t e = pos[i];
  edges[2 * e] = (int32_t)(k >> lbits);
  edges[2 * e + 1] = (int32_t)(k & ((1ull << lbits) - 1ull));
}

cudaError_t launch_unique_scatter(const unsigned long long* keys, int64_t m, const int64_t* pos,
                                  int lbits, int32_t* edges, cudaStream_t s, int64_t* launches) {
  if (m <= 0) return cudaSuccess;
  ++*launches;
  k_unique_scatter<<<grid_for(m, 256), 256, 0, s>>>(keys, m, pos, lbits, edges);
  return cudaGetLastError();
}

__global__ void k_copy_i32(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                           int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

cudaError_t launch_copy_i32(const int32_t* src, int32_t* dst, int64_t n, cudaStream_t s,
                            int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  ++*launches;
  k_copy_i32<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace bm
