// sort.cu — device-wide exclusive scan and stable LSD radix sort (steps C, D2).
//
// Scan: three phases (tile sums -> one-CTA scan of the sums -> tile scan +
// offset), 4096 elements per tile.
// Radix sort: 8-bit digits, per pass (1) per-tile 256-bin histograms stored
// digit-major, (2) exclusive scan of the histogram matrix, (3) stable scatter
// where each tile is processed in 16 rounds of 256 keys; ranks inside a round
// come from __match_any_sync (peers with the same digit in the warp) plus
// per-warp digit counts in shared memory, so equal keys keep their input
// order (LSD stability).
#include "internal.cuh"

namespace bm {

constexpr unsigned FM = 0xffffffffu;
constexpr int SCAN_NT = 512, SCAN_IPT = 8, SCAN_TILE = SCAN_NT * SCAN_IPT;

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

__global__ void __launch_bounds__(SCAN_NT) k_scan_partial(const int64_t* __restrict__ in,
                                                         int64_t n, int64_t* __restrict__ part) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k)
    if (base + k < n) s += in[base + k];
  int64_t tot;
  block_excl_scan<SCAN_NT>(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_top(int64_t* __restrict__ part, int64_t nb,
                                                   int64_t* __restrict__ total) {
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < nb; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const int64_t v = i < nb ? part[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<1024>(v, &tot);
    if (i < nb) part[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_down(const int64_t* __restrict__ in, int64_t n,
                                                      const int64_t* __restrict__ part,
                                                      int64_t* __restrict__ out) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  int64_t v[SCAN_IPT];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int64_t ex = block_excl_scan<SCAN_NT>(s, nullptr) + part[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
}

size_t scan_temp_bytes(int64_t n) {
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  return (size_t)(nb + 1) * sizeof(int64_t);
}

cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp,
                               int64_t* total_dev, cudaStream_t s, int64_t* launches) {
  if (n <= 0) {
    if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(int64_t), s);
    return cudaSuccess;
  }
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  int64_t* part = (int64_t*)temp;
  k_scan_partial<<<(unsigned)nb, SCAN_NT, 0, s>>>(in, n, part);
  k_scan_top<<<1, 1024, 0, s>>>(part, nb, total_dev);
  k_scan_down<<<(unsigned)nb, SCAN_NT, 0, s>>>(in, n, part, out);
  *launches += 3;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ radix sort
constexpr int RS_NT = 256, RS_ROUNDS = 16, RS_TILE = RS_NT * RS_ROUNDS, RS_BINS = 256;

__global__ void __launch_bounds__(RS_NT) k_rs_hist(const unsigned long long* __restrict__ keys,
                                                  int64_t n, int shift, int bits,
                                                  int64_t* __restrict__ hist, int64_t nblk) {
  __shared__ int h[RS_BINS];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned mask = (1u << bits) - 1u;
  const int64_t t0 = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = t0 + r * RS_NT + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)(keys[i] >> shift) & mask], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_NT) k_rs_scatter(const unsigned long long* __restrict__ in,
                                                     unsigned long long* __restrict__ out,
                                                     int64_t n, int shift, int bits,
                                                     const int64_t* __restrict__ off,
                                                     int64_t nblk) {
  __shared__ int64_t run[RS_BINS];
  __shared__ int wcnt[RS_NT / 32][RS_BINS];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned mask = (1u << bits) - 1u;
  run[tid] = off[(int64_t)tid * nblk + blockIdx.x];
  const int64_t t0 = (int64_t)blockIdx.x * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = t0 + r * RS_NT + tid;
    if (t0 + r * RS_NT >= n) break;  // uniform across the CTA
    const bool valid = i < n;
    const unsigned long long key = valid ? in[i] : 0ull;
    const int dig = valid ? (int)((unsigned)(key >> shift) & mask) : (RS_BINS + lane);
    const unsigned peers = __match_any_sync(FM, dig);
    const int intra = __popc(peers & ((1u << lane) - 1u));
#pragma unroll
    for (int ww = 0; ww < RS_NT / 32; ++ww) wcnt[ww][tid] = 0;
    __syncthreads();
    if (valid && intra == 0) wcnt[w][dig] = __popc(peers);
    __syncthreads();
    if (valid) {
      int64_t rank = run[dig] + intra;
      for (int ww = 0; ww < w; ++ww) rank += wcnt[ww][dig];
      out[rank] = key;
    }
    __syncthreads();
    int add = 0;
#pragma unroll
    for (int ww = 0; ww < RS_NT / 32; ++ww) add += wcnt[ww][tid];
    run[tid] += add;
    __syncthreads();
  }
}

size_t radix_temp_bytes(int64_t n) {
  int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
  if (nblk < 1) nblk = 1;
  size_t hist = (size_t)nblk * RS_BINS * sizeof(int64_t);
  return 2 * hist + scan_temp_bytes(nblk * RS_BINS) + 256;
}

cudaError_t radix_sort_u64(unsigned long long** keys, unsigned long long** alt, int64_t n,
                           int lo_bit, int hi_bit, void* temp, cudaStream_t s,
                           int64_t* launches) {
  if (n <= 1 || hi_bit <= lo_bit) return cudaSuccess;
  int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
  int64_t* hist = (int64_t*)temp;
  int64_t* off = hist + nblk * RS_BINS;
  void* stemp = (void*)(off + nblk * RS_BINS);
  for (int sh = lo_bit; sh < hi_bit; sh += 8) {
    int bits = hi_bit - sh < 8 ? hi_bit - sh : 8;
    k_rs_hist<<<(unsigned)nblk, RS_NT, 0, s>>>(*keys, n, sh, bits, hist, nblk);
    ++*launches;
    cudaError_t e = exclusive_scan_i64(hist, off, nblk * RS_BINS, stemp, nullptr, s, launches);
    if (e != cudaSuccess) return e;
    k_rs_scatter<<<(unsigned)nblk, RS_NT, 0, s>>>(*keys, *alt, n, sh, bits, off, nblk);
    ++*launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    unsigned long long* t = *keys;
    *keys = *alt;
    *alt = t;
  }
  return cudaSuccess;
}

}  // namespace bm
