// tc.cu — step B on the 5th-gen tensor cores: the Gram-trick membership
// contraction (d^2(q,x) = d^2(q,0) + d^2(x,0) - 2 sum_j q_j x_j,
// with the norms "precomputed and stored").
//
// Structure (one persistent CTA per SM; 12 warps, or 20 for the lean tf32
// membership instances):
//   warp 0      TMA producer: the CTA's resident A block (RA x 128 point rows,
//               all K atoms) once per work unit, then B (landmark) tiles of
//               BN rows one 128-byte K atom per pipeline stage (or, resident
//               B, the launch's whole landmark operand once).
//   warp 1      MMA issuer (one elected thread): tcgen05.mma kind::tf32 (fp32
//               data pre-rounded to tf32) or kind::i8 (exact int32), A and B
//               from 128B-swizzled K-major shared memory, D in TMEM; two TMEM
//               accumulator buffers of RA x BN columns so the epilogue of tile
//               t overlaps the MMAs of tile t+1; tf32 adds one K=8 MMA per
//               tile that folds the per-column constant into the accumulator.
//   warp 2      TMEM allocator.
//   warps 4..   epilogue warpgroups (2, or 4 when lean), each owning a slice of
//               every tile's columns; warp w reads TMEM lanes 32 (w % 4)..:
//               a max over the accumulators against a per-row constant is the
//               "every pair out" test; the rare survivors are classified in /
//               band and staged in shared memory, flushed to global with one
//               atomic per flush.  Lean instances (tf32 membership, unpruned,
//               e.g. C2 / C5 cosine): 32-column loads, the TMEM buffer released
//               before staged keys are flushed and band pairs re-decided.
//   L1T (the L1 thermometer-code contraction): two role
//   warps (producer; MMA issuer that also allocates TMEM) and four epilogue
//   warpgroups (576 threads); the accumulator's sign is the candidate mask,
//   candidates pass an 8-bit SAD bound, survivors get the fp64 decision.
// Float exactness: with x, l rounded to tf32 and fp32
// accumulation, |acc - x.l| <= C (|x|^2 + |l|^2)/2 with a global constant C;
// the per-row/per-column thresholds fold that bound in, so "out" and "in"
// decisions are certain and every other pair is re-decided inline by the
// epilogue lanes with the oracle's fp64 formula (pair_in_fp64, B').
#include <cuda.h>
#include <math.h>

#include "internal.cuh"
#include "tc.cuh"

namespace bm {
namespace tc {

constexpr unsigned FULLM = 0xffffffffu;

// Column constants of landmark j: cb_j =
// round_down(n_l/2 - C2 n_l) folded into the MMA as the exact tf32 split
// -cb = -(hi + mid + lo); d_j = round_up(n_l/2 + C2 n_l - cb_j) for the in-test.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x));
  return __uint_as_float(t);
}
__device__ __forceinline__ void tc_col_consts(double nl, double C2, int64_t j, float* ca,
                                              float* cb, float* colk) {
  const float c = __double2float_rd(0.5 * nl - C2 * nl);
  const float hi = tf32_rna(c);
  const float r1 = c - hi;              // exact
  const float mid = tf32_rna(r1);
  const float lo = r1 - mid;            // exact, <= 3 significant bits
  cb[j] = c;
  ca[j] = __double2float_ru(0.5 * nl + C2 * nl - (double)c);
  float* k = colk + j * 8;
  k[0] = -hi;
  k[1] = -mid;
  k[2] = -lo;
#pragma unroll
  for (int i = 3; i < 8; ++i) k[i] = 0.f;
}
// cosine columns: no constant (acc = cosine); a zero landmark gets acc' = +1e30
// and d_j = +inf, so every pair with it is re-decided by the fp64 zero rule
__device__ __forceinline__ void tc_col_consts_cos(double nl, int64_t j, float* ca, float* cb,
                                                  float* colk) {
  const bool zero = nl == 0.0;
  cb[j] = zero ? -1e30f : 0.f;
  ca[j] = zero ? INFINITY : 0.f;
  float* k = colk + j * 8;
  k[0] = zero ? 1e30f : 0.f;
#pragma unroll
  for (int i = 1; i < 8; ++i) k[i] = 0.f;
}
__device__ __forceinline__ void tc_col_inert(int64_t j, float* ca, float* cb, float* colk) {
  // padding column: acc' = acc - 1e38 never exceeds a row threshold (>= -1e37)
  cb[j] = INFINITY;
  ca[j] = INFINITY;
  float* k = colk + j * 8;
  k[0] = -1e38f;
#pragma unroll
  for (int i = 1; i < 8; ++i) k[i] = 0.f;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// diagnostics (BM_TC_TRACE=2): cycles a role spends in wait k, accumulated per
// thread and summed per CTA into args.wtrace[block][16] (off: wtrace null)
// (compiled in only with -DBM_TC_WTRACE: a diagnostic build, BM_NVCC_EXTRA)
#ifdef BM_TC_WTRACE
#define TC_TWAIT(k, stmt)                      \
  do {                                         \
    if (args.wtrace) {                         \
      const long long _t0 = clock64();         \
      stmt;                                    \
      wacc[k] += clock64() - _t0;              \
    } else {                                   \
      stmt;                                    \
    }                                          \
  } while (0)
#else
#define TC_TWAIT(k, stmt) \
  do {                    \
    stmt;                 \
  } while (0)
#endif
// diagnostics (BM_TC_TRACE=3, diagnostic builds): CTA 0's clock64 at stage k
// of tile i: 0 MMA before its buffer wait, 1 after it, 2 after the commit,
// 3 epilogue warp 4 sees the accumulator, 4 it releases the buffer
#ifdef BM_TC_WTRACE
#define TC_TL(i, k)                                                               \
  do {                                                                            \
    if (args.tline && blockIdx.x == 0 && (i) < 512) args.tline[(i) * 5 + (k)] = clock64(); \
  } while (0)
#else
#define TC_TL(i, k) \
  do {              \
  } while (0)
#endif
// diagnostics: stamp slot k of this CTA (no-op unless a trace buffer is given)
#define TC_STAMP(k) \
  do { \
    if (args.trace) args.trace[blockIdx.x * 16 + (k)] = gtimer(); \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// the same with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing try_wait, so many
// waiting warps do not take issue slots from the working ones
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(su32(b)),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* tm, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tm),
               "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t saddr) {   // shared-space load (no generic path)
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t acc) {
  if constexpr (KIND == TC_TF32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
// Warp-wide forms for the MMA role: the whole warp runs the issue loop
// (convergent, so the descriptors stay in uniform registers) and one elected
// lane issues the instruction (elect.sync inside the asm).
template <int KIND>
__device__ __forceinline__ void mma_w(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                      uint32_t acc) {
  if constexpr (KIND == TC_TF32) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync r|q, 0xffffffff;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync r|q, 0xffffffff;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
__device__ __forceinline__ void commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t.reg .b32 r;\n\telect.sync r|q, 0xffffffff;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          su32(bar))
      : "memory");
}
// 64 consecutive columns of the warp's 32 TMEM lanes in one load
__device__ __forceinline__ void tmem_ld64_nowait(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
        "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
        "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
        "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
        "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait64(uint32_t (&v)[64]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
      : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
        "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
        "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
        "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31]),
        "+r"(v[32]), "+r"(v[33]), "+r"(v[34]), "+r"(v[35]), "+r"(v[36]), "+r"(v[37]), "+r"(v[38]), "+r"(v[39]),
        "+r"(v[40]), "+r"(v[41]), "+r"(v[42]), "+r"(v[43]), "+r"(v[44]), "+r"(v[45]), "+r"(v[46]), "+r"(v[47]),
        "+r"(v[48]), "+r"(v[49]), "+r"(v[50]), "+r"(v[51]), "+r"(v[52]), "+r"(v[53]), "+r"(v[54]), "+r"(v[55]),
        "+r"(v[56]), "+r"(v[57]), "+r"(v[58]), "+r"(v[59]), "+r"(v[60]), "+r"(v[61]), "+r"(v[62]), "+r"(v[63])
      :
      : "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 B apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// Shared-memory matrix descriptor: K-major, 32-byte swizzle (one 8-element
// tf32 K step per row), 8-row groups 256 B apart.
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(256u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)6u << 61;
  return d;
}

template <int KIND>
constexpr uint32_t make_idesc(int M, int N) {
  // c_format [4,6): 1 = F32, 2 = S32; a/b format [7,10)/[10,13): TF32 = 2,
  // u8 = 0, s8 = 1; a/b major bits 15/16 = 0 (K-major); N>>3 at 17; M>>4 at 24.
  return (KIND == TC_TF32 ? (1u << 4) | (2u << 7) | (2u << 10)
                          : (2u << 4) | ((KIND == TC_S8 ? 1u : 0u) << 7) |
                                ((KIND == TC_S8 ? 1u : 0u) << 10)) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// EG: epilogue warpgroups (2, or 4 for the lean tf32 membership instances)
template <int RA, int BN, int KATOMS, int STAGES, int ABUF, bool FOLD, bool BRES = false,
          int MODE = TC_MODE_MEMBER, int EG = 2>
struct Smem {
  static constexpr int A_ATOM = 128 * 128;                 // 128 rows x 128 B
  // ABUF == 0 (K streaming, wide rows): no resident A block; every stage
  // carries the unit's A atom after the tile's B atom
  static constexpr bool KS = ABUF == 0;
  static constexpr int A_BYTES = KS ? 0 : RA * KATOMS * A_ATOM;   // one A buffer
  static constexpr int B_STAGE = BN * 128 + (KS ? A_ATOM : 0);
  static constexpr int B_BYTES = STAGES * B_STAGE;
  static constexpr int EPI_WARPS = 4 * EG;                // epilogue warpgroups x 4
  // staging slots per warp (the same total for 2 or 4 groups)
  // (L1T: every pair is staged as a band pair; in-ball keys are written by
  // the fp64 decision itself, so the key slots go unused)
  static constexpr int KW =
      MODE == TC_MODE_L1T ? 8 : (FOLD ? 64 : (KATOMS > 4 ? 96 : 128)) * 2 / EG;
  static constexpr int BW = MODE == TC_MODE_L1T ? 64 : KW;
  static constexpr int NBUF = 512 / (RA * BN);              // TMEM accumulator buffers
  // fold tiles (tf32): A ones [128 rows x 32 B], B constants [2 slots][BN rows x 32 B]
  static constexpr int AK_OFF = ABUF * A_BYTES + B_BYTES;
  static constexpr int BK_SLOT = BN * 32;
  static constexpr int NBK = BRES ? STAGES : 2;            // fold constant slots
  static constexpr int COL_OFF = AK_OFF + (FOLD ? 128 * 32 + NBK * BK_SLOT : 0);
  static constexpr int COL_BYTES = BN * 4;   // per-buffer column constants: c_j (int8) / d_j (tf32)
  // (tf32 with resident B keeps every d_j of the launch in DJ below instead)
  // (the lean epilogue, EG == 4, reads a candidate's d_j from global memory and
  // needs no slot: no copy may be left in flight when the CTA exits)
  static constexpr bool COLSLOT =
      (MODE == TC_MODE_MEMBER || MODE == TC_MODE_ADJ) && !(FOLD && BRES) && EG != 4;
  static constexpr int BAR_OFF = COL_OFF + (COLSLOT ? NBUF * COL_BYTES : 0);
  static constexpr int NQR = MODE == TC_MODE_L1T ? 4 : 0;   // L1T: unit row-word ring slots
  static constexpr int NBARS = 2 * STAGES + 2 * ABUF + 3 * NBUF + 5 + 2 * NQR;
  static constexpr int CNT_OFF = BAR_OFF + NBARS * 8;     // tmem slot + per-warp counts
  static constexpr int BUF_OFF = CNT_OFF + 256;   // tmem slot + 2 x 16 warp counts
  // resident B (tf32): the launch's in-test offsets d_j, staged once for the rare path
  static constexpr int DJ_OFF = (BUF_OFF + EPI_WARPS * (KW + BW) * 8 + 15) & ~15;
  static constexpr int DJ_BYTES = (BRES && FOLD) ? STAGES * BN * 4 : 0;
  // L1T: the launch's landmark 8-bit rows (<= 1024 columns x 4 words), column order
  static constexpr int Q8_OFF = DJ_OFF + DJ_BYTES;
  static constexpr int Q8_BYTES = MODE == TC_MODE_L1T ? 1024 * 16 : 0;
  // L1T: the 8-bit rows of a unit's 128 points, a ring of NQR slots filled by
  // the producer (one bulk copy per unit) and released by the epilogue warps
  static constexpr int QR_OFF = Q8_OFF + Q8_BYTES;
  static constexpr int QR_SLOT = 128 * 16;
  static constexpr int TOTAL = QR_OFF + NQR * QR_SLOT + 1024;  // + align slack
};

// 32 consecutive columns of the warp's 32 TMEM lanes
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
// 64 consecutive columns of the warp's 32 TMEM lanes, the low 16 bits of two
// adjacent columns packed per register (column 2i in bits 0-15, 2i+1 in 16-31)
__device__ __forceinline__ void tmem_ld64p_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
      : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
        "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
        "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
        "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
      :
      : "memory");
}

// 3-input max (one FMNMX3); inline PTX keeps the caller's reduction tree as
// written (the compiler re-associates fmaxf chains into two long chains)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// max of 32 accumulators: four independent 3-input chains
__device__ __forceinline__ float max32(const uint32_t (&v)[32]) {
  float m[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    m[k] = fmax3(__uint_as_float(v[k]), __uint_as_float(v[4 + k]), __uint_as_float(v[8 + k]));
#pragma unroll
  for (int i = 12; i < 28; i += 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      m[k] = fmax3(m[k], __uint_as_float(v[i + k]), __uint_as_float(v[i + 4 + k]));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) m[k] = fmaxf(m[k], __uint_as_float(v[28 + k]));
  return fmax3(fmax3(m[0], m[1], m[2]), m[3], m[3]);
}

// v[i] for a run-time i in [0, 32) without local memory: a 5-level select tree
__device__ __forceinline__ uint32_t sel32(const uint32_t (&v)[32], int i) {
  uint32_t a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (i & 1) ? v[2 * k + 1] : v[2 * k];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (i & 2) ? a[2 * k + 1] : a[2 * k];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = (i & 4) ? a[2 * k + 1] : a[2 * k];
#pragma unroll
  for (int k = 0; k < 2; ++k) a[k] = (i & 8) ? a[2 * k + 1] : a[2 * k];
  return (i & 16) ? a[1] : a[0];
}

// B': the oracle's fp64 decision for points p, q (ascending coordinates, no
// contraction; cosine with the zero-vector rule, A6/A7).
__device__ __noinline__ bool pair_in_fp64(const float* xrows, int xstride, int dd, int cosine,
                                          double eps, double eps2, int64_t p, int64_t q,
                                          double* dist) {
  const float* x = xrows + p * (int64_t)xstride;
  const float* y = xrows + q * (int64_t)xstride;
  // coordinates are loaded 16 at a time (independent loads in flight together:
  // one memory latency per 16 dimensions instead of one per dimension); the
  // fp64 sums still run in ascending coordinate order
  constexpr int G = 16;
  if (cosine) {
    double dot = 0.0, xx = 0.0, yy = 0.0;
    for (int k0 = 0; k0 < dd; k0 += G) {
      float xa[G], ya[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        xa[i] = k0 + i < dd ? __ldg(x + k0 + i) : 0.f;
        ya[i] = k0 + i < dd ? __ldg(y + k0 + i) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (k0 + i < dd) {
          const double a = (double)xa[i], b = (double)ya[i];
          dot = __dadd_rn(dot, __dmul_rn(a, b));
          xx = __dadd_rn(xx, __dmul_rn(a, a));
          yy = __dadd_rn(yy, __dmul_rn(b, b));
        }
      }
    }
    if (xx == 0.0 && yy == 0.0) *dist = 0.0;
    else if (xx == 0.0 || yy == 0.0) *dist = 1.0;
    else *dist = __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(xx), __dsqrt_rn(yy))));
    return *dist < eps;
  }
  double sacc = 0.0;
  for (int k0 = 0; k0 < dd; k0 += G) {
    float xa[G], ya[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      xa[i] = k0 + i < dd ? __ldg(x + k0 + i) : 0.f;
      ya[i] = k0 + i < dd ? __ldg(y + k0 + i) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      if (k0 + i < dd) {
        const double t = __dsub_rn((double)xa[i], (double)ya[i]);
        sacc = __dadd_rn(sacc, __dmul_rn(t, t));
      }
    }
  }
  *dist = __dsqrt_rn(sacc);
  return sacc < eps2;
}

// B' for L1 (the thermometer path): the oracle's fp64 Manhattan distance,
// sum_j |x_j - y_j| in ascending j (reading A8).  A separate function: one
// more argument on pair_in_fp64's call made the tf32 instances spill.
__device__ __noinline__ bool pair_in_fp64_l1(const float* xrows, int xstride, int dd, double eps,
                                             int64_t p, int64_t q, double* dist) {
  const float* x = xrows + p * (int64_t)xstride;
  const float* y = xrows + q * (int64_t)xstride;
  constexpr int G = 16;
  double sacc = 0.0;
  for (int k0 = 0; k0 < dd; k0 += G) {
    float xa[G], ya[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      xa[i] = k0 + i < dd ? __ldg(x + k0 + i) : 0.f;
      ya[i] = k0 + i < dd ? __ldg(y + k0 + i) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < G; ++i)
      if (k0 + i < dd) sacc = __dadd_rn(sacc, fabs(__dsub_rn((double)xa[i], (double)ya[i])));
  }
  *dist = sacc;
  return sacc < eps;
}

// ------------------------------------------------------------------ kernel
// warps 0-3 roles, 4.. epilogue (two or four warpgroups, tc_groups below)

// BRES (B resident): the launch's whole landmark operand (<= STAGES tiles of
// one K atom) and its fold constants are loaded once per CTA and stay in
// shared memory; only the point blocks stream.  Without it every work unit
// re-reads the same B tiles, and 148 SMs reading the same lines at once is
// bounded by the L2 slices that hold them (measured: C5 cosine, d = 16).
// PR: the launch is pruned (cells.cu; args.act, row_pt, col_pos set) — a
// separate instance, so the unpruned kernels carry none of its code.
// Epilogue warpgroups of an instance: the lean tf32 membership instances (the
// TMEM-read-latency-bound small-d contractions, e.g. C5 cosine at d = 16) run
// four, so that each SM sub-partition has four warps' loads in flight
template <int KIND, int BN, int MODE, bool PR>
constexpr bool tc_lean() {
#ifdef BM_TC_NOLEAN   // A/B diagnostics: every instance on the generic epilogue
  return false;
#else
  return (KIND == TC_TF32 && MODE == TC_MODE_MEMBER && !PR && BN == 256) ||
         (MODE == TC_MODE_L1T && BN == 256);
#endif
}
template <int KIND, int BN, int MODE, bool PR>
// L1T epilogue warpgroups: 4 (64 columns per warp) with two role warps
// (576 threads, 92 registers, no spills): C5 L1 contraction 832 ms; 2 groups
// (128 columns per warp, 137 registers): 891 ms; 4 groups beside four role
// warps (640 threads, 96 registers with spills to a nearly all-shared-memory
// L1): 991 ms (same box each)
#ifndef BM_L1T_EG
#define BM_L1T_EG 4
#endif
constexpr int tc_groups() {
  if (MODE == TC_MODE_L1T) return BM_L1T_EG;   // (2 or 4 groups: 128 or 64 columns per warp)
  return tc_lean<KIND, BN, MODE, PR>() ? 4 : 2;
}
// role warps ahead of the epilogue: warp 0 TMA producer, warp 1 MMA issuer,
// warp 2 TMEM allocator, warp 3 idle; the epilogue warps follow (TMEM lane
// quadrant = warp % 4, so every four consecutive epilogue warps cover the 128
// lanes).  L1T drops the two spare warps (the MMA warp allocates TMEM): with
// four epilogue groups its 576 threads fit 92 registers without spills
// (C5 L1 contraction 891 -> 832 ms against two groups)
template <int MODE>
constexpr int tc_rolew() {
  return MODE == TC_MODE_L1T ? 2 : 4;
}
template <int KIND, int BN, int MODE, bool PR>
constexpr int tc_threads() {
  return 32 * tc_rolew<MODE>() + 128 * tc_groups<KIND, BN, MODE, PR>();
}

template <int KIND, int RA, int BN, int KATOMS, int STAGES, int ABUF, int MODE, bool BRES,
          bool PR>
__global__ void __launch_bounds__(tc_threads<KIND, BN, MODE, PR>(), 1)
    k_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
         const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmO,
         TcArgs args) {
  // tf32: the column constant is folded into the contraction by one extra K=8
  // MMA per tile (ones x {-cb_hi, -cb_mid, -cb_lo}), so the epilogue's test is
  // a plain max over the accumulators
  constexpr bool FOLD = KIND == TC_TF32 && MODE != TC_MODE_GRAM;
  // LEAN (tf32 membership, unpruned, BN = 256): four epilogue groups, each
  // reads its 64 columns of a tile in one load and releases the TMEM buffer
  // before classifying
  constexpr bool LEAN = tc_lean<KIND, BN, MODE, PR>();
  constexpr int EG = tc_groups<KIND, BN, MODE, PR>();
  using S = Smem<RA, BN, KATOMS, STAGES, ABUF, FOLD, BRES, MODE, EG>;
  static_assert(!BRES || KATOMS == 1, "resident B: one K atom per tile");
  constexpr int BUFCOLS = RA * BN;
  constexpr int NBUF = 512 / BUFCOLS;   // TMEM accumulator buffers (2 at BN=256, 4 at BN=128)
  static_assert(NBUF >= 2 && NBUF * BUFCOLS <= 512, "TMEM: accumulator buffers must fit 512 columns");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(RA == 1, "one 128-row block per unit (N = BN MMAs, A double-buffered)");
  static_assert(MODE != TC_MODE_L1T || LEAN, "L1T runs the lean epilogue");
  constexpr int ATOM_ELEMS = KIND == TC_TF32 ? 32 : 128;
  constexpr uint32_t IDESC = make_idesc<KIND>(128, BN);
  constexpr bool KS = S::KS;
  static_assert(!KS || (RA == 1 && !BRES && !PR), "K streaming: plain instances only");
  // K streaming moves only the atoms the rows occupy (KATOMS is the maximum)
  const int n_atoms = KS ? (args.ksteps + 3) / 4 : KATOMS;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                                  // [ABUF][RA][KATOMS] atoms
  uint8_t* sB = sm + ABUF * S::A_BYTES;
  uint64_t* bars = (uint64_t*)(sm + S::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* a_full = bars + 2 * STAGES;             // [ABUF]
  uint64_t* a_empty = a_full + ABUF;                // [ABUF]
  uint64_t* t_full = a_empty + ABUF;                // [NBUF]
  uint64_t* t_empty = t_full + NBUF;                // [NBUF]
  uint64_t* c_full = t_empty + NBUF;                // [NBUF] column constants of TMEM buffer b
  uint64_t* bk_full = c_full + NBUF;                // [2] fold: B constant slots
  uint64_t* bk_empty = bk_full + 2;                 // [2]
  uint64_t* ak_full = bk_empty + 2;                 // fold: A ones tile
  uint64_t* qr_full = ak_full + 1;                  // L1T: [NQR] unit row words landed
  uint64_t* qr_empty = qr_full + S::NQR;            // L1T: [NQR] released by the epilogue
  float* scol = (float*)(sm + S::COL_OFF);          // [NBUF][BN] (int8)
  uint8_t* sAK = sm + S::AK_OFF;                    // fold: [128][32 B]
  uint8_t* sBK = sAK + 128 * 32;                    // fold: [2][BN][32 B]
  uint32_t* tmem_slot = (uint32_t*)(sm + S::CNT_OFF);
  uint32_t* kcount = tmem_slot + 1;                  // [EPI_WARPS]
  uint32_t* bcount = kcount + S::EPI_WARPS;          // [EPI_WARPS]
  unsigned long long* kbuf = (unsigned long long*)(sm + S::BUF_OFF);   // [EPI_WARPS][KW]
  unsigned long long* bbuf = kbuf + S::EPI_WARPS * S::KW;            // [EPI_WARPS][BW]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long wacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // BM_TC_TRACE=2 wait cycles
  // (slot 1 also counts the producer's fold-constant slot waits, 9 the MMA's)
  auto wflush = [&](int k0, int k1) {
    if (!args.wtrace) return;
    for (int k = k0; k < k1; ++k)
      if (wacc[k]) atomicAdd(args.wtrace + blockIdx.x * 16 + k, (unsigned long long)wacc[k]);
  };
  if (threadIdx.x == 0) TC_STAMP(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < ABUF; ++b) {
      mbar_init(&a_full[b], 1);
      mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], S::EPI_WARPS);   // every epilogue warp drains every buffer
      mbar_init(&c_full[b], 1);
    }
    mbar_init(&bk_full[0], 1);
    mbar_init(&bk_full[1], 1);
    mbar_init(&bk_empty[0], 1);
    mbar_init(&bk_empty[1], 1);
    mbar_init(ak_full, 1);
    for (int b = 0; b < S::NQR; ++b) {
      mbar_init(&qr_full[b], 1);
      mbar_init(&qr_empty[b], S::EPI_WARPS);
    }
    for (int w = 0; w < S::EPI_WARPS; ++w) {
      kcount[w] = 0;
      bcount[w] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    if constexpr (FOLD) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
  }
  if (warp == (tc_rolew<MODE>() == 2 ? 1 : 2)) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TC_STAMP(1);
  pdl_wait();   // everything above overlaps the previous kernel's tail
  // one persistent wave: the next kernel may be launched now (its CTAs start as
  // these exit and wait for this grid's completion in their own pdl_wait)
  pdl_trigger();
  if (threadIdx.x == 0) TC_STAMP(2);

  // Work units = (block of RA*128 point rows, chunk of BN-wide landmark tiles),
  // enough units to balance the grid; the column count may live on the device
  // (fused greedy tile), so every role derives the same schedule here.
  const int64_t n_cols =
      args.l_count_dev ? min((int64_t)*args.l_count_dev, args.L) : args.L;
  const int64_t lpos0 = args.l_total_dev ? (int64_t)*args.l_total_dev - n_cols : 0;
  const int64_t n_tiles = (n_cols + BN - 1) / BN;
  // (a single A buffer of wide rows (C4: 112 KB) is reloaded per unit without
  // overlap, so those instances split the columns only below two row blocks per CTA)
  constexpr int64_t UPC = (ABUF == 1 && KATOMS >= 4) ? 2 : 4;   // target units per CTA
  int64_t n_chunks = (UPC * (int64_t)gridDim.x + args.n_mblk - 1) / args.n_mblk;
  n_chunks = max((int64_t)1, min(n_chunks, n_tiles));
  const int64_t tiles_per_chunk = n_tiles > 0 ? (n_tiles + n_chunks - 1) / n_chunks : 1;
  n_chunks = n_tiles > 0 ? (n_tiles + tiles_per_chunk - 1) / tiles_per_chunk : 0;
  const int64_t n_units = args.n_mblk * n_chunks;
  // pruning: may the unit's row block hold an in-ball pair with a landmark of
  // tile t?  The row block's live-chunk bitmap (args.act_words words: byte t =
  // the 8 chunks of tile t) is loaded once per unit, one unit ahead, by every
  // role; every role evaluates the same predicate, so they skip the same tiles.
  constexpr int AWM = PR ? 8 : 1;   // <= 32 tiles of 256 columns (kBigT)
  struct ActW {
    uint32_t m;        // live tiles (bit t: tile t has a live chunk)
    uint32_t w[AWM];   // chunk bytes (loaded by the epilogue only)
  };
  auto tile_bits = [&](const ActW& ab, int64_t t) -> uint32_t {
    if constexpr (!PR) return 0xffu;
    const int i = (int)(t >> 2);
    uint32_t x = ab.w[0];
#pragma unroll
    for (int k = 1; k < AWM; ++k) x = i == k ? ab.w[k] : x;
    return (x >> (8 * (int)(t & 3))) & 0xffu;
  };
  // A2 (adjacency): a tile whose first column is at or after the row block's
  // last row holds no strictly-lower pair and is skipped (its words are
  // never read: the resolve kernels read only words v <= a / 32 of row a)
  auto tile_active = [&](const ActW& ab, int64_t mb, int64_t t) -> bool {
    if constexpr (MODE == TC_MODE_ADJ) return t * BN < (mb + 1) * RA * 128;
    if constexpr (PR) return t < 32 && ((ab.m >> t) & 1u);
    return true;
  };
  // a unit none of whose tiles is live is skipped whole (no A block load)
  auto unit_active_scan = [&](const ActW& ab, int64_t mb, int64_t t0, int64_t t1) -> bool {
    if constexpr (!PR && MODE != TC_MODE_ADJ) return true;
    for (int64_t t = t0; t < t1; ++t)
      if (tile_active(ab, mb, t)) return true;
    return false;
  };
  // Live tiles of a unit as a bit mask (bit t = tile t), so that the roles
  // visit only the live tiles instead of testing every tile of the unit
  // (pruned launches: <= 32 tiles, ~2 live; A2: the lower-triangle tiles).
  const bool use_mask = (PR || MODE == TC_MODE_ADJ) && n_tiles <= 32;
  auto live_tiles = [&](const ActW& ab, int64_t mb, int64_t t0, int64_t t1) -> uint32_t {
    uint32_t m = 0u;
    if constexpr (MODE == TC_MODE_ADJ) {
      const int64_t te = min(t1, ((mb + 1) * RA * 128 + BN - 1) / BN);
      m = te > 0 ? (te >= 32 ? 0xffffffffu : (1u << te) - 1u) : 0u;
    } else if constexpr (PR) {
      m = ab.m;
    }
    const uint32_t lo = t0 >= 32 ? 0u : (0xffffffffu << t0);
    const uint32_t hi = t1 >= 32 ? 0xffffffffu : ((1u << t1) - 1u);
    return m & lo & hi;
  };
  // first live tile after t (or a sentinel past every range)
  auto next_live = [&](uint32_t m, int64_t t) -> int64_t {
    const uint32_t r = t >= 31 ? 0u : (m & ~((2u << t) - 1u));
    return r ? (int64_t)(__ffs(r) - 1) : (int64_t)1 << 40;
  };
  auto first_live = [&](uint32_t m) -> int64_t {
    return m ? (int64_t)(__ffs(m) - 1) : (int64_t)1 << 40;
  };
  auto unit_active = [&](const ActW& ab, int64_t mb, int64_t t0, int64_t t1) -> bool {
    if (use_mask) return live_tiles(ab, mb, t0, t1) != 0u;
    return unit_active_scan(ab, mb, t0, t1);
  };

  // the live-chunk words of unit u
  // the live-tile mask of unit u (act layout per row block: [mask, chunk words])
  const int64_t act_stride = (int64_t)args.act_words + 1;
  auto act_of = [&](int64_t u) -> ActW {
    ActW r;
    r.m = PR ? 0u : 0xffffffffu;
#pragma unroll
    for (int k = 0; k < AWM; ++k) r.w[k] = PR ? 0u : 0xffffffffu;
    if constexpr (PR) {
      if (u < n_units) r.m = __ldg(args.act + (u / n_chunks) * act_stride);
    }
    return r;
  };
  // ... and, for the epilogue, its chunk words too
  auto act_of_full = [&](int64_t u) -> ActW {
    ActW r = act_of(u);
    if constexpr (PR) {
      if (u < n_units) {
        const uint32_t* p = args.act + (u / n_chunks) * act_stride + 1;
#pragma unroll
        for (int k = 0; k < AWM; ++k) r.w[k] = k < args.act_words ? __ldg(p + k) : 0u;
      }
    }
    return r;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0, a_ph = 0;   // a_ph bit b: parity of A buffer b's next release
      uint32_t bk_ph = 0;             // fold: bit b = parity of B constant slot b's release
      int64_t tk = 0;                 // tiles issued by this CTA
      int64_t ui = 0;                 // units issued by this CTA
      if constexpr (FOLD) {
        mbar_expect_tx(ak_full, 128u * 32u);
        tma_load_2d(sAK, &tmO, ak_full, 0, 0);
      }
      if constexpr (BRES) {   // the whole (<= STAGES tiles) landmark operand, once
        if (blockIdx.x < n_units)
          for (int64_t t = 0; t < n_tiles; ++t) {
            mbar_expect_tx(&full[t], (uint32_t)(S::B_STAGE + (FOLD ? S::BK_SLOT : 0)));
            tma_load_2d(sB + t * S::B_STAGE, &tmB, &full[t], 0, (int)(t * BN));
            if constexpr (FOLD)
              tma_load_2d(sBK + t * S::BK_SLOT, &tmK, &full[t], 0, (int)(t * BN));
          }
      }
      ActW act_next = act_of(blockIdx.x);
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int64_t mb = u / n_chunks, ch = u % n_chunks;
        const int64_t t0 = ch * tiles_per_chunk, t1 = min(n_tiles, t0 + tiles_per_chunk);
        const ActW uact = act_next;
        act_next = act_of(u + gridDim.x);
        if (!unit_active(uact, mb, t0, t1)) continue;
        if (ui == 0) TC_STAMP(3);
        if constexpr (!KS) {
          const int ab = (int)(ui % ABUF);
          if (ui >= ABUF) {             // wait until the MMAs of unit ui - ABUF released it
            TC_TWAIT(1, mbar_wait(&a_empty[ab], (a_ph >> ab) & 1u));
            a_ph ^= 1u << ab;
          }
          uint8_t* sAb = sA + ab * S::A_BYTES;
          mbar_expect_tx(&a_full[ab], (uint32_t)S::A_BYTES);
          for (int r = 0; r < RA; ++r)
            for (int ka = 0; ka < KATOMS; ++ka)
              tma_load_2d(sAb + (r * KATOMS + ka) * S::A_ATOM, &tmA, &a_full[ab],
                          ka * ATOM_ELEMS, (int)(mb * RA * 128 + r * 128));
        }
        if constexpr (S::NQR > 0) {   // L1T: the unit's 8-bit rows for the epilogue
          const int qs = (int)(ui % S::NQR);
          if (ui >= S::NQR) mbar_wait(&qr_empty[qs], (uint32_t)((ui / S::NQR - 1) & 1));
          const uint32_t qb = (uint32_t)(128 * args.nq * 4);
          mbar_expect_tx(&qr_full[qs], qb);
          bulk_load(sm + S::QR_OFF + qs * S::QR_SLOT, args.qrows + mb * 128 * args.nq, qb,
                    &qr_full[qs]);
        }
        // warm L2 with the next unit's point block while this one computes
        const int64_t un = u + gridDim.x;
        if (!KS && un < n_units && un / n_chunks != mb) {
          for (int r = 0; r < RA; ++r)
            for (int ka = 0; ka < KATOMS; ++ka)
              tma_prefetch_2d(&tmA, ka * ATOM_ELEMS, (int)((un / n_chunks) * RA * 128 + r * 128));
        }
        const uint32_t lmask = use_mask ? live_tiles(uact, mb, t0, t1) : 0u;
        for (int64_t t = use_mask ? first_live(lmask) : t0; t < t1 && !BRES;
             t = use_mask ? next_live(lmask, t) : t + 1) {
          if (!use_mask && !tile_active(uact, mb, t)) continue;
          for (int ka = 0; ka < n_atoms; ++ka) {
            TC_TWAIT(0, mbar_wait(&empty[stage], phase ^ 1u));
            mbar_expect_tx(&full[stage], (uint32_t)S::B_STAGE);
            tma_load_2d(sB + stage * S::B_STAGE, &tmB, &full[stage], ka * ATOM_ELEMS,
                        (int)(t * BN));
            if constexpr (KS)   // the unit's A atom ka rides in the same stage
              tma_load_2d(sB + stage * S::B_STAGE + BN * 128, &tmA, &full[stage],
                          ka * ATOM_ELEMS, (int)(mb * 128));
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          if constexpr (FOLD) {   // the tile's column constants, two slots
            const int sl = (int)(tk & 1);
            if (tk >= 2) {
              TC_TWAIT(1, mbar_wait(&bk_empty[sl], (bk_ph >> sl) & 1u));
              bk_ph ^= 1u << sl;
            }
            mbar_expect_tx(&bk_full[sl], (uint32_t)S::BK_SLOT);
            tma_load_2d(sBK + sl * S::BK_SLOT, &tmK, &bk_full[sl], 0, (int)(t * BN));
          }
          ++tk;
        }
        ++ui;
      }
      TC_STAMP(4);
      wflush(0, 2);
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer (the whole warp runs the loop; one elected
      // lane issues each tcgen05 instruction)
      int stage = 0;
      uint32_t phase = 0, a_ph = 0;
      uint32_t use[NBUF] = {};
      int buf = 0;
      const int ksteps = args.ksteps;  // 32-byte K steps actually needed
      int64_t ui = 0;
      int64_t tk = 0;                  // tiles issued (fold: B constant slot = tk & 1)
      if constexpr (FOLD) mbar_wait(ak_full, 0u);
      uint32_t res_seen = 0u;   // BRES: resident tiles already waited for
      unsigned long long n_run = 0ull, n_skip = 0ull;
      ActW act_next = act_of(blockIdx.x);
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int64_t mb = u / n_chunks, ch = u % n_chunks;
        const int64_t t0 = ch * tiles_per_chunk, t1 = min(n_tiles, t0 + tiles_per_chunk);
        const ActW uact = act_next;
        act_next = act_of(u + gridDim.x);
        if (!unit_active(uact, mb, t0, t1)) {
          n_skip += t1 - t0;
          continue;
        }
        const int ab = KS ? 0 : (int)(ui % (ABUF > 0 ? ABUF : 1));
        if constexpr (!KS) {
          TC_TWAIT(2, mbar_wait(&a_full[ab], (a_ph >> ab) & 1u));
          a_ph ^= 1u << ab;
          fence_after();
        }
        if (ui == 0 && lane == 0) TC_STAMP(5);
        const uint8_t* sAb = sA + ab * S::A_BYTES;
        const uint32_t lmask = use_mask ? live_tiles(uact, mb, t0, t1) : 0u;
        if (use_mask) n_skip += (t1 - t0) - __popc(lmask);
        for (int64_t t = use_mask ? first_live(lmask) : t0; t < t1;
             t = use_mask ? next_live(lmask, t) : t + 1) {
          if (!use_mask && !tile_active(uact, mb, t)) {
            ++n_skip;
            continue;
          }
          ++n_run;
          if (lane == 0) TC_TL(tk, 0);
          TC_TWAIT(3, mbar_wait(&t_empty[buf], (use[buf] & 1u) ^ 1u));
          if (lane == 0) TC_TL(tk, 1);
          fence_after();
          // int8: the tile's per-column constants c_j into this buffer's slot
          // (tf32 without resident B: the tile's in-test offsets d_j, read by
          // the epilogue's classification, land in the same slot)
          if constexpr (S::COLSLOT) {
            if (lane == 0) {   // one thread of the (convergent) MMA warp
              mbar_expect_tx(&c_full[buf], (uint32_t)S::COL_BYTES);
              bulk_load(scol + buf * BN,
                        FOLD ? (const void*)(args.col_a + t * BN)
                             : (const void*)(args.col_c + t * BN),
                        (uint32_t)S::COL_BYTES, &c_full[buf]);
            }
            __syncwarp();
          }
          const uint32_t dcol = tmem + (uint32_t)(buf * BUFCOLS);
          // the last tile of a ragged column range issues a narrower MMA
          // (N rounded up to 32; the padding columns carry inert constants)
          const int64_t left = n_cols - t * BN;
          const uint32_t nt = left >= BN ? (uint32_t)BN : (uint32_t)((left + 31) / 32 * 32);
          const uint32_t idesc = (IDESC & ~(0x3Fu << 17)) | ((nt >> 3) << 17);
          if constexpr (BRES) {
            if (!((res_seen >> t) & 1u)) {   // first use: the resident tile has landed
              mbar_wait(&full[t], 0u);
              fence_after();
              res_seen |= 1u << t;
            }
            const uint32_t bbase = su32(sB + t * S::B_STAGE);
            const uint32_t abase = su32(sAb);
#ifndef BM_TC_DIAG_NODATA
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              if (ks < ksteps)
                mma_w<KIND>(dcol, sdesc(abase + ks * 32), sdesc(bbase + ks * 32), idesc,
                          ks != 0 ? 1u : 0u);
#endif
#ifndef BM_TC_DIAG_NOFOLD
            if constexpr (FOLD)
              mma_w<KIND>(dcol, sdesc32(su32(sAK)), sdesc32(su32(sBK + t * S::BK_SLOT)), idesc, 1u);
#endif
          }
          for (int ka = 0; ka < n_atoms && !BRES; ++ka) {
            TC_TWAIT(4, mbar_wait(&full[stage], phase));
            fence_after();
            const uint32_t bbase = su32(sB + stage * S::B_STAGE);
#pragma unroll
            for (int r = 0; r < RA; ++r) {
              const uint32_t abase = KS ? bbase + (uint32_t)(BN * 128)
                                        : su32(sAb + (r * KATOMS + ka) * S::A_ATOM);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                if (ka * 4 + ks < ksteps)
                  mma_w<KIND>(dcol + (uint32_t)(r * BN), sdesc(abase + ks * 32),
                            sdesc(bbase + ks * 32), idesc, (ka | ks) != 0 ? 1u : 0u);
              }
            }
            commit_w(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          if constexpr (FOLD && !BRES) {   // acc' = x.l - cb_j: ones x {-cb_hi, -cb_mid, -cb_lo}
            const int sl = (int)(tk & 1);
            TC_TWAIT(9, mbar_wait(&bk_full[sl], (uint32_t)((tk >> 1) & 1)));
            fence_after();
            mma_w<KIND>(dcol, sdesc32(su32(sAK)), sdesc32(su32(sBK + sl * S::BK_SLOT)), idesc, 1u);
            commit_w(&bk_empty[sl]);
          }
          commit_w(&t_full[buf]);
          if (lane == 0) TC_TL(tk, 2);
          ++tk;
          ++use[buf];
          buf = buf + 1 == NBUF ? 0 : buf + 1;
        }
        if constexpr (!KS) commit_w(&a_empty[ab]);
        ++ui;
      }
      if ((MODE == TC_MODE_MEMBER || MODE == TC_MODE_L1T) && args.stats && lane == 0) {
        if (n_run) atomicAdd(&args.stats->tc_tiles_run, n_run);
        if (n_skip) atomicAdd(&args.stats->tc_tiles_skip, n_skip);
      }
      if (lane == 0) {
        TC_STAMP(6);
        wflush(2, 5);
        wflush(9, 10);
      }
    }
  } else if (warp >= tc_rolew<MODE>()) {
    // ---------------- epilogue: warps 4-7 take the first half of every tile's
    // columns, warps 8-11 the second half; warp w reads TMEM lanes 32*(w%4)..
    const int ew = warp - tc_rolew<MODE>(), grp = ew >> 2, q = warp & 3;
    // resident B: the in-test offsets of all the launch's columns in shared memory
    float* sdj = reinterpret_cast<float*>(sm + S::DJ_OFF);
    if constexpr (S::DJ_BYTES > 0) {
      for (int64_t j = threadIdx.x - 32 * tc_rolew<MODE>(); j < n_tiles * BN; j += 128 * EG)
        sdj[j] = __ldg(args.col_a + j);
      asm volatile("bar.sync 1, %0;" ::"n"(128 * EG) : "memory");   // the epilogue warps only
    }
    // L1T: the columns' 8-bit rows (4 words each, zero padded) staged once, so
    // the candidate filter reads shared memory instead of two dependent
    // global loads (launches of <= 1024 columns with <= 4 words per row)
    uint32_t* sq8 = reinterpret_cast<uint32_t*>(sm + S::Q8_OFF);
    // L1T: the 8-bit SAD bound of the CUDA-core path,
    // computed once into shared memory (an fp64 divide: kept out of the loop)
    uint32_t* sthr8 = bcount + S::EPI_WARPS;
    const bool q8s = S::Q8_BYTES > 0;   // (dispatch_l1t: nq == 4, <= 1024 columns)
    if constexpr (S::Q8_BYTES > 0) {
      if (threadIdx.x == 32 * tc_rolew<MODE>()) *sthr8 = l1q_threshold(args.qparam, args.eps, args.d);
      if (q8s) {
        for (int64_t t = threadIdx.x - 32 * tc_rolew<MODE>(); t < n_cols * 4; t += 128 * EG) {
          const int64_t j = t >> 2;
          const int w = (int)(t & 3);
          sq8[t] = w < args.nq ? __ldg(args.qrows + (int64_t)__ldg(args.lm_idx + j) * args.nq + w)
                               : 0u;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(128 * EG) : "memory");   // the epilogue warps only
    }
    unsigned long long* kb = kbuf + ew * S::KW;
    unsigned long long* bb = bbuf + ew * S::BW;
    uint32_t* kc = kcount + ew;
    uint32_t* bc = bcount + ew;
    // flush this warp's staged keys / band pairs to global (warp-collective)
    // B': one band pair (p << 32 | tile column) re-decided with the oracle's
    // fp64 formula (ascending coordinates, no contraction); an in-ball pair
    // becomes a key at once (per-lane, so callable from divergent code)
    // key position of tile column j (sorted columns under pruning)
    auto kpos = [&](int64_t j) -> int64_t {
      if constexpr (PR) return (int64_t)__ldg(args.col_pos + j);
      return j;
    };
    auto recheck = [&](unsigned long long bk) {
      const int64_t p = (int64_t)(bk >> 32), j = (int64_t)(bk & 0xffffffffull);
      if (j >= n_cols || p >= args.n) return;   // padding rows / columns never qualify
      const int64_t qp = args.lm_idx[j];
      double dist;
      bool in;
      if constexpr (MODE == TC_MODE_L1T)
        in = pair_in_fp64_l1(args.xrows, args.xstride, args.d, args.eps, p, qp, &dist);
      else
        in = pair_in_fp64(args.xrows, args.xstride, args.d, args.cosine, args.eps, args.eps2, p,
                          qp, &dist);
      if (fabs(dist - args.eps) <= args.tie_abs) {
        const unsigned long long k = atomicAdd(&args.stats->near_ties, 1ull);
        if ((int64_t)k < args.tie_cap && args.ties) {
          args.ties[3 * k] = p;
          args.ties[3 * k + 1] = qp;
          args.ties[3 * k + 2] = in ? 1 : 0;
        }
      }
      if (in) {
        if (args.covered) args.covered[p] = 1;
        const unsigned long long g = atomicAdd(args.key_count, 1ull);
        if ((int64_t)g < args.key_cap)
          args.keys[g] = ((unsigned long long)p << args.lbits) |
                         (unsigned long long)(lpos0 + kpos(j));
      }
    };
    auto flush = [&](void) {
      __syncwarp();
      const uint32_t kn = min(*kc, (uint32_t)S::KW), bn = min(*bc, (uint32_t)S::BW);
      unsigned long long g0 = 0;
      if (lane == 0) {
        if (kn) g0 = atomicAdd(args.key_count, (unsigned long long)kn);
        if (bn) atomicAdd(&args.stats->band_pairs, (unsigned long long)bn);
      }
      g0 = __shfl_sync(FULLM, g0, 0);
      for (uint32_t i = lane; i < kn; i += 32)
        if ((int64_t)(g0 + i) < args.key_cap) args.keys[g0 + i] = kb[i];
      for (uint32_t i = lane; i < bn; i += 32) recheck(bb[i]);
      __syncwarp();
      if (lane == 0) {
        *kc = 0;
        *bc = 0;
      }
      __syncwarp();
    };
    // append one pair (cls 1: in -> key; cls 2: band -> staged for the
    // recheck); beyond the staging capacity it is handled at once
    auto append = [&](int cls, unsigned long long key) {
      uint32_t* cnt = cls == 1 ? kc : bc;
      unsigned long long* buf_s = cls == 1 ? kb : bb;
      const uint32_t cap = cls == 1 ? S::KW : S::BW;
      const uint32_t k = atomicAdd(cnt, 1u);
      if (k < cap) {
        buf_s[k] = key;
      } else if (cls == 1) {
        const unsigned long long g = atomicAdd(args.key_count, 1ull);
        if ((int64_t)g < args.key_cap) args.keys[g] = key;
      } else {
        atomicAdd(&args.stats->band_pairs, 1ull);
        recheck(key);
      }
    };
    // L1T: 8-bit SAD of this lane's row (w words in registers) against column j
    auto l1t_sad = [&](const uint32_t (&rq)[4], int64_t j) -> uint32_t {
      uint32_t sad = 0u;
      {   // staged rows (nq <= 4: the padding words are zero on both sides)
        uint32_t a, b, c, e;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(e)
                     : "r"(su32(sq8 + j * 4)));
        sad = vsad4(rq[0], a, sad);
        sad = vsad4(rq[1], b, sad);
        sad = vsad4(rq[2], c, sad);
        sad = vsad4(rq[3], e, sad);
      }
      return sad;
    };
    if constexpr (LEAN && MODE == TC_MODE_L1T) {
      // ---- lean L1 epilogue (four groups, group g owns
      // columns [64 g, 64 g + 64) of every tile, warp q TMEM lanes 32 q ..):
      // the sign bits of the folded accumulators (SADq - cut < 0: not proven
      // out) become two 32-bit masks, the TMEM buffer goes back to the MMA
      // issuer, then each candidate passes the 8-bit SAD bound (rows staged in
      // shared memory) and the survivors are decided in fp64 (B')
      constexpr int NP = BN / EG / 64;   // packed 64-column loads per warp and tile
      static_assert(NP * 64 * EG == BN, "L1T: whole 64-column loads per group");
      const long long epi_t0 = args.wtrace ? clock64() : 0;
      uint32_t phase = 0;
      uint32_t tcnt = 0;
      const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(grp * (BN / EG));
      const uint32_t* qr_base = reinterpret_cast<const uint32_t*>(sm + S::QR_OFF);
      const uint32_t th8 = lds32(su32(sthr8));   // (constant per launch)
      const uint32_t kc_a = su32(kc), bc_a = su32(bc), sq8_a = su32(sq8);
      uint32_t uu = 0;   // units seen (the producer's ring order)
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++uu) {
        const int64_t mb = n_chunks == 1 ? u : u / n_chunks, ch = n_chunks == 1 ? 0 : u % n_chunks;
        const int t0 = (int)(ch * tiles_per_chunk), t1 = (int)min(n_tiles, t0 + tiles_per_chunk);
        const int64_t prow = mb * 128 + q * 32 + lane;
        const int qs = (int)(uu % S::NQR);
        // this lane's 8-bit row in the unit's ring slot (read on a candidate)
        const uint32_t* qrow = qr_base + qs * (S::QR_SLOT / 4) + (q * 32 + lane) * args.nq;
        // (every warp waits for the slot's copy before it releases the slot, so
        // the producer never re-arms a barrier whose copy is still in flight;
        // the copy was issued with the unit's A block and has long landed)
        TC_TWAIT(9, mbar_wait(&qr_full[qs], (uu / S::NQR) & 1u));   // (L1T diagnostics: slot 9)
        for (int t = t0; t < t1; ++t) {
          const uint32_t buf = tcnt & (uint32_t)(NBUF - 1);
          TC_TWAIT(5, mbar_wait(&t_full[buf], (phase >> buf) & 1u));
          if (ew == 0 && lane == 0) TC_TL(tcnt, 3);
          phase ^= 1u << buf;
          fence_after();
          const uint32_t ta = tlane + buf * (uint32_t)BUFCOLS;
          // the group's columns in 64-column loads, two 16-bit accumulators per
          // register (|SADq - cut| < 2^15); per 4 columns one byte permute
          // gathers the 4 sign bytes, and 8 of those make a 32-bit mask whose
          // bit 8 i + m is the sign of column 4 m + i
          uint32_t cm[2 * NP];
#ifdef BM_TC_WTRACE
          const long long s6 = clock64();
#endif
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            uint32_t v[32];
            tmem_ld64p_nowait(ta + 64u * p, v);
            tmem_wait32(v);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t m = 0u;
#pragma unroll
              for (int mm = 0; mm < 8; ++mm) {
                const uint32_t r = __byte_perm(v[16 * h + 2 * mm], v[16 * h + 2 * mm + 1], 0x7531);
                m |= (r >> (7 - mm)) & (0x01010101u << mm);
              }
              cm[2 * p + h] = m;
            }
          }
          // (columns past the tile's landmarks and rows past n hold zero
          // operands: acc = 0, never a candidate)
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_empty[buf]);
          if (ew == 0 && lane == 0) TC_TL(tcnt, 4);
#ifdef BM_TC_WTRACE
          const long long s7 = clock64();
          wacc[6] += s7 - s6;   // (L1T diagnostics: slot 6 = TMEM load + masks + release)
#endif
          ++tcnt;
          const int64_t jg = (int64_t)t * BN + grp * (BN / EG);
          if (jg + 64 * NP > n_cols) {   // a ragged last tile: its MMA wrote the first
            // columns only; the rest of the buffer holds an earlier tile's sums
#pragma unroll
            for (int h = 0; h < 2 * NP; ++h)
#pragma unroll
              for (int b = 0; b < 32; ++b)
                if (jg + 32 * h + 4 * (b & 7) + (b >> 3) >= n_cols) cm[h] &= ~(1u << b);
          }
          // candidates (a few per lane and tile): the 8-bit SAD bound, rows
          // staged in shared memory; survivors go to the fp64 decision
          uint32_t anyc = 0u;
#pragma unroll
          for (int h = 0; h < 2 * NP; ++h) anyc |= cm[h];
          if (__any_sync(FULLM, anyc != 0u)) {
            uint32_t rq[4];
            {
              uint32_t a, b2, c, e;
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(a), "=r"(b2), "=r"(c), "=r"(e)
                           : "r"(su32(qrow)));
              rq[0] = a;   // (dispatch_l1t: nq == 4)
              rq[1] = b2;
              rq[2] = c;
              rq[3] = e;
            }
            // (32-bit masks, 32-bit column index, two independent SAD chains:
            // the loop is per-lane and latency-bound)
            const uint32_t jg32 = (uint32_t)jg;
#pragma unroll
            for (int h = 0; h < 2 * NP; ++h) {
              uint32_t cand = cm[h];
              while (cand) {
                const uint32_t b = 31u - (uint32_t)__clz((int)(cand & (0u - cand)));
                cand &= cand - 1u;
                // bit b of mask h -> column
                const uint32_t j = jg32 + 32u * h + 4u * (b & 7u) + (b >> 3);
                uint32_t a0, a1, a2, a3;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                             : "r"(sq8_a + j * 16u));
                const uint32_t sad = vsad4(rq[1], a1, vsad4(rq[0], a0, 0u)) +
                                     vsad4(rq[3], a3, vsad4(rq[2], a2, 0u));
                if (sad < th8)
                  append(2, ((unsigned long long)prow << 32) | (unsigned long long)j);
              }
            }
          }
          __syncwarp();
          if (lds32(kc_a) > S::KW / 2 || lds32(bc_a) > S::BW / 2) flush();
#ifdef BM_TC_WTRACE
          wacc[7] += clock64() - s7;   // (L1T diagnostics: slot 7 = candidates + flush)
#endif
        }
        __syncwarp();   // the unit's row words go back to the producer
        if (lane == 0) mbar_arrive(&qr_empty[qs]);
      }
      if (args.wtrace) wacc[8] += clock64() - epi_t0;
    } else if constexpr (LEAN) {
      // ---- lean tf32 membership epilogue (four groups; group g owns columns
      // [g BN/4, (g + 1) BN/4) of every tile, warp q TMEM lanes 32 q ..).  Per
      // tile: BN/128 32-column loads, a max over the accumulators (the column
      // constant is folded into the MMA, so "every pair is out" is one
      // compare), one vote; only a warp with a candidate re-reads its columns
      // and classifies them.  32-bit state, 32 data registers: the 640-thread
      // CTA stays within 96 registers without spills.
      constexpr int NL = BN / EG / 32;   // 32-column loads per tile and warp
      const long long epi_t0 = args.wtrace ? clock64() : 0;
      uint32_t phase = 0;
      uint32_t tcnt = 0;
      const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(grp * (BN / EG));
      float nlo = 0.f, nhi = 0.f;
      auto lrows = [&](int64_t u) {
        if (u < n_units) {
          const int64_t pr = (u / n_chunks) * 128 + q * 32 + lane;
          nlo = __ldcg(args.row_lo + pr);
          nhi = __ldcg(args.row_hi + pr);
        }
      };
      lrows(blockIdx.x);
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int64_t mb = u / n_chunks, ch = u % n_chunks;
        const int t0 = (int)(ch * tiles_per_chunk), t1 = (int)min(n_tiles, t0 + tiles_per_chunk);
        const int64_t prow = mb * 128 + q * 32 + lane;
        const float rlo = nlo, rhi = nhi;
        lrows(u + gridDim.x);
        for (int t = t0; t < t1; ++t) {
          const uint32_t buf = tcnt & (uint32_t)(NBUF - 1);
          TC_TWAIT(5, mbar_wait(&t_full[buf], (phase >> buf) & 1u));
          if (ew == 0 && lane == 0) TC_TL(tcnt, 3);
          phase ^= 1u << buf;
          fence_after();
          const uint32_t ta = tlane + buf * (uint32_t)BUFCOLS;
          uint32_t v[32];
          float mx;
          TC_TWAIT(6, tmem_ld32_nowait(ta, v); tmem_wait32(v));
          mx = max32(v);
          if constexpr (NL == 2) {
            TC_TWAIT(6, tmem_ld32_nowait(ta + 32u, v); tmem_wait32(v));
            mx = fmaxf(mx, max32(v));
          }
          // (columns past a ragged last tile hold stale values: they only send
          // the warp down the rare path, which classifies columns < n_cols)
#ifdef BM_TC_DIAG   // timing experiments only (results invalid): no rare path
          if (false) {
#else
          if (__any_sync(FULLM, mx > rlo)) {
#endif
            // rare path: re-read the chunks (32 data registers keep the
            // 640-thread CTA spill-free), candidates (not certainly out)
            // become keys (certainly in) or staged band pairs (B')
            for (int k = 0; k < NL; ++k) {
              const int64_t j0 = (int64_t)t * BN + grp * (BN / EG) + k * 32;
              if (j0 >= n_cols) break;
              tmem_ld32_nowait(ta + 32u * k, v);
              tmem_wait32(v);
              uint32_t cand = 0u;
#pragma unroll
              for (int i = 0; i < 32; ++i) cand |= (__uint_as_float(v[i]) > rlo ? 1u : 0u) << i;
              if (prow >= args.n || j0 + 32 > n_cols)   // padding rows / columns never qualify
                cand &= prow >= args.n ? 0u : (uint32_t)((1ull << (n_cols - j0)) - 1ull);
              while (cand) {
                const int i = __ffs(cand) - 1;
                cand &= cand - 1u;
                const int64_t j = j0 + i;
                const float dji = S::DJ_BYTES > 0 ? sdj[j] : __ldg(args.col_a + j);
                if (__uint_as_float(sel32(v, i)) - dji > rhi) {
                  if (args.covered) args.covered[prow] = 1;
                  append(1, ((unsigned long long)prow << args.lbits) |
                                (unsigned long long)(lpos0 + j));
                } else {
                  append(2, ((unsigned long long)prow << 32) | (unsigned long long)j);
                }
              }
            }
          }
          // the buffer goes back to the MMA issuer before any staged keys are
          // written out and band pairs re-decided (global atomics, fp64 rows)
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_empty[buf]);
          if (ew == 0 && lane == 0) TC_TL(tcnt, 4);
          ++tcnt;
          if (*kc > S::KW / 2 || *bc > S::BW / 2) TC_TWAIT(7, flush());
        }
      }
      if (args.wtrace) wacc[8] += clock64() - epi_t0;
    }
    uint32_t phase = 0;   // bit b: parity of the next completion of buffer b
    int64_t tcount = 0;   // tiles seen, in the MMA issuer's order (buffer = tcount % NBUF)
    // row constants of the next unit are loaded one unit ahead
    float nlo[RA], nhi[RA];
    int32_t nint[RA];
    int64_t nppt[RA];   // pruning: original point of each row, loaded one unit ahead
    auto load_rows = [&](int64_t u) {
      if (u >= n_units) return;
      const int64_t mbn = u / n_chunks;
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        const int64_t pr = mbn * RA * 128 + r * 128 + q * 32 + lane;
        if constexpr (PR) nppt[r] = pr < args.n ? (int64_t)__ldg(args.row_pt + pr) : pr;
        if constexpr (KIND == TC_TF32) {
          nlo[r] = __ldcg(args.row_lo + pr);
          nhi[r] = __ldcg(args.row_hi + pr);
        } else {
          nint[r] = __ldcg(args.row_r + pr);
        }
      }
    };
    load_rows(blockIdx.x);
    unsigned long long ck_run = 0ull, ck_skip = 0ull;   // chunks of this warp's rows
    ActW act_next = act_of_full(blockIdx.x);
    const long long epi_t0 = args.wtrace ? clock64() : 0;
    for (int64_t u = LEAN ? n_units : (int64_t)blockIdx.x; u < n_units; u += gridDim.x) {
      const int64_t mb = u / n_chunks, ch = u % n_chunks;
      const ActW uact = act_next;
      act_next = act_of_full(u + gridDim.x);
      const int64_t t0 = ch * tiles_per_chunk, t1 = min(n_tiles, t0 + tiles_per_chunk);
      int64_t prow[RA];
      float rlo[RA], rhi[RA];
      int32_t rint[RA];
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        prow[r] = mb * RA * 128 + r * 128 + q * 32 + lane;   // < n_pad
        if constexpr (KIND == TC_TF32) {
          rlo[r] = nlo[r];
          rhi[r] = nhi[r];
        } else {
          rint[r] = nint[r];
        }
      }
      // pruning: original point of each row (loaded with the row constants)
      int64_t ppt[RA];
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        if constexpr (PR) ppt[r] = nppt[r];
        else ppt[r] = prow[r];
      }
      load_rows(u + gridDim.x);
      const uint32_t lmask = use_mask ? live_tiles(uact, mb, t0, t1) : 0u;
      for (int64_t t = use_mask ? first_live(lmask) : t0; t < t1;
           t = use_mask ? next_live(lmask, t) : t + 1) {
        if (!use_mask && !tile_active(uact, mb, t)) continue;
        // both groups drain every tile: group g takes its half of the columns
        const int buf = (int)(tcount % NBUF);
        const uint32_t ph = (phase >> buf) & 1u;    // parity of buffer buf's next fill
        TC_TWAIT(5, mbar_wait(&t_full[buf], ph));
        if (ew == 0 && lane == 0) TC_TL(tcount, 3);
        if (tcount < 2 && q == 0 && lane == 0) TC_STAMP(7 + grp);
        if constexpr (S::COLSLOT) TC_TWAIT(5, mbar_wait(&c_full[buf], ph));
        phase ^= 1u << buf;
        fence_after();
        const float* colb = scol + buf * BN;   // tile's col_b (tf32) / col_c (int8) in smem
        // TMEM -> registers 32 columns at a time, the next chunk's load in
        // flight while this one is classified (va / vb ping-pong)
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BUFCOLS);
        constexpr int NCH = RA * (BN / 32);
        uint32_t vv[64];   // two chunks per TMEM load
        // chunks the (possibly narrower) MMA of this tile wrote, this group's half
        const int64_t left = n_cols - t * BN;
        const int nch = RA == 1 && left < BN ? (int)((left + 31) / 32) : NCH;
        const int cbeg = grp * (NCH / EG), cend = min(nch, (grp + 1) * (NCH / EG));
        auto caddr = [&](int c) {
          return trow + (uint32_t)((c / (BN / 32)) * BN + (c % (BN / 32)) * 32);
        };
        auto chunk = [&](int c, uint32_t (&v)[32]) {
          const int r = RA == 1 ? 0 : c / (BN / 32), cc = RA == 1 ? c : c % (BN / 32);
          {
            const int64_t j0 = t * BN + cc * 32;
            if constexpr (MODE == TC_MODE_PROBE_LDONLY) {
              uint32_t x = 0u;
#pragma unroll
              for (int i = 0; i < 32; ++i) x ^= v[i];
              if (x == 0x9e3779b9u && prow[r] < 0) args.keys[0] = x;   // keeps the loads live
              return;
            }
            if constexpr (MODE == TC_MODE_GRAM) {
              if (prow[r] < args.n) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (j0 + i < n_cols) args.gram[prow[r] * n_cols + j0 + i] = v[i];
              }
              return;
            }
            if constexpr (MODE == TC_MODE_ADJ) {
              // A2: bit i of word j0/32 of candidate a = [cand j0+i adjacent to a],
              // strictly lower triangle (j < a), rows and columns < nc
              const int64_t a = prow[r];
              const uint32_t tri = j0 >= a ? 0u : (j0 + 32 <= a ? FULLM : ((1u << (a - j0)) - 1u));
              uint32_t mask = 0u;
              if constexpr (KIND == TC_TF32) {
                float dj[32];
                const float4* d4 = reinterpret_cast<const float4*>(colb + cc * 32);   // smem slot
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                  const float4 q4 = d4[i4];
                  dj[4 * i4] = q4.x;
                  dj[4 * i4 + 1] = q4.y;
                  dj[4 * i4 + 2] = q4.z;
                  dj[4 * i4 + 3] = q4.w;
                }
                uint32_t cand = 0u;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const float x = __uint_as_float(v[i]);
                  cand |= (x > rlo[r] ? 1u : 0u) << i;
                  mask |= (x - dj[i] > rhi[r] ? 1u : 0u) << i;
                }
                mask &= tri;
                uint32_t band = cand & ~mask & tri;
                if (a < n_cols) {
                  while (band) {   // B': fp64 decision of the band pairs
                    const int i = __ffs(band) - 1;
                    band &= band - 1u;
                    double dist;
                    if (pair_in_fp64(args.xrows, args.xstride, args.d, args.cosine, args.eps,
                                     args.eps2, args.lm_idx[a], args.lm_idx[j0 + i], &dist))
                      mask |= 1u << i;
                  }
                }
              } else {
                const int4* cc4 = reinterpret_cast<const int4*>(colb + cc * 32);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                  const int4 c = cc4[i4];
                  mask |= (2 * (int)v[4 * i4 + 0] - c.x > rint[r] ? 1u : 0u) << (4 * i4);
                  mask |= (2 * (int)v[4 * i4 + 1] - c.y > rint[r] ? 1u : 0u) << (4 * i4 + 1);
                  mask |= (2 * (int)v[4 * i4 + 2] - c.z > rint[r] ? 1u : 0u) << (4 * i4 + 2);
                  mask |= (2 * (int)v[4 * i4 + 3] - c.w > rint[r] ? 1u : 0u) << (4 * i4 + 3);
                }
                mask &= tri;
              }
              if (a < n_cols) {
                args.adj[(j0 >> 5) * (int64_t)args.adj_T + a] = mask;
                adj_list_push(args.nz, a, j0 >> 5, mask);
              }
              return;
            }
            // fast path: one compare per 32 pairs decides "all out"
            bool surv;
            if constexpr (KIND == TC_TF32) {
              // acc' = x.l - cb_j straight from the MMA: max over 32 columns
              float m[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) m[k] = __uint_as_float(v[k]);
#pragma unroll
              for (int i = 4; i < 32; i += 8) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  m[k] = fmaxf(m[k], fmaxf(__uint_as_float(v[i + 2 * k]),
                                           __uint_as_float(v[i + 2 * k + 1])));
              }
              surv = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])) > rlo[r];
            } else {
              const int4* cc4 = reinterpret_cast<const int4*>(colb + cc * 32);
              int m[4] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN};
#pragma unroll
              for (int i4 = 0; i4 < 8; ++i4) {
                const int4 c = cc4[i4];
                m[0] = max(m[0], 2 * (int)v[4 * i4 + 0] - c.x);
                m[1] = max(m[1], 2 * (int)v[4 * i4 + 1] - c.y);
                m[2] = max(m[2], 2 * (int)v[4 * i4 + 2] - c.z);
                m[3] = max(m[3], 2 * (int)v[4 * i4 + 3] - c.w);
              }
              surv = max(max(m[0], m[1]), max(m[2], m[3])) > rint[r];
            }
            if (__any_sync(FULLM, surv)) {
              // rare path: column masks of candidates (not certainly out) and
              // certain-in pairs, then one append per set bit
              if constexpr (!PR) {
                // unpruned instances: candidate mask only; the certain-in
                // test per candidate column (select tree + one d_j load)
                uint32_t cand = 0u;
                if (surv) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) {
                    if constexpr (KIND == TC_TF32) {
                      cand |= (__uint_as_float(v[i]) > rlo[r] ? 1u : 0u) << i;
                    } else {
                      cand |= (2 * (int)v[i] - __ldg(args.col_c + j0 + i) > rint[r] ? 1u : 0u) << i;
                    }
                  }
                }
                // candidates only (a few per chunk): the certain-in test of
                // column i takes its accumulator by a select tree and its d_j by
                // one load, instead of testing all 32 columns
                while (cand) {
                  const int i = __ffs(cand) - 1;
                  cand &= cand - 1u;
                  const int64_t j = j0 + i;
                  bool in = true;
                  if constexpr (KIND == TC_TF32) {
                    const float dji = S::DJ_BYTES > 0 ? sdj[j] : colb[cc * 32 + i];
                    in = __uint_as_float(sel32(v, i)) - dji > rhi[r];
                  }
                  if (in) {
                    if (args.covered) args.covered[ppt[r]] = 1;
                    append(1, ((unsigned long long)ppt[r] << args.lbits) |
                                  (unsigned long long)(lpos0 + kpos(j)));
                  } else {
                    append(2, ((unsigned long long)ppt[r] << 32) | (unsigned long long)j);
                  }
                }
              } else {
                // pruned instances (sparse survivors): both masks at once
                // (measured: the per-candidate form slowed C3's pruned kernel
                // 71 -> 80 ms)
                uint32_t cand = 0u, inm = 0u;
                float dj[32];   // tf32 in-test offsets of the chunk (warp-uniform loads)
                if constexpr (KIND == TC_TF32) {
                  const float4* d4 = reinterpret_cast<const float4*>(
                      S::DJ_BYTES > 0 ? (const float*)(sdj + j0) : colb + cc * 32);
#pragma unroll
                  for (int i4 = 0; i4 < 8; ++i4) {
                    float4 q4;
                    q4 = d4[i4];   // shared memory (resident d_j or the tile's slot)
                    dj[4 * i4] = q4.x;
                    dj[4 * i4 + 1] = q4.y;
                    dj[4 * i4 + 2] = q4.z;
                    dj[4 * i4 + 3] = q4.w;
                  }
                }
                if (surv) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) {
                    if constexpr (KIND == TC_TF32) {
                      const float a = __uint_as_float(v[i]);
                      cand |= (a > rlo[r] ? 1u : 0u) << i;
                      inm |= (a - dj[i] > rhi[r] ? 1u : 0u) << i;
                    } else {
                      cand |= (2 * (int)v[i] - __ldg(args.col_c + j0 + i) > rint[r] ? 1u : 0u) << i;
                    }
                  }
                  if constexpr (KIND != TC_TF32) inm = cand;
                }
                while (cand) {
                  const int i = __ffs(cand) - 1;
                  cand &= cand - 1u;
                  const int64_t j = j0 + i;
                  if ((inm >> i) & 1u) {
                    if (args.covered) args.covered[ppt[r]] = 1;
                    append(1, ((unsigned long long)ppt[r] << args.lbits) |
                                  (unsigned long long)(lpos0 + kpos(j)));
                  } else {
                    append(2, ((unsigned long long)ppt[r] << 32) | (unsigned long long)j);
                  }
                }
              }
              __syncwarp();
              if (*kc > S::KW / 2 || *bc > S::BW / 2) TC_TWAIT(7, flush());
            }
          }
        };
        if constexpr (MODE != TC_MODE_PROBE_NOLD) {
          // 64 columns per load (a past-the-end half is read and discarded)
#pragma unroll 1
          const uint32_t tb = tile_bits(uact, t);   // this tile's live chunks
          for (int c = cbeg; c < cend; c += 2) {
            if constexpr (PR) {
              const int nck = c + 1 < cend ? 2 : 1;
              if (((tb >> c) & (nck == 2 ? 3u : 1u)) == 0u) {
                ck_skip += nck;
                continue;   // no landmark of these 64 columns can be near this row block
              }
              ck_run += nck;
            }
            TC_TWAIT(6, tmem_ld64_nowait(caddr(c), vv); tmem_wait64(vv));
            chunk(c, *reinterpret_cast<uint32_t(*)[32]>(&vv[0]));
            if (c + 1 < cend) chunk(c + 1, *reinterpret_cast<uint32_t(*)[32]>(&vv[32]));
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[buf]);
        if (ew == 0 && lane == 0) TC_TL(tcount, 4);
        ++tcount;
      }
    }
    if (!LEAN && args.wtrace) wacc[8] += clock64() - epi_t0;
    flush();
    if (q == 0 && lane == 0) TC_STAMP(9 + grp);
    if (lane == 0) wflush(5, 9);
    // every chunk is read by the four warps of its group (32 rows each): count
    // it once, from warp q == 0
    if (MODE == TC_MODE_MEMBER && args.stats && q == 0 && lane == 0) {
      if (ck_run) atomicAdd(&args.stats->tc_chunks_run, ck_run);
      if (ck_skip) atomicAdd(&args.stats->tc_chunks_skip, ck_skip);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) TC_STAMP(11);
  if (warp == (tc_rolew<MODE>() == 2 ? 1 : 2)) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

// ------------------------------------------------------------ host helpers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-D K-major operand [rows][row_bytes], box = (128 bytes of K) x box_rows, 128B swizzle.
static cudaError_t make_tmap(CUtensorMap* tm, const void* base, int kind, int64_t k_elems,
                             int64_t rows, int64_t row_bytes, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const int esz = kind == TC_TF32 ? 4 : 1;
  cuuint64_t dims[2] = {(cuuint64_t)k_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, kind == TC_TF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// fp32 [rows][8] tile map, box 8 x box_rows, 32-byte swizzle (fold operands)
static cudaError_t make_tmap8(CUtensorMap* tm, const void* base, int64_t rows, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {8, (cuuint64_t)rows};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {8, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int KIND, int RA, int BN, int KATOMS, int STAGES, int ABUF, int MODE, bool BRES = false,
          bool PR = false>
static cudaError_t launch_cfg(const TcPlan& P, TcArgs a, cudaStream_t s) {
  constexpr bool FOLD = KIND == TC_TF32 && MODE != TC_MODE_GRAM;
  using S = Smem<RA, BN, KATOMS, STAGES, ABUF, FOLD, BRES, MODE, tc_groups<KIND, BN, MODE, PR>()>;
  static_assert(S::TOTAL <= 232448, "shared memory");
  CUtensorMap tA, tB, tK, tO;
  cudaError_t e = make_tmap(&tA, P.xop, KIND, P.k_elems, P.n_rows, P.row_bytes, 128);
  if (e != cudaSuccess) return e;
  e = make_tmap(&tB, P.lop, KIND, P.k_elems, P.l_rows, P.row_bytes, BN);
  if (e != cudaSuccess) return e;
  if (FOLD) {
    if (!a.colk || !P.ones) return cudaErrorInvalidValue;
    e = make_tmap8(&tK, a.colk, P.l_rows, BN);
    if (e != cudaSuccess) return e;
    e = make_tmap8(&tO, P.ones, 128, 128);
    if (e != cudaSuccess) return e;
  } else {
    tK = tB;
    tO = tB;
  }
  if (PR != (a.act != nullptr)) return cudaErrorInvalidValue;   // instance / arguments agree
  auto kern = k_tc<KIND, RA, BN, KATOMS, STAGES, ABUF, MODE, BRES, PR>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL);
  if (e != cudaSuccess) return e;
  a.n_mblk = (P.n_rows + RA * 128 - 1) / (RA * 128);
  // persistent grid: one CTA per SM (the schedule is derived on the device)
  int64_t grid = P.num_sms;
  if (!a.l_count_dev) {
    const int64_t n_tiles = (a.L + BN - 1) / BN;
    int64_t chunks = (4 * grid + a.n_mblk - 1) / a.n_mblk;
    chunks = chunks < 1 ? 1 : (chunks > n_tiles ? n_tiles : chunks);
    if (a.n_mblk * chunks < grid) grid = a.n_mblk * chunks;
  }
  if (grid < 1) grid = 1;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(tc_threads<KIND, BN, MODE, PR>()),
                    (size_t)S::TOTAL, s, tA, tB,
                    tK, tO, a);
}

// Configuration table: every configuration
// issues M=128 x N=256 MMAs (N=64 MMAs measured ~3x slower per flop on B200);
// a unit = 128 point rows (A, double-buffered when it fits) against a chunk
// of 256-wide landmark tiles streamed one 128-byte K atom per stage.
//   K <= 256 bytes (tf32 d <= 64, int8 d <= 256): 4 stages, 2 A buffers
//   K <= 512 bytes (tf32 d <= 128):               4 stages, 1 A buffer
//   K <= 896 bytes (int8 d <= 896):               3 stages, 1 A buffer
//   K <= 4096 bytes (tf32 d <= 1024, int8 d <= 4096): 4 stages of (B atom + A atom),
//                                                 no resident A block (ABUF = 0)
// resident B applies when every CTA's units share one column chunk (enough
// point blocks: n_chunks = 1 for any column count) and the launch's columns
// fit the stage ring (the fused greedy tile: <= 1024 columns)
static bool bres_ok(const TcPlan& P, const TcArgs& a, int stages, int bn = 256) {
  const int64_t n_mblk = (P.n_rows + 127) / 128;
  return n_mblk >= 4 * (int64_t)P.num_sms && (a.L + bn - 1) / bn <= stages;
}

template <int MODE>
static cudaError_t dispatch(const TcPlan& P, const TcArgs& a, cudaStream_t s) {
  // one-atom rows get their own instance: a wider template would move (and
  // TMA-zero-fill) a second, all-padding K atom for every A block and B tile
  if (P.kind == TC_TF32) {
    // pruned launches (the fused greedy tile, <= 1024 columns: B stays
    // resident for one-atom rows); for two atoms the A stream is the bound, so
    // more A buffers in flight at the cost of one B stage
    if constexpr (MODE == TC_MODE_MEMBER) {
      if (a.act && P.katoms == 1 && a.L <= 4 * 256)
        return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, MODE, true, true>(P, a, s);
      if (a.act && P.katoms == 1)   // big greedy tiles (> 1024 columns): B streams
        return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, MODE, false, true>(P, a, s);
      if (a.act && P.katoms <= 2)
        return launch_cfg<TC_TF32, 1, 256, 2, 3, 3, MODE, false, true>(P, a, s);
      if (a.act) return cudaErrorNotSupported;
    }
    if (P.katoms == 1 && bres_ok(P, a, 4))
      return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, MODE, true>(P, a, s);
    if (P.katoms == 1) return launch_cfg<TC_TF32, 1, 256, 1, 4, 2, MODE>(P, a, s);
    if (P.katoms <= 2) return launch_cfg<TC_TF32, 1, 256, 2, 4, 2, MODE>(P, a, s);
    if (P.katoms <= 4) return launch_cfg<TC_TF32, 1, 256, 4, 4, 1, MODE>(P, a, s);
    // wide rows (the paper's D up to 1000): A atoms stream with the B atoms
    if (P.katoms <= 32) return launch_cfg<TC_TF32, 1, 256, 32, 4, 0, MODE>(P, a, s);
    return cudaErrorNotSupported;
  }
  if (P.kind == TC_U8) {
    if (P.katoms == 1) return launch_cfg<TC_U8, 1, 256, 1, 4, 2, MODE>(P, a, s);
    if (P.katoms <= 2) return launch_cfg<TC_U8, 1, 256, 2, 4, 2, MODE>(P, a, s);
    if (P.katoms <= 7) return launch_cfg<TC_U8, 1, 256, 7, 3, 1, MODE>(P, a, s);
    if (P.katoms <= 32) return launch_cfg<TC_U8, 1, 256, 32, 4, 0, MODE>(P, a, s);
    return cudaErrorNotSupported;
  }
  if (P.katoms == 1) return launch_cfg<TC_S8, 1, 256, 1, 4, 2, MODE>(P, a, s);
  if (P.katoms <= 2) return launch_cfg<TC_S8, 1, 256, 2, 4, 2, MODE>(P, a, s);
  if (P.katoms <= 7) return launch_cfg<TC_S8, 1, 256, 7, 3, 1, MODE>(P, a, s);
  if (P.katoms <= 32) return launch_cfg<TC_S8, 1, 256, 32, 4, 0, MODE>(P, a, s);
  return cudaErrorNotSupported;
}

int tc_bn_for(int kind, int katoms) { return 256; }
int tc_rows_for(int kind, int katoms) { return 128; }
bool tc_supported(int kind, int katoms) {
  return katoms <= 32;   // 4096-byte rows: tf32 d <= 1024, int8 d <= 4096
}

// mode: TC_MODE_MEMBER / TC_MODE_PROBE_LDONLY / TC_MODE_PROBE_NOLD on the
// production configuration for tf32 with K <= 64
template <int BN, int ST, int KA>
static cudaError_t probe_cfg(const TcPlan& P, const TcArgs& a, int mode, cudaStream_t s) {
  if (mode == TC_MODE_PROBE_LDONLY)
    return launch_cfg<TC_TF32, 1, BN, KA, ST, 2, TC_MODE_PROBE_LDONLY>(P, a, s);
  if (mode == TC_MODE_PROBE_NOLD)
    return launch_cfg<TC_TF32, 1, BN, KA, ST, 2, TC_MODE_PROBE_NOLD>(P, a, s);
  return launch_cfg<TC_TF32, 1, BN, KA, ST, 2, TC_MODE_MEMBER>(P, a, s);
}
// mode + 16 * cfg: cfg 0 = N=256 tiles (2 TMEM buffers), cfg 1 = N=128 (4 buffers)
cudaError_t launch_tc_probe(const TcPlan& P, const TcArgs& a, int mode, cudaStream_t s) {
  if (P.kind != TC_TF32 || P.katoms > 2) return cudaErrorNotSupported;
  if (mode & 32) {
    if (P.katoms != 1 || !bres_ok(P, a, 4)) return cudaErrorNotSupported;
    const int m = mode & 15;
    if (m == TC_MODE_PROBE_LDONLY)
      return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, TC_MODE_PROBE_LDONLY, true>(P, a, s);
    if (m == TC_MODE_PROBE_NOLD)
      return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, TC_MODE_PROBE_NOLD, true>(P, a, s);
    return launch_cfg<TC_TF32, 1, 256, 1, 4, 3, TC_MODE_MEMBER, true>(P, a, s);
  }
  if ((mode >> 4) == 1) return probe_cfg<128, 8, 2>(P, a, mode & 15, s);
  if (P.katoms == 1) return probe_cfg<256, 4, 1>(P, a, mode & 15, s);
  return probe_cfg<256, 4, 2>(P, a, mode & 15, s);
}

cudaError_t launch_tc_adj(const TcPlan& Pc, const TcArgs& ac, cudaStream_t s, int64_t* launches) {
  ++*launches;
  return dispatch<TC_MODE_ADJ>(Pc, ac, s);
}

// L1 on tensor cores: signed int8 thermometer operands of one or two K atoms
static cudaError_t dispatch_l1t(const TcPlan& P, const TcArgs& a, cudaStream_t s) {
  if (P.kind != TC_S8 || !a.qrows || !a.qparam || a.nq != 4 || a.L > 1024)
    return cudaErrorInvalidValue;
  if (P.katoms == 1 && bres_ok(P, a, 4))
    return launch_cfg<TC_S8, 1, 256, 1, 4, 3, TC_MODE_L1T, true>(P, a, s);
  if (P.katoms == 1) return launch_cfg<TC_S8, 1, 256, 1, 4, 2, TC_MODE_L1T>(P, a, s);
  if (P.katoms == 2) return launch_cfg<TC_S8, 1, 256, 2, 3, 2, TC_MODE_L1T>(P, a, s);
  if (P.katoms == 3) return launch_cfg<TC_S8, 1, 256, 3, 3, 2, TC_MODE_L1T>(P, a, s);
  return cudaErrorNotSupported;
}

cudaError_t launch_tc(const TcPlan& P, const TcArgs& a, cudaStream_t s, int64_t* launches) {
  ++*launches;
  if (a.l1t) return dispatch_l1t(P, a, s);
  if (a.gram) return dispatch<TC_MODE_GRAM>(P, a, s);
  return dispatch<TC_MODE_MEMBER>(P, a, s);
}

// ------------------------------------------------------------ prep kernels
// Operand rows: fp32 rounded to tf32 (cvt.rna) or raw int8 bytes, K padded
// with zeros to row_bytes; norms in fp64 (float) / int32 (int).
// G lanes per row (a power of two, at most 8), lanes stride over the row
__global__ void k_tc_prep_f32(const float* __restrict__ X, int64_t n, int d, int row_elems,
                              int cosine, int G, float* __restrict__ xop,
                              double* __restrict__ nrm, DevStats* stats) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = gt / G;
  const int lane = (int)(gt % G);
  const bool live = p < n;
  const float* x = X + p * (int64_t)d;
  float* o = xop + p * (int64_t)row_elems;
  double ss = 0.0;
  bool fin = true;
  for (int j = lane; live && j < d; j += G) {
    const float v = x[j];
    fin = fin && isfinite(v);
    ss = __dadd_rn(ss, __dmul_rn((double)v, (double)v));
  }
  for (int k = G / 2; k > 0; k >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, k);
  if (!live) return;
  // cosine: operand x / |x| (fp64 norm), a zero row stays zero
  const double sc = cosine ? (ss > 0.0 ? 1.0 / sqrt(ss) : 0.0) : 1.0;
  for (int j = lane; j < row_elems; j += G) {
    const float v = j < d ? (cosine ? (float)((double)x[j] * sc) : x[j]) : 0.f;
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
    o[j] = __uint_as_float(t);
  }
  if (!fin) atomicExch(&stats->nonfinite, 1);
  if (lane == 0) nrm[p] = ss;
}

__global__ void k_tc_prep_int(const uint8_t* __restrict__ X, int64_t n, int d, int row_bytes,
                              int is_u8, uint8_t* __restrict__ xop, int32_t* __restrict__ nrm) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const uint8_t* x = X + p * (int64_t)d;
  uint8_t* o = xop + p * (int64_t)row_bytes;
  int32_t ss = 0;
  for (int j = lane; j < row_bytes; j += 32) {
    const uint8_t v = j < d ? x[j] : 0;
    o[j] = v;
    const int iv = is_u8 ? (int)v : (int)(int8_t)v;
    ss += iv * iv;
  }
  for (int k = 16; k > 0; k >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, k);
  if (lane == 0) nrm[p] = ss;
}

// per-row constants; rows >= n get +inf / INT_MAX
__global__ void k_tc_rows_f32(const double* __restrict__ nrm, int64_t n, int64_t n_pad, double C2,
                              double eps2, double tau, float* __restrict__ lo,
                              float* __restrict__ hi) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pad) return;
  if (p >= n) {
    lo[p] = INFINITY;
    hi[p] = INFINITY;
    return;
  }
  const double np = nrm[p];
  const double g = 0.5 * (np - eps2);
  lo[p] = __double2float_rd(g - C2 * np - tau);
  hi[p] = __double2float_ru(g + C2 * np + tau);
}

__global__ void k_tc_rows_cos(const double* __restrict__ nrm, int64_t n, int64_t n_pad,
                              double eps, double m, float* __restrict__ lo,
                              float* __restrict__ hi) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pad) return;
  if (p >= n) {
    lo[p] = INFINITY;
    hi[p] = INFINITY;
    return;
  }
  if (nrm[p] == 0.0) {   // zero vector: every live pair to the fp64 zero rule
    lo[p] = -1e37f;       // (padding columns sit at -1e38, below it)
    hi[p] = INFINITY;
    return;
  }
  // out if cos <= 1 - eps - tie - m, in if cos > 1 - eps + tie + m (tie: 1e-6 eps)
  lo[p] = __double2float_rd(1.0 - eps - 1.0000005e-6 * eps - m);
  hi[p] = __double2float_ru(1.0 - eps + 1.0000005e-6 * eps + m);
}

cudaError_t launch_tc_rows_cos(const TcPlan& P, const void* nrm, int64_t n, double eps, double m,
                               TcArgs& a, cudaStream_t s, int64_t* launches) {
  ++*launches;
  const unsigned g = (unsigned)((P.n_pad + 255) / 256);
  k_tc_rows_cos<<<g, 256, 0, s>>>((const double*)nrm, n, P.n_pad, eps, m, (float*)a.row_lo,
                                  (float*)a.row_hi);
  return cudaGetLastError();
}

__global__ void k_tc_rows_int(const int32_t* __restrict__ nrm, int64_t n, int64_t n_pad,
                              int32_t lo_i, int32_t* __restrict__ r) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pad) return;
  // in iff n_p + n_l - 2 acc < lo_i  <=>  2 acc - n_l > n_p - lo_i
  r[p] = p < n ? nrm[p] - lo_i : INT_MAX;
}

// gather landmark operand rows + per-column constants; columns >= L are inert
__global__ void k_tc_gather_lm(const uint8_t* __restrict__ xop, int64_t row_bytes,
                               const int32_t* __restrict__ lm, int64_t L, int64_t l_pad,
                               uint8_t* __restrict__ lop) {
  const int64_t j = blockIdx.x;
  const uint4* src = j < L ? reinterpret_cast<const uint4*>(xop + (int64_t)lm[j] * row_bytes)
                           : nullptr;
  uint4* dst = reinterpret_cast<uint4*>(lop + j * row_bytes);
  for (int64_t i = threadIdx.x; i < row_bytes / 16; i += blockDim.x)
    dst[i] = src ? src[i] : make_uint4(0, 0, 0, 0);
}

__global__ void k_tc_cols_f32(const double* __restrict__ nrm, const int32_t* __restrict__ lm,
                              int64_t L, int64_t l_pad, double C2, int cosine,
                              float* __restrict__ ca, float* __restrict__ cb,
                              float* __restrict__ colk) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l_pad) return;
  if (j >= L) tc_col_inert(j, ca, cb, colk);
  else if (cosine) tc_col_consts_cos(nrm[lm[j]], j, ca, cb, colk);
  else tc_col_consts(nrm[lm[j]], C2, j, ca, cb, colk);
}

__global__ void k_tc_cols_int(const int32_t* __restrict__ nrm, const int32_t* __restrict__ lm,
                              int64_t L, int64_t l_pad, int32_t* __restrict__ cc) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l_pad) return;
  cc[j] = j < L ? nrm[lm[j]] : (1 << 30);
}

// Fused greedy tile: landmark operand rows + column constants for the tile's
// new landmarks (count on the device); columns >= count are inert.
__global__ void k_tc_tile_lm(const uint8_t* __restrict__ xop, int64_t row_bytes,
                             const int32_t* __restrict__ new_lm,
                             const int32_t* __restrict__ l_count_dev, int kind, int cosine,
                             const void* __restrict__ nrm, double C2, uint8_t* __restrict__ lop,
                             float* __restrict__ ca, float* __restrict__ cb,
                             float* __restrict__ colk, int32_t* __restrict__ cc,
                             int64_t n_lm_blocks, const uint32_t* __restrict__ bmask,
                             const uint32_t* __restrict__ cmask,
                             const uint32_t* __restrict__ tmask, int64_t nblk, int act_words,
                             uint32_t* __restrict__ act) {
  pdl_wait();
  pdl_trigger();   // one wave
  if (blockIdx.x >= n_lm_blocks) {
    // pruning (cells.cu): per row block, which 32-column chunks of this tile
    // may hold an in-ball pair — act_words words per block for k_tc (byte t =
    // the chunks of 256-column tile t); a tile whose cell mask misses the
    // block's near cells is skipped without looking at its chunks
    __shared__ uint32_t scm[(kBigT / 32) * 8];
    __shared__ uint32_t stm[(kBigT / 256) * 8];
    const int64_t cnt = *l_count_dev;
    const int ntl = (int)((cnt + 255) / 256);
    for (int t = threadIdx.x; t < ntl * 64; t += blockDim.x) scm[t] = cmask[t];
    for (int t = threadIdx.x; t < ntl * 8; t += blockDim.x) stm[t] = tmask[t];
    __syncthreads();
    const int64_t b = (blockIdx.x - n_lm_blocks) * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    uint32_t bm[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) bm[w] = bmask[b * 8 + w];
    uint32_t live = 0u;   // word 0: the live tiles
    for (int wd = 0; wd < act_words; ++wd) {
      uint32_t bits = 0u;
      for (int tt = 0; tt < 4; ++tt) {
        const int t = 4 * wd + tt;
        if (t >= ntl) break;
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) any |= bm[w] & stm[t * 8 + w];
        if (!any) continue;
        for (int c = 0; c < 8; ++c) {
          uint32_t x = 0u;
#pragma unroll
          for (int w = 0; w < 8; ++w) x |= bm[w] & scm[(t * 8 + c) * 8 + w];
          bits |= (x != 0u ? 1u : 0u) << (8 * tt + c);
        }
        if ((bits >> (8 * tt)) & 0xffu) live |= 1u << t;
      }
      act[b * (act_words + 1) + 1 + wd] = bits;
    }
    act[b * (act_words + 1)] = live;
    return;
  }
  const int64_t j = blockIdx.x;
  const int64_t cnt = *l_count_dev;
  const bool live = j < cnt;
  const int32_t pt = live ? new_lm[j] : 0;
  const uint4* src = reinterpret_cast<const uint4*>(xop + (int64_t)pt * row_bytes);
  uint4* dst = reinterpret_cast<uint4*>(lop + j * row_bytes);
  for (int64_t i = threadIdx.x; i < row_bytes / 16; i += blockDim.x)
    dst[i] = live ? src[i] : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    if (kind == TC_TF32) {
      if (!live) tc_col_inert(j, ca, cb, colk);
      else if (cosine) tc_col_consts_cos(((const double*)nrm)[pt], j, ca, cb, colk);
      else tc_col_consts(((const double*)nrm)[pt], C2, j, ca, cb, colk);
    } else {
      cc[j] = live ? ((const int32_t*)nrm)[pt] : (1 << 30);
    }
  }
}

cudaError_t launch_tc_tile_landmarks(const TcPlan& P, const void* nrm, const int32_t* new_lm,
                                     const int32_t* l_count_dev, double C2, TcArgs& a,
                                     cudaStream_t s, int64_t* launches) {
  ++*launches;
  // (pruned launches: extra CTAs fold the row-block and chunk cell masks into
  // a.act in the same launch)
  const int64_t nblk = a.act ? (P.n_rows + 127) / 128 : 0;
  const int64_t extra = (nblk + 63) / 64;
  return launch_pdl(k_tc_tile_lm, dim3((unsigned)(P.l_rows + extra)), dim3(64), 0, s,
                    (const uint8_t*)P.xop, P.row_bytes, new_lm, l_count_dev, P.kind, P.cosine,
                    nrm, C2,
                    (uint8_t*)P.lop, (float*)a.col_a, (float*)a.col_b, (float*)a.colk,
                    (int32_t*)a.col_c, (int64_t)P.l_rows, a.act_bmask, a.act_cmask,
                    a.act_tmask, nblk, a.act_words, (uint32_t*)a.act);
}


// per-row thresholds of one row (norm nrm of its point), DESIGN.md 7.2
__device__ __forceinline__ void tc_row_consts(const RowParams& rp, const void* nrm, int64_t pt,
                                              bool live, int64_t j, float* lo, float* hi,
                                              int32_t* rr) {
  if (!rp.tf32) {
    rr[j] = live ? ((const int32_t*)nrm)[pt] - rp.lo_i : INT_MAX;
    return;
  }
  if (!live) {
    lo[j] = INFINITY;
    hi[j] = INFINITY;
    return;
  }
  const double np = ((const double*)nrm)[pt];
  if (rp.cosine) {
    if (np == 0.0) {
      lo[j] = -1e37f;
      hi[j] = INFINITY;
    } else {
      lo[j] = __double2float_rd(1.0 - rp.eps - 1.0000005e-6 * rp.eps - rp.m);
      hi[j] = __double2float_ru(1.0 - rp.eps + 1.0000005e-6 * rp.eps + rp.m);
    }
    return;
  }
  const double g = 0.5 * (np - rp.eps2);
  lo[j] = __double2float_rd(g - rp.C2 * np - rp.tau);
  hi[j] = __double2float_ru(g + rp.C2 * np + rp.tau);
}

// A2 on tensor cores: candidate j of the tile = unc[j] (j < nc): operand row,
// row thresholds and column constants; rows / columns >= nc are inert.
__global__ void k_tc_tile_cand(const uint8_t* __restrict__ xop, int64_t row_bytes,
                               const int32_t* __restrict__ unc,
                               const int32_t* __restrict__ n_unc_dev, int T, RowParams rp,
                               const void* __restrict__ nrm, double C2,
                               uint8_t* __restrict__ cop, float* __restrict__ rlo,
                               float* __restrict__ rhi, int32_t* __restrict__ rr,
                               float* __restrict__ ca, float* __restrict__ cb,
                               float* __restrict__ colk, int32_t* __restrict__ cc) {
  pdl_wait();
  pdl_trigger();   // one wave
  const int64_t j = blockIdx.x;
  const int64_t nc = min((int64_t)T, (int64_t)*n_unc_dev);
  const bool live = j < nc;
  const int32_t pt = live ? unc[j] : 0;
  const uint4* src = reinterpret_cast<const uint4*>(xop + (int64_t)pt * row_bytes);
  uint4* dst = reinterpret_cast<uint4*>(cop + j * row_bytes);
  for (int64_t i = threadIdx.x; i < row_bytes / 16; i += blockDim.x)
    dst[i] = live ? src[i] : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc_row_consts(rp, nrm, pt, live, j, rlo, rhi, rr);
    if (rp.tf32) {
      if (!live) tc_col_inert(j, ca, cb, colk);
      else if (rp.cosine) tc_col_consts_cos(((const double*)nrm)[pt], j, ca, cb, colk);
      else tc_col_consts(((const double*)nrm)[pt], C2, j, ca, cb, colk);
    } else {
      cc[j] = live ? ((const int32_t*)nrm)[pt] : (1 << 30);
    }
  }
}

cudaError_t launch_tc_tile_cand(const TcPlan& P, const TcPlan& Pc, const void* nrm,
                                const int32_t* unc, const int32_t* n_unc_dev, int T, double C2,
                                const RowParams& rp, TcArgs& ac, cudaStream_t s,
                                int64_t* launches) {
  ++*launches;
  return launch_pdl(k_tc_tile_cand, dim3((unsigned)Pc.l_rows), dim3(64), 0, s,
                    (const uint8_t*)P.xop, P.row_bytes, unc, n_unc_dev, T, rp, nrm, C2,
                    (uint8_t*)Pc.lop, (float*)ac.row_lo, (float*)ac.row_hi, (int32_t*)ac.row_r,
                    (float*)ac.col_a, (float*)ac.col_b, (float*)ac.colk, (int32_t*)ac.col_c);
}

cudaError_t launch_tc_prep(const void* X, int dtype, int64_t n, int d, const TcPlan& P,
                           void* nrm, DevStats* stats, cudaStream_t s, int64_t* launches) {
  ++*launches;
  // G lanes per row, each striding over its row: 8 lanes cover a 32-float
  // (128-byte) row in four coalesced 32-byte passes with a quarter of the
  // threads and shuffles a warp per row would need
  int G = 1;
  while (G < 8 && G < (int)(P.row_bytes / 4)) G *= 2;
  if (dtype == BM_F32)
    k_tc_prep_f32<<<(unsigned)((n * G + 255) / 256), 256, 0, s>>>(
        (const float*)X, n, d, (int)(P.row_bytes / 4), P.cosine, G, (float*)P.xop,
        (double*)nrm, stats);
  else   // integer rows: one warp per row
    k_tc_prep_int<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>((const uint8_t*)X, n, d, (int)P.row_bytes, dtype == BM_U8,
                                    (uint8_t*)P.xop, (int32_t*)nrm);
  return cudaGetLastError();
}

cudaError_t launch_tc_rows(const TcPlan& P, const void* nrm, int64_t n, double C2, double eps2,
                           double tau, int32_t lo_i, TcArgs& a, cudaStream_t s,
                           int64_t* launches) {
  ++*launches;
  const unsigned g = (unsigned)((P.n_pad + 255) / 256);
  if (P.kind == TC_TF32)
    k_tc_rows_f32<<<g, 256, 0, s>>>((const double*)nrm, n, P.n_pad, C2, eps2, tau,
                                    (float*)a.row_lo, (float*)a.row_hi);
  else
    k_tc_rows_int<<<g, 256, 0, s>>>((const int32_t*)nrm, n, P.n_pad, lo_i, (int32_t*)a.row_r);
  return cudaGetLastError();
}

cudaError_t launch_tc_landmarks(const TcPlan& P, const void* nrm, const int32_t* lm, int64_t L,
                                double C2, TcArgs& a, cudaStream_t s, int64_t* launches) {
  *launches += 2;
  k_tc_gather_lm<<<(unsigned)P.l_rows, 128, 0, s>>>((const uint8_t*)P.xop, P.row_bytes, lm, L,
                                                    P.l_rows, (uint8_t*)P.lop);
  const unsigned g = (unsigned)((P.l_rows + 255) / 256);
  if (P.kind == TC_TF32)
    k_tc_cols_f32<<<g, 256, 0, s>>>((const double*)nrm, lm, L, P.l_rows, C2, P.cosine,
                                    (float*)a.col_a, (float*)a.col_b, (float*)a.colk);
  else
    k_tc_cols_int<<<g, 256, 0, s>>>((const int32_t*)nrm, lm, L, P.l_rows, (int32_t*)a.col_c);
  return cudaGetLastError();
}

// ---- L1 on tensor cores: thermometer operands
// byte j B + k of a point row = -2 if level(x_j) > k else 0 (k < B); bytes
// dB..dB+2 = 1 (they meet the landmark's n_l), dB+3..dB+5 = n_p - cut in
// three signed bytes (they meet the landmark's 1s); a landmark row holds the
// bits as 0/1, n_l in three bytes, then 1,1,1.  So the s8 contraction gives
// acc = -2 <T(x), T(l)> + n_l + n_p - cut = SADq - cut.
__device__ __forceinline__ int l1t_chunk(int v, int k) {   // v split into 3 signed bytes
  const int c0 = v < -128 ? -128 : (v > 127 ? 127 : v);
  const int v1 = v - c0;
  const int c1 = v1 < -128 ? -128 : (v1 > 127 ? 127 : v1);
  return k == 0 ? c0 : (k == 1 ? c1 : v1 - c1);
}

// one warp per point: lane j < d bins coordinate j; every lane writes 8 bytes
// of the row (B >= 8, so 8 consecutive bytes span at most two coordinates)
__global__ void k_l1t_prep(const float* __restrict__ X, int64_t n, int d, int B, int row_bytes,
                           const double* __restrict__ qparam, double eps,
                           uint8_t* __restrict__ xop, int32_t* __restrict__ nrm) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const double mn = qparam[0], mx = qparam[1];
  const double st = mx > mn ? (mx - mn) / (double)(B + 1) : 1.0;
  int lv = 0;
  if (lane < d) {
    const double t = floor(((double)__ldg(X + p * (int64_t)d + lane) - mn) / st);
    lv = t < 0.0 ? 0 : (t > (double)B ? B : (int)t);
  }
  int np = lv;
  for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
  const int r = np - l1t_cut(qparam, eps, d, B);
  const int dB = d * B;
  // the folded constant bytes dB .. dB + 5 (1, 1, 1 and n_p - cut in three
  // signed bytes), little-endian from byte dB
  const uint64_t tail = 0x010101ull | ((uint64_t)(uint8_t)(int8_t)l1t_chunk(r, 0) << 24) |
                        ((uint64_t)(uint8_t)(int8_t)l1t_chunk(r, 1) << 32) |
                        ((uint64_t)(uint8_t)(int8_t)l1t_chunk(r, 2) << 40);
  auto bytemask = [](int nb) -> uint64_t {   // the low nb bytes (clamped to 0 .. 8)
    return nb >= 8 ? ~0ull : (nb <= 0 ? 0ull : ((1ull << (8 * nb)) - 1ull));
  };
  for (int h = 0; h < row_bytes; h += 256) {   // (rows of up to 512 bytes: two passes)
    const int b0 = h + lane * 8;
    const int ja = min(b0 / B, 31), jb = min((b0 + 7) / B, 31);
    const int la = __shfl_sync(0xffffffffu, lv, ja), lb = __shfl_sync(0xffffffffu, lv, jb);
    if (b0 >= row_bytes) continue;
    // byte i of the 8 is level kk + i of coordinate ja while kk + i < B (set
    // iff i < la - kk), else level kk + i - B of coordinate jb (set iff
    // i < lb + B - kk): two byte-prefix masks instead of a per-byte loop
    const int kk = b0 - ja * B, e1 = B - kk;
    uint64_t m = bytemask(max(0, min(min(8, e1), la - kk)));
    if (e1 < 8) m |= bytemask(max(e1, min(8, e1 + lb))) & ~bytemask(e1);
    uint64_t v = m & 0xfefefefefefefefeull;   // -2 per set level
    if (b0 + 8 > dB) {   // past the coordinates: the constant bytes, then zeros
      v &= bytemask(max(0, dB - b0));
      const int off = b0 - dB;   // (-8, row_bytes)
      if (off < 6) v |= off >= 0 ? (tail >> (8 * off)) : (tail << (8 * -off));
    }
    *reinterpret_cast<uint2*>(xop + p * (int64_t)row_bytes + b0) =
        make_uint2((uint32_t)v, (uint32_t)(v >> 32));
  }
  if (lane == 0) nrm[p] = np;
}

cudaError_t launch_l1t_prep(const float* X, int64_t n, int d, const TcPlan& P,
                            const double* qparam, double eps, int32_t* nrm, cudaStream_t s,
                            int64_t* launches) {
  const int B = l1t_bytes_per_coord(d);
  if (B == 0 || P.row_bytes > 512 || P.kind != TC_S8 || d * B + 6 > P.row_bytes)
    return cudaErrorInvalidValue;
  ++*launches;
  k_l1t_prep<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(
      X, n, d, B, (int)P.row_bytes, qparam, eps, (uint8_t*)P.xop, nrm);
  return cudaGetLastError();
}

// one warp per landmark row of the tile's operand (zero beyond the count)
__global__ void k_l1t_tile_lm(const uint8_t* __restrict__ xop, int row_bytes,
                              const int32_t* __restrict__ new_lm,
                              const int32_t* __restrict__ l_count_dev,
                              const int32_t* __restrict__ nrm, int d, int B, int64_t l_rows,
                              uint8_t* __restrict__ lop) {
  pdl_wait();
  pdl_trigger();   // one wave
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= l_rows) return;
  const bool live = j < (int64_t)*l_count_dev;
  for (int b0 = lane * 8; b0 < row_bytes; b0 += 256) {
  uint2 out = make_uint2(0u, 0u);
  if (live) {
    const int32_t pt = new_lm[j];
    const int nl = nrm[pt];
    const uint2 a = *reinterpret_cast<const uint2*>(xop + (int64_t)pt * row_bytes + b0);
    const int dB = d * B;
    uint32_t w[2] = {(a.x >> 1) & 0x01010101u, (a.y >> 1) & 0x01010101u};   // -2 -> 1, 0 -> 0
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int b = b0 + k;
      if (b < dB) continue;
      int v = 0;
      if (b < dB + 3) v = l1t_chunk(nl, b - dB);
      else if (b < dB + 6) v = 1;
      const uint32_t m = 0xffu << (8 * (k & 3));
      w[k >> 2] = (w[k >> 2] & ~m) | ((uint32_t)(uint8_t)(int8_t)v << (8 * (k & 3)));
    }
    out = make_uint2(w[0], w[1]);
  }
  *reinterpret_cast<uint2*>(lop + j * (int64_t)row_bytes + b0) = out;
  }
}

cudaError_t launch_l1t_tile_landmarks(const TcPlan& P, const int32_t* nrm, const int32_t* new_lm,
                                      const int32_t* l_count_dev, int d, cudaStream_t s,
                                      int64_t* launches) {
  ++*launches;
  const int B = l1t_bytes_per_coord(d);
  return launch_pdl(k_l1t_tile_lm, dim3((unsigned)((P.l_rows * 32 + 255) / 256)), dim3(256), 0, s,
                    (const uint8_t*)P.xop, (int)P.row_bytes, new_lm, l_count_dev, nrm, d, B,
                    (int64_t)P.l_rows, (uint8_t*)P.lop);
}


}  // namespace tc
}  // namespace bm
