// tcgen05 peak microbenchmark (sm_100a): dense MMA throughput of one CTA per
// SM issuing back-to-back tcgen05.mma.cta_group::1 with M = 128, N = 256 from
// shared memory (128B-swizzled K-major, one 128-byte K atom per operand) into
// two alternating TMEM accumulators, no epilogue.  Measures the ceiling the
// membership contraction (tc.cu) is compared against: kind::tf32 (C2/C3/C5
// cosine), kind::i8 (C4) and kind::f16 with bf16 operands (cross-check against
// the cuBLAS bf16 figure in MEASURED_PEAKS.json).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_peak tc_peak.cu
//   ./tc_peak            # prints one JSON line per kind
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

enum { K_BF16 = 0, K_TF32 = 1, K_I8 = 2 };

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;   // 128-byte swizzle
  return d;
}
template <int KIND>
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  // c_format [4,6): 1 = F32, 2 = S32; a/b format [7,10)/[10,13):
  // f16 kind: BF16 = 1; tf32 kind: TF32 = 2; i8 kind: s8 = 1
  return (KIND == K_I8 ? (2u << 4) | (1u << 7) | (1u << 10)
                       : (1u << 4) | ((KIND == K_TF32 ? 2u : 1u) << 7) |
                             ((KIND == K_TF32 ? 2u : 1u) << 10)) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                    uint32_t acc) {
  if constexpr (KIND == K_TF32)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc)
                 : "memory");
  else if constexpr (KIND == K_I8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc)
                 : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc)
                 : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_peak(int iters, unsigned seed, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                 // 128 rows x 128 B
  uint8_t* sB = sm + 128 * 128;     // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  // operands: small pseudo-random values (finite for every kind)
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) {
    uint32_t h = (i * 2654435761u) ^ seed;
    h ^= h >> 13;
    uint32_t v = KIND == K_I8 ? (h & 0x3f3f3f3fu)
                              : (KIND == K_TF32 ? (0x3f800000u | (h & 0x007fe000u))
                                                : (0x3f803f80u | (h & 0x007f007fu)));
    ((uint32_t*)sm)[i] = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t ID = idesc<KIND>(128, 256);
    const uint32_t a = su32(sA), b = su32(sB);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it & 1) * 256);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)   // one 128-byte K atom = 4 MMAs
        mma<KIND>(d, sdesc(a + ks * 32), sdesc(b + ks * 32), ID, ks ? 1u : 0u);
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(su32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345678u) atomicAdd(sink, 1);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// TMEM read rate: every warp reads its 32-lane quadrant (warp % 4), all 512
// columns, with tcgen05.ld.32x32b.x64 (64 columns x 4 B per lane), repeatedly.
__global__ void __launch_bounds__(512, 1) k_tmem_read(int iters, int* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int c = 0; c < 512; c += 64) {
      uint32_t v[64];
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
          : "r"(tmem + (uint32_t)c)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 64; ++i) acc ^= v[i];
    }
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

static void run_tmem(int warps) {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);   // kHz
  int* sink;
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  k_tmem_read<<<sms, 32 * warps>>>(iters / 10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_tmem_read<<<sms, 32 * warps>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // bytes: every warp reads 32 lanes x 512 columns x 4 B per iteration
  const double bytes = (double)warps * 32 * 512 * 4 * iters * sms;
  const double gbs = bytes / (best * 1e-3) / 1e9;
  printf("{\"kind\": \"tmem_read\", \"warps\": %d, \"GB_per_s\": %.1f, \"B_per_clk_per_sm_at_max\": "
         "%.1f, \"ms\": %.4f, \"status\": \"%s\"}\n",
         warps, gbs, gbs * 1e9 / sms / (clk * 1e3), best, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

template <int KIND>
static void run(const char* name, int k_per_atom) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(k_peak<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* sink;
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  k_peak<KIND><<<sms, 128, smem>>>(iters / 10, 1u, sink);   // warm-up
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_peak<KIND><<<sms, 128, smem>>>(iters, 2u + r, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const cudaError_t err = cudaGetLastError();
  const double flops = 2.0 * 128 * 256 * (double)k_per_atom * iters * sms;
  printf("{\"kind\": \"%s\", \"tflops\": %.1f, \"ms\": %.4f, \"sms\": %d, \"mma\": "
         "\"M128 N256 K%d x4 per atom, cta_group::1\", \"status\": \"%s\"}\n",
         name, flops / (best * 1e-3) / 1e12, best, sms, k_per_atom / 4,
         cudaGetErrorString(err));
  cudaFree(sink);
}

int main() {
  run<K_BF16>("bf16", 64);   // 128 B = 64 bf16 per atom
  run<K_TF32>("tf32", 32);   // 32 tf32
  run<K_I8>("i8", 128);      // 128 int8
  for (int w : {4, 8, 16}) run_tmem(w);
  return 0;
}
