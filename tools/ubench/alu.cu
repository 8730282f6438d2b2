// Instruction-throughput microbenchmark (sm_100a): lane-instructions per
// second for the candidate inner-loop instructions of the CUDA-core pair
// kernels.  8 independent chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define ITERS 4096
#define CH 8

template <int OP>
__global__ void kern(float* out, float seed) {
  float a[CH];
  float2 a2[CH];
  unsigned u[CH];
  half2 h[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = seed + threadIdx.x + c;
    a2[c] = make_float2(a[c], a[c] + 1.f);
    u[c] = threadIdx.x * 7 + c;
    h[c] = __floats2half2_rn(a[c], a[c]);
  }
  const float b = seed * 0.5f, cc = seed * 0.25f;
  const float2 b2 = make_float2(b, cc);
  const unsigned ub = 0x01020304u ^ threadIdx.x;
  const half2 hb = __floats2half2_rn(b, cc);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) a[c] = a[c] + b;                       // FADD
      if (OP == 1) a[c] = fmaf(a[c], a[c], cc);           // FFMA (3 reg)
      if (OP == 2) a2[c] = __fadd2_rn(a2[c], b2);         // FADD2
      if (OP == 3) a2[c] = __ffma2_rn(a2[c], a2[c], b2);  // FFMA2
      if (OP == 4) a[c] = fmaxf(a[c], b + c);             // FMNMX
      if (OP == 5) u[c] = (unsigned)__dp4a((int)u[c], (int)ub, (int)u[c]);  // IDP4A
      if (OP == 6) u[c] = __vabsdiffu4(u[c], ub);         // VABSDIFF4
      if (OP == 7) a[c] = a[c] + fabsf(a[c] - b);         // FADD + FADD|.| (L1 pattern, 2 instr)
      if (OP == 8) h[c] = __hadd2(h[c], __habs2(__hsub2(h[c], hb)));  // HADD2 |.| pattern
      if (OP == 9) u[c] = __vsadu4(u[c], ub) + u[c];      // vsadu4
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c] + a2[c].x + a2[c].y + (float)u[c] + __low2float(h[c]);
  if (s == 1234.5f) out[0] = s;
}

template <int OP>
void run(const char* name, double instr_per_op) {
  float* out;
  cudaMalloc(&out, 4);
  kern<OP><<<148 * 8, 256>>>(out, 1.0f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<OP><<<148 * 8, 256>>>(out, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * 148 * 8 * 256 * (double)ITERS * CH;
  printf("%-28s %8.2f T ops/s  (%.2f T lane-instr/s)\n", name, ops / (ms * 1e-3) / 1e12,
         ops * instr_per_op / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz; issue peak 148*128*clk = %.2f T lane-instr/s\n", clk,
         148.0 * 128 * clk * 1e3 / 1e12);
  run<0>("FADD", 1);
  run<1>("FFMA 3-reg", 1);
  run<2>("FADD2 (per pair of lanes-ops)", 1);
  run<3>("FFMA2", 1);
  run<4>("FMNMX(+FADD)", 2);
  run<5>("IDP4A", 1);
  run<6>("VABSDIFF4", 1);
  run<7>("L1 f32 pattern (per dim)", 2);
  run<8>("L1 f16x2 pattern (per 2 dim)", 2);
  run<9>("VSADU4+IADD", 2);
  return 0;
}
