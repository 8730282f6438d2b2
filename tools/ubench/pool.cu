// Host-time of stream-ordered pool allocations under the cover build's
// allocation pattern (diagnosing multi-100-ms host stalls).
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

__global__ void touch(char* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1;
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;   // 0 own pool (threshold max), 1 default pool
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaMemPool_t mp;
  cudaMemPoolProps pr{};
  pr.allocType = cudaMemAllocationTypePinned;
  pr.location.type = cudaMemLocationTypeDevice;
  pr.location.id = 0;
  cudaMemPoolCreate(&mp, &pr);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  const size_t sizes[] = {(size_t)1231 << 20, (size_t)1231 << 20, (size_t)77 << 20, (size_t)147 << 20, (size_t)60 << 20};
  for (int it = 0; it < 12; ++it) {
    std::vector<void*> ps;
    double worst = 0; int wi = -1;
    auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < 5; ++k) {
      auto t = std::chrono::steady_clock::now();
      void* p;
      if (mode == 0) cudaMallocFromPoolAsync(&p, sizes[k], mp, s); else cudaMallocAsync(&p, sizes[k], s);
      double dt = ms_since(t);
      if (dt > worst) { worst = dt; wi = k; }
      touch<<<1184, 256, 0, s>>>((char*)p, sizes[k]);
      ps.push_back(p);
      if (k == 2) {   // free the two big ones mid-way, like the edges step
        auto tf = std::chrono::steady_clock::now();
        cudaFreeAsync(ps[0], s); cudaFreeAsync(ps[1], s);
        double df = ms_since(tf);
        if (df > worst) { worst = df; wi = 100 + k; }
      }
    }
    for (int k = 2; k < 5; ++k) cudaFreeAsync(ps[k], s);
    cudaStreamSynchronize(s);
    printf("iter %2d: total %8.2f ms, worst call %8.3f ms (#%d)\n", it, ms_since(t0), worst, wi);
  }
  return 0;
}
