// api.cu — C ABI (include/bm.h) and host orchestration of the cover build.
//
// Sequence on the caller's stream:
//   A0 prep -> greedy tiles {A2 adjacency, A3 resolve, A4 coverage, compaction}
//   (device-resident counts; the host checks termination once per batch of
//   tiles) -> B membership (+B' fp64 band) -> C sort + CSR both ways ->
//   D1 pair emission -> D2 radix sort -> D3 unique.
// Host<->device synchronisation: one count read-back per greedy batch, then
// M (membership count), P (pair count) and E (edge count).
#include <math.h>
#include <stdarg.h>
#include <time.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <algorithm>
#include <vector>

#include "internal.cuh"
#include "tc.cuh"

// diagnostics: per-CTA %globaltimer phase stamps of one traced k_tc launch
// (TC_STAMP slots, tc.cu), summarised to stderr
// diagnostics: per-role wait cycles of one traced k_tc launch (BM_TC_TRACE=2),
// medians over the CTAs, in microseconds at the nominal clock
static cudaError_t print_tc_wtrace(const unsigned long long* tr, int G, const char* tag,
                                   cudaStream_t s) {
  std::vector<unsigned long long> h((size_t)G * 16);
  cudaError_t e = cudaMemcpyAsync(h.data(), tr, sizeof(unsigned long long) * G * 16,
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  static const char* names[10] = {"P wait B stage", "P wait A buf/fold slot", "M wait A",
                                  "M wait TMEM buf", "M wait B data", "E wait acc (x8 warps)",
                                  "E tmem ld (x8)", "E flush (x8)", "E loop total (x8)",
                                  "M wait fold consts"};
  fprintf(stderr, "wtrace [%s]", tag);
  for (int k = 0; k < 10; ++k) {
    std::vector<double> v;
    for (int b = 0; b < G; ++b) v.push_back((double)h[b * 16 + k] / 1965.0);
    std::sort(v.begin(), v.end());
    fprintf(stderr, " | %s %.1f", names[k], v[v.size() / 2]);
  }
  fprintf(stderr, " us\n");
  return cudaSuccess;
}

// diagnostics (BM_TC_TRACE=3): CTA 0's per-tile timeline, mean cycles over
// tiles 32..511: MMA wait for a free buffer, MMA issue, commit -> epilogue
// sees the accumulator, epilogue hold of the buffer, tile period
static cudaError_t print_tc_tline(const unsigned long long* tl, const char* tag, cudaStream_t s) {
  std::vector<unsigned long long> h(512 * 5);
  cudaError_t e = cudaMemcpyAsync(h.data(), tl, sizeof(unsigned long long) * 512 * 5,
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  double a[5] = {0, 0, 0, 0, 0};
  int m = 0;
  for (int i = 32; i + 1 < 512; ++i) {
    const unsigned long long* r = &h[i * 5];
    if (!r[0] || !r[4] || !h[(i + 1) * 5 + 3]) break;
    a[0] += (double)(long long)(r[1] - r[0]);
    a[1] += (double)(long long)(r[2] - r[1]);
    a[2] += (double)(long long)(r[3] - r[2]);
    a[3] += (double)(long long)(r[4] - r[3]);
    a[4] += (double)(long long)(h[(i + 1) * 5 + 3] - r[3]);
    ++m;
  }
  if (m)
    fprintf(stderr,
            "tline [%s] tiles %d | MMA wait buf %.0f | MMA issue %.0f | commit->epi %.0f | "
            "epi hold %.0f | period %.0f clk\n",
            tag, m, a[0] / m, a[1] / m, a[2] / m, a[3] / m, a[4] / m);
  return cudaSuccess;
}

static cudaError_t print_tc_trace(const unsigned long long* tr, int G, const char* tag,
                                  cudaStream_t s) {
  std::vector<unsigned long long> h((size_t)G * 16);
  cudaError_t e = cudaMemcpyAsync(h.data(), tr, sizeof(unsigned long long) * G * 16,
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < G; ++b) t0 = h[b * 16] && h[b * 16] < t0 ? h[b * 16] : t0;
  static const char* names[12] = {"start", "prologue", "pdl", "A0 issued", "producer done",
                                  "A0 landed", "mma done", "epi0 first", "epi1 first",
                                  "epi0 done", "epi1 done", "end"};
  fprintf(stderr, "trace [%s]\n", tag);
  for (int k = 0; k < 12; ++k) {
    std::vector<double> v;
    for (int b = 0; b < G; ++b)
      if (h[b * 16 + k]) v.push_back((double)(h[b * 16 + k] - t0) * 1e-3);
    std::sort(v.begin(), v.end());
    if (!v.empty())
      fprintf(stderr, "trace %-14s min %8.2f  med %8.2f  max %8.2f us  (%zu CTAs)\n", names[k],
              v.front(), v[v.size() / 2], v.back(), v.size());
  }
  std::vector<int> ord(G);
  for (int b = 0; b < G; ++b) ord[b] = b;
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return h[x * 16 + 11] > h[y * 16 + 11]; });
  for (int i = 0; i < 4 && i < G; ++i) {
    const int b = ord[i];
    fprintf(stderr, "slow CTA %3d:", b);
    for (int k = 0; k < 12; ++k)
      fprintf(stderr, " %6.2f", h[b * 16 + k] ? (double)(h[b * 16 + k] - t0) * 1e-3 : -1.0);
    fprintf(stderr, "\n");
  }
  return cudaSuccess;
}


namespace {

thread_local std::string g_err;

bm_status set_err(bm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(expr)                                                                      \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      cudaGetLastError();                                                             \
      return set_err(BM_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),       \
                     __FILE__, __LINE__);                                             \
    }                                                                                 \
  } while (0)

// Device memory: a library-owned block cache.  Blocks are carved by
// cudaMalloc in size classes (8 per octave above 1 MiB, powers of two below,
// <= 12.5% slack) and, once released, kept on a free list of the (device,
// stream) they were last used on: a later allocation on the same stream reuses
// them with no synchronisation (stream order makes the reuse safe).  The CUDA
// stream-ordered pool was measured to stall the host for 100-600 ms in
// cudaMallocFromPoolAsync on this platform even with an unlimited release
// threshold; the cache has no such path.  bm_trim_memory() returns cached
// blocks to the system.
struct BlockCache {
  struct Key {
    int dev;
    cudaStream_t s;
    size_t cls;
    bool operator<(const Key& o) const {
      if (dev != o.dev) return dev < o.dev;
      if (s != o.s) return (uintptr_t)s < (uintptr_t)o.s;
      return cls < o.cls;
    }
  };
  std::mutex mu;
  std::map<Key, std::vector<void*>> free_;
  std::unordered_map<void*, std::pair<int, size_t>> live_;   // ptr -> (device, class)

  static size_t size_class(size_t b) {
    if (b <= 256) return 256;
    if (b <= ((size_t)1 << 20)) {
      size_t c = 256;
      while (c < b) c <<= 1;
      return c;
    }
    int lg = 63 - __builtin_clzll((unsigned long long)b);
    const size_t step = (size_t)1 << (lg - 3);
    return (b + step - 1) / step * step;
  }
  cudaError_t alloc(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const size_t cls = size_class(bytes);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_.find(Key{dev, s, cls});
      if (it != free_.end() && !it->second.empty()) {
        *p = it->second.back();
        it->second.pop_back();
        live_[*p] = {dev, cls};
        return cudaSuccess;
      }
    }
    e = cudaMalloc(p, cls);
    if (e == cudaErrorMemoryAllocation) {   // give cached blocks back, retry once
      cudaGetLastError();
      trim();
      e = cudaMalloc(p, cls);
    }
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    live_[*p] = {dev, cls};
    return cudaSuccess;
  }
  void release(void* p, cudaStream_t s) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu);
    auto it = live_.find(p);
    if (it == live_.end()) return;
    free_[Key{it->second.first, s, it->second.second}].push_back(p);
    live_.erase(it);
  }
  void trim() {
    std::map<Key, std::vector<void*>> victims;
    {
      std::lock_guard<std::mutex> lk(mu);
      victims.swap(free_);
    }
    if (victims.empty()) return;
    cudaDeviceSynchronize();   // blocks may still be in use by queued work
    for (auto& kv : victims)
      for (void* q : kv.second) cudaFree(q);
  }
};
BlockCache g_cache;

// Pinned host blocks for the host-buffer API's results (one block per cover,
// all six arrays carved from it): device->host copies into pinned memory run
// at full link speed and can be queued behind one synchronisation; pinning
// fresh pages on every call would cost more than the copies.
struct PinnedCache {
  std::mutex mu;
  std::map<size_t, std::vector<void*>> free_;
  static size_t size_class(size_t b) { return BlockCache::size_class(b < 4096 ? 4096 : b); }
  void* get(size_t bytes, size_t* cls_out) {
    const size_t cls = size_class(bytes);
    *cls_out = cls;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_.find(cls);
      if (it != free_.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, cls) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  void put(void* p, size_t cls) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu);
    free_[cls].push_back(p);
  }
  void trim() {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : free_)
      for (void* p : kv.second) cudaFreeHost(p);
    free_.clear();
  }
};
PinnedCache g_pinned;

// Allocations owned by one build call (stream-ordered on the call's stream).
struct Pool {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Pool(cudaStream_t st) : s(st) {}
  ~Pool() {
    for (void* p : ptrs)
      if (p) g_cache.release(p, s);
  }
  template <class T>
  bm_status alloc(T** out, size_t count) {
    void* p = nullptr;
    const size_t bytes = count * sizeof(T);
    cudaError_t e = g_cache.alloc(&p, bytes, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *out = nullptr;
      return set_err(e == cudaErrorMemoryAllocation ? BM_ENOMEM : BM_ECUDA,
                     "device allocation (%zu bytes): %s", bytes, cudaGetErrorString(e));
    }
    ptrs.push_back(p);
    *out = (T*)p;
    return BM_OK;
  }
  // remove from the pool (ownership moves to the bm_cover)
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) q = nullptr;
  }
  void free_now(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        g_cache.release(q, s);
        q = nullptr;
      }
  }
};

#define TRY(expr)                      \
  do {                                 \
    bm_status _st = (expr);            \
    if (_st != BM_OK) return _st;      \
  } while (0)

struct Priv {
  cudaStream_t stream;
  void* pinned;        // host-buffer covers: pinned block of landmarks + both CSRs
  size_t pinned_cls;
  void* pinned_e;      //   ... and of the edge list
  size_t pinned_e_cls;
};

// A per-thread side stream for the host-buffer API's result copies (they
// overlap the edge construction on the caller's stream)
static cudaStream_t side_stream() {
  static thread_local cudaStream_t s2 = nullptr;
  if (!s2 && cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess) s2 = nullptr;
  return s2;
}

int bits_for(int64_t v) {  // number of bits to represent 0..v (>= 1)
  int b = 1;
  while (b < 63 && (v >> b) != 0) ++b;
  return b;
}

float round_down_f(double v) {
  float f = (float)v;
  if ((double)f > v) f = nextafterf(f, -INFINITY);
  return f;
}
float round_up_f(double v) {
  float f = (float)v;
  if ((double)f < v) f = nextafterf(f, INFINITY);
  return f;
}

// Rigorous fp32 classification band.
bm::Thresh make_thresh(int kind, int d, double eps) {
  bm::Thresh t{};
  const double u = ldexp(1.0, -24);
  const double tie = 1e-6;
  t.eps = eps;
  t.eps2 = eps * eps;
  t.tie_rel = tie;
  t.cosine = kind == bm::K_COSF ? 1 : 0;
  if (kind == bm::K_L2F) {
    // |s - D| <= (d+3) u D (difference rounding, squaring, fp32 accumulation),
    // near tie |d-eps| <= 1e-6 eps  <=>  |D - eps^2| <= 2.000001e-6 eps^2
    double eta = (d + 3) * u * 1.01 + 1e-12;
    double tie2 = 2.000001e-6;
    t.lo_f = round_down_f(t.eps2 * (1.0 - tie2 - 2.0 * eta));
    t.hi_f = round_up_f(t.eps2 * (1.0 + tie2 + 2.0 * eta));
  } else if (kind == bm::K_L1F) {
    double eta = (d + 1) * u * 1.01 + 1e-12;
    t.lo_f = round_down_f(eps * (1.0 - tie - 2.0 * eta));
    t.hi_f = round_up_f(eps * (1.0 + tie + 2.0 * eta));
  } else if (kind == bm::K_COSF) {
    // |c_hat - c| <= (d+3) u (normalisation + fp32 dot), absolute
    double eta = (d + 3) * u * 1.01 + 1e-12;
    double c_in = (1.0 - eps) + tie * eps + 2.0 * eta;   // in  if c_hat >  c_in
    double c_out = (1.0 - eps) - tie * eps - 2.0 * eta;  // out if c_hat <= c_out
    t.lo_f = round_down_f(-c_in);                        // score = -c_hat
    t.hi_f = round_up_f(-c_out);
  } else if (kind == bm::K_L2I) {
    double K = ceil(t.eps2) - 1.0;  // largest integer d2 with (double)d2 < eps*eps
    double lo = K + 1.0;
    t.lo_i = lo > 2147483647.0 ? 2147483647 : (int32_t)lo;
  } else {
    double lo = ceil(eps);          // in iff s < ceil(eps)  <=>  (double)s < eps
    t.lo_i = lo > 2147483647.0 ? 2147483647 : (int32_t)lo;
  }
  return t;
}

// Initial capacity of the membership key buffer (8 B per key): M is unknown
// until the greedy ends.  16 keys per point covers every BASELINE config
// (C5: M/n ~ 10); a larger M triggers one exact-capacity recount
// (membership_full).  Bounded by a quarter of the free device memory.
int64_t initial_key_cap(int64_t n) {
  int64_t cap = n * 16 > (1 << 20) ? n * 16 : (1 << 20);
  static int64_t lim_of[bm::kMaxDevices] = {};   // an eighth of the device memory, in keys
  int64_t& lim = lim_of[bm::cur_device()];
  if (lim <= 0) {
    int dev = 0;
    cudaDeviceProp pr;
    lim = (cudaGetDevice(&dev) == cudaSuccess &&
           cudaGetDeviceProperties(&pr, dev) == cudaSuccess)
              ? (int64_t)(pr.totalGlobalMem / 8 / sizeof(unsigned long long))
              : (int64_t)1 << 28;
  }
  return cap > lim && lim > (1 << 20) ? lim : cap;
}

// Tensor-core band constant: |acc - x.l| <= c1
// |x||l|, c1 = operand rounding to tf32 (2u_t + u_t^2) + fp32 accumulation
// (4 K 2^-23, safety 2); the epilogue's roundings add 2^-22; |x||l| <=
// (n_p + n_l)/2, and 1.25 is a further safety factor.
// The column constant cb_j (|cb_j| <= n_l/2) is folded into the MMA as three
// more exact products, adding c3 |cb_j| with c3 = 4 (K+3) 2^-23 (1.001).
// Cosine on tensor cores: |acc - x.y/(|x||y|)| <= c1 (operands x/|x| within
// 2u of the exact unit vectors per coordinate, then rounded to tf32), plus
// 8u for the fp32 normalisation and 2^-20 slack.
double tc_cos_margin(int ksteps) {
  const double ut = ldexp(1.0, -11), u = ldexp(1.0, -24);
  const double K = 8.0 * ksteps + 3.0;
  const double c1 = 2.0 * ut + ut * ut + 4.0 * K * ldexp(1.0, -23) * (1.0 + ut) * (1.0 + ut);
  return 1.25 * (c1 * (1.0 + 4.0 * u) * (1.0 + 4.0 * u) + 8.0 * u + ldexp(1.0, -20));
}

// Tensor-core operand row pitch: whole 128-byte swizzle atoms.  Measured on
// B200 (tools/tc_probe_c2.py): TMA tiles of 48-byte rows (C2, d = 10) take
// 3.3x longer than the same tiles of 128-byte rows, and C5 cosine (64-byte
// rows) drops from 604 to 378 ms with the padded pitch.
int64_t tc_row_bytes(int d, int esz) {
  return (((int64_t)d * esz + 127) / 128) * 128;
}

// D: the bit-triangle edge path when it fits min(8 GiB, free / 4) of HBM
// D1 row-union emission pays when the witnessed pairs repeat across the
// points two balls share: at least this many pairs per landmark (C5: ~2000,
// C3 eps=8: 265, where the per-point emission is faster)
constexpr int64_t kRowsMinPairs = 512;
// the bit triangle is the default while it stays this small (L <~ 46000: its
// random atomics then mostly hit L2; C4's L = 7935 takes 8 MB)
constexpr double kTriAutoBytes = 256.0 * (1 << 20);

bool use_tri_bitmap(int64_t L, int flags) {
  if (flags & BM_FLAG_NO_EDGE_TRIANGLE) return false;
  const double bytes = 4.0 * (double)bm::tri_bitmap_words(L);
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  return bytes <= 8.0 * (1ull << 30) && bytes <= 0.25 * (double)fr;
}

double tc_band_c2(int ksteps) {
  const double ut = ldexp(1.0, -11);
  const double K = 8.0 * ksteps + 3.0;
  const double c1 = 2.0 * ut + ut * ut + 4.0 * K * ldexp(1.0, -23) * (1.0 + ut) * (1.0 + ut);
  const double c3 = 4.0 * K * ldexp(1.0, -23) * 1.001;
  return 1.25 * 0.5 * (c1 + c3 + ldexp(1.0, -22));
}

__global__ void k_iota(int32_t* a, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

// BM_TRACE=1: synchronise and print the host time of every traced sub-step
// (diagnostics only; off by default).
struct Trace {
  bool on;
  cudaStream_t s;
  double t0;
  static double now() {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  int level;
  explicit Trace(cudaStream_t st)
      : on(getenv("BM_TRACE") != nullptr && atoi(getenv("BM_TRACE")) == 1), s(st), t0(now()),
        level(getenv("BM_TRACE") ? atoi(getenv("BM_TRACE")) : 0) {}
  void operator()(const char* what) {
    if (level == 3) {   // host timestamps only (no synchronisation)
      const double t = now();
      fprintf(stderr, "[bm trace host] %-28s %9.3f ms\n", what, t - t0);
      t0 = t;
      return;
    }
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = now();
    fprintf(stderr, "[bm trace] %-28s %9.3f ms\n", what, t - t0);
    t0 = t;
  }
};

// Timing events come from a per-thread cache (creating and destroying CUDA
// events costs host time inside every timed build).
static cudaEvent_t cached_event(size_t i) {
  static thread_local std::vector<cudaEvent_t> evs;
  while (evs.size() <= i) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    evs.push_back(e);
  }
  return evs[i];
}

struct Timer {
  bool on;
  cudaStream_t s;
  cudaEvent_t ev[BM_NUM_STEPS];
  int n = 0;
  Timer(bool o, cudaStream_t st) : on(o), s(st) {
    if (on)
      for (int i = 0; i < BM_NUM_STEPS; ++i) ev[i] = cached_event((size_t)i);
  }
  void mark(int i) {
    if (on && ev[i]) cudaEventRecord(ev[i], s);
  }
};

// B' inside the contraction's epilogue: rows to re-decide band pairs from.
void set_recheck(bm::tc::TcArgs& ta, const void* xrows, int xstride, int d, const bm::Thresh& th,
                 const int32_t* lm_idx, int64_t* ties, int64_t tie_cap, bm::DevStats* stats) {
  ta.xrows = (const float*)xrows;
  ta.xstride = xstride;
  ta.d = d;
  ta.eps = th.eps;
  ta.eps2 = th.eps2;
  ta.tie_rel = th.tie_rel;
  ta.tie_abs = th.tie_rel * th.eps;
  ta.lm_idx = lm_idx;
  ta.cosine = th.cosine;
  ta.ties = ties;
  ta.tie_cap = tie_cap;
  ta.stats = stats;
}

// tf32 column-constant fold operands: B constants [l_rows][8] and the A ones tile.
// The fold's constant A tile ({1,1,1,0,...} x 128 rows) is the same for every
// build: one copy per device, written once on first use by an async copy on
// the caller's stream followed by a synchronisation of that stream, so the
// pointer is published only after the data has landed (a plain cudaMemcpy from
// pageable memory may return before the DMA completes and is not ordered
// against a non-blocking stream).
static const float* fold_ones_tile(cudaStream_t s) {
  static std::mutex mu;
  static const float* tiles[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!tiles[dev]) {
    static float h[128 * 8];
    for (int i = 0; i < 128 * 8; ++i) h[i] = (i & 7) < 3 ? 1.f : 0.f;
    float* d = nullptr;
    if (cudaMalloc(&d, sizeof h) != cudaSuccess) return nullptr;
    if (cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      cudaFree(d);
      return nullptr;
    }
    tiles[dev] = d;
  }
  return tiles[dev];
}

bm_status alloc_fold(Pool& pool, bm::tc::TcPlan& P, bm::tc::TcArgs& ta, cudaStream_t s,
                     int64_t* launches) {
  (void)launches;
  float* colk = nullptr;
  TRY(pool.alloc(&colk, (size_t)P.l_rows * 8));
  const float* ones = fold_ones_tile(s);
  if (!ones) return set_err(BM_ENOMEM, "fold constant tile allocation failed");
  ta.colk = colk;
  P.ones = ones;
  return BM_OK;
}

// Step B over all n points x all L landmarks in one pass (used only when the
// fused loop's key buffer overflowed: M is then known exactly and `keys` has
// room for it).  Keys are point << 32 | landmark position, as in the loop.
bm_status membership_full(Pool& pool, int kind, const bm::PairArgs& base, bm::tc::TcPlan P,
                          bool use_tc, const void* tc_nrm, const int32_t* lm, int64_t L,
                          int64_t n, int d, bm_dtype dtype, int nu, const bm::Thresh& th,
                          double C2, unsigned long long* keys, int64_t key_cap,
                          int64_t* ties_dev, int64_t tie_cap, bm::DevStats* stats,
                          cudaStream_t s, int64_t* launches, int64_t* M_out) {
  using namespace bm;
  CK(cudaMemsetAsync(&stats->key_count, 0, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(&stats->near_ties, 0, sizeof(unsigned long long), s));
  if (use_tc) {
    const int BN = tc::tc_bn_for(P.kind, P.katoms);
    P.l_rows = ((L + BN - 1) / BN) * BN;
    tc::TcArgs ta{};
    ta.n = n;
    ta.L = L;
    ta.ksteps = (int)(((int64_t)d * (dtype == BM_F32 ? 4 : 1) + 31) / 32);
    ta.lbits = 32;
    TRY(pool.alloc((uint8_t**)&P.lop, (size_t)P.l_rows * P.row_bytes));
    const int RB = tc::tc_rows_for(P.kind, P.katoms);
    P.n_pad = ((n + RB - 1) / RB) * RB;
    double tau = 0.0;
    if (P.kind == tc::TC_TF32) {
      float *rlo, *rhi, *ca, *cb;
      TRY(pool.alloc(&rlo, (size_t)P.n_pad));
      TRY(pool.alloc(&rhi, (size_t)P.n_pad));
      TRY(pool.alloc(&ca, (size_t)P.l_rows));
      TRY(pool.alloc(&cb, (size_t)P.l_rows));
      ta.row_lo = rlo;
      ta.row_hi = rhi;
      ta.col_a = ca;
      ta.col_b = cb;
      TRY(alloc_fold(pool, P, ta, s, launches));
      tau = 1.0000005e-6 * th.eps2 + th.eps2 * ldexp(1.0, -21);
    } else {
      int32_t *rr, *cc;
      TRY(pool.alloc(&rr, (size_t)P.n_pad));
      TRY(pool.alloc(&cc, (size_t)P.l_rows));
      ta.row_r = rr;
      ta.col_c = cc;
    }
    if (P.cosine) CK(tc::launch_tc_rows_cos(P, tc_nrm, n, th.eps, tc_cos_margin(ta.ksteps), ta, s,
                                            launches));
    else CK(tc::launch_tc_rows(P, tc_nrm, n, C2, th.eps2, tau, th.lo_i, ta, s, launches));
    CK(tc::launch_tc_landmarks(P, tc_nrm, lm, L, C2, ta, s, launches));
    ta.keys = keys;
    ta.key_count = &stats->key_count;
    ta.key_cap = key_cap;
    set_recheck(ta, base.xrows, 2 * nu, d, th, lm, ties_dev, tie_cap, stats);
    CK(tc::launch_tc(P, ta, s, launches));
    pool.free_now((void*)P.lop);
  } else {
    PairArgs m = base;
    m.qidx = nullptr;
    m.q_begin = 0;
    m.q_end = n;
    m.lidx = lm;
    m.l_begin = 0;
    m.l_end = L;
    m.lpos0 = 0;
    m.keys = keys;
    m.key_cap = key_cap;
    m.lbits = 32;
    m.ties = ties_dev;
    m.tie_cap = tie_cap;
    CK(launch_pairs(kind, MODE_MEMBER, m, n, s, launches));
  }
  unsigned long long kc = 0;
  CK(cudaMemcpyAsync(&kc, &stats->key_count, sizeof kc, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *M_out = (int64_t)kc;   // > key_cap: the keys were dropped, the caller resizes and reruns
  return BM_OK;
}

// Pinned host mailbox for the build's small device->host readbacks: a copy
// into pageable memory blocks the host until the stream reaches it, so two
// such copies cost two round trips; into pinned memory they are queued and one
// stream synchronisation covers them all.
struct Mailbox {
  int32_t hc[8];        // the greedy loop's counters (n_unc ping-pong, L, dL)
  bm::DevStats hs;      // statistics at the loop's last check
  bm::DevStats hs_end;  // statistics at the end of the build
  int64_t pe[2];        // edges: P (witnessed pairs), E
  int64_t ties[3 * 1024];   // the first near-tie triples (with the final synchronisation)
};
static Mailbox* mailbox() {
  static thread_local Mailbox* mb = nullptr;
  if (!mb && cudaMallocHost((void**)&mb, sizeof(Mailbox)) != cudaSuccess) mb = nullptr;
  return mb;
}

bm_status build_impl(const void* points, bm_dtype dtype, int64_t n, int32_t d, bm_metric metric,
                     double eps, cudaStream_t s, const bm_options* opts, bool host_in,
                     bm_cover** out) {
  using namespace bm;
  if (!out) return set_err(BM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!points) return set_err(BM_EINVAL, "points is NULL");
  if (n < 1) return set_err(BM_EINVAL, "n must be >= 1 (got %lld)", (long long)n);
  if (d < 1) return set_err(BM_EINVAL, "d must be >= 1 (got %d)", d);
  if (!(eps > 0.0) || !isfinite(eps)) return set_err(BM_EINVAL, "eps must be finite and > 0");
  if (n > 2147483646LL) return set_err(BM_EOVERFLOW, "n exceeds INT32_MAX-1");
  if (dtype != BM_F32 && dtype != BM_I8 && dtype != BM_U8)
    return set_err(BM_EUNSUPPORTED, "unsupported dtype %d", (int)dtype);
  if (metric != BM_L2 && metric != BM_L1 && metric != BM_COSINE)
    return set_err(BM_EUNSUPPORTED, "unsupported metric %d", (int)metric);
  if (dtype != BM_F32 && metric == BM_COSINE)
    return set_err(BM_EUNSUPPORTED, "cosine is supported for BM_F32 only");
  if (dtype != BM_F32 && d > 32768)
    return set_err(BM_EOVERFLOW, "integer path needs d <= 32768 for exact int32 arithmetic");
  bm_options o{};
  if (opts) {
    size_t sz = opts->struct_size > 0 && (size_t)opts->struct_size < sizeof o
                    ? (size_t)opts->struct_size : sizeof o;
    memcpy(&o, opts, sz);
  }
  if (o.tile != 0 && (o.tile < 32 || o.tile > kBigT || (o.tile % 32) != 0))
    return set_err(BM_EINVAL, "tile must be a multiple of 32 in [32, %d]", kBigT);
  const int64_t tie_cap = o.near_tie_cap > 0 ? o.near_tie_cap : 65536;
  if (o.select != BM_SELECT_GREEDY && o.select != BM_SELECT_FPS)
    return set_err(BM_EINVAL, "unknown landmark selection %d", o.select);
  const bool fps = o.select == BM_SELECT_FPS;
  if (fps && (o.fps_start < 0 || o.fps_start >= n))
    return set_err(BM_EINVAL, "fps_start must be in [0, n) (got %d)", o.fps_start);

  const int kind = dtype == BM_F32
                       ? (metric == BM_L2 ? K_L2F : (metric == BM_L1 ? K_L1F : K_COSF))
                       : (metric == BM_L2 ? K_L2I : K_L1I);
  const int nu_needed = dtype == BM_F32 ? (d + 1) / 2 : (d + 7) / 8;
  int nu = pick_nu(nu_needed);
  if (nu == 0) nu = nu_needed;
  const Thresh th = make_thresh(kind, d, eps);

  // Tensor-core membership contraction (tc.cu): Euclidean (Gram form) and
  // cosine (Gram of the normalised rows), K up to the configured atom counts.
  tc::TcPlan P{};
  P.kind = dtype == BM_F32 ? tc::TC_TF32 : (dtype == BM_U8 ? tc::TC_U8 : tc::TC_S8);
  P.cosine = metric == BM_COSINE ? 1 : 0;
  {
    const int esz = dtype == BM_F32 ? 4 : 1;
    P.row_bytes = tc_row_bytes(d, esz);
    P.k_elems = P.row_bytes / esz;
    P.katoms = (int)((P.row_bytes + 127) / 128);
  }
  // AUTO: tensor cores for Euclidean when the rows are wide or numerous
  // enough to fill the 128 x 256 tiles (measured: C2, d = 10, n = 1e5, is
  // faster on tcgen05; C1, n = 2e3, on CUDA cores)
  bool use_tc = (metric == BM_L2 || (metric == BM_COSINE && dtype == BM_F32)) &&
                tc::tc_supported(P.kind, P.katoms) &&
                (o.path == BM_PATH_TENSOR ||
                 (o.path == BM_PATH_AUTO && (d >= 32 || n >= 32768)));
  // L1 (fp32, d <= 16) on tensor cores: a signed int8
  // contraction of thermometer codes proves most pairs out, the rest pass the
  // 8-bit SAD bound and the fp64 decision; needs the 8-bit rows.  AUTO takes
  // it for n >= 65536 (C5 L1: contraction 0.91 s against 1.00 s for the
  // CUDA-core SAD pass, same box)
  const int l1t_B = (metric == BM_L1 && dtype == BM_F32) ? l1t_bytes_per_coord(d) : 0;
  const bool use_l1t = l1t_B > 0 && l1q_words(d) > 0 && !(o.flags & BM_FLAG_NO_L1_PREFILTER) &&
                       (o.path == BM_PATH_TENSOR || (o.path == BM_PATH_AUTO && n >= 65536));
  if (use_l1t) {
    use_tc = true;
    P.kind = tc::TC_S8;
    P.row_bytes = ((int64_t)d * l1t_B + 6 + 127) / 128 * 128;
    P.k_elems = P.row_bytes;
    P.katoms = (int)(P.row_bytes / 128);
  }
  if (o.path == BM_PATH_TENSOR && !use_tc)
    return set_err(BM_EUNSUPPORTED,
                   "tensor-core path supports L2 and cosine with d*elem <= %d bytes, "
                   "and fp32 L1 with d <= 16",
                   4096);

  int64_t launches = 0;
  Mailbox* mb = mailbox();
  if (!mb) return set_err(BM_ENOMEM, "pinned host mailbox allocation failed");
  Pool pool(s);
  Timer tm(o.timing != 0, s);
  Trace tr(s);
  tm.mark(0);

  // ---- A0 prep
  const void* dpoints = points;
  if (host_in) {
    size_t esz = dtype == BM_F32 ? 4 : 1;
    void* buf;
    TRY(pool.alloc((uint8_t**)&buf, (size_t)n * d * esz));
    CK(cudaMemcpyAsync(buf, points, (size_t)n * d * esz, cudaMemcpyHostToDevice, s));
    dpoints = buf;
  }
  uint2* rows = nullptr;
  uint2* xhat = nullptr;
  int32_t* inorm = nullptr;
  DevStats* stats = nullptr;
  tr("prep: start");
  TRY(pool.alloc(&rows, (size_t)n * nu));
  if (kind == K_COSF) TRY(pool.alloc(&xhat, (size_t)n * nu));
  if (kind == K_L2I) TRY(pool.alloc(&inorm, (size_t)n));
  TRY(pool.alloc(&stats, 1));
  CK(cudaMemsetAsync(stats, 0, sizeof(DevStats), s));
  tr("prep: allocs");
  CK(launch_prep(dpoints, dtype, n, d, kind, nu, rows, xhat, inorm, stats, s, &launches));
  tr("prep: launch");
  void* tc_nrm = nullptr;
  if (use_tc) {
    uint8_t* xop = nullptr;
    TRY(pool.alloc(&xop, (size_t)n * P.row_bytes));
    if (dtype == BM_F32) TRY(pool.alloc((double**)&tc_nrm, (size_t)n));
    else TRY(pool.alloc((int32_t**)&tc_nrm, (size_t)n));
    P.xop = xop;
    P.n_rows = n;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&P.num_sms, cudaDevAttrMultiProcessorCount, dev));
    if (!use_l1t) CK(tc::launch_tc_prep(dpoints, dtype, n, d, P, tc_nrm, stats, s, &launches));
  }
  // L1: 8-bit quantised rows for the membership prefilter (exact decisions unchanged)
  uint32_t* qrows = nullptr;
  double* qparam = nullptr;
  // (the tensor path reads whole 4-word rows: d <= 16 is zero padded to 4 words)
  const int nq = kind == K_L1F ? (use_l1t ? 4 : l1q_words(d)) : 0;
  if (nq > 0 && !(o.flags & BM_FLAG_NO_L1_PREFILTER)) {
    // (rows padded to a multiple of 128: the tensor path copies whole 128-row
    // blocks of them; the padding rows are never read as candidates)
    TRY(pool.alloc(&qrows, (size_t)((n + 127) / 128 * 128) * nq));
    TRY(pool.alloc(&qparam, 4));
    CK(launch_l1_quantize((const float*)dpoints, n, d, nq, qparam, qrows, s, &launches));
  }
  // ... and, on tensor cores, the thermometer operand over the same range
  if (use_l1t)
    CK(tc::launch_l1t_prep((const float*)dpoints, n, d, P, qparam, eps, (int32_t*)tc_nrm, s,
                           &launches));

  if (host_in) pool.free_now((void*)dpoints);

  // ---- tile-level pruning of the tensor-core membership (cells.cu): fp32
  // Euclidean, large n (the preparation costs ~1 ms at n = 1e6)
  const bool prune = use_tc && dtype == BM_F32 && metric == BM_L2 && P.katoms <= 2 &&
                     n >= 4 * kPruneCells && !(o.flags & BM_FLAG_NO_PRUNE) &&
                     (n >= 262144 || (o.flags & BM_FLAG_FORCE_PRUNE));
  // Greedy tile T (A11: the result does not depend on it).  Pruned tensor
  // launches (C3) take 8192 candidates: each tile's membership launch streams
  // the whole point operand from HBM once, so 8x fewer tiles move 8x fewer
  // bytes, and a row block meets ~8x more live landmarks per A load; A2 then
  // lists its non-zero words and k_resolve_big decides the sparse in-tile
  // graph in rounds.  Elsewhere 1024 (the single-CTA in-order resolve).
  const int T = o.tile > 0 ? o.tile : (prune ? kBigT : 1024);
  const bool big_tile = T > 1024;
  const int aw = (int)(((T + 255) / 256 + 3) / 4);   // live-chunk words per row block
  PruneState ps{};
  tc::TcPlan Pm{};   // the member kernel's plan: A operand in permuted order
  if (prune) {
    const int KWd = kPruneCells / 32;
    const int64_t nblk = (n + 127) / 128;
    TRY(pool.alloc(&ps.cell, (size_t)n));
    TRY(pool.alloc(&ps.rank, (size_t)kPruneCells));
    TRY(pool.alloc(&ps.pdist, (size_t)kPruneCells * kPruneCells));
    TRY(pool.alloc(&ps.perm, (size_t)n));
    TRY(pool.alloc(&ps.seg, (size_t)kPruneCells + 1));
    TRY(pool.alloc(&ps.center, (size_t)kPruneCells * d));
    TRY(pool.alloc(&ps.radius, (size_t)kPruneCells));
    TRY(pool.alloc(&ps.part, (size_t)kPruneCells * kPruneSplit * 128));
    TRY(pool.alloc(&ps.rad2, (size_t)kPruneCells));
    TRY(pool.alloc(&ps.near, (size_t)kPruneCells * KWd));
    TRY(pool.alloc(&ps.bmask, (size_t)nblk * KWd));
    TRY(pool.alloc(&ps.xop_perm, (size_t)n * P.row_bytes));
    TRY(pool.alloc(&ps.nrm_perm, (size_t)n));
    const int64_t Tq = ((T + 255) / 256) * 256;
    TRY(pool.alloc(&ps.col_pt, (size_t)Tq));
    TRY(pool.alloc(&ps.col_pos, (size_t)Tq));
    TRY(pool.alloc(&ps.cmask, (size_t)(Tq / 32) * KWd));
    TRY(pool.alloc(&ps.tmask, (size_t)(Tq / 256) * KWd));
    TRY(pool.alloc(&ps.act, (size_t)nblk * (aw + 1)));   // [live-tile mask, chunk words]
    unsigned long long *pk = nullptr, *pa = nullptr;
    void* ptemp = nullptr;
    TRY(pool.alloc(&pk, (size_t)n));
    TRY(pool.alloc(&pa, (size_t)n));
    TRY(pool.alloc((uint8_t**)&ptemp, radix_temp_bytes(n)));
    CK(prune_prepare((const float*)rows, 2 * nu, d, n, eps, (const uint8_t*)P.xop, P.row_bytes,
                     (const double*)tc_nrm, ps, ptemp, pk, pa, s, &launches));
    pool.free_now(pk);
    pool.free_now(pa);
    pool.free_now(ptemp);
    tr("prune prepare");
  }
  tr("prep");

  // ---- buffers of the fused greedy + membership loop
  const int64_t nL_max = n;  // L <= n
  int64_t key_cap = o.key_cap > 0 ? (int64_t)o.key_cap : initial_key_cap(n);
  const int adj_words = T / 32;
  int32_t *cnt = nullptr, *unc0 = nullptr, *unc1 = nullptr, *lm = nullptr, *new_lm = nullptr;
  uint32_t* adj = nullptr;
  uint8_t* covered = nullptr;
  unsigned long long* cstate = nullptr;
  unsigned long long* keys = nullptr;
  int64_t* ties_dev = nullptr;
  TRY(pool.alloc(&cnt, 8));  // [0],[1] n_unc ping-pong; [2] L; [3] dL; [4] compaction ticket
  TRY(pool.alloc(&unc0, (size_t)n));
  TRY(pool.alloc(&unc1, (size_t)n));
  TRY(pool.alloc(&lm, (size_t)nL_max));
  TRY(pool.alloc(&new_lm, (size_t)T));
  TRY(pool.alloc(&adj, (size_t)T * adj_words));
  TRY(pool.alloc(&covered, (size_t)n));
  TRY(pool.alloc(&cstate, (size_t)compact_state_words(n)));
  TRY(pool.alloc(&keys, (size_t)key_cap));
  TRY(pool.alloc(&ties_dev, (size_t)tie_cap * 3));
  AdjList nz{};   // A2's non-zero word list for k_resolve_big (big tiles only)
  if (big_tile) {
    TRY(pool.alloc(&nz.e, (size_t)kBigNzCap));
    TRY(pool.alloc(&nz.count, 1));
    nz.cap = (uint32_t)kBigNzCap;
    CK(cudaMemsetAsync(nz.count, 0, sizeof(uint32_t), s));
  }
  CK(cudaMemsetAsync(covered, 0, (size_t)n, s));
  CK(cudaMemsetAsync(cstate, 0, sizeof(unsigned long long) * compact_state_words(n), s));
  {
    int32_t init[8] = {(int32_t)n, 0, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(cnt, init, sizeof init, cudaMemcpyHostToDevice, s));
    k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(unc0, n);
    ++launches;
    CK(cudaGetLastError());
  }
  int32_t* uncb[2] = {unc0, unc1};
  const uint2* score_rows = kind == K_COSF ? xhat : rows;

  PairArgs base{};
  base.rows = score_rows;
  base.xrows = rows;
  base.inorm = inorm;
  base.n = n;
  base.nu = nu;
  base.d = d;
  base.th = th;
  base.stats = stats;
  base.qrows = qrows;   // (MODE_MEMBER with K_L1F only: the 8-bit prefilter)
  base.nq = nq;
  base.qparam = qparam;

  // tensor path: tile landmark operand [T_pad][row_bytes], column constants
  tc::TcArgs ta{};
  // A2 on tensor cores when the CUDA-core adjacency kernel would have to
  // re-read wide rows from memory (no register-resident width fits, e.g. C4)
  // (also for d >= 32: measured on C3, d = 64: 9.0 ms of A2 over 572 tiles on
  // tensor cores vs 12.0 ms on CUDA cores; C2, d = 10, is faster on CUDA cores)
  const bool tc_adj = use_tc && !use_l1t && (pick_nu(nu_needed) == 0 || d >= 32);
  tc::TcArgs ac{};      // A2 on tensor cores: candidate contraction
  tc::TcPlan Pc{};
  tc::RowParams rp{};
  double C2 = 0.0;
  double tau = 0.0;
  if (use_tc) {
    const int BN = tc::tc_bn_for(P.kind, P.katoms);
    const int RB = tc::tc_rows_for(P.kind, P.katoms);
    P.l_rows = ((T + BN - 1) / BN) * BN;
    P.n_pad = ((n + RB - 1) / RB) * RB;
    ta.n = n;
    ta.L = T;
    ta.ksteps = use_l1t ? (int)(((int64_t)d * l1t_B + 6 + 31) / 32)
                        : (int)(((int64_t)d * (dtype == BM_F32 ? 4 : 1) + 31) / 32);
    ta.lbits = 32;
    ta.l_count_dev = cnt + 3;
    ta.l_total_dev = cnt + 2;
    ta.covered = covered;
    TRY(pool.alloc((uint8_t**)&P.lop, (size_t)P.l_rows * P.row_bytes));
    if (P.kind == tc::TC_TF32) {
      float *rlo, *rhi, *ca, *cb;
      TRY(pool.alloc(&rlo, (size_t)P.n_pad));
      TRY(pool.alloc(&rhi, (size_t)P.n_pad));
      TRY(pool.alloc(&ca, (size_t)P.l_rows));
      TRY(pool.alloc(&cb, (size_t)P.l_rows));
      ta.row_lo = rlo;
      ta.row_hi = rhi;
      ta.col_a = ca;
      ta.col_b = cb;
      TRY(alloc_fold(pool, P, ta, s, &launches));
      C2 = tc_band_c2(ta.ksteps);
      tau = 1.0000005e-6 * th.eps2 + th.eps2 * ldexp(1.0, -21);
    } else if (!use_l1t) {   // (L1T: the row and column constants are folded into the operands)
      int32_t *rr, *cc;
      TRY(pool.alloc(&rr, (size_t)P.n_pad));
      TRY(pool.alloc(&cc, (size_t)P.l_rows));
      ta.row_r = rr;
      ta.col_c = cc;
    }
    if (P.cosine) CK(tc::launch_tc_rows_cos(P, tc_nrm, n, th.eps, tc_cos_margin(ta.ksteps), ta, s,
                                            &launches));
    else if (!use_l1t)
      CK(tc::launch_tc_rows(P, prune ? (const void*)ps.nrm_perm : tc_nrm, n, C2, th.eps2, tau,
                            th.lo_i, ta, s, &launches));
    ta.keys = keys;
    ta.key_count = &stats->key_count;
    ta.key_cap = key_cap;
    set_recheck(ta, rows, 2 * nu, d, th, prune ? ps.col_pt : new_lm, ties_dev, tie_cap, stats);
    if (use_l1t) {
      ta.l1t = 1;
      ta.qrows = qrows;
      ta.nq = nq;
      ta.qparam = qparam;
    }
    if (prune) {
      Pm = P;
      Pm.xop = ps.xop_perm;
      ta.row_pt = ps.perm;
      ta.col_pos = ps.col_pos;
      ta.act = ps.act;
      ta.act_bmask = ps.bmask;
      ta.act_cmask = ps.cmask;
      ta.act_tmask = ps.tmask;
      ta.act_words = aw;
    }
  }
  if (tc_adj) {
    // A2 on tensor cores: the tile's candidates x themselves (adjacency epilogue)
    rp.tf32 = P.kind == tc::TC_TF32;
    rp.cosine = P.cosine;
    rp.C2 = C2;
    rp.eps = th.eps;
    rp.eps2 = th.eps2;
    rp.tau = tau;
    rp.m = tc_cos_margin(ta.ksteps);
    rp.lo_i = th.lo_i;
    const int64_t Tp = ((T + 255) / 256) * 256;
    Pc = P;
    Pc.n_rows = Tp;
    Pc.l_rows = Tp;
    Pc.n_pad = Tp;
    uint8_t* cop = nullptr;
    TRY(pool.alloc(&cop, (size_t)Tp * P.row_bytes));
    Pc.xop = cop;
    Pc.lop = cop;
    ac.n = Tp;
    ac.L = T;
    ac.ksteps = ta.ksteps;
    ac.adj = adj;
    ac.adj_T = T;
    ac.nz = nz;
    if (rp.tf32) {
      float *rlo, *rhi, *ca, *cb, *colk;
      TRY(pool.alloc(&rlo, (size_t)Tp));
      TRY(pool.alloc(&rhi, (size_t)Tp));
      TRY(pool.alloc(&ca, (size_t)Tp));
      TRY(pool.alloc(&cb, (size_t)Tp));
      TRY(pool.alloc(&colk, (size_t)Tp * 8));
      ac.row_lo = rlo;
      ac.row_hi = rhi;
      ac.col_a = ca;
      ac.col_b = cb;
      ac.colk = colk;
    } else {
      int32_t *rr, *cc;
      TRY(pool.alloc(&rr, (size_t)Tp));
      TRY(pool.alloc(&cc, (size_t)Tp));
      ac.row_r = rr;
      ac.col_c = cc;
    }
    set_recheck(ac, rows, 2 * nu, d, th, nullptr, nullptr, 0, stats);
  }
  tm.mark(1);
  tr("greedy buffers");

  // ---- A1-A4 + B: blocked greedy, each tile's membership pass over all points
  // (SURVEY §3 (iii) variant: total membership work is exactly n * L).
  std::vector<cudaEvent_t> mev;   // per-tile membership kernel brackets (timing only)
  auto mark_member = [&](void) -> cudaError_t {
    if (!tm.on) return cudaSuccess;
    cudaEvent_t e = cached_event(BM_NUM_STEPS + mev.size());
    if (!e) return cudaErrorMemoryAllocation;
    mev.push_back(e);
    return cudaEventRecord(e, s);
  };

  // tiles are issued in batches between host termination checks (a tile after
  // the last one costs a few empty launches; a check costs a round trip)
  // BM_LOOP_PROFILE=1 (diagnostics): per-phase device time of the tile loop
  // (A2 / A3 / B incl. landmark operands / A4), printed to stderr
  static const bool loop_prof = getenv("BM_LOOP_PROFILE") != nullptr;
  unsigned long long* tc_trace = nullptr;   // BM_TC_TRACE=1: stamp every membership launch
  if (use_tc && getenv("BM_TC_TRACE"))
    TRY(pool.alloc(&tc_trace, (size_t)P.num_sms * 16 + 512 * 5));
  const bool tc_wmode = tc_trace && atoi(getenv("BM_TC_TRACE")) >= 2;
  const bool tc_tline = tc_trace && atoi(getenv("BM_TC_TRACE")) == 3;
  std::vector<std::pair<int, cudaEvent_t>> lev;
  auto loop_mark = [&](int phase) {
    if (!loop_prof) return;
    cudaEvent_t e = cached_event(4096 + lev.size());
    if (e && cudaEventRecord(e, s) == cudaSuccess) lev.emplace_back(phase, e);
  };
  int64_t tile = 0;
  // tiles per host check: 3 first (the C2-size covers finish in three), then
  // the remaining count predicted from the rate at which the uncovered list
  // has been shrinking (each check costs a round trip, each tile after the
  // last one a few empty launches)
  int batch = 3;
  int64_t unc_start = n;
  int nonfinite_checked = 0;
  if (fps) {
    // NEXT-2: farthest point sampling selects the landmarks (fps.cu), then one
    // membership pass of all points against the ascending landmark list
    CK(cudaStreamSynchronize(s));
    int nf = 0;
    CK(cudaMemcpy(&nf, &stats->nonfinite, sizeof nf, cudaMemcpyDeviceToHost));
    if (nf) return set_err(BM_EINVAL, "points contain a non-finite coordinate");
    const int g = fps_max_candidates();
    double *mind = nullptr, *cval = nullptr;
    int64_t* cidx = nullptr;
    int32_t* seq = nullptr;
    TRY(pool.alloc(&mind, (size_t)n));
    TRY(pool.alloc(&seq, (size_t)n));
    TRY(pool.alloc(&cval, (size_t)2 * g));
    TRY(pool.alloc(&cidx, (size_t)2 * g));
    const double thr = metric == BM_L2 ? eps * eps : eps;
    // float L2 / L1: points in spatial (cell) order so that each warp of the
    // selection kernel can skip the landmarks that cannot lower its minima
    int32_t* fperm = nullptr;
    if ((kind == K_L2F || kind == K_L1F) && d <= 128 && n >= 4 * kPruneCells &&
        !(o.flags & BM_FLAG_NO_PRUNE)) {
      int32_t *fcell = nullptr, *frank = nullptr;
      float* fpd = nullptr;
      unsigned long long *fk = nullptr, *fa = nullptr;
      void* ftemp = nullptr;
      TRY(pool.alloc(&fperm, (size_t)n));
      TRY(pool.alloc(&fcell, (size_t)n));
      TRY(pool.alloc(&frank, (size_t)kPruneCells));
      TRY(pool.alloc(&fpd, (size_t)kPruneCells * kPruneCells));
      TRY(pool.alloc(&fk, (size_t)n));
      TRY(pool.alloc(&fa, (size_t)n));
      TRY(pool.alloc((uint8_t**)&ftemp, radix_temp_bytes(n)));
      CK(cell_order((const float*)rows, 2 * nu, d, n, fcell, frank, fpd, &fk, &fa, ftemp, fperm, s,
                    &launches));
    }
    tm.mark(6);
    CK(launch_fps(rows, inorm, nu, d, kind, n, thr, o.fps_start, mind, seq, cnt + 2, cval, cidx,
                  fperm, s));
    tm.mark(7);
    ++launches;
    int32_t hl = 0;
    CK(cudaMemcpyAsync(&hl, cnt + 2, sizeof hl, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    unsigned long long *lk = nullptr, *lalt = nullptr;
    void* temp = nullptr;
    TRY(pool.alloc(&lk, (size_t)hl));
    TRY(pool.alloc(&lalt, (size_t)hl));
    TRY(pool.alloc((uint8_t**)&temp, radix_temp_bytes(hl)));
    CK(launch_fps_keys(seq, hl, lk, s, &launches));
    const BitRange r[1] = {{0, bits_for(n > 1 ? n - 1 : 1)}};
    CK(radix_sort_u64(&lk, &lalt, hl, r, 1, temp, s, &launches));
    CK(launch_unpack_low(lk, hl, 0xffffffffull, lm, s, &launches));
    int64_t Mf = 0;
    CK(mark_member());
    TRY(membership_full(pool, kind, base, P, use_tc && !use_l1t, tc_nrm, lm, hl, n, d, dtype, nu, th, C2,
                        keys, key_cap, ties_dev, tie_cap, stats, s, &launches, &Mf));
    CK(mark_member());
    if (Mf > key_cap) {
      pool.free_now(keys);
      key_cap = Mf;
      TRY(pool.alloc(&keys, (size_t)key_cap));
      TRY(membership_full(pool, kind, base, P, use_tc && !use_l1t, tc_nrm, lm, hl, n, d, dtype, nu, th, C2,
                          keys, key_cap, ties_dev, tie_cap, stats, s, &launches, &Mf));
      if (Mf > key_cap) return set_err(BM_ECUDA, "membership recount exceeded its exact size");
    }
  }
  for (; !fps;) {
    for (int b = 0; b < batch; ++b, ++tile) {
      const int cur = (int)(tile & 1), nxt = cur ^ 1;
      loop_mark(0);
      // A2: adjacency among the candidates unc[0 .. nc)
      PairArgs a = base;
      a.qidx = uncb[cur];
      a.q_begin = 0;
      a.q_end = T;
      a.q_end_dev = cnt + cur;
      a.lidx = uncb[cur];
      a.l_begin = 0;
      a.l_end = T;
      a.l_end_dev = cnt + cur;
      a.adj = adj;
      a.adj_words = adj_words;
      a.nz = nz;
      if (tc_adj) {
        ac.l_count_dev = cnt + cur;
        ac.lm_idx = uncb[cur];
        CK(tc::launch_tc_tile_cand(P, Pc, tc_nrm, uncb[cur], cnt + cur, T, C2, rp, ac, s,
                                   &launches));
        CK(tc::launch_tc_adj(Pc, ac, s, &launches));
      } else {
        CK(launch_pairs(kind, MODE_ADJ, a, T, s, &launches));
      }
      loop_mark(1);
      // A3: in-order resolve, append landmarks (resets the tile's counters)
      {
        const PruneTile pt = prune ? PruneTile{ps.cell, ps.rank, ps.col_pt, ps.col_pos, ps.cmask,
                                               ps.tmask}
                                   : PruneTile{};
        if (big_tile)
          CK(launch_resolve_big(adj, nz, uncb[cur], cnt + cur, T, lm, cnt + 2, new_lm, cnt + 3,
                                stats, cnt + 4, nullptr, s, &launches, pt,
                                (o.flags & BM_FLAG_DENSE_RESOLVE) ? 1 : 0));
        else
          CK(launch_resolve(adj, adj_words, uncb[cur], cnt + cur, T, lm, cnt + 2, new_lm,
                            cnt + 3, stats, cnt + 4, nullptr, s, &launches, pt));
      }
      loop_mark(2);
      // B (+A4 marks): membership of every point in the new balls
      if (use_tc) {
        if (use_l1t)
          CK(tc::launch_l1t_tile_landmarks(P, (const int32_t*)tc_nrm, new_lm, cnt + 3, d, s,
                                           &launches));
        else
          CK(tc::launch_tc_tile_landmarks(P, tc_nrm, prune ? ps.col_pt : new_lm, cnt + 3, C2, ta,
                                          s, &launches));
        CK(mark_member());
        if (tc_trace) {   // diagnostics: phase stamps of this launch (synchronises)
          CK(cudaMemsetAsync(tc_trace, 0, sizeof(unsigned long long) * (P.num_sms * 16 + 512 * 5), s));
          if (tc_wmode) ta.wtrace = tc_trace;
          else ta.trace = tc_trace;
          if (tc_tline) ta.tline = tc_trace + P.num_sms * 16;
        }
        CK(tc::launch_tc(prune ? Pm : P, ta, s, &launches));
        CK(mark_member());
        if (tc_trace) {
          char tag[64];
          snprintf(tag, sizeof tag, "membership tile %lld", (long long)tile);
          if (tc_wmode) CK(print_tc_wtrace(tc_trace, P.num_sms, tag, s));
          else CK(print_tc_trace(tc_trace, P.num_sms, tag, s));
          if (tc_tline) CK(print_tc_tline(tc_trace + P.num_sms * 16, tag, s));
          ta.trace = nullptr;
          ta.wtrace = nullptr;
          ta.tline = nullptr;
        }
      } else {
        PairArgs m = base;
        m.qidx = nullptr;
        m.q_begin = 0;
        m.q_end = n;
        m.lidx = new_lm;
        m.l_begin = 0;
        m.l_end = T;
        m.l_end_dev = cnt + 3;
        m.l_total_dev = cnt + 2;
        m.keys = keys;
        m.key_cap = key_cap;
        m.lbits = 32;
        m.ties = ties_dev;
        m.tie_cap = tie_cap;
        m.covered = covered;
        m.qrows = qrows;
        m.nq = nq;
        m.qparam = qparam;
        CK(mark_member());
        CK(launch_pairs(kind, MODE_MEMBER, m, n, s, &launches));
        CK(mark_member());
      }
      loop_mark(3);
      // A4: keep the still-uncovered points after the tile, in order
      CK(launch_compact_unc(covered, uncb[cur], cnt + cur, T, uncb[nxt], cnt + nxt, cstate,
                            cnt + 4, (uint32_t)(tile + 1), n, s, &launches));
      loop_mark(4);
    }
    // one round trip: the counters and the statistics together
    CK(cudaMemcpyAsync(mb->hc, cnt, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&mb->hs, stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!nonfinite_checked) {
      if (mb->hs.nonfinite) return set_err(BM_EINVAL, "points contain a non-finite coordinate");
      nonfinite_checked = 1;
    }
    const int64_t unc_now = mb->hc[tile & 1];
    if (unc_now == 0) break;
    const double per_tile = (double)(unc_start - unc_now) / (double)tile;
    int64_t est = per_tile > 0.0 ? (int64_t)ceil((double)unc_now / per_tile) : 2 * batch;
    batch = (int)std::min<int64_t>(64, std::max<int64_t>(1, std::min<int64_t>(est, 2 * batch)));
  }
  tm.mark(2);
  tr("greedy+membership loop");
  if (loop_prof && !lev.empty()) {
    cudaEventSynchronize(lev.back().second);
    double acc[5] = {0, 0, 0, 0, 0};
    for (size_t i = 0; i + 1 < lev.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, lev[i].second, lev[i + 1].second);
      acc[lev[i].first] += t;
    }
    fprintf(stderr, "loop profile (ms): tiles %lld  A2 %.4f  A3 %.4f  B %.4f  A4 %.4f  gaps %.4f\n",
            (long long)tile, acc[0], acc[1], acc[2], acc[3], acc[4]);
  }

  DevStats hs{};
  int32_t hL = 0;
  if (fps) {
    CK(cudaMemcpyAsync(&mb->hs, stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(mb->hc, cnt, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  // (greedy: the loop's last check read both after all of its work)
  hs = mb->hs;
  hL = mb->hc[2];
  const int64_t L = hL;
  pool.free_now(unc0);
  pool.free_now(unc1);
  pool.free_now(covered);
  pool.free_now(cstate);

  // ---- B fallback: the key buffer overflowed; recompute the membership alone
  // with the exact capacity (the greedy's coverage decisions were unaffected)
  const int lbits = bits_for(L > 1 ? L - 1 : 1);
  const int pbits = bits_for(n > 1 ? n - 1 : 1);
  int64_t M = (int64_t)hs.key_count;
  if (M > key_cap) {
    pool.free_now(keys);
    key_cap = M;
    TRY(pool.alloc(&keys, (size_t)key_cap));
    TRY(membership_full(pool, kind, base, P, use_tc && !use_l1t, tc_nrm, lm, L, n, d, dtype, nu, th, C2,
                        keys, key_cap, ties_dev, tie_cap, stats, s, &launches, &M));
    if (M > key_cap) return set_err(BM_ECUDA, "membership recount exceeded its exact size");
    CK(cudaMemcpyAsync(&hs, stats, sizeof hs, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  tm.mark(3);

  // ---- C CSR both ways.  keys = point << 32 | landmark position: a stable
  // sort on the position bits and then the point bits gives the point-major
  // order; a further stable sort on the position bits alone gives the
  // landmark-major order with the points of each ball still ascending.
  // (n * L <= 2^30: both CSRs from two bit matrices instead, no sort)
  int64_t* pt_ptr = nullptr;
  int32_t* pt_lm = nullptr;
  int64_t* ball_ptr = nullptr;
  int32_t* ball_idx = nullptr;
  TRY(pool.alloc(&pt_ptr, (size_t)n + 1));
  TRY(pool.alloc(&pt_lm, (size_t)(M > 0 ? M : 1)));
  TRY(pool.alloc(&ball_ptr, (size_t)L + 1));
  TRY(pool.alloc(&ball_idx, (size_t)(M > 0 ? M : 1)));
  if (n * L <= kCsrBitmapMaxBits) {
    uint32_t* cbits = nullptr;
    void* ctemp = nullptr;
    TRY(pool.alloc(&cbits, (size_t)csr_bitmap_words(n, L)));
    TRY(pool.alloc((uint8_t**)&ctemp, csr_bitmap_temp_bytes(n, L)));
    tr("csr alloc");
    CK(csr_from_keys_bitmap(keys, M, n, L, cbits, ctemp, pt_ptr, pt_lm, ball_ptr, ball_idx, s,
                            &launches));
    pool.free_now(cbits);
    pool.free_now(ctemp);
    pool.free_now(keys);
  } else {
    unsigned long long* alt = nullptr;
    void* rtemp = nullptr;
    TRY(pool.alloc(&alt, (size_t)(M > 0 ? M : 1)));
    TRY(pool.alloc((uint8_t**)&rtemp, radix_temp_bytes(M)));
    const unsigned long long lo32 = 0xffffffffull;
    const BitRange pm[2] = {{0, lbits}, {32, 32 + pbits}};
    const BitRange lmaj[1] = {{0, lbits}};
    tr("csr alloc");
    CK(radix_sort_u64(&keys, &alt, M, pm, 2, rtemp, s, &launches));
    tr("csr sort point-major");
    CK(launch_unpack_low(keys, M, lo32, pt_lm, s, &launches));
    CK(launch_segment_ptr(keys, M, 32, lo32, n, pt_ptr, s, &launches));
    CK(radix_sort_u64(&keys, &alt, M, lmaj, 1, rtemp, s, &launches));
    CK(launch_unpack_high(keys, M, ball_idx, s, &launches));
    CK(launch_segment_ptr(keys, M, 0, lo32, L, ball_ptr, s, &launches));
    pool.free_now(keys);
    pool.free_now(alt);
    pool.free_now(rtemp);
  }
  tm.mark(4);
  tr("csr rest");

  // host-buffer API: landmarks and both CSRs go back on a side stream while
  // the edges are built (one pinned block; the edges follow at the end)
  uint8_t* hblk = nullptr;
  size_t hcls = 0, hoff[5] = {0, 0, 0, 0, 0};
  cudaStream_t s2 = nullptr;
  // on any early return: let the side-stream copies finish before the pool
  // releases the device arrays, and give the pinned block back
  struct SideGuard {
    cudaStream_t& st;
    uint8_t*& blk;
    size_t& cls;
    ~SideGuard() {
      if (st) cudaStreamSynchronize(st);
      if (blk) g_pinned.put(blk, cls);
    }
  } side_guard{s2, hblk, hcls};
  if (host_in) {
    const size_t hsz[5] = {sizeof(int32_t) * (size_t)L, sizeof(int64_t) * (size_t)(L + 1),
                           sizeof(int32_t) * (size_t)M, sizeof(int64_t) * (size_t)(n + 1),
                           sizeof(int32_t) * (size_t)M};
    const void* hsrc[5] = {lm, ball_ptr, ball_idx, pt_ptr, pt_lm};
    size_t total = 0;
    for (int i = 0; i < 5; ++i) {
      hoff[i] = total;
      total += (hsz[i] + 255) & ~(size_t)255;
    }
    hblk = (uint8_t*)g_pinned.get(total, &hcls);
    if (!hblk) return set_err(BM_ENOMEM, "pinned host allocation for the results failed");
    s2 = side_stream();
    cudaEvent_t ev = cached_event(8100);
    if (!s2 || !ev) return set_err(BM_ECUDA, "side stream / event creation failed");
    CK(cudaEventRecord(ev, s));
    CK(cudaStreamWaitEvent(s2, ev, 0));
    for (int i = 0; i < 5; ++i)
      if (hsz[i]) CK(cudaMemcpyAsync(hblk + hoff[i], hsrc[i], hsz[i], cudaMemcpyDeviceToHost, s2));
  }

  // ---- D1-D3 edges (edges.cu)
  int64_t NP = 0;  // P = sum_p C(t_p, 2) witnessed pairs
  int64_t E = 0;
  int32_t* edges = nullptr;
  int64_t* ptot = nullptr;
  bool pe_pending = false;
  TRY(pool.alloc(&ptot, 2));
  if (L >= 2 && L <= kEdgeBitmapMaxL) {
    // L x L bit matrix: no pair buffer, no sort; one host sync for (P, E)
    uint32_t* bits = nullptr;
    void* etemp = nullptr;
    const int64_t cap = L * (L - 1) / 2;
    TRY(pool.alloc(&bits, (size_t)edge_bitmap_words(L)));
    TRY(pool.alloc((uint8_t**)&etemp, edge_lb_temp_bytes(edge_bitmap_words(L))));
    TRY(pool.alloc(&edges, (size_t)(2 * cap)));
    CK(launch_edge_bits(pt_ptr, pt_lm, n, L, bits, (unsigned long long*)ptot, s, &launches));
    tr("edges: bits");
    CK(launch_bits_compact(bits, L, edges, cap, ptot + 1, etemp, s, &launches));
    // (P, E) arrive with the final synchronisation (edges holds the full capacity)
    CK(cudaMemcpyAsync(mb->pe, ptot, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, s));
    pe_pending = true;
    pool.free_now(bits);
    pool.free_now(etemp);
  } else if (L >= 2 && !(o.flags & (BM_FLAG_EDGE_POINT_PAIRS | BM_FLAG_EDGE_ROWS)) &&
             ((o.flags & BM_FLAG_EDGE_TRIANGLE) || 4.0 * (double)tri_bitmap_words(L) <= kTriAutoBytes) &&
             use_tri_bitmap(L, o.flags)) {
    // strictly-upper bit triangle: no pair buffer, no sort (edges.cu)
    uint32_t* bits = nullptr;
    int64_t *rcnt = nullptr, *roff = nullptr;
    void* stemp = nullptr;
    TRY(pool.alloc(&bits, (size_t)tri_bitmap_words(L)));
    TRY(pool.alloc(&rcnt, (size_t)L));
    TRY(pool.alloc(&roff, (size_t)L));
    TRY(pool.alloc((uint8_t**)&stemp, scan_temp_bytes(L)));
    CK(launch_tri_bits(pt_ptr, pt_lm, n, L, bits, (unsigned long long*)ptot, s, &launches));
    CK(launch_tri_rowcount(bits, L, rcnt, s, &launches));
    CK(exclusive_scan_i64(rcnt, roff, L, stemp, ptot + 1, s, &launches));
    int64_t h2[2];
    CK(cudaMemcpyAsync(h2, ptot, sizeof h2, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    NP = h2[0];
    E = h2[1];
    TRY(pool.alloc(&edges, (size_t)(2 * E > 0 ? 2 * E : 1)));
    if (E > 0) CK(launch_tri_emit(bits, L, roff, edges, s, &launches));
    tr("edges: triangle");
    pool.free_now(bits);
    pool.free_now(rcnt);
    pool.free_now(roff);
    pool.free_now(stemp);
  } else if (L >= 2) {
    // D1 -> D2 radix sort -> D3 unique.  D1 is the row-union emission
    // (deduplicated per ball row item) when the points' landmark rows repeat
    // their pairs enough for it to pay (P >= kRowsMinPairs L: C5), else the
    // per-point emission of every witnessed pair (C3)
    int64_t *pcnt = nullptr, *poff = nullptr, *icnt = nullptr, *ioff = nullptr;
    void* stemp = nullptr;
    TRY(pool.alloc(&pcnt, (size_t)n));
    TRY(pool.alloc(&poff, (size_t)n));
    TRY(pool.alloc((uint8_t**)&stemp, scan_temp_bytes(n > L ? n : L)));
    CK(launch_pair_counts(pt_ptr, n, pcnt, s, &launches));
    CK(exclusive_scan_i64(pcnt, poff, n, stemp, ptot, s, &launches));
    CK(cudaMemcpyAsync(&NP, ptot, sizeof NP, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    tr("edges count");
    const bool rows = !(o.flags & BM_FLAG_EDGE_POINT_PAIRS) &&
                      ((o.flags & BM_FLAG_EDGE_ROWS) || NP >= kRowsMinPairs * L);
    unsigned long long* kc = nullptr;   // [0] keys emitted, [1] pairs met
    int64_t n_items = 0;
    if (rows && NP > 0) {
      TRY(pool.alloc(&icnt, (size_t)L));
      TRY(pool.alloc(&ioff, (size_t)L));
      TRY(pool.alloc(&kc, 2));
      CK(cudaMemsetAsync(kc, 0, 2 * sizeof(unsigned long long), s));
      CK(launch_row_items(ball_ptr, L, icnt, s, &launches));
      CK(exclusive_scan_i64(icnt, ioff, L, stemp, ptot + 1, s, &launches));
      CK(cudaMemcpyAsync(&n_items, ptot + 1, sizeof n_items, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    if (rows) {
      if (NP > 0) {
        unsigned long long *ek = nullptr, *ea = nullptr;
        int32_t* irow = nullptr;
        TRY(pool.alloc(&irow, (size_t)n_items));
        CK(launch_item_rows(ioff, icnt, L, irow, s, &launches));
        TRY(pool.alloc(&ek, (size_t)NP));   // at most one key per witnessed pair
        CK(launch_row_pairs(ball_ptr, ball_idx, pt_ptr, pt_lm, n, L, ioff, irow, n_items, lbits, ek,
                            NP, kc, kc + 1, s, &launches));
        int64_t NK = 0, NV = 0;
        CK(cudaMemcpyAsync(&NK, kc, sizeof NK, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&NV, kc + 1, sizeof NV, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (getenv("BM_ROWS_TRACE"))
          fprintf(stderr, "rows: L %lld M %lld items %lld pairs %lld visits %lld keys %lld\n",
                  (long long)L, (long long)M, (long long)n_items, (long long)NP, (long long)NV,
                  (long long)NK);
        tr("edges: row pairs");
        if (NK > NP || NV != NP)
          return set_err(BM_ECUDA, "row-union edge emission: %lld keys / %lld pairs met for %lld pairs",
                         (long long)NK, (long long)NV, (long long)NP);
        void *et = nullptr, *ct = nullptr;
        TRY(pool.alloc(&ea, (size_t)(NK > 0 ? NK : 1)));
        TRY(pool.alloc((uint8_t**)&et, radix_temp_bytes(NK)));
        const BitRange er[1] = {{0, 2 * lbits}};
        CK(radix_sort_u64(&ek, &ea, NK, er, 1, et, s, &launches));
        pool.free_now(et);
        // (2 NK int32 fit the sort's spare buffer of NK keys)
        int32_t* etmp = (int32_t*)ea;
        TRY(pool.alloc((uint8_t**)&ct, edge_lb_temp_bytes(NK)));
        CK(launch_unique_compact(ek, NK, lbits, etmp, ptot + 1, ct, s, &launches));
        CK(cudaMemcpyAsync(&E, ptot + 1, sizeof E, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        TRY(pool.alloc(&edges, (size_t)(2 * E > 0 ? 2 * E : 1)));
        if (E > 0)
          CK(cudaMemcpyAsync(edges, etmp, sizeof(int32_t) * 2 * E, cudaMemcpyDeviceToDevice, s));
        tr("edges: rows sorted, unique");
        pool.free_now(ek);
        pool.free_now(ea);
        pool.free_now(ct);
        pool.free_now(irow);
      }
    } else {
      if (NP > 0) {
        unsigned long long *ek = nullptr, *ea = nullptr;
        int32_t* etmp = nullptr;
        void *et = nullptr, *ct = nullptr;
        TRY(pool.alloc(&ek, (size_t)NP));
        TRY(pool.alloc(&ea, (size_t)NP));
        TRY(pool.alloc((uint8_t**)&et, radix_temp_bytes(NP)));
        tr("edges alloc");
        CK(launch_pair_emit(pt_ptr, pt_lm, n, poff, lbits, ek, s, &launches));
        tr("edges emit");
        const BitRange er[1] = {{0, 2 * lbits}};
        CK(radix_sort_u64(&ek, &ea, NP, er, 1, et, s, &launches));
        tr("edges sort");
        pool.free_now(et);
        etmp = (int32_t*)ea;   // the sort's spare buffer holds 2 NP int32
        TRY(pool.alloc((uint8_t**)&ct, edge_lb_temp_bytes(NP)));
        CK(launch_unique_compact(ek, NP, lbits, etmp, ptot + 1, ct, s, &launches));
        tr("edges: compact launched");
        CK(cudaMemcpyAsync(&E, ptot + 1, sizeof E, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        tr("edges: E readback");
        TRY(pool.alloc(&edges, (size_t)(2 * E > 0 ? 2 * E : 1)));
        tr("edges: alloc exact");
        if (E > 0)
          CK(cudaMemcpyAsync(edges, etmp, sizeof(int32_t) * 2 * E, cudaMemcpyDeviceToDevice, s));
        tr("edges: copy");
        pool.free_now(ek);
        tr("edges: free ek");
        pool.free_now(ea);
        tr("edges: free ea");
        pool.free_now(ct);
      }
    }
    pool.free_now(pcnt);
    pool.free_now(poff);
    pool.free_now(stemp);
    if (icnt) pool.free_now(icnt);
    if (ioff) pool.free_now(ioff);
    if (kc) pool.free_now(kc);
    tr("edges: frees");
  }
  if (!edges) TRY(pool.alloc(&edges, 1));
  int32_t* landmarks = nullptr;
  TRY(pool.alloc(&landmarks, (size_t)(L > 0 ? L : 1)));
  tr("landmarks alloc");
  CK(launch_copy_i32(lm, landmarks, L, s, &launches));
  tm.mark(5);
  tr("edges rest");

  // ---- results (the first near ties ride along with the final synchronisation)
  CK(cudaMemcpyAsync(&mb->hs_end, stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(mb->ties, ties_dev, sizeof(int64_t) * 3 * std::min<int64_t>(tie_cap, 1024),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  hs = mb->hs_end;
  if (pe_pending) {
    NP = mb->pe[0];
    E = mb->pe[1];
  }
  bm_cover* c = (bm_cover*)calloc(1, sizeof(bm_cover));
  Priv* pv = (Priv*)calloc(1, sizeof(Priv));
  if (!c || !pv) {
    free(c);
    free(pv);
    return set_err(BM_ENOMEM, "host allocation failed");
  }
  pv->stream = s;
  c->priv = pv;
  c->n = n;
  c->d = d;
  c->dtype = dtype;
  c->metric = metric;
  c->eps = eps;
  c->n_landmarks = L;
  c->n_members = M;
  c->n_edges = E;
  c->n_witness_pairs = NP;
  c->n_pair_evals = n * L;
  c->n_greedy_evals = (int64_t)hs.greedy_evals;
  c->n_band_pairs = (int64_t)hs.band_pairs;
  c->n_near_ties = (int64_t)hs.near_ties;
  c->n_greedy_tiles = (int64_t)hs.tiles;
  c->n_tc_tiles_run = (int64_t)hs.tc_tiles_run;
  c->n_tc_tiles_skipped = (int64_t)hs.tc_tiles_skip;
  c->n_tc_chunks_run = (int64_t)hs.tc_chunks_run;
  c->n_tc_chunks_skipped = (int64_t)hs.tc_chunks_skip;
  c->path_used = use_tc ? BM_PATH_TENSOR : BM_PATH_CUDA_CORE;
  c->tile_used = T;
  const int64_t nst = c->n_near_ties < tie_cap ? c->n_near_ties : tie_cap;
  c->n_near_ties_stored = nst;
  if (nst > 0) {
    c->near_tie_pairs = (int64_t*)malloc(sizeof(int64_t) * 3 * nst);
    if (c->near_tie_pairs) {
      if (nst <= 1024) memcpy(c->near_tie_pairs, mb->ties, sizeof(int64_t) * 3 * nst);
      else CK(cudaMemcpy(c->near_tie_pairs, ties_dev, sizeof(int64_t) * 3 * nst,
                         cudaMemcpyDeviceToHost));
    }
  }
  if (tm.on) {
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&c->step_ms[i], tm.ev[i], tm.ev[i + 1]);
    cudaEventElapsedTime(&c->step_ms[BM_STEP_TOTAL], tm.ev[0], tm.ev[5]);
    float km = 0.f;
    for (size_t i = 0; i + 1 < mev.size(); i += 2) {
      float t = 0.f;
      cudaEventElapsedTime(&t, mev[i], mev[i + 1]);
      km += t;
    }
    c->step_ms[BM_STEP_MEMBER_KERNEL] = km;
    if (fps) cudaEventElapsedTime(&c->step_ms[BM_STEP_SELECT], tm.ev[6], tm.ev[7]);
  }
  c->n_member_launches = (int64_t)(mev.size() / 2);
  c->n_launches = launches;
  if (host_in) {
    c->on_host = 1;
    pv->pinned = hblk;
    pv->pinned_cls = hcls;
    c->landmarks = (int32_t*)(hblk + hoff[0]);
    c->ball_ptr = (int64_t*)(hblk + hoff[1]);
    c->ball_idx = (int32_t*)(hblk + hoff[2]);
    c->pt_ptr = (int64_t*)(hblk + hoff[3]);
    c->pt_lm = (int32_t*)(hblk + hoff[4]);
    hblk = nullptr;   // owned by the cover now
    // the edge list (its size is known now), then both streams
    const size_t esz = sizeof(int32_t) * 2 * (size_t)E;
    uint8_t* eblk = (uint8_t*)g_pinned.get(esz, &pv->pinned_e_cls);
    pv->pinned_e = eblk;
    if (!eblk) {
      // the side stream may still be copying into the block the cover now
      // owns: let it finish before bm_free hands the block back to the cache
      cudaStreamSynchronize(s2);
      bm_free(c);
      return set_err(BM_ENOMEM, "pinned host allocation for the results failed");
    }
    c->edges = (int32_t*)eblk;
    if (esz) CK(cudaMemcpyAsync(eblk, edges, esz, cudaMemcpyDeviceToHost, s));
    cudaError_t e = cudaStreamSynchronize(s);
    const cudaError_t e2 = cudaStreamSynchronize(s2);
    if (e == cudaSuccess) e = e2;
    if (e != cudaSuccess) {
      bm_free(c);
      return set_err(BM_ECUDA, "device-to-host copy of the results failed");
    }
  } else {
    c->landmarks = landmarks;
    c->ball_ptr = ball_ptr;
    c->ball_idx = ball_idx;
    c->pt_ptr = pt_ptr;
    c->pt_lm = pt_lm;
    c->edges = edges;
    for (void* p : {(void*)landmarks, (void*)ball_ptr, (void*)ball_idx, (void*)pt_ptr,
                    (void*)pt_lm, (void*)edges})
      pool.release(p);
  }
  *out = c;
  g_err.clear();
  return BM_OK;
}

}  // namespace

extern "C" {

bm_status bm_cover_build_ex(const void* points, bm_dtype dtype, int64_t n, int32_t d,
                            bm_metric metric, double eps, void* stream, const bm_options* opts,
                            bm_cover** out) {
  try {
    return build_impl(points, dtype, n, d, metric, eps, (cudaStream_t)stream, opts, false, out);
  } catch (...) {
    return set_err(BM_ENOMEM, "unexpected host exception");
  }
}

bm_status bm_cover_build(const void* points, bm_dtype dtype, int64_t n, int32_t d,
                         bm_metric metric, double eps, void* stream, bm_cover** out) {
  return bm_cover_build_ex(points, dtype, n, d, metric, eps, stream, nullptr, out);
}

bm_status bm_cover_build_host(const void* host_points, bm_dtype dtype, int64_t n, int32_t d,
                              bm_metric metric, double eps, void* stream,
                              const bm_options* opts, bm_cover** out) {
  try {
    return build_impl(host_points, dtype, n, d, metric, eps, (cudaStream_t)stream, opts, true,
                      out);
  } catch (...) {
    return set_err(BM_ENOMEM, "unexpected host exception");
  }
}

void bm_free(bm_cover* c) {
  if (!c) return;
  Priv* pv = (Priv*)c->priv;
  if (c->on_host) {
    if (pv && pv->pinned) {
      g_pinned.put(pv->pinned, pv->pinned_cls);
      if (pv->pinned_e) g_pinned.put(pv->pinned_e, pv->pinned_e_cls);
    } else {
      free(c->landmarks);
      free(c->ball_ptr);
      free(c->ball_idx);
      free(c->pt_ptr);
      free(c->pt_lm);
      free(c->edges);
    }
  } else {
    cudaStream_t s = pv ? pv->stream : nullptr;
    for (void* p : {(void*)c->landmarks, (void*)c->ball_ptr, (void*)c->ball_idx,
                    (void*)c->pt_ptr, (void*)c->pt_lm, (void*)c->edges})
      g_cache.release(p, s);
  }
  free(c->near_tie_pairs);
  free(pv);
  free(c);
}

const char* bm_last_error(void) { return g_err.c_str(); }

bm_status bm_color(const bm_cover* c, const void* values, bm_dtype vtype, bm_agg agg,
                   double alpha, double* out, void* stream) {
  using namespace bm;
  if (!c || !values || !out) return set_err(BM_EINVAL, "NULL argument");
  if (c->on_host) return set_err(BM_EINVAL, "bm_color needs a device cover");
  if (vtype != BM_F32 && vtype != BM_I32)
    return set_err(BM_EUNSUPPORTED, "values must be BM_F32 or BM_I32");
  if ((int)agg < 0 || (int)agg > BM_AGG_RANGE) return set_err(BM_EUNSUPPORTED, "unknown aggregator");
  if (agg == BM_AGG_TRIMMED && !(alpha >= 0.0 && alpha < 0.5))
    return set_err(BM_EINVAL, "trimmed mean needs 0 <= alpha < 0.5");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t L = c->n_landmarks, M = c->n_members;
  const int is_int = vtype == BM_I32;
  if (L == 0) return BM_OK;
  if (agg == BM_AGG_MEDIAN || agg == BM_AGG_TRIMMED || agg == BM_AGG_MODE) {
    Pool pool(s);
    unsigned long long *keys = nullptr, *alt = nullptr;
    void* rt = nullptr;
    TRY(pool.alloc(&keys, (size_t)(M > 0 ? M : 1)));
    TRY(pool.alloc(&alt, (size_t)(M > 0 ? M : 1)));
    TRY(pool.alloc((uint8_t**)&rt, radix_temp_bytes(M)));
    CK(launch_color_keys(c->ball_ptr, c->ball_idx, L, values, is_int, keys, s));
    const BitRange r[2] = {{0, 32}, {32, 32 + bits_for(L > 1 ? L - 1 : 1)}};
    int64_t launches = 0;
    CK(radix_sort_u64(&keys, &alt, M, r, 2, rt, s, &launches));
    CK(launch_color_order(c->ball_ptr, L, keys, is_int, (int)agg, alpha, out, s));
  } else {
    CK(launch_color_reduce(c->ball_ptr, c->ball_idx, L, values, is_int, (int)agg, out, s));
  }
  CK(cudaGetLastError());
  return BM_OK;
}

bm_status bm_skeleton(const bm_cover* c, int32_t k, int32_t* out, int64_t capacity,
                      int64_t* count, int64_t max_emit, void* stream) {
  using namespace bm;
  if (!c || !count || (capacity > 0 && !out)) return set_err(BM_EINVAL, "NULL argument");
  if (c->on_host) return set_err(BM_EINVAL, "bm_skeleton needs a device cover");
  if (k < 1 || k > 7) return set_err(BM_EUNSUPPORTED, "k must be in [1, 7]");
  const int64_t L = c->n_landmarks, n = c->n;
  const int r = k + 1;
  const int lbits = bits_for(L > 1 ? L - 1 : 1);
  if ((int64_t)r * lbits > 64) return set_err(BM_EUNSUPPORTED, "(k+1) * bits(L-1) exceeds 64");
  if (max_emit <= 0) max_emit = (int64_t)1 << 31;
  cudaStream_t s = (cudaStream_t)stream;
  *count = 0;
  Pool pool(s);
  int64_t *cnt = nullptr, *off = nullptr, *tot = nullptr;
  void* st = nullptr;
  TRY(pool.alloc(&cnt, (size_t)n));
  TRY(pool.alloc(&off, (size_t)n));
  TRY(pool.alloc(&tot, 2));
  TRY(pool.alloc((uint8_t**)&st, scan_temp_bytes(n)));
  int64_t launches = 0;
  CK(launch_simplex_counts(c->pt_ptr, n, r, cnt, s));
  CK(exclusive_scan_i64(cnt, off, n, st, tot, s, &launches));
  int64_t NP = 0;
  CK(cudaMemcpyAsync(&NP, tot, sizeof NP, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (NP > max_emit)
    return set_err(BM_EOVERFLOW, "%lld witnessed subsets exceed max_emit", (long long)NP);
  if (NP == 0) return BM_OK;
  unsigned long long *keys = nullptr, *alt = nullptr;
  void *rt = nullptr, *ut = nullptr;
  int32_t* tmp = nullptr;
  TRY(pool.alloc(&keys, (size_t)NP));
  TRY(pool.alloc(&alt, (size_t)NP));
  TRY(pool.alloc((uint8_t**)&rt, radix_temp_bytes(NP)));
  CK(launch_simplex_emit(c->pt_ptr, c->pt_lm, n, r, lbits, off, keys, s));
  const BitRange br[1] = {{0, r * lbits}};
  CK(radix_sort_u64(&keys, &alt, NP, br, 1, rt, s, &launches));
  TRY(pool.alloc(&tmp, (size_t)NP * r));
  TRY(pool.alloc((uint8_t**)&ut, simplex_unique_temp_bytes(NP)));
  CK(launch_simplex_unique(keys, NP, r, lbits, tmp, NP, tot + 1, ut, s));
  int64_t E = 0;
  CK(cudaMemcpyAsync(&E, tot + 1, sizeof E, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *count = E;
  const int64_t ncopy = E < capacity ? E : capacity;
  if (ncopy > 0) {
    CK(cudaMemcpyAsync(out, tmp, sizeof(int32_t) * r * ncopy, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return BM_OK;
}

bm_status bm_trim_memory(void) {
  g_cache.trim();
  g_pinned.trim();
  return BM_OK;
}

int32_t bm_version(void) { return (BM_VERSION_MAJOR << 16) | BM_VERSION_MINOR; }

bm_status bm_debug_radix_sort_u64(uint64_t* keys, int64_t n, int32_t bits, void* stream) {
  if (!keys || n < 0 || bits < 1 || bits > 64) return set_err(BM_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  Pool pool(s);
  unsigned long long* alt = nullptr;
  void* temp = nullptr;
  TRY(pool.alloc(&alt, (size_t)(n > 0 ? n : 1)));
  TRY(pool.alloc((uint8_t**)&temp, bm::radix_temp_bytes(n)));
  int64_t launches = 0;
  unsigned long long* k = (unsigned long long*)keys;
  const bm::BitRange r[1] = {{0, bits}};
  CK(bm::radix_sort_u64(&k, &alt, n, r, 1, temp, s, &launches));
  if (k != (unsigned long long*)keys)
    CK(cudaMemcpyAsync(keys, k, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  return BM_OK;
}

bm_status bm_debug_exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total,
                                      void* stream) {
  if (!in || !out || n < 0) return set_err(BM_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  Pool pool(s);
  void* temp = nullptr;
  int64_t* tot = nullptr;
  TRY(pool.alloc((uint8_t**)&temp, bm::scan_temp_bytes(n)));
  TRY(pool.alloc(&tot, 1));
  int64_t launches = 0;
  CK(bm::exclusive_scan_i64(in, out, n, temp, tot, s, &launches));
  int64_t h = 0;
  CK(cudaMemcpyAsync(&h, tot, sizeof h, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (total) *total = h;
  return BM_OK;
}

bm_status bm_debug_tc_gram(const void* points, bm_dtype dtype, int64_t n, int32_t d,
                           const int32_t* lm, int64_t L, uint32_t* out, void* stream) {
  using namespace bm;
  if (!points || !lm || !out || n < 1 || d < 1 || L < 1) return set_err(BM_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  tc::TcPlan P{};
  P.kind = dtype == BM_F32 ? tc::TC_TF32 : (dtype == BM_U8 ? tc::TC_U8 : tc::TC_S8);
  const int esz = dtype == BM_F32 ? 4 : 1;
  P.row_bytes = tc_row_bytes(d, esz);
  P.k_elems = P.row_bytes / esz;
  P.katoms = (int)((P.row_bytes + 127) / 128);
  if (!tc::tc_supported(P.kind, P.katoms)) return set_err(BM_EUNSUPPORTED, "d too large");
  Pool pool(s);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&P.num_sms, cudaDevAttrMultiProcessorCount, dev));
  uint8_t* xop = nullptr;
  void* nrm = nullptr;
  DevStats* stats = nullptr;
  TRY(pool.alloc(&xop, (size_t)n * P.row_bytes));
  TRY(pool.alloc((double**)&nrm, (size_t)n));
  TRY(pool.alloc(&stats, 1));
  CK(cudaMemsetAsync(stats, 0, sizeof(DevStats), s));
  P.xop = xop;
  P.n_rows = n;
  int64_t launches = 0;
  CK(tc::launch_tc_prep(points, dtype, n, d, P, nrm, stats, s, &launches));
  const int BN = tc::tc_bn_for(P.kind, P.katoms), RB = tc::tc_rows_for(P.kind, P.katoms);
  P.l_rows = ((L + BN - 1) / BN) * BN;
  P.n_pad = ((n + RB - 1) / RB) * RB;
  TRY(pool.alloc((uint8_t**)&P.lop, (size_t)P.l_rows * P.row_bytes));
  tc::TcArgs ta{};
  ta.n = n;
  ta.L = L;
  ta.ksteps = (int)(((int64_t)d * esz + 31) / 32);
  float *fa, *fb;
  TRY(pool.alloc(&fa, (size_t)P.l_rows * 2));
  fb = fa + P.l_rows;
  ta.col_a = fa;
  ta.col_b = fb;
  ta.col_c = (const int32_t*)fa;
  TRY(alloc_fold(pool, P, ta, s, &launches));
  CK(tc::launch_tc_landmarks(P, nrm, lm, L, 0.0, ta, s, &launches));
  ta.gram = out;
  CK(tc::launch_tc(P, ta, s, &launches));
  CK(cudaStreamSynchronize(s));
  return BM_OK;
}

bm_status bm_debug_tc_probe(const float* points, int64_t n, int32_t d, int64_t L, int32_t mode,
                            int32_t iters, float* ms_out, void* stream) {
  using namespace bm;
  if (!points || !ms_out || n < 1 || d < 1 || L < 1 || L > n || iters < 1)
    return set_err(BM_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  tc::TcPlan P{};
  P.kind = tc::TC_TF32;
  P.row_bytes = tc_row_bytes(d, 4);
  P.k_elems = P.row_bytes / 4;
  P.katoms = (int)((P.row_bytes + 127) / 128);
  if (P.katoms > 2) return set_err(BM_EUNSUPPORTED, "probe: d <= 64 only");
  Pool pool(s);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&P.num_sms, cudaDevAttrMultiProcessorCount, dev));
  uint8_t* xop = nullptr;
  double* nrm = nullptr;
  DevStats* stats = nullptr;
  int32_t* lm = nullptr;
  TRY(pool.alloc(&xop, (size_t)n * P.row_bytes));
  TRY(pool.alloc(&nrm, (size_t)n));
  TRY(pool.alloc(&stats, 1));
  TRY(pool.alloc(&lm, (size_t)L));
  CK(cudaMemsetAsync(stats, 0, sizeof(DevStats), s));
  P.xop = xop;
  P.n_rows = n;
  int64_t launches = 0;
  CK(tc::launch_tc_prep(points, BM_F32, n, d, P, nrm, stats, s, &launches));
  k_iota<<<(unsigned)((L + 255) / 256), 256, 0, s>>>(lm, L);
  const int BN = tc::tc_bn_for(P.kind, P.katoms), RB = tc::tc_rows_for(P.kind, P.katoms);
  P.l_rows = ((L + BN - 1) / BN) * BN;
  P.n_pad = ((n + RB - 1) / RB) * RB;
  TRY(pool.alloc((uint8_t**)&P.lop, (size_t)P.l_rows * P.row_bytes));
  tc::TcArgs ta{};
  ta.n = n;
  ta.L = L;
  ta.ksteps = (int)(((int64_t)d * 4 + 31) / 32);
  ta.lbits = 32;
  float *rlo, *rhi, *ca, *cb;
  TRY(pool.alloc(&rlo, (size_t)P.n_pad));
  TRY(pool.alloc(&rhi, (size_t)P.n_pad));
  TRY(pool.alloc(&ca, (size_t)P.l_rows));
  TRY(pool.alloc(&cb, (size_t)P.l_rows));
  ta.row_lo = rlo;
  ta.row_hi = rhi;
  ta.col_a = ca;
  ta.col_b = cb;
  TRY(alloc_fold(pool, P, ta, s, &launches));
  // eps tiny: every pair is certainly out, the epilogue takes its fast path only
  CK(tc::launch_tc_rows(P, nrm, n, tc_band_c2(ta.ksteps), 1e-30, 0.0, 0, ta, s, &launches));
  CK(tc::launch_tc_landmarks(P, nrm, lm, L, tc_band_c2(ta.ksteps), ta, s, &launches));
  unsigned long long *keys = nullptr, *kc = nullptr;
  TRY(pool.alloc(&keys, 1024));
  TRY(pool.alloc(&kc, 2));
  CK(cudaMemsetAsync(kc, 0, 16, s));
  ta.keys = keys;
  ta.key_count = kc;
  ta.key_cap = 1024;
  set_recheck(ta, points, d, d, make_thresh(K_L2F, d, 1e-15), lm, nullptr, 0, stats);
  CK(tc::launch_tc_probe(P, ta, mode, s));   // warm-up
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i) CK(tc::launch_tc_probe(P, ta, mode, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms / iters;
  if (mode & 256) {   // one traced launch: per-CTA %globaltimer stamps to stderr
    const int G = P.num_sms;
    unsigned long long* tr = nullptr;
    TRY(pool.alloc(&tr, (size_t)G * 16));
    CK(cudaMemsetAsync(tr, 0, sizeof(unsigned long long) * G * 16, s));
    ta.trace = tr;
    CK(tc::launch_tc_probe(P, ta, mode & 255, s));
    CK(print_tc_trace(tr, G, "probe", s));
  }
  return BM_OK;
}

bm_status bm_debug_resolve_tile(const uint32_t* adj, int32_t nc, uint8_t* lm_out, void* stream) {
  if (!adj || !lm_out || nc < 1 || nc > 1024) return set_err(BM_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  Pool pool(s);
  const int words = (nc + 31) / 32;
  uint32_t* dadj = nullptr;
  uint8_t* dlm = nullptr;
  // the library's layout is word-major: word v of candidate a at [v * 32 words + a]
  const int T = 32 * words;
  std::vector<uint32_t> wm((size_t)words * T, 0u);
  for (int a = 0; a < nc; ++a)
    for (int v = 0; v < words; ++v) wm[(size_t)v * T + a] = adj[(size_t)a * words + v];
  TRY(pool.alloc(&dadj, (size_t)words * T));
  TRY(pool.alloc(&dlm, (size_t)nc));
  CK(cudaMemcpyAsync(dadj, wm.data(), sizeof(uint32_t) * words * T, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  int64_t launches = 0;
  CK(bm::launch_resolve_debug(dadj, words, nc, dlm, s, &launches));
  if (getenv("BM_RESOLVE_BENCH")) {   // diagnostics: device time per resolve launch
    cudaEvent_t e0 = cached_event(8000), e1 = cached_event(8001);
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < 200; ++i) CK(bm::launch_resolve_debug(dadj, words, nc, dlm, s, &launches));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "resolve nc=%d: %.2f us per launch\n", nc, ms * 1e3f / 200.f);
  }
  CK(cudaMemcpyAsync(lm_out, dlm, nc, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return BM_OK;
}

}  // extern "C"
