// pairs.cu — kind dispatch for the CUDA-core pair kernel (pairs_impl.cuh).
#include "pairs_impl.cuh"

namespace bm {

template <int KIND>
cudaError_t launch_pairs_kind(int mode, const PairArgs& a, int64_t q_rows_max, cudaStream_t s);

cudaError_t launch_pairs(int kind, int mode, const PairArgs& a, int64_t q_rows_max,
                         cudaStream_t s, int64_t* launches) {
  ++*launches;
  switch (kind) {
    case K_L2F: return launch_pairs_kind<K_L2F>(mode, a, q_rows_max, s);
    case K_L1F: return launch_pairs_kind<K_L1F>(mode, a, q_rows_max, s);
    case K_COSF: return launch_pairs_kind<K_COSF>(mode, a, q_rows_max, s);
    case K_L2I: return launch_pairs_kind<K_L2I>(mode, a, q_rows_max, s);
    case K_L1I: return launch_pairs_kind<K_L1I>(mode, a, q_rows_max, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bm
