// pairs_l1i.cu — instantiation of the CUDA-core pair kernel for kind K_L1I
// (split per kind so the kernel variants compile in parallel).
#include "pairs_impl.cuh"
namespace bm {
BM_INSTANTIATE_PAIRS(K_L1I)
}
