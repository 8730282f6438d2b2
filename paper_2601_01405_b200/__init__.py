"""B200-native Ball Mapper cover construction (arxiv 2601.01405).

Public API (thin binding over the C ABI in include/bm.h):

    cover_build(points_cuda_tensor, metric, eps, ...) -> Cover
    cover_build_host(points_numpy, metric, eps, ...)  -> Cover (host arrays)
    color(cover, values_cuda_tensor, agg, alpha)      -> CUDA float64 [L]
    skeleton(cover, k)                                 -> CUDA int32 [count, k+1]

The hot path (greedy eps-net, ball membership, CSR, nerve 1-skeleton) and the
coloring / k-skeleton run in hand-written sm_100a kernels inside libbm_b200.so.
"""
from .bm import (BMError, Cover, color, cover_build, cover_build_host, load,  # noqa: F401
                 skeleton, trim_memory, EXPORTED, LIB_PATH)

__all__ = ["BMError", "Cover", "color", "cover_build", "cover_build_host", "load", "skeleton",
           "trim_memory"]
