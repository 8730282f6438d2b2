"""B200-native Ball Mapper cover construction (arxiv 2601.01405).

Public API (thin binding over the C ABI in include/bm.h):

    cover_build(points_cuda_tensor, metric, eps, ...) -> Cover
    cover_build_host(points_numpy, metric, eps, ...)  -> Cover (host arrays)

The hot path (greedy eps-net, ball membership, CSR, nerve 1-skeleton) runs in
hand-written sm_100a kernels inside libbm_b200.so.
"""
from .bm import (BMError, Cover, cover_build, cover_build_host, load,  # noqa: F401
                 EXPORTED, LIB_PATH)

__all__ = ["BMError", "Cover", "cover_build", "cover_build_host", "load"]
