"""Thin ctypes binding of include/bm.h (argument marshalling only).

Every step of the cover construction runs inside libbm_b200.so; this module
only converts torch / numpy buffers to pointers and wraps the returned
``bm_cover``.  There is no CPU fallback: if the library is missing, importing
or calling raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# BM_LIB_PATH (diagnostics only): load another build of the library, e.g. for A/B runs
LIB_PATH = os.environ.get("BM_LIB_PATH") or os.path.join(PKG, "libbm_b200.so")

BM_OK, BM_EINVAL, BM_EUNSUPPORTED, BM_ENOMEM, BM_ECUDA, BM_EOVERFLOW = range(6)
STATUS_NAMES = {0: "BM_OK", 1: "BM_EINVAL", 2: "BM_EUNSUPPORTED", 3: "BM_ENOMEM",
                4: "BM_ECUDA", 5: "BM_EOVERFLOW"}
METRIC = {"l2": 0, "l1": 1, "cos": 2, "cosine": 2}
DTYPE = {"f32": 0, "i8": 1, "u8": 2, "i32": 3}
AGG = {"mean": 0, "median": 1, "trimmed": 2, "min": 3, "max": 4, "mode": 5, "variance": 6,
       "range": 7}
PATH = {"auto": 0, "cuda_core": 1, "tensor": 2}
FLAG_NO_L1_PREFILTER = 1
FLAG_EDGE_POINT_PAIRS = 2
FLAG_NO_EDGE_TRIANGLE = FLAG_EDGE_POINT_PAIRS   # (former name)
FLAG_NO_PRUNE = 4
FLAG_FORCE_PRUNE = 8
FLAG_DENSE_RESOLVE = 16
FLAG_EDGE_TRIANGLE = 32
FLAG_EDGE_ROWS = 64
STEPS = ("prep", "greedy", "member", "csr", "edges", "total", "member_kernel", "select")

EXPORTED = ("bm_cover_build", "bm_cover_build_ex", "bm_cover_build_host", "bm_free",
            "bm_last_error", "bm_version", "bm_trim_memory", "bm_debug_radix_sort_u64",
            "bm_debug_exclusive_scan_i64", "bm_debug_resolve_tile", "bm_debug_tc_gram",
            "bm_debug_tc_probe", "bm_color", "bm_skeleton")


class BMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("tile", ctypes.c_int32),
                ("path", ctypes.c_int32), ("timing", ctypes.c_int32),
                ("near_tie_cap", ctypes.c_int64), ("key_cap", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("select", ctypes.c_int32), ("fps_start", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 3)]


class _Cover(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("metric", ctypes.c_int32), ("on_host", ctypes.c_int32), ("eps", ctypes.c_double),
                ("n_landmarks", ctypes.c_int64), ("landmarks", ctypes.c_void_p),
                ("n_members", ctypes.c_int64), ("ball_ptr", ctypes.c_void_p),
                ("ball_idx", ctypes.c_void_p), ("pt_ptr", ctypes.c_void_p),
                ("pt_lm", ctypes.c_void_p),
                ("n_edges", ctypes.c_int64), ("edges", ctypes.c_void_p),
                ("n_witness_pairs", ctypes.c_int64),
                ("n_pair_evals", ctypes.c_int64), ("n_greedy_evals", ctypes.c_int64),
                ("n_band_pairs", ctypes.c_int64), ("n_near_ties", ctypes.c_int64),
                ("n_near_ties_stored", ctypes.c_int64),
                ("near_tie_pairs", ctypes.POINTER(ctypes.c_int64)),
                ("n_greedy_tiles", ctypes.c_int64), ("n_launches", ctypes.c_int64),
                ("n_member_launches", ctypes.c_int64),
                ("path_used", ctypes.c_int32), ("tile_used", ctypes.c_int32),
                ("step_ms", ctypes.c_float * 8),
                ("n_tc_tiles_run", ctypes.c_int64), ("n_tc_tiles_skipped", ctypes.c_int64),
                ("n_tc_chunks_run", ctypes.c_int64), ("n_tc_chunks_skipped", ctypes.c_int64),
                ("priv", ctypes.c_void_p)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libbm_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2601_01405_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    pc = ctypes.POINTER(ctypes.POINTER(_Cover))
    lib.bm_cover_build.argtypes = [vp, i32, i64, i32, i32, dbl, vp, pc]
    lib.bm_cover_build_ex.argtypes = [vp, i32, i64, i32, i32, dbl, vp,
                                      ctypes.POINTER(_Options), pc]
    lib.bm_cover_build_host.argtypes = [vp, i32, i64, i32, i32, dbl, vp,
                                        ctypes.POINTER(_Options), pc]
    for f in (lib.bm_cover_build, lib.bm_cover_build_ex, lib.bm_cover_build_host):
        f.restype = i32
    lib.bm_free.argtypes = [ctypes.POINTER(_Cover)]
    lib.bm_free.restype = None
    lib.bm_last_error.restype = ctypes.c_char_p
    lib.bm_version.restype = i32
    lib.bm_trim_memory.restype = i32
    lib.bm_color.argtypes = [ctypes.POINTER(_Cover), vp, i32, i32, dbl, vp, vp]
    lib.bm_color.restype = i32
    lib.bm_skeleton.argtypes = [ctypes.POINTER(_Cover), i32, vp, i64, ctypes.POINTER(i64), i64,
                                vp]
    lib.bm_skeleton.restype = i32
    lib.bm_debug_radix_sort_u64.argtypes = [vp, i64, i32, vp]
    lib.bm_debug_radix_sort_u64.restype = i32
    lib.bm_debug_exclusive_scan_i64.argtypes = [vp, vp, i64, ctypes.POINTER(i64), vp]
    lib.bm_debug_exclusive_scan_i64.restype = i32
    lib.bm_debug_resolve_tile.argtypes = [vp, i32, vp, vp]
    lib.bm_debug_resolve_tile.restype = i32
    lib.bm_debug_tc_gram.argtypes = [vp, i32, i64, i32, vp, i64, vp, vp]
    lib.bm_debug_tc_gram.restype = i32
    lib.bm_debug_tc_probe.argtypes = [vp, i64, i32, i64, i32, i32, ctypes.POINTER(ctypes.c_float), vp]
    lib.bm_debug_tc_probe.restype = i32
    _lib = lib
    return lib


def _check(rc: int):
    if rc != BM_OK:
        raise BMError(rc, load().bm_last_error().decode())


SELECT = {"greedy": 0, "fps": 1}


def _options(tile=0, path="auto", timing=False, near_tie_cap=0, key_cap=0,
             flags=0, select="greedy", fps_start=0) -> _Options:
    o = _Options()
    o.struct_size = ctypes.sizeof(_Options)
    o.tile = int(tile)
    o.path = PATH[path] if isinstance(path, str) else int(path)
    o.timing = 1 if timing else 0
    o.near_tie_cap = int(near_tie_cap)
    o.key_cap = int(key_cap)
    o.flags = int(flags)
    o.select = SELECT[select] if isinstance(select, str) else int(select)
    o.fps_start = int(fps_start)
    return o


class _DevArray:
    """__cuda_array_interface__ view of a library-owned device array.  Holds a
    reference to the owning Cover, so a torch view (which keeps its source
    object alive) keeps the cover's memory from being handed back to the
    library's block cache while the view exists.  An explicit Cover.free()
    still releases it: views must not be used after that call."""

    def __init__(self, ptr, shape, typestr, owner=None):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}


@dataclass
class CoverStats:
    n_pair_evals: int
    n_greedy_evals: int
    n_band_pairs: int
    n_near_ties: int
    n_greedy_tiles: int
    n_launches: int
    n_member_launches: int
    path_used: int
    tile_used: int
    step_ms: dict
    tc_tiles_run: int = 0
    tc_tiles_skipped: int = 0
    tc_chunks_run: int = 0
    tc_chunks_skipped: int = 0


class Cover:
    """Owns one bm_cover.  Device arrays are exposed as torch tensors that
    alias library memory (valid until .free()); .numpy() copies to host."""

    def __init__(self, ptr):
        self._ptr = ptr
        c = ptr.contents
        self.n, self.d, self.eps = c.n, c.d, c.eps
        self.L, self.M, self.E = c.n_landmarks, c.n_members, c.n_edges
        self.P = c.n_witness_pairs
        self.on_host = bool(c.on_host)
        self.stats = CoverStats(c.n_pair_evals, c.n_greedy_evals, c.n_band_pairs,
                                c.n_near_ties, c.n_greedy_tiles, c.n_launches,
                                c.n_member_launches, c.path_used,
                                c.tile_used, {k: float(c.step_ms[i]) for i, k in
                                              enumerate(STEPS)},
                                c.n_tc_tiles_run, c.n_tc_tiles_skipped, c.n_tc_chunks_run,
                                c.n_tc_chunks_skipped)
        k = c.n_near_ties_stored
        if k > 0:
            self.near_ties = np.ctypeslib.as_array(c.near_tie_pairs, shape=(k, 3)).copy()
        else:
            self.near_ties = np.zeros((0, 3), dtype=np.int64)

    def _spec(self):
        c = self._ptr.contents
        return {"landmarks": (c.landmarks, (self.L,), "<i4"),
                "ball_ptr": (c.ball_ptr, (self.L + 1,), "<i8"),
                "ball_idx": (c.ball_idx, (self.M,), "<i4"),
                "pt_ptr": (c.pt_ptr, (self.n + 1,), "<i8"),
                "pt_lm": (c.pt_lm, (self.M,), "<i4"),
                "edges": (c.edges, (self.E, 2), "<i4")}

    def tensors(self) -> dict:
        """Zero-copy torch views of the device arrays (device covers only)."""
        if self.on_host:
            raise ValueError("host cover: use .numpy()")
        import torch
        out = {}
        for name, (p, shape, ts) in self._spec().items():
            if int(np.prod(shape)) == 0:
                dt = torch.int32 if ts == "<i4" else torch.int64
                out[name] = torch.zeros(shape, dtype=dt, device="cuda")
            else:
                out[name] = torch.as_tensor(_DevArray(p, shape, ts, owner=self), device="cuda")
        return out

    def numpy(self) -> dict:
        if self.on_host:
            out = {}
            for name, (p, shape, ts) in self._spec().items():
                ct = ctypes.c_int32 if ts == "<i4" else ctypes.c_int64
                n = int(np.prod(shape))
                if n == 0:
                    out[name] = np.zeros(shape, dtype=np.dtype(ts))
                else:
                    arr = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ct)), shape=(n,))
                    out[name] = arr.copy().reshape(shape)
            return out
        return {k: v.cpu().numpy() for k, v in self.tensors().items()}

    def free(self):
        if self._ptr is not None:
            load().bm_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _dtype_of(t) -> str:
    s = str(t.dtype)
    if s.endswith("float32"):
        return "f32"
    if s.endswith("uint8"):
        return "u8"
    if s.endswith("int8"):
        return "i8"
    raise ValueError(f"unsupported dtype {t.dtype}")


def cover_build(points, metric: str, eps: float, stream=None, tile: int = 0,
                path: str = "auto", timing: bool = False, near_tie_cap: int = 0,
                key_cap: int = 0, flags: int = 0, select: str = "greedy",
                fps_start: int = 0) -> Cover:
    """bm_cover_build_ex on a CUDA torch tensor [n, d] (row-major, contiguous)."""
    import torch
    if not (isinstance(points, torch.Tensor) and points.is_cuda):
        raise TypeError("points must be a CUDA torch tensor (use cover_build_host for host data)")
    if points.dim() != 2:
        raise ValueError("points must be 2-D [n, d]")
    points = points.contiguous()
    n, d = points.shape
    if stream is None:
        stream = torch.cuda.current_stream(points.device)
    sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    out = ctypes.POINTER(_Cover)()
    o = _options(tile, path, timing, near_tie_cap, key_cap, flags, select,
                 fps_start)
    lib = load()
    with torch.cuda.device(points.device):
        rc = lib.bm_cover_build_ex(ctypes.c_void_p(points.data_ptr()), DTYPE[_dtype_of(points)],
                                   n, d, METRIC[metric], float(eps), ctypes.c_void_p(sp),
                                   ctypes.byref(o), ctypes.byref(out))
    _check(rc)
    return Cover(out)


def cover_build_host(points: np.ndarray, metric: str, eps: float, stream=None, tile: int = 0,
                     path: str = "auto", timing: bool = False, near_tie_cap: int = 0,
                     key_cap: int = 0, flags: int = 0, select: str = "greedy",
                     fps_start: int = 0) -> Cover:
    """bm_cover_build_host on a host buffer (numpy array or CPU torch tensor,
    ideally pinned): copies in, builds, copies every result back to host."""
    import torch
    if isinstance(points, torch.Tensor):
        if points.is_cuda:
            raise TypeError("cover_build_host takes host memory")
        points = points.contiguous()
        ptr, (n, d), dt = points.data_ptr(), points.shape, _dtype_of(points)
    else:
        points = np.ascontiguousarray(points)
        ptr, (n, d) = points.ctypes.data, points.shape
        dt = {np.dtype(np.float32): "f32", np.dtype(np.int8): "i8",
              np.dtype(np.uint8): "u8"}[points.dtype]
    if stream is None:
        stream = torch.cuda.current_stream()
    sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    out = ctypes.POINTER(_Cover)()
    o = _options(tile, path, timing, near_tie_cap, key_cap, flags, select,
                 fps_start)
    rc = load().bm_cover_build_host(ctypes.c_void_p(ptr), DTYPE[dt], n, d, METRIC[metric],
                                    float(eps), ctypes.c_void_p(sp), ctypes.byref(o),
                                    ctypes.byref(out))
    _check(rc)
    return Cover(out)


def raw_build(ptr: int, dtype: str, n: int, d: int, metric: str, eps: float, stream: int = 0):
    """bm_cover_build with raw arguments (ABI tests: NULL pointers, bad sizes)."""
    out = ctypes.POINTER(_Cover)()
    rc = load().bm_cover_build(ctypes.c_void_p(ptr), DTYPE.get(dtype, dtype) if isinstance(
        dtype, str) else dtype, n, d, METRIC.get(metric, metric) if isinstance(metric, str)
        else metric, float(eps), ctypes.c_void_p(stream), ctypes.byref(out))
    return rc, (Cover(out) if rc == BM_OK else None)


def radix_sort_u64(keys, bits: int):
    """In-place device radix sort (diagnostic entry point)."""
    import torch
    assert keys.is_cuda and keys.dtype == torch.int64 and keys.is_contiguous()
    _check(load().bm_debug_radix_sort_u64(ctypes.c_void_p(keys.data_ptr()), keys.numel(), bits,
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return keys


def exclusive_scan_i64(x):
    import torch
    out = torch.empty_like(x)
    tot = ctypes.c_int64()
    _check(load().bm_debug_exclusive_scan_i64(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), x.numel(),
        ctypes.byref(tot), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out, tot.value


def resolve_tile(adj_words: np.ndarray, nc: int) -> np.ndarray:
    """A3 on the device from a host [nc, ceil(nc/32)] uint32 lower-triangular adjacency."""
    import torch
    adj_words = np.ascontiguousarray(adj_words, dtype=np.uint32)
    out = np.zeros(nc, dtype=np.uint8)
    _check(load().bm_debug_resolve_tile(
        ctypes.c_void_p(adj_words.ctypes.data), nc, ctypes.c_void_p(out.ctypes.data),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def tc_gram(points, landmarks):
    """Raw tcgen05 accumulators [n, L] (diagnostic; float32 for f32 input,
    int32 for int8 input) of points @ points[landmarks].T."""
    import torch
    assert points.is_cuda and landmarks.is_cuda and landmarks.dtype == torch.int32
    n, d = points.shape
    L = landmarks.numel()
    out = torch.empty((n, L), dtype=torch.int32, device=points.device)
    _check(load().bm_debug_tc_gram(
        ctypes.c_void_p(points.data_ptr()), DTYPE[_dtype_of(points)], n, d,
        ctypes.c_void_p(landmarks.data_ptr()), L, ctypes.c_void_p(out.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out.view(torch.float32) if _dtype_of(points) == "f32" else out


def trim_memory():
    """Return the library's cached device memory (its stream-ordered pool) to the system."""
    _check(load().bm_trim_memory())


def tc_probe(points, L: int, mode: int, iters: int = 10) -> float:
    """Mean launch time (ms) of the tcgen05 contraction with a probe epilogue
    (diagnostic entry point bm_debug_tc_probe)."""
    import torch
    assert points.is_cuda and points.dtype == torch.float32 and points.is_contiguous()
    ms = ctypes.c_float(0.0)
    n, d = points.shape
    _check(load().bm_debug_tc_probe(ctypes.c_void_p(points.data_ptr()), n, d, int(L), int(mode),
                                    int(iters), ctypes.byref(ms),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return float(ms.value)


def color(cov: "Cover", values, agg: str = "mean", alpha: float = 0.1):
    """bm_color: colour every landmark of a device cover.
    values: CUDA tensor [n] float32 (function values) or int32 (labels).
    Returns a CUDA float64 tensor [L]."""
    import torch
    if cov.on_host:
        raise ValueError("bm_color needs a device cover")
    if not (isinstance(values, torch.Tensor) and values.is_cuda) or values.numel() != cov.n:
        raise ValueError("values must be a CUDA tensor with one entry per point")
    vt = {torch.float32: DTYPE["f32"], torch.int32: DTYPE["i32"]}[values.dtype]
    values = values.contiguous()
    out = torch.empty(cov.L, dtype=torch.float64, device=values.device)
    _check(load().bm_color(cov._ptr, ctypes.c_void_p(values.data_ptr()), vt, AGG[agg],
                           float(alpha), ctypes.c_void_p(out.data_ptr()),
                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def skeleton(cov: "Cover", k: int = 2, max_emit: int = 0):
    """bm_skeleton: the k-simplices of the nerve as a CUDA int32 tensor [count, k+1]."""
    import torch
    cnt = ctypes.c_int64(0)
    lib = load()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _check(lib.bm_skeleton(cov._ptr, int(k), None, 0, ctypes.byref(cnt), int(max_emit), sp))
    out = torch.empty((max(cnt.value, 1), k + 1), dtype=torch.int32, device="cuda")
    _check(lib.bm_skeleton(cov._ptr, int(k), ctypes.c_void_p(out.data_ptr()), cnt.value,
                           ctypes.byref(cnt), int(max_emit), sp))
    return out[: cnt.value]
