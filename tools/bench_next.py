"""Measurements of the §8(f) rows (NEXT-1 coloring, NEXT-2 FPS, NEXT-3 k-skeleton)
on the BASELINE workloads.  One JSON line per measurement on stdout.

  python tools/bench_next.py [--reps 5] [--only color,skeleton,fps]

Timing: CUDA events on the current stream (the stream the library launches
on), warm-up first, median of --reps.  The oracle (oracle/extensions.py for
coloring and the k-skeleton, the C oracle's FPS) is timed beside it on the
host (one run, wall clock; FPS on a bounded prefix, stated per line).
Rooflines: algorithmic bytes per call (stated per line) over the measured
time, against MEASURED_PEAKS.json's HBM copy bandwidth.  FPS: per landmark step the kernel reads every row once and
reads + writes the running minimum (n * (row bytes + 16)), so its roofline is
that traffic x L over the selection kernel's own time (BM_STEP_SELECT).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from oracle import extensions as OX  # noqa: E402  (the oracle timed beside the GPU)
from oracle import oracle as O  # noqa: E402
from workloads import gen  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
ESZ = {"f32": 4, "i8": 1, "u8": 1}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), ts


def emit(**kw):
    print(json.dumps(kw), flush=True)


def bench_color(name, reps):
    w = gen.get(name)
    X = torch.from_numpy(gen.generate(w)).cuda()
    cov = bm.cover_build(X, w.metric, w.eps)
    rng = np.random.default_rng(3)
    f = torch.from_numpy(rng.normal(size=w.n).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, 7, size=w.n).astype(np.int32)).cuda()
    h = cov.numpy()
    fh, labh = f.cpu().numpy(), lab.cpu().numpy()
    for agg in ("mean", "variance", "min", "max", "range", "median", "trimmed", "mode"):
        vals = lab if agg == "mode" else f
        ms, _ = timed(lambda: bm.color(cov, vals, agg, 0.1), reps)
        t0 = time.perf_counter()
        OX.color(h["ball_ptr"], h["ball_idx"], labh if agg == "mode" else fh, agg, 0.1)
        oracle_ms = (time.perf_counter() - t0) * 1e3
        # reduce aggregators: ball_ptr (L+1)*8 + ball_idx M*4 + gathered values M*4 + out L*8
        # order aggregators add the per-ball sort: key write M*8 + sort (read+write per pass)
        byts = (cov.L + 1) * 8 + cov.M * 8 + cov.L * 8
        if agg in ("median", "trimmed", "mode"):
            byts += cov.M * 8 + cov.M * 8 * 2 * 2 + cov.M * 8
        emit(row="NEXT-1 color", workload=name, agg=agg, L=cov.L, M=cov.M, ms=round(ms, 4),
             algorithmic_bytes=byts, achieved_gbs=round(byts / ms / 1e6, 1),
             hbm_peak_gbs=PEAK, frac=round(byts / ms / 1e6 / PEAK, 4),
             oracle_ms=round(oracle_ms, 3), oracle_kind="oracle/extensions.py (numpy, 1 core)")


def bench_skeleton(name, reps, ks=(1, 2, 3)):
    w = gen.get(name)
    X = torch.from_numpy(gen.generate(w)).cuda()
    cov = bm.cover_build(X, w.metric, w.eps)
    ptr = cov.numpy()["pt_ptr"]
    deg = np.diff(np.asarray(ptr, dtype=np.int64))
    from math import comb
    h = cov.numpy()
    for k in ks:
        emitted = int(sum(comb(int(t), k + 1) for t in deg))
        ms, _ = timed(lambda: bm.skeleton(cov, k), reps)
        out = bm.skeleton(cov, k)
        t0 = time.perf_counter()
        OX.skeleton(h["pt_ptr"], h["pt_lm"], k)
        oracle_ms = (time.perf_counter() - t0) * 1e3
        # algorithmic bytes: row reads (pt_ptr, pt_lm) + the emitted keys written,
        # sorted (read + write per radix pass) and read once by the unique pass
        import math as _m
        passes = max(1, _m.ceil((k + 1) * max(1, (cov.L - 1).bit_length()) / 8))
        byts = 8 * (len(h["pt_ptr"])) + 4 * cov.M + emitted * 8 * (2 + 2 * passes)
        emit(row="NEXT-3 skeleton", workload=name, k=k, L=cov.L, M=cov.M,
             simplices=int(out.shape[0]), emitted_keys=emitted, ms=round(ms, 4),
             keys_per_s=round(emitted / ms * 1e3, 1), algorithmic_bytes=byts,
             achieved_gbs=round(byts / ms / 1e6, 1), hbm_peak_gbs=PEAK,
             frac=round(byts / ms / 1e6 / PEAK, 4), oracle_ms=round(oracle_ms, 3),
             oracle_kind="oracle/extensions.py (Python per point, 1 core)")


def bench_fps(name, reps, n=None):
    w = gen.get(name)
    X = torch.from_numpy(gen.generate(w, n)).cuda()
    nn = X.shape[0]
    g = bm.cover_build(X, w.metric, w.eps, timing=True)
    tg, _ = timed(lambda: bm.cover_build(X, w.metric, w.eps), reps)
    covs = []

    def run():
        covs.append(bm.cover_build(X, w.metric, w.eps, select="fps", timing=True))
    tf, _ = timed(run, reps)
    c = covs[-1]
    sel = statistics.median(cv.stats.step_ms["select"] for cv in covs[1:])
    row_bytes = w.d * ESZ[w.dtype]
    byts = nn * (row_bytes + 16) * c.L
    # the C oracle's FPS on a bounded prefix (seconds, OpenMP over the host cores)
    m = min(nn, 20000)
    Xh = gen.generate(w, m)
    t0 = time.perf_counter()
    so = O.fps(Xh, w.metric, w.eps)
    oracle_s = time.perf_counter() - t0
    emit(row="NEXT-2 fps", workload=name, n=nn, L_fps=c.L, L_greedy=g.L, M_fps=c.M, M_greedy=g.M,
         E_fps=c.E, E_greedy=g.E, greedy_build_ms=round(tg, 3), fps_build_ms=round(tf, 3),
         fps_select_ms=round(sel, 3), select_us_per_landmark=round(sel / c.L * 1e3, 3),
         algorithmic_bytes_select=byts, achieved_gbs=round(byts / sel / 1e6, 1),
         hbm_peak_gbs=PEAK,
         # float L2 / L1 FPS skips warps by bounding balls (fps.cu): the unpruned
         # bytes then overstate the traffic, so no fraction is claimed for them
         frac=None if (w.dtype == "f32" and w.metric in ("l2", "l1"))
         else round(byts / sel / 1e6 / PEAK, 4),
         warp_pruning=w.dtype == "f32" and w.metric in ("l2", "l1"),
         oracle_prefix_n=m, oracle_prefix_L=int(len(so)), oracle_select_s=round(oracle_s, 3),
         oracle_evals_per_s=round(m * len(so) / oracle_s, 1),
         gpu_evals_per_s=round(nn * c.L / (sel * 1e-3), 1),
         oracle_kind="oracle_fps (C, OpenMP)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="color,skeleton,fps")
    ap.add_argument("--fps-workloads", default="c1,c2,c4,c3_e8")
    a = ap.parse_args()
    bm.load()
    only = a.only.split(",")
    t0 = time.time()
    if "color" in only:
        for name in ("c2", "c4"):
            bench_color(name, a.reps)
    if "skeleton" in only:
        bench_skeleton("c1", a.reps)
        bench_skeleton("c2", a.reps)
    if "fps" in only:
        for name in a.fps_workloads.split(","):
            bench_fps(name, max(2, a.reps // 2) if name.startswith("c3") else a.reps)
    emit(row="done", seconds=round(time.time() - t0, 1))


if __name__ == "__main__":
    main()
