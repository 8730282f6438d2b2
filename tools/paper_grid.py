"""The paper's benchmark grid on the B200 path (second half).

PAPER.md:263 [§4]: n in {100, 500, 1000, 2000, 5000} x D in {10, 50, 100,
200, 500, 1000}, 65 trials per cell, Euclidean eps-net; §4.1 reports median
runtimes and speedups; §4.3 fits T(D) = k D^p by least squares on
log T = log k + p log D and reports p with R^2 (Table 1).  Inputs: uniform on
[0,1)^D, eps = 0.5 sqrt(D/6) (workloads/gen.py cube_cloud / cube_eps; DESIGN.md
reading G1).  The paper's comparison systems (Ball Tree, FAISS, pyBallMapper)
are out of scope; the oracle (C, OpenMP) is timed beside the GPU instead.

Per cell: median over trials of
  * device ms  — bm_cover_build on device-resident input, CUDA events;
  * e2e ms     — bm_cover_build_host from host numpy input to host numpy
                 output arrays (wall clock, copies included: what §4 times);
  * oracle ms  — the C oracle's cover (wall clock, --oracle-trials trials).
Fits: T(D) at each n and T(n) at each D, for e2e and device time (fit_power_law).

  python tools/paper_grid.py [--trials 65] [--oracle-trials 3] [--out FILE.jsonl]
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import gen  # noqa: E402


def fit_power_law(xs, ys) -> dict:
    """Least-squares line through (log x, log y) (P:326-332 [§4.3]): p = slope,
    k = exp(intercept), R^2 = 1 - SS_res / SS_tot in log space on the fit's own
    residuals."""
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    if x.size < 2 or x.size != y.size:
        raise ValueError("need >= 2 (x, y) pairs")
    if (x <= 0).any() or (y <= 0).any():
        raise ValueError("power-law fit needs positive values")
    if np.all(x == x[0]):
        raise ValueError("xs are all equal")
    lx, ly = np.log(x), np.log(y)
    mx, my = lx.mean(), ly.mean()
    p = float(((lx - mx) * (ly - my)).sum() / ((lx - mx) ** 2).sum())
    b = my - p * mx
    res = ly - (b + p * lx)
    ss_res = float((res ** 2).sum())
    ss_tot = float(((ly - my) ** 2).sum())
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return {"p": p, "k": float(math.exp(b)), "r2": r2}


def median(v):
    return statistics.median(v)


def run(trials: int, oracle_trials: int, ns, ds, out):
    import torch

    # the oracle's OpenMP threads must not spin on the host cores while the
    # GPU cells are timed (measured: 3x outliers in the cell after an oracle
    # call); the oracle runs in a second pass, after every GPU cell
    os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
    import paper_2601_01405_b200 as bm
    from oracle import oracle as O

    bm.load()
    cells = []
    t_start = time.time()
    for n in ns:
        for D in ds:
            eps = gen.cube_eps(D)
            dev, e2e = [], []
            L = M = E = None
            # every trial's cloud is generated (and uploaded) before the timed
            # runs, so they run back to back (host generation between runs let
            # the idle GPU change clocks: 10x outliers)
            Xh_all = [gen.cube_cloud(n, D, t) for t in range(trials)]
            Xd_all = [torch.from_numpy(x).cuda() for x in Xh_all]
            # warm-up (untimed): at least 3 covers and 0.3 s of
            # back-to-back GPU work, so the GPU leaves its idle clocks first
            # (the host-side generation above leaves it idle for up to a second)
            tw = time.perf_counter()
            for i in range(1000):
                bm.cover_build(Xd_all[i % trials], "l2", eps).free()
                torch.cuda.synchronize()
                if i >= 2 and time.perf_counter() - tw > 0.3:
                    break
            # no collector pass inside a timed call (the wrapper's Python work
            # after the library returns sits inside the event bracket)
            gc.collect()
            gc.disable()
            for t in range(trials):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                c = bm.cover_build(Xd_all[t], "l2", eps)
                b.record()
                torch.cuda.synchronize()
                dev.append(a.elapsed_time(b))
                if t == 0:
                    L, M, E = c.L, c.M, c.E
                c.free()
            bm.cover_build_host(Xh_all[0], "l2", eps)
            for t in range(trials):
                t0 = time.perf_counter()
                h = bm.cover_build_host(Xh_all[t], "l2", eps)
                e2e.append((time.perf_counter() - t0) * 1e3)
                del h
            gc.enable()
            del Xd_all
            rec = {"row": "NEXT-4 paper grid", "n": n, "D": D, "eps": eps, "L": L, "M": M, "E": E,
                   "trials": trials, "device_ms": round(median(dev), 4),
                   "device_ms_min": round(min(dev), 4), "device_ms_all": [round(x, 2) for x in dev],
                   "device_ms_p90": round(sorted(dev)[int(0.9 * (len(dev) - 1))], 4),
                   "e2e_ms": round(median(e2e), 4),
                   "oracle_trials": oracle_trials}
            cells.append(rec)
    for rec in cells:   # second pass: the oracle beside every cell
        n, D, eps = rec["n"], rec["D"], rec["eps"]
        orc = []
        for t in range(oracle_trials):
            Xh = gen.cube_cloud(n, D, t)
            t0 = time.perf_counter()
            o = O.cover(Xh, "l2", eps)
            orc.append((time.perf_counter() - t0) * 1e3)
            if t == 0:
                assert o.L == rec["L"], f"cell ({n}, {D}): oracle L {o.L} != GPU L {rec['L']}"
        rec["oracle_ms"] = round(median(orc), 3) if orc else None
        rec["speedup_e2e"] = round(median(orc) / rec["e2e_ms"], 1) if orc else None
        print(json.dumps(rec), flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")
    fits = []
    for key in ("e2e_ms", "device_ms", "oracle_ms"):
        for n in ns:
            row = [c for c in cells if c["n"] == n and c[key]]
            if len(row) >= 2:
                f = fit_power_law([c["D"] for c in row], [c[key] for c in row])
                fits.append({"row": "NEXT-4 fit", "time": key, "vs": "D", "at_n": n,
                             **{k: round(v, 4) for k, v in f.items()}})
        for D in ds:
            row = [c for c in cells if c["D"] == D and c[key]]
            if len(row) >= 2:
                f = fit_power_law([c["n"] for c in row], [c[key] for c in row])
                fits.append({"row": "NEXT-4 fit", "time": key, "vs": "n", "at_D": D,
                             **{k: round(v, 4) for k, v in f.items()}})
    for f in fits:
        print(json.dumps(f), flush=True)
        if out:
            out.write(json.dumps(f) + "\n")
    print(json.dumps({"row": "done", "seconds": round(time.time() - t_start, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=65)
    ap.add_argument("--oracle-trials", type=int, default=3)
    ap.add_argument("--n", default=",".join(map(str, gen.PAPER_GRID_N)))
    ap.add_argument("--D", default=",".join(map(str, gen.PAPER_GRID_D)))
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ns = [int(v) for v in a.n.split(",")]
    ds = [int(v) for v in a.D.split(",")]
    out = open(a.out, "w") if a.out else None
    run(a.trials, a.oracle_trials, ns, ds, out)


if __name__ == "__main__":
    main()
