#!/usr/bin/env python
"""Benchmark of the B200 Ball Mapper cover construction (BASELINE.json metric:
"point-landmark distance evals/sec and cover build time; % of B200 roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
    python bench.py --impl reference ...        # the CPU oracle arm

One step = one full bm_cover_build (greedy eps-net, membership, CSR, edges) of
the workload.  The default workload is BASELINE.json configs[1] (C2).  Inputs
are resident in HBM before the timed region; L2 is flushed (a 256 MiB write)
before every timed step, outside the step's CUDA-event bracket.  N > 1 runs N
independent replicas (the path does not shard across
GPUs in this build), one per rank, timed on the device, max over ranks.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "point-landmark distance evals/sec"
UNIT = "evals/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--n", type=int, default=0, help="prefix size (0 = the full workload)")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--path", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    return ap.parse_args(argv)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bm_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("BM_CLOCK_MS", "100")], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        sm_load = [s for s in sm if s > 500] or sm
        sm_load.sort()
        med = sm_load[len(sm_load) // 2] if sm_load else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def roofline_for(w, L, kernel_ms, n, peaks, path_used, step_ms, st=None):
    if path_used == 2:
        return roofline_tensor(w, L, kernel_ms, n, peaks, step_ms, st)
    return roofline_alu(w, L, kernel_ms, n, peaks)


def _traffic(w):
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            return json.load(open(tp)).get(w.name, {}).get("member_kernel_dram_bytes")
        except Exception:
            return None
    return None


def roofline_tensor(w, L, kernel_ms, n, peaks, step_ms, st=None):
    """tcgen05 contraction, two ceilings:
      tensor: 2*d algorithmic ops per pair (true d, not the padded K) against
        the measured bf16 peak x the nominal ratio (tf32 0.5, int8 2.0); burst
        figure for short steps, sustained for steps > 0.5 s;
      tmem: every pair's 4-byte accumulator is read from tensor memory once,
        against 64 B/clk/SM x 148 SMs x sm_max_mhz (the guide's LDTM rate,
        confirmed on this B200: 61 B/clk/SM with a TMEM-read-only epilogue,
        tools/tc_probe_c2.py mode 2).
    The reported bound is the ceiling the kernel is closer to (the binding
    one); the other is kept under "other"."""
    sustained = step_ms > 500.0
    bf16 = float(peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"])
    ratio = 0.5 if w.dtype == "f32" else 2.0
    peak = bf16 * ratio
    ks = kernel_ms * 1e-3
    # executed work: with the tile-level pruning (cells.cu) only the contracted
    # 128 x 256 tiles and the 128 x 32 chunks read from TMEM count against the
    # ceilings; without it (or on paths that do not report) every pair does
    tiles = getattr(st, "tc_tiles_run", 0) if st is not None else 0
    chunks = getattr(st, "tc_chunks_run", 0) if st is not None else 0
    ops = 2.0 * w.d * (tiles * 128.0 * 256.0 if tiles else float(n) * L)
    achieved = ops / ks / 1e12 if kernel_ms > 0 else 0.0
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    tmem_peak = 64.0 * 148 * clk / 1e9                      # GB/s
    tmem_bytes = (chunks * 128.0 * 32.0 if chunks else float(n) * L) * 4.0
    tmem_ach = tmem_bytes / ks / 1e9 if kernel_ms > 0 else 0.0
    kern = "k_tc (tcgen05 " + ("tf32" if w.dtype == "f32" else "int8") + ", per-tile)"
    tensor = {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3),
              "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
              "ops_per_pair": 2 * w.d,
              "peak_basis": f"measured bf16 {'sustained' if sustained else 'burst'} "
                            f"{bf16} x {ratio} (nominal {'tf32' if ratio == 0.5 else 'int8'} "
                            f"ratio)"}
    tmem = {"bound": "tmem", "achieved": round(tmem_ach, 1), "peak": round(tmem_peak, 1),
            "unit": "GB/s", "frac": round(tmem_ach / tmem_peak, 4),
            "bytes_per_pair": 4,
            "peak_basis": "64 B/clk/SM TMEM read (guide; 61 B/clk measured here) x 148 x "
                          f"{clk / 1e6:.0f} MHz"}
    main, other = (tmem, tensor) if tmem["frac"] > tensor["frac"] else (tensor, tmem)
    out = dict(main)
    out.update({"kernel": kern, "traffic": _traffic(w), "kernel_ms": round(kernel_ms, 5),
                "other": other,
                "work_basis": "executed tiles / TMEM chunks" if tiles else "n x L pairs",
                "decided_pairs_per_s": round(float(n) * L / ks, 1) if ks > 0 else None})
    if st is not None and (getattr(st, "tc_tiles_skipped", 0) or getattr(st, "tc_chunks_skipped", 0)):
        tt = st.tc_tiles_run + st.tc_tiles_skipped
        cc = st.tc_chunks_run + st.tc_chunks_skipped
        out["pruned"] = {"tiles_skipped_frac": round(st.tc_tiles_skipped / max(1, tt), 4),
                         "chunks_skipped_frac": round(st.tc_chunks_skipped / max(1, cc), 4)}
    return out


def roofline_alu(w, L, kernel_ms, n, peaks):
    """Dominant kernel = the membership pass (step B) on CUDA cores: bound
    'alu', algorithmic lane-instructions per pair against the issue rate of the
    unit doing the work (DESIGN.md §7 "Rooflines"):
      L1 f32 (8-bit SAD prefilter, d <= 64): ceil(d/4) VABSDIFF4 per pair, peak
        148 SM x 64 lanes x clock (half-rate instruction, measured 18.5 T/s);
      L2 f32 direct 2d (sub + fma), cosine d (fma), L1 f32 without the
        prefilter 2d, int L2 ceil(d/4) dp4a, int L1 2 ceil(d/4): peak
        148 SM x 128 lanes x clock (full-rate FP32/INT issue)."""
    d = w.d
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    if (w.dtype, w.metric) == ("f32", "l1") and d <= 64:
        per_pair, lanes, what = math.ceil(d / 4), 64, "VABSDIFF4 (half rate)"
    else:
        per_pair = {("f32", "l2"): 2 * d, ("f32", "l1"): 2 * d, ("f32", "cos"): d,
                    ("i8", "l2"): math.ceil(d / 4), ("u8", "l2"): math.ceil(d / 4),
                    ("i8", "l1"): 2 * math.ceil(d / 4), ("u8", "l1"): 2 * math.ceil(d / 4)}[
            (w.dtype, w.metric)]
        lanes, what = 128, "FP32/INT issue"
    peak = 148 * lanes * clk / 1e12
    ops = float(n) * L * per_pair
    achieved = ops / (kernel_ms * 1e-3) / 1e12 if kernel_ms > 0 else 0.0
    traffic = _traffic(w)
    return {"bound": "alu", "kernel": "k_pairs<MODE_MEMBER> (per-tile membership)",
            "achieved": round(achieved, 4),
            "peak": round(peak, 4), "unit": "Tinst/s", "frac": round(achieved / peak, 4),
            "traffic": traffic, "ops_per_pair": per_pair,
            "kernel_ms": round(kernel_ms, 5),
            "peak_basis": f"148 SM x {lanes} lanes x sm_max_mhz, {what} (DESIGN.md §7)"}


def cpu_baseline(w, X, budget_s: float):
    """The oracle as it stands on the host cores, bounded sample of the workload:
    the largest prefix whose greedy finishes within ~budget_s (full workload when
    it fits).  value = sample pairs (n_s * L_s) / oracle seconds."""
    from oracle import oracle as O
    cores = O.set_threads(0)
    n = X.shape[0]
    m = min(n, 20000)
    res = None
    while True:
        t0 = time.perf_counter()
        c = O.cover(X[:m], w.metric, w.eps)
        dt = time.perf_counter() - t0
        res = (m, c.L, dt)
        if m >= n or dt > budget_s / 4:
            break
        grow = max(2.0, min(8.0, (budget_s / 4) / max(dt, 1e-3)))
        m = min(n, int(m * math.sqrt(grow)))
    m, L, dt = res
    return {"value": m * L / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{'full' if m == n else 'prefix'} {w.name} n={m} (L={L}), 1 run, "
                      f"{dt:.2f}s", "seconds": round(dt, 3)}


# ----------------------------------------------------------------- arms
def max_over_ranks(x: float, world: int, device: str = "cuda") -> float:
    """Max of a per-rank time over all ranks (device timing rule: the job
    takes as long as its slowest replica).  Gloo on CPU tensors in the tests."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(world: int, pairs_per_replica: float, seconds: float) -> float:
    """Whole-job throughput: every replica evaluates pairs_per_replica pairs
    (weak scaling, no data-path collective), the job time is the max over ranks."""
    return world * pairs_per_replica / seconds


def run_reference(args):
    """--impl reference: the CPU oracle arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from workloads import gen
    w = gen.get(args.workload)
    X = gen.generate(w, args.n or None)
    cores = O.set_threads(0)
    # bounded sample per step: prefix sized so one step takes <= ~2 s
    m = min(X.shape[0], 20000)
    while True:
        t0 = time.perf_counter()
        O.cover(X[:m], w.metric, w.eps)
        dt = time.perf_counter() - t0
        if m >= X.shape[0] or dt > 0.5:
            break
        m = min(X.shape[0], m * 2)
    Xs = X[:m]
    for _ in range(args.warmup):
        O.cover(Xs, w.metric, w.eps)
    times, L = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c = O.cover(Xs, w.metric, w.eps)
        times.append(time.perf_counter() - t0)
        L = c.L
    ms = 1e3 * sum(times) / len(times)
    value = m * L / (ms * 1e-3)
    sample = f"{'full' if m == X.shape[0] else 'prefix'} {w.name} n={m} (L={L}) per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if w.dtype == "f32" else "int64", "data": "synthetic",
            "config": {"workload": w.name, "n": int(m), "d": w.d, "metric": w.metric,
                       "eps": w.eps, "L": int(L)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2601_01405_b200 as bm
    from workloads import gen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and not (world == 1 and args.gpus == 1):
        if world == 1:
            print(f"--gpus {args.gpus} needs torchrun with {args.gpus} ranks", file=sys.stderr)
            return 2
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = gen.get(args.workload)
    Xh = gen.generate(w, args.n or None)
    n, d = Xh.shape
    X = torch.from_numpy(Xh).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # the timed steps run without the library's per-step timing events: those
    # sit between the tile loop's kernels and break their programmatic
    # (PDL) overlap (measured: C2 0.41 ms plain vs 0.49 ms instrumented,
    # tools/timing_overhead.py); a separate instrumented pass below gives the
    # per-step breakdown and the membership kernel time for the roofline
    kw = dict(tile=args.tile, path=args.path, timing=False)
    kw_t = dict(tile=args.tile, path=args.path, timing=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    warm = max(args.warmup, 3)            # timing rule: >= 3 warm-up steps
    for _ in range(warm):
        bm.cover_build(X, w.metric, w.eps, **kw).free()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    # the sampler's start-up pause lets the clocks drop: two more untimed
    # steps, exactly as the timed ones (flush, events, build), bring them back
    for i in range(2):
        flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bm.cover_build(X, w.metric, w.eps, **kw).free()
        e1.record(stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier()
    covs_stats = []
    L = 0
    launches = 0
    import gc
    gc.collect()
    gc.disable()   # a collector pause between ev0 and the first launch would count
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                 # L2 flush outside the timed bracket
        ev[i][0].record(stream)
        cov = bm.cover_build(X, w.metric, w.eps, **kw)
        ev[i][1].record(stream)
        L, M, E, NPW = cov.L, cov.M, cov.E, cov.P
        launches += cov.stats.n_launches
        cov.free()
    barrier()
    gc.enable()
    clocks = sampler.stop()
    # instrumented pass (not timed): per-step breakdown, membership kernel time
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(i & 0xFF)
        cov = bm.cover_build(X, w.metric, w.eps, **kw_t)
        covs_stats.append(cov.stats)
        cov.free()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    ss = sorted(step_ms)
    step_stats = {"min": round(ss[0], 4), "median": round(ss[len(ss) // 2], 4),
                  "max": round(ss[-1], 4)}
    ms = max_over_ranks(ms, world)
    pairs = n * L
    value = whole_job_value(world, pairs, ms * 1e-3)

    # dominant kernel: membership pass, timed by library events on the launch stream
    kern_ms = sorted(s.step_ms["member_kernel"] for s in covs_stats)[len(covs_stats) // 2]
    kern_launches = covs_stats[-1].n_member_launches
    breakdown = {k: round(sorted(s.step_ms[k] for s in covs_stats)[len(covs_stats) // 2], 4)
                 for k in ("prep", "greedy", "member", "csr", "edges", "member_kernel")}
    peaks, peak_src = load_peaks()
    roof = roofline_for(w, L, kern_ms, n, peaks, covs_stats[-1].path_used, ms, covs_stats[-1])
    roof["peak_source"] = peak_src
    roof["share_of_step"] = round(kern_ms / ms, 4) if ms > 0 else None
    roof["launches_per_step"] = int(kern_launches)
    roof["avg_launch_ms"] = round(kern_ms / max(1, kern_launches), 5)
    roof["timing"] = ("CUDA events on the launch stream around every membership launch "
                      "(one per greedy tile), summed per step, median over the instrumented "
                      "steps (share_of_step relative to the uninstrumented step time)")

    # e2e through the public host-buffer entry point (H2D + D2H inside the timing)
    pinned = torch.from_numpy(Xh).pin_memory()
    e2e_times = []
    h2d = n * d * Xh.itemsize
    d2h = 0
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hc = bm.cover_build_host(pinned, w.metric, w.eps, tile=args.tile, path=args.path)
        e2e_times.append(time.perf_counter() - t0)
        d2h = 4 * hc.L + 8 * (hc.L + 1) + 4 * hc.M + 8 * (n + 1) + 4 * hc.M + 8 * hc.E
        hc.free()
    e2e_s = max_over_ranks(sorted(e2e_times)[len(e2e_times) // 2], world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, Xh, args.cpu_sample_seconds)

    last = covs_stats[-1]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"f32": "f32", "i8": "int8", "u8": "uint8"}[w.dtype],
            "data": "synthetic",
            "config": {"workload": w.name, "n": int(n), "d": int(d), "metric": w.metric,
                       "eps": w.eps, "L": int(L), "M": int(M), "E": int(E), "P": int(NPW),
                       "tile": int(last.tile_used), "path": ["auto", "cuda_core", "tensor"][
                           last.path_used], "l2": "flushed (256 MiB write) before each step",
                       "parallelism": "replicas" if world > 1 else "single"},
            "cover_ms": round(ms, 4),
            "step_ms_stats": step_stats, "step_ms_all": [round(x, 4) for x in step_ms],
            "breakdown_ms": breakdown,
            "breakdown_note": "library CUDA events per sub-step, separate instrumented steps "
                              "(the events break the tile loop's PDL overlap, so these sum to "
                              "more than ms_per_step)",
            "greedy": {"tiles": int(last.n_greedy_tiles), "evals": int(last.n_greedy_evals),
                       "band_pairs": int(last.n_band_pairs), "near_ties": int(last.n_near_ties)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": whole_job_value(world, pairs, e2e_s), "unit": UNIT, "seconds": round(e2e_s, 5),
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "clocks": clocks,
            "gpu_launches": int(launches)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
