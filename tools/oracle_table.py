"""The CPU oracle baseline table of SURVEY §8(d) "Oracle timing", run on the
GPU box's host: full C1, C2 and C4, prefixes of C3 (eps 2/4/8) and C5 (L1,
cosine) with the full-size time extrapolated as n * L_gpu / (prefix pairs per
second) and labelled so, plus the 1-thread time of C1 and C2.  Reports nproc,
the CPU model and the OpenMP thread count.  The oracle is run as it stands
(never tuned for this).

    python tools/oracle_table.py > profiles/oracle_table_r02.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from bench import cpu_model  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads import gen  # noqa: E402

PREFIX = {"c3_e2": 50_000, "c3_e4": 50_000, "c3_e8": 100_000, "c5_l1": 250_000,
          "c5_cos": 250_000}


def gpu_L(w, X):
    c = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps)
    L = c.L
    c.free()
    return L


def main():
    threads = O.set_threads(0)
    head = {"nproc": os.cpu_count(), "cpu_model": cpu_model(), "omp_threads": threads}
    print(json.dumps({"host": head}), flush=True)
    for name in ("c1", "c2", "c4", "c3_e2", "c3_e4", "c3_e8", "c5_l1", "c5_cos"):
        w = gen.get(name)
        X = gen.generate(w)
        m = PREFIX.get(name, len(X))
        t0 = time.perf_counter()
        c = O.cover(X[:m], w.metric, w.eps)
        dt = time.perf_counter() - t0
        rec = {"workload": name, "n_sample": m, "L_sample": c.L, "seconds": round(dt, 3),
               "pairs_per_s": m * c.L / dt, "threads": threads}
        if m < len(X):
            L = gpu_L(w, X)
            rec.update({"kind": "prefix", "L_full_gpu": L,
                        "extrapolated_full_s": round(len(X) * L / rec["pairs_per_s"], 1),
                        "note": "full-size oracle time EXTRAPOLATED from the prefix rate"})
        else:
            rec["kind"] = "full"
        if name in ("c1", "c2"):
            O.set_threads(1)
            t0 = time.perf_counter()
            O.cover(X, w.metric, w.eps)
            rec["seconds_1_thread"] = round(time.perf_counter() - t0, 3)
            O.set_threads(threads)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
