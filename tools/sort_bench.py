"""Radix-sort throughput on its own (diagnostics): python tools/sort_bench.py [n] [bits] [reps]

Times bm_debug_radix_sort_u64 on n uniformly random keys of `bits` bits with
CUDA events and reports the HBM rate on the algorithmic traffic of an LSD
sort: one histogram read (8 B / key) plus ceil(bits / 8) scatter passes of
8 B read + 8 B write per key.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_01405_b200 import bm as B  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 140_000_000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 39
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(0)
src = torch.randint(0, 2 ** bits, (n,), device="cuda", generator=g, dtype=torch.int64)
k = src.clone()
B.radix_sort_u64(k, bits)   # warm-up (allocations, attributes)
ok = bool(torch.equal(k, torch.sort(src).values))
passes = math.ceil(bits / 8)
traffic = n * 8 * (1 + 2 * passes)
ts = []
for _ in range(reps):
    k.copy_(src)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    B.radix_sort_u64(k, bits)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts)[len(ts) // 2]
print(f"radix sort n={n} bits={bits} passes={passes}: {ms:.3f} ms, "
      f"{traffic / ms / 1e6:.0f} GB/s on {traffic / 1e9:.2f} GB algorithmic, "
      f"{n / ms / 1e6:.2f} Gkeys/s, correct={ok}")
