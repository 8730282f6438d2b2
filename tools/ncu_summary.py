"""Summarise an `ncu --set full` report (.ncu-rep) into the metrics the
roofline cares about: duration, DRAM bytes, pipe utilisation, issue, occupancy.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import re
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe cycles %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe cycles %"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


# memory-hierarchy throughputs and the top stall reasons (any name matching)
EXTRA = re.compile(r"^(lts__t_(bytes|sectors)[^,]*(sum|pct_of_peak_sustained_elapsed)$"
                   r"|lts__throughput\.avg\.pct_of_peak_sustained_elapsed"
                   r"|l1tex__m_xbar2l1tex_read_bytes\.sum(\.per_second)?"
                   r"|l1tex__throughput\.avg\.pct_of_peak_sustained_active"
                   r"|smsp__average_warp(s|_latency)_issue_stalled_[a-z_]+_per_issue_active\.ratio)")


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no data")
        return
    h, units = rows[0], rows[1]
    tensor_cols = [c for c in h if "pipe_tc" in c or "tensor" in c and "pct" in c]
    for r in rows[2:]:
        print(f"kernel: {r[h.index('Kernel Name')]}")
        for key, label in WANT:
            if key in h:
                i = h.index(key)
                print(f"  {label:32s} {r[i]} {units[i]}")
        stalls = []
        for i, c in enumerate(h):
            if EXTRA.match(c) and r[i] not in ("", "n/a"):
                if "issue_stalled" in c:
                    try:
                        stalls.append((float(r[i].replace(",", "")), c))
                    except ValueError:
                        pass
                else:
                    print(f"  {c:60s} {r[i]} {units[i]}")
        for v, c in sorted(stalls, reverse=True)[:8]:
            print(f"  {c:60s} {v:.3f}")
        for c in tensor_cols:
            i = h.index(c)
            if r[i] not in ("", "0", "n/a"):
                print(f"  {c:60s} {r[i]} {units[i]}")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
