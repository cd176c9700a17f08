"""Extract the walk kernel's roofline evidence from an ncu --set full report
into profiles/ncu_walk_kernel.json (read by bench.py for roofline.traffic).

    python tools/ncu_to_json.py gpurun_out/prof_bench.ncu-rep L WALKS [N] > profiles/ncu_walk_kernel.json

N = steps per walk (default 8 * D): walk_steps = WALKS * N, from which
bench.py derives warp-instructions per walk step (dead ends are negligible at
n = 8 D; the captured launch's own step count can be passed instead).
"""
import csv
import json
import subprocess
import sys

rep, L, W = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
N = int(sys.argv[4]) if len(sys.argv) > 4 else 8 * ((L + 1) // 2)
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
names, units, vals = raw[0], raw[1], raw[2]


def get(key):
    if key not in names:
        return None
    v = vals[names.index(key)].replace(",", "")
    u = units[names.index(key)]
    try:
        x = float(v)
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}.get(u, 1)
    return x * scale


out = {
    "source": rep.split("/")[-1] + " (ncu --set full --clock-control none, one timed bench launch)",
    "L": L, "walks": W, "walk_steps": W * N,
    "kernel": vals[names.index("Kernel Name")] if "Kernel Name" in names else None,
    "duration_ns": get("gpu__time_duration.sum"),
    "dram_bytes": (get("dram__bytes_read.sum") or 0) + (get("dram__bytes_write.sum") or 0),
    "tensor_pipe_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": get("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "issue_busy_pct": get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "warps_per_sm": get("sm__warps_active.avg.per_cycle_active"),
    "registers": get("launch__registers_per_thread"),
    "inst_executed": get("smsp__inst_executed.sum"),
    "smem_wavefronts": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "smem_wavefronts_pct": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "smem_ld_bank_conflict_share": (get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum") or 0)
    / max(1.0, get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum") or 1.0),
}
print(json.dumps(out, indent=1))
