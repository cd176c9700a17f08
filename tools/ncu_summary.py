"""Summarise an ncu --set full capture: key metrics, per-opcode mix, top source lines."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


want = ["Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Executed Instructions", "No Eligible",
        "Eligible Warps Per Scheduler", "L1/TEX Cache Throughput", "Compute (SM) Throughput", "DRAM Throughput",
        "Grid Size", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"]
rows = list(csv.reader(run("--page", "details", "--csv").splitlines()))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
if len(raw) > 2:
    names, units, vals = raw[0], raw[1], raw[2]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_tensor.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
        if key in names:
            i = names.index(key)
            print(f"{key:70s} {vals[i]} {units[i]}")
sass = list(csv.reader(run("--page", "source", "--csv", "--print-source=sass").splitlines()))
h2 = sass[1]
data = [dict(zip(h2, r)) for r in sass[2:] if len(r) == len(h2)]
ie = lambda d: int(d["Instructions Executed"] or 0)
tot = sum(ie(d) for d in data) or 1
samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
c, s = Counter(), Counter()
for d in data:
    toks = d["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += ie(d)
    s[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print("\nopcode mix (inst%, stall-sample%):")
for op, v in c.most_common(16):
    print(f"  {op:10s} {v / tot * 100:6.2f}% {s[op] / samp * 100:6.2f}%")
keys = [k for k in h2 if k.startswith("stall_") and "(Not" not in k]
tots = {k: sum(int(d[k] or 0) for d in data) for k in keys}
print("stalls:", ", ".join(f"{k[6:]}={v / samp * 100:.1f}%" for k, v in sorted(tots.items(), key=lambda x: -x[1])[:8]))
wf = sum(int(d["L1 Wavefronts Shared"] or 0) for d in data)
wfi = sum(int(d["L1 Wavefronts Shared Ideal"] or 0) for d in data)
print(f"smem wavefronts {wf} (ideal {wfi}), total warp-instructions {tot}")
cs = list(csv.reader(run("--page", "source", "--csv", "--print-source=cuda,sass").splitlines()))
out, cur, hdr3 = [], None, None
for r in cs:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr3 = r
        continue
    if hdr3 and len(r) == len(hdr3) and r[2] == "-":
        try:
            out.append((int(r[7] or 0), int(r[4] or 0), cur, r[0], r[1][:88]))
        except ValueError:
            pass
t2 = sum(o[0] for o in out) or 1
s2 = sum(o[1] for o in out) or 1
out.sort(reverse=True)
print(f"\ntop source lines (inst%, stall%):")
for a, b, f, ln, src in out[:top]:
    print(f"  {a / t2 * 100:5.1f}% {b / s2 * 100:5.1f}%  {f}:{ln}  {src}")
