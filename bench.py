"""Benchmark: evaluated neighbours/s (NSE/s) of the SAW search at L=201.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One "step" = one batch of walks (BASELINE config 4): every GPU runs
`--walkers-per-gpu` (default 2^20) independent walks of n = 8*D steps at
L=201 with seeds derived on device from (master_seed=1, batch, global walker),
then the batch is merged across ranks (one NCCL all_gather of the per-rank
summaries, ~32 B per rank).
Weak scaling: per-GPU work is fixed as N grows.

value  = sum over ranks of steps*(D-1) / max over ranks of the device time of
         the K timed batches (CUDA events on the launching stream, L2 flushed
         between batches).
e2e    = the same metric through the reference-facing host-buffer drop-in
         (sk_saw_batch_host == _kernels.saw_batch): host seeds in, per-walk
         outputs out, copies inside the timed region.
--impl reference: the reference's CPU algorithm (the oracle port,
         oracle/sokol_oracle.c, all host cores) on a bounded sample of the
         same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L_DEFAULT = 201
METRIC = "evaluated neighbours/sec (NSE/s) at L=201"
UNIT = "NSE/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--length", type=int, default=L_DEFAULT)
    ap.add_argument("--walkers-per-gpu", type=int, default=1 << 20)
    ap.add_argument("--walk-factor", type=int, default=8)
    ap.add_argument("--master-seed", type=int, default=1)
    ap.add_argument("--variant", default="auto", choices=["auto", "scalar", "fast"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-walkers", type=int, default=0, help="walkers per e2e step (0 = walkers-per-gpu)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N>1 (gloo lets 2 ranks share one GPU in tests)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------ CPU baseline --
def cpu_baseline(L: int, walk_factor: int, master: int, seconds: float) -> dict:
    """The reference algorithm on all host cores (oracle port), bounded."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    oracle.build()
    cores = oracle.num_procs()
    d = (L + 1) // 2
    n = walk_factor * d
    per = 4 * cores  # walkers = 4 * os.cpu_count()
    oracle.batch_outputs(L, n, oracle.derive_walk_seeds(master, 10**6, cores))  # warm-up
    total = 0
    walks = 0
    t0 = time.perf_counter()
    b = 0
    while True:
        seeds = oracle.derive_walk_seeds(master, b, per)
        _, _, st, _ = oracle.batch_outputs(L, n, seeds)
        total += int(st.sum()) * (d - 1)
        walks += per
        b += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": total / el, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{walks} walks of L={L}, n={n} ({b} batches of {per}, master_seed={master}) in {el:.1f}s "
                      f"on {cores} threads (oracle/sokol_oracle.c, pthreads)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    L = args.length
    d = (L + 1) // 2
    # each step is a bounded sample (~seconds) of the same workload
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(L, args.walk_factor, args.master_seed, 1.0)
    for _ in range(args.steps):
        vals.append(cpu_baseline(L, args.walk_factor, args.master_seed, max(2.0, args.cpu_seconds / max(1, args.steps))))
    v = sum(x["value"] for x in vals) / len(vals)
    cb = dict(vals[-1])
    cb["value"] = v
    per_step_nse = 4 * cb["cores"] * 8 * d * (d - 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_nse / v * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic: random starts from derive_walk_seed(1, batch, walker)",
        "config": {"workload": f"L={L} throughput (bounded CPU sample per step)", "L": L, "n": args.walk_factor * d,
                   "walkers_per_step": 4 * cb["cores"]},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ native --
def run_native(args):
    import torch
    import torch.distributed as dist

    from paper_2210_15962_b200 import _lib, engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    gpu = local % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    pg = None
    if world > 1 or "MASTER_ADDR" in os.environ:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        pg = dist.group.WORLD
    mdev = dev if args.backend == "nccl" else torch.device("cpu")  # merge tensors live here
    lib = _lib.load()
    _lib.set_variant({"auto": 0, "scalar": 1, "fast": 2}[args.variant])

    L = args.length
    D = (L + 1) // 2
    nw = (D + 63) // 64
    n = args.walk_factor * D
    Wg = args.walkers_per_gpu
    begin = rank * Wg
    stream = torch.cuda.current_stream(dev)
    summ = torch.empty(engine.SUMMARY_WORDS, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def launch(batch):
        _lib.check(lib.sk_saw_batch(L, n, None, args.master_seed, batch, begin, Wg, None, None, None, None,
                                    summ.data_ptr(), stream.cuda_stream))

    def merge():
        loc = engine.decode_summary(summ.cpu().numpy().view(np.uint64), nw)
        if pg is None:
            return loc
        return engine.merge_across_ranks(loc, loc.steps_sum if loc else 0, nw, pg, mdev)

    for b in range(args.warmup):
        launch(1000 + b)
        merge()

    sampler = ClockSampler(gpu)
    sampler.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    total_steps = 0
    best = None
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for b in range(args.steps):
        flush.zero_()
        starts[b].record(stream)
        launch(b)
        res = merge()  # 80-byte D2H (+ one NCCL all_gather across ranks)
        ends[b].record(stream)
        total_steps += res.steps_sum
        if best is None or res.best_E < best:
            best = res.best_E
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([dev_ms], dtype=torch.float64, device=mdev)
    if pg is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    nse = total_steps * (D - 1)  # total_steps already summed over ranks by the merge
    value = nse / (dev_ms / 1e3)

    # ---- roofline of the walk kernel (one launch per step) ----------------
    roof = roofline(L, n, Wg, value / max(1, world), dev_ms, clocks)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: random starts from device-derived splitmix64 seeds (derive_walk_seed)",
        "config": {"workload": f"L={L} throughput: {Wg} walks/GPU/batch, walk_factor {args.walk_factor}, "
                               f"master_seed {args.master_seed}",
                   "L": L, "n": n, "walkers_per_gpu": Wg, "global_walkers": Wg * world,
                   "parallelism": f"walker-sharded x{world}", "variant": args.variant,
                   "l2": "flushed between batches (256 MiB memset); walk state is on-chip"},
        "walk_steps_per_s": value / (D - 1),
        "lag_terms_per_s": value * D,
        "best_E_seen": best,
        "wall_s": wall,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": 3 * args.steps,
    }
    if not args.no_e2e:
        line["e2e"] = e2e(args, lib, rank, world, mdev, pg)
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(L, args.walk_factor, args.master_seed, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        dist.destroy_process_group()


def e2e(args, lib, rank, world, dev, pg):
    """NSE/s through the host-buffer drop-in (sk_saw_batch_host)."""
    import torch
    import torch.distributed as dist

    from paper_2210_15962_b200 import _lib
    from paper_2210_15962_b200.runner import derive_walk_seed  # noqa: F401

    L = args.length
    D = (L + 1) // 2
    nw = (D + 63) // 64
    n = args.walk_factor * D
    W = args.e2e_walkers or args.walkers_per_gpu
    steps = max(1, min(args.steps, 3))
    seeds = [host_seeds(args.master_seed, 500 + b, rank * W, W) for b in range(steps + 1)]
    be = np.empty(W, np.int64)
    bw = np.empty((W, nw), np.uint64)
    st = np.empty(W, np.int64)
    dd = np.empty(W, np.uint8)

    def call(s):
        _lib.check(lib.sk_saw_batch_host(L, n, s.ctypes.data, W, be.ctypes.data, bw.ctypes.data,
                                         st.ctypes.data, dd.ctypes.data))

    call(seeds[-1])  # warm-up
    if pg is not None:
        dist.barrier()
    total = 0
    t0 = time.perf_counter()
    for b in range(steps):
        call(seeds[b])
        total += int(st.sum())
    el = time.perf_counter() - t0
    if pg is not None:
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        tn = torch.tensor([float(total)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dist.all_reduce(tn, op=dist.ReduceOp.SUM)
        el, total = float(te.item()), float(tn.item())
    return {"value": total * (D - 1) / el, "unit": UNIT, "h2d_bytes_per_step": W * 8,
            "d2h_bytes_per_step": W * (8 + 8 * nw + 8 + 1),
            "path": "sk_saw_batch_host (drop-in of _kernels.saw_batch, host numpy buffers)",
            "walkers_per_step": W, "steps": steps}


def host_seeds(master, batch, begin, W):
    """derive_walk_seed vectorised over walkers (runner.py:53-57)."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)

    def mix(z):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))

    with np.errstate(over="ignore"):
        h = mix(np.uint64(master) ^ np.uint64(0x9E3779B97F4A7C15))
        h = mix(h ^ np.uint64(batch))
        w = np.arange(begin, begin + W, dtype=np.uint64)
        return np.ascontiguousarray(mix(h ^ w) & M)


def mma_per_step(L: int) -> int:
    """mma.sync.m16n8k16 per walk step of the production evaluator
    (eval_tc.cuh, every L <= 1023): the sum over 128-neighbour tiles tau of
    the k-block range [mlo(tau), mhi(tau)]."""
    D = (L + 1) // 2
    NI = (D + 15) // 16
    MT = (NI + 7) // 8
    tot = 0
    for tau in range(MT):
        amax = min(8 * tau + 7, NI - 1)
        tot += (NI - 4 * tau - 1) - (-((amax + 1) >> 1)) + 1
    return tot


def roofline(L, n, W, nse_per_s_gpu, dev_ms, clocks):
    """The walk step is bound by on-chip throughput, not HBM:
    shared-memory wavefronts (128 B each, one per SM per clock) and
    instruction issue (4 warp-instructions per SM per clock).  Per walk step
    counts of both come from the committed ncu capture of this launch
    (profiles/ncu_walk_kernel.json) and are multiplied by the live steps/s;
    "bound" names the higher fraction.  The tensor pipe (HMMA count per step
    x steps/s against the measured mma.sync rate) and the lag-term INT32
    equivalence are reported beside it."""
    D = (L + 1) // 2
    steps_per_s = nse_per_s_gpu / (D - 1)
    peaks = load_peaks()
    ncu = load_ncu(L, W)
    mhz = clocks.get("sm_mhz") or 1965.0
    issue_peak = 148 * 4 * mhz * 1e6 / 1e9  # Gwarp-inst/s
    smem_peak = 148 * 128 * mhz * 1e6 / 1e9  # GB/s: one 128-byte shared-memory wavefront per SM per clock
    ips = ncu.get("inst_per_walk_step")
    wps = ncu.get("smem_wavefronts_per_walk_step")
    issue = ips * steps_per_s / 1e9 if ips else None
    smem = wps * 128 * steps_per_s / 1e9 if wps else None
    mma = mma_per_step(L)
    tau = nse_per_s_gpu * D
    cand = {"smem": (smem, smem_peak, "GB/s", "shared-memory data pipe: 148 SM x 128 B/clk (1 wavefront/clk) at the "
                     f"run's median SM clock ({mhz:.0f} MHz)"),
            "issue": (issue, issue_peak, "Gwarp-inst/s", "instruction issue: 148 SM x 4 schedulers x 1 warp-inst/clk "
                      f"at the run's median SM clock ({mhz:.0f} MHz)")}
    bound = max(cand, key=lambda k: (cand[k][0] or 0) / cand[k][1])
    achieved, peak, unit, src = cand[bound]
    return {
        "bound": bound,
        "achieved": achieved,
        "peak": peak,
        "unit": unit,
        "frac": achieved / peak if achieved else None,
        "traffic": ncu.get("traffic_bytes_per_launch"),
        "peak_source": src,
        "per_walk_step": {"warp_inst": ips, "smem_wavefronts": wps, "mma": mma},
        "issue": {"achieved": issue, "peak": issue_peak, "unit": "Gwarp-inst/s",
                  "frac": issue / issue_peak if issue else None},
        "smem": {"achieved": smem, "peak": smem_peak, "unit": "GB/s", "frac": smem / smem_peak if smem else None},
        "pipes": {
            "tensor": {"mma_per_step": mma, "achieved_mma_per_s": mma * steps_per_s,
                       "peak_mma_per_s": peaks["hmma_per_s"],
                       "frac": mma * steps_per_s / peaks["hmma_per_s"] if peaks["hmma_per_s"] else None,
                       "peak_source": peaks["hmma_src"]},
            "ncu": ncu,
        },
        "int32_equivalent": {
            "note": "equivalence metric, not a ceiling: lag-terms x 2 INT32 ops / measured IMAD peak; the "
                    "contraction runs on the tensor pipe, so values above 1 are expected",
            "achieved": tau * 2 / 1e12, "peak": peaks["int_tops"], "unit": "Tops/s",
            "frac": tau * 2 / 1e12 / peaks["int_tops"] if peaks["int_tops"] else None,
            "algorithmic_unit": "lag-term tau = one (neighbour, even lag) v(2v-C) MAC; D*(D-1) per walk step, "
                                f"D={D} per NSE",
            "tau_per_s_per_gpu": tau},
    }


def load_ncu(L, W):
    """DRAM traffic and pipe utilisation of the walk kernel from the committed
    ncu --set full capture of this bench's launch (profiles/ncu_walk_kernel.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_walk_kernel.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        d = json.load(f)
    out = {k: d[k] for k in ("source", "kernel", "tensor_pipe_pct", "alu_pipe_pct", "fma_pipe_pct", "lsu_pipe_pct",
                             "issue_busy_pct", "warps_per_sm", "registers", "smem_wavefronts_pct",
                             "smem_ld_bank_conflict_share", "stall_top")
           if k in d}
    if d.get("L") == L and d.get("inst_executed") and d.get("walk_steps"):
        out["inst_per_walk_step"] = d["inst_executed"] / d["walk_steps"]
        if d.get("smem_wavefronts"):
            out["smem_wavefronts_per_walk_step"] = d["smem_wavefronts"] / d["walk_steps"]
    if d.get("L") == L and d.get("walks") and d.get("dram_bytes") is not None:
        out["traffic_bytes_per_launch"] = d["dram_bytes"] * (W / d["walks"])
        out["traffic_note"] = f"dram read+write of one captured launch ({d['walks']} walks), scaled to {W} walks"
    return out


def load_peaks():
    """INT32 and mma.sync peaks: profiles/microbench_peaks.json (measured on
    B200 by tools/microbench.cu) if present, else the theoretical IMAD rate."""
    out = {"int_tops": 2 * 148 * 64 * 1.965e9 / 1e12, "int_src": "theoretical IMAD 64 lanes/clk/SM x 148 SM x 1965 MHz (x2 ops)",
           "hmma_per_s": None, "hmma_src": None}
    p = os.path.join(ROOT, "profiles", "microbench_peaks.json")
    if os.path.exists(p):
        with open(p) as f:
            mb = json.load(f)
        if mb.get("imad_tops"):
            out["int_tops"] = mb["imad_tops"]
            out["int_src"] = f"measured IMAD (profiles/microbench_peaks.json, {mb.get('when', '')})"
        if mb.get("hmma_m16n8k16_f16f32_per_s"):
            out["hmma_per_s"] = mb["hmma_m16n8k16_f16f32_per_s"]
            out["hmma_src"] = f"measured mma.sync.m16n8k16 f16->f32 (profiles/microbench_peaks.json, {mb.get('when', '')})"
    return out


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_native(a)
