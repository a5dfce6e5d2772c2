"""Benchmark of the B200 j2d5pt deep-temporal-blocking solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2|c1|c3a|c3b|c4|c5]

A bench "step" is one complete solve of the workload (e.g. C2 = all 10,000
Jacobi steps of a 1900^2 fp64 grid), inputs already resident in HBM
(generated on the device by the splitmix64 fill kernel, bit-identical to the
reference's random_interior). Metric (BASELINE.json): GCells/s = valid
cell-updates nx*ny*steps per second. Prints ONE JSON line on rank 0.

--impl reference times the reference's CPU algorithm on this host's cores:
the C restatement of jacobi_reference (oracle/j2d5pt_oracle.c, bitwise pinned
to the reference, pthreads over all host cores) on a bounded sample of the
same workload. The b200 line's cpu_baseline carries the same port plus the
BASELINE.md §4 legs with the reference's own structure (oracle/engine_port.py):
jacobi_reference's row-wise numpy loop on one pinned core, and the reference
DTB engine (run_dtb) with the B200 DeviceModel at threads=1 and threads=cores.

--gpus N > 1 runs the C5 weak-scaling series (32768 x 4096N fp64 y-slabs, one
rank per GPU, depth-16 halos) plus strong scaling at the fixed 32768^2; the
N=1 line (C2 headline) carries the same family's N=1 anchors under "c5".
Without a launcher, --gpus N > 1 re-launches itself under torch.distributed.run.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (nx, ny, steps, dtype, description)
    "c1": (256, 256, 100, "f64", "j2d5pt fp64 256x256, 100 steps (BASELINE config 1)"),
    "c2": (1900, 1900, 10000, "f64", "j2d5pt fp64 1900x1900, 10000 steps, smem-resident (BASELINE config 2)"),
    "c3a": (2700, 2700, 10000, "f32", "j2d5pt fp32 2700x2700, 10000 steps, smem-resident (BASELINE config 3)"),
    "c3b": (8192, 8192, 1000, "f32", "j2d5pt fp32 8192x8192, 1000 steps, streaming (BASELINE config 3)"),
    "c4": (16384, 16384, 1000, "f64", "j2d5pt fp64 16384x16384, 1000 steps, streaming (BASELINE config 4)"),
    # C5 weak-scaling series: 32768 x (4096 * N) fp64 y-slabs, depth-16 halo exchange
    "c5": (32768, 4096, 1000, "f64", "j2d5pt fp64 32768x(4096*N) y-slabs, 1000 steps, depth-16 "
                                     "NVLink halo exchange (BASELINE config 5, weak scaling)"),
}

METRIC = "j2d5pt GCells/s (fp64/fp32) at 1/2/4/8 B200 vs roofline and CPU reference"


def measured_peaks():
    """Roofline denominators: HBM from MEASURED_PEAKS.json (driver-written);
    smem and FP64/FP32 issue rates from this repo's B200 microbenchmarks
    (tools/microbench/peaks.cu, profiles/r01/microbench_peaks.log)."""
    peaks = {"hbm_gbs": 6545.3, "hbm_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        pass
    # microbench (148 SMs): LDS.128 235.2 B/SM/ns; DMUL/DADD 124.6 /SM/ns; FMUL/FADD 244.9 /SM/ns
    peaks["smem_gbs"] = 235.156 * 148
    peaks["fp64_gops"] = 124.563 * 148
    peaks["fp32_gops"] = 244.929 * 148
    return peaks


def ncu_traffic(kernel, dtype):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    newest committed ncu --set full capture (profiles/r02, else r01
    ncu_summary.json), or None."""
    summ = None
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_summary.json")) as fh:
                summ = json.load(fh)
            break
        except (OSError, ValueError):
            continue
    if summ is None:
        return None, None
    tag = "double" if dtype == "f64" else "float"
    for name, rec in summ.items():
        if name.startswith(kernel + "<" + tag):
            return rec["dram_bytes_read"] + rec["dram_bytes_write"], \
                f"{rec['capture']} ({rec['workload']}; DRAM read + write per launch of that capture)"
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    The nvidia-smi process is started when the sampler is created (before the
    warm-up: it takes a few hundred ms to deliver its first sample); `with
    sampler:` marks the timed window, and the summary keeps the samples that
    arrived inside it (or, for a window shorter than the 50 ms period, the
    first one after it)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []  # (arrival time, line)
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def __enter__(self):
        self.t0 = time.monotonic()
        return self

    def __exit__(self, *exc):
        self.t1 = time.monotonic()
        if self.proc is not None:
            # a window shorter than the sampling period: wait for one sample
            deadline = self.t1 + 1.0
            while (not any(ts >= self.t0 for ts, _ in self.lines)
                   and time.monotonic() < deadline and self.proc.poll() is None):
                time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = self.t1 if self.t1 is not None else float("inf")
        inside = [ln for ts, ln in self.lines if t0 <= ts <= t1 + 0.05]
        if not inside:
            after = [ln for ts, ln in self.lines if ts >= t0]
            inside = after[:1]
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_port():
    """The CPU port of the reference's path that can use every host core: the C
    restatement of jacobi_reference (oracle/j2d5pt_oracle.c, -ffp-contract=off,
    pthreads over rows; pinned bitwise to the reference), else the numpy one."""
    import os as _os
    import platform
    from oracle import jacobi_c, jacobi_numpy
    threads = _os.cpu_count() or 1
    model = platform.processor() or platform.machine()
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from oracle.ref import build_c_oracle
        build_c_oracle()

        def run(data, w, steps, dt):
            return jacobi_c(data, w, steps, dt, threads=threads)
        return run, threads, f"C port (pthreads, {threads} threads, {model})"
    except Exception:  # no C oracle on this host: the numpy restatement, one core
        return (lambda data, w, steps, dt: jacobi_numpy(data, w, steps, dt)), 1, \
            f"numpy port (1 core, {model})"


def _reference_legs(nx, ny):
    """BASELINE.md §4 legs with the reference's own structure
    (oracle/engine_port.py, bitwise-pinned to the reference's outputs):
    jacobi_reference's row-wise numpy loop on ONE pinned core, and the
    reference DTB engine run_dtb with the B200 DeviceModel (148 workers x
    232448 B) at threads=1 and threads=host cores, each on a bounded sample
    of whole time blocks (per-step cost is constant, so the rate carries)."""
    import numpy as np
    from oracle.engine_port import jacobi_rowwise, run_dtb_port
    from paper_2306_03336_b200 import DeviceModel, plan_device_tiles
    from paper_2306_03336_b200.grid import grid_new
    from paper_2306_03336_b200.prng import random_interior
    g = grid_new(nx, ny, random_interior(nx, ny, 1)).data
    w = (0.2, 0.2, 0.2, 1.0 - 4 * 0.2, 0.2)
    cores = os.cpu_count() or 1
    legs = []
    # 1. jacobi_reference on one core (single-threaded by contract)
    try:
        old = os.sched_getaffinity(0)
        pin = min(old)
        os.sched_setaffinity(0, {pin})
    except (AttributeError, OSError):
        old, pin = None, None
    try:
        t0 = time.perf_counter()
        jacobi_rowwise(g, w, 2)
        per = (time.perf_counter() - t0) / 2
        k = max(2, min(200, int(4.0 / per)))
        t0 = time.perf_counter()
        jacobi_rowwise(g, w, k)
        el = time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    legs.append({"leg": "jacobi_reference (oracle.py:19-34), row-wise numpy, 1 core"
                        + (f" (pinned to cpu {pin})" if pin is not None else ""),
                 "value": nx * ny * k / el / 1e9, "unit": "GCells/s", "cores": 1,
                 "sample": f"{nx}x{ny} f64, {k} steps, {el:.1f} s"})
    # 2. run_dtb (engine.py:305-326) with the B200 DeviceModel, one time block of T=2
    plan = plan_device_tiles((nx, ny), DeviceModel("b200", 148, 232448), 2)
    for threads in sorted({1, cores}):
        t0 = time.perf_counter()
        run_dtb_port(g, w, 2, plan, threads)
        el = time.perf_counter() - t0
        legs.append({"leg": f"run_dtb (engine.py:305-326), B200 DeviceModel 148 x 232448 B, "
                            f"t_depth 2, threads={threads}",
                     "value": nx * ny * 2 / el / 1e9, "unit": "GCells/s", "cores": threads,
                     "sample": f"{nx}x{ny} f64, one time block of 2 steps over "
                               f"{len(plan.tiles)} tiles, {el:.1f} s"})
    return legs


def cpu_reference_sample(nx, ny, dtype, budget_s=8.0, legs=True):
    """Time the reference algorithm (a bitwise-pinned CPU port of
    jacobi_reference, oracle.py:19-34) on all of this host's cores; with
    `legs`, also the reference-structured BASELINE.md §4 legs."""
    import numpy as np
    from paper_2306_03336_b200.grid import grid_new
    from paper_2306_03336_b200.prng import random_interior
    run, cores, what = _cpu_port()
    dt = np.float64 if dtype == "f64" else np.float32
    g = grid_new(nx, ny, random_interior(nx, ny, 1))
    w = (0.2, 0.2, 0.2, 1.0 - 4 * 0.2, 0.2)
    # per-step cost from a ~0.1 s calibration run (amortises the per-call
    # thread start and buffer copies), then ~budget_s of work
    n = 4
    while True:
        t0 = time.perf_counter()
        run(g.data, w, n, dt)
        el = time.perf_counter() - t0
        if el > 0.1 or n >= 1 << 20:
            break
        n *= 4
    steps = max(1, int(budget_s / (el / n)))
    t0 = time.perf_counter()
    run(g.data, w, steps, dt)
    el = time.perf_counter() - t0
    out = {"value": nx * ny * steps / el / 1e9, "unit": "GCells/s", "cores": cores,
           "kind": "port",
           "sample": f"{nx}x{ny} {dtype}, {steps} steps of the {what} restatement of "
                     f"jacobi_reference (oracle/, pinned to the reference), {el:.1f} s"}
    if legs:
        out["legs"] = _reference_legs(nx, ny)
    return out


def run_reference(args):
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    nx, ny, steps, dtype, desc = WORKLOADS[args.workload]
    import numpy as np
    from oracle import jacobi_numpy
    from paper_2306_03336_b200.grid import grid_new
    from paper_2306_03336_b200.prng import random_interior
    dt = np.float64 if dtype == "f64" else np.float32
    g = grid_new(nx, ny, random_interior(nx, ny, 1))
    w = (0.2, 0.2, 0.2, 1.0 - 4 * 0.2, 0.2)
    run, cores, what = _cpu_port()
    # bounded sample per bench step: ~2 s of the port's per-step cost (net of
    # the per-call overhead, which a long solve amortises)
    n = 4
    while True:
        t0 = time.perf_counter()
        run(g.data, w, n, dt)
        el = time.perf_counter() - t0
        if el > 0.1 or n >= 1 << 20:
            break
        n *= 4
    sample = max(1, min(steps, int(2.0 / (el / n))))
    for _ in range(args.warmup):
        run(g.data, w, sample, dt)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run(g.data, w, sample, dt)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = nx * ny * sample * args.steps / total / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GCells/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": desc, "nx": nx, "ny": ny, "solve_steps": steps,
                       "sample_steps_per_bench_step": sample},
            "cpu_baseline": {"value": value, "unit": "GCells/s", "cores": cores, "kind": "port",
                             "sample": f"{nx}x{ny} {dtype}, {sample} Jacobi steps per bench step "
                                       f"({what} restatement of jacobi_reference, bitwise "
                                       "pinned to the reference)"},
            "e2e": {"value": value, "unit": "GCells/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def slab_series(args, world, rank, local, ny, steps, exchange="auto"):
    """One C5-family measurement: a 32768 x ny fp64 domain in `world` y-slabs,
    one per rank (SlabSolver), depth-16 halos. Returns the whole-job rate
    (max over ranks) and the e2e leg, or None on ranks != 0."""
    import torch
    import torch.distributed as dist
    from paper_2306_03336_b200 import StencilWeights, j2d5pt_device, last_launch_count
    from paper_2306_03336_b200.prng import fill_random_rows_device
    from paper_2306_03336_b200.slab import SlabGeometry, SlabSolver
    nx, depth = WORKLOADS["c5"][0], 16
    dev = torch.device("cuda", local)
    geo = SlabGeometry(nx, ny, world, rank, depth)
    pitch = (nx + 2 + 31) // 32 * 32
    w = StencilWeights.diffusive(0.2)
    launches = [0]

    def local_solve(src, dst, lnx, lny, k):
        j2d5pt_device(src, dst, lnx, lny, w, k)
        launches[0] += last_launch_count()

    solver = SlabSolver(geo, local_solve, dist if world > 1 else None, exchange=exchange,
                        weights=w.astuple())
    a, b = solver.allocate(pitch, torch.float64, dev)

    def fresh():
        fill_random_rows_device(a, nx, ny, 1, geo.global_row0)
        solver.attach(a, b)

    def barrier():
        if world > 1:
            dist.barrier()

    clk = ClockSampler(local)  # started before the warm-up (first sample latency)
    for _ in range(args.warmup):
        fresh()
        solver.run(steps)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    total_ms = 0.0
    launches[0] = 0
    solver.launches = 0
    with clk:
        for _ in range(args.steps):
            fresh()
            torch.cuda.synchronize()
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            solver.run(steps)
            e.record(stream)
            torch.cuda.synchronize()
            barrier()
            total_ms += s.elapsed_time(e)
    launches_timed = launches[0] + solver.launches
    # e2e through the same public API: each rank's slab from pinned host
    # memory (H2D), the slab solve with its halo exchanges, the owned rows
    # back (D2H), all inside the timed window
    fresh()
    torch.cuda.synchronize()
    h_in = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
    h_in.copy_(a)
    h_out = torch.empty((geo.owned, pitch), dtype=a.dtype, pin_memory=True)
    e2e_ms = 0.0
    for _ in range(args.steps):
        torch.cuda.synchronize()
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        a.copy_(h_in, non_blocking=True)
        solver.attach(a, b)
        solver.run(steps)
        h_out.copy_(solver.owned_view(), non_blocking=True)
        e.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms += s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    mode = solver.exchange_mode
    solver.close()
    del a, b
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    cells = nx * ny * steps  # whole job
    return {
        "value": cells * args.steps / (total_ms * 1e-3) / 1e9, "unit": "GCells/s",
        "ms_per_step": total_ms / args.steps, "nx": nx, "ny": ny, "solve_steps": steps,
        "n_gpus": world, "depth": depth, "exchange": mode,
        "gpu_launches": launches_timed,
        "clocks": clk.summary(),
        "nvlink_halo_bytes_per_exchange_per_gpu":
            2 * depth * (nx + 2) * 8 * (2 if world > 2 else 1) if world > 1 else 0,
        "e2e": {"value": cells * args.steps / (e2e_ms * 1e-3) / 1e9, "unit": "GCells/s",
                "h2d_bytes_per_step": int(h_in.numel() * h_in.element_size()) * world,
                "d2h_bytes_per_step": int(h_out.numel() * h_out.element_size()) * world,
                "api": "paper_2306_03336_b200.slab.SlabSolver over j2d5pt_device "
                       "(dtb_j2d5pt_f64_dev), pinned host buffers per rank"},
    }


def run_slab(args, world, rank, local):
    """N > 1 (or --workload c5): the C5 weak series 32768 x (4096 N), plus
    strong scaling at the fixed 32768^2 under "strong"."""
    nx, rows_per_gpu, steps, dtype, desc = WORKLOADS["c5"]
    if args.solve_steps:
        steps = args.solve_steps
    weak = slab_series(args, world, rank, local, rows_per_gpu * world, steps)
    strong = None if args.no_strong else slab_series(args, world, rank, local, nx, steps)
    if rank != 0:
        return
    peaks = measured_peaks()
    per_gpu = weak["value"] / world
    ops = 6  # diffusive weights: the isotropic shared-product form (dtb_core.cuh)
    fp = {"achieved": per_gpu * ops, "peak": peaks["fp64_gops"], "unit": "Gop/s",
          "ops_per_cell": ops, "frac": per_gpu * ops / peaks["fp64_gops"]}
    line = {
        "metric": METRIC, "value": weak["value"], "unit": "GCells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": weak["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (splitmix64 random_interior seed 1, each slab filled on its GPU)",
        "config": {"workload": desc, "nx": nx, "ny": weak["ny"], "solve_steps": steps,
                   "depth": weak["depth"], "parallelism": f"y-slab x{world}",
                   "exchange": weak["exchange"], "l2": "inputs (>= 1 GB) larger than L2"},
        "roofline": dict(fp, bound="fp64_pipe", kernel="pipe_kernel", traffic=None),
        "rooflines": {"fp_pipe": fp},
        "nvlink_halo_bytes_per_exchange_per_gpu": weak["nvlink_halo_bytes_per_exchange_per_gpu"],
        "gpu_launches": weak["gpu_launches"],
        "clocks": weak["clocks"],
        "e2e": weak["e2e"],
        "strong": strong,
        # the CPU leg runs at N=1 only (bench contract)
        "cpu_baseline": (cpu_reference_sample(1900, 1900, dtype)
                         if not args.no_cpu and world == 1 else None),
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch
    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if world > 1 or args.workload == "c5":
        return run_slab(args, world, rank, local)
    line = run_single(args, world, rank, local)
    # the C5 family's N=1 anchors (the series --gpus N > 1 runs), measured
    # after the headline (the pipelined kernel runs at the power cap)
    if line is not None and args.workload == "c2" and not args.no_c5:
        c5_steps = args.solve_steps or WORKLOADS["c5"][2]
        line["c5"] = {"weak_n1": slab_series(args, 1, 0, local, WORKLOADS["c5"][1], c5_steps),
                      "strong_32768_n1": None if args.no_strong else
                      slab_series(args, 1, 0, local, WORKLOADS["c5"][0], c5_steps)}
    if line is not None:
        print(json.dumps(line), flush=True)


def run_single(args, world, rank, local):
    """The single-GPU workload line (C2 headline by default); None off rank 0."""
    import numpy as np
    import torch
    from paper_2306_03336_b200 import StencilWeights, j2d5pt_device, last_launch_count, plan_b200
    from paper_2306_03336_b200 import _native
    from paper_2306_03336_b200.prng import fill_random_device

    nx, ny, steps, dtype, desc = WORKLOADS[args.workload]
    if args.solve_steps:
        steps = args.solve_steps
    tdt = torch.float64 if dtype == "f64" else torch.float32
    elem = 8 if dtype == "f64" else 4
    w = StencilWeights.diffusive(0.2)
    dev = torch.device("cuda", local)
    a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=tdt, device=dev)  # 128-B pitch
    b = torch.empty_like(a)
    fill_random_device(a, nx, ny, 1, ghost=0.0)
    plan = plan_b200(nx, ny, elem, steps, 1)
    grid_bytes = a.numel() * elem
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    clk = ClockSampler(local)  # started before the warm-up (first sample latency)
    for _ in range(args.warmup):
        flush.fill_(0)  # also loads the flush and sleep kernels (lazy module loading
        torch.cuda._sleep(1)  # would stall the host inside the timed loop)
        j2d5pt_device(a, b, nx, ny, w, steps)
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    torch.cuda.synchronize()
    barrier()
    with clk:
        # solves are queued back to back, each bracketed by its own events, so
        # the ~20 us host cost of a call overlaps the previous solve and the
        # flush (it is part of the e2e leg below); multi-rank runs keep a
        # barrier per solve. A one-rank run first parks the stream on a ~5 ms
        # device sleep (outside every event pair) so that the host enqueues
        # the iterations ahead of the device: short solves (C1, ~0.1 ms)
        # would otherwise time the host's ~45 us call latency as device idle
        if world == 1:
            torch.cuda._sleep(10_000_000)
        for i in range(args.steps):
            flush.fill_(i)  # evict the grid from L2 between timed iterations
            if world > 1:
                torch.cuda.synchronize()
                barrier()
            ev[i][0].record(stream)
            j2d5pt_device(a, b, nx, ny, w, steps)
            ev[i][1].record(stream)
            launches += last_launch_count()
            if world > 1:
                torch.cuda.synchronize()
                barrier()
        torch.cuda.synchronize()
        barrier()
    ms = [s.elapsed_time(e) for s, e in ev]
    if os.environ.get("BENCH_DEBUG"):
        print("per-solve ms", [round(x, 4) for x in ms], file=sys.stderr)
    total_ms = sum(ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    cells = nx * ny * steps
    value = world * cells * args.steps / (total_ms * 1e-3) / 1e9

    # e2e through the public host API (H2D + solve + D2H from pinned host memory)
    e2e = None
    if rank == 0:
        host_in = torch.empty((ny + 2, nx + 2), dtype=tdt, pin_memory=True)
        host_in.copy_(a[:, :nx + 2].cpu())
        host_out = torch.empty_like(host_in).pin_memory()
        import ctypes
        lib = _native.lib()
        fn = lib.dtb_j2d5pt_f64 if dtype == "f64" else lib.dtb_j2d5pt_f32
        ct = ctypes.c_double if dtype == "f64" else ctypes.c_float
        wts = (ct * 5)(*w.astuple())
        rep = _native.DtbReport()
        call = lambda: fn(host_in.data_ptr(), host_out.data_ptr(), nx, ny, nx + 2, wts, steps,
                          1, None, 1, 1, 0, ctypes.byref(rep))
        if call() != 0:
            raise RuntimeError(_native.last_error())
        k = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(k):
            if call() != 0:
                raise RuntimeError(_native.last_error())
        el = time.perf_counter() - t0
        e2e = {"value": cells * k / el / 1e9, "unit": "GCells/s",
               "h2d_bytes_per_step": grid_bytes, "d2h_bytes_per_step": grid_bytes,
               "api": "dtb_j2d5pt_%s (include/dtb_b200.h) from pinned host buffers" % dtype}
        res = host_out.numpy()
        if not np.isfinite(res).all():
            raise RuntimeError("non-finite result")

    if rank != 0:
        return None
    peaks = measured_peaks()
    kernel_s = total_ms * 1e-3 / args.steps
    cells_per_s = cells / kernel_s
    fp_peak = peaks["fp64_gops"] if elem == 8 else peaks["fp32_gops"]
    # diffusive(0.2) has w == e == s == n: the kernels run the isotropic
    # shared-product form, 2 products + 4 sums = 6 rounded ops per cell update
    # (9 for general weights); the FP-pipe fraction counts the ops executed
    ops = 6
    rooflines = {
        "smem": {"achieved": cells_per_s * 2 * elem / 1e9, "peak": peaks["smem_gbs"], "unit": "GB/s",
                 "bytes_per_cell": 2 * elem, "peak_src": "microbench LDS.128 (profiles/r01/microbench_peaks.log)"},
        "fp_pipe": {"achieved": cells_per_s * ops / 1e9, "peak": fp_peak, "unit": "Gop/s",
                    "ops_per_cell": ops, "ops_per_cell_general_weights": 9,
                    "peak_src": "microbench DMUL/DADD (profiles/r01/microbench_peaks.log)"},
        "hbm": {"achieved": cells_per_s * 2 * elem / max(plan.halo, 1) / 1e9
                if plan.mode in ("streaming", "pipe") else grid_bytes * 2 / kernel_s / 1e9,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "peak_src": peaks["hbm_src"]},
    }
    for r in rooflines.values():
        r["frac"] = r["achieved"] / r["peak"]
    if plan.mode == "resident":
        # the north star's denominator: shared-memory bandwidth at 16 B/cell
        main = dict(rooflines["smem"], bound="smem")
    else:
        # streaming passes are FP-issue bound (HBM at 2*elem/h B/cell is far below peak)
        main = dict(rooflines["fp_pipe"], bound="fp64_pipe" if elem == 8 else "fp32_pipe")
    main["kernel"] = {"resident": "resident_kernel", "pipe": "pipe_kernel"}.get(plan.mode,
                                                                                "stream_kernel")
    main["traffic"], main["traffic_src"] = ncu_traffic(main["kernel"], dtype)
    line = {
        "metric": METRIC, "value": value, "unit": "GCells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (splitmix64 random_interior seed 1, generated on device)",
        "config": {"workload": desc, "nx": nx, "ny": ny, "solve_steps": steps,
                   "weights": "diffusive(0.2)", "l2": "256 MB buffer written between timed iterations",
                   "timing": "CUDA events around each solve; solves queued back to back (host call overlapped)",
                   "plan": {"mode": plan.mode, "halo": plan.halo, "lane_elems": plan.lane_elems,
                            "warps": plan.warps, "tiles": [plan.tiles_x, plan.tiles_y],
                            "ctas": plan.ctas, "smem_bytes": plan.smem_bytes}},
        "roofline": main,
        "rooflines": rooflines,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu_reference_sample(min(nx, 1900), min(ny, 1900), dtype,
                                             legs=not args.no_legs)
        if not args.no_cpu else None,
    }
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-legs", action="store_true",
                    help="cpu_baseline: only the all-core C port (skip the reference-structured legs)")
    ap.add_argument("--no-c5", action="store_true", help="N=1: skip the C5 family anchors")
    ap.add_argument("--no-strong", action="store_true", help="skip strong scaling at 32768^2")
    ap.add_argument("--solve-steps", type=int, default=0,
                    help="override the workload's Jacobi step count (quick runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # the timing rules require >= 3 warm-up steps
    if args.gpus < 1:
        ap.error("--gpus must be at least 1")
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # no launcher: one rank per GPU under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started "
                         f"WORLD_SIZE={world} ranks")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
