#!/usr/bin/env python
"""Benchmark of the B200 red-black SOR hot path (arXiv 1401.0763).

Metric (BASELINE.json): GLUP/s = interior grid-point updates per second
(rows*cols*iterations / t) and the HBM-roofline fraction of the dominant
kernel.

Default workload (N=1): BASELINE.json configs[2] "C3", the size the metric
and the 70%-of-roofline target are quoted on: 4096x4096 interior, fp64,
north=100, omega_opt(4096), 1000 fixed iterations then solve to
max|du| < 1e-8 with a check every iteration, continued on the same handle.
One step = reset the grid from the HBM-resident initial array, iterate(1000),
solve(1e-8).  `value` counts every iteration the step executed.

N>1 (torchrun, one process per GPU): the same grid split into row slabs
(strong scaling), halos over NCCL, allreduce-max for the stop test.

`--impl reference` times the CPU oracle (oracle/, plain C, threaded row-slab
variant = Algorithm 1's P workers) on this host's cores on a bounded sample
of the same workload; it is the reference arm for this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import sor_inputs as SI  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def g_nsm():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# SOR_BENCH_SHARE_GPU=1 (functional test of the N > 1 code path on a one-GPU
# box, never a measurement): every rank uses device 0, the process group is
# gloo, the dist handles run in lockstep (ranks sharing a GPU), no NCCL.
SHARE_GPU = os.environ.get("SOR_BENCH_SHARE_GPU") == "1"


def coll_dev():
    """Device of tensors passed to torch.distributed collectives."""
    return "cpu" if SHARE_GPU else "cuda"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference arm for this tier: the CPU oracle as it stands (no
    reference implementation exists), on the same fixed window as our arm's
    cpu_baseline; each step = the window at all cores, after the thread-scaling
    sweep (reported, not timed into `value`)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle
    cfg = SI.config(args.config, dtype=args.dtype)
    cores = len(os.sched_getaffinity(0))
    window = args.cpu_window
    init = cfg.init()
    for _ in range(args.warmup):
        u = oracle.to_storage(init, cfg.dtype)
        oracle.iterate(u, cfg.omega, 1, threads=cores)
    ts = []
    for _ in range(args.steps):
        u = oracle.to_storage(init, cfg.dtype)
        t0 = time.perf_counter()
        oracle.iterate(u, cfg.omega, window, threads=cores)
        ts.append(time.perf_counter() - t0)
    t = sum(ts)
    glups = cfg.rows * cfg.cols * window * args.steps / t / 1e9
    scaling = cpu_protocol(cfg, window, thread_counts(cores)) if args.steps > 0 else {}
    line = {
        "impl": "reference", "metric": "GLUP/s", "value": glups, "unit": "GLUP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic",
        "config": {"workload": f"{cfg.name} window: iterations 1..{window} of the {cfg.rows}x{cfg.cols} "
                               f"{cfg.dtype} grid from its initial state, per step", "impl": "CPU oracle "
                               "(oracle/sor_oracle.c, pthreads row slabs + barrier per phase, bitwise = serial oracle)"},
        "cpu_baseline": {"value": glups, "unit": "GLUP/s", "cores": cores, "kind": "oracle",
                         "sample": f"iterations 1..{window} of {cfg.name} per step, {args.steps} steps, all cores",
                         "threads": {k: round(v, 4) for k, v in scaling.items()}, "host": host_info()},
        "e2e": {"value": glups, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_info():
    """CPU model, sockets / NUMA nodes, host RAM (the CPU baseline's hardware)."""
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                if ln.startswith("physical id"):
                    sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 2 ** 20, 1)
    except OSError:
        pass
    numa = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")]) \
        if os.path.isdir("/sys/devices/system/node") else None
    return {"cpu_model": model, "sockets": len(sockets) or None, "numa_nodes": numa, "ram_gib": ram,
            "cores_available": len(os.sched_getaffinity(0))}


def thread_counts(cores):
    return sorted({t for t in (1, 2, 4, 8, cores) if t <= cores})


def cpu_protocol_child(cfg_name, dtype, window, threads):
    """The CPU-baseline protocol (the paper's thread scaling
    P:383-389): the oracle as it stands, on a fixed window -- iterations
    1..window of the workload from its initial grid -- once per thread count,
    one oracle call per window (threads spawned once).  Run in a clean child
    process, so nothing of the GPU process (driver threads, pinned buffers)
    shares the cores or the memory with it."""
    import oracle
    cfg = SI.config(cfg_name, dtype=dtype)
    init = cfg.init()
    out = {}
    for P in threads:
        rates = []
        for _ in range(3 if P >= 8 else 1):      # short windows at many threads: median of 3
            u = oracle.to_storage(init, cfg.dtype)
            t0 = time.perf_counter()
            oracle.iterate(u, cfg.omega, window, threads=P)
            dt = time.perf_counter() - t0
            rates.append(cfg.rows * cfg.cols * window / dt / 1e9)
        out[str(P)] = float(np.median(rates))
    return out


def cpu_protocol(cfg, window, threads):
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-protocol-child", "--config", cfg.name,
           "--dtype", cfg.dtype, "--cpu-window", str(window), "--cpu-threads", ",".join(map(str, threads))]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    if r.returncode != 0:
        raise RuntimeError("cpu protocol child failed: " + r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_baseline(cfg, window):
    """Oracle (as it stands) on this host's cores: the fixed-window protocol
    at 1/2/4/8/all threads; `value` is the all-cores rate."""
    cores = len(os.sched_getaffinity(0))
    ths = thread_counts(cores)
    rates = cpu_protocol(cfg, window, ths)
    return {"value": rates[str(cores)], "unit": "GLUP/s", "cores": cores, "kind": "oracle",
            "sample": (f"iterations 1..{window} of {cfg.name} ({cfg.rows}x{cfg.cols} {cfg.dtype}) from its "
                       f"initial grid, threaded oracle (P workers + barrier per phase), one call per window "
                       f"(median of 3 at >= 8 threads), clean child process"),
            "threads": {k: round(v, 4) for k, v in rates.items()},
            "host": host_info()}


# ------------------------------------------------------------------ NEXT rows
def run_next(args):
    """NEXT-2 (Jacobi on C3's grid, 1000 iterations, T-deep passes), NEXT-3
    (3-D SOR, 512^3 fp64, 50 iterations) and NEXT-4 (multi-colour / block
    red-black SOR on C3's grid, 200 iterations): the same JSON contract as the
    headline line, one GPU."""
    import torch

    import oracle
    import paper_1401_0763_b200 as P

    torch.cuda.set_device(0)
    pk, pk_kind = peaks()
    if args.method == "jacobi":
        cfg = SI.config("C3")
        init_h = cfg.init()
        iters, units = 1000, cfg.rows * cfg.cols
        T = args.T
        g = P.Grid.create(torch.from_numpy(init_h).cuda())
        g.set_kernel("temporal", T)
        run = lambda n: g.jacobi(n)                        # noqa: E731
        reset_d = lambda: g.reset(torch.from_numpy(init_h).cuda())  # noqa: E731
        bytes_per_update = 16.0 / T
        kname, workload = f"jacobi_kernel<f64,T={T},ck=0>", f"Jacobi (NEXT-2) on the C3 grid: 4096x4096 f64, {iters} iterations"
        elapsed = lambda: g.elapsed_ms                     # noqa: E731
        launches = lambda: g.stats["kernel_launches"]      # noqa: E731
    elif args.method in ("multicolor", "block"):
        cfg = SI.config("C3")
        init_h = cfg.init()
        iters, units = 200, cfg.rows * cfg.cols
        if args.method == "multicolor":
            ca, cb, nc = (int(x) for x in args.colours.split(","))
            var = P.Variant.multicolor(ca, cb, nc)
            kname = f"mc_kernel<f64> (colour ({ca}i+{cb}j) mod {nc}, {nc} phases in shared memory)"
            vdesc = f"multi-colour SOR (NEXT-4, reading N4-1), colour ({ca}i+{cb}j) mod {nc}"
        else:
            var = P.Variant.blocks(args.block)
            kname = f"bp_kernel<f64> (block {args.block}, red/black blocks in shared memory)"
            vdesc = f"block red-black SOR (NEXT-4, reading N4-2), {args.block}x{args.block} blocks"
        g = P.Grid.create(torch.from_numpy(init_h).cuda())
        run = lambda n: g.variant_iterate(var, cfg.omega, n)  # noqa: E731
        reset_d = lambda: g.reset(torch.from_numpy(init_h).cuda())  # noqa: E731
        bytes_per_update = 16.0
        workload = f"{vdesc} on the C3 grid: 4096x4096 f64, omega_opt, {iters} iterations"
        elapsed = lambda: g.elapsed_ms                     # noqa: E731
        launches = lambda: g.stats["kernel_launches"]      # noqa: E731
    else:
        n = 512
        init_h = SI.random_shell3d(n, n, n, seed=7)
        iters, units = 50, n ** 3
        g = P.Grid3D(init_h)
        k3 = "natural" if args.kernel == "natural" else "fused"
        g.set_kernel(k3)
        run = lambda k: g.iterate(1.9, k)                  # noqa: E731
        reset_d = None
        bytes_per_update = 32.0 if k3 == "natural" else 16.0
        kname = "k3d_half_sweep<f64> (red + black)" if k3 == "natural" else "k3d_tma<f64> (one pass)"
        workload = f"3-D red-black SOR (NEXT-3): 512^3 f64, omega 1.9, {iters} iterations, {k3} kernel"
        elapsed = lambda: g.elapsed_ms                     # noqa: E731
        launches = lambda: (2 if k3 == "natural" else 1) * iters  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        run(iters)
        flush.zero_()
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    t_dev, n_launch = 0.0, 0
    for _ in range(args.steps):
        if reset_d:
            reset_d()
        run(iters)
        t_dev += elapsed()
        n_launch += launches()
        flush.zero_()
    torch.cuda.synchronize()
    ck = clocks.stop()
    value = units * iters * args.steps / (t_dev * 1e-3) / 1e9
    achieved = value * bytes_per_update
    line = {
        "metric": "GLUP/s", "value": value, "unit": "GLUP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_dev / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "method": args.method,
                   "l2": "flushed between steps (256 MiB write); grids exceed the 126 MB L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": None, "kernel": kname,
                     "algorithmic_bytes_per_update": bytes_per_update, "peak_kind": pk_kind},
        "gpu_launches": n_launch, "clocks": ck,
    }
    # end to end through the C ABI from pinned host buffers
    hin = torch.from_numpy(init_h).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if args.method == "jacobi":
            g.reset(hin)
            g.jacobi(iters)
            g.download(hout)
        elif args.method in ("multicolor", "block"):
            g.reset(hin)
            run(iters)
            g.download(hout)
        else:
            g3 = P.Grid3D(hin.numpy())
            g3.set_kernel(k3)
            g3.iterate(1.9, iters)
            g3.download(hout.numpy())
            g3.close()
    t = time.perf_counter() - t0
    line["e2e"] = {"value": units * iters * args.steps / t / 1e9, "unit": "GLUP/s",
                   "h2d_bytes_per_step": hin.numel() * 8, "d2h_bytes_per_step": hout.numel() * 8}
    # the oracle, single thread, bounded sample of the same workload
    u = init_h.copy()
    k, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < args.cpu_budget:
        if args.method == "jacobi":
            oracle.jacobi_iterate(u, 2)
        elif args.method == "multicolor":
            oracle.multicolor_iterate(u, cfg.omega, 2, ca, cb, nc)
        elif args.method == "block":
            oracle.block_iterate(u, cfg.omega, 2, args.block)
        else:
            oracle.sor3d_iterate(u, 1.9, 1)
        k += 1 if args.method == "sor3d" else 2
    tc = time.perf_counter() - t0
    line["cpu_baseline"] = {"value": units * k / tc / 1e9, "unit": "GLUP/s", "cores": 1, "kind": "oracle",
                            "sample": f"first {k} iterations of the same grid, single-thread oracle, {tc:.1f} s"}
    g.close()
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ multi-GPU / C5
def ipc_self_check(P, SI, make_grid, rank):
    """IPC vs NCCL on this node: 61 iterations + a short solve of a 1024^2
    grid with random interior, grids compared bitwise on rank 0."""
    import torch
    import torch.distributed as dist
    try:
        cfg = SI.config("C2")
        init = SI.random_field(cfg.rows, cfg.cols, seed=3, lo=-10.0, hi=10.0)
        dinit = torch.from_numpy(init).cuda()
        res = {}
        for tr in ("nccl", "ipc"):
            g = make_grid(cfg, dinit, tr)
            g.set_kernel("temporal", 4)
            g.iterate(1.9, 61)
            r = g.solve(1.9, 1e-3, 4000, 1)
            out = g.download()
            res[tr] = (out, r.iters, r.max_change)
            g.close()
        ok = 1
        if rank == 0:
            a, b = res["nccl"], res["ipc"]
            ok = int(np.array_equal(a[0], b[0]) and a[1:] == b[1:])
        f = torch.tensor([ok], dtype=torch.int32, device=coll_dev())
        dist.broadcast(f, 0)
        return {"ok": bool(f.item()), "what": "iterate 61 + solve(1e-3) of a 1024^2 random field, T=4, "
                "IPC vs NCCL, bitwise"}
    except Exception as e:  # noqa: BLE001
        return {"ok": False, "error": str(e)[:300]}


def measure_c5(P, torch, dist, make_grid, transport, world, rank, local, args, pk, pk_kind, reps=3):
    """C5 (BJ configs[4]) at N GPUs: reset from the HBM-resident init, then
    iterate(omega_opt, 200), temporally blocked at T = 5 on one GPU (the
    deepest measured-best depth; multi-slab handles run T <= 4); device time,
    max over ranks."""
    cfg = SI.config("C5")
    init_h = cfg.init()
    init_d = torch.from_numpy(init_h).cuda() if (world == 1 or rank == 0) else None
    del init_h
    g = make_grid(cfg, init_d, transport)
    T = 5 if world == 1 else 4
    g.set_kernel("temporal", T)
    g.iterate(cfg.omega, cfg.iters)            # warm-up (tile tables, tensor maps)
    clocks = ClockSampler(local)
    clocks.start()
    ts, launches = [], 0
    for _ in range(reps):
        g.reset(init_d if (world == 1 or rank == 0) else None)
        if world > 1:
            dist.barrier()
        g.iterate(cfg.omega, cfg.iters)
        ms = g.elapsed_ms
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device=coll_dev())
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        ts.append(ms)
        launches += g.stats["kernel_launches"]
    ck = clocks.stop()
    rows_local = g.stats["row_hi"] - g.stats["row_lo"]
    g.close()
    ms = float(np.median(ts))
    value = cfg.rows * cfg.cols * cfg.iters / (ms * 1e-3) / 1e9
    t_launch = ms / (launches / reps)
    bpl = 16 * rows_local * cfg.cols  # one HBM pass (read + write each cell) per launch of T iterations
    achieved = bpl / (t_launch * 1e-3) / 1e9
    alu_peak = g_nsm() * 64 * 1.965e9 / 1e12
    alu_achieved = 7 * rows_local * cfg.cols * T / (t_launch * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f)
        kfam = "wave2_kernel" if (world == 1 and os.environ.get("SOR_WAVE2", "1") != "0") else "wave_kernel"
        traffic = tr.get(f"C5:{kfam}<f64,T={T},ck=0>", {}).get("dram_bytes_per_launch")
    return {"metric": "GLUP/s", "value": value, "unit": "GLUP/s", "ms": ms, "reps_ms": ts,
            "workload": f"C5: {cfg.rows}x{cfg.cols} f64, random edges seed 7, omega={cfg.omega!r}, "
                        f"{cfg.iters} iterations, T={T}, median of {reps}",
            "n_gpus": world, "scaling": "strong",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "kernel": ("wave2_kernel" if (world == 1 and os.environ.get("SOR_WAVE2", "1") != "0")
                                    else "wave_kernel") + f"<f64,T={T},ck=0>", "algorithmic_bytes_per_launch": bpl,
                         "avg_launch_ms": t_launch, "peak_kind": pk_kind,
                         "fp64_pipe": {"achieved_tflops": alu_achieved, "peak_tflops": alu_peak,
                                       "frac": alu_achieved / alu_peak,
                                       "note": "7 FP64 instructions per update (no FMA), ghost work excluded; "
                                               "peak = SMs x 64 x 1.965 GHz"}},
            "clocks": ck}


# ------------------------------------------------------------------ our arm
def measure_small(P, torch):
    """BJ configs[0] and configs[1] (the latency configs) on one GPU with the
    register-resident K7 kernel (SOR_KERNEL_RESIDENT): C1 solved on one CTA
    with the stop test on the device, C2 iterated on one block per SM with
    T = 3 passes; device time of the call (CUDA events), best of 5, grid
    reset from HBM before each run.  The per-iteration time is the figure of
    merit (both grids are L2/register resident; there is no HBM roofline)."""
    out = {}
    for name, T in (("C1", 1), ("C2", 3)):
        cfg = SI.config(name)
        dinit = torch.from_numpy(cfg.init()).cuda()
        with P.Grid.create(dinit) as g:
            g.set_kernel("resident", T)
            best, iters = 1e30, 0
            for rep in range(6):
                g.reset(dinit)
                if name == "C1":
                    iters = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1).iters
                else:
                    g.iterate(cfg.omega, cfg.iters)
                    iters = cfg.iters
                if rep:
                    best = min(best, g.elapsed_ms)
            launches = g.stats["kernel_launches"]
        out[name] = {"us_per_iteration": best * 1e3 / iters, "iterations": iters, "ms": best,
                     "glups": cfg.rows * cfg.cols * iters / (best * 1e-3) / 1e9, "kernel_launches": launches,
                     "kernel": "resident (K7)", "temporal_depth": T}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--kernel", default="temporal")
    ap.add_argument("--T", type=int, default=4)
    ap.add_argument("--no-solve", action="store_true", help="fixed iterations only")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="NEXT rows: single-thread oracle budget (s)")
    ap.add_argument("--cpu-window", type=int, default=96,
                    help="CPU baseline / reference arm: iterations 1..W of the workload")
    ap.add_argument("--cpu-threads", default=None)
    ap.add_argument("--cpu-protocol-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N>1: halo/max transport (ipc: device-initiated pushes over CUDA IPC)")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (32768^2) sub-record")
    ap.add_argument("--no-small", action="store_true", help="skip the C1/C2 (latency configs) sub-record")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--method", default="sor", choices=["sor", "jacobi", "sor3d", "multicolor", "block"],
                    help="sor: the headline path; jacobi / sor3d / multicolor, block: the NEXT-2 / NEXT-3 / "
                         "NEXT-4 rows (1 GPU)")
    ap.add_argument("--colours", default="1,1,4", help="multicolor: ca,cb,nc (colour (ca*i+cb*j) mod nc)")
    ap.add_argument("--block", type=int, default=8, help="block: block side B")
    args = ap.parse_args()
    if args.dtype is None:
        args.dtype = "f32" if args.config == "C4F32" else "f64"
    if args.cpu_protocol_child:
        rates = cpu_protocol_child(args.config, args.dtype, args.cpu_window,
                                   [int(x) for x in args.cpu_threads.split(",")])
        print(json.dumps(rates), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference(args)
    if args.method != "sor":
        return run_next(args)

    import torch
    import torch.distributed as dist

    import paper_1401_0763_b200 as P

    rank, world, local = env_rank()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    if SHARE_GPU:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = SI.config(args.config, dtype=args.dtype)
    iters_fixed = cfg.iters
    do_solve = cfg.tol is not None and not args.no_solve
    init_h = cfg.init()
    init_d = torch.from_numpy(init_h).cuda()

    def bcast_id(make):
        uid = make() if rank == 0 else bytes(128)
        tb = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(coll_dev())
        dist.broadcast(tb, 0)
        return bytes(tb.cpu().numpy().tobytes())

    def make_grid(c, dinit, transport):
        """One handle of config c: single GPU, or row slabs over `transport`."""
        if world == 1:
            return P.Grid.create(dinit, dtype=c.dtype)
        if transport == "ipc":
            return P.Grid.create_dist_ipc(dinit if rank == 0 else None, rank, world, local,
                                          bcast_id(P.ipc_unique_id), dtype=c.dtype, rows=c.rows, cols=c.cols)
        return P.Grid.create_dist(dinit if rank == 0 else None, rank, world, local, bcast_id(P.nccl_unique_id),
                                  dtype=c.dtype, rows=c.rows, cols=c.cols)

    transport, transport_check = args.transport, None
    if world > 1 and SHARE_GPU:
        transport, transport_check = "ipc", {"ok": True, "what": "skipped: SOR_BENCH_SHARE_GPU test mode (no NCCL)"}
    elif world > 1 and transport == "ipc":
        # the device-initiated path is checked against the NCCL path on this
        # node before it is timed (a short iterate + solve, bitwise); any
        # mismatch or error falls back to NCCL and says so in the JSON line
        transport_check = ipc_self_check(P, SI, make_grid, rank)
        if not transport_check.get("ok"):
            transport = "nccl"
    g = make_grid(cfg, init_d, transport)
    g.set_kernel(args.kernel, args.T if args.kernel == "temporal" else 1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(record):
        g.reset(init_d)
        g.iterate(cfg.omega, iters_fixed, want_delta=True)
        t_it = g.elapsed_ms
        st = g.stats
        n_iter = iters_fixed
        n_launch = st["kernel_launches"]
        solve_iters, t_sv, sv_launch, sv_passes = 0, 0.0, 0, 0
        if do_solve:
            r = g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every)
            solve_iters = r.iters
            n_iter += r.iters
            t_sv = g.elapsed_ms
            s2 = g.stats
            sv_launch = s2["kernel_launches"]
            sv_passes = s2["hbm_passes"]
            n_launch += sv_launch
        if record is not None:
            record.append({"iters": n_iter, "solve_iters": solve_iters, "t_iterate_ms": t_it,
                           "iterate_launches": st["kernel_launches"], "launches": n_launch,
                           "hbm_passes": st["hbm_passes"], "t_solve_ms": t_sv, "solve_launches": sv_launch,
                           "solve_passes": sv_passes})

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(None)
        flush.zero_()
    clocks = ClockSampler(local)
    recs = []
    barrier()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step(recs)
        flush.zero_()      # L2 flush between steps (256 MiB > 126 MB L2)
    ev1.record()
    barrier()
    ck = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([ms_total], dtype=torch.float64, device=coll_dev())
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    iters_total = sum(r["iters"] for r in recs)
    updates = cfg.rows * cfg.cols * iters_total
    value = updates / (ms_total * 1e-3) / 1e9

    # dominant kernel roofline.  Both phases launch one wave_kernel per HBM pass
    # (the stop test is fused into it); the solve phase (per-iteration
    # max-change, ck=3) takes most of the step when present.
    pk, pk_kind = peaks()
    esz = 8 if cfg.dtype == "f64" else 4
    T_eff = args.T if args.kernel == "temporal" else 1
    t_it_total = sum(r["t_iterate_ms"] for r in recs)
    t_sv_total = sum(r["t_solve_ms"] for r in recs)
    solve_dominant = t_sv_total > t_it_total
    # the skew-2 schedule (wave2_kernel) runs T >= 2 on one GPU unless SOR_WAVE2=0
    kfam = "wave2_kernel" if (T_eff >= 2 and world == 1 and os.environ.get("SOR_WAVE2", "1") != "0") else "wave_kernel"
    if solve_dominant:
        t_launch_ms = t_sv_total / sum(r["solve_launches"] for r in recs)
        kname = f"{kfam}<{cfg.dtype},T={T_eff},ck={4 if T_eff > 1 else 1}> (solve phase)"
    else:
        t_launch_ms = t_it_total / sum(r["iterate_launches"] for r in recs)
        kname = f"{kfam}<{cfg.dtype},T={T_eff},ck=0> (fixed-iteration phase)"
    rows_local = g.stats["row_hi"] - g.stats["row_lo"]
    bytes_per_launch = 2 * esz * rows_local * cfg.cols          # read X_{k0} + write X_{k0+T}, once each
    achieved = bytes_per_launch / (t_launch_ms * 1e-3) / 1e9
    it_glups = cfg.rows * cfg.cols * iters_fixed * len(recs) / (t_it_total * 1e-3) / 1e9
    sv_glups = (cfg.rows * cfg.cols * sum(r["solve_iters"] for r in recs) / (t_sv_total * 1e-3) / 1e9
                if t_sv_total > 0 else None)
    # FP64 pipe roofline of the same launch: 7 flops per update (+1 for |delta|
    # when measured), peak = 148 SMs x 64 FP64 lanes x max SM clock
    flops_per_update = 7 + (1 if solve_dominant else 0)
    alu_peak = g_nsm() * 64 * 1.965e9 / 1e12
    alu_achieved = flops_per_update * rows_local * cfg.cols * T_eff / (t_launch_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f)
        key = f"{cfg.name}:{kname}"
        if key in tr:
            traffic = tr[key]["dram_bytes_per_launch"]

    line = {
        "metric": "GLUP/s", "value": value, "unit": "GLUP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic",
        "config": {
            "workload": (f"{cfg.name}: {cfg.rows}x{cfg.cols} interior {cfg.dtype}, {cfg.kind}, "
                         f"omega={cfg.omega!r}, {iters_fixed} fixed iterations"
                         + (f" + solve to max|du|<{cfg.tol:g} (check every {cfg.check_every})" if do_solve else "")),
            "kernel": args.kernel, "temporal_depth": args.T if args.kernel == "temporal" else 1,
            "iterations_per_step": iters_total / len(recs),
            "solve_iterations": recs[-1]["solve_iters"],
            "l2": "flushed between steps (256 MiB write); grid planes 2x134 MB exceed the 126 MB L2",
            "parallelism": (f"row slabs x{world}, halos and max join over {transport}"
                            if world > 1 else "single GPU"),
        },
        "fixed_phase_glups": it_glups,
        "solve_phase_glups": sv_glups,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "kernel": kname,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "avg_launch_ms": t_launch_ms, "peak_kind": pk_kind,
                     "effective_frac_16B_per_update": (value * 2 * esz) / pk["hbm_gbs"],
                     "fp64_pipe": {"achieved_tflops": alu_achieved, "peak_tflops": alu_peak,
                                   "frac": alu_achieved / alu_peak,
                                   "note": "no FMA: each op is one FP64 instruction; peak = SMs x 64 x 1.965 GHz"}},
        "gpu_launches": sum(r["launches"] for r in recs),
        "clocks": ck,
    }

    # end-to-end through the C ABI with host buffers (H2D + D2H inside timing).
    # N > 1: rank 0 passes the pinned host init (the library scatters the
    # slabs) and receives the gathered grid; time = max over ranks.
    if not args.no_e2e:
        hin = torch.from_numpy(init_h).pin_memory() if rank == 0 else None
        hout = torch.empty_like(hin).pin_memory() if rank == 0 else None
        barrier()
        t0 = time.perf_counter()
        e_iters = 0
        for _ in range(args.steps):
            g.reset(hin)
            g.iterate(cfg.omega, iters_fixed, want_delta=True)
            e_iters += iters_fixed
            if do_solve:
                e_iters += g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every).iters
            g.download(hout)
        t = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=coll_dev())
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        nbytes = init_h.size * 8
        line["e2e"] = {"value": cfg.rows * cfg.cols * e_iters / t / 1e9, "unit": "GLUP/s",
                       "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}
    if transport_check is not None:
        line["transport_check"] = transport_check
    g.close()
    del g
    # BJ's metric also names 32768^2: the C5 sub-record (BJ configs[4]:
    # 32768x32768 f64, omega_opt, 200 iterations, temporally blocked T=4)
    if not args.no_c5 and args.config == "C3":
        line["c5"] = measure_c5(P, torch, dist, make_grid, transport, world, rank, local, args, pk, pk_kind)
    if rank == 0 and world == 1 and args.config == "C3" and not args.no_small:
        line["small_configs"] = measure_small(P, torch)
    if rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_window)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
