"""Why did round 1's two CPU-baseline numbers differ (3.0 vs 5.6 GLUP/s on the
same box)?  Times the threaded oracle on C3 with both round-1 protocols and
the round-2 one, in a process that holds a CUDA context and GPU buffers (as
bench.py's cpu_baseline leg did) and in a clean process:
  A  round-1 bench leg:      2 iterations per oracle call (threads re-spawned per call)
  B  round-1 reference arm:  32 iterations per call, after 5 warm-up iterations
  C  round-2 protocol:       iterations 1..96 from the initial grid, one call
Usage: python tools/cpu_gap_probe.py [--cuda]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import sor_inputs as SI  # noqa: E402

if "--cuda" in sys.argv:
    import torch
    x = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    x.zero_()
    torch.cuda.synchronize()
cfg = SI.config("C3")
cores = len(os.sched_getaffinity(0))
n = cfg.rows * cfg.cols


def rate(chunk, total, warm):
    u = oracle.to_storage(cfg.init(), "f64")
    if warm:
        oracle.iterate(u, cfg.omega, warm, threads=cores)
    k, t0 = 0, time.perf_counter()
    while k < total:
        oracle.iterate(u, cfg.omega, chunk, threads=cores)
        k += chunk
    return n * k / (time.perf_counter() - t0) / 1e9


tag = "cuda-process" if "--cuda" in sys.argv else "clean-process"
print(f"{tag} cores={cores} A(chunk2,1..192)={rate(2, 192, 0):.3f} B(chunk32,6..197)={rate(32, 192, 5):.3f} "
      f"C(window96)={rate(96, 96, 0):.3f} GLUP/s", flush=True)
