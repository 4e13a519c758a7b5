"""Writes tests/golden/paper_replay_4096.json with the CPU oracle only (no CUDA
path involved): the paper's protocol at its own size [P:100, P:375, P:383] --
4096 x 4096, north = 1, omega = 0.376, eps = 1e-5, K = 4000 -- run by the
threaded oracle (bitwise = serial, pin P14) to convergence; records the
iteration count, the checked max-change (hex) and the SHA-256 of the final
(rows+2) x (cols+2) float64 grid.  The oracle needs minutes here (fp64
subnormals appear ahead of the under-relaxed diffusion front), so the GPU
test compares with this stored result instead of re-running it."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("PAPER")
u = cfg.init()
t0 = time.time()
rep = oracle.solve(u, cfg.omega, cfg.tol, cfg.maxit, cfg.check_every, threads=len(os.sched_getaffinity(0)))
out = {"config": "PAPER (4096x4096, north 1, omega 0.376, eps 1e-5, K 4000) [P:100, P:375, P:383]",
       "converged": rep.status == 0, "iters": rep.iters, "checks": rep.checks,
       "max_change_hex": float(rep.max_change).hex(), "grid_sha256": hashlib.sha256(u.tobytes()).hexdigest(),
       "shape": list(u.shape), "writer": "tools/make_golden_paper_replay.py (oracle only)",
       "oracle_seconds": round(time.time() - t0, 1)}
with open(os.path.join(ROOT, "tests", "golden", "paper_replay_4096.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out)
