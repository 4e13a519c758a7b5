"""bench.py's JSON-line contract (the driver parses it).  The reference arm
runs on CPU (`-m "not gpu"`); our arm needs a B200 (`-m gpu`)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-window", "2"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert "1" in cb["threads"] and str(cb["cores"]) in cb["threads"] and cb["host"]["cores_available"] >= 1
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_headline_line():
    d = _run(["--steps", "2", "--warmup", "3", "--cpu-window", "4", "--no-c5"], 900)
    assert BASE_KEYS <= set(d) and d["metric"] == "GLUP/s" and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] and r["peak"] > 0 and r["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"] and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["solve_iterations"] == 12480 and d["config"]["iterations_per_step"] == 13480
    assert set(d["cpu_baseline"]["threads"]) >= {"1", str(d["cpu_baseline"]["cores"])}


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["jacobi", "sor3d"])
def test_next_rows_lines(method):
    d = _run(["--method", method, "--steps", "2", "--warmup", "3", "--cpu-budget", "1"], 900)
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["roofline"]["frac"] > 0 and d["gpu_launches"] > 0


@pytest.mark.gpu
def test_two_rank_bench_on_one_gpu():
    """The N > 1 code path of bench.py (torchrun, dist-IPC handles, rank-0
    scatter / gather, max over ranks) as a functional check on a one-GPU box:
    SOR_BENCH_SHARE_GPU=1 puts both ranks on device 0 (lockstep, gloo); the
    number it prints is not a measurement."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-c5", "--cpu-window", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, SOR_BENCH_SHARE_GPU="1"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "ipc" in d["config"]["parallelism"]
    assert d["config"]["solve_iterations"] == 12480 and d["e2e"]["value"] > 0
