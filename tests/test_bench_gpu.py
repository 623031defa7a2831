"""bench.py contract on the GPU: one JSON line with the required keys, N=1 and
the N=2 torchrun path (both ranks on the one B200 over gloo: plumbing only)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_c1_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup", "3",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])


def test_bench_two_ranks_plumbing():
    env = dict(os.environ, TPF_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--config", "c1",
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    # the N > 1 steps go through shard.solve_sharded; its final gather reassembles both slices
    g = d["shard_gather"]
    assert g["gathered_cases"] == 2 * d["config"]["tau_per_gpu"] and g["own_slice_bitwise"]
    assert d["config"]["converged"] == 2 * d["config"]["tau_per_gpu"]


def test_bench_c4_pass_line():
    """Config C4: the probabilistic-PF pass (generation + solve + statistics) over every scenario."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "c4", "--scenarios", "4", "--tau", "65536",
                        "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["steps"] == 4 and d["config"]["cases"] == 4 * 65536 and d["scaling"] == "strong"
    assert d["result"]["nonconverged"] == 0 and 0.9 < d["result"]["vmin_min"] < d["result"]["vmax_max"] <= 1.0


def test_bench_c64_line():
    """The complex64 twin is reported as its own line (north_star: "a complex64 mode reported separately")."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--dtype", "c64", "--steps", "3",
                        "--warmup", "3", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["dtype"] == "c64" and d["value"] > 0
    assert d["roofline"]["kernel"] == "dense_c64_kernel" and 0 < d["roofline"]["frac"] < 1
    assert d["config"]["converged"] == d["config"]["tau_per_gpu"]
    assert d["e2e"]["h2d_bytes_per_step"] == 34 * 8760 * 8


def test_bench_default_line_with_sparse_half():
    """The driver's default invocation: C2 dense plus the nested C3 sparse object (full size; ~1 min)."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--cpu-seconds", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] == 2 * 3
    sp = d["sparse"]
    assert sp["value"] > 0 and sp["roofline"]["bound"] == "hbm" and 0 < sp["roofline"]["frac"] < 1


def test_bench_c5_line():
    """Config C5 (b = 1,000, the device-side loop + persistent tail) at a small tau."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "c5", "--tau", "2000", "--steps", "2", "--warmup",
                        "3", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] >= 2 * 4
    assert d["roofline"]["bound"] == "tensor" and 0 < d["roofline"]["frac"] < 1
