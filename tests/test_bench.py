"""bench.py keeps the driver's contract: one JSON line with the required keys
(our arm and the --impl reference arm), rank != 0 silent, N > 1 control flow."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([sys.executable, *args], cwd=ROOT, env=e, capture_output=True, text=True,
                       timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p, lines


def test_reference_arm_contract():
    _, lines = _run(["bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
                     "--warmup", "1"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_are_silent():
    _, lines = _run(["bench.py", "--impl", "reference", "--config", "c1", "--steps", "1",
                     "--warmup", "0"], env={"RANK": "1", "WORLD_SIZE": "2"})
    assert lines == []


@pytest.mark.gpu
def test_bench_line_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _, lines = _run(["bench.py", "--config", "c2", "--steps", "3", "--warmup", "3",
                     "--cpu-budget", "1"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1 and r["peak"] > 0
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 4 * d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_bench_two_ranks_share_one_gpu():
    """N = 2 control flow (P2P attach via CUDA IPC, barriers, max over ranks,
    e2e, teardown order) with both ranks on cuda:0 (PIKO_BENCH_SHARE_GPU)."""
    import socket
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    _, lines = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                     "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py",
                     "--gpus", "2", "--config", "c2", "--steps", "3", "--warmup", "3"],
                    env={"PIKO_BENCH_SHARE_GPU": "1"})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "p2p" in d["config"]["parallelism"] and d["value"] > 0
