"""bench.py contract on a small problem: the single-GPU arm, the torchrun
multi-GPU arm (one rank) and the reference arm each print one JSON line with
the keys the driver reads."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(cmd, env=None):
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


SMALL = ["--divisions", "24", "--steps", "40", "--warmup", "3", "--e2e-steps", "3", "--tled-steps", "10",
         "--f64-steps", "10"]


def test_bench_single_gpu_line():
    line = _run([sys.executable, "bench.py", *SMALL, "--cpu-steps", "2", "--sub-configs", "cfg1,cfg2"])
    assert KEYS <= set(line) and line["n_gpus"] == 1 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["e2e"]["value"] < line["value"]
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and r["achieved"] > 0
    assert line["gpu_launches"] == 2 * 40 and line["clocks"]["samples"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] > 0 and cb["same_config"] and cb["threads_1"]["cores"] == 1
    assert r["traffic_stale"] in (None, True, False) and len(r["source_hash"]) == 16
    for name in ("cfg1", "cfg2"):
        sub = line["sub_configs"][name]
        assert sub["status"] == 0 and sub["ms_per_step"] > 0 and sub["step_frac"] > 0, sub
    assert line["tled"]["status"] == 0
    assert line["f64"]["status"] == 0 and line["f64"]["ms_per_step"] > 0
    assert line["e2e_run"]["value"] > 0 and line["e2e_run"]["steps"] == 40


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_multi_gpu_arm_one_rank():
    line = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                 "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1", *SMALL],
                env={"DJG_BENCH_FORCE_MULTI": "1"})
    assert KEYS <= set(line) and line["scaling"] == "strong" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["value"] < line["value"]
    assert line["partition"]["neighbors"] == 0


def test_bench_reference_arm():
    line = _run([sys.executable, "bench.py", "--impl", "reference", "--divisions", "24", "--steps", "3",
                 "--warmup", "1"])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["same_config"] and line["config"]["divisions"] == 24 and line["steps"] == 3 and line["warmup"] == 3
    assert line["threads_1"]["value"] > 0 and line["tled"]["value"] > 0
