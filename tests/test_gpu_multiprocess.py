"""The peer-memory multi-GPU step across processes: torchrun
with 2 ranks on the one GPU of the test box (tests/mp_peer_worker.py). This
runs the CUDA-IPC mapping (djg_peer_ipc_export / djg_peer_ipc_open), peer
stores through foreign pointers, system-scope mailbox release/acquire and
the agreement between two processes -- everything but NVLink itself -- bit
for bit against one engine, inversion agreement and SkipAndReport counts
included. The ranks step in host lockstep, so no kernel waits on the other
process (kernels of two processes on one GPU are time-sliced; see
DistributedEngine.step_lockstep). NCCL cannot run two ranks on one GPU:
the NCCL transport's send/recv stays unexercised until a multi-GPU box."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_memory_two_processes_one_gpu():
    env = {**os.environ, "CUDA_VISIBLE_DEVICES": os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]}
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "tests/mp_peer_worker.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:] + p.stderr[-2000:]
    res = json.loads(lines[0])
    assert res["world"] == 2
    for name in ("smooth_t4_f32", "smooth_h8_ti_f64", "box_local_t4_f32", "abort_inversion", "skip_and_report"):
        c = res[name]
        assert c["halo_send"] > 0, (name, c)
        assert c["bitwise_u"] and c["bitwise_u_prev"] and c["reports_match"], (name, c)
    assert res["abort_inversion"]["single"][0] in (4, 5)
    assert res["skip_and_report"]["single"][3] > 0
