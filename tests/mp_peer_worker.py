"""Worker of tests/test_gpu_multiprocess.py (launched by torchrun, 2 ranks,
both on cuda:0, gloo for the host side): the peer-memory multi-GPU step
across PROCESSES -- every rank maps the other rank's displacement buffers and
mailbox with CUDA IPC (djg_peer_ipc_export / djg_peer_ipc_open), its node
kernel stores the halo into them through the foreign pointers and posts its
status with system-scope release, k_wait_agree acquires and agrees. Steps
run in host lockstep (DistributedEngine.step_lockstep), so no kernel waits on
the other process. Rank 0 checks the assembled global state against one
engine, bit for bit, for a smooth run, an inversion halt (Abort) and
SkipAndReport counts; prints one JSON line."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("DJG_PEER_TIMEOUT_MS", "1000")  # safety net: never spin longer than this

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, mesh_spec  # noqa: E402
from paper_2106_14189_b200 import _abi as A  # noqa: E402
from paper_2106_14189_b200.parallel import DistributedEngine  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(0)
out = {"rank": rank, "world": dist.get_world_size()}


def single(spec, steps):
    with GpuDjEngine(Scenario(spec)) as e:
        r = e.step(steps, raise_on_failure=False)
        u, up, _ = e.get_state()
    return u, up, r


def case(name, spec, steps, method="rcb"):
    de = DistributedEngine(spec if method == "box-local" else Scenario(spec), device=0, transport="p2p",
                           method=method)
    r = de.step_lockstep(steps)
    g = de.gather_global()
    reps = [None] * dist.get_world_size()
    dist.all_gather_object(reps, (r.status, r.step, r.first_inverted, r.inverted_count, r.inverted_steps))
    if rank == 0:
        u1, up1, r1 = single(spec, steps)
        U, UP, step = g
        want = (r1.status, r1.step, r1.first_inverted, r1.inverted_count, r1.inverted_steps)
        out[name] = {"bitwise_u": bool(np.array_equal(U, u1)), "bitwise_u_prev": bool(np.array_equal(UP, up1)),
                     "reports_match": all(tuple(x) == want for x in reps), "single": want,
                     "parts": [list(x) for x in reps], "halo_send": de.part.info["send_total"]}
    dist.barrier()


case("smooth_t4_f32", box_spec(kind="T4", model="NH", divisions=8, precision=4, ramp_steps=120), 120)
case("smooth_h8_ti_f64", box_spec(kind="H8", model="TI", divisions=7, precision=8, ramp_steps=80), 80)
case("box_local_t4_f32", box_spec(kind="T4", model="NH", divisions=(9, 8, 10), precision=4, ramp_steps=100), 100,
     method="box-local")
case("abort_inversion", box_spec(kind="T4", divisions=3, extent=(0.1,) * 3, precision=8, target=-0.09,
                                 ramp_steps=3, fix_all_axes=True), 50)
sc0 = Scenario(box_spec(kind="T4", divisions=4, extent=(0.1, 0.1, 0.1), precision=8))
img = sc0.image()
nodes, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
bottom = [n for n in range(len(nodes)) if nodes[n, 2] == 0.0]
top = [n for n in range(len(nodes)) if nodes[n, 2] == nodes[:, 2].max()]
case("skip_and_report", mesh_spec(nodes, conn, kind="T4", precision=8, fixed=[(n, a) for n in bottom for a in range(3)],
                                  prescribed=[(n, 2, -0.35, 2e-4) for n in top], dt=1e-5, alpha=0.0,
                                  policy=A.DJG_SKIP_AND_REPORT), 40)
if rank == 0:
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
