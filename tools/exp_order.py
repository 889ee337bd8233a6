"""Timing experiment: element processing order (storage permutation) vs
k_element time on cfg5. Builds permuted meshes (timing only: a permuted
mesh changes the reference's summation order, the product permutes
internally)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402
from paper_2106_14189_b200.spec import mesh_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
only = set(sys.argv[2:])
sc = Scenario(config_spec(name, precision=4))
img = sc.image()
nodes = img["nodes"].reshape(-1, 3).astype(np.float64)
conn = img["conn"].reshape(-1, 4)
E = conn.shape[0]
sc.close()
cen = nodes[conn].mean(axis=1)
lo, hi = cen.min(0), cen.max(0)
d = round((E / 6) ** (1 / 3))
h = (hi - lo).max() / d
rng = np.random.default_rng(0)
u0 = (rng.standard_normal(nodes.size) * 1e-4).astype(np.float32)


def run(tag, perm):
    if only and tag not in only:
        return
    c = conn[perm] if perm is not None else conn
    spec = mesh_spec(nodes, c, kind="T4", model="NH", precision=4, fixed=[(0, 0)])
    s = Scenario(spec)
    with GpuDjEngine(s) as eng:
        eng.set_state(u0, u0, 0)
        eng.step(3, raise_on_failure=False)
        ms_e, ms_n, _ = eng.profile_steps(20)
        print(json.dumps(dict(order=tag, k_element_us=round(ms_e / 20 * 1e3, 1), k_node_us=round(ms_n / 20 * 1e3, 1),
                              pipe=eng.info()["pipelined"])), flush=True)
    s.close()


run("original", None)
q = np.floor((cen - lo) / h).astype(np.int64)
for b in (2, 3, 4, 8):
    key = ((q[:, 2] // b) * (d // b + 1) + q[:, 1] // b) * (1 << 40) + q[:, 0] * (1 << 20) + \
          (q[:, 1] % b) * b + (q[:, 2] % b)
    run(f"pencil{b}", np.argsort(key, kind="stable"))
# Morton order of cells
def spread(x):
    x = x.astype(np.uint64)
    out = np.zeros_like(x)
    for i in range(21):
        out |= ((x >> np.uint64(i)) & np.uint64(1)) << np.uint64(3 * i)
    return out
mk = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
run("morton", np.argsort(mk, kind="stable"))
