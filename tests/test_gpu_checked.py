"""The bounds-checked engine (paper_2106_14189_b200/_build_checked, built with
DJG_CHECKS=1: every gathered node id and every slot position is checked on
the device, a violation traps) runs every kernel family without a trap and
gives the same bits as the default build.

compute-sanitizer is not available on the GPU pool, so these checks are the
out-of-bounds net: each workload runs in a child process (a trapped kernel
poisons its CUDA context) against both libraries."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2106_14189_b200" / "_build_checked" / "libdjg.so"

WORKLOAD = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, config_spec
from paper_2106_14189_b200 import _abi as A
from paper_2106_14189_b200.parallel import EmulatedParts

out = {}
def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()

def run(name, spec, steps, flags=0, **kw):
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=flags, **kw) as eng:
        rep = eng.step(steps, raise_on_failure=False)
        u, up, st = eng.get_state()
        if name == "t4_nh":
            nxt, r2 = eng.advance_host(u, up, st)
            out["advance_host"] = [digest(nxt), r2.status]
    out[name] = [digest(u, up), rep.status, rep.step]

run("t4_nh", config_spec("cfg1", precision=4), 200)
run("t4_nh_f64", box_spec(kind="T4", divisions=(5, 4, 6), precision=8, ramp_steps=100), 100)
run("h8_ti", box_spec(kind="H8", model="TI", divisions=5, precision=4, ramp_steps=100), 100)
run("h8_ot_f64", box_spec(kind="H8", model="OT", divisions=4, precision=8, ramp_steps=100), 100)
run("t4_mr", box_spec(kind="T4", model="MR", divisions=5, precision=4, ramp_steps=100), 100)
run("t4_i57", box_spec(kind="T4", model="I57", divisions=4, precision=8, ramp_steps=100), 100)
run("t4_dev", box_spec(kind="T4", model="OT", divisions=6, precision=4, ramp_steps=100), 100,
    flags=A.DJG_FLAG_DEVICE_PRECOMPUTE, device_csr=True)
run("t4_tled", box_spec(kind="T4", divisions=6, precision=4, ramp_steps=100), 100, flags=A.DJG_FLAG_TLED)
run("t4_nopipe", box_spec(kind="T4", model="TI", divisions=6, precision=4, ramp_steps=100), 100,
    flags=A.DJG_FLAG_NO_PIPE)
for transport in ("copy", "p2p"):
    spec = box_spec(kind="T4", model="NH", divisions=6, precision=4, ramp_steps=80)
    em = EmulatedParts(Scenario(spec), 3, transport=transport)
    reps = em.step(80)
    u, up, step = em.global_state()
    em.close()
    out["parts_" + transport] = [digest(u, up), max(r.status for r in reps), step]
print(json.dumps(out))
"""


def _run(lib: Path) -> dict:
    env = dict(os.environ, DJG_LIB_PATH=str(lib))
    p = subprocess.run([sys.executable, "-c", WORKLOAD, str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, f"{lib}: rc={p.returncode}\n{p.stdout[-2000:]}\n{p.stderr[-3000:]}"
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_checked_build_no_trap_same_bits():
    if not CHECKED.exists():
        pytest.fail(f"{CHECKED} missing: build with `python -c 'import __graft_entry__ as g; g.build()'`")
    default = ROOT / "paper_2106_14189_b200" / "_build" / "libdjg.so"
    a, b = _run(CHECKED), _run(default)
    assert a.keys() == b.keys()
    for k in a:
        assert a[k] == b[k], k
        assert a[k][1] == 0, (k, a[k])
    assert np.all([v[1] == 0 for v in b.values()])
