"""Soak parity run: a SURVEY config (default cfg5: T4-NH d=203, 50.2M tets,
20 % compression ramp) for its full step protocol on the GPU, against the CPU
oracle on the host cores; prints one JSON line (bitwise verdict, max relative
error, timings). Minutes of host time: run on the GPU box, not in the test
suite.  usage: soak.py [cfg] [steps] [ext|ramp] [4|8]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 550
ext = len(sys.argv) > 3 and sys.argv[3] == "ext"  # the reference bench's +1 % extension ramp
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 4
spec = (config_spec(cfg, precision=prec, target=0.01, ramp_steps=steps) if ext
        else config_spec(cfg, precision=prec))
t0 = time.perf_counter()
sc = Scenario(spec)
with GpuDjEngine(sc) as eng:
    t1 = time.perf_counter()
    rep = eng.step(steps, raise_on_failure=False)
    t2 = time.perf_counter()
    u, up, st = eng.get_state()
sc.close()
t3 = time.perf_counter()
ur, upr, rr = oracle.run(spec, steps, "oracle")
t4 = time.perf_counter()
out = {
    "config": f"{cfg} f{8 * prec}, " + ("+1 % extension ramp" if ext else "SURVEY load (20 % compression)"),
    "steps": steps, "gpu_status": rep.status, "gpu_step": rep.step, "oracle": rr,
    "bitwise_u": bool(np.array_equal(u, ur)), "bitwise_u_prev": bool(np.array_equal(up, upr)),
    "rel_max_err": oracle.rel_max_err(u, ur), "max_abs_u": float(np.abs(ur).max()),
    "gpu_build_s": t1 - t0, "gpu_steps_s": t2 - t1, "oracle_s": t4 - t3,
}
print(json.dumps(out), flush=True)
