"""Multi-part soak: a SURVEY config split into k parts (EmulatedParts on one
device, both transports) for its full step protocol, against one engine;
prints one JSON line per transport. usage: soak_parts.py [cfg] [steps] [k] [4|8]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402
from paper_2106_14189_b200.parallel import EmulatedParts  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1100
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 4
spec = config_spec(cfg, precision=prec)
sc = Scenario(spec)
with GpuDjEngine(sc) as eng:
    r1 = eng.step(steps, raise_on_failure=False)
    u1, up1, _ = eng.get_state()
for transport, overlap in (("copy", True), ("p2p", False)):
    t0 = time.perf_counter()
    em = EmulatedParts(sc, k, transport=transport)
    reps = em.step(steps, overlap=overlap)
    u, up, step = em.global_state()
    em.close()
    print(json.dumps({"config": f"{cfg} f{8 * prec}, SURVEY load", "parts": k, "transport": transport,
                      "overlapped": overlap, "steps": steps, "single_status": r1.status, "single_step": r1.step,
                      "parts_status": max(r.status for r in reps), "parts_step": step,
                      "bitwise_u": bool(np.array_equal(u, u1)), "bitwise_u_prev": bool(np.array_equal(up, up1)),
                      "wall_s": time.perf_counter() - t0}), flush=True)
