"""Developer probe: is the GPU step bit-identical to the CPU oracle?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import oracle
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, config_spec

cases = [(k, m, p, d, s) for k in ("T4", "H8") for m in ("NH", "TI", "OT", "MR") for p in (4, 8) for d, s in [(4, 300)]]
cases += [("T4", "NH", 4, 12, 2000), ("H8", "NH", 4, 22, 2000), ("T4", "NH", 8, 12, 2000), ("H8", "TI", 4, 16, 500)]
for kind, model, prec, d, steps in cases:
    spec = box_spec(kind=kind, model=model, divisions=d, precision=prec, ramp_steps=steps)
    sc = Scenario(spec)
    with GpuDjEngine(sc) as eng:
        eng.step(steps)
        u, up, _ = eng.get_state()
    ur, upr, _ = oracle.run(spec, steps, "oracle")
    ndiff = int(np.count_nonzero(u != ur))
    print(f"{kind}-{model} f{8*prec} d={d} steps={steps}: bitwise={np.array_equal(u, ur) and np.array_equal(up, upr)} "
          f"ndiff={ndiff}/{u.size} rel={oracle.rel_max_err(u, ur):.2e}", flush=True)
