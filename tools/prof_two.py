"""Developer tool: one cfg, two engines (DJG_FLAG_WINDOW and the
default pipeline), a few plain steps each -- for one ncu capture holding
both element kernels."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec
from paper_2106_14189_b200 import _abi as A

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = Scenario(config_spec(name, precision=4, target=0.01, ramp_steps=100000))
for fl in (A.DJG_FLAG_WINDOW, 0):
    with GpuDjEngine(sc, flags=A.DJG_FLAG_NO_GRAPH | fl) as eng:
        r = eng.step(steps)
    print(name, fl, "steps", r.step, "status", r.status)
