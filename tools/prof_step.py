"""Developer tool: build one SURVEY config and run W+K plain (non-graph)
steps, for ncu launch lists and full captures."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec
from paper_2106_14189_b200 import _abi as A

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sc = Scenario(config_spec(name, precision=prec, target=0.01, ramp_steps=100000))
with GpuDjEngine(sc, flags=A.DJG_FLAG_NO_GRAPH) as eng:
    r = eng.step(steps)
print(name, "steps", r.step, "status", r.status)
