"""Developer A/B: f64 kernel times on SURVEY configs (DJG_LIB_PATH variant)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402

for name in sys.argv[1:] or ["cfg3", "cfg5"]:
    sc = Scenario(config_spec(name, precision=8, target=0.01, ramp_steps=100000))
    with GpuDjEngine(sc) as eng:
        eng.step(3)
        e, n, t = eng.profile_steps(20)
        print(json.dumps(dict(cfg=name, prec=8, k_element_us=round(e / 20 * 1e3, 1), k_node_us=round(n / 20 * 1e3, 1))),
              flush=True)
    sc.close()
