"""Developer A/B probe: k_element / k_node device time for a library variant
(DJG_LIB_PATH) on one configuration; prints the run status so timing
experiments that break the physics are visible."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402

for name in sys.argv[1:] or ["cfg5"]:
    sc = Scenario(config_spec(name, precision=4, target=0.01, ramp_steps=100000))
    import os
    eng = GpuDjEngine(sc, flags=int(os.environ.get("DJG_FLAGS", "0")))
    pipe = eng.info()["pipelined"]
    eng.step(3, raise_on_failure=False)
    ms_e, ms_n, ms_t = eng.profile_steps(20)
    r = eng.sync()
    print(json.dumps(dict(cfg=name, k_element_us=round(ms_e / 20 * 1e3, 1), k_node_us=round(ms_n / 20 * 1e3, 1),
                          status=r.status, steps=r.step, pipe=pipe)), flush=True)
    eng.close()
    sc.close()
