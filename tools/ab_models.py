"""Developer A/B: element-kernel (DJG_KIND, default T4) time per material model and precision for
a library variant (DJG_LIB_PATH) and flag set (DJG_FLAGS); args 'MODEL:PREC'."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec  # noqa: E402

divs = int(os.environ.get("DJG_DIVS", "120"))
kind = os.environ.get("DJG_KIND", "T4")
flags = int(os.environ.get("DJG_FLAGS", "0"))
for arg in sys.argv[1:]:
    model, prec = arg.split(":")
    sc = Scenario(box_spec(kind=kind, model=model, divisions=divs, precision=int(prec), target=0.01,
                           ramp_steps=100000))
    with GpuDjEngine(sc, flags=flags) as eng:
        info = eng.info()
        eng.step(3, raise_on_failure=False)
        e, n, t = eng.profile_steps(20)
        r = eng.sync()
        print(json.dumps(dict(kind=kind, model=model, prec=prec, flags=flags, k_element_us=round(e / 20 * 1e3, 1),
                              k_node_us=round(n / 20 * 1e3, 1), status=r.status, compact=info.get("compact"),
                              pipe=info["pipelined"])), flush=True)
    sc.close()
