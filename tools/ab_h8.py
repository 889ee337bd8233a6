"""Developer A/B: H8 element/node kernel times per material, full vs compact
record (DJG_LIB_PATH selects the library variant)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec  # noqa: E402
from paper_2106_14189_b200 import _abi as A  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for prec in (4, 8):
    for model in ("NH", "TI", "OT", "MR"):
        sc = Scenario(box_spec(kind="H8", model=model, divisions=d, precision=prec, target=0.01, ramp_steps=100000))
        out = {"model": model, "prec": prec}
        for name, fl in (("full", A.DJG_FLAG_FULL_RECORD), ("compact", A.DJG_FLAG_COMPACT)):
            with GpuDjEngine(sc, flags=fl) as eng:
                eng.step(3)
                e, n, t = eng.profile_steps(20)
                out[name] = round(e / 20 * 1e3, 1)
                out["node"] = round(n / 20 * 1e3, 1)
        print(json.dumps(out), flush=True)
        sc.close()
