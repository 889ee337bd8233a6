"""Developer A/B: node-windowed element kernel vs the global-gather pipeline
(the default) on one configuration: graph-replay time per step, the
per-kernel split, and bitwise equality of the two states after the run."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14189_b200 import GpuDjEngine, Scenario, _abi as A, config_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sc = Scenario(config_spec(name, precision=prec, target=0.01, ramp_steps=100000))
res = {}
states = {}
for label, flags in (("win", A.DJG_FLAG_WINDOW), ("nowin", 0), ("win2", A.DJG_FLAG_WINDOW)):
    with GpuDjEngine(sc, flags=flags) as eng:
        info = eng.info()
        eng.step(10)
        s = torch.cuda.ExternalStream(eng.stream)
        out = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            eng.step_async(K)
            b.record(s)
            b.synchronize()
            eng.sync()
            out.append(round(a.elapsed_time(b) / K * 1e3, 1))
        e, n, t = eng.profile_steps(50)
        status = eng.sync().status
        states[label] = eng.get_state()[0]
        res[label] = dict(graph_us=out, k_element_us=round(e / 50 * 1e3, 1), k_node_us=round(n / 50 * 1e3, 1),
                          status=status, windowed=info["windowed"], window_tiles=info["window_tiles"],
                          device_gb=round(info["device_bytes"] / 1e9, 2))
res["bitwise"] = bool(np.array_equal(states["win"], states["nowin"]))
print(json.dumps(dict(cfg=name, prec=prec, **res)), flush=True)
