"""Developer A/B: graph-replay time per step (the bench's timed path) for a
library variant (DJG_LIB_PATH) on one configuration."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 300
sc = Scenario(config_spec(name, precision=4, target=0.01, ramp_steps=100000))
with GpuDjEngine(sc) as eng:
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
print(json.dumps(dict(cfg=name, graph_us=out, k_element_us=round(e / 50 * 1e3, 1), k_node_us=round(n / 50 * 1e3, 1),
                      sum_us=round(t / 50 * 1e3, 1))), flush=True)
