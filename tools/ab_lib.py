"""Developer A/B: graph-replay step time and per-kernel split of the default
engine for each library variant given (paths to libdjg.so, "" = in-tree),
one process per variant, interleaved twice."""
import json
import os
import subprocess
import sys

cfg = sys.argv[1]
libs = sys.argv[2:]
code = r'''
import json, sys, torch
sys.path.insert(0, ".")
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec
sc = Scenario(config_spec(sys.argv[1], precision=4, target=0.01, ramp_steps=100000))
with GpuDjEngine(sc) as eng:
    eng.step(10)
    s = torch.cuda.ExternalStream(eng.stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = int(sys.argv[2])
    torch.cuda.synchronize(); a.record(s); eng.step_async(K); b.record(s); b.synchronize()
    st = eng.sync().status
    e, n, t = eng.profile_steps(30)
    print(json.dumps(dict(graph_us=round(a.elapsed_time(b) / K * 1e3, 1), k_element_us=round(e / 30 * 1e3, 1),
                          k_node_us=round(n / 30 * 1e3, 1), status=st)))
'''
K = "100" if cfg == "cfg5" else "1000"
for rnd in range(2):
    for lib in libs:
        env = dict(os.environ)
        if lib:
            env["DJG_LIB_PATH"] = lib
        out = subprocess.run([sys.executable, "-c", code, cfg, K], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(json.dumps(dict(cfg=cfg, lib=lib or "default", round=rnd, res=line)), flush=True)
