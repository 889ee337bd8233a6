"""Developer A/B: graph-replay step time and per-kernel split of the default
engine under environment variants ("NAME=VALUE[,NAME=VALUE]" or "" for
none), one process per variant, interleaved twice. Optional --lib PATH
selects a library variant for all runs; AB_FLAGS=<int> sets the engine flags.  usage: ab_env.py cfg5 "" "DJG_X=0" ..."""
import json
import os
import subprocess
import sys

cfg = sys.argv[1]
variants = sys.argv[2:]
code = r'''
import json, sys, torch
sys.path.insert(0, ".")
from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec
import os
sc = Scenario(config_spec(sys.argv[1], precision=int(sys.argv[3]), target=0.01, ramp_steps=100000))
with GpuDjEngine(sc, flags=int(os.environ.get("AB_FLAGS", "0"))) as eng:
    info = eng.info()
    eng.step(10)
    s = torch.cuda.ExternalStream(eng.stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = int(sys.argv[2])
    torch.cuda.synchronize(); a.record(s); eng.step_async(K); b.record(s); b.synchronize()
    st = eng.sync().status
    e, n, t = eng.profile_steps(30)
    u = eng.get_state()[0]
import hashlib
print(json.dumps(dict(graph_us=round(a.elapsed_time(b) / K * 1e3, 1), k_element_us=round(e / 30 * 1e3, 1),
                      k_node_us=round(n / 30 * 1e3, 1), status=st, cap=info["slot_capacity"],
                      windowed=info["windowed"], u_hash=hashlib.sha1(u.tobytes()).hexdigest()[:12])))
'''
K = "100" if cfg == "cfg5" else "1000"
prec = os.environ.get("AB_PREC", "4")
for rnd in range(2):
    for v in variants:
        env = dict(os.environ)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            env[k] = val
        out = subprocess.run([sys.executable, "-c", code, cfg, K, prec], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(json.dumps(dict(cfg=cfg, variant=v or "default", round=rnd, res=line)), flush=True)
