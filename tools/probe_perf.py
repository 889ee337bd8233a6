"""Developer probe: per-kernel device time and roofline fraction of the step
on the SURVEY §8(d) configurations (not the bench contract; see bench.py)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec

PEAK = 6552.0  # MEASURED_PEAKS.json hbm_gbs
C = {("T4", "NH"): 92, ("T4", "TI"): 140, ("H8", "NH"): 224, ("H8", "TI"): 272}


def algo_bytes(kind, model, N, E, prec=4):
    npe = 4 if kind == "T4" else 8
    c = C[(kind, model)]
    if prec == 4:
        return E * (32 * npe + c) + 57 * N
    return E * (56 * npe + 2 * c) + 109 * N


def main(names):
    for name in names:
        from paper_2106_14189_b200.spec import CONFIGS
        cf = CONFIGS[name]
        for prec in (4,):
            t0 = time.perf_counter()
            sc = Scenario(config_spec(name, precision=prec, target=0.01, ramp_steps=100000))
            t1 = time.perf_counter()
            import os
            eng = GpuDjEngine(sc, flags=int(os.environ.get('DJG_FLAGS', '0')))
            t2 = time.perf_counter()
            eng.step(10)
            ms_e, ms_n, ms_t = eng.profile_steps(50)
            eng.set_state(None, None, 0)
            eng.step(5)
            import ctypes
            # graph-replayed wall time per step
            t3 = time.perf_counter()
            eng.step(200)
            t4 = time.perf_counter()
            B = algo_bytes(cf["kind"], cf["model"], sc.num_nodes, sc.num_elements, prec)
            step_ms = (t4 - t3) / 200 * 1e3
            out = dict(cfg=name, prec=prec, N=sc.num_nodes, E=sc.num_elements, build_s=round(t1 - t0, 2),
                       create_s=round(t2 - t1, 2), k_element_us=round(ms_e / 50 * 1e3, 2),
                       k_node_us=round(ms_n / 50 * 1e3, 2), step_us_events=round(ms_t / 50 * 1e3, 2),
                       step_us_graph=round(step_ms * 1e3, 2),
                       roofline_frac=round(B / (step_ms * 1e-3) / 1e9 / PEAK, 3),
                       el_steps_per_s=round(sc.num_elements / (step_ms * 1e-3) / 1e9, 3), info=eng.info())
            print(json.dumps(out), flush=True)
            eng.close()
            sc.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
