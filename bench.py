#!/usr/bin/env python
"""DJ-TLED explicit-dynamics benchmark (BASELINE.json metric: element-steps/s
and time per explicit step on B200).

Default workload: SURVEY §8(d) cfg5 / BASELINE configs[4] -- unit cube,
4-node tets, divisions 203 (8,489,664 nodes, 50,192,562 elements),
neo-Hookean (bench_material), float32, zmin fixed, zmax ramped +1% in z
over the run (the reference bench's loading, bench.hpp:52-72), dt = 0.5
critical_dt, alpha = relaxation_alpha. One "step" = one advance_step: element
forces -> CSR gather -> central-difference update.

  value     element-steps/s with the problem resident in HBM, device time from
            CUDA events on the engine stream (max over ranks)
  e2e       the same metric through the public C-ABI with host state: every
            step uploads u_curr/u_prev from pinned host memory, advances one
            step and reads u_curr back (advance_step with a host SimState)
  roofline  k_element's algorithmic bytes / its average event-timed duration
            against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the unmodified reference (oracle/_ref, all host threads) on a
            bounded sample of the same workload

`--impl reference` times the reference's own CPU implementation instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np

METRIC = "DJ-TLED element-steps/sec at 1/2/4/8 B200; time per explicit step"
UNIT = "element-steps/s"
# Hot-constant bytes per element in f32.
CONST_BYTES = {("T4", "NH"): 92, ("T4", "TI"): 140, ("H8", "NH"): 224, ("H8", "TI"): 272,
               ("T4", "OT"): 188, ("H8", "OT"): 320, ("T4", "MR"): 320, ("H8", "MR"): 452}
SAMPLE_DIVISIONS = 70   # reference CPU sample: cfg3-sized T4 box (2,058,000 elements)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algo_bytes(kind: str, model: str, N: int, E: int, prec: int) -> dict:
    """SURVEY §8(d) algorithmic bytes per step, split by kernel."""
    npe = 4 if kind == "T4" else 8
    C = CONST_BYTES[(kind, model)] * (prec // 4)
    r = prec  # bytes per Real
    # k_element: conn 4npe + slot index 4npe + constants C + force write 3r*npe per
    # element; gathered u (3r) once per node.
    k1 = E * (8 * npe + C + 3 * r * npe) + 3 * r * N
    # k_node: force read 3r*npe per element; u_curr, u_prev read, u_next write,
    # c1, CSR row length 4, BC code 1 per node.
    k2 = E * 3 * r * npe + N * (10 * r + 5)
    return {"k_element": k1, "k_node": k2, "step": k1 + k2}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference_sample(steps: int, warmup: int, kind: str, model: str, precision: int) -> dict:
    """The unmodified reference's advance_step loop (oracle/_ref) on the host,
    all threads, on a bounded sample of the workload. Falls back to the C
    restatement (kind "port") only where the reference library is absent."""
    import oracle
    from paper_2106_14189_b200.spec import box_spec
    threads = os.cpu_count() or 1
    spec = box_spec(kind=kind, model=model, divisions=SAMPLE_DIVISIONS, precision=precision, target=0.01,
                    ramp_steps=warmup + steps)
    E = SAMPLE_DIVISIONS ** 3 * (6 if kind == "T4" else 1)
    if oracle.have("ref"):
        sec = oracle.ref_time_steps(spec, warmup, steps, threads, 0)
        kind_s = "reference"
    else:
        t0 = time.perf_counter()
        oracle.run(spec, warmup, "oracle", threads=threads)
        t1 = time.perf_counter()
        oracle.run(spec, warmup + steps, "oracle", threads=threads)
        t2 = time.perf_counter()
        sec = ((t2 - t1) - (t1 - t0)) / steps
        kind_s = "port"
    return {"value": E / sec, "unit": UNIT, "cores": threads, "kind": kind_s,
            "ms_per_step": sec * 1e3,
            "sample": f"{kind}-{model} box d={SAMPLE_DIVISIONS} ({E} elements), {warmup} warm-up + {steps} timed "
                      f"advance_step calls, f{8 * precision}, OMP threads={threads}"}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    steps = max(args.steps, 1)
    cb = cpu_reference_sample(steps, max(args.warmup, 1), args.kind, args.model, args.precision)
    line = {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == 4 else "f64",
        "data": "synthetic (generate_box unit cube, bench_material)",
        "config": {"workload": f"cfg5 reference sample: {args.kind}-{args.model} box d={SAMPLE_DIVISIONS}",
                   "kind": args.kind, "material": args.model, "divisions": SAMPLE_DIVISIONS},
        "impl": "reference",
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def our_arm(args):
    import torch

    from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec

    rank, world, local = dist_env()
    device = local
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    if world > 1:
        raise SystemExit("multi-GPU partitioned stepping is not wired into bench.py yet")

    K, W = args.steps, max(args.warmup, 3)
    total = W + K + args.e2e_steps + 8
    spec = box_spec(kind=args.kind, model=args.model, divisions=args.divisions, precision=args.precision,
                    target=0.01, ramp_steps=total)
    t0 = time.perf_counter()
    sc = Scenario(spec)
    t1 = time.perf_counter()
    eng = GpuDjEngine(sc, device=device)
    t2 = time.perf_counter()
    log(f"[bench] N={sc.num_nodes} E={sc.num_elements} build {t1 - t0:.1f}s create {t2 - t1:.1f}s "
        f"device {eng.info()['device_bytes'] / 1e9:.2f} GB")
    N, E = sc.num_nodes, sc.num_elements

    eng.step(W)                          # warm-up (graphs captured, clocks up)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(device)
    clocks.start()
    ms_e, ms_n, ms_tot = eng.profile_steps(K)   # CUDA events on the engine stream
    rep = eng.sync()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if rep.status != 0 or rep.steps_done != K:
        raise SystemExit(f"timed run failed: {rep}")
    ms_step = ms_tot / K
    if dist:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = E * world / (ms_step * 1e-3)

    # Graph-replayed steps (no per-kernel events) for reference.
    s = torch.cuda.ExternalStream(eng.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    eng.step_async(K)
    ev1.record(s)
    ev1.synchronize()
    eng.sync()
    ms_graph = ev0.elapsed_time(ev1) / K

    # e2e: advance_step with a host-resident SimState through the public API.
    rdt = np.float32 if args.precision == 4 else np.float64
    u_h = torch.empty(3 * N, dtype=torch.float32 if args.precision == 4 else torch.float64).pin_memory()
    up_h = torch.empty_like(u_h).pin_memory()
    u_out = torch.empty_like(u_h).pin_memory()
    uc, upv, st = eng.get_state()
    u_h.numpy()[:] = uc
    up_h.numpy()[:] = upv
    lib = __import__("paper_2106_14189_b200._abi", fromlist=["x"]).load_library()
    import ctypes as C
    from paper_2106_14189_b200 import _abi as A
    h = eng._h
    step_c = C.c_int64(st)
    rep_c = A.djg_report()
    pu, pup, pout = (C.c_void_p(t.data_ptr()) for t in (u_h, up_h, u_out))
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        lib.djg_set_state(h, pu, pup, step_c.value)
        rc = lib.djg_step(h, 1, C.byref(rep_c))
        lib.djg_get_state(h, pout, pup, C.byref(step_c))
        if rc:
            raise SystemExit(f"e2e step failed rc={rc}")
        pu, pout = pout, pu
    te1 = time.perf_counter()
    e2e_ms = (te1 - te0) / args.e2e_steps * 1e3
    rbytes = args.precision
    h2d = 2 * 3 * N * rbytes
    d2h = 2 * 3 * N * rbytes

    hbm, peak_kind = peaks()
    B = algo_bytes(args.kind, args.model, N, E, args.precision)
    k1_ms = ms_e / K
    achieved = B["k_element"] / (k1_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == 4 else "f64",
        "data": "synthetic (generate_box unit cube, bench_material NH, +1% z-extension ramp)",
        "config": {"workload": f"cfg5: {args.kind}-{args.model} unit cube d={args.divisions}",
                   "kind": args.kind, "material": args.model, "divisions": args.divisions,
                   "num_nodes": N, "num_elements": E, "parallelism": f"{world} GPU",
                   "l2": "inputs larger than L2 (state ~%.1f GB)" % (eng.info()["device_bytes"] / 1e9)},
        "e2e": {"value": E / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms,
                "mode": "per step: H2D u_curr+u_prev (pinned), djg_step(1), D2H u_curr+u_prev"},
        "roofline": {"bound": "hbm", "kernel": "k_element", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None, "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": B["k_element"], "launch_ms": k1_ms,
                     "step_frac": B["step"] / (ms_step * 1e-3) / 1e9 / hbm,
                     "k_node_ms": ms_n / K, "k_node_frac": B["k_node"] / (ms_n / K * 1e-3) / 1e9 / hbm},
        "ms_per_step_graph": ms_graph,
        "gpu_launches": 2 * K,
        "clocks": clk,
        "time_per_step_us": ms_step * 1e3,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_sample(args.cpu_steps, 2, args.kind, args.model, args.precision)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    eng.close()
    sc.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="T4")
    ap.add_argument("--model", default="NH")
    ap.add_argument("--divisions", type=int, default=203)
    ap.add_argument("--precision", type=int, default=4, choices=[4, 8])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()
