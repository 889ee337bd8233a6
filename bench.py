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
  e2e       the same metric through the public C-ABI with host state
            (djg_advance_host): every step uploads u_curr/u_prev from pinned
            host memory, advances one step and reads the new u_curr back
  roofline  k_element's algorithmic bytes / its average event-timed duration
            against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the unmodified reference (oracle/_ref) on the same workload:
            all host threads (and one thread), a bounded number of steps

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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# Kernel sources whose content the committed ncu traffic numbers belong to.
KERNEL_SOURCES = ("paper_2106_14189_b200/csrc/cuda/kernels.cuh", "paper_2106_14189_b200/csrc/cuda/engine.cu",
                  "paper_2106_14189_b200/csrc/common/element_math.hpp")


def source_hash() -> str:
    """sha256 (first 16 hex digits) of the kernel sources, as
    tools/ncu_traffic.py records it next to each capture."""
    import hashlib
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        h.update((ROOT / f).read_bytes())
    return h.hexdigest()[:16]


def measured_traffic(workload: str, kernel_prefix: str):
    """DRAM bytes per launch of a kernel from the newest committed ncu launch
    list of the same workload (profiles/r*/ncu_traffic.json, made by
    tools/ncu_traffic.py from `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum`): (bytes, source, stale). `stale` is True when the
    capture's kernel-source hash differs from the sources built here."""
    for p in sorted((ROOT / "profiles").glob("r*/ncu_traffic.json"), reverse=True):
        d = json.loads(p.read_text()).get(workload)
        if not d:
            continue
        for k, v in d["kernels"].items():
            if k.startswith(kernel_prefix):
                src = f"{p.relative_to(ROOT).parent}/{d['source']} ({k}, ncu, per launch)"
                return v["dram_bytes_per_launch"], src, d.get("source_hash") != source_hash()
    return None, None, None


def measured_issue(workload: str, kernel_prefix: str):
    """ncu's smsp__issue_active (fraction of peak) of the kernel from the
    newest ncu_traffic.json that recorded it, or None."""
    for p in sorted((ROOT / "profiles").glob("r*/ncu_traffic.json"), reverse=True):
        d = json.loads(p.read_text()).get(workload)
        if not d:
            continue
        for k, v in d["kernels"].items():
            if k.startswith(kernel_prefix) and v.get("issue_active_pct") is not None:
                return v["issue_active_pct"] / 100
    return None


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
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes ~0.1-0.3 s to report: wait for its first line so
            # short timed regions are sampled too
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
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


def _mem_available() -> int:
    """Host bytes this process may still allocate: MemAvailable, capped by
    the cgroup limit when there is one."""
    avail = 1 << 62
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    for p in ("/sys/fs/cgroup/memory.max", "/sys/fs/cgroup/memory/memory.limit_in_bytes"):
        try:
            v = open(p).read().strip()
            if v.isdigit():
                avail = min(avail, int(v))
        except OSError:
            pass
    return avail


def _peak_rss_gb() -> float:
    import resource
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20


def _ref_host_bytes(kind: str, d: int, precision: int, tled: bool) -> int:
    """Peak host memory of the reference's DjEngine on a d^3 box: the AoS
    ElementConstants (1196 B f32 / 2384 B f64, every optional block
    allocated), the 16-byte CSR pairs, connectivity and the
    element-force scratch; TLED adds its 236 B (f32) record while the DJ
    model is still alive."""
    npe = 4 if kind == "T4" else 8
    E = d ** 3 * (6 if kind == "T4" else 1)
    rec = 1196 if precision == 4 else 2384
    per = rec + npe * (16 + 4 + 3 * precision) + (236 * precision // 4 if tled else 0)
    return int(E * per * 1.1) + (2 << 30)


def cpu_reference_protocol(args, warmup: int, steps: int, one_thread: bool, tled: bool) -> dict:
    """SURVEY §8(d)'s CPU path on the bench workload itself: the unmodified
    reference (oracle/_ref: DjEngine + advance_step, the bench.hpp:87-95
    loop), built with build_threads = all host threads (solver.hpp:264-267;
    the build is not timed), then `warmup` + `steps` timed steps on all host
    threads, 1 + 2 steps on one thread, and the same all-thread protocol on
    the reference's TledEngine for the paper's DJ/TLED ratio. Falls back to
    the C restatement (kind "port") only where the reference library is
    absent, and to a smaller box only when host memory cannot hold the
    reference's AoS constants (same_config false, said in `sample`)."""
    import oracle
    from paper_2106_14189_b200.spec import box_spec
    threads = os.cpu_count() or 1
    d = args.divisions
    need = _ref_host_bytes(args.kind, d, args.precision, tled)
    avail = _mem_available()
    note = ""
    while need > avail and d > 8:
        d = int(d * 0.8)
        need = _ref_host_bytes(args.kind, d, args.precision, tled)
    if d != args.divisions:
        note = (f"; host memory {avail / 2**30:.0f} GiB cannot hold the reference's cfg d={args.divisions} "
                f"constants: sampled d={d}")
    E = d ** 3 * (6 if args.kind == "T4" else 1)
    spec = box_spec(kind=args.kind, model=args.model, divisions=d, precision=args.precision, target=0.01,
                    ramp_steps=warmup + steps)
    out = {"nproc": threads, "divisions": d, "num_elements": E, "same_config": d == args.divisions,
           "omp_proc_bind": os.environ.get("OMP_PROC_BIND")}
    if oracle.have("ref"):
        runs = [(threads, warmup, steps)] + ([(1, 1, 2)] if one_thread else [])
        secs, build = oracle.ref_time_protocol(spec, 0, threads, runs)
        out.update(kind="reference", sec=secs[0], build_s=build)
        if one_thread:
            out["threads_1"] = {"value": E / secs[1], "unit": UNIT, "ms_per_step": secs[1] * 1e3, "cores": 1,
                                "sample": "1 warm-up + 2 timed advance_step calls, 1 thread"}
        if tled:
            tsecs, tbuild = oracle.ref_time_protocol(spec, 2, threads, [(threads, warmup, steps)])
            out["tled"] = {"value": E / tsecs[0], "unit": UNIT, "ms_per_step": tsecs[0] * 1e3, "cores": threads,
                           "dj_over_tled_time": secs[0] / tsecs[0], "build_s": tbuild,
                           "sample": f"reference TledEngine, {warmup} warm-up + {steps} timed steps, "
                                     f"{threads} threads (paper Table 5 ratio)"}
    else:
        t0 = time.perf_counter()
        oracle.run(spec, warmup, "oracle", threads=threads)
        t1 = time.perf_counter()
        oracle.run(spec, warmup + steps, "oracle", threads=threads)
        t2 = time.perf_counter()
        out.update(kind="port", sec=((t2 - t1) - (t1 - t0)) / steps, build_s=None)
    sec = out["sec"]
    out.update(value=E / sec, unit=UNIT, cores=threads, ms_per_step=sec * 1e3,
               sample=f"{args.kind}-{args.model} box d={d} ({E} elements), {warmup} warm-up + {steps} timed "
                      f"advance_step calls, f{8 * args.precision}, {threads} threads (all host threads), "
                      f"build_threads={threads} (build untimed){note}")
    return out


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # SURVEY §8(d)'s cfg5 CPU protocol is 3 warm-up + 10 timed steps: the
    # driver's K is capped there so the arm ends within a few minutes, and
    # the 3 warm-up steps are kept (the first steps after a multi-threaded
    # build run several times slower while the kernel settles the freshly
    # touched pages).
    W, K = 3, min(max(args.steps, 1), 10)
    cb = cpu_reference_protocol(args, W, K, one_thread=True, tled=True)
    line = {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": K,
        "warmup": W, "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if args.precision == 4 else "f64",
        "data": "synthetic (generate_box unit cube, bench_material, +1% z-extension ramp)",
        "config": {"workload": f"{cfg_name(args)}: {args.kind}-{args.model} unit cube d={cb['divisions']}",
                   "kind": args.kind, "material": args.model, "divisions": cb["divisions"],
                   "num_elements": cb["num_elements"], "parallelism": f"{cb['nproc']} host threads"},
        "impl": "reference",
        "same_config": cb["same_config"],
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "nproc": cb["nproc"], "build_s": cb["build_s"], "host_peak_rss_gb": _peak_rss_gb(),
        "steps_note": f"SURVEY §8(d)'s CPU protocol: 3 warm-up + min(K, 10) timed steps (asked K={args.steps}, W={args.warmup})",
    }
    for k in ("threads_1", "tled"):
        if k in cb:
            line[k] = cb[k]
    print(json.dumps(line), flush=True)


def _cpu_baseline_line(args):
    """cpu_baseline: the reference on the bench workload itself, a bounded
    number of steps (2 warm-up + 3 timed on all threads, 1 + 2 on one)."""
    try:
        cb = cpu_reference_protocol(args, 2, args.cpu_steps, one_thread=True, tled=False)
        r = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        r.update(same_config=cb["same_config"], nproc=cb["nproc"], ms_per_step=cb["ms_per_step"])
        if "threads_1" in cb:
            r["threads_1"] = cb["threads_1"]
        return r
    except Exception as ex:  # reported, not fatal
        return {"value": None, "error": str(ex)}


def element_kernel_prefix(info) -> str:
    if info.get("fused"):
        return "k_box_step"
    if info.get("windowed"):
        return "k_element_win"
    return "k_element_pipe" if info.get("pipelined") else "k_element<"


def sub_config(name: str, device: int, warmup: int = 100, steps: int = 1000) -> dict:
    """SURVEY §8(d)'s roofline gate on cfg3 / cfg4 (one GPU, f32): graph
    replay, `warmup` untimed + `steps` timed steps (events on the engine
    stream), the per-kernel split from profile_steps, the step's fraction of
    the HBM peak on algorithmic bytes and the element kernel's fraction on the
    DRAM bytes ncu measured for it (moved_frac)."""
    import torch

    from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec
    from paper_2106_14189_b200.spec import CONFIGS
    c = CONFIGS[name]
    sc = Scenario(config_spec(name, precision=4, target=0.01, ramp_steps=warmup + steps + 200))
    N, E = sc.num_nodes, sc.num_elements
    with GpuDjEngine(sc, device=device) as eng:
        info = eng.info()
        eng.step(warmup)
        s = torch.cuda.ExternalStream(eng.stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        eng.step_async(steps)
        b.record(s)
        b.synchronize()
        rep = eng.sync()
        me, mn, _ = eng.profile_steps(100)
    sc.close()
    ms = a.elapsed_time(b) / steps
    hbm, _ = peaks()
    B = algo_bytes(c["kind"], c["model"], N, E, 4)
    traffic, src, stale = measured_traffic(name, element_kernel_prefix(info))
    k1 = me / 100
    fused = bool(info.get("fused"))  # one kernel: its algorithmic bytes are the step's
    return {"workload": f"{name}: {c['kind']}-{c['model']} unit cube d={c['divisions']}", "num_elements": E,
            "num_nodes": N, "steps": steps, "warmup": warmup, "status": rep.status, "ms_per_step": ms,
            "value": E / (ms * 1e-3), "unit": UNIT, "kernel": element_kernel_prefix(info), "fused": int(fused),
            "lattice": int(info.get("lattice", 0)), "k_element_ms": k1, "k_node_ms": mn / 100,
            "step_frac": B["step"] / (ms * 1e-3) / 1e9 / hbm,
            "k_element_frac": B["step" if fused else "k_element"] / (k1 * 1e-3) / 1e9 / hbm,
            "moved_frac": (traffic / (k1 * 1e-3) / 1e9 / hbm) if traffic else None, "traffic": traffic,
            "traffic_source": src, "traffic_stale": stale,
            "issue_active": measured_issue(name, element_kernel_prefix(info))}


# SURVEY §8(d) config names, keyed by (kind, material, divisions).
CFG_NAMES = {("T4", "NH", 12): "cfg1", ("H8", "NH", 22): "cfg2", ("T4", "NH", 70): "cfg3",
             ("H8", "TI", 100): "cfg4", ("T4", "NH", 203): "cfg5"}


def cfg_name(args):
    return CFG_NAMES.get((args.kind, args.model, args.divisions), "custom")


def _line(args, world, K, W, E, ms_step, value, extra):
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if args.precision == 4 else "f64",
        "data": "synthetic (generate_box unit cube, bench_material, +1% z-extension ramp)",
        "config": {"workload": f"{cfg_name(args)}: {args.kind}-{args.model} unit cube d={args.divisions}",
                   "kind": args.kind, "material": args.model, "divisions": args.divisions,
                   "num_elements": E, "parallelism": f"{world} GPU" + (f" ({args.partition.upper()} partition, {args.transport} halo)" if world > 1 else "")},
        "time_per_step_us": ms_step * 1e3,
    }
    line.update(extra)
    return line


def our_arm(args):
    import torch

    from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec

    rank, world, local = dist_env()
    device = local
    torch.cuda.set_device(device)
    if world > 1 or os.environ.get("DJG_BENCH_FORCE_MULTI") == "1":
        return multi_arm(args, rank, world, device)

    K, W = args.steps, max(args.warmup, 3)
    total = W + 3 * K + args.e2e_steps + 8
    spec = box_spec(kind=args.kind, model=args.model, divisions=args.divisions, precision=args.precision,
                    target=0.01, ramp_steps=total)
    t0 = time.perf_counter()
    sc = Scenario(spec)
    t1 = time.perf_counter()
    eng = GpuDjEngine(sc, device=device)
    t2 = time.perf_counter()
    info = eng.info()
    log(f"[bench] N={sc.num_nodes} E={sc.num_elements} build {t1 - t0:.1f}s create {t2 - t1:.1f}s "
        f"device {info['device_bytes'] / 1e9:.2f} GB")
    N, E = sc.num_nodes, sc.num_elements

    eng.step(W)                          # warm-up (graphs captured, clocks up)
    torch.cuda.synchronize()
    clocks = ClockSampler(device)
    clocks.start()
    # Timed region 1: per-kernel CUDA events on the engine stream.
    ms_e, ms_n, ms_tot = eng.profile_steps(K)
    rep = eng.sync()
    # Timed region 2: the production path (CUDA graph replay), events on the
    # engine stream around the whole region.
    s = torch.cuda.ExternalStream(eng.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(s)
    eng.step_async(K)
    ev1.record(s)
    ev1.synchronize()
    rep2 = eng.sync()
    clk = clocks.stop()
    if rep.status != 0 or rep2.status != 0 or rep.steps_done != K or rep2.steps_done != K:
        raise SystemExit(f"timed run failed: {rep} {rep2}")
    ms_graph = ev0.elapsed_time(ev1) / K
    ms_step = ms_graph
    value = E / (ms_step * 1e-3)

    # e2e: advance_step with a host-resident SimState through the public C-ABI.
    import ctypes as C

    from paper_2106_14189_b200 import _abi as A
    lib = A.load_library()
    tdt = torch.float32 if args.precision == 4 else torch.float64
    u_h = torch.empty(3 * N, dtype=tdt).pin_memory()
    up_h = torch.empty_like(u_h).pin_memory()
    u_out = torch.empty_like(u_h).pin_memory()
    uc, upv, st = eng.get_state()
    u_h.numpy()[:] = uc
    up_h.numpy()[:] = upv
    h = eng._h
    step_c = C.c_int64(st)
    rep_c = A.djg_report()
    # Host SimState rotation: the step's inputs (u_curr, u_prev) go up, the
    # result u_curr comes back; the next u_prev is the host's previous u_curr.
    cur, prev, spare = (C.c_void_p(t.data_ptr()) for t in (u_h, up_h, u_out))
    lib.djg_advance_host(h, cur, prev, step_c.value, spare, C.byref(rep_c))  # untimed: first-call setup
    step_c.value = rep_c.step
    cur, prev, spare = spare, cur, prev
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        rc = lib.djg_advance_host(h, cur, prev, step_c.value, spare, C.byref(rep_c))
        if rc:
            raise SystemExit(f"e2e step failed rc={rc}")
        step_c.value = rep_c.step
        cur, prev, spare = spare, cur, prev
    te1 = time.perf_counter()
    e2e_ms = (te1 - te0) / args.e2e_steps * 1e3 if args.e2e_steps > 0 else 1.0
    # The run_simulation path (solver.hpp:205-258) through the C-ABI: the
    # host SimState goes up once (djg_set_state from pinned host), K steps
    # run on the device (graph replay, failure checks on the device), the
    # state comes back (djg_get_state); wall clock around all of it.
    ru = C.c_int64(0)
    torch.cuda.synchronize()
    tr0 = time.perf_counter()
    if lib.djg_set_state(h, C.c_void_p(u_h.data_ptr()), C.c_void_p(up_h.data_ptr()), step_c.value):
        raise SystemExit("djg_set_state failed")
    if lib.djg_step(h, K, C.byref(rep_c)) or rep_c.steps_done != K:
        raise SystemExit(f"run path failed: status {rep_c.status}")
    if lib.djg_get_state(h, C.c_void_p(u_h.data_ptr()), C.c_void_p(up_h.data_ptr()), C.byref(ru)):
        raise SystemExit("djg_get_state failed")
    tr1 = time.perf_counter()
    run_ms = (tr1 - tr0) / K * 1e3
    rbytes = args.precision

    hbm, peak_kind = peaks()
    B = algo_bytes(args.kind, args.model, N, E, args.precision)
    k1_ms = ms_e / K
    fused = bool(info.get("fused"))
    # the fused box step is the whole step in one kernel: its algorithmic
    # bytes are the step's
    algo_k1 = B["step"] if fused else B["k_element"]
    achieved = algo_k1 / (k1_ms * 1e-3) / 1e9
    traffic, traffic_src, stale, issue = None, None, None, None
    if cfg_name(args) != "custom" and args.precision == 4:
        traffic, traffic_src, stale = measured_traffic(cfg_name(args), element_kernel_prefix(info))
        issue = measured_issue(cfg_name(args), element_kernel_prefix(info))
    extra = {
        "e2e": {"value": E / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 2 * 3 * N * rbytes,
                "d2h_bytes_per_step": 3 * N * rbytes, "ms_per_step": e2e_ms,
                "mode": ("per step: djg_advance_host -- advance_step with a host SimState: H2D u_curr and "
                         "u_prev from pinned host, region by region (8 tapered runs of node layers; u_curr and "
                         "u_prev on two copy streams), the fused box step launched on each region's layers as "
                         "soon as they have landed, each region's new u_curr D2H on the other copy direction "
                         "behind the next region; the next u_prev is the host's previous u_curr; wall clock"
                         if fused else
                         "per step: djg_advance_host -- advance_step with a host SimState: H2D u_curr and "
                         "u_prev from pinned host (u_curr in 8 chunks, each element chunk starting once the node "
                         "prefix it reads has landed; u_prev in 4 tapered chunks gating the node-update chunks), one "
                         "step, D2H the new u_curr chunk by chunk on the other copy direction; the next u_prev "
                         "is the host's previous u_curr; wall clock")} if args.e2e_steps > 0 else None,
        "e2e_run": {"value": E / (run_ms * 1e-3), "unit": UNIT, "steps": K, "ms_per_step": run_ms,
                    "h2d_bytes": 2 * 3 * N * rbytes, "d2h_bytes": 2 * 3 * N * rbytes,
                    "mode": "run_simulation path: djg_set_state (host SimState up once), djg_step(K) on the "
                            "device, djg_get_state (state back); wall clock over the whole call sequence"},
        "roofline": {"bound": "hbm", "kernel": "k_box_step (fused step)" if fused else "k_element",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "moved_frac": (traffic / (k1_ms * 1e-3) / 1e9 / hbm) if traffic else None,
                     "traffic_stale": stale, "source_hash": source_hash(),
                     "issue_active": issue,
                     "note": ("the fused step keeps the element forces on chip: it moves ~0.6 GB per cfg5 step "
                              "against the two-kernel step's 8.2 GB, so HBM is not its bound -- instruction issue "
                              "is (issue_active: ncu smsp__issue_active of the same capture); with engine.lattice = 1 the tets' "
                              "records come from the verified per-class table instead of a per-tet rebuild "
                              "(DESIGN.md §4). " if fused else
                              "moved_frac is the kernel's efficiency: measured DRAM bytes (traffic, ncu, capture "
                              "of the same kernel sources unless traffic_stale) / event-timed launch / peak. ") +
                             "achieved/frac use SURVEY §8(d)'s algorithmic bytes (the reference's hot-field set, "
                             "12-byte force rows); the compact record and the fused step move fewer bytes, so "
                             "frac exceeds 1 and is not an efficiency figure",
                     "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": algo_k1, "launch_ms": k1_ms,
                     "k_node_ms": ms_n / K,
                     "k_node_frac": None if fused else B["k_node"] / (ms_n / K * 1e-3) / 1e9 / hbm,
                     "step_algorithmic_bytes": B["step"], "step_frac": B["step"] / (ms_step * 1e-3) / 1e9 / hbm},
        "ms_per_step_events_per_kernel": ms_tot / K,
        "gpu_launches": (1 if fused else 2) * K,
        "clocks": clk,
        "engine": {k: info[k] for k in ("slabs", "kernels_per_step", "device_bytes", "slot_capacity", "pipelined",
                                        "fused", "lattice")},
    }
    extra["config"] = None
    line = _line(args, 1, K, W, E, ms_step, value, {k: v for k, v in extra.items() if k != "config"})
    if args.sub_configs:
        line["sub_configs"] = {}
        for name in args.sub_configs.split(","):
            try:
                line["sub_configs"][name] = sub_config(name, device)
            except Exception as ex:  # reported, not fatal
                line["sub_configs"][name] = {"error": str(ex)}
    line["config"]["num_nodes"] = N
    line["config"]["l2"] = "inputs larger than L2 (state %.1f GB resident)" % (info["device_bytes"] / 1e9)
    eng.close()
    # The paper's comparison path on the same problem: conventional TLED
    # element forces with the same gather/update (DJG_FLAG_TLED), graph replay.
    if args.tled_steps > 0:
        from paper_2106_14189_b200 import _abi as A

        def replay(flags):
            with GpuDjEngine(sc, device=device, flags=flags) as teng:
                teng.step(W)
                ts = torch.cuda.ExternalStream(teng.stream)
                t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0e.record(ts)
                teng.step_async(args.tled_steps)
                t1e.record(ts)
                t1e.synchronize()
                return t0e.elapsed_time(t1e) / args.tled_steps, teng.sync().status
        tled_ms, tstatus = replay(A.DJG_FLAG_TLED)
        line["tled"] = {"ms_per_step": tled_ms, "value": E / (tled_ms * 1e-3), "unit": UNIT,
                        "dj_over_tled_time": ms_step / tled_ms, "status": tstatus,
                        "note": "paper Table 5 ratio (CPU: 0.70-0.88) on the same problem and the same kernel "
                                "shape: DJ-TLED (this line's step) against conventional TLED (DJG_FLAG_TLED), "
                                "both in the fused box step on the lattice table when the line's step is fused; "
                                "two_kernel: both as element kernel + CSR gather / update kernel"}
        if info.get("fused"):
            dj2_ms, _ = replay(A.DJG_FLAG_NO_FUSED)
            tl2_ms, _ = replay(A.DJG_FLAG_TLED | A.DJG_FLAG_NO_FUSED)
            line["tled"]["two_kernel"] = {"dj_ms": dj2_ms, "tled_ms": tl2_ms, "dj_over_tled_time": dj2_ms / tl2_ms}
    sc.close()
    # SURVEY §8(d)'s secondary precision: the same problem in f64 (graph
    # replay, events on the engine stream; per-kernel split from
    # profile_steps).
    if args.f64_steps > 0 and args.precision == 4:
        spec8 = box_spec(kind=args.kind, model=args.model, divisions=args.divisions, precision=8, target=0.01,
                         ramp_steps=W + 2 * args.f64_steps + 8)
        sc8 = Scenario(spec8)
        with GpuDjEngine(sc8, device=device) as e8:
            e8.step(W)
            me, mn, _ = e8.profile_steps(args.f64_steps)
            s8 = torch.cuda.ExternalStream(e8.stream)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a0.record(s8)
            e8.step_async(args.f64_steps)
            a1.record(s8)
            a1.synchronize()
            r8 = e8.sync()
        sc8.close()
        ms8 = a0.elapsed_time(a1) / args.f64_steps
        line["f64"] = {"ms_per_step": ms8, "value": E / (ms8 * 1e-3), "unit": UNIT, "status": r8.status,
                       "k_element_ms": me / args.f64_steps, "k_node_ms": mn / args.f64_steps,
                       "steps": args.f64_steps, "note": "same mesh and load in double precision (secondary metric)"}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline_line(args)
    print(json.dumps(line), flush=True)


def multi_arm(args, rank, world, device):
    """Strong scaling: the cfg5 mesh partitioned over `world` ranks (RCB),
    halo exchange + failure agreement per step over NCCL."""
    import torch
    import torch.distributed as dist

    from paper_2106_14189_b200 import Scenario, box_spec
    from paper_2106_14189_b200.parallel import DistributedEngine

    dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    K, W = args.steps, max(args.warmup, 3)
    total = W + K + 8
    spec = box_spec(kind=args.kind, model=args.model, divisions=args.divisions, precision=args.precision,
                    target=0.01, ramp_steps=total)
    t0 = time.perf_counter()
    if args.partition == "box":
        # part-local setup: this rank builds only its part from the box spec
        de = DistributedEngine(spec, device=device, method="box-local", transport=args.transport)
    else:
        de = DistributedEngine(Scenario(spec), device=device, method=args.partition, transport=args.transport)
    t1 = time.perf_counter()
    pi = de.part.info
    E = pi["global_elements"]
    setup = torch.tensor([t1 - t0, _peak_rss_gb()], dtype=torch.float64, device="cuda")
    dist.all_reduce(setup, op=dist.ReduceOp.MAX)
    log(f"[bench rank {rank}] local E={pi['num_elements']} owned N={pi['num_owned']} "
        f"neighbors={pi['num_neighbors']} halo send={pi['send_total']} setup {t1 - t0:.1f}s "
        f"peak RSS {_peak_rss_gb():.2f} GB")
    de.step(W)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(device) if rank == 0 else None
    if clocks:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(de.stream)
    de.step_async(K)
    ev1.record(de.stream)
    ev1.synchronize()
    rep = de.eng.sync()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop() if clocks else None
    ms = torch.tensor([ev0.elapsed_time(ev1) / K], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item())
    if rep.status != 0:
        raise SystemExit(f"rank {rank}: timed run failed: {rep}")
    value = E / (ms_step * 1e-3)

    # e2e: the same run loop with a host-resident SimState per rank: every step
    # uploads the rank's u_curr/u_prev (pinned), advances one step (kernels +
    # halo exchange + agreement) and reads the new u_curr back; wall clock,
    # max over ranks.
    import ctypes as C

    from paper_2106_14189_b200 import _abi as A
    lib = A.load_library()
    eng = de.eng
    tdt = torch.float32 if args.precision == 4 else torch.float64
    nloc = 3 * pi["num_nodes"]
    uc, upv, st = eng.get_state()
    bufs = [torch.empty(nloc, dtype=tdt).pin_memory() for _ in range(3)]
    bufs[0].numpy()[:] = uc
    bufs[1].numpy()[:] = upv
    cur, prev, spare = (C.c_void_p(b.data_ptr()) for b in bufs)
    step_c = C.c_int64(st)
    rep_c = A.djg_report()
    torch.cuda.synchronize()
    dist.barrier()
    te0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        lib.djg_set_state(eng._h, cur, prev, step_c.value)
        if lib.djg_step(eng._h, 1, C.byref(rep_c)):
            raise SystemExit(f"rank {rank}: e2e step failed")
        lib.djg_get_state(eng._h, spare, None, C.byref(step_c))
        cur, prev, spare = spare, cur, prev
    e2e_local = (time.perf_counter() - te0) / args.e2e_steps * 1e3
    e2e_t = torch.tensor([e2e_local, float(2 * nloc * args.precision), float(nloc * args.precision)],
                         dtype=torch.float64, device="cuda")
    mx = e2e_t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    tot = e2e_t.clone()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    e2e_ms = float(mx[0].item())

    hbm, peak_kind = peaks()
    B = algo_bytes(args.kind, args.model, pi["num_owned"], pi["num_elements"], args.precision)
    per_step = 2 + (pi["send_total"] > 0) + (pi["recv_total"] > 0) + 2
    if rank == 0:
        extra = {
            "roofline": {"bound": "hbm", "kernel": "step (per GPU)", "achieved": B["step"] / (ms_step * 1e-3) / 1e9,
                         "peak": hbm, "unit": "GB/s", "frac": B["step"] / (ms_step * 1e-3) / 1e9 / hbm,
                         "traffic": None, "peak_source": peak_kind,
                         "note": "rank-0 local elements incl. ghosts / max-over-ranks step time"},
            "e2e": {"value": E / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(tot[1].item()),
                    "d2h_bytes_per_step": int(tot[2].item()), "ms_per_step": e2e_ms,
                    "mode": "per rank and step: djg_set_state (H2D local u_curr+u_prev from pinned host), "
                            "djg_step(1) (kernels, halo exchange, agreement), djg_get_state (D2H the new local "
                            "u_curr); wall clock, max over ranks; bytes summed over ranks"},
            "gpu_launches": K * per_step,
            "gpu_launches_note": "rank 0: element, node, halo pack / unpack, status, agree per step (NCCL kernels "
                                 "not counted)",
            "clocks": clk,
            "partition": {"method": "box (part-local build)" if args.partition == "box" else args.partition,
                          "local_elements": pi["num_elements"], "owned_elements": pi["owned_elements"],
                          "halo_send_nodes": pi["send_total"], "neighbors": pi["num_neighbors"],
                          "setup_s_max_over_ranks": float(setup[0].item()),
                          "host_peak_rss_gb_max_over_ranks": float(setup[1].item())},
        }
        print(json.dumps(_line(args, world, K, W, E, ms_step, value, extra)), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="T4")
    ap.add_argument("--model", default="NH")
    ap.add_argument("--divisions", type=int, default=203)
    ap.add_argument("--precision", type=int, default=4, choices=[4, 8])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--tled-steps", type=int, default=100)
    ap.add_argument("--f64-steps", type=int, default=50, help="also time the f64 problem (0: skip)")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--sub-configs", default="cfg3,cfg4",
                    help="also time these SURVEY configs on one GPU (roofline gate), '' to skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU halo / agreement: peer-memory stores from the node kernel (default) or NCCL")
    ap.add_argument("--partition", default="box", choices=["box", "rcb", "metis"],
                    help="multi-GPU partition: blocks of the box's cell grid, each rank building only its part "
                         "(default), or -- from the global problem -- coordinate bisection / METIS k-way")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()
