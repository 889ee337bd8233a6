"""Problem specifications (djg_scenario_spec) built from Python.

Mirrors the inputs the reference's CLI and bench hand to the solver:
`bench_material` (bench.hpp:12-25), `generate_box` (mesh.hpp:208-264), the
zmin-fixed / zmax-ramped loading of bench::detail::time_steps
(bench.hpp:52-72) and of SURVEY §8(d), dt = safety * critical_dt and
alpha = relaxation_alpha (solver.hpp:330-339).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi as A

# SURVEY §8(d) configurations (BASELINE.json configs[0..4]).
CONFIGS = {
    "cfg1": dict(kind="T4", model="NH", divisions=12, steps=2000),
    "cfg2": dict(kind="H8", model="NH", divisions=22, steps=2000),
    "cfg3": dict(kind="T4", model="NH", divisions=70, steps=1100),
    "cfg4": dict(kind="H8", model="TI", divisions=100, steps=1100),
    "cfg5": dict(kind="T4", model="NH", divisions=203, steps=550),
}


def bench_material(model: int | str) -> A.djg_material_params:
    """bench_material (bench.hpp:12-25); I57 (the fifth/seventh-invariant
    energy of test_forces.cpp:248-271, no bench counterpart): eta5 = 1.6 mu,
    eta7 = 1.3 mu (the test's 800 / 650 over mu = 500), oblique fibres."""
    if isinstance(model, str):
        model = A.MODEL_NAMES[model]
    m = A.djg_material_params()
    m.model = model
    m.mu, m.kappa, m.rho = 6567.0, 326210.0, 1060.0
    m.fibre_a[0] = 1.0
    m.fibre_b[1] = 1.0
    if model in (A.DJG_TI, A.DJG_OT):
        m.eta_a = 2 * 6567.0
    if model == A.DJG_OT:
        m.eta_b = 2 * 6567.0
    if model == A.DJG_MR:
        m.mu = 0.0
        m.c10, m.c01 = 6567.0 / 2, 3000.0
    if model == A.DJG_I57:
        m.eta_a, m.eta_b = 1.6 * 6567.0, 1.3 * 6567.0
        m.fibre_a[1] = 1.0
        m.fibre_b[2] = 1.0
    return m


def material(model: str | int, mu=0.0, kappa=0.0, rho=0.0, eta_a=0.0, eta_b=0.0, c10=0.0, c01=0.0,
             fibre_a=(1.0, 0.0, 0.0), fibre_b=(0.0, 1.0, 0.0)) -> A.djg_material_params:
    m = A.djg_material_params()
    m.model = A.MODEL_NAMES[model] if isinstance(model, str) else model
    m.mu, m.kappa, m.rho, m.eta_a, m.eta_b, m.c10, m.c01 = mu, kappa, rho, eta_a, eta_b, c10, c01
    for i in range(3):
        m.fibre_a[i] = fibre_a[i]
        m.fibre_b[i] = fibre_b[i]
    return m


@dataclass
class Spec:
    """A djg_scenario_spec plus the numpy arrays its pointers alias."""
    c: A.djg_scenario_spec
    keep: list = field(default_factory=list)

    @property
    def precision(self) -> int:
        return self.c.precision

    @property
    def dtype(self):
        return np.float32 if self.c.precision == 4 else np.float64

    @property
    def npe(self) -> int:
        return A.npe_of(self.c.kind)

    def ref(self):
        return C.byref(self.c)


def _kind(kind) -> int:
    return A.KIND_NAMES[kind] if isinstance(kind, str) else int(kind)


def box_spec(kind="T4", model="NH", divisions=12, precision=4, ramp_steps=2000, target=-0.2, safety=0.5,
             extent=(1.0, 1.0, 1.0), fix_all_axes=True, alpha=None, dt=None, policy=A.DJG_ABORT,
             mat: A.djg_material_params | None = None, c_hg=0.1) -> Spec:
    """Unit-cube problem of SURVEY §8(d): zmin fixed, zmax ramped along z."""
    s = A.djg_scenario_spec()
    s.precision = precision
    s.kind = _kind(kind)
    divs = divisions if isinstance(divisions, (tuple, list)) else (divisions,) * 3
    for i in range(3):
        s.divisions[i] = int(divs[i])
        s.extent[i] = float(extent[i])
    s.material = mat if mat is not None else bench_material(model)
    s.c_hg = c_hg
    s.bc_mode = 1
    s.fix_all_axes = 1 if fix_all_axes else 0
    s.target = target
    s.ramp_steps = ramp_steps
    s.safety = safety
    s.dt = 0.0 if dt is None else float(dt)
    s.alpha_mode = 0 if alpha is None else 1
    s.alpha = 0.0 if alpha is None else float(alpha)
    s.policy = policy
    return Spec(s)


def mesh_spec(nodes: np.ndarray, conn: np.ndarray, kind="T4", model="NH", precision=4,
              mat: A.djg_material_params | None = None, fixed=(), prescribed=(), dt=None, safety=0.5,
              alpha=None, policy=A.DJG_ABORT, c_hg=0.1) -> Spec:
    """Caller mesh with explicit BCs: fixed = [(node, axis)], prescribed =
    [(node, axis, target, t_total)] (BoundaryConditions, mesh.hpp:41-71)."""
    s = A.djg_scenario_spec()
    s.precision = precision
    s.kind = _kind(kind)
    nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1)
    conn = np.ascontiguousarray(conn, dtype=np.int32).reshape(-1)
    keep = [nodes, conn]
    s.num_nodes = nodes.size // 3
    s.num_elements = conn.size // A.npe_of(s.kind)
    s.nodes = A.typed_ptr(nodes, C.c_double)
    s.conn = A.typed_ptr(conn, C.c_int32)
    s.material = mat if mat is not None else bench_material(model)
    s.c_hg = c_hg
    s.bc_mode = 2
    fx = np.array([f[0] for f in fixed], dtype=np.int32)
    fa = np.array([f[1] for f in fixed], dtype=np.int32)
    pn = np.array([p[0] for p in prescribed], dtype=np.int32)
    pa = np.array([p[1] for p in prescribed], dtype=np.int32)
    pt = np.array([p[2] for p in prescribed], dtype=np.float64)
    pT = np.array([p[3] for p in prescribed], dtype=np.float64)
    keep += [fx, fa, pn, pa, pt, pT]
    s.n_fixed = fx.size
    s.fixed_node = A.typed_ptr(fx, C.c_int32) if fx.size else None
    s.fixed_axis = A.typed_ptr(fa, C.c_int32) if fx.size else None
    s.n_prescribed = pn.size
    if pn.size:
        s.presc_node = A.typed_ptr(pn, C.c_int32)
        s.presc_axis = A.typed_ptr(pa, C.c_int32)
        s.presc_target = A.typed_ptr(pt, C.c_double)
        s.presc_t_total = A.typed_ptr(pT, C.c_double)
    s.safety = safety
    s.dt = 0.0 if dt is None else float(dt)
    s.alpha_mode = 0 if alpha is None else 1
    s.alpha = 0.0 if alpha is None else float(alpha)
    s.policy = policy
    return Spec(s, keep)


def config_spec(name: str, precision=4, ramp_steps=None, **kw) -> Spec:
    """Spec of a SURVEY §8(d) configuration (cfg1..cfg5)."""
    c = CONFIGS[name]
    return box_spec(kind=c["kind"], model=c["model"], divisions=c["divisions"], precision=precision,
                    ramp_steps=c["steps"] if ramp_steps is None else ramp_steps, **kw)


def box_counts(kind, divisions) -> tuple[int, int]:
    d = divisions if isinstance(divisions, (tuple, list)) else (divisions,) * 3
    n = (d[0] + 1) * (d[1] + 1) * (d[2] + 1)
    e = d[0] * d[1] * d[2] * (6 if _kind(kind) == A.DJG_T4 else 1)
    return n, e
