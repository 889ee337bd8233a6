"""Python mirror of the reference's solver interface over libdjg's C-ABI.

Names, argument meaning and error behaviour follow the reference
(solver.hpp / djtled_force.hpp / core.hpp) so tests read like its own:

  Scenario            DjModel::build + lump_mass + DofConstraints +
                      UpdateCoeffs + critical_dt + relaxation_alpha inputs
                      (native C++ builder, include/djg_host.h)
  GpuDjEngine         DjEngine (solver.hpp:261-284) with the state resident
                      on the B200: assemble() is Engine::assemble,
                      advance_step()/step() are advance_step, run_simulation()
                      is run_simulation (solver.hpp:98-258)
  SimulationError     core.hpp:44-57 (kind ElementInversion / Divergence,
                      index = element id / failing step)

Every call goes to the CUDA engine; a missing library raises (no fallback).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _abi as A
from .spec import Spec


class ConfigError(ValueError):
    """ConfigError / MeshError (core.hpp:28-42)."""


class CudaError(RuntimeError):
    pass


class SimulationError(RuntimeError):
    """SimulationError (core.hpp:44-57)."""
    ElementInversion = "ElementInversion"
    Divergence = "Divergence"

    def __init__(self, kind: str, message: str, index: int):
        super().__init__(message)
        self.kind = kind
        self.index = index


def _lib():
    return A.load_library()


class Scenario:
    """A fully prepared problem (host side, native C++ builder)."""

    def __init__(self, spec: Spec, threads: int = 0):
        self.spec = spec
        h = C.c_void_p()
        rc = _lib().djg_scenario_build(spec.ref(), threads, C.byref(h))
        if rc != A.DJG_OK:
            raise ConfigError(_lib().djg_scenario_error().decode())
        self._h = h
        sc = A.djg_image_scalars()
        _lib().djg_scenario_scalars(self._h, C.byref(sc))
        self.scalars = {name: getattr(sc, name) for name, _ in sc._fields_}
        self.num_nodes = sc.num_nodes
        self.num_elements = sc.num_elements
        self.npe = sc.npe
        self.nconst = sc.nconst
        self.dt = sc.dt

    @property
    def dtype(self):
        return self.spec.dtype

    def image(self) -> dict:
        n, e, npe, nc, dt = self.num_nodes, self.num_elements, self.npe, self.nconst, self.dtype
        img = {
            "nodes": np.zeros(3 * n, dt), "conn": np.zeros(npe * e, np.int32),
            "csr_offsets": np.zeros(n + 1, np.int64), "csr_elem": np.zeros(npe * e, np.int64),
            "csr_local": np.zeros(npe * e, np.int32), "consts": np.zeros(e * nc, dt),
            "mass": np.zeros(n, dt), "c1": np.zeros(n, dt), "massless": np.zeros(n, np.uint8),
            "dof_kind": np.zeros(3 * n, np.uint8), "dof_target": np.zeros(3 * n, dt),
            "dof_t_total": np.zeros(3 * n, dt),
        }
        p = A.djg_image_ptrs()
        for k, v in img.items():
            setattr(p, k, v.ctypes.data_as(C.c_void_p))
        _lib().djg_scenario_image(self._h, C.byref(p))
        return img

    def desc(self, device: int = 0, flags: int = 0) -> A.djg_desc:
        d = A.djg_desc()
        _lib().djg_scenario_desc(self._h, device, C.byref(d))
        d.flags = flags
        return d

    def close(self):
        if getattr(self, "_h", None):
            _lib().djg_scenario_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class StepReport:
    steps_done: int
    step: int
    first_inverted: int
    inverted_count: int
    inverted_steps: int
    fail_step: int
    diverged: bool
    status: int

    @classmethod
    def from_c(cls, r: A.djg_report) -> "StepReport":
        return cls(r.steps_done, r.step, r.first_inverted, r.inverted_count, r.inverted_steps, r.fail_step,
                   bool(r.diverged), r.status)


class GpuDjEngine:
    """DjEngine on the B200 with the simulation state resident in HBM."""

    def __init__(self, scenario: Scenario, device: int = 0, flags: int = 0, device_csr: bool = False):
        """device_csr: build the node adjacency / slot layout on the GPU
        (with DJG_FLAG_DEVICE_PRECOMPUTE) instead of passing the host CSR."""
        self.scenario = scenario
        self.dtype = scenario.dtype
        self.num_nodes = scenario.num_nodes
        self.num_elements = scenario.num_elements
        h = C.c_void_p()
        d = scenario.desc(device, flags)
        if device_csr:
            d.csr_offsets = d.csr_elem = d.csr_local = None
        rc = _lib().djg_create(C.byref(d), C.byref(h))
        if rc != A.DJG_OK:
            msg = _lib().djg_create_error().decode()
            raise (CudaError if rc == A.DJG_E_CUDA else ConfigError)(msg)
        self._h = h

    # -- plumbing
    def _check(self, rc: int):
        if rc in (A.DJG_OK, A.DJG_E_INVERSION, A.DJG_E_DIVERGENCE, A.DJG_E_PEER):
            return rc
        msg = _lib().djg_last_error(self._h).decode()
        raise (CudaError if rc == A.DJG_E_CUDA else ConfigError)(msg)

    def _vec(self, a):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=self.dtype).reshape(-1)
        if a.size != 3 * self.num_nodes:
            raise ConfigError(f"expected {3 * self.num_nodes} DOFs, got {a.size}")
        return a

    def close(self):
        if getattr(self, "_h", None):
            _lib().djg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- SimState
    def set_state(self, u_curr=None, u_prev=None, step: int = 0):
        u, up = self._vec(u_curr), self._vec(u_prev)
        self._check(_lib().djg_set_state(self._h, A.ptr(u), A.ptr(up), step))

    def set_external(self, r_ext=None):
        self._check(_lib().djg_set_external(self._h, A.ptr(self._vec(r_ext))))

    def get_state(self):
        u = np.empty(3 * self.num_nodes, self.dtype)
        up = np.empty(3 * self.num_nodes, self.dtype)
        st = C.c_int64()
        self._check(_lib().djg_get_state(self._h, A.ptr(u), A.ptr(up), C.byref(st)))
        return u, up, st.value

    @property
    def u_curr(self):
        return self.get_state()[0]

    # -- Engine::assemble (solver.hpp:269-272)
    def assemble(self, u=None, threads: int = 0, policy=None):
        """Internal forces at u (default: the current state). Returns
        (f or None, {"first_inverted", "inverted_count"}) like AssembleStats;
        under Abort with an inversion f is None (the reference does not gather)."""
        del threads, policy  # the reference's OpenMP knob; policy is fixed at construction
        uu = self._vec(u)
        f = np.zeros(3 * self.num_nodes, self.dtype)
        st = A.djg_assemble_stats()
        rc = self._check(_lib().djg_assemble(self._h, A.ptr(uu), A.ptr(f), C.byref(st)))
        stats = {"first_inverted": st.first_inverted, "inverted_count": st.inverted_count}
        return (None if rc == A.DJG_E_INVERSION else f), stats

    # -- advance_step / run loop
    def step(self, nsteps: int = 1, raise_on_failure: bool = True) -> StepReport:
        rep = A.djg_report()
        rc = self._check(_lib().djg_step(self._h, nsteps, C.byref(rep)))
        r = StepReport.from_c(rep)
        if raise_on_failure and rc != A.DJG_OK:
            raise_for(r)
        return r

    def advance_host(self, u_curr, u_prev, step: int, out=None):
        """advance_step with a host SimState (djg_advance_host): one step from
        (u_curr, u_prev, step); returns (new u_curr, StepReport)."""
        u, up = self._vec(u_curr), self._vec(u_prev)
        if out is None:
            out = np.empty(3 * self.num_nodes, self.dtype)
        elif not (isinstance(out, np.ndarray) and out.dtype == self.dtype and out.size == 3 * self.num_nodes
                  and out.flags["C_CONTIGUOUS"] and out.flags["WRITEABLE"]):
            # the library writes 3N Reals through this pointer
            raise ConfigError(f"out must be a writeable C-contiguous {np.dtype(self.dtype).name} array of "
                              f"{3 * self.num_nodes} DOFs")
        rep = A.djg_report()
        self._check(_lib().djg_advance_host(self._h, A.ptr(u), A.ptr(up), step, A.ptr(out), C.byref(rep)))
        return out, StepReport.from_c(rep)

    def step_async(self, nsteps: int):
        self._check(_lib().djg_step_async(self._h, nsteps))

    def sync(self) -> StepReport:
        rep = A.djg_report()
        self._check(_lib().djg_sync(self._h, C.byref(rep)))
        return StepReport.from_c(rep)

    def profile_steps(self, nsteps: int):
        """(ms in k_element, ms in k_node, ms total) over nsteps, CUDA events."""
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        self._check(_lib().djg_profile_steps(self._h, nsteps, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def stream(self) -> int:
        return int(_lib().djg_stream(self._h) or 0)

    def info(self) -> dict:
        i = A.djg_engine_info()
        self._check(_lib().djg_get_info(self._h, C.byref(i)))
        return {name: getattr(i, name) for name, _ in i._fields_}

    def device_consts(self) -> np.ndarray:
        """The per-element record held on the device (E x n)."""
        n = int(_lib().djg_get_consts(self._h, None))
        out = np.zeros((self.num_elements, n), self.dtype)
        _lib().djg_get_consts(self._h, A.ptr(out))
        return out

    def lump_mass(self) -> np.ndarray:
        """lump_mass on the device (engines built with device_csr)."""
        out = np.zeros(self.num_nodes, self.dtype)
        self._check(_lib().djg_lump_mass(self._h, A.ptr(out)))
        return out

    def min_char_length(self) -> float:
        v = C.c_double()
        self._check(_lib().djg_min_char_length(self._h, C.byref(v)))
        return v.value

    def slot_map(self) -> np.ndarray:
        out = np.zeros(self.scenario.npe * self.num_elements, np.int32)
        self._check(_lib().djg_get_slot_map(self._h, A.ptr(out)))
        return out


def raise_for(r: StepReport):
    """run_simulation's failure mapping (solver.hpp:229-239)."""
    if r.status == A.DJG_E_DIVERGENCE:
        raise SimulationError(SimulationError.Divergence,
                              f"solution diverged at step {r.fail_step}; reduce the time step", r.fail_step)
    if r.status == A.DJG_E_INVERSION:
        raise SimulationError(SimulationError.ElementInversion,
                              f"element {r.first_inverted} inverted at step {r.fail_step}", r.first_inverted)
    if r.status == A.DJG_E_PEER:
        raise CudaError(f"peer-memory step {r.fail_step}: a part did not post its step within the wait limit")


@dataclass
class RunResult:
    u_curr: np.ndarray
    u_prev: np.ndarray
    steps: int
    wall_seconds: float
    mean_step_seconds: float
    inverted_steps: int


def run_simulation(engine: GpuDjEngine, t_end: float | None = None, num_steps: int | None = None,
                   initial=None) -> RunResult:
    """run_simulation (solver.hpp:205-258): from rest (or `initial` =
    (u_curr, u_prev)) for ceil(t_end/dt - 1e-9) steps, or an explicit
    num_steps. Raises SimulationError on inversion (Abort) or divergence."""
    if num_steps is None:
        if t_end is None or t_end < 0:
            raise ConfigError("t_end must be >= 0")
        num_steps = int(np.ceil(float(t_end) / float(engine.scenario.dt) - 1e-9))
    if initial is not None:
        engine.set_state(initial[0], initial[1], 0)
    else:
        engine.set_state(None, None, 0)
    t0 = time.perf_counter()
    r = engine.step(num_steps, raise_on_failure=True)
    wall = time.perf_counter() - t0
    u, up, step = engine.get_state()
    return RunResult(u, up, step, wall, wall / num_steps if num_steps else 0.0, r.inverted_steps)
