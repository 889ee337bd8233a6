"""TEST INFRASTRUCTURE ONLY — CPU checkers for the DJ-TLED hot path.

Two libraries, both built by oracle/Makefile:
  * `oracle`  (_build/libdjoracle.so): the plain-C restatement of the
    reference algorithm (djo_impl.h), always available;
  * `ref`     (_ref/libdjref.so): the unmodified reference headers behind a
    thin C-ABI (ref_driver.cpp); built only where /root/reference exists,
    shipped prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and its
--impl reference arm) may import this package. The product never does.
Parity pinned: tests/test_oracle.py checks `oracle` against `ref` bit for bit
and against the committed fixtures in tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_2106_14189_b200 import _abi as A
from paper_2106_14189_b200.spec import Spec

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "_build" / "libdjoracle.so"
REF_LIB = HERE / "_ref" / "libdjref.so"

_libs: dict[str, C.CDLL] = {}


def build(quiet=True) -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def have(which: str) -> bool:
    return (ORACLE_LIB if which == "oracle" else REF_LIB).exists()


def lib(which: str = "oracle") -> C.CDLL:
    if which in _libs:
        return _libs[which]
    path = ORACLE_LIB if which == "oracle" else REF_LIB
    if not path.exists():
        raise RuntimeError(f"{which} library missing at {path}; run `make -C oracle`")
    L = C.CDLL(str(path))
    P = C.POINTER
    if which == "oracle":
        L.djo_image.argtypes = [P(A.djg_scenario_spec), C.c_int32, P(A.djg_image_ptrs), P(A.djg_image_scalars)]
        L.djo_run.argtypes = [P(A.djg_scenario_spec), C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, P(A.djg_report)]
        L.djo_assemble.argtypes = [P(A.djg_scenario_spec), C.c_int32, C.c_void_p, C.c_void_p,
                                   P(A.djg_assemble_stats)]
        L.djo_element_force_rec.argtypes = [C.c_int32, C.c_int32, P(A.djg_material_params), C.c_void_p,
                                            C.c_void_p, C.c_void_p]
        L.djo_element_record.argtypes = [C.c_int32, C.c_int32, P(A.djg_material_params), C.c_double,
                                         P(C.c_double), C.c_void_p]
        L.djo_libm_cbrt.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64]
        L.djo_restated_cbrt.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64]
    else:
        L.djref_image.argtypes = [P(A.djg_scenario_spec), P(A.djg_image_ptrs), P(A.djg_image_scalars)]
        L.djref_run.argtypes = [P(A.djg_scenario_spec), C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, P(A.djg_report), P(C.c_double)]
        L.djref_assemble.argtypes = [P(A.djg_scenario_spec), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                     P(A.djg_assemble_stats)]
        L.djref_element_force.argtypes = [C.c_int32, C.c_int32, P(A.djg_material_params), C.c_double,
                                          P(C.c_double), P(C.c_double), P(C.c_double), C.c_int32]
        L.djref_time_steps.argtypes = [P(A.djg_scenario_spec), C.c_int64, C.c_int64, C.c_int32, C.c_int32]
        L.djref_time_steps.restype = C.c_double
        L.djref_time_protocol.argtypes = [P(A.djg_scenario_spec), C.c_int32, C.c_int32, C.c_int32, P(C.c_int32),
                                          P(C.c_int64), P(C.c_int64), P(C.c_double), P(C.c_double)]
        L.djref_error.restype = C.c_char_p
    _libs[which] = L
    return L


def _empty_image(spec: Spec, n: int, e: int, nconst: int) -> dict:
    dt = spec.dtype
    npe = spec.npe
    return {
        "nodes": np.zeros(3 * n, dt), "conn": np.zeros(npe * e, np.int32),
        "csr_offsets": np.zeros(n + 1, np.int64), "csr_elem": np.zeros(npe * e, np.int64),
        "csr_local": np.zeros(npe * e, np.int32), "consts": np.zeros(e * nconst, dt),
        "mass": np.zeros(n, dt), "c1": np.zeros(n, dt), "massless": np.zeros(n, np.uint8),
        "dof_kind": np.zeros(3 * n, np.uint8), "dof_target": np.zeros(3 * n, dt),
        "dof_t_total": np.zeros(3 * n, dt),
    }


def _ptrs(img: dict) -> A.djg_image_ptrs:
    p = A.djg_image_ptrs()
    for k, v in img.items():
        setattr(p, k, v.ctypes.data_as(C.c_void_p))
    return p


def scalars_dict(sc: A.djg_image_scalars) -> dict:
    return {name: getattr(sc, name) for name, _ in sc._fields_}


def image(spec: Spec, which="oracle", threads=0) -> tuple[dict, dict]:
    """Fully built problem arrays + scalars from the oracle or the reference."""
    L = lib(which)
    sc = A.djg_image_scalars()
    if which == "oracle":
        rc = L.djo_image(spec.ref(), threads, None, C.byref(sc))
    else:
        rc = L.djref_image(spec.ref(), None, C.byref(sc))
    if rc:
        raise RuntimeError(f"{which} image failed rc={rc}")
    nconst = A.const_count(spec.c.kind, spec.c.material.model)
    img = _empty_image(spec, sc.num_nodes, sc.num_elements, nconst)
    p = _ptrs(img)
    if which == "oracle":
        rc = L.djo_image(spec.ref(), threads, C.byref(p), C.byref(sc))
    else:
        rc = L.djref_image(spec.ref(), C.byref(p), C.byref(sc))
    if rc:
        raise RuntimeError(f"{which} image failed rc={rc}")
    return img, scalars_dict(sc)


def run(spec: Spec, steps: int, which="oracle", threads=0, u0=None, up0=None, r_ext=None, engine=0):
    """steps x advance_step from rest (or u0/up0). Returns (u_curr, u_prev, report)."""
    L = lib(which)
    sc = A.djg_image_scalars()
    if which == "oracle":
        L.djo_image(spec.ref(), threads, None, C.byref(sc))
    else:
        L.djref_image(spec.ref(), None, C.byref(sc))
    n = sc.num_nodes
    u = np.zeros(3 * n, spec.dtype)
    up = np.zeros(3 * n, spec.dtype)
    rep = A.djg_report()
    conv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=spec.dtype)
    u0, up0, r_ext = conv(u0), conv(up0), conv(r_ext)
    if which == "oracle":
        assert engine == 0, "the C oracle restates the DJ-TLED path only"
        L.djo_run(spec.ref(), steps, threads, A.ptr(u0), A.ptr(up0), A.ptr(r_ext), A.ptr(u), A.ptr(up), C.byref(rep))
    else:
        assert r_ext is None
        secs = C.c_double()
        L.djref_run(spec.ref(), steps, threads, engine, A.ptr(u0), A.ptr(up0), A.ptr(u), A.ptr(up), C.byref(rep),
                    C.byref(secs))
    return u, up, rep.as_dict()


def assemble(spec: Spec, u: np.ndarray, which="oracle", threads=0, engine=0):
    L = lib(which)
    u = np.ascontiguousarray(u, dtype=spec.dtype)
    f = np.zeros_like(u)
    st = A.djg_assemble_stats()
    if which == "oracle":
        L.djo_assemble(spec.ref(), threads, A.ptr(u), A.ptr(f), C.byref(st))
    else:
        L.djref_assemble(spec.ref(), threads, engine, A.ptr(u), A.ptr(f), C.byref(st))
    return f, {"first_inverted": st.first_inverted, "inverted_count": st.inverted_count}


def element_record(precision, kind, mat, coords, c_hg=0.1):
    npe = A.npe_of(kind)
    dt = np.float32 if precision == 4 else np.float64
    rec = np.zeros(A.const_count(kind, mat.model), dt)
    x = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1)
    rc = lib("oracle").djo_element_record(precision, kind, C.byref(mat), c_hg, A.typed_ptr(x, C.c_double),
                                          A.ptr(rec))
    if rc:
        raise ValueError("degenerate element")
    return rec


def element_force_rec(precision, kind, mat, rec, u):
    npe = A.npe_of(kind)
    dt = np.float32 if precision == 4 else np.float64
    u = np.ascontiguousarray(u, dtype=dt).reshape(-1)
    f = np.zeros(3 * npe, dt)
    rc = lib("oracle").djo_element_force_rec(precision, kind, C.byref(mat), A.ptr(np.ascontiguousarray(rec, dt)),
                                             A.ptr(u), A.ptr(f))
    return (f if rc == 0 else None)


def ref_element_force(precision, kind, mat, coords, u, c_hg=0.1, engine=0):
    npe = A.npe_of(kind)
    x = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1)
    uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    f = np.zeros(3 * npe, np.float64)
    rc = lib("ref").djref_element_force(precision, kind, C.byref(mat), c_hg, A.typed_ptr(x, C.c_double),
                                        A.typed_ptr(uu, C.c_double), A.typed_ptr(f, C.c_double), engine)
    return f if rc == 0 else None


def ref_time_steps(spec: Spec, warmup: int, steps: int, threads: int = 0, engine: int = 0) -> float:
    """Mean seconds per step of the reference's own advance_step loop."""
    r = lib("ref").djref_time_steps(spec.ref(), warmup, steps, threads, engine)
    if r < 0:
        raise RuntimeError(lib("ref").djref_error().decode())
    return r


def ref_time_protocol(spec: Spec, engine: int, build_threads: int, runs) -> tuple[list[float], float]:
    """One reference problem built with `build_threads` (engine 0 DjEngine,
    2 TledEngine), then for each (threads, warmup, steps) in `runs` the
    advance_step loop from rest: mean seconds per timed step, and the build
    time in seconds."""
    n = len(runs)
    th = (C.c_int32 * n)(*[r[0] for r in runs])
    wu = (C.c_int64 * n)(*[r[1] for r in runs])
    st = (C.c_int64 * n)(*[r[2] for r in runs])
    secs = (C.c_double * n)()
    b = C.c_double()
    rc = lib("ref").djref_time_protocol(spec.ref(), engine, build_threads, n, th, wu, st, secs, C.byref(b))
    if rc:
        raise RuntimeError(lib("ref").djref_error().decode())
    return list(secs), b.value


def rel_max_err(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / max|b| (SURVEY §8(c) parity metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b), initial=0.0))
