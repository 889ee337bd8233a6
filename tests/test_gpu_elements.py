"""Element-level GPU parity on the reference's own random states.

`tests/golden/elements.npz` holds 40 random element states per kind (the
generators of the reference tests, oracles.hpp:126-157 / test_forces.cpp:
161-182) with the forces the UNMODIFIED reference computes for them
(`element_force` + `hourglass_force`, djtled_force.hpp:36-95; TLED:
tled_force.hpp), made by tests/golden/make_golden.py. Here every state runs
through the CUDA element kernels: the 40 elements of a kind become one mesh
of disjoint elements (element i owns nodes npe*i .. npe*i+npe-1), so the
engine's assembled internal force at a node is exactly that element's force
row (+0 + row in the CSR gather). The gate is bitwise equality, for every
kind x material x precision and every element-kernel form (pipelined with
the compact record, full record, one-shot, device precompute, node windows,
TLED).

Near-inversion states (det tJ -> 0+) and cube-root edge cases (J at and
around powers of two and 1) are generated here and checked against the
reference (oracle/_ref) where it is built, else against the C oracle.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2106_14189_b200 import GpuDjEngine, Scenario, material
from paper_2106_14189_b200 import _abi as A
from paper_2106_14189_b200.spec import bench_material, mesh_spec

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
KINDS = {"T4": A.DJG_T4, "H8": A.DJG_H8}
I57_TEST = material("I57", mu=500.0, kappa=2000.0, rho=1000.0, eta_a=800.0, eta_b=650.0,
                    fibre_a=(0.3, -0.5, 0.81), fibre_b=(-0.62, 0.1, 0.4))
FORMS = {"default": 0, "full": A.DJG_FLAG_FULL_RECORD, "nopipe": A.DJG_FLAG_NO_PIPE,
         "device": A.DJG_FLAG_DEVICE_PRECOMPUTE, "window": A.DJG_FLAG_WINDOW}


def element_mesh(X, kind, mat, prec, policy=A.DJG_ABORT):
    """Disjoint elements: coordinates X[i] (npe x 3) for element i."""
    n, npe = X.shape[0], X.shape[1]
    nodes = X.reshape(-1, 3)
    conn = np.arange(n * npe, dtype=np.int32).reshape(n, npe)
    # one fixed DOF keeps the scenario builder's BC tables non-empty; the
    # assembled forces do not depend on BCs
    return mesh_spec(nodes, conn, kind=kind, precision=prec, mat=mat, fixed=[(0, 0)], dt=1e-6, alpha=0.0,
                     policy=policy)


def gpu_forces(X, U, kind, mat, prec, flags=0, policy=A.DJG_ABORT):
    spec = element_mesh(X, kind, mat, prec, policy)
    dt = np.float32 if prec == 4 else np.float64
    with GpuDjEngine(Scenario(spec), flags=flags) as eng:
        f, st = eng.assemble(U.reshape(-1).astype(dt))
        info = eng.info()
    return f, st, info


def same(a, b):
    """Bitwise up to the sign of zero (== semantics)."""
    return a.shape == b.shape and bool(np.all(a == b))


@pytest.mark.parametrize("form", list(FORMS))
@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_golden_states_bitwise(kind, model, prec, form):
    g = np.load(GOLDEN / "elements.npz")
    X, U, F = g[f"{kind}_coords"], g[f"{kind}_u"], g[f"{kind}_{model}_f{8 * prec}"]
    f, st, info = gpu_forces(X, U, kind, bench_material(model), prec, FORMS[form])
    assert st["inverted_count"] == 0 and f is not None
    if form == "window" and info["pipelined"] and kind == "T4":
        assert info["windowed"] == 1
    got = f.astype(np.float64).reshape(F.shape)
    bad = [i for i in range(len(F)) if not same(got[i], F[i])]
    assert not bad, f"{len(bad)} of {len(F)} elements differ, first {bad[0]}: {got[bad[0]]} vs {F[bad[0]]}"


@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("name", ["I57", "I57x"])
@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_golden_states_i57(kind, name, prec):
    """The I5 / I7 force terms (djtled_force.hpp:58-65) on the device, against
    the reference's element_force with the test energy of test_forces.cpp:248-271."""
    g = np.load(GOLDEN / "elements.npz")
    X, U, F = g[f"{kind}_coords"], g[f"{kind}_u"], g[f"{kind}_{name}_f{8 * prec}"]
    m = bench_material("I57") if name == "I57" else I57_TEST
    f, st, _ = gpu_forces(X, U, kind, m, prec)
    assert same(f.astype(np.float64).reshape(F.shape), F)


@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_golden_states_tled(kind, model):
    """The device TLED element kernel against the reference TledEngine's
    element forces (tled_force.hpp) on the same 40 states (f64 fixtures)."""
    g = np.load(GOLDEN / "elements.npz")
    X, U, F = g[f"{kind}_coords"], g[f"{kind}_u"], g[f"{kind}_{model}_tled_f64"]
    f, st, _ = gpu_forces(X, U, kind, bench_material(model), 8, A.DJG_FLAG_TLED)
    assert same(f.reshape(F.shape), F)


def _base(kind):
    if kind == "T4":
        return np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    return np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                     [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)


def _edge_states(kind):
    """Elements deformed by F = [[1, s, 0], [0, 1, 0], [0, 0, lam]] (J = lam):
    near-inversion (lam -> 0+), cube-root edge cases (lam at / next to 1 and
    powers of two), and a slightly rotated copy of each."""
    lams = [0.5, 1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 3e-7, 1.0, 1 + 2.0 ** -23, 1 - 2.0 ** -24, 1 + 2.0 ** -52,
            2.0, 4.0, 8.0, 0.25, 0.125, 1.5, 3.0, 0.7937005259840998]
    X0 = _base(kind) * 0.37 + 0.11
    th = 0.3
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
    X, U = [], []
    for lam in lams:
        for s in (0.0, 0.2):
            for rot in (False, True):
                Fm = np.array([[1, s, 0], [0, 1, 0], [0, 0, lam]])
                if rot:
                    Fm = R @ Fm
                X.append(X0)
                U.append(X0 @ (Fm - np.eye(3)).T)
    return np.array(X), np.array(U)


@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("model", ["NH", "TI"])
@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_near_inversion_and_cbrt_edges(kind, model, prec):
    X, U = _edge_states(kind)
    m = bench_material(model)
    which = "ref" if oracle.have("ref") else "oracle"
    want, ok = [], []
    for i in range(len(X)):
        if which == "ref":
            # the reference converts its double inputs to Real itself
            u = U[i].astype(np.float32 if prec == 4 else np.float64).astype(np.float64)
            r = oracle.ref_element_force(prec, KINDS[kind], m, X[i], u)
        else:
            rec = oracle.element_record(prec, KINDS[kind], m, X[i])
            r = oracle.element_force_rec(prec, KINDS[kind], m, rec, U[i].astype(np.float32 if prec == 4 else np.float64))
        ok.append(r is not None)
        want.append(np.zeros(3 * len(X[i])) if r is None else np.asarray(r, np.float64).reshape(-1))
    for form in ("default", "nopipe"):
        f, st, _ = gpu_forces(X, U, kind, m, prec, FORMS[form], policy=A.DJG_SKIP_AND_REPORT)
        assert st["inverted_count"] == ok.count(False)
        got = f.astype(np.float64).reshape(len(X), -1)
        bad = [i for i in range(len(X)) if not same(got[i], want[i])]
        assert not bad, (form, which, bad[:5])


def test_inverted_element_reported_like_the_reference():
    """An element pushed through zero volume: the device reports it (Abort:
    lowest inverted element id, no gather), as the reference's assemble does."""
    X, U = _edge_states("T4")
    lam_neg = np.array([[1, 0, 0], [0, 1, 0], [0, 0, -1e-3]])
    U = U.copy()
    U[7] = X[7] @ (lam_neg - np.eye(3)).T
    U[23] = X[23] @ (lam_neg - np.eye(3)).T
    f, st, _ = gpu_forces(X, U, "T4", bench_material("NH"), 4)
    assert f is None and st["first_inverted"] == 7
    f, st, _ = gpu_forces(X, U, "T4", bench_material("NH"), 4, policy=A.DJG_SKIP_AND_REPORT)
    assert f is not None and st["inverted_count"] == 2
    assert not np.any(f.reshape(len(X), -1)[[7, 23]])
