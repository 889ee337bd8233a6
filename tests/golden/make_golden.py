"""Generates tests/golden/*.npz from the UNMODIFIED reference
(oracle/_ref/libdjref.so, built from /root/reference/proj/include by
oracle/Makefile). Run in the authoring container:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the CPU oracle (tests/test_oracle.py) on machines where the
reference is absent (the GPU box).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2106_14189_b200 import _abi as A  # noqa: E402
from paper_2106_14189_b200.spec import bench_material, box_spec, material  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, kind, model, divisions, precision, steps, extra spec kwargs)
RUNS = [
    ("t4_nh_d3_f32", "T4", "NH", 3, 4, 200, {}),
    ("t4_nh_d3_f64", "T4", "NH", 3, 8, 200, {}),
    ("h8_nh_d3_f32", "H8", "NH", 3, 4, 200, {}),
    ("h8_ti_d3_f32", "H8", "TI", 3, 4, 200, {}),
    ("h8_ti_d3_f64", "H8", "TI", 3, 8, 200, {}),
    ("t4_ti_d3_f32", "T4", "TI", 3, 4, 150, {}),
    ("t4_ot_d2_f64", "T4", "OT", 2, 8, 100, {}),
    ("h8_mr_d2_f64", "H8", "MR", 2, 8, 100, {}),
    ("t4_mr_d2_f32", "T4", "MR", 2, 4, 100, {}),
    ("t4_nh_d3_ext_f32", "T4", "NH", (3, 4, 2), 4, 120, {"target": 0.01, "fix_all_axes": False}),
]


def run_fixture(name, kind, model, d, prec, steps, kw):
    spec = box_spec(kind=kind, model=model, divisions=d, precision=prec, ramp_steps=steps, **kw)
    img, sc = oracle.image(spec, "ref")
    u, up, rep = oracle.run(spec, steps, "ref")
    arrs = {f"img_{k}": v for k, v in img.items()}
    arrs.update({f"sc_{k}": np.array(v) for k, v in sc.items()})
    arrs.update({f"rep_{k}": np.array(v) for k, v in rep.items()})
    np.savez_compressed(OUT / f"run_{name}.npz", u=u, up=up, steps=steps,
                        spec=np.array([kind, model, str(d), str(prec), repr(kw)]), **arrs)


TLED_RUNS = [
    ("t4_nh_d3_f32", "T4", "NH", 3, 4, 150),
    ("h8_ti_d3_f64", "H8", "TI", 3, 8, 150),
    ("t4_mr_d2_f64", "T4", "MR", 2, 8, 100),
    ("h8_ot_d2_f32", "H8", "OT", 2, 4, 100),
]


def tled_fixture(name, kind, model, d, prec, steps):
    """The reference's conventional TLED engine (tled_force.hpp) on the same box."""
    spec = box_spec(kind=kind, model=model, divisions=d, precision=prec, ramp_steps=steps)
    u, up, rep = oracle.run(spec, steps, "ref", engine=1)
    np.savez_compressed(OUT / f"tled_{name}.npz", u=u, up=up, steps=steps,
                        spec=np.array([kind, model, str(d), str(prec)]),
                        **{f"rep_{k}": np.array(v) for k, v in rep.items()})


def failure_fixtures():
    # Inversion (test_solver.cpp:214-241) under both policies, and divergence
    # (test_solver.cpp:192-212).
    from paper_2106_14189_b200.spec import mesh_spec
    spec0 = box_spec(kind="T4", divisions=1, extent=(0.1, 0.1, 0.1), precision=8)
    img, _ = oracle.image(spec0, "ref")
    nodes, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
    bottom = [n for n in range(8) if nodes[n, 2] == 0.0]
    top = [n for n in range(8) if nodes[n, 2] > 0.0]
    out = {}
    for pol in (A.DJG_ABORT, A.DJG_SKIP_AND_REPORT):
        spec = mesh_spec(nodes, conn, kind="T4", precision=8, fixed=[(n, a) for n in bottom for a in range(3)],
                         prescribed=[(n, 2, -0.5, 1e-4) for n in top], dt=1e-4, alpha=0.0, policy=pol)
        u, up, rep = oracle.run(spec, 100, "ref")
        out[f"inv{pol}_u"] = u
        for k, v in rep.items():
            out[f"inv{pol}_{k}"] = np.array(v)
    _, sc = oracle.image(box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8), "ref")
    spec = box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8, target=0.05,
                    dt=10 * sc["critical_dt"], alpha=10.0, ramp_steps=1)
    u, up, rep = oracle.run(spec, 500, "ref")
    out["div_u"] = u
    out["div_dt"] = np.array(10 * sc["critical_dt"])
    for k, v in rep.items():
        out[f"div_{k}"] = np.array(v)
    np.savez_compressed(OUT / "failures.npz", nodes=nodes, conn=conn, bottom=np.array(bottom), top=np.array(top),
                        **out)


def element_fixtures():
    """Random element states (oracles.hpp:126-157 style): coordinates jittered
    around the unit element, small admissible displacements; DJ forces from
    the reference for every kind x material, f64 and f32."""
    rng = np.random.default_rng(2106)
    out = {}
    for kind_name, kind in (("T4", A.DJG_T4), ("H8", A.DJG_H8)):
        npe = A.npe_of(kind)
        if kind == A.DJG_T4:
            base = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
        else:
            base = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                             [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)
        X, U = [], []
        while len(X) < 40:
            x = base * rng.uniform(0.5, 2.0) + rng.uniform(-0.15, 0.15, base.shape)
            u = rng.uniform(-0.1, 0.1, base.shape) * np.abs(x).max()
            # keep states whose DJ force exists (no inversion) in both precisions
            m = bench_material("NH")
            if oracle.ref_element_force(8, kind, m, x, u) is None:
                continue
            X.append(x)
            U.append(u)
        X, U = np.array(X), np.array(U)
        out[f"{kind_name}_coords"] = X
        out[f"{kind_name}_u"] = U
        for model in ("NH", "TI", "OT", "MR"):
            m = bench_material(model)
            for prec in (4, 8):
                F = np.array([oracle.ref_element_force(prec, kind, m, X[i], U[i]) for i in range(len(X))])
                out[f"{kind_name}_{model}_f{8 * prec}"] = F
                if prec == 8:
                    T = np.array([oracle.ref_element_force(8, kind, m, X[i], U[i], engine=1) for i in range(len(X))])
                    out[f"{kind_name}_{model}_tled_f64"] = T
        # DJG_I57: the reference's I5 / I7 force terms driven by the test
        # energy of test_forces.cpp:248-271 (no TLED form): the bench-scale
        # parameters, and the test's own moduli with oblique fibres.
        for name, m in (("I57", bench_material("I57")), ("I57x", I57_TEST)):
            for prec in (4, 8):
                F = np.array([oracle.ref_element_force(prec, kind, m, X[i], U[i]) for i in range(len(X))])
                out[f"{kind_name}_{name}_f{8 * prec}"] = F
    np.savez_compressed(OUT / "elements.npz", **out)


# test_forces.cpp:251: mu 500, kappa 2000, eta5 800, eta7 650 (fibres fixed
# oblique unit-length-free vectors instead of the test's random draws)
I57_TEST = material("I57", mu=500.0, kappa=2000.0, rho=1000.0, eta_a=800.0, eta_b=650.0,
                    fibre_a=(0.3, -0.5, 0.81), fibre_b=(-0.62, 0.1, 0.4))


if __name__ == "__main__":
    if not oracle.have("ref"):
        raise SystemExit("oracle/_ref/libdjref.so missing: run `make -C oracle` where /root/reference exists")
    for r in RUNS:
        run_fixture(*r)
    for r in TLED_RUNS:
        tled_fixture(*r)
    failure_fixtures()
    element_fixtures()
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))
