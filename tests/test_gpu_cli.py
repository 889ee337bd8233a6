"""djg command-line tool on the GPU: the reference CLI's end-to-end checks
(tests/test_cli.cpp) plus bitwise parity of the exported field with the CPU
oracle on the same config."""
import numpy as np
import pytest

import oracle
from cli_util import CLI, read_report, read_vtk_field, run_cli, tiny_run_config, write
from paper_2106_14189_b200 import Scenario, box_spec, material, mesh_spec
from paper_2106_14189_b200 import _abi as A

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not CLI.exists(), reason="djg not built")]


def oracle_field(precision, steps, kind="T4", divisions=2, extent=0.1, policy=A.DJG_ABORT, dt=None):
    """The tiny config's problem built in Python: box nodes from the same
    generator, zmin fixed (all axes), zmax ramped along z to 0.005 over 0.02 s,
    dt = 0.8 critical_dt, alpha = 100."""
    dtype = np.float32 if precision == 4 else np.float64
    sc = Scenario(box_spec(kind=kind, divisions=divisions, extent=(extent,) * 3, precision=precision))
    img = sc.image()
    x = img["nodes"].reshape(-1, 3)
    conn = img["conn"]
    z = x[:, 2]
    lo, hi = z.min(), z.max()
    eps = dtype(1e-9) * (hi - lo)
    bottom = np.nonzero(np.abs(z - lo) <= eps)[0]
    top = np.nonzero(np.abs(z - hi) <= eps)[0]
    t = dtype(0.005), dtype(0.02)
    spec = mesh_spec(x.astype(np.float64), conn.reshape(-1, 4 if kind == "T4" else 8), kind=kind,
                     precision=precision, mat=material("NH", mu=float(dtype(6567)), kappa=float(dtype(326210)),
                                                       rho=float(dtype(1060))),
                     fixed=[(int(n), a) for n in bottom for a in range(3)],
                     prescribed=[(int(n), 2, float(t[0]), float(t[1])) for n in top],
                     dt=dt, safety=float(dtype(0.8)), alpha=float(dtype(100)), policy=policy)
    u, up, rep = oracle.run(spec, steps, "oracle")
    return u, rep


@pytest.mark.parametrize("precision", ["double", "single"])
def test_run_writes_artifacts_bitwise_with_oracle(tmp_path, precision):
    """test_cli.cpp:52-58 + parity: the exported field == the CPU oracle."""
    cfg = write(tmp_path / "run.cfg", tiny_run_config(tmp_path))
    rc, out, err = run_cli("run", cfg, "--precision", precision)
    assert rc == 0, err
    rep = read_report(tmp_path / "report.txt")
    assert out.startswith("djtled run report")
    steps = int(rep["steps"])
    assert steps == 13 and "mean_step_us" in rep and rep["engine"] == "djtled"
    field = (tmp_path / "out.vtk").read_text()
    assert "DATASET UNSTRUCTURED_GRID" in field and "VECTORS displacement" in field
    prec = 4 if precision == "single" else 8
    assert f"POINTS 27 {'float' if prec == 4 else 'double'}" in field
    dtype = np.float32 if prec == 4 else np.float64
    u = read_vtk_field(tmp_path / "out.vtk", dtype)
    ur, rr = oracle_field(prec, steps)
    assert rr["status"] == 0 and np.array_equal(u, ur)
    assert float(rep["max_disp"]) == pytest.approx(float(np.abs(ur).max()), rel=1e-11)


def test_repeated_runs_bit_identical(tmp_path):
    """test_cli.cpp:123-131"""
    cfg = write(tmp_path / "run.cfg", tiny_run_config(tmp_path))
    assert run_cli("run", cfg)[0] == 0
    first = (tmp_path / "out.vtk").read_text()
    assert run_cli("run", cfg)[0] == 0
    assert (tmp_path / "out.vtk").read_text() == first


def test_gross_instability_fails_like_the_reference(tmp_path):
    """test_cli.cpp:76-84 with enough steps to fail: dt = 0.05 (30x the bound).
    Abort: the first inverted element at step 3 -> exit 4; report policy:
    inversions skipped until the state turns non-finite -> exit 5; strict
    stability refuses to start -> exit 3. Element id and steps == the oracle."""
    base = tiny_run_config(tmp_path).replace("dt = auto", "dt = 0.05").replace("t_end = 0.02", "t_end = 1")
    cfg = write(tmp_path / "u.cfg", base)
    _, ra = oracle_field(8, 20, dt=0.05)
    rc, _, err = run_cli("run", cfg)
    assert rc == 4 and ra["status"] == 4
    assert f"element {ra['first_inverted']} inverted at step {ra['fail_step']}" in err, err
    _, rr = oracle_field(8, 20, dt=0.05, policy=A.DJG_SKIP_AND_REPORT)
    rc, _, err = run_cli("run", cfg, "--on-inversion", "report")
    assert rc == 5 and rr["status"] == 5
    assert f"solution diverged at step {rr['fail_step']}" in err, err
    assert run_cli("run", cfg, "--strict-stability")[0] == 3


def test_inversion_exit_code_and_report_policy(tmp_path):
    """A crushing prescribed displacement inverts elements: exit 4 under
    abort; under --on-inversion report the run completes and counts steps."""
    cfg = tiny_run_config(tmp_path).replace("prescribe = zmax z 0.005 0.02", "prescribe = zmax z -0.5 0.002")
    path = write(tmp_path / "inv.cfg", cfg)
    rc, _, err = run_cli("run", path)
    assert rc == 4 and "inverted at step" in err, err
    rc, _, err = run_cli("run", path, "--on-inversion", "report")
    assert rc in (0, 5), err
    if rc == 0:
        assert int(read_report(tmp_path / "report.txt")["inverted_steps"]) > 0


def test_compare_reports_consistent_rmse(tmp_path):
    """test_cli.cpp:86-115: rmse tiny and equal to the rmse of the two fields."""
    cfg = write(tmp_path / "cmp.cfg", tiny_run_config(tmp_path, "both"))
    rc, out, err = run_cli("compare", cfg)
    assert rc == 0, err
    rep = read_report(tmp_path / "report.txt")
    rmse = float(rep["rmse"])
    assert rmse < 1e-9
    u_dj = read_vtk_field(tmp_path / "out_djtled.vtk", np.float64)
    u_tl = read_vtk_field(tmp_path / "out_tled.vtk", np.float64)
    assert u_dj.size == u_tl.size == 27 * 3
    assert np.sqrt(np.mean((u_dj - u_tl) ** 2)) == pytest.approx(rmse, abs=1e-12)
    assert "ratio" in rep and "nre_histogram" in out


def test_tled_engine_run(tmp_path):
    cfg = write(tmp_path / "t.cfg", tiny_run_config(tmp_path, "tled"))
    rc, _, err = run_cli("run", cfg)
    assert rc == 0, err
    assert read_report(tmp_path / "report.txt")["engine"] == "tled"


def test_bench_writes_documented_csv(tmp_path):
    """test_cli.cpp:133-145"""
    extra = ("[bench]\nextent = 0.1\ndivisions = 2\nkinds = T4\nmaterials = NH\nwarmup = 2\n"
             f"steps = 10\nthreads = 1\ncsv = {tmp_path}/bench.csv\n")
    cfg = write(tmp_path / "b.cfg", tiny_run_config(tmp_path, extra=extra))
    rc, _, err = run_cli("bench", cfg)
    assert rc == 0, err
    csv = (tmp_path / "bench.csv").read_text()
    assert csv.startswith("dofs,kind,material,engine,threads,mean_step_us,ratio\n")
    assert "81,T4,NH,djtled,1," in csv and "81,T4,NH,tled,1," in csv


def test_binary_mesh_and_npy_field_match_text_path(tmp_path):
    """A mesh file (text and binary) and a .npy field give the same bits as
    the generated box."""
    cfg = write(tmp_path / "run.cfg", tiny_run_config(tmp_path))
    assert run_cli("run", cfg)[0] == 0
    ref = read_vtk_field(tmp_path / "out.vtk", np.float64)
    # export the box as a mesh file through a tiny Python writer (reference format)
    sc = Scenario(box_spec(kind="T4", divisions=2, extent=(0.1,) * 3, precision=8))
    img = sc.image()
    x, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
    lines = ["djtled-mesh 1", f"nodes {len(x)}"] + [" ".join(repr(float(v)) for v in p) for p in x]
    lines += [f"elements T4 {len(conn)}"] + [" ".join(str(int(i)) for i in c) for c in conn]
    write(tmp_path / "box.mesh", "\n".join(lines) + "\n")
    assert run_cli("convert", tmp_path / "box.mesh", tmp_path / "box.djgmesh")[0] == 0
    for mesh in ("box.mesh", "box.djgmesh"):
        text = tiny_run_config(tmp_path).replace("generate = box\nkind = T4\nextent = 0.1\ndivisions = 2 2 2",
                                                 f"file = {mesh}").replace("out.vtk", "out.npy")
        rc, _, err = run_cli("run", write(tmp_path / "m.cfg", text))
        assert rc == 0, err
        u = np.load(tmp_path / "out.npy")
        assert u.shape == (27, 3) and np.array_equal(u.reshape(-1), ref)
