"""djg command-line tool, host side (no GPU): config parsing, error
handling and exit codes of the reference CLI (tools/djtled_main.cpp:13-20,
config.hpp; tests/test_cli.cpp, tests/test_config.cpp), and mesh I/O."""
import numpy as np
import pytest

from cli_util import CLI, read_report, run_cli, tiny_run_config, write

pytestmark = pytest.mark.skipif(not CLI.exists(), reason="djg not built")


def test_usage_without_subcommand():
    rc, _, err = run_cli()
    assert rc == 1 and "usage" in err


@pytest.mark.parametrize("edit,code,msg", [
    (lambda c: c + "[mesh]\nwhat = 1\n", 2, "unknown key 'what' in [mesh]"),              # test_cli.cpp:70-74
    (lambda c: c.replace("generate = box\nkind = T4\nextent = 0.1\ndivisions = 2 2 2",
                         "file = does_not_exist.mesh"), 2, "cannot open mesh file"),     # test_cli.cpp:60-68
    (lambda c: c + "[extra]\nx = 1\n", 2, "unknown section [extra]"),
    (lambda c: c.replace("mu = 6567", "mu = 6567\nmu = 1"), 2, "duplicate key 'mu' in [material]"),
    (lambda c: c.replace("rho = 1060\n", ""), 2, "missing key 'rho' in [material]"),
    (lambda c: c.replace("model = NH", "model = XX"), 2, "unknown material model 'XX'"),
    (lambda c: c.replace("kind = T4", "kind = P6"), 2, "unknown element kind 'P6'"),
    (lambda c: c.replace("divisions = 2 2 2", "divisions = 2 2"), 2, "divisions needs 1 or 3 values"),
    (lambda c: c.replace("divisions = 2 2 2", "divisions = 2 x 2"), 2, "cannot parse divisions"),
    (lambda c: c.replace("mu = 6567", "mu = 6567abc"), 2, "trailing characters in mu"),
    (lambda c: c.replace("safety = 0.8", "safety = 1.5"), 2, "safety must be in (0, 1]"),
    (lambda c: c.replace("alpha = 100", "alpha = -1"), 2, "alpha must be >= 0"),
    (lambda c: c.replace("t_end = 0.02", "t_end = -1"), 2, "t_end must be >= 0"),
    (lambda c: c.replace("dt = auto", "dt = 0"), 2, "dt must be positive"),
    (lambda c: c.replace("fix = zmin all", "fix = top all"), 2, "unknown plane selector 'top'"),
    (lambda c: c.replace("fix = zmin all", "fix = zmin xq"), 2, "unknown axis 'q' in fix rule"),
    (lambda c: c.replace("prescribe = zmax z 0.005 0.02", "prescribe = zmax z 0.005"), 2,
     "prescribe rule needs"),
    (lambda c: c.replace("prescribe = zmax z 0.005 0.02", "prescribe = zmax w 0.005 0.02"), 2, "unknown axis 'w'"),
    (lambda c: c.replace("prescribe = zmax z 0.005 0.02", "prescribe = zmax z 0.005 0"), 2,
     "prescribe ramp duration must be positive"),
    (lambda c: c.replace("prescribe = zmax z 0.005 0.02", "prescribe = zmin z 0.005 0.02"), 2,
     "appears in more than one boundary condition"),
    (lambda c: c.replace("engine = djtled", "engine = cuda"), 2, "unknown engine 'cuda'"),
    (lambda c: c.replace("engine = djtled", "engine = both"), 2, "engine = both is only valid for 'compare'"),
    (lambda c: c.replace("threads = 1", "threads = 0"), 2, "threads must be >= 1 or auto"),
    (lambda c: c + "[run]\non_inversion = maybe\n", 2, "on_inversion must be abort or report"),
    (lambda c: c.replace("[mesh]\n", "[mesh\n"), 2, "line 1: unterminated section header"),
    (lambda c: "key = 1\n" + c, 2, "line 1: key 'key' outside any [section]"),
    (lambda c: c.replace("kind = T4", "kind T4"), 2, "line 3: expected 'key = value'"),
])
def test_config_errors_exit_with_config_code(tmp_path, edit, code, msg):
    cfg = write(tmp_path / "bad.cfg", edit(tiny_run_config(tmp_path)))
    rc, _, err = run_cli("run", cfg)
    assert rc == code, err
    assert msg in err, err
    assert not (tmp_path / "report.txt").exists()


def test_compare_demands_engine_both(tmp_path):
    """test_cli.cpp:117-121"""
    cfg = write(tmp_path / "cmp.cfg", tiny_run_config(tmp_path, "djtled"))
    rc, _, err = run_cli("compare", cfg)
    assert rc == 2 and "compare requires engine = both" in err


def test_strict_stability_refuses_unstable_dt(tmp_path):
    """test_cli.cpp:76-84: dt far above the bound -> exit 3 before any step
    (the stability check runs on the host)."""
    cfg = write(tmp_path / "u.cfg", tiny_run_config(tmp_path).replace("dt = auto", "dt = 0.05"))
    rc, _, err = run_cli("run", cfg, "--strict-stability")
    assert rc == 3 and "exceeds the stability bound" in err


def test_bad_options(tmp_path):
    cfg = write(tmp_path / "run.cfg", tiny_run_config(tmp_path))
    assert run_cli("run", cfg, "--precision", "half")[0] == 1
    assert run_cli("run", cfg, "--on-inversion", "ignore")[0] == 1
    assert run_cli("run", cfg, "--engine", "cpu")[0] == 1
    assert run_cli("frobnicate", cfg)[0] == 1


def _box_text(tmp_path):
    # the reference's mesh file format (mesh.hpp:105-115)
    text = ("djtled-mesh 1\n# a comment\nnodes 5\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n1 1 1\n"
            "elements T4 2\n0 1 2 3\n1 2 3 4\n")
    return write(tmp_path / "two.mesh", text)


@pytest.mark.parametrize("precision", ["single", "double"])
def test_mesh_convert_round_trip(tmp_path, precision):
    src = _box_text(tmp_path)
    rc, _, err = run_cli("convert", src, tmp_path / "two.djgmesh", "--precision", precision)
    assert rc == 0, err
    rc, _, err = run_cli("convert", tmp_path / "two.djgmesh", tmp_path / "back.mesh", "--precision", precision)
    assert rc == 0, err
    back = (tmp_path / "back.mesh").read_text().split("\n")
    assert back[0] == "djtled-mesh 1" and back[1] == "nodes 5" and back[7] == "elements T4 2"
    assert back[8:10] == ["0 1 2 3", "1 2 3 4"]
    assert np.array_equal(np.array(" ".join(back[2:7]).split(), float),
                          np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1, 1, 1], float))


@pytest.mark.parametrize("text,msg", [
    ("djtled-mesh 2\nnodes 0\nelements T4 0\n", "unsupported mesh format version 2"),
    ("nodes 1\n", "expected header 'djtled-mesh 1'"),
    ("djtled-mesh 1\nnodes 2\n0 0 0\n", "unexpected end of file"),
    ("djtled-mesh 1\nnodes 1\n0 0\n", "malformed node coordinates"),
    ("djtled-mesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements T4 1\n0 1 2\n", "expected 4 node indices"),
    ("djtled-mesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements T4 1\n0 1 2 3 0\n", "too many node indices"),
    ("djtled-mesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements Q4 1\n0 1 2 3\n", "unknown element kind 'Q4'"),
    ("djtled-mesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements T4 1\n0 1 2 9\n", "out of range"),
    ("djtled-mesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements T4 1\n0 2 1 3\n",
     "non-positive reference Jacobian determinant"),
])
def test_mesh_file_errors(tmp_path, text, msg):
    src = write(tmp_path / "bad.mesh", text)
    rc, _, err = run_cli("convert", src, tmp_path / "out.mesh")
    assert rc == 2 and msg in err, err


def test_mesh_file_config_excludes_generator_keys(tmp_path):
    _box_text(tmp_path)
    cfg = tiny_run_config(tmp_path).replace("generate = box\n", "file = two.mesh\n")
    rc, _, err = run_cli("run", write(tmp_path / "f.cfg", cfg))
    assert rc == 2 and "file excludes generator keys" in err


def test_prescribe_rule_must_select_nodes(tmp_path):
    # a mesh whose zmax plane is a single node; prescribing xmax of a flat
    # mesh selects the whole mesh -- use a config on a degenerate selector
    _box_text(tmp_path)
    cfg = ("[mesh]\nfile = two.mesh\n[material]\nmodel = NH\nmu = 6567\nkappa = 326210\nrho = 1060\n"
           "[bc]\nfix = zmin all\nprescribe = zmin x 0.1 1\n[time]\nt_end = 0.001\nalpha = relax\n")
    rc, _, err = run_cli("run", write(tmp_path / "p.cfg", cfg))
    assert rc == 2 and "more than one boundary condition" in err
