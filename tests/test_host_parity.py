"""The product's native host builder (libdjg.so, include/djg_host.h) produces
bit-identical engine inputs to the reference and the oracle: mesh, CSR
adjacency, hot constants, masses, dt, alpha, DOF constraints, update
coefficients. No GPU needed."""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2106_14189_b200 import ConfigError, Scenario, box_spec, mesh_spec
from paper_2106_14189_b200 import _abi as A

GOLDEN = Path(__file__).resolve().parent / "golden"


def same(a, b):
    return a.shape == b.shape and bool(np.all(a == b))


@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR", "I57"])
@pytest.mark.parametrize("prec", [4, 8])
def test_builder_matches_oracle(kind, model, prec):
    spec = box_spec(kind=kind, model=model, divisions=(4, 3, 5), precision=prec, ramp_steps=321)
    sc = Scenario(spec, threads=3)
    img = sc.image()
    ref, scal = oracle.image(spec, "oracle")
    for k in img:
        assert same(img[k], ref[k]), k
    for k in ("dt", "critical_dt", "alpha", "c2", "c3", "ramp_t_total", "wave_speed", "nconst"):
        assert sc.scalars[k] == scal[k], k


@pytest.mark.skipif(not oracle.have("ref"), reason="reference library not built here")
@pytest.mark.parametrize("kind,model", [("T4", "NH"), ("H8", "TI"), ("T4", "MR"), ("H8", "OT")])
def test_builder_matches_reference(kind, model):
    spec = box_spec(kind=kind, model=model, divisions=5, precision=4, ramp_steps=1000, fix_all_axes=False,
                    target=0.01)
    img = Scenario(spec).image()
    ref, _ = oracle.image(spec, "ref")
    for k in img:
        assert same(img[k], ref[k]), k


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("run_*.npz"))[:4], ids=lambda p: p.stem)
def test_builder_matches_golden(path):
    g = np.load(path)
    kind, model, d, prec, kw = g["spec"]
    spec = box_spec(kind=kind, model=model, divisions=eval(d), precision=int(prec), ramp_steps=int(g["steps"]),
                    **eval(kw))  # noqa: S307
    img = Scenario(spec).image()
    for k, v in img.items():
        assert same(v, g[f"img_{k}"]), k


def test_builder_thread_count_independent():
    spec = box_spec(kind="H8", model="TI", divisions=9, precision=4, ramp_steps=100)
    a = Scenario(spec, threads=1).image()
    b = Scenario(spec, threads=7).image()
    for k in a:
        assert same(a[k], b[k]), k


def test_explicit_mesh_two_tets_sharing_a_face():
    """test_forces.cpp:379-408 mesh: two tets sharing face (1,2,3)."""
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], float)
    conn = np.array([0, 1, 2, 3, 4, 2, 1, 3], np.int32)
    spec = mesh_spec(nodes, conn, kind="T4", precision=8, fixed=[(0, 0)], prescribed=[(4, 2, 0.01, 1.0)])
    img = Scenario(spec).image()
    ref, _ = oracle.image(spec, "oracle")
    for k in img:
        assert same(img[k], ref[k]), k
    assert list(img["csr_offsets"]) == [0, 1, 3, 5, 7, 8]


def test_config_errors():
    """ConfigError / MeshError conditions (mesh.hpp:55-92, 208-213)."""
    with pytest.raises(ConfigError):
        Scenario(box_spec(extent=(0.0, 1.0, 1.0)))
    with pytest.raises(ConfigError):
        Scenario(box_spec(divisions=(1, 0, 1)))
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    with pytest.raises(ConfigError, match="element 0"):  # inverted tet
        Scenario(mesh_spec(nodes, np.array([0, 2, 1, 3], np.int32)))
    with pytest.raises(ConfigError, match="more than one"):
        Scenario(mesh_spec(nodes, np.array([0, 1, 2, 3], np.int32), fixed=[(0, 1)], prescribed=[(0, 1, 0.1, 1.0)]))
    with pytest.raises(ConfigError, match="ramp duration"):
        Scenario(mesh_spec(nodes, np.array([0, 1, 2, 3], np.int32), prescribed=[(0, 1, 0.1, 0.0)]))
    with pytest.raises(ConfigError, match="out of range"):
        Scenario(mesh_spec(nodes, np.array([0, 1, 2, 9], np.int32)))
    m = box_spec().c.material
    m.kappa = -1.0
    with pytest.raises(ConfigError, match="bulk modulus"):
        Scenario(box_spec(mat=m))


def test_const_count_and_layout():
    lib = A.load_library()
    for kind in (A.DJG_T4, A.DJG_H8):
        for model in range(4):
            assert lib.djg_const_count(kind, model) == A.const_count(kind, model)
    assert A.const_count(A.DJG_T4, A.DJG_NH) * 4 == 92
    assert A.const_count(A.DJG_H8, A.DJG_TI) * 4 == 272
