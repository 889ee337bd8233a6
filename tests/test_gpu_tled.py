"""Conventional TLED on the GPU (tled_force.hpp): the same
slots, gather and update as the DJ-TLED step with the TLED element kernel.
Gate: bit-identical to the reference's own TledEngine (oracle/_ref) and to
its committed fixtures (tests/golden/tled_*.npz)."""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, config_spec
from paper_2106_14189_b200 import _abi as A

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def run(spec, steps, flags=A.DJG_FLAG_TLED):
    with GpuDjEngine(Scenario(spec), flags=flags) as eng:
        rep = eng.step(steps, raise_on_failure=False)
        u, up, _ = eng.get_state()
        info = eng.info()
    return u, up, rep, info


@pytest.mark.skipif(not oracle.have("ref"), reason="reference library not built")
@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
def test_tled_bitwise_vs_reference_tled(kind, model, precision):
    spec = box_spec(kind=kind, model=model, divisions=4, precision=precision, ramp_steps=300)
    u, up, rep, info = run(spec, 300)
    assert info["formulation"] == 1
    ur, upr, rr = oracle.run(spec, 300, "ref", engine=1)
    assert rep.status == rr["status"] == 0 and rep.step == rr["step"]
    assert np.array_equal(u, ur) and np.array_equal(up, upr)
    assert np.abs(ur).max() > 0.1


@pytest.mark.parametrize("flags", [A.DJG_FLAG_TLED, A.DJG_FLAG_TLED | A.DJG_FLAG_NO_PIPE], ids=["pipe", "nopipe"])
@pytest.mark.parametrize("path", sorted(GOLDEN.glob("tled_*.npz")), ids=lambda p: p.stem)
def test_tled_vs_golden(path, flags):
    g = np.load(path)
    kind, model, d, prec = g["spec"]
    steps = int(g["steps"])
    spec = box_spec(kind=kind, model=model, divisions=int(d), precision=int(prec), ramp_steps=steps)
    u, up, rep, _ = run(spec, steps, flags)
    assert np.array_equal(u, g["u"]) and np.array_equal(up, g["up"])


@pytest.mark.skipif(not oracle.have("ref"), reason="reference library not built")
def test_tled_cfg2_and_dj_agree():
    """cfg2 (H8 NH + hourglass), 1000 steps: TLED == reference TLED bitwise,
    and DJ-TLED vs TLED within the reference's own DJ/TLED f32 spread
    (1.8e-6 .. 6.0e-6)."""
    spec = config_spec("cfg2", precision=4, ramp_steps=2000)
    u_t, _, _, _ = run(spec, 1000)
    ur, _, _ = oracle.run(spec, 1000, "ref", engine=1)
    assert np.array_equal(u_t, ur)
    u_d, _, _, _ = run(spec, 1000, flags=0)
    assert oracle.rel_max_err(u_d, u_t) < 1e-5


def test_tled_inversion_semantics():
    spec = box_spec(kind="T4", divisions=1, extent=(0.1, 0.1, 0.1), precision=8, target=-0.5, dt=1e-4,
                    alpha=0.0, ramp_steps=1)
    u, up, rep, _ = run(spec, 100)
    assert rep.status == A.DJG_E_INVERSION and rep.first_inverted >= 0
    if oracle.have("ref"):
        ur, upr, rr = oracle.run(spec, 100, "ref", engine=1)
        assert (rep.first_inverted, rep.fail_step) == (rr["first_inverted"], rr["fail_step"])
        assert np.array_equal(u, ur)


def _moved_box(d, model):
    """A generated T4 box with one interior node moved off the coordinate
    lattice (the fused step then streams the B0 / V0 planes)."""
    from paper_2106_14189_b200 import mesh_spec
    img = Scenario(box_spec(kind="T4", divisions=d, precision=4)).image()
    x = img["nodes"].reshape(-1, 3).astype(np.float64)
    x[3 + (d[0] + 1) * (2 + (d[1] + 1) * 3), 0] += 0.013
    z = x[:, 2]
    bottom, top = np.flatnonzero(z == z.min()), np.flatnonzero(z == z.max())
    return mesh_spec(x, img["conn"].reshape(-1, 4), kind="T4", model=model, precision=4,
                     fixed=[(int(n), a) for n in bottom for a in range(3)],
                     prescribed=[(int(n), 2, -0.04, 1e-3) for n in top])


@pytest.mark.parametrize("model", ["NH", "TI", "OT"])
@pytest.mark.parametrize("d", [(5, 4, 6), (17, 9, 33), "moved"])
def test_tled_fused_box_step(model, d):
    """TLED in the fused box step (k_box_step<..., TLED>): all four rows of a
    tet kept in shared memory, the record from the lattice table (generated
    box) or streamed from the B0 / V0 planes (a node off the lattice) --
    bit-identical to the two-kernel TLED step and to the reference's
    TledEngine."""
    spec = _moved_box((6, 5, 7), model) if d == "moved" else \
        box_spec(kind="T4", model=model, divisions=d, precision=4, ramp_steps=200)
    u, up, rep, info = run(spec, 200, A.DJG_FLAG_TLED | A.DJG_FLAG_FUSED)
    assert info["fused"] == 1 and info["formulation"] == 1 and info["lattice"] == (d != "moved"), info
    u2, up2, rep2, info2 = run(spec, 200, A.DJG_FLAG_TLED | A.DJG_FLAG_NO_FUSED)
    assert info2["fused"] == 0
    assert rep.status == rep2.status == 0 and rep.step == rep2.step
    assert np.array_equal(u, u2) and np.array_equal(up, up2)
    if oracle.have("ref"):
        ur, upr, rr = oracle.run(spec, 200, "ref", engine=1)
        assert np.array_equal(u, ur) and np.array_equal(up, upr)
    assert np.abs(u).max() > 0


@pytest.mark.parametrize("policy", [A.DJG_ABORT, A.DJG_SKIP_AND_REPORT])
def test_tled_fused_inversion(policy):
    """TLED fused under a crushing load: same halt / counts / state as the
    two-kernel TLED step."""
    spec = box_spec(kind="T4", divisions=(9, 7, 8), extent=(0.1, 0.1, 0.1), precision=4, target=-0.09,
                    ramp_steps=3, fix_all_axes=True, policy=policy)
    outs = []
    for flags in (A.DJG_FLAG_FUSED, A.DJG_FLAG_NO_FUSED):
        u, up, r, info = run(spec, 60, A.DJG_FLAG_TLED | flags)
        outs.append((r, u, up))
    (r1, u1, up1), (r2, u2, up2) = outs
    assert (r1.status, r1.step, r1.first_inverted, r1.inverted_count, r1.inverted_steps) == \
        (r2.status, r2.step, r2.first_inverted, r2.inverted_count, r2.inverted_steps), (r1, r2)
    assert r1.inverted_count > 0
    assert np.array_equal(u1, u2) and np.array_equal(up1, up2)


@pytest.mark.parametrize("model", ["NH", "TI"])
def test_tled_fused_box_step_f64(model):
    spec = box_spec(kind="T4", model=model, divisions=(7, 5, 9), precision=8, ramp_steps=200)
    u, up, rep, info = run(spec, 200, A.DJG_FLAG_TLED | A.DJG_FLAG_FUSED)
    assert info["fused"] == 1 and info["lattice"] == 1
    u2, up2, rep2, _ = run(spec, 200, A.DJG_FLAG_TLED | A.DJG_FLAG_NO_FUSED)
    assert rep.status == rep2.status == 0
    assert np.array_equal(u, u2) and np.array_equal(up, up2) and np.abs(u).max() > 0
