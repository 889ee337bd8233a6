"""GPU parity: the sm_100a engine (through libdjg's C-ABI) against the CPU
oracle (itself bit-identical to the reference, tests/test_oracle.py) on the
same inputs.

The gate is BITWISE equality of u_curr and u_prev (== semantics, so only the
sign of an exact zero may differ): the engine mirrors the reference's
evaluation order, is compiled with --fmad=false, sums each node's element
rows in ascending element order, and restates glibc's cbrt. The SURVEY §8(c)
tolerances (1e-5 float, 1e-10 double) are asserted as well, as the contract
floor, and integers (CSR, slot map) are exact.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2106_14189_b200 import (GpuDjEngine, Scenario, SimulationError, box_spec, config_spec, material,
                                   mesh_spec)
from paper_2106_14189_b200 import _abi as A

pytestmark = pytest.mark.gpu

TOL = {4: 1e-5, 8: 1e-10}


def run_gpu(spec, steps, **kw):
    sc = Scenario(spec)
    with GpuDjEngine(sc, **kw) as eng:
        rep = eng.step(steps, raise_on_failure=False)
        u, up, step = eng.get_state()
    return u, up, rep


def check_run(spec, steps, tol=None, exact=True, flags=0):
    u, up, rep = run_gpu(spec, steps, flags=flags)
    ur, upr, rr = oracle.run(spec, steps, "oracle")
    assert rep.step == rr["step"] and rep.status == rr["status"], (rep, rr)
    tol = TOL[spec.precision] if tol is None else tol
    e1, e2 = oracle.rel_max_err(u, ur), oracle.rel_max_err(up, upr)
    assert e1 <= tol and e2 <= tol, (e1, e2)
    if exact:
        assert np.array_equal(u, ur) and np.array_equal(up, upr), \
            f"not bit-identical: {np.count_nonzero(u != ur)} of {u.size} DOFs differ (rel {e1:.2e})"
    assert np.max(np.abs(ur)) > 0
    return e1


@pytest.mark.parametrize("precision", [4, 8])
def test_cfg1_t4_nh_2000_steps(precision):
    """BASELINE configs[0]: unit cube T4 (10,368 el) NH, 20% compression."""
    err = check_run(config_spec("cfg1", precision=precision), 2000)
    print(f"cfg1 f{8 * precision}: {err:.3e}")


@pytest.mark.parametrize("precision", [4, 8])
def test_cfg2_h8_nh_hourglass_2000_steps(precision):
    """BASELINE configs[1]: unit cube H8 (10,648 el) NH + hourglass control."""
    err = check_run(config_spec("cfg2", precision=precision), 2000)
    print(f"cfg2 f{8 * precision}: {err:.3e}")


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR", "I57"])
@pytest.mark.parametrize("mode", ["default", "slabs", "nopipe"])
def test_materials_small(kind, model, precision, mode, monkeypatch):
    flags = 0
    if mode == "slabs":
        monkeypatch.setenv("DJG_SLAB_KB", "64")
        flags = A.DJG_FLAG_SLABS
    elif mode == "nopipe":
        flags = A.DJG_FLAG_NO_PIPE
    check_run(box_spec(kind=kind, model=model, divisions=4, precision=precision, ramp_steps=300), 300, flags=flags)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
@pytest.mark.parametrize("flags", [A.DJG_FLAG_COMPACT, A.DJG_FLAG_FULL_RECORD, A.DJG_FLAG_DEVICE_PRECOMPUTE,
                                   A.DJG_FLAG_COMPACT | A.DJG_FLAG_DEVICE_PRECOMPUTE,
                                   A.DJG_FLAG_FULL_RECORD | A.DJG_FLAG_DEVICE_PRECOMPUTE])
def test_compact_and_device_precompute_bitwise(kind, model, precision, flags):
    check_run(box_spec(kind=kind, model=model, divisions=4, precision=precision, ramp_steps=300), 300, flags=flags)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
@pytest.mark.parametrize("flags", [0, A.DJG_FLAG_FULL_RECORD, A.DJG_FLAG_TLED, A.DJG_FLAG_DEVICE_PRECOMPUTE])
def test_pipeline_partial_tiles(model, precision, flags):
    """k_element_pipe on a mesh whose element count is not a multiple of the
    128-element tile (720 tets: 5 full tiles + 80), with record tail planes
    and rank words whose copies round up to 16 bytes. (f64 Mooney-Rivlin keeps
    the full record by default; its compact pipeline is forced here.)"""
    if model == "MR" and not flags & (A.DJG_FLAG_FULL_RECORD | A.DJG_FLAG_TLED):
        flags |= A.DJG_FLAG_COMPACT
    spec = box_spec(kind="T4", model=model, divisions=(5, 4, 6), precision=precision, ramp_steps=250)
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=flags) as eng:
        # full f64 records of the anisotropic models exceed the stage budget
        assert eng.info()["pipelined"] == 1 or (flags & A.DJG_FLAG_FULL_RECORD)
    if flags & A.DJG_FLAG_TLED:
        return  # TLED parity is tests/test_gpu_tled.py
    check_run(spec, 250, flags=flags)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
@pytest.mark.parametrize("flags", [0, A.DJG_FLAG_FULL_RECORD, A.DJG_FLAG_DEVICE_PRECOMPUTE])
def test_node_windows_bitwise(model, precision, flags):
    """k_element_win (DJG_FLAG_WINDOW): each tile's node rows staged by
    bulk copies beside precomputed slot positions -- every T4 tile of the
    box fits its window, partial last tile included; bit-identical to the
    oracle."""
    if model == "MR" and not flags & A.DJG_FLAG_FULL_RECORD:
        flags |= A.DJG_FLAG_COMPACT
    spec = box_spec(kind="T4", model=model, divisions=(5, 4, 6), precision=precision, ramp_steps=250)
    with GpuDjEngine(Scenario(spec), flags=flags | A.DJG_FLAG_WINDOW) as eng:
        info = eng.info()
    if info["pipelined"]:
        assert info["windowed"] == 1 and info["window_tiles"] == 6, info
    check_run(spec, 250, flags=flags | A.DJG_FLAG_WINDOW)


def test_node_windows_mixed_tiles():
    """A box whose node ids are permuted in the upper half only: tiles of the
    lower half fit their windows, the others fall back to the staged
    connectivity + global gather; both kinds of tile in one launch, the
    multi-step graph and the host-state step, bit-identical."""
    rng = np.random.default_rng(5)
    img = Scenario(box_spec(kind="T4", divisions=(8, 6, 10), precision=4)).image()
    x = img["nodes"].reshape(-1, 3).astype(np.float64)
    conn = img["conn"].reshape(-1, 4)
    N = len(x)
    perm = np.arange(N)
    hi = np.flatnonzero(x[:, 2] > 0.5)
    perm[hi] = rng.permutation(hi)          # old node i -> new id perm[i]
    xn = np.empty_like(x)
    xn[perm] = x
    cn = perm[conn].astype(np.int32)
    z = xn[:, 2]
    bottom = np.flatnonzero(z == z.min())
    top = np.flatnonzero(z == z.max())
    for prec in (4, 8):
        spec = mesh_spec(xn, cn, kind="T4", precision=prec, fixed=[(int(n), a) for n in bottom for a in range(3)],
                         prescribed=[(int(n), 2, -0.04, 1e-3) for n in top])
        sc = Scenario(spec)
        with GpuDjEngine(sc, flags=A.DJG_FLAG_WINDOW) as eng:
            info = eng.info()
            ntiles = (sc.num_elements + 127) // 128
            assert 0 < info["window_tiles"] < ntiles, info
        check_run(spec, 200, flags=A.DJG_FLAG_WINDOW)
        check_run(spec, 200, flags=A.DJG_FLAG_WINDOW | A.DJG_FLAG_NO_GRAPH)


@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT"])
@pytest.mark.parametrize("divisions", [(5, 4, 6), (17, 9, 33), (16, 16, 16), (33, 2, 5), (1, 1, 1)])
def test_fused_box_step_bitwise(divisions, model, kind):
    """k_box_step (DJG_FLAG_FUSED): one kernel per step on a generated box --
    element forces into shared memory, each node folding its tets' rows in
    ascending element id, the update -- bit-identical to the oracle, on boxes
    whose sides are and are not multiples of the 16 x 16 x 16 tile."""
    spec = box_spec(kind=kind, model=model, divisions=divisions, precision=4, ramp_steps=200)
    with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
        info = eng.info()
        assert info["fused"] == 1 and info["lattice"] == (kind == "T4")
    check_run(spec, 200, flags=A.DJG_FLAG_FUSED)


@pytest.mark.parametrize("model", ["NH", "TI", "OT"])
@pytest.mark.parametrize("divisions", [(5, 4, 6), (17, 9, 33), (1, 1, 1)])
def test_fused_box_step_f64(divisions, model):
    """The fused T4 step in double precision (f64 rows and records, one
    block per SM): bit-identical to the oracle, with and without the lattice
    table."""
    spec = box_spec(kind="T4", model=model, divisions=divisions, precision=8, ramp_steps=200)
    with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
        info = eng.info()
        assert info["fused"] == 1 and info["lattice"] == 1
    check_run(spec, 200, flags=A.DJG_FLAG_FUSED)


def test_fused_box_step_f64_off_lattice(monkeypatch):
    monkeypatch.setenv("DJG_LATTICE", "0")
    spec = box_spec(kind="T4", model="TI", divisions=(9, 8, 7), precision=8, ramp_steps=200)
    with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
        info = eng.info()
        assert info["fused"] == 1 and info["lattice"] == 0
    check_run(spec, 200, flags=A.DJG_FLAG_FUSED)


def _box_with_nodes(divisions, move, **kw):
    """A generated T4 box's connectivity with its node coordinates moved by
    move(x) (fixed bottom face, prescribed top face)."""
    img = Scenario(box_spec(kind="T4", divisions=divisions, precision=4)).image()
    x = move(img["nodes"].reshape(-1, 3).astype(np.float64))
    z = x[:, 2]
    bottom, top = np.flatnonzero(z == z.min()), np.flatnonzero(z == z.max())
    return mesh_spec(x, img["conn"].reshape(-1, 4), kind="T4", precision=4,
                     fixed=[(int(n), a) for n in bottom for a in range(3)],
                     prescribed=[(int(n), 2, -0.04, 1e-3) for n in top], **kw)


@pytest.mark.parametrize("axis", [0, 2])
def test_fused_lattice_one_ulp_off(axis):
    """One interior node moved by a single float ulp: the per-axis classes
    (taken along the box's edges) do not see it, the check of every tet's
    record against its class entry does -- the table is refused (lattice = 0)
    and the step stays bit-identical to the oracle."""
    d = (8, 7, 9)

    def nudge(x):
        x = x.copy()
        n = 4 + (d[0] + 1) * (3 + (d[1] + 1) * 5)  # node (4, 3, 5)
        x[n, axis] = float(np.nextafter(np.float32(x[n, axis]), np.float32(2)))
        return x
    spec = _box_with_nodes(d, nudge)
    with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
        info = eng.info()
        assert info["fused"] == 1 and info["lattice"] == 0, info
    check_run(spec, 120, flags=A.DJG_FLAG_FUSED)


@pytest.mark.parametrize("model", ["NH", "TI", "OT"])
def test_fused_lattice_table(model, monkeypatch):
    """The fused T4 step's lattice table (build_lattice): on a graded lattice
    (x_i = (i / n)^2: a class per interval, hundreds of class triples) the
    table is used and bit-identical to the oracle; on the same box with one
    interior node moved off the lattice the table check fails on the tets
    around it and the step rebuilds every record (lattice = 0), still
    bit-identical; DJG_LATTICE=0 gives the rebuild on the generated box."""
    d = (11, 7, 9)
    graded = _box_with_nodes(d, lambda x: x * x, model=model)

    def off_lattice(x):
        x = x.copy()
        n = 3 + 12 * (4 + 8 * 5)  # node (3, 4, 5)
        x[n, 0] += 0.013
        return x
    moved = _box_with_nodes(d, off_lattice, model=model)
    for spec, want in ((graded, 1), (moved, 0)):
        with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
            info = eng.info()
            assert info["fused"] == 1 and info["lattice"] == want, info
        check_run(spec, 150, flags=A.DJG_FLAG_FUSED)
    monkeypatch.setenv("DJG_LATTICE", "0")
    spec = box_spec(kind="T4", model=model, divisions=d, precision=4, ramp_steps=150)
    with GpuDjEngine(Scenario(spec), flags=A.DJG_FLAG_FUSED) as eng:
        assert eng.info()["lattice"] == 0
    check_run(spec, 150, flags=A.DJG_FLAG_FUSED)


@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("policy", [A.DJG_ABORT, A.DJG_SKIP_AND_REPORT])
def test_fused_box_step_inversion(policy, kind):
    """The fused step under a crushing load: Abort halts on the same element
    and step with the same state as the two-kernel step (the fused kernel has
    already written u_next when it learns of the inversion; the step is not
    closed, so the state stays), SkipAndReport gives the same counts (each
    inversion counted once, by the tile owning the cell)."""
    spec = box_spec(kind=kind, divisions=(9, 7, 8), extent=(0.1, 0.1, 0.1), precision=4, target=-0.09,
                    ramp_steps=3, fix_all_axes=True, policy=policy)
    outs = []
    for flags in (A.DJG_FLAG_FUSED, A.DJG_FLAG_NO_FUSED):
        with GpuDjEngine(Scenario(spec), flags=flags) as eng:
            r = eng.step(60, raise_on_failure=False)
            outs.append((r, *eng.get_state()))
    (r1, u1, up1, s1), (r2, u2, up2, s2) = outs
    assert (r1.status, r1.step, r1.first_inverted, r1.inverted_count, r1.inverted_steps) == \
        (r2.status, r2.step, r2.first_inverted, r2.inverted_count, r2.inverted_steps), (r1, r2)
    assert r1.inverted_count > 0
    assert np.array_equal(u1, u2) and np.array_equal(up1, up2)
    ur, upr, rr = oracle.run(spec, 60, "oracle")
    assert (r1.status, r1.first_inverted, r1.inverted_count) == (rr["status"], rr["first_inverted"],
                                                                 rr["inverted_count"])
    assert np.array_equal(u1, ur)


@pytest.mark.parametrize("kind,model,d", [("T4", "NH", 96), ("H8", "TI", 100)])
def test_fused_box_step_large_vs_two_kernel(kind, model, d):
    """A 96^3 T4 box (5.3M tets) and cfg4 (1M hexes, TI) against the
    two-kernel step on the same device, 300 steps, bitwise (u and u_prev)."""
    spec = box_spec(kind=kind, model=model, divisions=d, precision=4, target=0.01, ramp_steps=300)
    sc = Scenario(spec)
    res = []
    for flags in (A.DJG_FLAG_FUSED, A.DJG_FLAG_NO_FUSED):
        with GpuDjEngine(sc, flags=flags) as eng:
            res.append(eng.info()["fused"])
            eng.step(300)
            res.append(eng.get_state())
    assert res[0] == 1 and res[2] == 0
    assert np.array_equal(res[1][0], res[3][0]) and np.array_equal(res[1][1], res[3][1])


@pytest.mark.parametrize("flags", [A.DJG_FLAG_COMPACT, A.DJG_FLAG_DEVICE_PRECOMPUTE, A.DJG_FLAG_TLED])
def test_i57_full_record_only(flags):
    """DJG_I57 (the I5 / I7 test energy) runs on the host-built full record;
    the compact, device-precompute and TLED forms are refused loudly."""
    sc = Scenario(box_spec(kind="T4", model="I57", divisions=2, precision=4))
    with GpuDjEngine(sc) as eng:
        info = eng.info()
        assert info["compact"] == 0 and info["pipelined"] == 0 and info["nconst"] == 137
    with pytest.raises(Exception, match="I57"):
        GpuDjEngine(sc, flags=flags)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_i57_longer_run(kind, precision):
    """The fifth/seventh-invariant terms over a 600-step compression, bitwise."""
    check_run(box_spec(kind=kind, model="I57", divisions=(4, 3, 5), precision=precision, ramp_steps=600), 600)


def test_pipeline_selection():
    """T4 and f32 compact H8 run the bulk-copy pipeline by default; DJG_FLAG_NO_PIPE and the
    larger H8 records the one-shot kernel."""
    for kind, flags, want in (("T4", 0, 1), ("T4", A.DJG_FLAG_NO_PIPE, 0), ("H8", 0, 1),
                              ("H8", A.DJG_FLAG_FULL_RECORD, 0)):
        sc = Scenario(box_spec(kind=kind, divisions=3, precision=4))
        with GpuDjEngine(sc, flags=flags) as eng:
            assert eng.info()["pipelined"] == want, (kind, flags)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("model", ["NH", "TI", "OT", "MR"])
def test_device_precompute_equals_host_precompute(kind, model, precision):
    """build_element_constants on the GPU == on the host (== the reference),
    bit for bit, every field of every element."""
    spec = box_spec(kind=kind, model=model, divisions=(5, 4, 6), precision=precision)
    sc = Scenario(spec)
    host = sc.image()["consts"].reshape(sc.num_elements, -1)
    with GpuDjEngine(sc, flags=A.DJG_FLAG_DEVICE_PRECOMPUTE | A.DJG_FLAG_FULL_RECORD) as eng:
        dev = eng.device_consts()
    assert np.array_equal(dev, host)
    with GpuDjEngine(sc, flags=A.DJG_FLAG_DEVICE_PRECOMPUTE | A.DJG_FLAG_COMPACT) as eng:
        dev_c = eng.device_consts()
    with GpuDjEngine(sc, flags=A.DJG_FLAG_COMPACT) as eng:
        host_c = eng.device_consts()
    assert np.array_equal(dev_c, host_c)
    if kind == "T4":
        assert dev_c.shape[1] == 0  # compact T4: no record, J0 is rebuilt from the coordinates
    else:
        assert np.array_equal(dev_c[:, :11], host[:, :11])  # J0, det J0, V0


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
@pytest.mark.parametrize("flags", [A.DJG_FLAG_COMPACT, A.DJG_FLAG_COMPACT | A.DJG_FLAG_DEVICE_PRECOMPUTE])
def test_compact_cfg_2000_steps(cfg, flags):
    check_run(config_spec(cfg, precision=4), 2000, flags=flags)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_slab_path_cfg(cfg, monkeypatch):
    monkeypatch.setenv("DJG_SLAB_KB", "64")
    check_run(config_spec(cfg, precision=4), 500, flags=A.DJG_FLAG_SLABS)


def test_slab_schedule_on_large_mesh():
    sc = Scenario(config_spec("cfg3", precision=4))
    with GpuDjEngine(sc) as eng:  # cfg3's default: the fused step on the lattice table
        info = eng.info()
        assert info["fused"] == 1 and info["lattice"] == 1 and info["kernels_per_step"] == 1
    with GpuDjEngine(sc, flags=A.DJG_FLAG_NO_FUSED) as eng:
        assert eng.info()["slabs"] == 1 and eng.info()["kernels_per_step"] == 2
    with GpuDjEngine(sc, flags=A.DJG_FLAG_SLABS) as eng:
        info = eng.info()
    assert info["slabs"] > 1 and info["kernels_per_step"] == 2 * info["slabs"]
    assert info["slab_elements"] * info["npe"] * 16 <= 40 << 20


@pytest.mark.parametrize("kind,model", [("T4", "NH"), ("H8", "TI"), ("T4", "MR")])
def test_many_slabs_bitwise(kind, model, monkeypatch):
    """Small slabs (64 KB of rows: several slabs even on small meshes)."""
    monkeypatch.setenv("DJG_SLAB_KB", "64")
    spec = box_spec(kind=kind, model=model, divisions=14, precision=4, ramp_steps=300)
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=A.DJG_FLAG_SLABS) as eng:
        assert eng.info()["slabs"] >= 3
    check_run(spec, 300, flags=A.DJG_FLAG_SLABS)
    check_run(spec, 300, flags=A.DJG_FLAG_SLABS | A.DJG_FLAG_NO_DISCARD)


@pytest.mark.slow
def test_cfg3_slab_vs_two_kernel_bitwise():
    spec = config_spec("cfg3", precision=4, target=0.01, ramp_steps=1000)
    a = run_gpu(spec, 50)[0]  # fused (lattice table)
    b = run_gpu(spec, 50, flags=A.DJG_FLAG_SLABS)[0]
    c = run_gpu(spec, 50, flags=A.DJG_FLAG_SLABS | A.DJG_FLAG_NO_DISCARD)[0]
    d = run_gpu(spec, 50, flags=A.DJG_FLAG_NO_FUSED)[0]
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)


@pytest.mark.parametrize("flags", [A.DJG_FLAG_SLABS | A.DJG_FLAG_NO_DISCARD, A.DJG_FLAG_NO_GRAPH | A.DJG_FLAG_SLABS,
                                   A.DJG_FLAG_NO_GRAPH])
def test_variants_bitwise_cfg2(flags, monkeypatch):
    monkeypatch.setenv("DJG_SLAB_KB", "64")
    check_run(config_spec("cfg2", precision=4), 400, flags=flags)


@pytest.mark.parametrize("precision", [4, 8])
def test_cfg4_shape_h8_ti(precision):
    """configs[3] material/element on a smaller cube (d=16)."""
    check_run(box_spec(kind="H8", model="TI", divisions=16, precision=precision, ramp_steps=400), 400)


@pytest.mark.slow
def test_cfg3_first_200_steps():
    """configs[2] at full size (2,058,000 T4): first 200 steps vs the oracle."""
    check_run(config_spec("cfg3", precision=4, ramp_steps=1100), 200)


@pytest.mark.slow
def test_cfg5_full_size_bitwise():
    """BASELINE configs[4] at full size (50,192,562 tets, the bench problem
    and loading): 8 steps of a fast +1 % extension ramp, bit-identical to the
    CPU oracle (all host threads)."""
    spec = config_spec("cfg5", precision=4, target=0.01, ramp_steps=8)
    with GpuDjEngine(Scenario(spec)) as eng:
        assert eng.info()["fused"] == 1  # the default step on cfg5: one fused kernel
    check_run(spec, 8)
    check_run(spec, 8, flags=A.DJG_FLAG_NO_FUSED)


@pytest.mark.slow
@pytest.mark.parametrize("load", ["extension", "compression"])
def test_cfg5_soak_550_steps(load):
    """SURVEY §8(d)'s cfg5 protocol length on the full 50,192,562-tet mesh
    against the CPU oracle on the host cores: the +1 % extension ramp for all
    550 steps, bit-identical (u and u_prev); the 20 % compression ramp, which
    inverts elements at step 118 -- same abort step, same first inverted
    element and count, same retained state."""
    if load == "extension":
        spec = config_spec("cfg5", precision=4, target=0.01, ramp_steps=550)
    else:
        spec = config_spec("cfg5", precision=4)
    u, up, rep = run_gpu(spec, 550)
    ur, upr, rr = oracle.run(spec, 550, "oracle")
    assert (rep.status, rep.step, rep.first_inverted, rep.inverted_count) == \
        (rr["status"], rr["step"], rr["first_inverted"], rr["inverted_count"]), (rep, rr)
    if load == "compression":
        assert rr["status"] == A.DJG_E_INVERSION and rr["fail_step"] == 118
    else:
        assert rr["status"] == 0 and rr["step"] == 550
    assert np.array_equal(u, ur) and np.array_equal(up, upr)


@pytest.mark.slow
def test_cfg4_first_100_steps():
    """configs[3] at full size (1,000,000 H8 TI): first 100 steps vs the oracle."""
    check_run(config_spec("cfg4", precision=4, ramp_steps=1100), 100)


@pytest.mark.parametrize("precision", [4, 8])
def test_assemble_random_state(precision):
    """Engine::assemble at a random admissible state equals the oracle's."""
    spec = box_spec(kind="T4", model="MR", divisions=(3, 4, 5), precision=precision, extent=(0.1, 0.1, 0.1))
    sc = Scenario(spec)
    rng = np.random.default_rng(13)
    u = rng.uniform(-0.003, 0.003, 3 * sc.num_nodes)
    with GpuDjEngine(sc) as eng:
        f, st = eng.assemble(u)
    fr, sr = oracle.assemble(spec, u)
    assert st["first_inverted"] == -1 and sr["first_inverted"] == -1
    assert np.array_equal(f, fr)


def test_slot_map_is_a_bijection_consistent_with_csr():
    spec = box_spec(kind="H8", model="NH", divisions=(5, 3, 4))
    sc = Scenario(spec)
    img = sc.image()
    with GpuDjEngine(sc) as eng:
        slots = eng.slot_map()
        info = eng.info()
    npe = 8
    assert len(np.unique(slots)) == slots.size
    assert slots.min() >= 0 and slots.max() < info["slot_capacity"]
    off, ce, cl = img["csr_offsets"], img["csr_elem"], img["csr_local"]
    N = sc.num_nodes
    for n in range(N):
        for k, p in enumerate(range(off[n], off[n + 1])):
            base = 32 * k + (n % 32)
            pos = slots[ce[p] * npe + cl[p]]
            assert (pos - base) % 32 == 0  # slot k of node n in lane n%32 of its slice


def test_rest_stays_at_rest():
    """test_solver.cpp:52-66 (no loads, from rest). Element forces at rest
    cancel only to rounding (the reference itself drifts to ~1e-17 m here),
    so the field must stay at that noise level, as the oracle's does."""
    spec = box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8, alpha=0.0, dt=1e-4)
    spec.c.bc_mode = 0
    u, up, rep = run_gpu(spec, 20)
    ur, _, rr = oracle.run(spec, 20, "oracle")
    assert rep.status == 0 and rep.step == 20 == rr["step"]
    assert np.max(np.abs(u)) < 1e-15 and np.max(np.abs(ur)) < 1e-15


def test_fixed_and_ramp_exact_every_frame():
    """test_solver.cpp:144-166: fixed DOFs exactly 0, ramped DOFs exactly
    min(dt*s/T, 1)*target at every one of 200 frames."""
    spec = box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8, target=0.03, alpha=50.0)
    sc = Scenario(spec)
    img = sc.image()
    dt = sc.dt
    T = sc.scalars["ramp_t_total"]
    kinds = img["dof_kind"]
    with GpuDjEngine(sc) as eng:
        for s in range(1, 201):
            eng.step(1)
            u = eng.get_state()[0]
            assert np.all(u[kinds == A.DJG_FIXED] == 0.0)
            s_ = (dt * float(s)) / T
            expect = (1.0 if s_ >= 1.0 else s_) * 0.03
            assert np.all(u[kinds == A.DJG_PRESCRIBED] == expect)


def test_deterministic_repeats():
    spec = box_spec(kind="H8", model="NH", divisions=6, precision=4, ramp_steps=300)
    a = run_gpu(spec, 300)[0]
    b = run_gpu(spec, 300)[0]
    c = run_gpu(spec, 300, flags=A.DJG_FLAG_NO_GRAPH)[0]
    d = run_gpu(spec, 300, flags=A.DJG_FLAG_SLABS)[0]
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)


def test_resume_from_state_is_bitwise():
    """run_simulation's `initial` hook (solver.hpp:209-214)."""
    spec = box_spec(kind="T4", model="TI", divisions=5, precision=4, ramp_steps=400)
    sc = Scenario(spec)
    with GpuDjEngine(sc) as eng:
        eng.step(400)
        u_full = eng.get_state()[0]
        eng.set_state(None, None, 0)
        eng.step(150)
        u, up, st = eng.get_state()
    with GpuDjEngine(sc) as eng2:
        eng2.set_state(u, up, st)
        eng2.step(250)
        assert np.array_equal(eng2.get_state()[0], u_full)


def test_external_force_matches_oracle():
    spec = box_spec(kind="T4", divisions=3, precision=8, target=0.0, ramp_steps=100)
    sc = Scenario(spec)
    rng = np.random.default_rng(5)
    r = rng.uniform(-1.0, 1.0, 3 * sc.num_nodes)
    with GpuDjEngine(sc) as eng:
        eng.set_external(r)
        eng.step(100)
        u = eng.get_state()[0]
    ur, _, _ = oracle.run(spec, 100, "oracle", r_ext=r)
    assert np.array_equal(u, ur)


def test_inversion_abort_reports_min_element_and_keeps_state():
    """test_solver.cpp:214-241: the top face is driven through the bottom."""
    sc0 = Scenario(box_spec(kind="T4", divisions=1, extent=(0.1, 0.1, 0.1), precision=8))
    img = sc0.image()
    nodes, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
    bottom = [n for n in range(8) if nodes[n, 2] == 0.0]
    top = [n for n in range(8) if nodes[n, 2] > 0.0]
    fixed = [(n, a) for n in bottom for a in range(3)]
    presc = [(n, 2, -0.5, 1e-4) for n in top]
    spec = mesh_spec(nodes, conn, kind="T4", precision=8, fixed=fixed, prescribed=presc, dt=1e-4, alpha=0.0)
    u, up, rep = run_gpu(spec, 100)
    ur, upr, rr = oracle.run(spec, 100, "oracle")
    assert rep.status == A.DJG_E_INVERSION == rr["status"]
    assert rep.first_inverted == rr["first_inverted"] >= 0
    assert (rep.fail_step, rep.step) == (rr["fail_step"], rr["step"])
    assert np.array_equal(u, ur) and np.array_equal(up, upr)
    with pytest.raises(SimulationError) as ei:
        with GpuDjEngine(Scenario(spec)) as eng:
            eng.step(100)
    assert ei.value.kind == SimulationError.ElementInversion and ei.value.index == rr["first_inverted"]
    # Skip-and-report keeps going and counts the inverted steps.
    spec.c.policy = A.DJG_SKIP_AND_REPORT
    _, _, rep2 = run_gpu(spec, 100)
    _, _, rr2 = oracle.run(spec, 100, "oracle")
    assert rep2.inverted_steps > 0
    assert (rep2.status, rep2.step, rep2.inverted_steps) == (rr2["status"], rr2["step"], rr2["inverted_steps"])


def test_divergence_detector():
    """test_solver.cpp:192-212: dt = 10 x critical."""
    sc0 = Scenario(box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8))
    spec = box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8, target=0.05,
                    dt=10 * sc0.scalars["critical_dt"], alpha=10.0, ramp_steps=1)
    spec.c.ramp_steps = 1
    u, up, rep = run_gpu(spec, 500)
    ur, upr, rr = oracle.run(spec, 500, "oracle")
    assert rep.status in (A.DJG_E_DIVERGENCE, A.DJG_E_INVERSION)
    assert (rep.status, rep.step, rep.fail_step) == (rr["status"], rr["step"], rr["fail_step"])
    with pytest.raises(SimulationError):
        sc = Scenario(spec)
        with GpuDjEngine(sc) as eng:
            eng.step(500)


def _wave_speed(m, dtype):
    """dilatational_wave_speed (material.hpp:117-120) in Real."""
    kappa, rho = dtype(m.kappa), dtype(m.rho)
    mu = dtype(2) * (dtype(m.c10) + dtype(m.c01)) if m.model == A.DJG_MR else dtype(m.mu)
    return np.sqrt((kappa + dtype(4) / dtype(3) * mu) / rho).astype(dtype)


@pytest.mark.parametrize("precision", [4, 8])
@pytest.mark.parametrize("kind,model", [("T4", "NH"), ("T4", "TI"), ("T4", "MR"), ("H8", "NH"), ("H8", "OT")])
def test_device_layout_and_precompute(kind, model, precision):
    """with DJG_FLAG_DEVICE_PRECOMPUTE and no caller CSR the
    adjacency (stable radix sort by node), slot ranks, slices, lump_mass and
    characteristic lengths are built on the GPU: identical slot map, masses
    == the host builder (== the reference) bit for bit, critical_dt equal,
    and the run bit-identical to the oracle."""
    dtype = np.float32 if precision == 4 else np.float64
    spec = box_spec(kind=kind, model=model, divisions=(5, 4, 6), precision=precision, ramp_steps=250)
    sc = Scenario(spec)
    img = sc.image()
    fl = A.DJG_FLAG_DEVICE_PRECOMPUTE
    with GpuDjEngine(sc, flags=fl) as host_layout:
        smap = host_layout.slot_map()
        info_h = host_layout.info()
    with GpuDjEngine(sc, flags=fl, device_csr=True) as eng:
        assert np.array_equal(eng.slot_map(), smap)
        info = eng.info()
        for k in ("slot_capacity", "num_slots", "pipelined", "compact"):
            assert info[k] == info_h[k], k
        assert np.array_equal(eng.lump_mass(), img["mass"])
        dt = dtype(eng.min_char_length()) / _wave_speed(spec.c.material, dtype)
        assert dtype(dt) == dtype(sc.scalars["critical_dt"])
        rep = eng.step(250, raise_on_failure=False)
        u, up, _ = eng.get_state()
    ur, upr, rr = oracle.run(spec, 250, "oracle")
    assert rep.status == rr["status"] == 0 and np.array_equal(u, ur) and np.array_equal(up, upr)


def test_device_layout_rejects_bad_connectivity():
    spec = box_spec(kind="T4", divisions=2, precision=4)
    sc = Scenario(spec)
    d = sc.desc(0, A.DJG_FLAG_DEVICE_PRECOMPUTE)
    d.csr_offsets = d.csr_elem = d.csr_local = None
    conn = np.ctypeslib.as_array(C.cast(C.c_void_p(d.conn), C.POINTER(C.c_int32)), shape=(sc.num_elements * 4,)).copy()
    conn[7] = sc.num_nodes + 3
    d.conn = conn.ctypes.data_as(C.c_void_p)
    h = C.c_void_p()
    rc = A.load_library().djg_create(C.byref(d), C.byref(h))
    assert rc == A.DJG_E_CONFIG and b"out of range" in A.load_library().djg_create_error()


@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_unstructured_numbering_and_isolated_node(kind):
    """A box with randomly permuted node ids and element order, jittered
    coordinates and one isolated (massless, element-less) node: irregular
    CSR rows and slices, bit-identical to the oracle."""
    rng = np.random.default_rng(7)
    sc = Scenario(box_spec(kind=kind, divisions=(5, 4, 6), precision=8))
    img = sc.image()
    npe = 4 if kind == "T4" else 8
    x = img["nodes"].reshape(-1, 3)
    conn = img["conn"].reshape(-1, npe)
    h = 1.0 / 6
    x = x + rng.uniform(-0.08 * h, 0.08 * h, x.shape)
    perm = rng.permutation(len(x))          # new id of old node i = inv[i]
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(x))
    xn = np.vstack([x[perm], [[2.0, 2.0, 2.0]]])  # + isolated node
    cn = inv[conn][rng.permutation(len(conn))]
    z = xn[:-1, 2]
    bottom = np.flatnonzero(np.abs(z - z.min()) < 1e-12)
    top = np.flatnonzero(np.abs(z - z.max()) < 1e-12)
    for prec in (8, 4):
        spec = mesh_spec(xn, cn, kind=kind, precision=prec, fixed=[(int(n), a) for n in bottom for a in range(3)],
                         prescribed=[(int(n), 2, -0.03, 1e-3) for n in top])
        check_run(spec, 200)


def test_high_valence_node_uses_two_byte_ranks():
    """A fan of 300 tets around one axis: its two hub nodes have 300 incident
    elements (> 256: 16-bit slot ranks), bit-identical to the oracle."""
    M = 300
    ang = 2 * np.pi * np.arange(M) / M
    ring = np.c_[np.cos(ang), np.sin(ang), np.zeros(M)]
    x = np.vstack([[0.0, 0.0, 0.0], [0.0, 0.0, 1.0], ring])
    conn = []
    for i in range(M):
        t = [0, 2 + i, 2 + (i + 1) % M, 1]
        a, b, c, d = x[t]
        if np.linalg.det(np.c_[b - a, c - a, d - a]) < 0:
            t[1], t[2] = t[2], t[1]
        conn.append(t)
    conn = np.array(conn, np.int32)
    for prec in (4, 8):
        spec = mesh_spec(x, conn, kind="T4", precision=prec,
                         fixed=[(n, a) for n in range(2, 2 + M) for a in range(3)] + [(0, a) for a in range(3)],
                         prescribed=[(1, 2, -0.05, 2e-3), (1, 0, 0.02, 2e-3)])
        check_run(spec, 300)


def _nh_ref():
    return material("NH", mu=6567.0, kappa=326210.0, rho=1060.0)


def test_small_strain_extension_matches_linear_modulus():
    """test_solver.cpp:265-284: 1 % uniaxial extension of a 0.1 m cube (roller
    at zmin), relaxed to steady state on the GPU; the zmax face reaction from
    the GPU assemble (reaction_force, solver.hpp:312-325) is within 5 % of
    E * strain * area, E = 9 kappa mu / (3 kappa + mu); the field is
    bit-identical to the oracle."""
    from paper_2106_14189_b200 import run_simulation
    spec = box_spec(kind="T4", divisions=3, extent=(0.1,) * 3, precision=8, mat=_nh_ref(), target=0.001,
                    fix_all_axes=False, safety=0.5)
    sc = Scenario(spec)
    t_total = 0.1
    steps_ramp = int(round(t_total / sc.dt))
    spec = box_spec(kind="T4", divisions=3, extent=(0.1,) * 3, precision=8, mat=_nh_ref(), target=0.001,
                    fix_all_axes=False, safety=0.5, ramp_steps=steps_ramp)
    sc = Scenario(spec)
    with GpuDjEngine(sc) as eng:
        res = run_simulation(eng, t_end=1.5)
        f, st = eng.assemble(res.u_curr)
    assert st["first_inverted"] == -1 and f is not None
    x = sc.image()["nodes"].reshape(-1, 3)
    top = np.flatnonzero(np.abs(x[:, 2] - 0.1) < 1e-12)
    reaction = f.reshape(-1, 3)[top, 2].sum()
    e_mod = 9.0 * 326210.0 * 6567.0 / (3.0 * 326210.0 + 6567.0)
    assert reaction == pytest.approx(e_mod * 0.01 * 0.1 * 0.1, rel=0.05)
    ur, _, rr = oracle.run(spec, res.steps, "oracle")
    assert np.array_equal(res.u_curr, ur)


def test_heavy_damping_decays_to_steady_state():
    """test_solver.cpp:168-190: with the relaxation damping the kinetic-energy
    proxy sum m |u - u_prev|^2 / dt^2 / 2 peaks and decays below 1e-12 of
    its peak after 1.2 s of a 20 % extension (all-axes fixed base)."""
    spec = box_spec(kind="T4", divisions=2, extent=(0.1,) * 3, precision=8, mat=_nh_ref(), target=0.02, safety=0.5)
    sc0 = Scenario(spec)
    spec = box_spec(kind="T4", divisions=2, extent=(0.1,) * 3, precision=8, mat=_nh_ref(), target=0.02, safety=0.5,
                    ramp_steps=int(round(0.1 / sc0.dt)))
    sc = Scenario(spec)
    mass = sc.image()["mass"]
    steps = int(np.ceil(1.2 / sc.dt))
    ke = []
    with GpuDjEngine(sc) as eng:
        for s in range(0, steps, 25):
            eng.step(min(25, steps - s))
            u, up, _ = eng.get_state()
            v = (u - up).reshape(-1, 3) / sc.dt
            ke.append(0.5 * float(np.sum(mass[:, None] * v * v)))
    assert max(ke) > 0 and ke[-1] < 1e-12 * max(ke)


def test_t_end_zero_returns_initial_field():
    """test_solver.cpp:107-119."""
    from paper_2106_14189_b200 import run_simulation
    spec = box_spec(kind="T4", divisions=1, extent=(0.1,) * 3, precision=8, mat=_nh_ref(), dt=1e-4)
    spec.c.bc_mode = 0
    with GpuDjEngine(Scenario(spec)) as eng:
        r = run_simulation(eng, t_end=0.0)
    assert r.steps == 0 and not np.any(r.u_curr)


@pytest.mark.parametrize("precision", [4, 8])
def test_advance_host_matches_device_loop(precision):
    """djg_advance_host (one step from a host SimState, u_prev upload
    overlapped with the element kernel) == the device-resident loop, bit for
    bit, step by step; a failing step hands back the unchanged state."""
    spec = box_spec(kind="T4", model="TI", divisions=5, precision=precision, ramp_steps=120)
    sc = Scenario(spec)
    with GpuDjEngine(sc) as ref:
        ref.step(120)
        u_ref, up_ref, _ = ref.get_state()
    with GpuDjEngine(sc) as eng:
        n3 = 3 * sc.num_nodes
        u, up = np.zeros(n3, spec.dtype), np.zeros(n3, spec.dtype)
        for s in range(120):
            un, rep = eng.advance_host(u, up, s)
            assert rep.status == 0 and rep.step == s + 1 and rep.steps_done == 1
            u, up = un, u
    assert np.array_equal(u, u_ref) and np.array_equal(up, up_ref)
    # inversion: status 4, state handed back unchanged
    inv = box_spec(kind="T4", divisions=2, extent=(0.1,) * 3, precision=8, target=-0.09, ramp_steps=2)
    with GpuDjEngine(Scenario(inv)) as e2:
        n3 = 3 * e2.num_nodes
        u, up = np.zeros(n3), np.zeros(n3)
        for s in range(40):
            un, rep = e2.advance_host(u, up, s)
            if rep.status:
                assert rep.status in (A.DJG_E_INVERSION, A.DJG_E_DIVERGENCE) and np.array_equal(un, u)
                break
            u, up = un, u
        else:
            pytest.fail("the crushing ramp never failed")


def test_advance_host_chunked_readback():
    """A mesh with >= 1024 node slices: the host-state step updates the nodes
    in 4 chunks whose results go back while the next chunk computes; same bits
    as the device loop."""
    spec = box_spec(kind="T4", model="NH", divisions=33, precision=4, target=0.01, ramp_steps=30)
    sc = Scenario(spec)
    assert (sc.num_nodes + 31) // 32 >= 1024
    with GpuDjEngine(sc) as ref:
        ref.step(30)
        u_ref, up_ref, _ = ref.get_state()
    with GpuDjEngine(sc) as eng:
        n3 = 3 * sc.num_nodes
        u, up = np.zeros(n3, np.float32), np.zeros(n3, np.float32)
        for s in range(30):
            un, rep = eng.advance_host(u, up, s)
            assert rep.status == 0
            u, up = un, u
    assert np.array_equal(u, u_ref) and np.array_equal(up, up_ref) and np.abs(u).max() > 0


@pytest.mark.parametrize("kind,model,d,prec", [("T4", "NH", (40, 41, 45), 4), ("T4", "TI", (12, 9, 33), 4),
                                                ("H8", "TI", (41, 40, 40), 4), ("T4", "NH", (5, 4, 6), 4),
                                                ("T4", "OT", (10, 11, 36), 8)])
@pytest.mark.parametrize("tled", [False, True])
def test_advance_host_fused_regions(kind, model, d, prec, tled):
    """The host-state step on the fused box step (advance_host_box): region
    by region (8 tapered runs of node layers when the box has >= 32 layers,
    else one launch) -- uploads, partial k_box_step launches, read-back --
    the same bits as the device-resident loop of the same engine and of the
    two-kernel step; an Abort step hands back the state."""
    if tled and kind == "H8":
        pytest.skip("TLED fused step: T4 only")
    flags = A.DJG_FLAG_FUSED | (A.DJG_FLAG_TLED if tled else 0)
    spec = box_spec(kind=kind, model=model, divisions=d, precision=prec, target=0.01, ramp_steps=25)
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=(A.DJG_FLAG_TLED if tled else 0) | A.DJG_FLAG_NO_FUSED) as ref:
        ref.step(25)
        u_ref, up_ref, _ = ref.get_state()
    with GpuDjEngine(sc, flags=flags) as eng:
        assert eng.info()["fused"] == 1
        n3 = 3 * sc.num_nodes
        u, up = np.zeros(n3, spec.dtype), np.zeros(n3, spec.dtype)
        for st in range(25):
            un, rep = eng.advance_host(u, up, st)
            assert rep.status == 0 and rep.step == st + 1
            u, up = un, u
    assert np.array_equal(u, u_ref) and np.array_equal(up, up_ref) and np.abs(u).max() > 0


@pytest.mark.parametrize("kind,prec,tled,off", [("T4", 4, False, 0), ("T4", 4, False, 1), ("T4", 4, True, 0),
                                                ("H8", 4, False, 0), ("T4", 8, False, 0)])
def test_advance_host_fused_pinned(kind, prec, tled, off):
    """The host-state step on page-locked host arrays (the bench's e2e
    shape), aligned and not: same bits as the device loop."""
    import torch
    flags = A.DJG_FLAG_FUSED | (A.DJG_FLAG_TLED if tled else 0)
    d = (40, 41, 45) if kind == "T4" else (41, 40, 40)
    spec = box_spec(kind=kind, model="TI", divisions=d, precision=prec, target=0.01, ramp_steps=12)
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=flags) as ref:
        ref.step(12)
        u_ref, up_ref, _ = ref.get_state()
    tdt = torch.float32 if prec == 4 else torch.float64
    n3 = 3 * sc.num_nodes
    # off = 1: rows not 16-byte aligned (the kernels' scalar path)
    bufs = [torch.zeros(n3 + 4, dtype=tdt).pin_memory()[off:n3 + off].numpy() for _ in range(3)]
    with GpuDjEngine(sc, flags=flags) as eng:
        u, up, nxt = bufs
        for st in range(12):
            _, rep = eng.advance_host(u, up, st, out=nxt)
            assert rep.status == 0 and rep.step == st + 1
            u, up, nxt = nxt, u, up
    assert np.array_equal(u, u_ref) and np.array_equal(up, up_ref) and np.abs(u).max() > 0


def test_advance_host_fused_inversion():
    """A crushing ramp through the fused host-state step: the same failing
    step, status and counts as the device loop; the state handed back."""
    spec = box_spec(kind="T4", divisions=(9, 7, 40), extent=(0.1, 0.1, 0.4), precision=4, target=-0.35,
                    ramp_steps=3, fix_all_axes=True, policy=A.DJG_ABORT)
    sc = Scenario(spec)
    with GpuDjEngine(sc, flags=A.DJG_FLAG_FUSED) as ref:
        rr = ref.step(60, raise_on_failure=False)
    assert rr.status != 0
    with GpuDjEngine(sc, flags=A.DJG_FLAG_FUSED) as eng:
        n3 = 3 * sc.num_nodes
        u, up = np.zeros(n3, np.float32), np.zeros(n3, np.float32)
        for st in range(60):
            un, rep = eng.advance_host(u, up, st)
            if rep.status:
                assert rep.status == rr.status and st == rr.step and rep.first_inverted == rr.first_inverted
                assert np.array_equal(un, u)
                break
            u, up = un, u
        else:
            pytest.fail("no failing step")


@pytest.mark.parametrize("kind,d", [("T4", 33), ("H8", 40)])
def test_advance_host_chunked_permuted_nodes(kind, d):
    """Chunked host-state step on a mesh whose node ids are randomly permuted:
    every element chunk reads nodes from the whole id range (each waits for
    the full u_curr upload); same bits as the device loop."""
    img = Scenario(box_spec(kind=kind, divisions=d, precision=4)).image()
    nodes, conn = img["nodes"].reshape(-1, 3).astype(np.float64), img["conn"].reshape(-1, 4 if kind == "T4" else 8)
    N = nodes.shape[0]
    perm = np.random.default_rng(11).permutation(N)
    nodes_p = np.empty_like(nodes)
    nodes_p[perm] = nodes
    conn_p = perm[conn].astype(np.int32)
    bottom = np.flatnonzero(nodes_p[:, 2] == 0.0)
    top = np.flatnonzero(nodes_p[:, 2] == nodes_p[:, 2].max())
    spec = mesh_spec(nodes_p, conn_p, kind=kind, precision=4, fixed=[(n, a) for n in bottom for a in range(3)],
                     prescribed=[(n, 2, 0.01, 1e-3) for n in top])
    sc = Scenario(spec)
    assert (sc.num_nodes + 31) // 32 >= 1024
    with GpuDjEngine(sc) as ref:
        ref.step(20)
        u_ref, up_ref, _ = ref.get_state()
    with GpuDjEngine(sc) as eng:
        n3 = 3 * sc.num_nodes
        u, up = np.zeros(n3, np.float32), np.zeros(n3, np.float32)
        for st in range(20):
            un, rep = eng.advance_host(u, up, st)
            assert rep.status == 0
            u, up = un, u
    assert np.array_equal(u, u_ref) and np.array_equal(up, up_ref) and np.abs(u).max() > 0


def test_descriptor_limits_fail_loudly():
    """32-bit slot indexing: more than INT32_MAX element-nodes is refused with
    a config error before any device work; so is an empty mesh."""
    spec = box_spec(kind="T4", divisions=2, precision=4)
    sc = Scenario(spec)
    lib = A.load_library()
    d = sc.desc(0, 0)
    d.num_elements = (1 << 31) // 4 + 1
    h = C.c_void_p()
    assert lib.djg_create(C.byref(d), C.byref(h)) == A.DJG_E_CONFIG
    assert b"32-bit" in lib.djg_create_error()
    d = sc.desc(0, 0)
    d.num_elements = 0
    assert lib.djg_create(C.byref(d), C.byref(h)) == A.DJG_E_CONFIG
    assert b"nodes and elements" in lib.djg_create_error()
