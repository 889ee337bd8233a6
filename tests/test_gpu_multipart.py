"""Multi-part step on one GPU: every part is a real engine running the real
kernels (local elements, owned nodes, halo pack/unpack, failure agreement);
the halo moves by device copies between the parts' buffers, so no kernel ever
waits on another. k parts must be bit-identical to one engine."""
import socket

import numpy as np
import pytest

import oracle
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, mesh_spec
from paper_2106_14189_b200 import _abi as A
from paper_2106_14189_b200.parallel import EmulatedParts

pytestmark = pytest.mark.gpu


def single(spec, steps):
    sc = Scenario(spec)
    with GpuDjEngine(sc) as eng:
        rep = eng.step(steps, raise_on_failure=False)
        u, up, st = eng.get_state()
    return u, up, rep


@pytest.mark.parametrize("overlap", [False, True], ids=["sequential", "overlapped"])
@pytest.mark.parametrize("nparts", [2, 3, 4, 8])
@pytest.mark.parametrize("kind,model,prec", [("T4", "NH", 4), ("H8", "TI", 4), ("T4", "MR", 8)])
def test_parts_bitwise_equal_single_gpu(nparts, kind, model, prec, overlap):
    """k parts == 1 GPU bit for bit, with the halo exchanged after the step or
    (overlapped) at the next step's start, behind the interior elements."""
    spec = box_spec(kind=kind, model=model, divisions=8, precision=prec, ramp_steps=200)
    u1, up1, r1 = single(spec, 200)
    em = EmulatedParts(Scenario(spec), nparts)
    reps = em.step(200, overlap=overlap)
    u, up, step = em.global_state()
    em.close()
    assert step == 200 == r1.step and all(r.step == 200 and r.status == 0 for r in reps)
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("cfg,nparts,steps", [("cfg1", 2, 400), ("cfg1", 4, 400), ("cfg1", 8, 400),
                                              ("cfg3", 8, 40)])
def test_parts_cfg_bitwise(cfg, nparts, steps, prec):
    """1 GPU == k parts bit for bit on cfg1 / cfg3, f32 and f64
    (overlapped step, peer-memory transport for k = 8)."""
    from paper_2106_14189_b200 import config_spec
    spec = config_spec(cfg, precision=prec)
    u1, up1, r1 = single(spec, steps)
    em = EmulatedParts(Scenario(spec), nparts, transport="p2p" if nparts == 8 else "copy")
    reps = em.step(steps, overlap=True) if nparts != 8 else em.step(steps)
    u, up, step = em.global_state()
    em.close()
    assert all(r.status == 0 for r in reps) and step == steps == r1.step
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


@pytest.mark.parametrize("nparts", [2, 3, 8])
@pytest.mark.parametrize("kind,model,prec", [("T4", "NH", 4), ("H8", "TI", 8)])
def test_parts_peer_memory_transport_bitwise(nparts, kind, model, prec):
    """The peer-memory step (node kernel stores the halo into the other parts'
    buffers, mailbox agreement): k parts == 1 GPU bit for bit."""
    spec = box_spec(kind=kind, model=model, divisions=7, precision=prec, ramp_steps=150)
    u1, up1, r1 = single(spec, 150)
    em = EmulatedParts(Scenario(spec), nparts, transport="p2p")
    reps = em.step(150)
    u, up, step = em.global_state()
    em.close()
    assert all(r.status == 0 for r in reps) and step == 150
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


def test_parts_metis_partition_bitwise():
    """Graph (METIS k-way) partitions: same bits as one GPU, overlapped step."""
    for kind, model in (("T4", "NH"), ("H8", "OT")):
        spec = box_spec(kind=kind, model=model, divisions=7, precision=4, ramp_steps=150)
        u1, up1, r1 = single(spec, 150)
        for nparts, transport in ((3, "copy"), (8, "copy"), (5, "p2p")):
            em = EmulatedParts(Scenario(spec), nparts, method="metis", transport=transport)
            reps = em.step(150, overlap=transport == "copy")
            u, up, step = em.global_state()
            em.close()
            assert all(r.status == 0 for r in reps) and step == 150
            assert np.array_equal(u, u1) and np.array_equal(up, up1)


@pytest.mark.parametrize("transport", ["copy", "p2p"])
@pytest.mark.parametrize("nparts", [2, 3, 8])
@pytest.mark.parametrize("kind,model,prec", [("T4", "NH", 4), ("H8", "TI", 8)])
def test_parts_box_local_bitwise(kind, model, prec, nparts, transport):
    """Parts built part-locally from the box spec (no global mesh or problem,
    Partition.box_local): bit-identical to one engine."""
    spec = box_spec(kind=kind, model=model, divisions=(9, 7, 8), precision=prec, ramp_steps=150)
    u1, up1, r1 = single(spec, 150)
    em = EmulatedParts(spec, nparts, method="box-local", transport=transport)
    reps = em.step(150, overlap=transport == "copy")
    u, up, step = em.global_state()
    em.close()
    assert all(r.status == 0 for r in reps) and step == 150
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


@pytest.mark.parametrize("overlap", [False, True, "p2p"], ids=["sequential", "overlapped", "peer-memory"])
def test_parts_agree_on_inversion(overlap):
    """The crushing case of test_solver.cpp:214-241 split in two: every part
    halts at the same state, reporting the same (global) element."""
    sc0 = Scenario(box_spec(kind="T4", divisions=2, extent=(0.1, 0.1, 0.1), precision=8))
    img = sc0.image()
    nodes, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
    bottom = [n for n in range(len(nodes)) if nodes[n, 2] == 0.0]
    top = [n for n in range(len(nodes)) if nodes[n, 2] == nodes[:, 2].max()]
    spec = mesh_spec(nodes, conn, kind="T4", precision=8, fixed=[(n, a) for n in bottom for a in range(3)],
                     prescribed=[(n, 2, -0.5, 1e-4) for n in top], dt=1e-4, alpha=0.0)
    u1, up1, r1 = single(spec, 100)
    ur, upr, rr = oracle.run(spec, 100, "oracle")
    assert r1.status == A.DJG_E_INVERSION and r1.first_inverted == rr["first_inverted"]
    if overlap == "p2p":
        em = EmulatedParts(Scenario(spec), 2, transport="p2p")
        reps = em.step(100)
    else:
        em = EmulatedParts(Scenario(spec), 2)
        reps = em.step(100, overlap=overlap)
    u, up, step = em.global_state()
    em.close()
    for r in reps:
        assert r.status == A.DJG_E_INVERSION
        assert r.first_inverted == r1.first_inverted and r.step == r1.step
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


@pytest.mark.parametrize("nparts", [2, 3, 4])
@pytest.mark.parametrize("transport", ["sequential", "overlapped", "p2p"])
def test_parts_skip_and_report_counts(nparts, transport):
    """SkipAndReport over a crushing load: elements invert on several steps,
    some of them ghosts held by more than one part. Every part reports the
    single-GPU (= reference) inverted_count and inverted_steps: an inversion
    is counted only on the part that owns the element and the step counts are
    summed by the agreement."""
    sc0 = Scenario(box_spec(kind="T4", divisions=4, extent=(0.1, 0.1, 0.1), precision=8))
    img = sc0.image()
    nodes, conn = img["nodes"].reshape(-1, 3), img["conn"].reshape(-1, 4)
    bottom = [n for n in range(len(nodes)) if nodes[n, 2] == 0.0]
    top = [n for n in range(len(nodes)) if nodes[n, 2] == nodes[:, 2].max()]
    spec = mesh_spec(nodes, conn, kind="T4", precision=8, fixed=[(n, a) for n in bottom for a in range(3)],
                     prescribed=[(n, 2, -0.35, 2e-4) for n in top], dt=1e-5, alpha=0.0,
                     policy=A.DJG_SKIP_AND_REPORT)
    steps = 60
    u1, up1, r1 = single(spec, steps)
    ur, upr, rr = oracle.run(spec, steps, "oracle")
    assert (r1.inverted_count, r1.inverted_steps, r1.status) == (rr["inverted_count"], rr["inverted_steps"],
                                                                 rr["status"])
    assert r1.inverted_count > r1.inverted_steps > 1, r1  # several elements on several steps
    if transport == "p2p":
        em = EmulatedParts(Scenario(spec), nparts, transport="p2p")
        reps = em.step(steps)
    else:
        em = EmulatedParts(Scenario(spec), nparts)
        reps = em.step(steps, overlap=transport == "overlapped")
    u, up, step = em.global_state()
    em.close()
    for r in reps:
        assert (r.inverted_count, r.inverted_steps, r.status, r.step) == \
            (r1.inverted_count, r1.inverted_steps, r1.status, r1.step), (r, r1)
    assert np.array_equal(u, u1) and np.array_equal(up, up1)


def test_peer_setup_rejects_out_of_range_destinations():
    """djg_peer_setup bounds-checks every halo destination against the peer's
    node count before any peer store can run."""
    from paper_2106_14189_b200.engine import ConfigError
    from paper_2106_14189_b200.parallel import _halo, peer_destinations
    spec = box_spec(kind="T4", divisions=4, precision=4, ramp_steps=50)
    em = EmulatedParts(Scenario(spec), 2, transport="p2p")
    try:
        ptrs = [e.peer_export() for e in em.engs]
        halos = [_halo(p) for p in em.parts]
        node, part, index = peer_destinations(halos, 0)
        assert len(index) > 0
        counts = [h[5] for h in halos]
        bad = list(index)
        bad[0] = counts[part[0]]  # one past the peer's last node
        with pytest.raises(ConfigError, match="outside the peer"):
            em.engs[0].peer_setup(2, 0, ptrs, (node, part, bad), counts)
        with pytest.raises(ConfigError, match="node counts"):
            em.engs[0].peer_setup(2, 0, ptrs, (node, part, index), [counts[0] + 1, counts[1]])
    finally:
        em.close()


def test_peer_wait_is_bounded(monkeypatch):
    """A part whose peer never posts its step: the agreement kernel gives up
    after DJG_PEER_TIMEOUT_MS and halts the part with DJG_E_PEER instead of
    spinning on the GPU (one kernel waits here, on a flag no kernel will
    write: nothing else has to run concurrently)."""
    monkeypatch.setenv("DJG_PEER_TIMEOUT_MS", "200")
    spec = box_spec(kind="T4", divisions=4, precision=4, ramp_steps=50)
    em = EmulatedParts(Scenario(spec), 2, transport="p2p")
    try:
        e0 = em.engs[0]
        e0.step_peer_local()
        e0.sync()
        e0.step_peer_agree()
        r = e0.sync()
        assert r.status == A.DJG_E_PEER, r
        e0.step_async(3)  # a halted part runs no further steps
        assert e0.sync().status == A.DJG_E_PEER
    finally:
        em.close()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("engine_comm", [True, False, "p2p"], ids=["engine-nccl", "python-driver", "peer-memory"])
def test_distributed_engine_single_rank_nccl(engine_comm):
    """The torch.distributed (NCCL) driver on one rank: same bits as the
    plain engine (the halo is empty, the status allreduce is real). With
    engine_comm the engine's own NCCL communicator runs inside its CUDA
    graphs (djg_comm_init)."""
    import torch
    import torch.distributed as dist
    from paper_2106_14189_b200.parallel import DistributedEngine
    spec = box_spec(kind="H8", model="NH", divisions=6, precision=4, ramp_steps=100)
    u1, _, _ = single(spec, 100)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        kw = dict(transport="p2p") if engine_comm == "p2p" else dict(engine_comm=engine_comm)
        de = DistributedEngine(Scenario(spec), device=0, **kw)
        r = de.step(100)
        U, UP, step = de.gather_global()
        assert r.status == 0 and step == 100
        assert np.array_equal(U, u1)
        # failure agreement through the allreduce: an inverting problem halts
        # at the same step and element as the plain engine
        inv = box_spec(kind="T4", divisions=3, extent=(0.1,) * 3, precision=8, target=-0.09, ramp_steps=3,
                       fix_all_axes=True)
        with GpuDjEngine(Scenario(inv)) as e1:
            r1 = e1.step(50, raise_on_failure=False)
        de2 = DistributedEngine(Scenario(inv), device=0, **kw)
        r2 = de2.step(50, raise_on_failure=False)
        assert r1.status in (A.DJG_E_INVERSION, A.DJG_E_DIVERGENCE)
        assert r1.status == r2.status and r1.fail_step == r2.fail_step and r1.first_inverted == r2.first_inverted
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", [4, 8])
def test_halo_pack_unpack_against_host_indexing(prec):
    """SURVEY §8(e) halo-only unit test: djg_halo_pack gathers exactly the
    current displacements of the part's send list (host re-assembly from the
    global state through node_l2g), and djg_halo_unpack writes exactly the
    receive list."""
    import torch
    from paper_2106_14189_b200.parallel import Partition, PartEngine
    spec = box_spec(kind="T4", model="NH", divisions=6, precision=prec)
    sc = Scenario(spec)
    rng = np.random.default_rng(5)
    dt = np.float32 if prec == 4 else np.float64
    tdt = torch.float32 if prec == 4 else torch.float64
    ug = rng.uniform(-1, 1, 3 * sc.num_nodes).astype(dt)
    upg = rng.uniform(-1, 1, 3 * sc.num_nodes).astype(dt)
    for me in range(3):
        part = Partition(sc, 3, me)
        with PartEngine(part) as pe:
            for step in (0, 1, 2):  # every buffer phase
                pe.set_global_state(ug, upg, step)
                ns, nr = part.send_nodes.size, part.recv_nodes.size
                assert ns > 0 and nr > 0
                buf = torch.zeros((ns, 4), dtype=tdt, device="cuda")
                pe.halo_pack(buf.data_ptr())
                torch.cuda.synchronize()
                want = ug.reshape(-1, 3)[part.node_l2g[part.send_nodes]]
                assert np.array_equal(buf.cpu().numpy()[:, :3], want)
                vals = torch.from_numpy(rng.uniform(-1, 1, (nr, 4)).astype(dt)).cuda()
                pe.halo_unpack(vals.data_ptr())
                torch.cuda.synchronize()
                u, up, st = pe.get_state()
                u = u.reshape(-1, 3)
                assert np.array_equal(u[part.recv_nodes], vals.cpu().numpy()[:, :3]) and st == step
                others = np.setdiff1d(np.arange(part.num_nodes), part.recv_nodes)
                assert np.array_equal(u[others], ug.reshape(-1, 3)[part.node_l2g[others]])
