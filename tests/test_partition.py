"""Multi-GPU decomposition checked on the CPU: partition and
halo invariants, and a world_size-2 gloo run of the partitioned step
(oracle element forces, ordered gather, central difference, halo exchange)
that must be bit-identical to the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2106_14189_b200 import Scenario, box_spec
from paper_2106_14189_b200 import _abi as A
from paper_2106_14189_b200.parallel import Partition, element_parts


@pytest.mark.parametrize("method", ["rcb", "metis"])
@pytest.mark.parametrize("kind", ["T4", "H8"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
def test_partition_invariants(kind, nparts, method):
    sc = Scenario(box_spec(kind=kind, divisions=(6, 5, 7), precision=4))
    img = sc.image()
    npe = sc.npe
    conn = img["conn"].reshape(-1, npe)
    parts = [Partition(sc, nparts, p, method) for p in range(nparts)]
    # owned nodes: an exact cover of the mesh
    owned = np.concatenate([p.node_l2g[: p.num_owned] for p in parts])
    assert np.array_equal(np.sort(owned), np.arange(sc.num_nodes))
    owner = np.empty(sc.num_nodes, np.int64)
    for i, p in enumerate(parts):
        owner[p.node_l2g[: p.num_owned]] = i
    ep = element_parts(sc, nparts, method)
    counts = np.bincount(ep, minlength=nparts)
    if method == "rcb":
        assert counts.min() >= sc.num_elements // nparts - 1
    else:  # METIS k-way: within its default 3 % imbalance, every part non-empty
        assert counts.min() > 0 and counts.max() <= 1.031 * sc.num_elements / nparts + 1
    for i, p in enumerate(parts):
        # local elements: exactly those touching an owned node; interior ones
        # (no ghost node) first, then boundary ones, each ascending global id
        want = np.flatnonzero((owner[conn] == i).any(axis=1))
        assert np.array_equal(np.sort(p.elem_l2g), want)
        ni = p.info["interior_elements"]
        interior = (owner[conn[p.elem_l2g]] == i).all(axis=1)
        assert interior[:ni].all() and not interior[ni:].any()
        assert np.all(np.diff(p.elem_l2g[:ni]) > 0) and np.all(np.diff(p.elem_l2g[ni:]) > 0)
        # ghosts: the other nodes of those elements, ascending
        ghosts = np.setdiff1d(np.unique(conn[want]), p.node_l2g[: p.num_owned])
        assert np.array_equal(p.node_l2g[p.num_owned:], ghosts)
        # owned nodes have their complete CSR rows locally
        limg = p.image()
        loff = limg["csr_offsets"]
        for n in range(p.num_owned):
            g = p.node_l2g[n]
            assert loff[n + 1] - loff[n] == img["csr_offsets"][g + 1] - img["csr_offsets"][g]
            # ... in ascending GLOBAL element id (the summation order)
            row = p.elem_l2g[limg["csr_elem"][loff[n]:loff[n + 1]]]
            assert np.array_equal(row, img["csr_elem"][img["csr_offsets"][g]:img["csr_offsets"][g + 1]])
    # halo symmetry: what p sends q is what q receives from p, in the same order
    for i, p in enumerate(parts):
        for k, q in enumerate(p.neighbors.tolist()):
            pq = parts[q]
            j = pq.neighbors.tolist().index(i)
            sent = p.node_l2g[p.send_nodes[p.send_off[k]:p.send_off[k + 1]]]
            got = pq.node_l2g[pq.recv_nodes[pq.recv_off[j]:pq.recv_off[j + 1]]]
            assert np.array_equal(sent, got) and np.all(np.diff(sent) > 0)
            assert np.all(owner[got] == i)


def test_partition_is_deterministic():
    sc = Scenario(box_spec(kind="T4", divisions=7, precision=8))
    a = element_parts(sc, 8)
    b = element_parts(Scenario(box_spec(kind="T4", divisions=7, precision=8)), 8)
    assert np.array_equal(a, b)
    m1 = element_parts(sc, 8, "metis")
    m2 = element_parts(Scenario(box_spec(kind="T4", divisions=7, precision=8)), 8, "metis")
    assert np.array_equal(m1, m2)
    p1, p2 = Partition(sc, 8, 5), Partition(sc, 8, 5)
    assert np.array_equal(p1.node_l2g, p2.node_l2g) and np.array_equal(p1.send_nodes, p2.send_nodes)


# ----------------------------------------------------------------- gloo run

def _cpu_part_steps(part: Partition, spec, steps, exchange):
    """advance_step restricted to one part, in the reference's arithmetic:
    oracle element forces, per-node left-fold gather in CSR order, central
    difference with BCs, then the halo exchange of owned boundary nodes."""
    img = part.image()
    npe, nc, R = part.npe, part.nconst, part.dtype
    conn = img["conn"].reshape(-1, npe)
    consts = img["consts"].reshape(-1, nc)
    off, ce, cl = img["csr_offsets"], img["csr_elem"], img["csr_local"]
    kinds, tgt, ttot = img["dof_kind"], img["dof_target"], img["dof_t_total"]
    c1, massless = img["c1"], img["massless"]
    sc = part.scenario.scalars
    c2, c3, dt = R(sc["c2"]), R(sc["c3"]), R(sc["dt"])
    u = np.zeros((part.num_nodes, 3), R)
    up = np.zeros_like(u)
    mat = spec.c.material
    for step in range(steps):
        rows = np.stack([oracle.element_force_rec(spec.precision, spec.c.kind, mat, consts[e], u[conn[e]])
                         .reshape(npe, 3) for e in range(len(conn))])
        un = np.zeros_like(u)
        t_next = dt * R(step + 1)
        for n in range(part.num_owned):
            f = [R(0), R(0), R(0)]
            for p in range(off[n], off[n + 1]):
                for i in range(3):
                    f[i] = R(f[i] + rows[ce[p], cl[p], i])
            for i in range(3):
                k = kinds[3 * n + i]
                if k == A.DJG_FIXED:
                    v = R(0)
                elif k == A.DJG_PRESCRIBED:
                    s = R(t_next / ttot[3 * n + i])
                    v = R((R(1) if s >= R(1) else s) * tgt[3 * n + i])
                elif massless[n]:
                    v = R(0)
                else:
                    v = R(R(R(c1[n] * R(R(0) - f[i])) + R(c2 * u[n, i])) + R(c3 * up[n, i]))
                un[n, i] = v
        exchange(un)
        up, u = u, un
    return u[: part.num_owned], up[: part.num_owned]


def _gloo_worker(rank, world, port, q, method="rcb"):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec = box_spec(kind="T4", model="TI", divisions=3, precision=4, ramp_steps=40)
    sc = Scenario(spec)
    part = Partition(sc, world, rank, method)

    def exchange(un):
        reqs, bufs = [], []
        for k, nb in enumerate(part.neighbors.tolist()):
            s = un[part.send_nodes[part.send_off[k]:part.send_off[k + 1]]]
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(s)), nb))
            r = torch.zeros((part.recv_off[k + 1] - part.recv_off[k], 3), dtype=torch.float32)
            reqs.append(dist.irecv(r, nb))
            bufs.append((k, r))
        for w in reqs:
            w.wait()
        for k, r in bufs:
            un[part.recv_nodes[part.recv_off[k]:part.recv_off[k + 1]]] = r.numpy()

    u, up = _cpu_part_steps(part, spec, 40, exchange)
    q.put((rank, part.node_l2g[: part.num_owned], u, up))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("method", ["rcb", "metis"])
def test_gloo_two_ranks_bitwise_equal_single_process(method):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q, method)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = box_spec(kind="T4", model="TI", divisions=3, precision=4, ramp_steps=40)
    ur, upr, _ = oracle.run(spec, 40, "oracle")
    ur, upr = ur.reshape(-1, 3), upr.reshape(-1, 3)
    covered = np.zeros(len(ur), bool)
    for rank, ids, u, up in res:
        assert np.array_equal(u, ur[ids]) and np.array_equal(up, upr[ids])
        covered[ids] = True
    assert covered.all() and np.abs(ur).max() > 0.05


@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("kind,model", [("T4", "NH"), ("H8", "TI"), ("T4", "OT")])
@pytest.mark.parametrize("nparts", [1, 2, 3, 5, 8])
def test_box_local_build_equals_global_extraction(kind, model, nparts, prec):
    """Partition.box_local builds part p of the box partition from the spec
    alone; it must equal the part djg_partition_build_method(DJG_PART_BOX)
    extracts from the global problem: maps, halo lists, element ownership,
    local connectivity, coordinates, records and CSR, and on every owned
    node the mass, update coefficient and BCs (ghost-node masses are partial
    locally and never used: only owned nodes are updated)."""
    spec = box_spec(kind=kind, model=model, divisions=(7, 5, 6), precision=prec, ramp_steps=100)
    sc = Scenario(spec)
    parts = [Partition.box_local(spec, nparts, p) for p in range(nparts)]
    for p in range(nparts):
        glob = Partition(sc, nparts, p, "box")
        loc = Partition.box_local(spec, nparts, p,
                                  reduce_min=lambda x: _global_lmin(spec, nparts))
        assert loc.info == glob.info
        for f in ("node_l2g", "elem_l2g", "elem_owned", "neighbors", "send_off", "recv_off", "send_nodes",
                  "recv_nodes"):
            assert np.array_equal(getattr(loc, f), getattr(glob, f)), f
        a, b = loc.image(), glob.image()
        no = loc.num_owned
        for f in ("nodes", "conn", "csr_offsets", "csr_elem", "csr_local", "consts"):
            assert np.array_equal(a[f], b[f]), f
        for f in ("mass", "c1", "massless"):
            assert np.array_equal(a[f][:no], b[f][:no]), f
        for f in ("dof_kind", "dof_target", "dof_t_total"):
            assert np.array_equal(a[f][: 3 * no], b[f][: 3 * no]), f
        da, db = loc.desc(), glob.desc()
        for f in ("dt", "c2", "c3"):
            assert getattr(da, f) == getattr(db, f), f
    # every element is owned by exactly one part; owned nodes cover the mesh
    owned = np.concatenate([p.node_l2g[: p.num_owned] for p in parts])
    assert np.array_equal(np.sort(owned), np.arange(sc.num_nodes))
    oe = np.concatenate([p.elem_l2g[p.elem_owned.astype(bool)] for p in parts])
    assert np.array_equal(np.sort(oe), np.arange(sc.num_elements))


def _global_lmin(spec, nparts):
    """min over the parts of their local minimum characteristic length (what
    a rank obtains with an allreduce(MIN))."""
    out = []
    for p in range(nparts):
        h = A.C.c_void_p()
        x = A.C.c_double()
        assert A.load_library().djg_partition_build_box(spec.ref(), nparts, p, A.C.byref(h), A.C.byref(x)) == 0
        A.load_library().djg_partition_free(h)
        out.append(x.value)
    return min(out)
