"""Multi-GPU DJ-TLED step: one process (rank) per GPU.

The mesh is split by the native host partitioner (include/djg_host.h,
djg_partition_*): each rank owns a set of nodes, computes every element that
touches them (ghost elements included) in ascending global element id, and
after each step exchanges the fresh displacement of boundary nodes with its
neighbors. Owned nodes sum exactly the rows a single GPU sums, in the same
order, so a k-rank run is bit-identical to the 1-GPU run.

Per step, all enqueued on the engine's CUDA stream (no host synchronisation):
  djg_step_async(1) -> djg_halo_pack -> NCCL send/recv with each neighbor ->
  djg_halo_unpack -> djg_step_status -> NCCL allreduce (MAX; SUM of the counts) -> djg_step_agree

`EmulatedParts` runs all parts in one process on one device, exchanging the
halo with device copies (no kernel ever waits on another): it is how the
multi-part path is tested on a single GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .engine import ConfigError, GpuDjEngine, Scenario, StepReport, raise_for


def _lib():
    return A.load_library()


class Partition:
    """Host-side local problem of part `part` of `nparts`: extracted from a
    built global Scenario, or (Partition.box_local) built alone from a box
    spec without the global mesh."""

    def __init__(self, scenario: Scenario, nparts: int, part: int, method: str = "rcb"):
        self.scenario = scenario
        h = C.c_void_p()
        if _lib().djg_partition_build_method(scenario._h, nparts, part, A.PART_METHODS[method], C.byref(h)) != A.DJG_OK:
            raise ConfigError(_lib().djg_scenario_error().decode())
        self._load(h, scenario.dtype, scenario.npe, scenario.nconst)
        self.dt = scenario.dt

    @classmethod
    def box_local(cls, spec, nparts: int, part: int, reduce_min=None) -> "Partition":
        """Part `part` of the box partition (DJG_PART_BOX) of a generated-box
        spec, built from the spec alone (djg_partition_build_box): the rank's
        host memory and setup time scale with its part, not the mesh.
        reduce_min(x) returns the minimum of x over all parts (the global
        minimum characteristic length behind dt); None for a single part."""
        obj = cls.__new__(cls)
        obj.scenario = None
        h = C.c_void_p()
        lmin = C.c_double()
        if _lib().djg_partition_build_box(spec.ref(), nparts, part, C.byref(h), C.byref(lmin)) != A.DJG_OK:
            raise ConfigError(_lib().djg_scenario_error().decode())
        g = reduce_min(lmin.value) if reduce_min is not None else lmin.value
        if _lib().djg_partition_finish(h, g) != A.DJG_OK:
            _lib().djg_partition_free(h)
            raise ConfigError(_lib().djg_scenario_error().decode())
        obj._load(h, spec.dtype, spec.npe, A.const_count(spec.c.kind, spec.c.material.model))
        obj.dt = obj.desc().dt
        return obj

    @classmethod
    def box_local_all(cls, spec, nparts: int) -> list["Partition"]:
        """Every part of the box partition built part-locally in one process
        (single-device emulation): the minimum characteristic length is
        reduced over the parts' own builds, as ranks would with allreduce."""
        hs, mins = [], []
        for p in range(nparts):
            h = C.c_void_p()
            lmin = C.c_double()
            if _lib().djg_partition_build_box(spec.ref(), nparts, p, C.byref(h), C.byref(lmin)) != A.DJG_OK:
                raise ConfigError(_lib().djg_scenario_error().decode())
            hs.append(h)
            mins.append(lmin.value)
        out = []
        for h in hs:
            if _lib().djg_partition_finish(h, min(mins)) != A.DJG_OK:
                raise ConfigError(_lib().djg_scenario_error().decode())
            obj = cls.__new__(cls)
            obj.scenario = None
            obj._load(h, spec.dtype, spec.npe, A.const_count(spec.c.kind, spec.c.material.model))
            obj.dt = obj.desc().dt
            out.append(obj)
        return out

    def _load(self, h, dtype, npe: int, nconst: int):
        self._h = h
        i = A.djg_partition_info()
        _lib().djg_partition_get_info(self._h, C.byref(i))
        self.info = {name: getattr(i, name) for name, _ in i._fields_}
        nb = max(i.num_neighbors, 0)
        self.neighbors = np.zeros(nb, np.int32)
        self.send_off = np.zeros(nb + 1, np.int64)
        self.recv_off = np.zeros(nb + 1, np.int64)
        self.send_nodes = np.zeros(i.send_total, np.int32)
        self.recv_nodes = np.zeros(i.recv_total, np.int32)
        _lib().djg_partition_halo(self._h, A.ptr(self.neighbors), A.ptr(self.send_off), A.ptr(self.recv_off),
                                  A.ptr(self.send_nodes), A.ptr(self.recv_nodes))
        self.node_l2g = np.zeros(i.num_nodes, np.int64)
        self.elem_l2g = np.zeros(i.num_elements, np.int64)
        _lib().djg_partition_maps(self._h, A.ptr(self.node_l2g), A.ptr(self.elem_l2g))
        self.elem_owned = np.zeros(i.num_elements, np.uint8)  # elements this part reports inversions of
        _lib().djg_partition_owned_elements(self._h, A.ptr(self.elem_owned))
        self.num_owned = i.num_owned
        self.num_nodes = i.num_nodes
        self.num_elements = i.num_elements
        self.dtype = dtype
        self.npe = npe
        self.nconst = nconst

    def image(self) -> dict:
        n, e, npe, nc, dt = self.num_nodes, self.num_elements, self.npe, self.nconst, self.dtype
        img = {
            "nodes": np.zeros(3 * n, dt), "conn": np.zeros(npe * e, np.int32),
            "csr_offsets": np.zeros(n + 1, np.int64), "csr_elem": np.zeros(npe * e, np.int64),
            "csr_local": np.zeros(npe * e, np.int32), "consts": np.zeros(e * nc, dt),
            "mass": np.zeros(n, dt), "c1": np.zeros(n, dt), "massless": np.zeros(n, np.uint8),
            "dof_kind": np.zeros(3 * n, np.uint8), "dof_target": np.zeros(3 * n, dt),
            "dof_t_total": np.zeros(3 * n, dt),
        }
        p = A.djg_image_ptrs()
        for k, v in img.items():
            setattr(p, k, v.ctypes.data_as(C.c_void_p))
        _lib().djg_partition_image(self._h, C.byref(p))
        return img

    def desc(self, device: int = 0, flags: int = 0) -> A.djg_desc:
        d = A.djg_desc()
        _lib().djg_partition_desc(self._h, device, C.byref(d))
        d.flags = flags
        return d

    def close(self):
        if getattr(self, "_h", None):
            _lib().djg_partition_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def element_parts(scenario: Scenario, nparts: int, method: str = "rcb") -> np.ndarray:
    out = np.zeros(scenario.num_elements, np.int32)
    if _lib().djg_element_parts_method(scenario._h, nparts, A.PART_METHODS[method], A.ptr(out)) != A.DJG_OK:
        raise ConfigError(_lib().djg_scenario_error().decode())
    return out


class PartEngine(GpuDjEngine):
    """GpuDjEngine on a part's local problem, with its halo lists."""

    def __init__(self, part: Partition, device: int = 0, flags: int = 0):
        self.scenario = part  # duck-typed: desc(), dtype, num_nodes, num_elements, npe, dt
        self.part = part
        self.dtype = part.dtype
        self.num_nodes = part.num_nodes
        self.num_elements = part.num_elements
        h = C.c_void_p()
        d = part.desc(device, flags)
        if _lib().djg_create(C.byref(d), C.byref(h)) != A.DJG_OK:
            raise ConfigError(_lib().djg_create_error().decode())
        self._h = h
        self._check(_lib().djg_set_partition(self._h, part.num_owned, A.ptr(part.elem_l2g)))
        self._check(_lib().djg_set_halo(self._h, part.send_nodes.size, A.ptr(part.send_nodes),
                                        part.recv_nodes.size, A.ptr(part.recv_nodes)))
        self._check(_lib().djg_set_interior(self._h, part.info["interior_elements"]))
        self._check(_lib().djg_set_counted_elements(self._h, A.ptr(part.elem_owned)))

    def set_global_state(self, u_curr=None, u_prev=None, step: int = 0):
        l2g = self.part.node_l2g
        loc = lambda g: None if g is None else np.asarray(g, self.dtype).reshape(-1, 3)[l2g].reshape(-1)
        self.set_state(loc(u_curr), loc(u_prev), step)

    def owned_state(self):
        u, up, step = self.get_state()
        n = self.part.num_owned
        return u.reshape(-1, 3)[:n], up.reshape(-1, 3)[:n], step

    def halo_pack(self, dev_ptr: int):
        self._check(_lib().djg_halo_pack(self._h, C.c_void_p(dev_ptr)))

    def halo_unpack(self, dev_ptr: int):
        self._check(_lib().djg_halo_unpack(self._h, C.c_void_p(dev_ptr)))

    # -- peer-memory transport (djg_peer_*)
    def peer_export(self) -> list[int]:
        out = (C.c_void_p * 4)()
        self._check(_lib().djg_peer_export(self._h, out))
        return [int(v or 0) for v in out]

    def peer_ipc_export(self) -> bytes:
        buf = C.create_string_buffer(4 * 64)
        self._check(_lib().djg_peer_ipc_export(self._h, buf))
        return buf.raw

    def peer_ipc_open(self, handles: bytes) -> list[int]:
        out = (C.c_void_p * 4)()
        self._check(_lib().djg_peer_ipc_open(self._h, C.create_string_buffer(handles, 4 * 64), out))
        return [int(v or 0) for v in out]

    def peer_setup(self, nparts: int, part: int, ptrs: list[list[int]], dests, num_nodes):
        """ptrs[q]: part q's 4 device pointers; dests: peer_destinations();
        num_nodes[q]: part q's local node count (the destination bounds)."""
        peer_u = (C.c_void_p * (3 * nparts))(*[p[i] for p in ptrs for i in range(3)])
        peer_mail = (C.c_void_p * nparts)(*[p[3] for p in ptrs])
        counts = np.ascontiguousarray(num_nodes, np.int64)
        node, dpart, index = (np.ascontiguousarray(a, np.int32) for a in dests)
        self._check(_lib().djg_peer_setup(self._h, nparts, part, peer_u, peer_mail, A.ptr(counts), int(node.size),
                                          A.ptr(node), A.ptr(dpart), A.ptr(index)))

    def step_peer_local(self):
        self._check(_lib().djg_step_peer_local(self._h))

    def step_peer_agree(self):
        self._check(_lib().djg_step_peer_agree(self._h))

    def step_interior(self):
        self._check(_lib().djg_step_interior(self._h))

    def step_boundary(self):
        self._check(_lib().djg_step_boundary(self._h))

    def step_status(self, dev_ptr: int):
        self._check(_lib().djg_step_status(self._h, C.c_void_p(dev_ptr)))

    def step_agree(self, dev_ptr: int):
        self._check(_lib().djg_step_agree(self._h, C.c_void_p(dev_ptr)))


def peer_destinations(halos: list, me: int):
    """Halo destinations of part `me` for the peer-memory transport: owned
    node i of my send block to part q lands on q's ghost node at the same
    position of q's receive block from me (the blocks list the same global
    nodes in the same order). halos[q] = (neighbors, send_off, recv_off,
    send_nodes, recv_nodes) of part q."""
    nb, s_off, _, s_nodes, _ = halos[me][:5]
    node, part, index = [], [], []
    for k, q in enumerate(list(nb)):
        qnb, _, q_roff, _, q_rnodes = halos[q][:5]
        j = list(qnb).index(me)
        send = s_nodes[s_off[k]:s_off[k + 1]]
        recv = q_rnodes[q_roff[j]:q_roff[j + 1]]
        assert len(send) == len(recv)
        node.extend(send.tolist())
        part.extend([q] * len(send))
        index.extend(recv.tolist())
    return node, part, index


def _spec_of(scenario):
    """The Spec behind a Scenario (or a Spec itself): the part-local build
    reads only the box spec."""
    return getattr(scenario, "spec", scenario)


def _halo(p: "Partition"):
    return (p.neighbors.copy(), p.send_off.copy(), p.recv_off.copy(), p.send_nodes.copy(), p.recv_nodes.copy(),
            p.num_nodes)


def _torch_dtype(dtype):
    import torch
    return torch.float32 if dtype == np.float32 else torch.float64


class DistributedEngine:
    """This rank's part of a multi-GPU run over torch.distributed (NCCL).

    engine_comm=True (default): torch.distributed only distributes an NCCL
    unique id; the engine then runs every step -- kernels, halo send/recv,
    status allreduce -- itself, CUDA-graph captured (djg_comm_init).
    engine_comm=False: the same sequence driven from Python per step with
    torch.distributed P2P / allreduce (reference driver for tests)."""

    def __init__(self, scenario: Scenario, device: int, group=None, flags: int = 0, engine_comm: bool = True,
                 method: str = "rcb", transport: str = "nccl"):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device
        self.engine_comm = engine_comm
        if method == "box-local":
            # this rank's part from the box spec alone (no global mesh); the
            # global minimum characteristic length through the group
            def reduce_min(x):
                vals = [None] * self.world
                dist.all_gather_object(vals, float(x), group=group)
                return min(vals)
            self.part = Partition.box_local(_spec_of(scenario), self.world, self.rank, reduce_min)
        else:
            self.part = Partition(scenario, self.world, self.rank, method)
        self.eng = PartEngine(self.part, device, flags)
        tdt = _torch_dtype(self.part.dtype)
        dev = torch.device("cuda", device)
        self.send = torch.zeros((max(self.part.send_nodes.size, 1), 4), dtype=tdt, device=dev)
        self.recv = torch.zeros((max(self.part.recv_nodes.size, 1), 4), dtype=tdt, device=dev)
        self.status = torch.zeros(3, dtype=torch.int64, device=dev)  # djg_step_status: MAX, MAX, SUM
        self.stream = torch.cuda.ExternalStream(self.eng.stream, device=dev)
        self.transport = transport
        if transport == "p2p":
            # peer-memory step: map every other rank's buffers (CUDA IPC) and
            # let the engine store the halo into them from its node kernel
            handles = [None] * self.world
            dist.all_gather_object(handles, self.eng.peer_ipc_export(), group=group)
            halos = [None] * self.world
            dist.all_gather_object(halos, _halo(self.part), group=group)
            ptrs = [self.eng.peer_export() if q == self.rank else self.eng.peer_ipc_open(handles[q])
                    for q in range(self.world)]
            self.eng.peer_setup(self.world, self.rank, ptrs, peer_destinations(halos, self.rank),
                                [h[5] for h in halos])
            dist.barrier(group=group)
            self.engine_comm = True  # the engine drives every step
        elif engine_comm:
            uid = C.create_string_buffer(128)
            if self.rank == 0 and _lib().djg_comm_unique_id(uid) != A.DJG_OK:
                raise RuntimeError(_lib().djg_create_error().decode())
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            uid = C.create_string_buffer(box[0], 128)
            p = self.part
            nb = np.ascontiguousarray(p.neighbors, np.int32)
            self.eng._check(_lib().djg_comm_init(self.eng._h, uid, self.world, self.rank, int(nb.size), A.ptr(nb),
                                                 A.ptr(p.send_off), A.ptr(p.recv_off)))

    def _exchange(self):
        dist = self.dist
        ops = []
        p = self.part
        for k, nb in enumerate(p.neighbors.tolist()):
            s0, s1 = int(p.send_off[k]), int(p.send_off[k + 1])
            r0, r1 = int(p.recv_off[k]), int(p.recv_off[k + 1])
            if s1 > s0:
                ops.append(dist.P2POp(dist.isend, self.send[s0:s1], nb, self.group))
            if r1 > r0:
                ops.append(dist.P2POp(dist.irecv, self.recv[r0:r1], nb, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def step_async(self, nsteps: int):
        import torch
        if self.engine_comm:
            self.eng.step_async(nsteps)
            return
        with torch.cuda.stream(self.stream):
            for _ in range(nsteps):
                self.eng.step_async(1)
                self.eng.halo_pack(self.send.data_ptr())
                self._exchange()
                self.eng.halo_unpack(self.recv.data_ptr())
                self.eng.step_status(self.status.data_ptr())
                self.dist.all_reduce(self.status[:2], op=self.dist.ReduceOp.MAX, group=self.group)
                self.dist.all_reduce(self.status[2:], op=self.dist.ReduceOp.SUM, group=self.group)
                self.eng.step_agree(self.status.data_ptr())

    def step(self, nsteps: int, raise_on_failure=True) -> StepReport:
        start = self.eng.get_state()[2]
        self.step_async(nsteps)
        r = self.eng.sync()
        r.steps_done = r.step - start
        if raise_on_failure and r.status != A.DJG_OK:
            raise_for(r)
        return r

    def step_lockstep(self, nsteps: int) -> StepReport:
        """Peer-memory step with a host barrier between each step's local part
        (element kernel, node kernel with its peer stores and mailbox posts)
        and the agreement: by the time any rank's k_wait_agree runs, every
        rank's posts have completed, so no kernel ever waits on another
        process's kernel. For ranks that share one GPU (processes on one
        device are time-sliced: a kernel spinning on another process's flag
        is not guaranteed to see it run). Same kernels, IPC mappings,
        system-scope release/acquire and agreement as the graph-captured step;
        counts summed over the steps."""
        if self.transport != "p2p":
            raise ConfigError("step_lockstep drives the peer-memory transport")
        acc = None
        for _ in range(nsteps):
            self.eng.step_peer_local()
            self.eng.sync()
            self.dist.barrier(group=self.group)
            self.eng.step_peer_agree()
            r = self.eng.sync()
            self.dist.barrier(group=self.group)
            if acc is not None:
                r.steps_done += acc.steps_done
                r.inverted_count += acc.inverted_count
                r.inverted_steps += acc.inverted_steps
            acc = r
        return acc

    def gather_global(self):
        """All ranks' owned displacements assembled into global arrays (rank 0
        gets the result; others return None)."""
        import torch
        u, up, step = self.eng.owned_state()
        ids = torch.from_numpy(self.part.node_l2g[: self.part.num_owned].copy())
        objs = [None] * self.world
        self.dist.all_gather_object(objs, (ids.numpy(), u, up), group=self.group)
        if self.rank != 0:
            return None
        n = self.part.info["global_nodes"]
        U = np.zeros((n, 3), self.part.dtype)
        UP = np.zeros((n, 3), self.part.dtype)
        for g, a, b in objs:
            U[g] = a
            UP[g] = b
        return U.reshape(-1), UP.reshape(-1), step


class EmulatedParts:
    """All parts of a decomposition in one process on one device: the same
    engines and kernels as DistributedEngine, the halo moved with device
    copies and the failure agreement reduced on the device. For tests."""

    def __init__(self, scenario: Scenario, nparts: int, device: int = 0, flags: int = 0, method: str = "rcb",
                 transport: str = "copy"):
        import torch
        self.torch = torch
        if method == "box-local":
            self.parts = Partition.box_local_all(_spec_of(scenario), nparts)
        else:
            self.parts = [Partition(scenario, nparts, p, method) for p in range(nparts)]
        self.engs = [PartEngine(p, device, flags) for p in self.parts]
        self.transport = transport
        if transport == "p2p":
            ptrs = [e.peer_export() for e in self.engs]
            halos = [_halo(p) for p in self.parts]
            for i, e in enumerate(self.engs):
                e.peer_setup(nparts, i, ptrs, peer_destinations(halos, i), [h[5] for h in halos])
        tdt = _torch_dtype(scenario.dtype)
        dev = torch.device("cuda", device)
        self.send = [torch.zeros((max(p.send_nodes.size, 1), 4), dtype=tdt, device=dev) for p in self.parts]
        self.recv = [torch.zeros((max(p.recv_nodes.size, 1), 4), dtype=tdt, device=dev) for p in self.parts]
        self.status = [torch.zeros(3, dtype=torch.int64, device=dev) for _ in self.parts]
        self.global_nodes = self.parts[0].info["global_nodes"]

    def _sync(self):
        for e in self.engs:
            e.sync()

    def _exchange(self):
        # receiver q's block from p = sender p's block to q (same global order)
        for q, pq in enumerate(self.parts):
            for k, p in enumerate(pq.neighbors.tolist()):
                pp = self.parts[p]
                j = pp.neighbors.tolist().index(q)
                r0, r1 = int(pq.recv_off[k]), int(pq.recv_off[k + 1])
                s0, s1 = int(pp.send_off[j]), int(pp.send_off[j + 1])
                assert r1 - r0 == s1 - s0
                if r1 > r0:
                    self.recv[q][r0:r1].copy_(self.send[p][s0:s1])
        self.torch.cuda.synchronize()

    def _agree(self):
        torch = self.torch
        st = torch.stack(self.status)
        red = torch.cat([st[:, :2].max(dim=0).values, st[:, 2:].sum(dim=0)])
        torch.cuda.synchronize()  # red is produced on torch's stream, read on the engines'
        for e in self.engs:
            e.step_agree(red.data_ptr())
        self._sync()

    def step(self, nsteps: int, overlap: bool = False):
        """overlap=False: local step, then halo exchange and agreement.
        overlap=True: the order of the engine's overlapped NCCL step -- halo
        pack and interior elements, exchange, unpack, boundary elements and
        node update, agreement. Returns one report per part over the whole
        call (each engine call covers one step: the counts are summed)."""
        acc = [None] * len(self.engs)
        for _ in range(nsteps):
            self._step1(overlap)
            for i, e in enumerate(self.engs):
                r = e.sync()
                if acc[i] is not None:
                    r.steps_done += acc[i].steps_done
                    r.inverted_count += acc[i].inverted_count
                    r.inverted_steps += acc[i].inverted_steps
                acc[i] = r
        return acc if nsteps > 0 else [e.sync() for e in self.engs]

    def _step1(self, overlap: bool):
        if self.transport == "p2p":
            # every part's step (its node kernel stores the halo into the
            # other parts' buffers and posts its status) before any part
            # waits: no kernel ever waits for another one here
            for e in self.engs:
                e.step_peer_local()
            self._sync()
            for e in self.engs:
                e.step_peer_agree()
            self._sync()
            return
        if overlap:
            for p, e in enumerate(self.engs):
                e.halo_pack(self.send[p].data_ptr())
                e.step_interior()
            self._sync()
            self._exchange()
            for p, e in enumerate(self.engs):
                e.halo_unpack(self.recv[p].data_ptr())
                e.step_boundary()
                e.step_status(self.status[p].data_ptr())
        else:
            for e in self.engs:
                e.step_async(1)
            for p, e in enumerate(self.engs):
                e.halo_pack(self.send[p].data_ptr())
            self._sync()
            self._exchange()
            for p, e in enumerate(self.engs):
                e.halo_unpack(self.recv[p].data_ptr())
                e.step_status(self.status[p].data_ptr())
        self._sync()
        self._agree()

    def set_global_state(self, u=None, up=None, step=0):
        for e in self.engs:
            e.set_global_state(u, up, step)

    def global_state(self):
        U = np.zeros((self.global_nodes, 3), self.parts[0].dtype)
        UP = np.zeros_like(U)
        step = None
        for p, e in zip(self.parts, self.engs):
            u, up, step = e.owned_state()
            U[p.node_l2g[: p.num_owned]] = u
            UP[p.node_l2g[: p.num_owned]] = up
        return U.reshape(-1), UP.reshape(-1), step

    def close(self):
        for e in self.engs:
            e.close()
