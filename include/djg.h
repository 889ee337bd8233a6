/*
 * djg.h — C-ABI of the B200 DJ-TLED explicit-dynamics engine (libdjg.so).
 *
 * What it replaces. The reference is a header-only C++ library with no FFI;
 * its de-facto operator interface for the hot path is the duck-typed Engine
 * concept consumed by advance_step / run_simulation:
 *
 *   AssembleStats Engine::assemble(const std::vector<Real>& u,
 *                                  std::vector<Real>& f, int threads,
 *                                  InversionPolicy policy)
 *        /root/reference/proj/include/djtled/solver.hpp:269-272 (DjEngine)
 *   StepOutcome advance_step(SimState&, Engine&, const UpdateCoeffs&,
 *                            const DofConstraints&, Real dt, int threads,
 *                            InversionPolicy, std::vector<Real>& u_next)
 *        solver.hpp:98-153
 *   RunResult run_simulation(Engine&, node_mass, DofConstraints, RunParams,
 *                            hook, const SimState* initial)
 *        solver.hpp:205-258
 *
 * Plugging the GPU in at `assemble` would move 2x3N Reals over PCIe per
 * step, so this ABI sits one level up: the whole step and the run loop, with
 * the state resident in HBM. Each entry point names the reference call it
 * replaces. Ownership: the caller owns every host array; djg_create deep
 * copies them. A handle is not thread-safe (like DjEngine, whose elem_f_ is
 * mutable, solver.hpp:283); calls are synchronous unless suffixed _async.
 * No exception crosses the ABI: functions return djg_status codes and
 * djg_last_error() holds the message.
 */
#ifndef DJG_H
#define DJG_H

#include <stddef.h>
#include <stdint.h>

#include "djg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Canonical per-element hot-field record (Reals, this order), the subset of
 * ElementConstants<Real> (precompute.hpp:170-201) the step reads:
 *   [0..8]   J0, row-major, J[i][j] = dx_j/dxi_i       (element.hpp:380)
 *   [9]      det_J0          [10] V0
 *   [11..16] m1[6]           [17..22] I1m (xx,yy,zz,xy,xz,yz)
 *   TI, OT:  m4[6], I4m[6]
 *   OT:      m6[6], I6m[6]
 *   MR:      M2 (21, packed upper Sym6, core.hpp:282-305), I2m[6] (6 x 6)
 *   I57:     M5 (21), I5m[6] (6 x 6), M7 (21), I7m[6] (6 x 6)  (full record only)
 *   H8:      k_hg, hg_gamma[4][8]
 */
#define DJG_CONST_BASE 23
int32_t djg_const_count(int32_t kind, int32_t model);

typedef struct djg_engine djg_engine;

/* Engine construction inputs: everything DjEngine + UpdateCoeffs +
 * DofConstraints hold after precompute (solver.hpp:18-33,64-87,264-267). */
typedef struct djg_desc {
    int32_t precision;          /* sizeof(Real): 4 or 8 */
    int32_t kind;               /* djg_element_kind */
    int64_t num_nodes;
    int64_t num_elements;
    const int32_t* conn;        /* npe*E, Mesh::conn (mesh.hpp:24) */
    const void* consts;         /* E*nconst Reals, canonical record above */
    int32_t nconst;             /* must equal djg_const_count(kind, material.model) */
    int32_t inversion_policy;   /* djg_inversion_policy */
    const int64_t* csr_offsets; /* N+1, NodeElementAdjacency (mesh.hpp:299-320); */
    const int64_t* csr_elem;    /*   NULL -> rebuilt from conn by the same   */
    const int32_t* csr_local;   /*   ascending-element counting sort          */
    const uint8_t* dof_kind;    /* 3N  DofConstraints::kind (NULL: all free) */
    const void* dof_target;     /* 3N Real */
    const void* dof_t_total;    /* 3N Real */
    const void* c1;             /* N Real  UpdateCoeffs::c1 (NULL: configure later) */
    const uint8_t* massless;    /* N       UpdateCoeffs::massless */
    double c2, c3;              /* UpdateCoeffs::c2/c3 (Real values) */
    double dt;                  /* Real value */
    djg_material_params material;
    int32_t device;             /* CUDA ordinal */
    uint32_t flags;             /* DJG_FLAG_* */
    const void* nodes;          /* 3N Reals, reference coordinates (DJG_FLAG_DEVICE_PRECOMPUTE) */
    double c_hg;                /* hourglass coefficient (DJG_FLAG_DEVICE_PRECOMPUTE) */
} djg_desc;

/* Flags */
#define DJG_FLAG_NO_GRAPH 1u    /* launch kernels one by one instead of CUDA graphs */
#define DJG_FLAG_SLABS 2u       /* pipeline each step as L2-sized element slabs (bit-identical) */
#define DJG_FLAG_NO_DISCARD 4u  /* slab step: keep consumed force rows in L2 (no discard) */
#define DJG_FLAG_COMPACT 8u     /* keep J0, det J0, V0 (+ H8 k_hg, gamma) per element in HBM;
                                   the element kernel rebuilds the m / I tensors in registers
                                   with the precompute's own arithmetic (bitwise) */
#define DJG_FLAG_DEVICE_PRECOMPUTE 16u /* build the per-element record on the GPU from
                                          nodes + conn (desc.consts may be NULL) */
#define DJG_FLAG_FULL_RECORD 32u /* keep the full record in HBM (default for
                                    Mooney-Rivlin in f64 and on H8; otherwise
                                    the compact record) */
#define DJG_FLAG_TLED 64u        /* conventional TLED element forces (tled_force.hpp), the
                                    paper's comparison path; record built on the device */
#define DJG_FLAG_NO_PIPE 128u    /* one-shot element kernel instead of the bulk-copy
                                    pipelined one (k_element_pipe); bit-identical */
#define DJG_FLAG_NO_FUSED 512u  /* keep the two-kernel step (element kernel + gather/update)
                                    on a generated box, where the default is one fused
                                    kernel per step (k_box_step, no force slots in HBM)
                                    once the box gives every block enough column layers */
#define DJG_FLAG_FUSED 1024u     /* the fused box step on any generated T4 box it supports,
                                    however small (bit-identical either way) */
#define DJG_FLAG_WINDOW 256u     /* pipelined element kernel with node windows: each
                                    tile's node rows staged in shared memory by bulk
                                    copies next to its slot positions (k_element_win);
                                    bit-identical. Opt-in: faster on L2-resident meshes
                                    (cfg3), slower on cfg5 */

/* DjEngine(mesh, material, c_hg) (solver.hpp:264-267) at the mesh level:
 * the library runs the precompute (build_element_constants,
 * precompute.hpp:206-255) and NodeElementAdjacency::build (mesh.hpp:299-320)
 * itself, bit-identically to the reference, then uploads. The step data
 * (masses, BCs, dt, alpha) follows with djg_configure_step, like the
 * reference's run_simulation(engine, node_mass, bc, params). */
typedef struct djg_mesh_desc {
    int32_t precision;          /* sizeof(Real) */
    int32_t kind;               /* djg_element_kind */
    int64_t num_nodes;
    int64_t num_elements;
    const void* nodes;          /* 3N Reals, Mesh::nodes (mesh.hpp:23) */
    const int32_t* conn;        /* npe*E, Mesh::conn */
    djg_material_params material;
    double c_hg;                /* hourglass coefficient (0.1 = default_hourglass_coefficient) */
    int32_t inversion_policy;
    int32_t device;
    uint32_t flags;
    int32_t threads;            /* host threads for the precompute (0 = all) */
} djg_mesh_desc;
int djg_create_from_mesh(const djg_mesh_desc* desc, djg_engine** out);

/* Precompute results on the device, for an engine created with
 * DJG_FLAG_DEVICE_PRECOMPUTE and no caller CSR (its adjacency, slot ranks
 * and slices are then built on the GPU too):
 *   djg_lump_mass        lump_mass(mesh, material.rho, elems)  precompute.hpp:275-287
 *                        -> N Reals, bit-identical to the host function
 *   djg_min_char_length  min over elements of characteristic_length
 *                        (precompute.hpp:303-319), the numerator of
 *                        critical_dt = l_min / wave_speed (:323-331); Real
 *                        widened to double.
 * Other engines return DJG_E_CONFIG. */
int djg_lump_mass(djg_engine* eng, void* mass);
int djg_min_char_length(djg_engine* eng, double* l_min);

/* UpdateCoeffs::build(node_mass, dt, alpha) (solver.hpp:70-86) +
 * DofConstraints (solver.hpp:11-39): everything advance_step needs besides
 * the engine. dof_kind NULL = all free. Real values widened to double. */
typedef struct djg_step_desc {
    const void* node_mass;      /* N Reals (lump_mass) */
    const uint8_t* dof_kind;    /* 3N  DofConstraints::kind */
    const void* dof_target;     /* 3N Reals */
    const void* dof_t_total;    /* 3N Reals */
    double dt;
    double alpha;
} djg_step_desc;
int djg_configure_step(djg_engine* eng, const djg_step_desc* step);

/* The InversionPolicy argument of Engine::assemble / RunParams::on_inversion. */
int djg_set_policy(djg_engine* eng, int32_t policy);

/* DjEngine ctor + UpdateCoeffs::build + DofConstraints::build
 * (solver.hpp:264-267, 70-86, 18-33). Validates shapes, uploads, builds the
 * CSR-ordered force-slot layout on the device. */
int djg_create(const djg_desc* desc, djg_engine** out);
void djg_destroy(djg_engine* eng);

/* SimState assignment (solver.hpp:41-57; run_simulation's `initial`,
 * solver.hpp:209,214). u_curr/u_prev: 3N Reals (NULL -> zeros). Clears any
 * halted inversion/divergence condition. */
int djg_set_state(djg_engine* eng, const void* u_curr, const void* u_prev, int64_t step);
/* SimState::r_ext (solver.hpp:44). NULL -> identically zero (the default). */
int djg_set_external(djg_engine* eng, const void* r_ext);
/* SimState readback: u_curr/u_prev 3N Reals each (either may be NULL). */
int djg_get_state(djg_engine* eng, void* u_curr, void* u_prev, int64_t* step);

/* nsteps x advance_step (solver.hpp:98-153) with the loop semantics of
 * run_simulation (solver.hpp:225-239): stops at the first failing step and
 * leaves the state at the last good step. Returns DJG_OK,
 * DJG_E_INVERSION (report->first_inverted = min inverted element id) or
 * DJG_E_DIVERGENCE (report->fail_step = state.step + 1). */
int djg_step(djg_engine* eng, int64_t nsteps, djg_report* report);
/* advance_step (solver.hpp:98-153) with a host SimState, in one call: uploads
 * u_curr and u_prev (3N Reals each) in chunks -- each element chunk starts as
 * soon as the u_curr nodes it reads have landed, each node-update chunk when
 * its u_prev chunk has -- runs one step from `step`, writes the new u_curr to
 * u_next chunk by chunk (or u_curr unchanged when the step failed) and fills
 * the report. For loops whose state lives on the host; pinned host buffers
 * let the copies overlap. */
int djg_advance_host(djg_engine* eng, const void* u_curr, const void* u_prev, int64_t step, void* u_next,
                     djg_report* report);

/* Asynchronous variant for timing: enqueue nsteps on the engine stream and
 * return. djg_sync waits and fills the report. */
int djg_step_async(djg_engine* eng, int64_t nsteps);
int djg_sync(djg_engine* eng, djg_report* report);
/* The engine's cudaStream_t (for CUDA events / external streams). */
void* djg_stream(djg_engine* eng);

/* Engine::assemble (solver.hpp:269-272 -> assemble_internal,
 * djtled_force.hpp:163-209): internal forces f (3N Reals) at displacement u
 * (3N Reals; NULL -> the current state). Under Abort with an inverted element
 * f is not written, as in the reference. */
int djg_assemble(djg_engine* eng, const void* u, void* f_int, djg_assemble_stats* stats);

/* Per-kernel timing of nsteps steps: device milliseconds spent in the
 * element-force kernel and in the gather+update kernel (CUDA events on the
 * engine stream). Advances the state like djg_step. */
int djg_profile_steps(djg_engine* eng, int64_t nsteps, float* ms_element, float* ms_node,
                      float* ms_total);

/*
 * Multi-GPU step, one engine per part (djg_partition_desc).
 * Per step, on the engine stream, with the communication in between done by
 * the caller's NCCL (or any transport):
 *   djg_step_async(eng, 1)              local elements, owned nodes
 *   djg_halo_pack(eng, send)            owned nodes others reference -> send
 *   <exchange send/recv with the neighbors>
 *   djg_halo_unpack(eng, recv)          recv -> ghost nodes
 *   djg_step_status(eng, status)        int64[3] step summary of this part
 *   <allreduce over parts: MAX of words 0-1, SUM of word 2>
 *   djg_step_agree(eng, reduced)        every part halts at the same state
 * status[0]: 2 inversion halt, 1 divergence, 0 none; status[1]: -(global id
 * of the first inverted element) or INT64_MIN; status[2]: inverted elements
 * this part reports for the step (its own elements only, see
 * djg_set_counted_elements) -- the reduced sum is the step's global count,
 * accumulated by djg_step_agree into the report's inverted_count /
 * inverted_steps on every part.
 * Halo buffers hold one 16-byte (f32) / 32-byte (f64) node record per entry.
 */
int djg_set_partition(djg_engine* eng, int64_t num_owned, const int64_t* elem_l2g);
int djg_set_halo(djg_engine* eng, int64_t nsend, const int32_t* send_nodes, int64_t nrecv, const int32_t* recv_nodes);
/* Multi-part inversion counting: counted[e] = 1 for the local elements this
 * part reports (djg_partition_owned_elements), 0 for ghost copies, so every
 * inverted element is counted once over all parts. Without it a part counts
 * every element it computes. */
int djg_set_counted_elements(djg_engine* eng, const uint8_t* counted);
int djg_halo_pack(djg_engine* eng, void* dev_send);
int djg_halo_unpack(djg_engine* eng, const void* dev_recv);
int djg_step_status(djg_engine* eng, int64_t* dev_status);
int djg_step_agree(djg_engine* eng, const int64_t* dev_reduced);

/* Engine-driven multi-GPU step over NCCL (no host work per step). Rank 0
 * creates a 128-byte NCCL unique id and the caller distributes it; every rank
 * then calls djg_comm_init (collectively) with its neighbour ranks and the
 * halo offsets of djg_partition_halo. From then on djg_step / djg_step_async
 * run, per step and CUDA-graph captured: the local step, halo pack, one
 * grouped ncclSend/ncclRecv per neighbour, unpack, status, ncclAllReduce(MAX)
 * and the agreement -- bit-identical to one GPU. libnccl.so.2 is resolved at
 * run time (the process's, e.g. torch.distributed's). */
int djg_comm_unique_id(void* id128);
/* Overlapped multi-part step: the part's local elements [0, num_interior)
 * reference no ghost node (djg_partition_info.interior_elements; the
 * partitioner orders them first). With a communicator the captured step
 * becomes: halo pack -> {interior elements || NCCL halo send/recv} -> unpack
 * -> boundary elements -> node update -> status allreduce -> agreement, the
 * exchange hidden behind the interior elements (the ghost values used are
 * those of the step start, as before). Without one, a caller drives the same
 * order itself: djg_halo_pack, djg_step_interior, <exchange>,
 * djg_halo_unpack, djg_step_boundary, djg_step_status, <allreduce>,
 * djg_step_agree. */
/* Peer-memory multi-GPU step (no NCCL on the step path): every part's node
 * kernel stores the new displacement of the owned nodes other parts reference
 * straight into their buffers over NVLink, and posts its step status into
 * every part's mailbox; a one-warp kernel waits for all parts and agrees.
 *   djg_peer_export      this engine's 4 device pointers (3 displacement
 *                        buffers, mailbox) -- single-process use
 *   djg_peer_ipc_export  their CUDA IPC handles (4 x 64 bytes), for other ranks
 *   djg_peer_ipc_open    map another rank's 4 handles -> 4 device pointers
 *   djg_peer_setup       every part's pointers (peer_u: 3 per part, peer_mail:
 *                        1 per part, own included), every part's local node
 *                        count (peer_num_nodes: the destination bounds) and
 *                        this part's halo destinations: owned node
 *                        dest_node[i] -> part dest_part[i], local node
 *                        dest_index[i] < peer_num_nodes[dest_part[i]]
 * Then djg_step runs element kernel -> node kernel with peer stores ->
 * wait/agree per step, graph-captured. The wait is bounded: a part whose
 * peers do not post within DJG_PEER_TIMEOUT_MS (default 10 s) halts with
 * DJG_E_PEER instead of spinning forever. djg_step_peer_local /
 * djg_step_peer_agree split one step for single-device emulation. */
int djg_peer_export(djg_engine* eng, void** ptrs4);
int djg_peer_ipc_export(djg_engine* eng, void* handles);
int djg_peer_ipc_open(djg_engine* eng, const void* handles, void** ptrs4);
int djg_peer_setup(djg_engine* eng, int32_t nparts, int32_t part, const void* const* peer_u,
                   const void* const* peer_mail, const int64_t* peer_num_nodes, int64_t ndest,
                   const int32_t* dest_node, const int32_t* dest_part, const int32_t* dest_index);
int djg_step_peer_local(djg_engine* eng);
int djg_step_peer_agree(djg_engine* eng);
int djg_set_interior(djg_engine* eng, int64_t num_interior);
int djg_step_interior(djg_engine* eng);
int djg_step_boundary(djg_engine* eng);
int djg_comm_init(djg_engine* eng, const void* id128, int32_t nranks, int32_t rank, int32_t num_neighbors,
                  const int32_t* neighbors, const int64_t* send_off, const int64_t* recv_off);

/* Layout facts for roofline accounting and tests. */
typedef struct djg_engine_info {
    int64_t num_nodes, num_elements;
    int64_t num_slots;          /* npe*E */
    int64_t slot_capacity;      /* force-slot buffer entries (sliced layout incl. padding) */
    int64_t device_bytes;       /* device memory held by the engine */
    int32_t npe, nconst, const_planes, precision;
    int32_t kernels_per_step;   /* kernel launches per step */
    int32_t sm_count;
    int32_t slabs;              /* element slabs per step (2 kernels each) */
    int32_t compact;            /* 1: compact per-element record in HBM */
    int64_t slab_elements;      /* elements per slab */
    int32_t formulation;        /* 0 DJ-TLED, 1 TLED (DJG_FLAG_TLED) */
    int32_t pipelined;          /* element kernel streams tiles through shared memory */
    int32_t windowed;           /* ... with each tile's node rows staged as windows */
    int64_t window_tiles;       /* tiles whose nodes fit a window (the rest gather) */
    int32_t fused;              /* 1: one fused kernel per step (generated box, k_box_step) */
    int32_t lattice;            /* 1: the fused step reads its records from the lattice table */
} djg_engine_info;
int djg_get_info(djg_engine* eng, djg_engine_info* info);

/* Debug/test: copy the engine's force-slot position table (npe*E int32, the
 * position of (element, local) in the sliced slot buffer) to the host. */
int djg_get_slot_map(djg_engine* eng, int32_t* slot_pos);

/* Test hook: the per-element record held on the device as E x n Reals
 * (n = nconst, or in compact mode 12: J0, det J0, V0, pad -- 45 for H8:
 * + k_hg, gamma). Returns n
 * (out may be NULL to query it), -1 on error. */
int64_t djg_get_consts(djg_engine* eng, void* out);

/* Test hook: the device cube root the element kernel uses (a restatement of
 * the host libm's, see kernels.cuh) over n Reals. */
int djg_debug_cbrt(int32_t precision, const void* in, void* out, int64_t n, int32_t device);

const char* djg_last_error(djg_engine* eng);
const char* djg_status_string(int32_t status);
/* Last error of a failed djg_create (no handle). */
const char* djg_create_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DJG_H */
