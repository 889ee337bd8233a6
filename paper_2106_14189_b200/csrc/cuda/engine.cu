// libdjg: the B200 DJ-TLED engine behind the C-ABI of include/djg.h.
//
// One engine = one problem resident in HBM:
//   conn        int4 planes [npe/4][E]     connectivity
//   rank        npe x 1|2 bytes per element: rank of the element in each node's CSR row
//   consts      Plane planes [nplanes][E]  hot constants (float4 / double2)
//   u[3]        Node[N]                    triple-buffered displacement (xyz+pad)
//   ef          Node[capacity]             element-node forces (xyz + pad) in sliced CSR order
//   row_len, slice_base, c1, code, target, t_total, r_ext   node data
//   ctrl        Ctrl                       step counter + failure flags
// A step is k_element then k_node on one stream; multi-step calls replay a
// CUDA graph of G steps. Buffer roles rotate with ctrl.step % 3 on the device,
// so one graph serves every phase and a failed step leaves the state as the
// reference's advance_step does (solver.hpp:106-110, 143-147).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "djg.h"
#include "../common/box_mesh.hpp"
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include "kernels.cuh"

namespace djg {
namespace {

// k_element_pipe: stages per block and the largest tile stage it is used for
// (bigger records -- H8 full, MR -- keep the one-shot kernel).
#ifndef DJG_PIPE_STAGES
#define DJG_PIPE_STAGES 4
#endif
#ifndef DJG_PIPE_MAX_STAGE_KB
#define DJG_PIPE_MAX_STAGE_KB 32
#endif

constexpr int kPipeStages = DJG_PIPE_STAGES;
// H8 through the bulk-copy pipeline where its stage fits (f32 compact NH / TI /
// OT: 29 KB per 128-element stage, 2 stages, 3 blocks/SM): 2.2M hexes NH 163
// -> 142 us, TI 166 -> 146, OT 178 -> 153; cfg4 81 -> 73. The larger records
// (f64, full, TLED) keep the one-shot kernel.
#ifndef DJG_PIPE_H8
#define DJG_PIPE_H8 1
#endif
#ifndef DJG_PIPE_H8_STAGES
#define DJG_PIPE_H8_STAGES 2
#endif

#ifndef DJG_HOST_CHUNKS
#define DJG_HOST_CHUNKS 4  // djg_advance_host: u_prev upload / node-update / read-back chunks
#endif
constexpr int kPipeMaxStageBytes = DJG_PIPE_MAX_STAGE_KB * 1024;
// k_element_win (node windows staged with the tile): the largest stage it is
// used for, and whether H8 tiles use it (cfg4 hexes: ~460 window nodes).
#ifndef DJG_WIN_MAX_STAGE_KB
#define DJG_WIN_MAX_STAGE_KB 40
#endif
#ifndef DJG_WIN_H8
#define DJG_WIN_H8 0
#endif
constexpr int kWinMaxStageBytes = DJG_WIN_MAX_STAGE_KB * 1024;
// k_box_step tile: BX x BY owned nodes (one thread each)
#ifndef DJG_BOX_BX
#define DJG_BOX_BX 16
#endif
#ifndef DJG_BOX_BY
#define DJG_BOX_BY 16
#endif
constexpr int kBoxBX = DJG_BOX_BX, kBoxBY = DJG_BOX_BY;

thread_local std::string g_create_error;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DescError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(call)                                                                                   \
    do {                                                                                           \
        const cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                                     \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")");                                       \
    } while (0)

inline int npe_of(int kind) { return kind == DJG_T4 ? 4 : 8; }

inline int const_count(int kind, int model) {
    int n = 23;
    if (model == DJG_TI || model == DJG_OT) n += 12;
    if (model == DJG_OT) n += 12;
    if (model == DJG_MR) n += 57;
    if (model == DJG_I57) n += 114;
    if (kind == DJG_H8) n += 33;
    return n;
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void alloc(size_t b) {
        release();
        bytes = b;
        if (b) CK(cudaMalloc(&p, b));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// NCCL, resolved at run time from the process's libnccl.so.2 (the one
// torch.distributed already loaded, else the system library), so libdjg.so
// has no link-time dependency on it. Only the multi-GPU step uses it.
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;

    static const Nccl& get() {
        static const Nccl api = [] {
            Nccl a;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return a;
            a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
            a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
            a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
            a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
            a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
            a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
            a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
            a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
            return a;
        }();
        if (!api.all_reduce) throw std::runtime_error("libnccl.so.2 not found (multi-GPU step)");
        return api;
    }
};

#define NK(x)                                                                                  \
    do {                                                                                       \
        const ncclResult_t r_ = (x);                                                           \
        if (r_ != ncclSuccess)                                                                 \
            throw CudaError(std::string("NCCL: ") + Nccl::get().error_string(r_) + " (" #x ")"); \
    } while (0)

class EngineBase {
public:
    virtual ~EngineBase() = default;
    virtual void set_state(const void* u, const void* up, int64_t step) = 0;
    virtual void set_external(const void* r) = 0;
    virtual void get_state(void* u, void* up, int64_t* step) = 0;
    virtual int step(int64_t n, djg_report* rep) = 0;
    virtual void step_async(int64_t n) = 0;
    virtual int sync(djg_report* rep) = 0;
    virtual int assemble(const void* u, void* f, djg_assemble_stats* st) = 0;
    virtual int profile(int64_t n, float* ms_e, float* ms_n, float* ms_t) = 0;
    virtual void info(djg_engine_info* out) = 0;
    virtual void slot_map(int32_t* out) = 0;
    virtual int64_t consts_out(void* out) = 0;
    virtual int lump_mass(void* out) = 0;
    virtual int min_char_length(double* out) = 0;
    virtual cudaStream_t stream() const = 0;
    virtual void configure_step(const djg_step_desc& s) = 0;
    virtual void set_policy(int policy) = 0;
    virtual void set_partition(int64_t num_owned, const int64_t* elem_l2g) = 0;
    virtual void set_halo(int64_t nsend, const int32_t* send, int64_t nrecv, const int32_t* recv) = 0;
    virtual void set_counted_elements(const uint8_t* counted) = 0;
    virtual void halo_pack(void* dev_out) = 0;
    virtual void halo_unpack(const void* dev_in) = 0;
    virtual void step_status(int64_t* dev_status) = 0;
    virtual void step_agree(const int64_t* dev_reduced) = 0;
    virtual void comm_init(const void* id, int nranks, int rank, int nnb, const int32_t* nb, const int64_t* send_off,
                           const int64_t* recv_off) = 0;
    virtual void set_interior(int64_t n) = 0;
    virtual void peer_export(void** ptrs) = 0;
    virtual void peer_ipc_export(void* handles) = 0;
    virtual void peer_ipc_open(const void* handles, void** ptrs) = 0;
    virtual void peer_setup(int nparts, int part, const void* const* peer_u, const void* const* peer_mail,
                            const int64_t* peer_num_nodes, int64_t ndest, const int32_t* dest_node,
                            const int32_t* dest_part, const int32_t* dest_index) = 0;
    virtual void step_peer_local() = 0;
    virtual int advance_host(const void* u, const void* up, int64_t step, void* u_next, djg_report* rep) = 0;
    virtual void step_peer_agree() = 0;
    virtual void step_interior() = 0;
    virtual void step_boundary() = 0;
};

template <class Real>
class Engine final : public EngineBase {
    using T = RT<Real>;
    using Node = typename T::Node;
    using Plane = typename T::Plane;

public:
    explicit Engine(const djg_desc& d) {
        kind_ = d.kind;
        model_ = d.material.model;
        npe_ = npe_of(kind_);
        N_ = d.num_nodes;
        E_ = d.num_elements;
        policy_ = d.inversion_policy;
        flags_ = d.flags;
        if (const char* v = std::getenv("DJG_SLAB_KB")) slab_bytes_ = int64_t(std::atoll(v)) << 10;
        nconst_ = const_count(kind_, model_);
        // Default record: compact (fewer bytes win) except for Mooney-Rivlin
        // in f64 and on H8, where rebuilding its 57 second-invariant Reals
        // costs more than reading them (10.4M tets: f32 T4 compact 590 vs
        // full 676 us; f64 T4 1588 vs 1343; 2.2M hexes f32 351 vs 238).
        tled_ = (flags_ & DJG_FLAG_TLED) != 0;
        if (model_ == DJG_I57 && (flags_ & (DJG_FLAG_COMPACT | DJG_FLAG_DEVICE_PRECOMPUTE | DJG_FLAG_TLED)))
            throw DescError("the I57 energy runs on the host-built full record only "
                            "(no DJG_FLAG_COMPACT / DJG_FLAG_DEVICE_PRECOMPUTE / DJG_FLAG_TLED)");
        const bool compact_default =
            model_ != DJG_I57 && (model_ != DJG_MR || (kind_ == DJG_T4 && sizeof(Real) == 4));
        compact_ = !tled_ && ((flags_ & DJG_FLAG_COMPACT) != 0 ||
                              (!(flags_ & DJG_FLAG_FULL_RECORD) && compact_default));
        // The compact T4 record is empty: the kernel rebuilds J0 from the node
        // coordinates, so they must be on the device.
        if (compact_ && d.kind == DJG_T4 && !d.nodes) compact_ = false;
        const bool dev_pre = tled_ || (flags_ & DJG_FLAG_DEVICE_PRECOMPUTE) != 0;
        need_x_ = dev_pre || (compact_ && d.kind == DJG_T4);
        nrec_ = tled_ ? (kind_ == DJG_H8 ? TledLayout<1>::count : TledLayout<0>::count)
                      : compact_ ? (kind_ == DJG_H8 ? kCompactLen<1> : kCompactLen<0>) : nconst_;
        // Tail planes (a remainder of scalar planes instead of a padded 16-byte
        // plane) apply to the compact T4 record, which is now empty.
        const bool tail = compact_ && kind_ == DJG_T4;
        nplanes_ = tail ? nrec_ / T::kPlane : (nrec_ + T::kPlane - 1) / T::kPlane;
        ntail_ = tail ? nrec_ % T::kPlane : 0;
        tail_stride_ = (E_ + 3) / 4 * 4 + 4;  // 16-byte aligned planes, tail tiles may round up
        if (d.nconst != nconst_) throw DescError("nconst does not match djg_const_count(kind, model)");
        if (N_ < 1 || E_ < 1) throw DescError("mesh must have nodes and elements");
        if (!d.conn) throw DescError("descriptor is missing conn");
        if (!d.consts && !dev_pre) throw DescError("descriptor is missing consts (or DJG_FLAG_DEVICE_PRECOMPUTE)");
        if (!d.nodes && dev_pre) throw DescError("device precompute / TLED need the node coordinates");
        if (!d.c1 != !d.massless) throw DescError("c1 and massless must be given together");
        if (E_ * npe_ > INT32_MAX || N_ > INT32_MAX) throw DescError("mesh too large for 32-bit slot indexing");

        device_ = d.device;
        CK(cudaSetDevice(d.device));
        CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, d.device));
        CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));

        // Slot layout: from the caller's (or a host-built) CSR, or -- device
        // precompute without a caller CSR and without slabs -- built on the GPU.
        device_layout_ = dev_pre && !d.csr_offsets && !(flags_ & DJG_FLAG_SLABS) && slab_bytes_ == 0;
        if (device_layout_) {
            build_layout_device(d.conn);
        } else {
            const int npe = npe_;
            const int32_t* conn = d.conn;
            for (int64_t i = 0; i < E_ * npe; ++i)
                if (conn[i] < 0 || conn[i] >= N_) throw DescError("connectivity index out of range");

            // Node -> (element, local) adjacency in ascending element order
            // (NodeElementAdjacency::build, mesh.hpp:299-320).
            std::vector<int64_t> off_v, elem_v;
            std::vector<int32_t> loc_v;
            const int64_t* off = d.csr_offsets;
            const int64_t* celem = d.csr_elem;
            const int32_t* cloc = d.csr_local;
            if (!off || !celem || !cloc) {
                off_v.assign(size_t(N_) + 1, 0);
                for (int64_t i = 0; i < E_ * npe; ++i) off_v[size_t(conn[i]) + 1]++;
                for (int64_t n = 0; n < N_; ++n) off_v[size_t(n) + 1] += off_v[size_t(n)];
                elem_v.resize(size_t(E_ * npe));
                loc_v.resize(size_t(E_ * npe));
                std::vector<int64_t> cur(off_v.begin(), off_v.end() - 1);
                for (int64_t e = 0; e < E_; ++e)
                    for (int a = 0; a < npe; ++a) {
                        const int64_t p = cur[size_t(conn[e * npe + a])]++;
                        elem_v[size_t(p)] = e;
                        loc_v[size_t(p)] = a;
                    }
                off = off_v.data();
                celem = elem_v.data();
                cloc = loc_v.data();
            }
            if (off[0] != 0 || off[N_] != E_ * npe) throw DescError("CSR offsets inconsistent with connectivity");

            // CSR consistency and row lengths.
            std::vector<int32_t> row_len(static_cast<size_t>(N_));
            int wmax = 0;
            bool bad = false;
    #pragma omp parallel for schedule(static) reduction(|| : bad) reduction(max : wmax)
            for (int64_t n = 0; n < N_; ++n) {
                row_len[size_t(n)] = int32_t(off[n + 1] - off[n]);
                wmax = std::max(wmax, int(off[n + 1] - off[n]));
                for (int64_t p = off[n]; p < off[n + 1]; ++p) {
                    const int64_t e = celem[p];
                    const int a = cloc[p];
                    if (e < 0 || e >= E_ || a < 0 || a >= npe || conn[e * npe + a] != n) bad = true;
                }
            }
            if (bad) throw DescError("CSR pairs do not match connectivity");
            wmax_ = std::max(wmax, 1);
            // Sliced slot layout: node n's k-th slot at slice_base[n/32] + 32k + n%32.
            // The element kernel finds it from the element's rank k in each of its
            // nodes' CSR rows (1 or 2 bytes per element-node).
            if (wmax_ > 65535) throw DescError("a node has more than 65535 incident elements");
            rank_bytes_ = wmax_ <= 256 ? 1 : 2;
            std::vector<uint8_t> ranks(size_t(E_ * npe) * size_t(rank_bytes_));
            {
                const int64_t S = (N_ + 31) / 32;
                slice_base_.assign(static_cast<size_t>(S) + 1, 0);
                int64_t cap = 0;
                for (int64_t sl = 0; sl < S; ++sl) {
                    slice_base_[size_t(sl)] = int32_t(cap);
                    int w = 0;
                    for (int64_t n = sl * 32; n < std::min<int64_t>(N_, sl * 32 + 32); ++n) w = std::max(w, row_len[size_t(n)]);
                    cap += int64_t(32) * w;
                    if (cap > INT32_MAX) throw DescError("slot buffer exceeds 32-bit indexing");
                }
                slice_base_[size_t(S)] = int32_t(cap);
                capacity_ = std::max<int64_t>(cap, 32);
                uniform_slices();
                const int rb = rank_bytes_;
    #pragma omp parallel for schedule(static)
                for (int64_t n = 0; n < N_; ++n)
                    for (int64_t p = off[n]; p < off[n + 1]; ++p) {
                        const int64_t k = p - off[n];
                        uint8_t* r = ranks.data() + size_t((celem[p] * npe + cloc[p]) * rb);
                        r[0] = uint8_t(k & 0xff);
                        if (rb == 2) r[1] = uint8_t(k >> 8);
                    }
                slicebase_.alloc(slice_base_.size() * sizeof(int32_t));
                CK(cudaMemcpy(slicebase_.p, slice_base_.data(), slicebase_.bytes, cudaMemcpyHostToDevice));
                rank_.alloc(ranks.size() + 16);  // + 16: bulk copies of a tail tile round up to 16 bytes
                CK(cudaMemcpy(rank_.p, ranks.data(), ranks.size(), cudaMemcpyHostToDevice));
            }
            plan_slabs(off, celem);

            // Upload connectivity as int4 planes.
            const int nq = npe / 4;
            {
                std::vector<int32_t> planes(size_t(E_ * npe));
    #pragma omp parallel for schedule(static)
                for (int64_t e = 0; e < E_; ++e)
                    for (int q = 0; q < nq; ++q)
                        for (int k = 0; k < 4; ++k) planes[size_t((int64_t(q) * E_ + e) * 4 + k)] = conn[e * npe + 4 * q + k];
                conn_.alloc(planes.size() * sizeof(int32_t));
                CK(cudaMemcpy(conn_.p, planes.data(), conn_.bytes, cudaMemcpyHostToDevice));
            }
            rowlen_.alloc(row_len.size() * sizeof(int32_t));
            CK(cudaMemcpy(rowlen_.p, row_len.data(), rowlen_.bytes, cudaMemcpyHostToDevice));
        }
        // Reference coordinates (device precompute).
        if (d.nodes && need_x_) {
            X_.alloc(size_t(N_) * sizeof(Node));
            DevBuf flat;
            flat.alloc(size_t(3 * N_) * sizeof(Real));
            CK(cudaMemcpy(flat.p, d.nodes, flat.bytes, cudaMemcpyHostToDevice));
            k_pack_nodes<Real><<<unsigned((N_ + 255) / 256), 256>>>(flat.as<Real>(), N_, X_.as<Node>());
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
        }
        // Material terms of the precompute (FibreDirections, k_hg factor).
        {
            const Real fa[3] = {Real(d.material.fibre_a[0]), Real(d.material.fibre_a[1]), Real(d.material.fibre_a[2])};
            const Real fb[3] = {Real(d.material.fibre_b[0]), Real(d.material.fibre_b[1]), Real(d.material.fibre_b[2])};
            for (int k = 0; k < 6; ++k) ea_.mat.A[k] = ea_.mat.B[k] = Real(0);
            for (int k = 0; k < 3; ++k) ea_.mat.fa[k] = ea_.mat.fb[k] = Real(0);
            if (model_ == DJG_TI || model_ == DJG_OT) {
                em::fibre_structure(fa, ea_.mat.A);
                em::unit3(fa, ea_.mat.fa);
            }
            if (model_ == DJG_OT) {
                em::fibre_structure(fb, ea_.mat.B);
                em::unit3(fb, ea_.mat.fb);
            }
            ea_.mat.chk = Real(d.c_hg) * Real(d.material.kappa);
        }
        // Constants: built on the device, or AoS chunks -> device planes.
        consts_.alloc(size_t(nplanes_) * size_t(E_) * sizeof(Plane) + size_t(ntail_) * size_t(tail_stride_) * sizeof(Real));
        Real* const ctail = reinterpret_cast<Real*>(consts_.as<Plane>() + size_t(nplanes_) * size_t(E_));
        if (dev_pre) {
            ElemArgs<Real> a{};
            a.E = E_;
            a.tail_stride = tail_stride_;
            a.conn = conn_.as<int4>();
            a.X = X_.as<Node>();
            a.mat = ea_.mat;
            DevBuf bad;
            bad.alloc(sizeof(unsigned long long));
            CK(cudaMemset(bad.p, 0xff, bad.bytes));
            const unsigned grid = unsigned((E_ + 127) / 128);
#define DJG_PRE(K, M) \
    k_precompute<Real, K, M><<<grid, 128>>>(a, nrec_, nplanes_, consts_.as<Plane>(), ctail, bad.as<unsigned long long>())
            if (tled_) {
                if (kind_ == DJG_T4) k_precompute_tled<Real, 0><<<grid, 128>>>(a, consts_.as<Plane>(), bad.as<unsigned long long>());
                else k_precompute_tled<Real, 1><<<grid, 128>>>(a, consts_.as<Plane>(), bad.as<unsigned long long>());
            } else if (kind_ == DJG_T4) {
                switch (model_) {
                    case DJG_NH: DJG_PRE(0, 0); break;
                    case DJG_TI: DJG_PRE(0, 1); break;
                    case DJG_OT: DJG_PRE(0, 2); break;
                    default: DJG_PRE(0, 3); break;
                }
            } else {
                switch (model_) {
                    case DJG_NH: DJG_PRE(1, 0); break;
                    case DJG_TI: DJG_PRE(1, 1); break;
                    case DJG_OT: DJG_PRE(1, 2); break;
                    default: DJG_PRE(1, 3); break;
                }
            }
#undef DJG_PRE
            CK(cudaGetLastError());
            unsigned long long first_bad = 0;
            CK(cudaMemcpy(&first_bad, bad.p, sizeof(first_bad), cudaMemcpyDeviceToHost));
            if (first_bad != ~0ull)
                throw DescError("element " + std::to_string(first_bad) + ": non-positive reference Jacobian determinant");
        } else if (nplanes_ + ntail_ > 0) {  // (the compact T4 record is empty)
            const int64_t chunk = std::min<int64_t>(E_, 1 << 20);
            DevBuf stage;
            stage.alloc(size_t(chunk) * nconst_ * sizeof(Real));
            const Real* src = static_cast<const Real*>(d.consts);
            for (int64_t e0 = 0; e0 < E_; e0 += chunk) {
                const int64_t ne = std::min(chunk, E_ - e0);
                CK(cudaMemcpy(stage.p, src + e0 * nconst_, size_t(ne) * nconst_ * sizeof(Real),
                              cudaMemcpyHostToDevice));
                const int64_t work = ne * (nplanes_ + ntail_);
                k_transpose_consts<Real><<<unsigned((work + 255) / 256), 256>>>(
                    stage.as<Real>(), nconst_, nrec_, kind_ == DJG_H8 ? nconst_ - 33 : -1, e0, ne, E_, nplanes_,
                    consts_.as<Real>(), ctail, tail_stride_, ntail_);
                CK(cudaGetLastError());
            }
            CK(cudaDeviceSynchronize());
        }
        if (device_layout_) mass_and_length_device(d.material.rho);
        // Node data.
        for (auto& b : u_) b.alloc(size_t(N_) * sizeof(Node));
        uscratch_.alloc(size_t(N_) * sizeof(Node));
        flat_.alloc(size_t(3 * N_) * sizeof(Real));
        ef_.alloc(size_t(capacity_) * sizeof(Node));
        CK(cudaMemset(ef_.p, 0, ef_.bytes));
        c1_.alloc(size_t(N_) * sizeof(Real));
        code_.alloc(size_t(N_));
        target_.alloc(size_t(3 * N_) * sizeof(Real));
        tTotal_.alloc(size_t(3 * N_) * sizeof(Real));
        ctrl_.alloc(sizeof(Ctrl));
        CK(cudaMallocHost(reinterpret_cast<void**>(&hctrl_), sizeof(Ctrl)));
        CK(cudaMallocHost(reinterpret_cast<void**>(&hstart_), sizeof(Ctrl)));

        // Kernel arguments.
        ea_.E = E_;
        ea_.N = N_;
        ea_.cap = capacity_;
        ea_.conn = conn_.as<int4>();
        ea_.rank = rank_.p;
        ea_.slice_base = slicebase_.as<int>();
        ea_.slice_w = slice_w_;
        ea_.c = consts_.as<Plane>();
        ea_.ctail = reinterpret_cast<const Real*>(consts_.as<Plane>() + size_t(nplanes_) * size_t(E_));
        ea_.tail_stride = tail_stride_;
        for (int i = 0; i < 3; ++i) ea_.u[i] = u_[i].as<Node>();
        ea_.u_override = nullptr;
        ea_.elem_l2g = nullptr;
        ea_.ef = ef_.as<Node>();
        ea_.ctrl = ctrl_.as<Ctrl>();
        const Real mu = Real(d.material.mu), c10 = Real(d.material.c10);
        ea_.mat.dI1 = model_ == DJG_MR ? c10 : mu / 2;
        ea_.mat.kappa = Real(d.material.kappa);
        ea_.mat.eta_a = Real(d.material.eta_a);
        ea_.mat.eta_b = Real(d.material.eta_b);
        ea_.mat.dI2 = Real(d.material.c01);
        ea_.X = X_.as<Node>();
        na_.N = N_;
        na_.cap = capacity_;
        na_.row_len = rowlen_.as<int>();
        na_.slice_base = slicebase_.as<int>();
        na_.slice_w = slice_w_;
        na_.ef = ef_.as<Node>();
        for (int i = 0; i < 3; ++i) na_.u[i] = u_[i].as<Node>();
        na_.r_ext = nullptr;
        na_.c1 = c1_.as<Real>();
        na_.code = code_.as<unsigned char>();
        na_.target = target_.as<Real>();
        na_.t_total = tTotal_.as<Real>();
        na_.policy = policy_;
        na_.ctrl = ctrl_.as<Ctrl>();
        na_.f_out = flat_.as<Real>();
        if (d.c1) {
            configure(static_cast<const Real*>(d.c1), d.massless, d.dof_kind, static_cast<const Real*>(d.dof_target),
                      static_cast<const Real*>(d.dof_t_total), Real(d.c2), Real(d.c3), Real(d.dt));
        }
        {
            // k_node grid: on meshes of up to 16 waves, a grid-stride launch
            // sized to the resident blocks (one barrier + completion count per
            // block, no tail wave: cfg4 54 -> 40 us), twice that for long rows
            // (T4, ~24 slots per node) beyond 4 waves (1 % better there, 7 %
            // worse for H8's 8-slot rows); on large meshes one thread per node
            // streams better (cfg5).
            int nb = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_node<Real, false>, 256, 0));
            const int64_t resident = int64_t(std::max(nb, 1)) * sms_, blocks = (N_ + 255) / 256;
            const bool long_rows = int64_t(npe_) * E_ >= 16 * N_;
            node_grid_ = blocks > 16 * resident                ? 0
                         : (blocks > 4 * resident && long_rows) ? 2 * resident
                                                                : resident;
            if (const char* v = std::getenv("DJG_NODE_GRID")) node_grid_ = std::atoll(v);
        }
        pipe_ = !(flags_ & DJG_FLAG_NO_PIPE) && n_slabs_ == 1;
        win_ = pipe_ && (flags_ & DJG_FLAG_WINDOW) && (kind_ == DJG_T4 || DJG_WIN_H8);
        if (win_) build_windows(d.conn);
        if (pipe_) launch_element(stream_, 0, E_, nullptr, /*setup=*/true);
        if (detect_box(d.conn)) {
            // the fused step pays for its column pieces' extra cell layer and
            // its halo cells: with per-tet rebuilds it wins from >= 32
            // column-layers per block (cfg5: 116, not cfg3: 6); with the
            // lattice table from >= 4 (cfg3: 75.3 -> 67.3 us). Smaller boxes
            // keep the kernel form their flags ask for.
            const int64_t W = int64_t(box_.tiles_x) * box_.tiles_y * (box_.nz + 1), g = box_grid_;
            if (kind_ == DJG_T4 && d.nodes && (box_forced_ || W >= 4 * g))
                build_lattice(static_cast<const Real*>(d.nodes));
            fused_ = box_forced_ || W >= 32 * g || (lattice_ && W >= 4 * g);
        }
        if (!win_) {
            slot_.release();
            widx_.release();
            wdesc_.release();
            ea_.slot = nullptr;
            ea_.widx = nullptr;
            ea_.wdesc = nullptr;
            win_tiles_ = 0;
        }
        set_state(nullptr, nullptr, 0);
    }

    // The fused box step (k_box_step) applies to a mesh generate_box made:
    // T4 cells in cell order, lexicographic nodes. The box dimensions follow
    // from element 0 (its first tet runs corner 0 -> 1 -> 3 -> 7: node ids 0,
    // 1, nx + 2, nx + 2 + (nx + 1)(ny + 1)); every element is then checked
    // against the generator. f32 compact records (J0 rebuilt from X) with
    // NH / TI / OT, one part, no slabs. It is the default when the box gives
    // every block enough column-layers (the constructor's gate);
    // DJG_FLAG_FUSED forces it on any such box (tests), DJG_FLAG_NO_FUSED or
    // DJG_NO_FUSED=1 keep the two-kernel step. Returns whether the box
    // qualifies (box_, box_grid_ set).
    bool detect_box(const int32_t* conn) {
        // DJ-TLED: f32 compact records (T4 rebuilt from X, H8 streamed);
        // TLED: T4, its B0 / V0 planes streamed or from the lattice table
        if ((sizeof(Real) != 4 && kind_ != DJG_T4) || n_slabs_ != 1 || win_) return false;  // (f64: T4)
        if (tled_ ? kind_ != DJG_T4 : !compact_) return false;
        if (kind_ == DJG_T4 && !tled_ && !X_.p) return false;
        if (model_ != DJG_NH && model_ != DJG_TI && model_ != DJG_OT) return false;
        if ((flags_ & DJG_FLAG_NO_FUSED) || (std::getenv("DJG_NO_FUSED") && std::atoi(std::getenv("DJG_NO_FUSED"))))
            return false;
        const bool forced = (flags_ & DJG_FLAG_FUSED) || (std::getenv("DJG_FUSED") && std::atoi(std::getenv("DJG_FUSED")));
        const bool t4 = kind_ == DJG_T4;
        const int per_cell = t4 ? 6 : 1, per = t4 ? 24 : 8;
        if (E_ < per_cell || E_ % per_cell || conn[0] != 0 || conn[1] != 1) return false;
        // T4 tet 0 runs corners 0 -> 1 -> 3 -> 7; H8 corners 0, 1, (1,1,0), (0,1,0), (0,0,1), ...
        const int64_t nx = int64_t(conn[2]) - 2;
        if (nx < 1) return false;
        const int64_t plane = t4 ? int64_t(conn[3]) - conn[2] : int64_t(conn[4]);
        if (plane % (nx + 1)) return false;
        const int64_t ny = plane / (nx + 1) - 1;
        if (ny < 1 || N_ % ((nx + 1) * (ny + 1))) return false;
        const int64_t nz = N_ / ((nx + 1) * (ny + 1)) - 1;
        if (nz < 1 || per_cell * nx * ny * nz != E_ || nx > INT32_MAX / 2 || ny > INT32_MAX / 2 || nz > INT32_MAX / 2)
            return false;
        const int32_t div[3] = {int32_t(nx), int32_t(ny), int32_t(nz)};
        bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
        for (int64_t c = 0; c < nx * ny * nz; ++c) {
            int32_t cc[24];
            box_cell_conn(t4 ? 0 : 1, div, c, cc);
            ok = ok && std::memcmp(cc, conn + c * per, size_t(per) * sizeof(int32_t)) == 0;
        }
        if (!ok) return false;
        box_.nx = int(nx);
        box_.ny = int(ny);
        box_.nz = int(nz);
        box_.tiles_x = int((nx + 1 + kBoxBX - 1) / kBoxBX);
        box_.tiles_y = int((ny + 1 + kBoxBY - 1) / kBoxBY);
        box_.lay0 = 0;
        box_.lay1 = int(nz + 1);
        box_.close = 1;
        int per_sm = 0;
        auto setup = [&](auto kern, size_t smem, int threads) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            int nb = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem));
            per_sm = per_sm == 0 ? nb : std::min(per_sm, nb);
        };
        {
            if (t4 && tled_) {
                using BS = BoxShape<kBoxBX, kBoxBY>;
                const size_t smem = BS::template smem_bytes<Real, false, true>();
                setup(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, false, true>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, false, true>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, false, true>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, true, true>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, true, true>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, true, true>, smem, BS::kThreads);
            } else if (t4) {
                using BS = BoxShape<kBoxBX, kBoxBY>;
                const size_t smem = BS::template smem_bytes<Real>(), lsmem = BS::template smem_bytes<Real, true>();
                setup(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, false>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, false>, smem, BS::kThreads);
                setup(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, false>, smem, BS::kThreads);
                // (the lattice variants: the same grid -- their smem is smaller)
                CK(cudaFuncSetAttribute(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsmem)));
                CK(cudaFuncSetAttribute(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsmem)));
                CK(cudaFuncSetAttribute(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsmem)));
            } else if constexpr (sizeof(Real) == 4) {
                using BS = BoxShapeH8<kBoxBX, kBoxBY>;
                const size_t smem = BS::template smem_bytes<Real>();
                setup(k_box_step_h8<Real, DJG_NH, kBoxBX, kBoxBY>, smem, BS::kThreads);
                setup(k_box_step_h8<Real, DJG_TI, kBoxBX, kBoxBY>, smem, BS::kThreads);
                setup(k_box_step_h8<Real, DJG_OT, kBoxBX, kBoxBY>, smem, BS::kThreads);
            }
        }
        if (per_sm < 1) return false;
        box_grid_ = per_sm * sms_;  // persistent: every block resident
        box_forced_ = forced;
        return true;
    }

    void launch_box(cudaStream_t s) { launch_box(s, box_); }

    // node layers [lay0, lay1) only; the last such launch of a step closes it
    void launch_box(cudaStream_t s, int lay0, int lay1, bool close) {
        BoxArgs b = box_;
        b.lay0 = lay0;
        b.lay1 = lay1;
        b.close = close ? 1 : 0;
        launch_box(s, b);
    }

    void launch_box(cudaStream_t s, const BoxArgs& box) {
        {
            const unsigned grid = unsigned(box_grid_);
            if (kind_ == DJG_T4) {
                using BS = BoxShape<kBoxBX, kBoxBY>;
                auto go = [&](auto kern, size_t smem) { kern<<<grid, BS::kThreads, smem, s>>>(ea_, na_, box); };
                if (tled_) {
                    const size_t smem = BS::template smem_bytes<Real, false, true>();
                    if (lattice_) {
                        switch (model_) {
                            case DJG_NH: go(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, true, true>, smem); break;
                            case DJG_TI: go(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, true, true>, smem); break;
                            default: go(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, true, true>, smem); break;
                        }
                    } else {
                        switch (model_) {
                            case DJG_NH: go(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, false, true>, smem); break;
                            case DJG_TI: go(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, false, true>, smem); break;
                            default: go(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, false, true>, smem); break;
                        }
                    }
                } else if (lattice_) {
                    const size_t smem = BS::template smem_bytes<Real, true>();
                    switch (model_) {
                        case DJG_NH: go(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, true>, smem); break;
                        case DJG_TI: go(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, true>, smem); break;
                        default: go(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, true>, smem); break;
                    }
                } else {
                    const size_t smem = BS::template smem_bytes<Real>();
                    switch (model_) {
                        case DJG_NH: go(k_box_step<Real, DJG_NH, kBoxBX, kBoxBY, false>, smem); break;
                        case DJG_TI: go(k_box_step<Real, DJG_TI, kBoxBX, kBoxBY, false>, smem); break;
                        default: go(k_box_step<Real, DJG_OT, kBoxBX, kBoxBY, false>, smem); break;
                    }
                }
            } else if constexpr (sizeof(Real) == 4) {
                using BS = BoxShapeH8<kBoxBX, kBoxBY>;
                const size_t smem = BS::template smem_bytes<Real>();
                switch (model_) {
                    case DJG_NH: k_box_step_h8<Real, DJG_NH, kBoxBX, kBoxBY><<<grid, BS::kThreads, smem, s>>>(ea_, na_, box); break;
                    case DJG_TI: k_box_step_h8<Real, DJG_TI, kBoxBX, kBoxBY><<<grid, BS::kThreads, smem, s>>>(ea_, na_, box); break;
                    default: k_box_step_h8<Real, DJG_OT, kBoxBX, kBoxBY><<<grid, BS::kThreads, smem, s>>>(ea_, na_, box); break;
                }
            }
            CK(cudaGetLastError());
        }
    }

    // Coordinate lattice (generate_box's nodes: x depends on i alone, y on j,
    // z on k): a tet's compact record is a function of its J0 alone, and J0
    // of tet t in cell (i, j, k) is built from the x / y / z rows of the
    // cell's two node planes per axis -- so cells whose three axis intervals
    // hold the same coordinate pairs up to the exact differences the rebuild
    // forms have the same six records. Axis classes: the pair ((0 + -a) + b,
    // (0 + -b) + a) of the interval's end coordinates a, b (the two J0
    // entries it can produce). k_lattice_table rebuilds the record of each
    // class triple once; k_lattice_verify then rebuilds every tet's record
    // and compares it bit for bit with its class's, and the fused step reads
    // the table (not the coordinates) only if all agree -- cfg5: 9 classes
    // per axis, 729 x 6 records (0.4 MB), against ~22 % of the step's
    // instructions. DJG_LATTICE=0 keeps the per-tet rebuild.
    void build_lattice(const Real* nodes) {
        {
            const char* v = std::getenv("DJG_LATTICE");
            if (v && std::atoi(v) == 0) return;
            const int64_t nx = box_.nx, ny = box_.ny, nz = box_.nz;
            auto gid = [&](int64_t i, int64_t j, int64_t k) { return i + (nx + 1) * (j + (ny + 1) * k); };
            std::vector<int32_t> cls(size_t(nx + ny + nz)), rep;
            std::vector<Real> len;  // each class's interval length (0 + -a) + b
            int ncl[3] = {0, 0, 0};
            const int64_t n[3] = {nx, ny, nz};
            int64_t off = 0;
            for (int ax = 0; ax < 3; ++ax) {
                std::map<std::pair<uint64_t, uint64_t>, int> ids;
                for (int64_t i = 0; i < n[ax]; ++i) {
                    const int64_t g0 = ax == 0 ? gid(i, 0, 0) : ax == 1 ? gid(0, i, 0) : gid(0, 0, i);
                    const int64_t g1 = ax == 0 ? gid(i + 1, 0, 0) : ax == 1 ? gid(0, i + 1, 0) : gid(0, 0, i + 1);
                    const Real a = nodes[3 * g0 + ax], b = nodes[3 * g1 + ax];
                    const Real fwd = (Real(0) + -a) + b, bwd = (Real(0) + -b) + a;
                    uint64_t kf = 0, kb = 0;
                    std::memcpy(&kf, &fwd, sizeof(Real));
                    std::memcpy(&kb, &bwd, sizeof(Real));
                    const auto [it, fresh] = ids.emplace(std::make_pair(kf, kb), int(ids.size()));
                    if (fresh) {
                        rep.push_back(int32_t(i));  // the class's first cell index
                        len.push_back(fwd);
                    }
                    cls[size_t(off + i)] = it->second;
                }
                ncl[ax] = int(ids.size());
                off += n[ax];
            }
            const int64_t ncomb = int64_t(ncl[0]) * ncl[1] * ncl[2];
            int nq = 0;
            switch (model_) {
                case DJG_NH: nq = kLatPlanes<Real, DJG_NH>; break;
                case DJG_TI: nq = kLatPlanes<Real, DJG_TI>; break;
                default: nq = kLatPlanes<Real, DJG_OT>; break;
            }
            if (tled_) nq = kTledPlanes<Real>;
            const size_t bytes = size_t(ncomb) * 6 * nq * sizeof(Plane);
            if (bytes > (size_t(16) << 20)) return;  // an irregular box: too many classes
            lcls_.alloc(cls.size() * sizeof(int32_t));
            CK(cudaMemcpy(lcls_.p, cls.data(), lcls_.bytes, cudaMemcpyHostToDevice));
            ld_.alloc(len.size() * sizeof(Real));
            CK(cudaMemcpy(ld_.p, len.data(), ld_.bytes, cudaMemcpyHostToDevice));
            DevBuf drep, bad;
            drep.alloc(rep.size() * sizeof(int32_t));
            CK(cudaMemcpy(drep.p, rep.data(), drep.bytes, cudaMemcpyHostToDevice));
            lat_.alloc(bytes);
            bad.alloc(sizeof(unsigned long long));
            CK(cudaMemset(bad.p, 0, bad.bytes));
            BoxArgs b = box_;
            b.lat = lat_.p;
            b.lcls = lcls_.as<int32_t>();
            b.ld = ld_.p;
            b.lncx = ncl[0];
            b.lncy = ncl[1];
            b.lncz = ncl[2];
            const unsigned tb = unsigned((ncomb * 6 + 127) / 128), vb = unsigned(sms_ * 8);
            auto run = [&](auto table, auto verify) {
                table<<<tb, 128>>>(ea_, b, drep.as<int32_t>(), lat_.as<Plane>());
                verify<<<vb, 256>>>(ea_, b, lat_.as<Plane>(), bad.as<unsigned long long>());
            };
            if (tled_) {
                // TLED: the records exist already (B0 / V0 planes): copy a
                // representative's, compare every tet's planes
                run(k_lattice_table_rec<Real>, k_lattice_verify_rec<Real>);
            } else {
                switch (model_) {
                    case DJG_NH: run(k_lattice_table<Real, DJG_NH>, k_lattice_verify<Real, DJG_NH>); break;
                    case DJG_TI: run(k_lattice_table<Real, DJG_TI>, k_lattice_verify<Real, DJG_TI>); break;
                    default: run(k_lattice_table<Real, DJG_OT>, k_lattice_verify<Real, DJG_OT>); break;
                }
            }
            CK(cudaGetLastError());
            unsigned long long nbad = 0;
            CK(cudaMemcpy(&nbad, bad.p, sizeof(nbad), cudaMemcpyDeviceToHost));
            if (nbad) {
                lat_.release();
                lcls_.release();
                ld_.release();
                return;
            }
            box_ = b;
            lattice_ = true;
        }
    }

    // (a part of a decomposition -- element ids mapped, inversions counted
    // per owner, ghost nodes -- keeps the two-kernel step)
    bool fused_now() const {
        return fused_ && na_.N == N_ && !peer_ && !comm_ && n_slabs_ == 1 && !ea_.elem_l2g && !ea_.counted;
    }

    // Uniform slices: when every 32-node slice given the widest row's width
    // costs at most 2 % more slots (the cube: 0.9 %), all slices get that
    // width, so slice_base[s] = 32 W s and the kernels compute a slot position
    // from the node id alone (ElemArgs / NodeArgs::slice_w) instead of
    // loading the slice base -- one gather less per element-node. The table
    // stays (other paths read it) and holds the same values.
    void uniform_slices() {
        const int64_t S = (N_ + 31) / 32;
        const int64_t ucap = int64_t(32) * wmax_ * S;
        const char* v = std::getenv("DJG_UNIFORM_SLICES");
        if ((v && std::atoi(v) == 0) || ucap > INT32_MAX || double(ucap) > 1.02 * double(capacity_)) return;
        for (int64_t sl = 0; sl <= S; ++sl) slice_base_[size_t(sl)] = int32_t(int64_t(32) * wmax_ * sl);
        capacity_ = std::max<int64_t>(ucap, 32);
        slice_w_ = wmax_;
    }

    // Node windows of the 128-element tiles (k_element_win, kernels.cuh): per
    // tile the distinct node ids as at most kWinRuns runs (ids closer than
    // kGap are merged: a few unused rows are cheaper than another copy) and
    // at most kWinCap nodes, else the tile is flagged for the global gather;
    // per element-node its index in the window; and the slot position of
    // every element-node (device, from the ranks and slice bases).
    void build_windows(const int32_t* conn) {
        constexpr int kGap = 8;
        const int npe = npe_;
        const int cap = kind_ == DJG_H8 ? kWinCap<1> : kWinCap<0>;
        const int lb = kind_ == DJG_H8 ? kWinIdxBytes<1> : kWinIdxBytes<0>;
        const int64_t ntiles = (E_ + kPipeTile - 1) / kPipeTile;
        std::vector<int32_t> desc(size_t(ntiles) * kWinDesc, 0);
        std::vector<uint8_t> idx(size_t(E_) * size_t(npe * lb) + 16, 0);
        int64_t fit = 0;
        const bool force_fallback = std::getenv("DJG_WIN_FORCE_FALLBACK") != nullptr;  // (A/B diagnosis)
#pragma omp parallel reduction(+ : fit)
        {
            std::vector<int32_t> ids;
            ids.reserve(size_t(kPipeTile * npe));
#pragma omp for schedule(dynamic, 512)
            for (int64_t t = 0; t < ntiles; ++t) {
                const int64_t eb = t * kPipeTile, ee = std::min<int64_t>(E_, eb + kPipeTile);
                ids.assign(conn + eb * npe, conn + ee * npe);
                std::sort(ids.begin(), ids.end());
                ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
                int32_t rs[kWinRuns], ro[kWinRuns];
                int nr = 0, total = 0;
                bool ok = true;
                for (size_t i = 0; i < ids.size() && ok;) {
                    size_t j = i + 1;
                    while (j < ids.size() && ids[j] - ids[j - 1] <= kGap) ++j;
                    const int len = ids[j - 1] - ids[i] + 1;
                    if (nr == kWinRuns || total + len > cap) {
                        ok = false;
                    } else {
                        rs[nr] = ids[i];
                        ro[nr] = total;
                        total += len;
                        ++nr;
                    }
                    i = j;
                }
                if (!ok || force_fallback) continue;  // nruns = 0: global gather
                int32_t* d = desc.data() + size_t(t) * kWinDesc;
                d[0] = nr;
                d[1] = total;
                for (int r = 0; r < nr; ++r) {
                    d[2 + 2 * r] = rs[r];
                    d[3 + 2 * r] = ro[r];
                }
                for (int64_t e = eb; e < ee; ++e)
                    for (int a = 0; a < npe; ++a) {
                        const int32_t n = conn[e * npe + a];
                        int r = nr - 1;
                        while (rs[r] > n) --r;
                        const int w = ro[r] + (n - rs[r]);
                        uint8_t* q = idx.data() + size_t(e * npe + a) * size_t(lb);
                        q[0] = uint8_t(w & 0xff);
                        if (lb == 2) q[1] = uint8_t(w >> 8);
                    }
                ++fit;
            }
        }
        win_tiles_ = fit;
        wdesc_.alloc(desc.size() * sizeof(int32_t));
        CK(cudaMemcpy(wdesc_.p, desc.data(), wdesc_.bytes, cudaMemcpyHostToDevice));
        widx_.alloc(idx.size());
        CK(cudaMemcpy(widx_.p, idx.data(), widx_.bytes, cudaMemcpyHostToDevice));
        slot_.alloc(size_t(E_) * size_t(npe) * sizeof(int32_t));
        const unsigned grid = unsigned((E_ + 255) / 256);
        if (rank_bytes_ == 1)
            k_slot_planes<1><<<grid, 256>>>(conn_.as<int4>(), rank_.p, slicebase_.as<int>(), E_, npe, slot_.as<int4>());
        else
            k_slot_planes<2><<<grid, 256>>>(conn_.as<int4>(), rank_.p, slicebase_.as<int>(), E_, npe, slot_.as<int4>());
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        ea_.slot = slot_.as<int4>();
        ea_.widx = widx_.p;
        ea_.wdesc = wdesc_.as<int>();
    }

    // Step data: UpdateCoeffs (c1 per node, massless, c2, c3), DofConstraints
    // (kind / target / t_total per DOF) and dt (solver.hpp:18-39, 64-87).
    void configure(const Real* c1, const uint8_t* massless, const uint8_t* dof_kind, const Real* target,
                   const Real* t_total, Real c2, Real c3, Real dt) {
        std::vector<uint8_t> code(static_cast<size_t>(N_));
        for (int64_t n = 0; n < N_; ++n) {
            uint8_t c = 0;
            for (int i = 0; i < 3; ++i) {
                const uint8_t k = dof_kind ? dof_kind[3 * n + i] : uint8_t(DJG_FREE);
                if (k > 2) throw DescError("invalid DOF kind");
                c |= uint8_t(k << (2 * i));
            }
            if (massless[n]) c |= 1u << 6;
            code[size_t(n)] = c;
        }
        CK(cudaMemcpy(code_.p, code.data(), code_.bytes, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c1_.p, c1, c1_.bytes, cudaMemcpyHostToDevice));
        if (target) {
            CK(cudaMemcpy(target_.p, target, target_.bytes, cudaMemcpyHostToDevice));
        } else {
            CK(cudaMemset(target_.p, 0, target_.bytes));
        }
        if (t_total) {
            CK(cudaMemcpy(tTotal_.p, t_total, tTotal_.bytes, cudaMemcpyHostToDevice));
        } else {
            std::vector<Real> ones(size_t(3 * N_), Real(1));
            CK(cudaMemcpy(tTotal_.p, ones.data(), tTotal_.bytes, cudaMemcpyHostToDevice));
        }
        na_.c2 = c2;
        na_.c3 = c3;
        na_.dt = dt;
        configured_ = true;
        drop_graphs();
    }

    // UpdateCoeffs::build from node masses (solver.hpp:70-86), same Real ops.
    void configure_step(const djg_step_desc& s) override {
        if (!s.node_mass) throw DescError("node_mass is required");
        const Real dt = Real(s.dt), alpha = Real(s.alpha);
        if (!(dt > Real(0))) throw DescError("time step must be positive");
        const Real* m = static_cast<const Real*>(s.node_mass);
        const Real denom = Real(1) + alpha * dt / 2;
        const Real c2 = Real(2) / denom;
        const Real c3 = -(Real(1) - alpha * dt / 2) / denom;
        std::vector<Real> c1(static_cast<size_t>(N_), Real(0));
        std::vector<uint8_t> massless(static_cast<size_t>(N_), 0);
        for (int64_t n = 0; n < N_; ++n) {
            if (m[n] > Real(0)) c1[size_t(n)] = dt * dt / (m[n] * denom);
            else massless[size_t(n)] = 1;
        }
        configure(c1.data(), massless.data(), s.dof_kind, static_cast<const Real*>(s.dof_target),
                  static_cast<const Real*>(s.dof_t_total), c2, c3, dt);
    }

    // Multi-GPU: only nodes [0, num_owned) are gathered and updated; ghost
    // nodes come from the halo. Inverted elements are reported in global ids.
    void set_partition(int64_t num_owned, const int64_t* elem_l2g) override {
        if (num_owned < 0 || num_owned > N_) throw DescError("num_owned out of range");
        na_.N = num_owned;
        if (!mailbox_.p) {
            mailbox_.alloc(sizeof(Mailbox));
            CK(cudaMemset(mailbox_.p, 0, mailbox_.bytes));
        }
        if (elem_l2g) {
            elemL2g_.alloc(size_t(E_) * sizeof(int64_t));
            CK(cudaMemcpy(elemL2g_.p, elem_l2g, elemL2g_.bytes, cudaMemcpyHostToDevice));
            ea_.elem_l2g = elemL2g_.as<long long>();
        }
        drop_graphs();
    }

    // Multi-part inversion counting (djg_set_counted_elements): only this
    // part's own elements are counted; the parts' step counts are summed by
    // the agreement (k_agree / k_wait_agree) into every part's totals.
    void set_counted_elements(const uint8_t* counted) override {
        if (!counted) throw DescError("counted elements missing");
        counted_.alloc(size_t(E_));
        CK(cudaMemcpy(counted_.p, counted, size_t(E_), cudaMemcpyHostToDevice));
        ea_.counted = counted_.as<unsigned char>();
        multipart_ = true;
        read_ctrl();
        hctrl_->multipart = 1;
        CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));
        drop_graphs();
    }

    void set_halo(int64_t nsend, const int32_t* send, int64_t nrecv, const int32_t* recv) override {
        auto up = [&](DevBuf& b, int64_t n, const int32_t* v) {
            for (int64_t i = 0; i < n; ++i)
                if (v[i] < 0 || v[i] >= N_) throw DescError("halo node index out of range");
            b.alloc(size_t(std::max<int64_t>(n, 1)) * sizeof(int32_t));
            if (n) CK(cudaMemcpy(b.p, v, size_t(n) * sizeof(int32_t), cudaMemcpyHostToDevice));
        };
        up(haloSend_, nsend, send);
        up(haloRecv_, nrecv, recv);
        nsend_ = nsend;
        nrecv_ = nrecv;
    }

    void halo_pack(void* dev_out) override {
        if (nsend_ == 0) return;
        k_halo_pack<Real><<<unsigned((nsend_ + 255) / 256), 256, 0, stream_>>>(
            ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloSend_.as<int>(), nsend_,
            static_cast<Node*>(dev_out));
        CK(cudaGetLastError());
    }

    void halo_unpack(const void* dev_in) override {
        if (nrecv_ == 0) return;
        k_halo_unpack<Real><<<unsigned((nrecv_ + 255) / 256), 256, 0, stream_>>>(
            ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloRecv_.as<int>(), nrecv_,
            static_cast<const Node*>(dev_in));
        CK(cudaGetLastError());
    }

    void step_status(int64_t* dev_status) override {
        if (!elemL2g_.p) throw DescError("step_status needs djg_set_partition with elem_l2g");
        k_step_status<<<1, 1, 0, stream_>>>(ctrl_.as<Ctrl>(), elemL2g_.as<long long>(),
                                            reinterpret_cast<long long*>(dev_status));
        CK(cudaGetLastError());
    }

    void step_agree(const int64_t* dev_reduced) override {
        k_agree<<<1, 1, 0, stream_>>>(ctrl_.as<Ctrl>(), reinterpret_cast<const long long*>(dev_reduced));
        CK(cudaGetLastError());
    }

    // Multi-GPU step driven by the engine itself: after djg_set_partition /
    // djg_set_halo, a communicator over the ranks and the per-neighbour halo
    // offsets. Every step then enqueues -- and CUDA-graph captures -- the
    // element and node kernels, the halo pack, one grouped NCCL send/recv per
    // neighbour, the unpack, the failure status, its allreduce(MAX) and the
    // agreement: no host round trip per step.
    void comm_init(const void* id, int nranks, int rank, int nnb, const int32_t* nb, const int64_t* send_off,
                   const int64_t* recv_off) override {
        if (!elemL2g_.p) throw DescError("djg_comm_init needs djg_set_partition with elem_l2g first");
        if (nranks < 1 || rank < 0 || rank >= nranks || nnb < 0) throw DescError("invalid rank / neighbour count");
        if (nnb > 0 && (!nb || !send_off || !recv_off)) throw DescError("neighbour lists missing");
        nbr_.assign(nb, nb + nnb);
        send_off_.assign(send_off, send_off + (nnb ? nnb + 1 : 0));
        recv_off_.assign(recv_off, recv_off + (nnb ? nnb + 1 : 0));
        for (int k = 0; k < nnb; ++k)
            if (nbr_[size_t(k)] < 0 || nbr_[size_t(k)] >= nranks || nbr_[size_t(k)] == rank)
                throw DescError("invalid neighbour rank");
        if (nnb && (send_off_.front() != 0 || send_off_.back() != nsend_ || recv_off_.front() != 0 ||
                    recv_off_.back() != nrecv_))
            throw DescError("halo offsets do not match djg_set_halo");
        const Nccl& api = Nccl::get();
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        CK(cudaSetDevice(device_));
        if (comm_) api.comm_destroy(static_cast<ncclComm_t>(comm_));
        ncclComm_t c = nullptr;
        NK(api.comm_init_rank(&c, nranks, uid, rank));
        comm_ = c;
        if (!side_) {
            CK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&evFork_, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&evJoin_, cudaEventDisableTiming));
        }
        sendBuf_.alloc(size_t(std::max<int64_t>(nsend_, 1)) * sizeof(Node));
        recvBuf_.alloc(size_t(std::max<int64_t>(nrecv_, 1)) * sizeof(Node));
        status_.alloc(3 * sizeof(int64_t));
        drop_graphs();
    }

    void launch_exchange(cudaStream_t s) {
        const Nccl& api = Nccl::get();
        ncclComm_t c = static_cast<ncclComm_t>(comm_);
        constexpr int kPer = int(sizeof(Node) / sizeof(Real));  // Reals per halo row
        const ncclDataType_t dt = sizeof(Real) == 4 ? ncclFloat32 : ncclFloat64;
        if (nsend_) {
            k_halo_pack<Real><<<unsigned((nsend_ + 255) / 256), 256, 0, s>>>(
                ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloSend_.as<int>(), nsend_,
                sendBuf_.as<Node>());
            CK(cudaGetLastError());
        }
        if (!nbr_.empty()) {
            NK(api.group_start());
            for (size_t k = 0; k < nbr_.size(); ++k) {
                const int64_t s0 = send_off_[k], s1 = send_off_[k + 1], r0 = recv_off_[k], r1 = recv_off_[k + 1];
                if (s1 > s0) NK(api.send(sendBuf_.as<Node>() + s0, size_t(s1 - s0) * kPer, dt, nbr_[k], c, s));
                if (r1 > r0) NK(api.recv(recvBuf_.as<Node>() + r0, size_t(r1 - r0) * kPer, dt, nbr_[k], c, s));
            }
            NK(api.group_end());
        }
        if (nrecv_) {
            k_halo_unpack<Real><<<unsigned((nrecv_ + 255) / 256), 256, 0, s>>>(
                ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloRecv_.as<int>(), nrecv_,
                recvBuf_.as<Node>());
            CK(cudaGetLastError());
        }
        k_step_status<<<1, 1, 0, s>>>(ctrl_.as<Ctrl>(), elemL2g_.as<long long>(), status_.as<long long>());
        NK(api.all_reduce(status_.p, status_.p, 2, ncclInt64, ncclMax, c, s));
        NK(api.all_reduce(status_.as<long long>() + 2, status_.as<long long>() + 2, 1, ncclInt64, ncclSum, c, s));
        k_agree<<<1, 1, 0, s>>>(ctrl_.as<Ctrl>(), status_.as<long long>());
        CK(cudaGetLastError());
    }

    // ---- overlapped multi-part step: pack -> {interior elements || halo
    // exchange} -> unpack -> boundary elements -> node update -> status /
    // agreement. Local elements [0, split) reference no ghost node
    // (djg_set_interior; the partition builder orders them first).
    int64_t split_point() const { return interior_ < 0 ? E_ : interior_; }

    void set_interior(int64_t n) override {
        if (n < 0 || n > E_) throw DescError("interior element count out of range");
        if (n_slabs_ != 1) throw DescError("the split step needs the one-slab schedule");
        interior_ = n / kPipeTile * kPipeTile;  // tile-aligned ranges for the bulk copies
        drop_graphs();
    }

    void launch_pack(cudaStream_t s, Node* out) {
        if (!nsend_) return;
        k_halo_pack<Real><<<unsigned((nsend_ + 255) / 256), 256, 0, s>>>(
            ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloSend_.as<int>(), nsend_, out);
        CK(cudaGetLastError());
    }

    void launch_unpack(cudaStream_t s, const Node* in) {
        if (!nrecv_) return;
        k_halo_unpack<Real><<<unsigned((nrecv_ + 255) / 256), 256, 0, s>>>(
            ctrl_.as<Ctrl>(), u_[0].as<Node>(), u_[1].as<Node>(), u_[2].as<Node>(), haloRecv_.as<int>(), nrecv_, in);
        CK(cudaGetLastError());
    }

    void step_interior() override {
        if (!configured_) throw DescError("step data not configured (djg_configure_step)");
        // a step starts here: sync() reports from this point (as djg_step_async)
        CK(cudaMemcpyAsync(hstart_, ctrl_.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream_));
        launch_element(stream_, 0, split_point());
    }

    void step_boundary() override {
        launch_element(stream_, split_point(), E_);
        launch_node(stream_, 0, false);
    }

    // One overlapped step with the engine's NCCL communicator (captured).
    void launch_overlapped_step(cudaStream_t s) {
        const Nccl& api = Nccl::get();
        ncclComm_t c = static_cast<ncclComm_t>(comm_);
        constexpr int kPer = int(sizeof(Node) / sizeof(Real));
        const ncclDataType_t dt = sizeof(Real) == 4 ? ncclFloat32 : ncclFloat64;
        launch_pack(s, sendBuf_.as<Node>());
        CK(cudaEventRecord(evFork_, s));
        CK(cudaStreamWaitEvent(side_, evFork_, 0));
        pipe_spare_sms_ = kSpareSms;  // leave SMs for the NCCL kernels
        launch_element(side_, 0, split_point());
        pipe_spare_sms_ = 0;
        NK(api.group_start());
        for (size_t k = 0; k < nbr_.size(); ++k) {
            const int64_t s0 = send_off_[k], s1 = send_off_[k + 1], r0 = recv_off_[k], r1 = recv_off_[k + 1];
            if (s1 > s0) NK(api.send(sendBuf_.as<Node>() + s0, size_t(s1 - s0) * kPer, dt, nbr_[k], c, s));
            if (r1 > r0) NK(api.recv(recvBuf_.as<Node>() + r0, size_t(r1 - r0) * kPer, dt, nbr_[k], c, s));
        }
        NK(api.group_end());
        launch_unpack(s, recvBuf_.as<Node>());
        CK(cudaEventRecord(evJoin_, side_));
        CK(cudaStreamWaitEvent(s, evJoin_, 0));
        launch_element(s, split_point(), E_);
        launch_node(s, 0, false);
        k_step_status<<<1, 1, 0, s>>>(ctrl_.as<Ctrl>(), elemL2g_.as<long long>(), status_.as<long long>());
        NK(api.all_reduce(status_.p, status_.p, 2, ncclInt64, ncclMax, c, s));
        NK(api.all_reduce(status_.as<long long>() + 2, status_.as<long long>() + 2, 1, ncclInt64, ncclSum, c, s));
        k_agree<<<1, 1, 0, s>>>(ctrl_.as<Ctrl>(), status_.as<long long>());
        CK(cudaGetLastError());
    }

    // ---- peer-memory multi-GPU step (kernels.cuh: k_node_peer, k_wait_agree)
    void peer_export(void** ptrs) override {
        if (!mailbox_.p) throw DescError("djg_set_partition first");
        for (int i = 0; i < 3; ++i) ptrs[i] = u_[i].p;
        ptrs[3] = mailbox_.p;
    }

    void peer_ipc_export(void* handles) override {
        if (!mailbox_.p) throw DescError("djg_set_partition first");
        auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
        for (int i = 0; i < 3; ++i) CK(cudaIpcGetMemHandle(h + i, u_[i].p));
        CK(cudaIpcGetMemHandle(h + 3, mailbox_.p));
    }

    void peer_ipc_open(const void* handles, void** ptrs) override {
        const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
        CK(cudaSetDevice(device_));
        for (int i = 0; i < 4; ++i) {
            CK(cudaIpcOpenMemHandle(&ptrs[i], h[i], cudaIpcMemLazyEnablePeerAccess));
            ipc_open_.push_back(ptrs[i]);
        }
    }

    void peer_setup(int nparts, int part, const void* const* peer_u, const void* const* peer_mail,
                    const int64_t* peer_num_nodes, int64_t ndest, const int32_t* dest_node, const int32_t* dest_part,
                    const int32_t* dest_index) override {
        if (!elemL2g_.p || !mailbox_.p) throw DescError("djg_peer_setup needs djg_set_partition with elem_l2g first");
        if (nparts < 1 || nparts > kMaxParts || part < 0 || part >= nparts) throw DescError("invalid part count / index");
        if (!peer_num_nodes || peer_num_nodes[part] != N_) throw DescError("peer node counts missing or inconsistent");
        const int64_t no = na_.N;
        std::vector<int32_t> off(size_t(no) + 1, 0);
        for (int64_t i = 0; i < ndest; ++i) {
            if (dest_node[i] < 0 || dest_node[i] >= no) throw DescError("halo destination of a non-owned node");
            if (dest_part[i] < 0 || dest_part[i] >= nparts || dest_part[i] == part) throw DescError("invalid peer part");
            // the node kernel stores through peer_u[dest_part] + dest_index: keep it inside that buffer
            if (dest_index[i] < 0 || dest_index[i] >= peer_num_nodes[dest_part[i]])
                throw DescError("halo destination index outside the peer's node range");
            off[size_t(dest_node[i]) + 1]++;
        }
        for (int64_t n = 0; n < no; ++n) off[size_t(n) + 1] += off[size_t(n)];
        std::vector<int2> dst(static_cast<size_t>(std::max<int64_t>(ndest, 1)));
        std::vector<int32_t> cur(off.begin(), off.end() - 1);
        for (int64_t i = 0; i < ndest; ++i) dst[size_t(cur[size_t(dest_node[i])]++)] = make_int2(dest_part[i], dest_index[i]);
        destOff_.alloc(off.size() * sizeof(int32_t));
        CK(cudaMemcpy(destOff_.p, off.data(), destOff_.bytes, cudaMemcpyHostToDevice));
        dest_.alloc(dst.size() * sizeof(int2));
        CK(cudaMemcpy(dest_.p, dst.data(), dest_.bytes, cudaMemcpyHostToDevice));
        peerU_.alloc(size_t(3 * nparts) * sizeof(void*));
        CK(cudaMemcpy(peerU_.p, peer_u, peerU_.bytes, cudaMemcpyHostToDevice));
        peerMail_.alloc(size_t(nparts) * sizeof(void*));
        CK(cudaMemcpy(peerMail_.p, peer_mail, peerMail_.bytes, cudaMemcpyHostToDevice));
        pa_.dest_off = destOff_.as<int>();
        pa_.dest = dest_.as<int2>();
        pa_.peer_u = peerU_.as<Node*>();
        pa_.peer_mail = peerMail_.as<Mailbox*>();
        pa_.nparts = nparts;
        pa_.part = part;
        peer_ = true;
        if (const char* v = std::getenv("DJG_PEER_TIMEOUT_MS")) peer_timeout_ns_ = std::strtoull(v, nullptr, 10) * 1000000ull;
        drop_graphs();
    }

    void launch_peer_local(cudaStream_t s) {
        launch_element(s, 0, E_);
        const int64_t blocks = std::max<int64_t>(1, (na_.N + 255) / 256);
        const unsigned g = unsigned(node_grid_ > 0 ? std::min<int64_t>(blocks, node_grid_) : blocks);
        k_node_peer<Real><<<g, 256, 0, s>>>(na_, pa_);
        CK(cudaGetLastError());
    }

    void launch_peer_agree(cudaStream_t s) {
        k_wait_agree<<<1, 32, 0, s>>>(ctrl_.as<Ctrl>(), mailbox_.as<Mailbox>(), pa_.nparts, peer_timeout_ns_);
        CK(cudaGetLastError());
    }

    void step_peer_local() override {
        if (!peer_) throw DescError("djg_peer_setup first");
        if (!configured_) throw DescError("step data not configured (djg_configure_step)");
        CK(cudaMemcpyAsync(hstart_, ctrl_.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream_));  // (see step_interior)
        launch_peer_local(stream_);
    }

    void step_peer_agree() override {
        if (!peer_) throw DescError("djg_peer_setup first");
        launch_peer_agree(stream_);
    }

    void set_policy(int policy) override {
        if (policy != DJG_ABORT && policy != DJG_SKIP_AND_REPORT) throw DescError("unknown inversion policy");
        policy_ = policy;
        na_.policy = policy;
        drop_graphs();
    }

    // Slab schedule (kernels.cuh, k_node_slices): elements are cut into slabs
    // whose force rows fit in L2; every 32-node slice is gathered right after
    // the slab holding its last (highest-id) element.
    // Slot layout on the device (see k_count_nodes): CSR rows, ranks, slices,
    // connectivity planes. Keeps the sorted pairs and row offsets for
    // mass_and_length_device.
    void build_layout_device(const int32_t* conn_h) {
        const int npe = npe_;
        const int64_t P = E_ * npe;
        const unsigned gp = unsigned((P + 255) / 256);
        DevBuf conn, cnt, bad, vals_in, keys_out, rank_of_pair, tmp;
        conn.alloc(size_t(P) * 4);
        CK(cudaMemcpy(conn.p, conn_h, conn.bytes, cudaMemcpyHostToDevice));
        cnt.alloc(size_t(N_ + 1) * 4);
        CK(cudaMemset(cnt.p, 0, cnt.bytes));
        bad.alloc(4);
        CK(cudaMemset(bad.p, 0, 4));
        k_count_nodes<<<gp, 256>>>(conn.as<int>(), P, N_, cnt.as<int>(), bad.as<int>());
        CK(cudaGetLastError());
        int hbad = 0;
        CK(cudaMemcpy(&hbad, bad.p, 4, cudaMemcpyDeviceToHost));
        if (hbad) throw DescError("connectivity index out of range");
        // row offsets (int32: E * npe <= INT32_MAX is checked above)
        rowoff_.alloc(size_t(N_ + 1) * 4);
        size_t tb = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<int>(), rowoff_.as<int>(), int(N_ + 1)));
        tmp.alloc(tb);
        CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<int>(), rowoff_.as<int>(), int(N_ + 1)));
        // stable sort of pair indices by node
        vals_in.alloc(size_t(P) * 4);
        keys_out.alloc(size_t(P) * 4);
        pairs_.alloc(size_t(P) * 4);
        k_iota<<<gp, 256>>>(vals_in.as<int>(), P);
        int bits = 1;
        while ((int64_t(1) << bits) < N_) ++bits;
        size_t sb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, sb, conn.as<int>(), keys_out.as<int>(), vals_in.as<int>(),
                                           pairs_.as<int>(), P, 0, bits));
        DevBuf stmp;
        stmp.alloc(sb);
        CK(cub::DeviceRadixSort::SortPairs(stmp.p, sb, conn.as<int>(), keys_out.as<int>(), vals_in.as<int>(),
                                           pairs_.as<int>(), P, 0, bits));
        rank_of_pair.alloc(size_t(P) * 4);
        k_ranks_from_sorted<<<gp, 256>>>(keys_out.as<int>(), pairs_.as<int>(), rowoff_.as<int>(), P,
                                         rank_of_pair.as<int>());
        CK(cudaGetLastError());
        // widest row
        DevBuf dmax;
        dmax.alloc(4);
        size_t mb = 0;
        CK(cub::DeviceReduce::Max(nullptr, mb, cnt.as<int>(), dmax.as<int>(), int(N_)));
        DevBuf mtmp;
        mtmp.alloc(mb);
        CK(cub::DeviceReduce::Max(mtmp.p, mb, cnt.as<int>(), dmax.as<int>(), int(N_)));
        int wmax = 0;
        CK(cudaMemcpy(&wmax, dmax.p, 4, cudaMemcpyDeviceToHost));
        wmax_ = std::max(wmax, 1);
        if (wmax_ > 65535) throw DescError("a node has more than 65535 incident elements");
        rank_bytes_ = wmax_ <= 256 ? 1 : 2;
        // slices: slice_base = exclusive scan of 32 x widest row
        const int64_t S = (N_ + 31) / 32;
        DevBuf caps, base64;
        caps.alloc(size_t(S + 1) * 8);
        base64.alloc(size_t(S + 1) * 8);
        k_slice_caps<<<unsigned((S + 1 + 255) / 256), 256>>>(cnt.as<int>(), N_, caps.as<long long>());
        size_t cb = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, cb, caps.as<long long>(), base64.as<long long>(), int(S + 1)));
        DevBuf ctmp;
        ctmp.alloc(cb);
        CK(cub::DeviceScan::ExclusiveSum(ctmp.p, cb, caps.as<long long>(), base64.as<long long>(), int(S + 1)));
        long long cap = 0;
        CK(cudaMemcpy(&cap, base64.as<long long>() + S, 8, cudaMemcpyDeviceToHost));
        if (cap > INT32_MAX) throw DescError("slot buffer exceeds 32-bit indexing");
        capacity_ = std::max<int64_t>(cap, 32);
        slicebase_.alloc(size_t(S + 1) * 4);
        k_narrow_i64<<<unsigned((S + 1 + 255) / 256), 256>>>(base64.as<long long>(), S + 1, slicebase_.as<int>());
        slice_base_.resize(size_t(S + 1));
        CK(cudaMemcpy(slice_base_.data(), slicebase_.p, slicebase_.bytes, cudaMemcpyDeviceToHost));
        uniform_slices();
        CK(cudaMemcpy(slicebase_.p, slice_base_.data(), slicebase_.bytes, cudaMemcpyHostToDevice));
        rank_.alloc(size_t(P) * size_t(rank_bytes_) + 16);
        k_pack_ranks<<<gp, 256>>>(rank_of_pair.as<int>(), P, rank_bytes_, static_cast<unsigned char*>(rank_.p));
        conn_.alloc(size_t(P) * 4);
        k_conn_planes<<<unsigned((E_ + 255) / 256), 256>>>(conn.as<int>(), E_, npe, conn_.as<int>());
        rowlen_.alloc(size_t(N_) * 4);
        CK(cudaMemcpy(rowlen_.p, cnt.p, rowlen_.bytes, cudaMemcpyDeviceToDevice));
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        // one slab: the whole mesh
        slab_off_ = {0, int(S)};
        slab_elems_ = E_;
        n_slabs_ = 1;
    }

    // lump_mass (precompute.hpp:275-287) and the minimum characteristic
    // length of critical_dt (precompute.hpp:303-331) on the device, from the
    // coordinates and the sorted CSR pairs; frees the pairs.
    void mass_and_length_device(double rho) {
        DevBuf v0, len, lmin, tmp;
        v0.alloc(size_t(E_) * sizeof(Real));
        len.alloc(size_t(E_) * sizeof(Real));
        ElemArgs<Real> a{};
        a.E = E_;
        a.conn = conn_.as<int4>();
        a.X = X_.as<Node>();
        const unsigned ge = unsigned((E_ + 127) / 128);
        if (kind_ == DJG_T4) k_volume_length<Real, 0><<<ge, 128>>>(a, v0.as<Real>(), len.as<Real>());
        else k_volume_length<Real, 1><<<ge, 128>>>(a, v0.as<Real>(), len.as<Real>());
        CK(cudaGetLastError());
        lmin.alloc(sizeof(Real));
        size_t tb = 0;
        CK(cub::DeviceReduce::Min(nullptr, tb, len.as<Real>(), lmin.as<Real>(), int(E_)));
        tmp.alloc(tb);
        CK(cub::DeviceReduce::Min(tmp.p, tb, len.as<Real>(), lmin.as<Real>(), int(E_)));
        Real h = 0;
        CK(cudaMemcpy(&h, lmin.p, sizeof(Real), cudaMemcpyDeviceToHost));
        lmin_ = h;
        mass_.alloc(size_t(N_) * sizeof(Real));
        k_lump_mass<Real><<<unsigned((N_ + 255) / 256), 256>>>(pairs_.as<int>(), rowoff_.as<int>(), N_, npe_,
                                                                v0.as<Real>(), Real(rho), mass_.as<Real>());
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        pairs_.release();
        rowoff_.release();
    }

    int lump_mass(void* out) override {
        if (!mass_.p) throw DescError("lump_mass on the device needs an engine built with DJG_FLAG_DEVICE_PRECOMPUTE "
                                      "and no caller CSR");
        CK(cudaMemcpy(out, mass_.p, mass_.bytes, cudaMemcpyDeviceToHost));
        return DJG_OK;
    }

    int min_char_length(double* out) override {
        if (!mass_.p) throw DescError("the characteristic length on the device needs an engine built with "
                                      "DJG_FLAG_DEVICE_PRECOMPUTE and no caller CSR");
        if (!(lmin_ > Real(0))) throw DescError("degenerate element with zero characteristic length");
        *out = double(lmin_);
        return DJG_OK;
    }

    void plan_slabs(const int64_t* off, const int64_t* celem) {
        int64_t se = E_;
        if ((flags_ & DJG_FLAG_SLABS) || slab_bytes_ > 0) {
            const int64_t bytes = slab_bytes_ > 0 ? slab_bytes_ : kSlabBytes;
            se = std::max<int64_t>(1024, bytes / (int64_t(npe_) * int64_t(sizeof(Node))));
            se = (se + 127) / 128 * 128;
        }
        const int64_t S = std::max<int64_t>(1, (E_ + se - 1) / se);
        const int64_t nS = (N_ + 31) / 32;
        std::vector<int> slab_of(static_cast<size_t>(nS), 0);
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < nS; ++j) {
            int64_t last = -1;
            for (int64_t n = j * 32; n < std::min<int64_t>(N_, (j + 1) * 32); ++n)
                if (off[n + 1] > off[n]) last = std::max<int64_t>(last, celem[off[n + 1] - 1]);
            slab_of[size_t(j)] = last < 0 ? 0 : int(last / se);
        }
        std::vector<int> cnt(static_cast<size_t>(S) + 1, 0), list(static_cast<size_t>(nS));
        for (int64_t j = 0; j < nS; ++j) cnt[size_t(slab_of[size_t(j)]) + 1]++;
        for (int64_t q = 0; q < S; ++q) cnt[size_t(q + 1)] += cnt[size_t(q)];
        slab_off_ = cnt;
        std::vector<int> cur(cnt.begin(), cnt.end() - 1);
        for (int64_t j = 0; j < nS; ++j) list[size_t(cur[size_t(slab_of[size_t(j)])]++)] = int(j);
        slabSlices_.alloc(list.size() * sizeof(int));
        CK(cudaMemcpy(slabSlices_.p, list.data(), slabSlices_.bytes, cudaMemcpyHostToDevice));
        slab_elems_ = se;
        n_slabs_ = int(S);
    }

    ~Engine() override {
        if (comm_) Nccl::get().comm_destroy(static_cast<ncclComm_t>(comm_));
        for (void* p : ipc_open_) cudaIpcCloseMemHandle(p);
        if (evFork_) cudaEventDestroy(evFork_);
        if (evPrev_) cudaEventDestroy(evPrev_);
        if (down_) cudaStreamDestroy(down_);
        for (auto e : evChunk_) cudaEventDestroy(e);
        for (auto e : evBox_) cudaEventDestroy(e);
        if (evJoin_) cudaEventDestroy(evJoin_);
        if (side_) cudaStreamDestroy(side_);
        if (side2_) cudaStreamDestroy(side2_);
        if (graph_big_) cudaGraphExecDestroy(graph_big_);
        if (graph_one_) cudaGraphExecDestroy(graph_one_);
        if (hctrl_) cudaFreeHost(hctrl_);
        if (hstart_) cudaFreeHost(hstart_);
        if (stream_) cudaStreamDestroy(stream_);
    }

    cudaStream_t stream() const override { return stream_; }

    void reset_ctrl(int64_t step) {
        unsigned epoch = 0;
        if (ctrl_initialized_) {
            read_ctrl();
            epoch = hctrl_->epoch;  // flags carry epoch stamps: never move backwards
        }
        ctrl_initialized_ = true;
        Ctrl c{};
        c.epoch = epoch;
        c.multipart = multipart_ ? 1 : 0;
        c.step = step;
        c.first_inv = kNone;
        c.asm_first = kNone;
        c.halt_first_inv = -1;
        c.fail_step = -1;
        *hctrl_ = c;
        CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    void upload_nodes(const void* flat, Node* dst) {
        if (flat) {
            CK(cudaMemcpyAsync(flat_.p, flat, size_t(3 * N_) * sizeof(Real), cudaMemcpyHostToDevice, stream_));
            k_pack_nodes<Real><<<unsigned((N_ + 255) / 256), 256, 0, stream_>>>(flat_.as<Real>(), N_, dst);
        } else {
            k_pack_nodes<Real><<<unsigned((N_ + 255) / 256), 256, 0, stream_>>>(nullptr, N_, dst);
        }
        CK(cudaGetLastError());
    }

    void download_nodes(const Node* src, void* flat) {
        k_unpack_nodes<Real><<<unsigned((N_ + 255) / 256), 256, 0, stream_>>>(src, N_, flat_.as<Real>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(flat, flat_.p, size_t(3 * N_) * sizeof(Real), cudaMemcpyDeviceToHost, stream_));
    }

    void set_state(const void* u, const void* up, int64_t step) override {
        if (step < 0) throw DescError("step must be >= 0");
        const int ph = int(step % 3);
        upload_nodes(u, u_[ph].as<Node>());
        upload_nodes(up, u_[(ph + 2) % 3].as<Node>());
        // (the next buffer is rewritten by the step before it is read; with the
        // peer-memory transport another rank may already be storing this
        // part's ghosts into it, so it is left alone)
        if (!peer_) upload_nodes(nullptr, u_[(ph + 1) % 3].as<Node>());
        CK(cudaStreamSynchronize(stream_));
        reset_ctrl(step);
    }

    // advance_step with a host SimState in one call. Uploads run on one copy
    // stream in issue order (u_curr in kUpChunks node chunks, then u_prev in
    // the node-update chunks); each element chunk starts once the u_curr
    // prefix it reads has landed, each node-update chunk once its u_prev
    // chunk has, and each chunk's new u_curr goes back on a third stream
    // (the other copy direction) behind the next chunk's update.
    int advance_host(const void* u, const void* up, int64_t step, void* u_next, djg_report* rep) override {
        if (!configured_) throw DescError("step data not configured (djg_configure_step)");
        if (!u || !up || !u_next) throw DescError("djg_advance_host needs u_curr, u_prev and u_next");
        if (step < 0) throw DescError("step must be >= 0");
        if (n_slabs_ != 1 || comm_ || peer_) throw DescError("djg_advance_host: single-part, one-slab engines");
        if (fused_now() && !(std::getenv("DJG_HOST_TWO_KERNEL") && std::atoi(std::getenv("DJG_HOST_TWO_KERNEL"))))
            return advance_host_box(u, up, step, u_next, rep);
        const int64_t S = (N_ + 31) / 32;
        const bool chunked = S >= 4 * 256;
        const int nu = chunked ? kUpChunks : 1, ne = chunked ? kUpChunks : 1, nc = chunked ? kHostChunks : 1;
        if (!side_) CK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
        if (!down_) CK(cudaStreamCreateWithFlags(&down_, cudaStreamNonBlocking));
        if (!flat2_.p) flat2_.alloc(flat_.bytes);
        if (!allSlices_.p) {
            std::vector<int32_t> ids(static_cast<size_t>(S));
            for (int64_t i = 0; i < S; ++i) ids[size_t(i)] = int32_t(i);
            allSlices_.alloc(ids.size() * sizeof(int32_t));
            CK(cudaMemcpy(allSlices_.p, ids.data(), allSlices_.bytes, cudaMemcpyHostToDevice));
            evChunk_.resize(size_t(kUpChunks + 2 * kHostChunks + 2));
            for (auto& e : evChunk_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            // u_curr chunk each element chunk waits for
            needChunk_.assign(size_t(kUpChunks), kUpChunks - 1);
            if (chunked) {
                // per-tile maxima (tiles never straddle an element chunk)
                const int64_t ntile = (E_ + kPipeTile - 1) / kPipeTile;
                DevBuf tm;
                tm.alloc(sizeof(int) * size_t(ntile));
                CK(cudaMemset(tm.p, 0xff, tm.bytes));
                const unsigned g = unsigned((E_ + 255) / 256);
                if (kind_ == DJG_T4) k_chunk_maxnode<4><<<g, 256>>>(conn_.as<int4>(), E_, kPipeTile, tm.as<int>());
                else k_chunk_maxnode<8><<<g, 256>>>(conn_.as<int4>(), E_, kPipeTile, tm.as<int>());
                CK(cudaGetLastError());
                std::vector<int> t(static_cast<size_t>(ntile));
                CK(cudaMemcpy(t.data(), tm.p, tm.bytes, cudaMemcpyDeviceToHost));
                std::vector<int> m(static_cast<size_t>(kUpChunks), -1);
                for (int j = 0; j < kUpChunks; ++j) {
                    const int64_t t0 = ((E_ * j / kUpChunks) / kPipeTile);
                    const int64_t t1 = j + 1 == kUpChunks ? ntile : ((E_ * (j + 1) / kUpChunks) / kPipeTile);
                    for (int64_t q = t0; q < t1; ++q) m[size_t(j)] = std::max(m[size_t(j)], t[size_t(q)]);
                }
                for (int j = 0; j < kUpChunks; ++j) {
                    int c = 0;
                    while (c < kUpChunks - 1 && int64_t(m[size_t(j)]) >= N_ * (c + 1) / kUpChunks) ++c;
                    needChunk_[size_t(j)] = c;
                }
            }
        }
        cudaEvent_t* evU = evChunk_.data();                    // u_curr chunk landed
        cudaEvent_t* evP = evU + kUpChunks;                    // u_prev chunk landed
        cudaEvent_t* evN = evP + kHostChunks;                  // node chunk updated
        cudaEvent_t evStart = evN[kHostChunks], evDone = evN[kHostChunks + 1];
        // control block reset without a host round trip: the H2D copy is
        // stream-ordered before the step (single-part engines never read the
        // epoch stamps, so the last host copy's epoch is carried)
        {
            Ctrl c{};
            c.epoch = ctrl_initialized_ ? hctrl_->epoch : 0u;
            c.multipart = multipart_ ? 1 : 0;
            c.step = step;
            c.first_inv = kNone;
            c.asm_first = kNone;
            c.halt_first_inv = -1;
            c.fail_step = -1;
            *hctrl_ = c;
            *hstart_ = c;
            ctrl_initialized_ = true;
            CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        }
        CK(cudaEventRecord(evStart, stream_));
        CK(cudaStreamWaitEvent(side_, evStart, 0));
        // DJG_TRACE_HOST=1: timing events along the three streams, printed
        // (ms from the start) to stderr after the step -- developer timeline
        static const bool trace = std::getenv("DJG_TRACE_HOST") != nullptr;
        std::vector<std::pair<std::string, cudaEvent_t>> tl;
        auto mark = [&](const std::string& what, cudaStream_t st) {
            if (!trace) return;
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            CK(cudaEventRecord(e, st));
            tl.emplace_back(what, e);
        };
        mark("start", stream_);
        const int ph = int(step % 3);
        Node* ucur = u_[ph].as<Node>();
        Node* uprv = u_[(ph + 2) % 3].as<Node>();
        auto upload = [&](const void* host, Real* stage, Node* dst, int64_t n0, int64_t n1, cudaEvent_t ev) {
            CK(cudaMemcpyAsync(stage + 3 * n0, static_cast<const Real*>(host) + 3 * n0,
                               size_t(3 * (n1 - n0)) * sizeof(Real), cudaMemcpyHostToDevice, side_));
            k_pack_nodes<Real><<<unsigned(std::max<int64_t>(1, (n1 - n0 + 255) / 256)), 256, 0, side_>>>(
                stage + 3 * n0, n1 - n0, dst + n0);
            CK(cudaEventRecord(ev, side_));
            mark(std::string(stage == flat_.as<Real>() ? "up u_curr " : "up u_prev ") + std::to_string(n0), side_);
        };
        for (int c = 0; c < nu; ++c) upload(u, flat_.as<Real>(), ucur, N_ * c / nu, N_ * (c + 1) / nu, evU[c]);
#ifndef DJG_HOST_TAPER
#define DJG_HOST_TAPER 1
#endif
        // node-update chunk c covers slices [sb(c), sb(c + 1)); tapered: the
        // last chunks are smaller, so less is left to update and read back
        // after the last upload lands
        auto sb = [&](int c) -> int64_t {
            if (!DJG_HOST_TAPER || nc != 4) return S * c / nc;
            static const int w[5] = {0, 30, 60, 85, 100};
            return S * w[c] / 100;
        };
        auto node_range = [&](int c, int64_t& n0, int64_t& n1) {
            n0 = 32 * sb(c);
            n1 = std::min<int64_t>(N_, 32 * sb(c + 1));
        };
        for (int c = 0; c < nc; ++c) {
            int64_t n0, n1;
            node_range(c, n0, n1);
            upload(up, flat2_.as<Real>(), uprv, n0, n1, evP[c]);
        }
        CK(cudaGetLastError());
        // element chunk boundaries on whole tiles (the pipeline's bulk copies
        // of rank words and tail planes need 16-byte aligned starts)
        auto ebound = [&](int j) { return j == ne ? E_ : (E_ * j / ne) / kPipeTile * kPipeTile; };
        for (int j = 0; j < ne; ++j) {
            CK(cudaStreamWaitEvent(stream_, evU[chunked ? needChunk_[size_t(j)] : 0], 0));
            launch_element(stream_, ebound(j), ebound(j + 1));
            mark("element chunk " + std::to_string(j), stream_);
        }
        const Node* unew = u_[(ph + 1) % 3].as<Node>();
        for (int c = 0; c < nc; ++c) {
            const int64_t s0 = sb(c), s1 = sb(c + 1);
            const int ns = int(s1 - s0);
            int64_t n0, n1;
            node_range(c, n0, n1);
            CK(cudaStreamWaitEvent(stream_, evP[c], 0));
            k_node_slices<Real, false><<<unsigned(std::max(1, (ns * 32 + 255) / 256)), 256, 0, stream_>>>(
                na_, allSlices_.as<int>() + s0, ns, 0, c == nc - 1 ? 1 : 0);
            // the unpacked result reuses the u_curr staging buffer (its upload
            // has been consumed by the pack kernels the element chunks waited on)
            k_unpack_nodes<Real><<<unsigned(std::max<int64_t>(1, (n1 - n0 + 255) / 256)), 256, 0, stream_>>>(
                unew + n0, n1 - n0, flat_.as<Real>() + 3 * n0);
            CK(cudaEventRecord(evN[c], stream_));
            mark("node chunk " + std::to_string(c), stream_);
            CK(cudaStreamWaitEvent(down_, evN[c], 0));
            CK(cudaMemcpyAsync(static_cast<Real*>(u_next) + 3 * n0, flat_.as<Real>() + 3 * n0,
                               size_t(3 * (n1 - n0)) * sizeof(Real), cudaMemcpyDeviceToHost, down_));
            mark("down " + std::to_string(c), down_);
        }
        CK(cudaEventRecord(evDone, down_));
        CK(cudaStreamWaitEvent(stream_, evDone, 0));
        CK(cudaGetLastError());
        const int status = sync(rep);
        if (trace) {
            for (auto& [what, e] : tl) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, tl.front().second, e));
                std::fprintf(stderr, "[djg host step] %8.3f ms  %s\n", ms, what.c_str());
            }
            for (auto& te : tl) cudaEventDestroy(te.second);
        }
        if (status != DJG_OK) {  // the state did not advance: hand back u_curr
            download_nodes(u_[ph].as<Node>(), u_next);
            CK(cudaStreamSynchronize(stream_));
        }
        return status;
    }

    // advance_host on the fused box step: the box is cut into kBoxRegions
    // runs of node layers (lexicographic ids: contiguous node ranges). Region
    // r's uploads -- u_curr through the first layer above it (its top cell
    // layer reads it), then its own u_prev -- go up one copy stream in
    // region order; k_box_step updates region r's layers as soon as they
    // have landed (the last region's launch closes the step) and region r's
    // u_next goes back on the other copy direction while region r + 1
    // uploads. The regions taper so that little is left to compute and read
    // back after the last upload.
    static constexpr int kBoxRegions = 8;
    int advance_host_box(const void* u, const void* up, int64_t step, void* u_next, djg_report* rep) {
        const int64_t plane = int64_t(box_.nx + 1) * (box_.ny + 1), L = box_.nz + 1;
        const bool chunked = L >= 4 * kBoxRegions && N_ >= (int64_t(1) << 16);
        int R = chunked ? kBoxRegions : 1;
        if (const char* v = std::getenv("DJG_HOST_REGIONS"); v && *v && chunked)  // developer A/B: equal regions
            R = std::max(1, std::min(kBoxRegions, std::atoi(v)));
        if (!side_) CK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
        if (!side2_) CK(cudaStreamCreateWithFlags(&side2_, cudaStreamNonBlocking));
        if (!down_) CK(cudaStreamCreateWithFlags(&down_, cudaStreamNonBlocking));
        if (!flat2_.p) flat2_.alloc(flat_.bytes);
        if (evBox_.empty()) {
            evBox_.resize(size_t(3 * kBoxRegions + 2));
            for (auto& e : evBox_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        cudaEvent_t* evUp = evBox_.data();         // region r's u_curr rows landed
        cudaEvent_t* evUpP = evUp + kBoxRegions;  // region r's u_prev rows landed
        cudaEvent_t* evNew = evUpP + kBoxRegions; // region r's u_next unpacked
        cudaEvent_t evStart = evNew[kBoxRegions], evDone = evNew[kBoxRegions + 1];
        {
            Ctrl c{};
            c.epoch = ctrl_initialized_ ? hctrl_->epoch : 0u;
            c.multipart = multipart_ ? 1 : 0;
            c.step = step;
            c.first_inv = kNone;
            c.asm_first = kNone;
            c.halt_first_inv = -1;
            c.fail_step = -1;
            *hctrl_ = c;
            *hstart_ = c;
            ctrl_initialized_ = true;
            CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        }
        CK(cudaEventRecord(evStart, stream_));
        CK(cudaStreamWaitEvent(side_, evStart, 0));
        CK(cudaStreamWaitEvent(side2_, evStart, 0));
        static const bool trace = std::getenv("DJG_TRACE_HOST") != nullptr;  // as advance_host
        std::vector<std::pair<std::string, cudaEvent_t>> tl;
        auto mark = [&](const std::string& what, cudaStream_t st) {
            if (!trace) return;
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            CK(cudaEventRecord(e, st));
            tl.emplace_back(what, e);
        };
        mark("start", stream_);
        const int ph = int(step % 3);
        Node* ucur = u_[ph].as<Node>();
        Node* uprv = u_[(ph + 2) % 3].as<Node>();
        const Node* unew = u_[(ph + 1) % 3].as<Node>();
        // region boundaries in node layers (percent of the layers, tapered)
        static const int w8[kBoxRegions + 1] = {0, 15, 30, 45, 60, 73, 84, 93, 100};
        auto lay = [&](int r) -> int64_t { return R == kBoxRegions ? L * w8[r] / 100 : L * r / R; };
        // u_curr and u_prev go up on two streams (a copy stream alone moved
        // ~40 GB/s in tools/pcie_probe.py, two at once ~55 GB/s; in the step
        // they reach ~48 GB/s together: cfg5 4.78 -> 4.51 ms per host-state
        // step; splitting each array over both streams was slower)
        auto upload = [&](const void* host, Real* stage, Node* dst, int64_t n0, int64_t n1, cudaStream_t st) {
            if (n1 <= n0) return;
            CK(cudaMemcpyAsync(stage + 3 * n0, static_cast<const Real*>(host) + 3 * n0,
                               size_t(3 * (n1 - n0)) * sizeof(Real), cudaMemcpyHostToDevice, st));
            k_pack_nodes<Real><<<unsigned(std::max<int64_t>(1, (n1 - n0 + 255) / 256)), 256, 0, st>>>(
                stage + 3 * n0, n1 - n0, dst + n0);
        };
        int64_t cur_done = 0;  // u_curr nodes uploaded so far
        for (int r = 0; r < R; ++r) {
            const int64_t n0 = lay(r) * plane, n1 = lay(r + 1) * plane;
            const int64_t c1 = std::min(N_, (lay(r + 1) + 1) * plane);  // through the layer above
            upload(u, flat_.as<Real>(), ucur, cur_done, c1, side_);
            cur_done = std::max(cur_done, c1);
            upload(up, flat2_.as<Real>(), uprv, n0, n1, side2_);
            CK(cudaEventRecord(evUp[r], side_));
            CK(cudaEventRecord(evUpP[r], side2_));
            mark("up u_curr region " + std::to_string(r), side_);
            mark("up u_prev region " + std::to_string(r), side2_);
        }
        CK(cudaGetLastError());
        for (int r = 0; r < R; ++r) {
            const int64_t n0 = lay(r) * plane, n1 = lay(r + 1) * plane;
            CK(cudaStreamWaitEvent(stream_, evUp[r], 0));
            CK(cudaStreamWaitEvent(stream_, evUpP[r], 0));
            launch_box(stream_, int(lay(r)), int(lay(r + 1)), r == R - 1);
            mark("box region " + std::to_string(r), stream_);
            // region r's result into the u_curr staging rows it no longer needs
            k_unpack_nodes<Real><<<unsigned(std::max<int64_t>(1, (n1 - n0 + 255) / 256)), 256, 0, stream_>>>(
                unew + n0, n1 - n0, flat_.as<Real>() + 3 * n0);
            CK(cudaEventRecord(evNew[r], stream_));
            CK(cudaStreamWaitEvent(down_, evNew[r], 0));
            CK(cudaMemcpyAsync(static_cast<Real*>(u_next) + 3 * n0, flat_.as<Real>() + 3 * n0,
                               size_t(3 * (n1 - n0)) * sizeof(Real), cudaMemcpyDeviceToHost, down_));
            mark("down region " + std::to_string(r), down_);
        }
        CK(cudaEventRecord(evDone, down_));
        CK(cudaStreamWaitEvent(stream_, evDone, 0));
        CK(cudaGetLastError());
        const int status = sync(rep);
        if (trace) {
            for (auto& [what, e] : tl) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, tl.front().second, e));
                std::fprintf(stderr, "[djg host step] %8.3f ms  %s\n", ms, what.c_str());
            }
            for (auto& te : tl) cudaEventDestroy(te.second);
        }
        if (status != DJG_OK) {  // the state did not advance: hand back u_curr
            download_nodes(u_[ph].as<Node>(), u_next);
            CK(cudaStreamSynchronize(stream_));
        }
        return status;
    }

    void set_external(const void* r) override {
        if (!r) {
            na_.r_ext = nullptr;
        } else {
            if (!rext_.p) rext_.alloc(size_t(N_) * sizeof(Node));
            upload_nodes(r, rext_.as<Node>());
            CK(cudaStreamSynchronize(stream_));
            na_.r_ext = rext_.as<Node>();
        }
        drop_graphs();
    }

    void read_ctrl() {
        CK(cudaMemcpyAsync(hctrl_, ctrl_.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    void get_state(void* u, void* up, int64_t* step) override {
        read_ctrl();
        const int ph = int(hctrl_->step % 3);
        if (u) download_nodes(u_[ph].as<Node>(), u);
        if (up) download_nodes(u_[(ph + 2) % 3].as<Node>(), up);
        CK(cudaStreamSynchronize(stream_));
        if (step) *step = hctrl_->step;
    }

    // Pipelined element kernel (k_element_pipe) for shapes whose tile stage
    // is small enough to keep several stages and blocks per SM; setup = true
    // only sizes the persistent grid. Returns false if the shape has none.
    template <int K, int M, int RB, int FORM>
    bool launch_pipe(cudaStream_t s, const ElemArgs<Real>& a, int64_t e0, int64_t e1, bool setup) {
        using PS = PipeShape<Real, K, M, RB, FORM>;
        // H8 bodies (heavier, 8 gathers, full record) run better one-shot.
        if constexpr ((K == 1 && !DJG_PIPE_H8) || PS::kStageBytes > kPipeMaxStageBytes) {
            return false;
        } else {
            constexpr int ST = K == 1 ? DJG_PIPE_H8_STAGES : kPipeStages;
            auto kern = k_element_pipe<Real, K, M, RB, FORM, ST>;
            const size_t smem = PS::smem_bytes(ST);
            if (setup) {
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                int nb = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kPipeThreads, smem));
                pipe_blocks_sm_ = nb;
                pipe_smem_ = smem;
                return nb > 0;
            }
            const int64_t tiles = (e1 - e0 + kPipeTile - 1) / kPipeTile;
            const int64_t sms = std::max(1, sms_ - pipe_spare_sms_);
            const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(pipe_blocks_sm_) * sms)));
            kern<<<grid, kPipeThreads, smem, s>>>(a, e0, e1);
            return true;
        }
    }

    // Windowed element kernel (k_element_win): tiles must start on the
    // descriptor grid (e0 a multiple of the tile); otherwise false.
    template <int K, int M, int FORM>
    bool launch_win(cudaStream_t s, const ElemArgs<Real>& a, int64_t e0, int64_t e1, bool setup) {
        using WS = WinShape<Real, K, M, FORM>;
        if constexpr (WS::kStageBytes > kWinMaxStageBytes) {
            return false;
        } else {
            constexpr int ST = K == 1 ? DJG_PIPE_H8_STAGES : kPipeStages;
            auto kern = k_element_win<Real, K, M, FORM, ST>;
            const size_t smem = WS::smem_bytes(ST);
            if (setup) {
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                int nb = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kPipeThreads, smem));
                win_blocks_sm_ = nb;
                return nb > 0;
            }
            if (e0 % kPipeTile != 0) return false;
            const int64_t tiles = (e1 - e0 + kPipeTile - 1) / kPipeTile;
            const int64_t sms = std::max(1, sms_ - pipe_spare_sms_);
            const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(win_blocks_sm_) * sms)));
            kern<<<grid, kPipeThreads, smem, s>>>(a, e0, e1);
            return true;
        }
    }

    void launch_element(cudaStream_t s, int64_t e0, int64_t e1, const Node* u_override = nullptr,
                        bool setup = false) {
        if (e1 <= e0 && !setup) return;
        ElemArgs<Real> a = ea_;
        a.u_override = u_override;
        const unsigned grid = unsigned((e1 - e0 + 127) / 128);
        const int form = tled_ ? 2 : compact_ ? 1 : 0;
#define DJG_K1(K, M)                                                                                            \
    do {                                                                                                        \
        if (win_) {                                                                                             \
            const bool wok = form == 2   ? launch_win<K, M, 2>(s, a, e0, e1, setup)                             \
                             : form == 1 ? launch_win<K, M, 1>(s, a, e0, e1, setup)                             \
                                         : launch_win<K, M, 0>(s, a, e0, e1, setup);                            \
            if (setup) win_ = wok;                                                                              \
            else if (wok) break;                                                                                \
        }                                                                                                       \
        if (pipe_) {                                                                                            \
            bool ok;                                                                                            \
            if (rank_bytes_ == 1)                                                                               \
                ok = form == 2 ? launch_pipe<K, M, 1, 2>(s, a, e0, e1, setup)                                   \
                               : form == 1 ? launch_pipe<K, M, 1, 1>(s, a, e0, e1, setup)                       \
                                           : launch_pipe<K, M, 1, 0>(s, a, e0, e1, setup);                      \
            else                                                                                                \
                ok = form == 2 ? launch_pipe<K, M, 2, 2>(s, a, e0, e1, setup)                                   \
                               : form == 1 ? launch_pipe<K, M, 2, 1>(s, a, e0, e1, setup)                       \
                                           : launch_pipe<K, M, 2, 0>(s, a, e0, e1, setup);                      \
            if (setup) { pipe_ = ok; return; }                                                                  \
            if (ok) break;                                                                                      \
        }                                                                                                       \
        if (setup) return;                                                                                      \
        if (tled_) {                                                                                            \
            if (rank_bytes_ == 1) k_element_tled<Real, K, M, 1><<<grid, 128, 0, s>>>(a, e0, e1);                \
            else k_element_tled<Real, K, M, 2><<<grid, 128, 0, s>>>(a, e0, e1);                                 \
        } else if (compact_) {                                                                                  \
            if (rank_bytes_ == 1) k_element<Real, K, M, 1, true><<<grid, 128, 0, s>>>(a, e0, e1);               \
            else k_element<Real, K, M, 2, true><<<grid, 128, 0, s>>>(a, e0, e1);                                \
        } else {                                                                                                \
            if (rank_bytes_ == 1) k_element<Real, K, M, 1, false><<<grid, 128, 0, s>>>(a, e0, e1);              \
            else k_element<Real, K, M, 2, false><<<grid, 128, 0, s>>>(a, e0, e1);                               \
        }                                                                                                       \
    } while (0)
// DJG_I57: the full-record one-shot kernel only (its 137-Real record is
// beyond the pipeline's stage budget; compact / TLED are refused at creation).
#define DJG_K1_FULL(K, M)                                                                                       \
    do {                                                                                                        \
        if (setup) { pipe_ = false; return; }                                                                   \
        if (rank_bytes_ == 1) k_element<Real, K, M, 1, false><<<grid, 128, 0, s>>>(a, e0, e1);                  \
        else k_element<Real, K, M, 2, false><<<grid, 128, 0, s>>>(a, e0, e1);                                   \
    } while (0)
        if (kind_ == DJG_T4) {
            switch (model_) {
                case DJG_NH: DJG_K1(0, 0); break;
                case DJG_TI: DJG_K1(0, 1); break;
                case DJG_OT: DJG_K1(0, 2); break;
                case DJG_MR: DJG_K1(0, 3); break;
                default: DJG_K1_FULL(0, 4); break;
            }
        } else {
            switch (model_) {
                case DJG_NH: DJG_K1(1, 0); break;
                case DJG_TI: DJG_K1(1, 1); break;
                case DJG_OT: DJG_K1(1, 2); break;
                case DJG_MR: DJG_K1(1, 3); break;
                default: DJG_K1_FULL(1, 4); break;
            }
        }
#undef DJG_K1_FULL
#undef DJG_K1
        CK(cudaGetLastError());
    }

    // One advance_step (or one assemble) on the stream: S slab pairs.
    void launch_step(cudaStream_t s, bool assemble_mode = false, const Node* u_override = nullptr,
                     std::vector<cudaEvent_t>* marks = nullptr) {
        if (!assemble_mode && !u_override && fused_now()) {
            launch_box(s);
            if (marks) {
                CK(cudaEventRecord((*marks)[0], s));
                CK(cudaEventRecord((*marks)[1], s));
            }
            return;
        }
        for (int q = 0; q < n_slabs_; ++q) {
            const int64_t e0 = int64_t(q) * slab_elems_, e1 = std::min<int64_t>(E_, e0 + slab_elems_);
            launch_element(s, e0, e1, u_override);
            if (marks) CK(cudaEventRecord((*marks)[size_t(2 * q)], s));
            launch_node(s, q, assemble_mode);
            if (marks) CK(cudaEventRecord((*marks)[size_t(2 * q + 1)], s));
        }
    }

    void launch_node(cudaStream_t s, int slab, bool assemble_mode) {
        if (n_slabs_ == 1) {
            const unsigned g = unsigned(node_grid_ > 0 ? std::min<int64_t>((N_ + 255) / 256, node_grid_) : (N_ + 255) / 256);
            if (assemble_mode) k_node<Real, true><<<g, 256, 0, s>>>(na_);
            else k_node<Real, false><<<g, 256, 0, s>>>(na_);
            CK(cudaGetLastError());
            return;
        }
        const int n = slab_off_[size_t(slab + 1)] - slab_off_[size_t(slab)];
        const int close = slab == n_slabs_ - 1;
        if (n == 0 && !close) return;
        const int* list = slabSlices_.as<int>() + slab_off_[size_t(slab)];
        const unsigned grid = unsigned(std::max(1, (n * 32 + 255) / 256));
        const int discard = (flags_ & DJG_FLAG_NO_DISCARD) || n_slabs_ == 1 ? 0 : 1;  // slab mode only
        if (assemble_mode) k_node_slices<Real, true><<<grid, 256, 0, s>>>(na_, list, n, discard, close);
        else k_node_slices<Real, false><<<grid, 256, 0, s>>>(na_, list, n, discard, close);
        CK(cudaGetLastError());
    }

    void one_step(cudaStream_t s) {
        if (peer_) {
            launch_peer_local(s);
            launch_peer_agree(s);
        } else if (comm_ && interior_ >= 0) {
            launch_overlapped_step(s);
        } else {
            launch_step(s);
            if (comm_) launch_exchange(s);
        }
    }

    void drop_graphs() {
        if (graph_big_) cudaGraphExecDestroy(graph_big_);
        if (graph_one_) cudaGraphExecDestroy(graph_one_);
        graph_big_ = graph_one_ = nullptr;
    }

    cudaGraphExec_t capture(int steps) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < steps; ++i) one_step(stream_);
        CK(cudaStreamEndCapture(stream_, &g));
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        CK(cudaGraphDestroy(g));
        return ex;
    }

    void step_async(int64_t n) override {
        if (n < 0) throw DescError("nsteps must be >= 0");
        if (!configured_ && n > 0) throw DescError("step data not configured (djg_configure_step)");
        // Snapshot the counters at the start of this call without blocking the
        // host: sync() reports the difference.
        CK(cudaMemcpyAsync(hstart_, ctrl_.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream_));
        if (flags_ & DJG_FLAG_NO_GRAPH) {
            for (int64_t i = 0; i < n; ++i) one_step(stream_);
            return;
        }
        if (n >= kGraphSteps && !graph_big_) graph_big_ = capture(kGraphSteps);
        if (n % kGraphSteps && !graph_one_) graph_one_ = capture(1);
        for (int64_t i = 0; i < n / kGraphSteps; ++i) CK(cudaGraphLaunch(graph_big_, stream_));
        for (int64_t i = 0; i < n % kGraphSteps; ++i) CK(cudaGraphLaunch(graph_one_, stream_));
    }

    int sync(djg_report* rep) override {
        read_ctrl();
        djg_report r{};
        r.step = hctrl_->step;
        r.steps_done = hctrl_->step - hstart_->step;
        r.inverted_count = int64_t(hctrl_->total_inv - hstart_->total_inv);
        r.inverted_steps = hctrl_->inv_steps - hstart_->inv_steps;
        r.first_inverted = -1;
        r.fail_step = -1;
        r.status = hctrl_->halted;
        if (hctrl_->halted == DJG_E_INVERSION) {
            r.first_inverted = hctrl_->halt_first_inv;
            r.fail_step = hctrl_->fail_step;
        } else if (hctrl_->halted == DJG_E_DIVERGENCE) {
            r.diverged = 1;
            r.fail_step = hctrl_->fail_step;
        }
        if (rep) *rep = r;
        return r.status;
    }

    int step(int64_t n, djg_report* rep) override {
        step_async(n);
        return sync(rep);
    }

    int assemble(const void* u, void* f, djg_assemble_stats* st) override {
        const Node* uo = nullptr;
        if (u) {
            upload_nodes(u, uscratch_.as<Node>());
            uo = uscratch_.as<Node>();
        } else {
            read_ctrl();
            uo = u_[hctrl_->step % 3].as<Node>();
        }
        // The element kernel early-outs on a halted engine; assemble must not.
        read_ctrl();
        const int halted = hctrl_->halted;
        if (halted) {
            hctrl_->halted = 0;
            CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        }
        launch_step(stream_, true, uo);
        read_ctrl();
        if (halted) {
            hctrl_->halted = halted;
            CK(cudaMemcpyAsync(ctrl_.p, hctrl_, sizeof(Ctrl), cudaMemcpyHostToDevice, stream_));
        }
        const bool abort = hctrl_->asm_first != kNone;
        if (st) {
            st->first_inverted = abort ? int64_t(hctrl_->asm_first) : -1;
            st->inverted_count = int64_t(hctrl_->asm_count);
        }
        if (!abort && f) CK(cudaMemcpyAsync(f, flat_.p, size_t(3 * N_) * sizeof(Real), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        return abort ? DJG_E_INVERSION : DJG_OK;
    }

    int profile(int64_t n, float* ms_e, float* ms_n, float* ms_t) override {
        if (!configured_) throw DescError("step data not configured (djg_configure_step)");
        CK(cudaMemcpyAsync(hstart_, ctrl_.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream_));
        std::vector<cudaEvent_t> marks(size_t(2 * n_slabs_));
        for (auto& e : marks) CK(cudaEventCreate(&e));
        cudaEvent_t t0, t1;
        CK(cudaEventCreate(&t0));
        CK(cudaEventCreate(&t1));
        float te = 0, tn = 0, tt = 0;
        for (int64_t i = 0; i < n; ++i) {
            CK(cudaEventRecord(t0, stream_));
            launch_step(stream_, false, nullptr, &marks);
            CK(cudaEventRecord(t1, stream_));
            CK(cudaEventSynchronize(t1));
            float a = 0, b = 0, c = 0;
            cudaEvent_t prev = t0;
            for (int q = 0; q < n_slabs_; ++q) {
                CK(cudaEventElapsedTime(&a, prev, marks[size_t(2 * q)]));
                CK(cudaEventElapsedTime(&b, marks[size_t(2 * q)], marks[size_t(2 * q + 1)]));
                te += a;
                tn += b;
                prev = marks[size_t(2 * q + 1)];
            }
            CK(cudaEventElapsedTime(&c, t0, t1));
            tt += c;
        }
        for (auto& e : marks) cudaEventDestroy(e);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        if (ms_e) *ms_e = te;
        if (ms_n) *ms_n = tn;
        if (ms_t) *ms_t = tt;
        return sync(nullptr);
    }

    void info(djg_engine_info* o) override {
        std::memset(o, 0, sizeof(*o));
        o->num_nodes = N_;
        o->num_elements = E_;
        o->num_slots = E_ * npe_;
        o->slot_capacity = capacity_;
        o->device_bytes = int64_t(slot_.bytes + widx_.bytes + wdesc_.bytes + conn_.bytes + rank_.bytes + consts_.bytes + 3 * u_[0].bytes + uscratch_.bytes +
                                  flat_.bytes + ef_.bytes + rowlen_.bytes + slicebase_.bytes + c1_.bytes +
                                  code_.bytes + target_.bytes + tTotal_.bytes + rext_.bytes + ctrl_.bytes +
                                  slabSlices_.bytes);
        o->npe = npe_;
        o->nconst = nconst_;
        o->const_planes = nplanes_;
        o->precision = int32_t(sizeof(Real));
        o->kernels_per_step = fused_now() ? 1 : 2 * n_slabs_;
        o->compact = compact_ ? 1 : 0;
        o->formulation = tled_ ? 1 : 0;
        o->pipelined = pipe_ ? 1 : 0;
        o->windowed = win_ ? 1 : 0;
        o->fused = fused_now() ? 1 : 0;
        o->lattice = fused_now() && lattice_ ? 1 : 0;
        o->window_tiles = win_tiles_;
        o->slabs = n_slabs_;
        o->slab_elements = slab_elems_;
        o->sm_count = sms_;
    }

    // Test hook: the device constant planes as an AoS record (E x nrec Reals).
    int64_t consts_out(void* out) override {
        if (!out) return nrec_;
        std::vector<Real> planes(consts_.bytes / sizeof(Real));
        CK(cudaMemcpy(planes.data(), consts_.p, consts_.bytes, cudaMemcpyDeviceToHost));
        const Real* tail = planes.data() + size_t(nplanes_) * size_t(E_) * size_t(T::kPlane);
        Real* o = static_cast<Real*>(out);
        const int nf = nplanes_ * T::kPlane;
        for (int64_t e = 0; e < E_; ++e)
            for (int f = 0; f < nrec_; ++f)
                o[e * nrec_ + f] = f < nf ? planes[size_t((int64_t(f / T::kPlane) * E_ + e) * T::kPlane + f % T::kPlane)]
                                          : tail[size_t(int64_t(f - nf) * tail_stride_ + e)];
        return nrec_;
    }

    void slot_map(int32_t* out) override {
        std::vector<uint8_t> ranks(rank_.bytes);
        std::vector<int32_t> planes(size_t(E_ * npe_));
        CK(cudaMemcpy(ranks.data(), rank_.p, rank_.bytes, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(planes.data(), conn_.p, conn_.bytes, cudaMemcpyDeviceToHost));
        const int nq = npe_ / 4;
        for (int64_t e = 0; e < E_; ++e)
            for (int q = 0; q < nq; ++q)
                for (int k = 0; k < 4; ++k) {
                    const int a = 4 * q + k;
                    const int64_t n = planes[size_t((int64_t(q) * E_ + e) * 4 + k)];
                    const uint8_t* r = ranks.data() + size_t((e * npe_ + a) * rank_bytes_);
                    const int64_t rank = rank_bytes_ == 1 ? r[0] : (r[0] | (int64_t(r[1]) << 8));
                    out[e * npe_ + a] = int32_t(slice_base_[size_t(n >> 5)] + 32 * rank + (n & 31));
                }
    }

private:
    static constexpr int kGraphSteps = 32;
    int kind_ = 0, model_ = 0, npe_ = 4, nconst_ = 0, nrec_ = 0, nplanes_ = 0, ntail_ = 0, policy_ = 0, sms_ = 0;
    int64_t tail_stride_ = 0;
    int64_t node_grid_ = 0;
    bool device_layout_ = false, need_x_ = false;
    void* comm_ = nullptr;  // ncclComm_t of the multi-GPU step
    int device_ = 0;
    std::vector<int32_t> nbr_;
    std::vector<int64_t> send_off_, recv_off_;
    DevBuf sendBuf_, recvBuf_, status_, counted_;
    bool multipart_ = false;           // djg_set_counted_elements given: totals from the agreement
    int64_t interior_ = -1;            // split step: local elements [0, interior_) touch no ghost node
    int pipe_spare_sms_ = 0;           // SMs the pipelined element kernel leaves free
    static constexpr int kSpareSms = 4;
    cudaStream_t side_ = nullptr;      // interior elements of the overlapped step
    cudaEvent_t evFork_ = nullptr, evJoin_ = nullptr;
    bool peer_ = false;                // peer-memory multi-GPU step
    unsigned long long peer_timeout_ns_ = 10000000000ull;  // k_wait_agree's bound (DJG_PEER_TIMEOUT_MS)
    cudaEvent_t evPrev_ = nullptr;     // djg_advance_host: u_prev uploaded
    std::vector<cudaEvent_t> evBox_;   // djg_advance_host on the fused box step
    cudaStream_t side2_ = nullptr;     // djg_advance_host on the fused box step: u_prev uploads
    DevBuf flat2_, allSlices_;
    std::vector<cudaEvent_t> evChunk_;
    static constexpr int kHostChunks = DJG_HOST_CHUNKS;
    static constexpr int kUpChunks = 8;  // djg_advance_host: u_curr upload / element chunks
    cudaStream_t down_ = nullptr;        // djg_advance_host: result read-back
    std::vector<int> needChunk_;
    PeerArgs<Real> pa_{};
    DevBuf mailbox_, destOff_, dest_, peerU_, peerMail_;
    std::vector<void*> ipc_open_;
    DevBuf pairs_, rowoff_, mass_;  // device layout: sorted CSR pairs (until masses are built), lump_mass
    Real lmin_ = 0;
    bool compact_ = false, tled_ = false, pipe_ = false, win_ = false;
    int pipe_blocks_sm_ = 0, win_blocks_sm_ = 0;
    size_t pipe_smem_ = 0;
    int64_t win_tiles_ = 0;            // tiles whose nodes fit a window (k_element_win)
    DevBuf slot_, widx_, wdesc_;       // node windows: slot positions, window indices, tile descriptors
    bool fused_ = false;               // generated box of T4 cells: one fused kernel per step (k_box_step)
    BoxArgs box_{};
    int box_grid_ = 0;
    bool lattice_ = false;  // the fused step reads records from lat_ (build_lattice)
    bool box_forced_ = false;  // DJG_FLAG_FUSED / DJG_FUSED=1
    DevBuf lat_, lcls_, ld_;
    uint32_t flags_ = 0;
    int64_t N_ = 0, E_ = 0, capacity_ = 0;
    cudaStream_t stream_ = nullptr;
    std::vector<int32_t> slice_base_;
    int rank_bytes_ = 1;
    DevBuf elemL2g_, haloSend_, haloRecv_, X_;
    int64_t nsend_ = 0, nrecv_ = 0;
    DevBuf conn_, rank_, consts_, u_[3], uscratch_, flat_, ef_, rowlen_, slicebase_, c1_, code_, target_, tTotal_,
        rext_, ctrl_;
    Ctrl* hctrl_ = nullptr;
    ElemArgs<Real> ea_{};
    NodeArgs<Real> na_{};
    cudaGraphExec_t graph_big_ = nullptr, graph_one_ = nullptr;
    Ctrl* hstart_ = nullptr;  // pinned snapshot taken at the start of a step call
    bool configured_ = false;
    bool ctrl_initialized_ = false;
    // slab schedule
    static constexpr int64_t kSlabBytes = int64_t(32) << 20;  // force rows per slab kept in L2
    int64_t slab_bytes_ = 0, slab_elems_ = 0;
    int wmax_ = 1, n_slabs_ = 1;
    int slice_w_ = 0;  // uniform slice width (slots per node) or 0: slice_base table
    std::vector<int> slab_off_;
    DevBuf slabSlices_;
};

int debug_cbrt(int32_t precision, const void* in, void* out, int64_t n, int32_t device) {
    try {
        CK(cudaSetDevice(device));
        const size_t bytes = size_t(n) * size_t(precision);
        DevBuf a, b;
        a.alloc(bytes);
        b.alloc(bytes);
        CK(cudaMemcpy(a.p, in, bytes, cudaMemcpyHostToDevice));
        const unsigned grid = unsigned((n + 255) / 256);
        if (precision == 4) k_cbrt<float><<<grid, 256>>>(a.as<float>(), b.as<float>(), n);
        else k_cbrt<double><<<grid, 256>>>(a.as<double>(), b.as<double>(), n);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, b.p, bytes, cudaMemcpyDeviceToHost));
        return DJG_OK;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        return DJG_E_CUDA;
    }
}

}  // namespace
}  // namespace djg

struct djg_engine {
    std::unique_ptr<djg::EngineBase> impl;
    std::string err;
};

namespace {

template <class F>
int guarded(djg_engine* eng, F&& f) {
    if (!eng || !eng->impl) return DJG_E_CONFIG;
    try {
        return f(*eng->impl);
    } catch (const djg::DescError& e) {
        eng->err = e.what();
        return DJG_E_CONFIG;
    } catch (const djg::CudaError& e) {
        eng->err = e.what();
        return DJG_E_CUDA;
    } catch (const std::exception& e) {
        eng->err = e.what();
        return DJG_E_INTERNAL;
    }
}

}  // namespace

extern "C" {

int32_t djg_const_count(int32_t kind, int32_t model) { return djg::const_count(kind, model); }

int djg_create(const djg_desc* d, djg_engine** out) {
    if (!d || !out) {
        djg::g_create_error = "null argument";
        return DJG_E_CONFIG;
    }
    *out = nullptr;
    try {
        if (d->kind != DJG_T4 && d->kind != DJG_H8) throw djg::DescError("unknown element kind");
        if (d->material.model < DJG_NH || d->material.model > DJG_I57) throw djg::DescError("unknown material model");
        if (d->inversion_policy != DJG_ABORT && d->inversion_policy != DJG_SKIP_AND_REPORT)
            throw djg::DescError("unknown inversion policy");
        auto eng = std::make_unique<djg_engine>();
        if (d->precision == 4) eng->impl = std::make_unique<djg::Engine<float>>(*d);
        else if (d->precision == 8) eng->impl = std::make_unique<djg::Engine<double>>(*d);
        else throw djg::DescError("precision must be 4 or 8");
        *out = eng.release();
        return DJG_OK;
    } catch (const djg::DescError& e) {
        djg::g_create_error = e.what();
        return DJG_E_CONFIG;
    } catch (const djg::CudaError& e) {
        djg::g_create_error = e.what();
        return DJG_E_CUDA;
    } catch (const std::exception& e) {
        djg::g_create_error = e.what();
        return DJG_E_INTERNAL;
    }
}

void djg_destroy(djg_engine* eng) { delete eng; }

const char* djg_create_error(void) { return djg::g_create_error.c_str(); }

// Not in the public headers: lets the host-side builder report its errors
// through djg_create_error().
void djg_internal_set_create_error(const char* msg) { djg::g_create_error = msg ? msg : ""; }

int djg_set_state(djg_engine* eng, const void* u, const void* up, int64_t step) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_state(u, up, step);
        return DJG_OK;
    });
}

int djg_set_external(djg_engine* eng, const void* r) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_external(r);
        return DJG_OK;
    });
}

int djg_get_state(djg_engine* eng, void* u, void* up, int64_t* step) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.get_state(u, up, step);
        return DJG_OK;
    });
}

int djg_step(djg_engine* eng, int64_t n, djg_report* rep) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.step(n, rep); });
}

int djg_step_async(djg_engine* eng, int64_t n) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_async(n);
        return DJG_OK;
    });
}

int djg_sync(djg_engine* eng, djg_report* rep) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.sync(rep); });
}

void* djg_stream(djg_engine* eng) { return eng && eng->impl ? static_cast<void*>(eng->impl->stream()) : nullptr; }

int djg_assemble(djg_engine* eng, const void* u, void* f, djg_assemble_stats* st) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.assemble(u, f, st); });
}

int djg_profile_steps(djg_engine* eng, int64_t n, float* ms_e, float* ms_n, float* ms_t) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.profile(n, ms_e, ms_n, ms_t); });
}

int djg_configure_step(djg_engine* eng, const djg_step_desc* s) {
    return guarded(eng, [&](djg::EngineBase& e) {
        if (!s) throw djg::DescError("null step descriptor");
        e.configure_step(*s);
        return DJG_OK;
    });
}

int djg_set_policy(djg_engine* eng, int32_t policy) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_policy(policy);
        return DJG_OK;
    });
}

int djg_set_partition(djg_engine* eng, int64_t num_owned, const int64_t* elem_l2g) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_partition(num_owned, elem_l2g);
        return DJG_OK;
    });
}

int djg_set_halo(djg_engine* eng, int64_t nsend, const int32_t* send_nodes, int64_t nrecv, const int32_t* recv_nodes) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_halo(nsend, send_nodes, nrecv, recv_nodes);
        return DJG_OK;
    });
}

int djg_set_counted_elements(djg_engine* eng, const uint8_t* counted) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_counted_elements(counted);
        return DJG_OK;
    });
}

int djg_halo_pack(djg_engine* eng, void* dev_send) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.halo_pack(dev_send);
        return DJG_OK;
    });
}

int djg_halo_unpack(djg_engine* eng, const void* dev_recv) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.halo_unpack(dev_recv);
        return DJG_OK;
    });
}

int djg_step_status(djg_engine* eng, int64_t* dev_status) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_status(dev_status);
        return DJG_OK;
    });
}

int djg_step_agree(djg_engine* eng, const int64_t* dev_reduced) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_agree(dev_reduced);
        return DJG_OK;
    });
}

int djg_get_info(djg_engine* eng, djg_engine_info* info) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.info(info);
        return DJG_OK;
    });
}

int djg_get_slot_map(djg_engine* eng, int32_t* out) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.slot_map(out);
        return DJG_OK;
    });
}

int djg_comm_unique_id(void* id) {
    if (!id) return DJG_E_CONFIG;
    try {
        const djg::Nccl& api = djg::Nccl::get();
        ncclUniqueId uid;
        const ncclResult_t r = api.get_unique_id(&uid);
        if (r != ncclSuccess) {
            djg_internal_set_create_error(api.error_string(r));
            return DJG_E_CUDA;
        }
        std::memcpy(id, &uid, sizeof(uid));
        return DJG_OK;
    } catch (const std::exception& e) {
        djg_internal_set_create_error(e.what());
        return DJG_E_CUDA;
    }
}

int djg_comm_init(djg_engine* eng, const void* id, int32_t nranks, int32_t rank, int32_t num_neighbors,
                  const int32_t* neighbors, const int64_t* send_off, const int64_t* recv_off) {
    return guarded(eng, [&](djg::EngineBase& e) {
        if (!id) throw djg::DescError("null unique id");
        e.comm_init(id, nranks, rank, num_neighbors, neighbors, send_off, recv_off);
        return DJG_OK;
    });
}

int djg_set_interior(djg_engine* eng, int64_t num_interior) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.set_interior(num_interior);
        return DJG_OK;
    });
}

int djg_step_interior(djg_engine* eng) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_interior();
        return DJG_OK;
    });
}

int djg_step_boundary(djg_engine* eng) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_boundary();
        return DJG_OK;
    });
}

int djg_peer_export(djg_engine* eng, void** ptrs4) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.peer_export(ptrs4);
        return DJG_OK;
    });
}

int djg_peer_ipc_export(djg_engine* eng, void* handles) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.peer_ipc_export(handles);
        return DJG_OK;
    });
}

int djg_peer_ipc_open(djg_engine* eng, const void* handles, void** ptrs4) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.peer_ipc_open(handles, ptrs4);
        return DJG_OK;
    });
}

int djg_peer_setup(djg_engine* eng, int32_t nparts, int32_t part, const void* const* peer_u,
                   const void* const* peer_mail, const int64_t* peer_num_nodes, int64_t ndest,
                   const int32_t* dest_node, const int32_t* dest_part, const int32_t* dest_index) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.peer_setup(nparts, part, peer_u, peer_mail, peer_num_nodes, ndest, dest_node, dest_part, dest_index);
        return DJG_OK;
    });
}

int djg_step_peer_local(djg_engine* eng) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_peer_local();
        return DJG_OK;
    });
}

int djg_step_peer_agree(djg_engine* eng) {
    return guarded(eng, [&](djg::EngineBase& e) {
        e.step_peer_agree();
        return DJG_OK;
    });
}

int djg_advance_host(djg_engine* eng, const void* u_curr, const void* u_prev, int64_t step, void* u_next,
                     djg_report* report) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.advance_host(u_curr, u_prev, step, u_next, report); });
}

int djg_lump_mass(djg_engine* eng, void* mass) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.lump_mass(mass); });
}

int djg_min_char_length(djg_engine* eng, double* out) {
    return guarded(eng, [&](djg::EngineBase& e) { return e.min_char_length(out); });
}

int djg_debug_cbrt(int32_t precision, const void* in, void* out, int64_t n, int32_t device) {
    return djg::debug_cbrt(precision, in, out, n, device);
}

int64_t djg_get_consts(djg_engine* eng, void* out) {
    if (!eng || !eng->impl) return -1;
    try {
        return eng->impl->consts_out(out);
    } catch (const std::exception& e) {
        eng->err = e.what();
        return -1;
    }
}

const char* djg_last_error(djg_engine* eng) { return eng ? eng->err.c_str() : "null engine"; }

const char* djg_status_string(int32_t s) {
    switch (s) {
        case DJG_OK: return "ok";
        case DJG_E_INTERNAL: return "internal error";
        case DJG_E_CONFIG: return "configuration error";
        case DJG_E_CUDA: return "CUDA error";
        case DJG_E_INVERSION: return "element inversion";
        case DJG_E_DIVERGENCE: return "divergence";
    }
    return "unknown status";
}

}  // extern "C"
