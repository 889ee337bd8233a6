// sm_100a kernels of one DJ-TLED explicit step.
//
//   k_element  (K1)  one thread per element: 128-bit streaming loads of the
//                    connectivity, force-slot positions and hot constants
//                    (structure of 16-byte planes), gather of the element's
//                    nodal displacements, the direct-Jacobian force of
//                    Table 3 / Eq. 10 (+ hourglass for H8), one 16-byte store
//                    per element node into its CSR slot.
//   k_node     (K2+K3) one thread per node: sums its slots in ascending
//                    element order (slots live in a sliced layout so lane i
//                    reads slot k of node i at a coalesced address), then the
//                    central-difference update with damping and BCs, the
//                    non-finite detector, and the end-of-step bookkeeping.
//
// Arithmetic mirrors the reference expression by expression, the file is
// compiled with --fmad=false, and cbrt restates glibc's algorithm, so a step
// reproduces the CPU reference bit for bit. No float atomics anywhere: the only atomics are
// the integer inversion/divergence flags (djtled_force.hpp:97-112,
// solver.hpp:115,137).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../common/element_math.hpp"

namespace djg {

// ------------------------------------------------------------------ types

struct alignas(32) double4a {
    double x, y, z, w;
};

template <class Real>
struct RT;

template <>
struct RT<float> {
    using Node = float4;    // xyz + pad: one 128-bit access per node / slot
    using Plane = float4;   // 4 Reals per constant plane
    static constexpr int kPlane = 4;
    __device__ static inline Node load_node(const Node* p) { return __ldg(p); }
    __device__ static inline Node load_stream(const Node* p) { return __ldcs(p); }
    __device__ static inline Node load_l2(const Node* p) { return __ldcg(p); }
    __device__ static inline void store_node(Node* p, float x, float y, float z) { *p = make_float4(x, y, z, 0.f); }
    __device__ static inline Plane load_plane(const Plane* p) { return __ldcs(p); }
};

template <>
struct RT<double> {
    using Node = double4a;  // xyz + pad, 32 bytes = one sector
    using Plane = double2;  // 2 Reals per constant plane
    static constexpr int kPlane = 2;
    __device__ static inline Node load_node(const Node* p) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        return {a.x, a.y, b.x, b.y};
    }
    __device__ static inline Node load_stream(const Node* p) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
        const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
        return {a.x, a.y, b.x, b.y};
    }
    __device__ static inline Node load_l2(const Node* p) {
        const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
        return {a.x, a.y, b.x, b.y};
    }
    __device__ static inline void store_node(Node* p, double x, double y, double z) {
        reinterpret_cast<double2*>(p)[0] = make_double2(x, y);
        reinterpret_cast<double2*>(p)[1] = make_double2(z, 0.0);
    }
    __device__ static inline Plane load_plane(const Plane* p) { return __ldcs(p); }
};

// Component k of a record plane; bit-for-bit equality (+0 and -0 distinct).
__device__ __forceinline__ float plane_at(const float4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
__device__ __forceinline__ double plane_at(const double2& v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ bool same_bits(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }
__device__ __forceinline__ bool same_bits(double a, double b) { return __double_as_longlong(a) == __double_as_longlong(b); }

// Record layout per (kind, model): offsets in the canonical record (djg.h).
template <int KIND, int MODEL>
struct Layout {
    static constexpr bool kI4 = MODEL == 1 || MODEL == 2;
    static constexpr bool kI6 = MODEL == 2;
    static constexpr bool kI2 = MODEL == 3;
    static constexpr bool kI57 = MODEL == 4;  // DJG_I57: I5 and I7 (full record only)
    static constexpr bool kH8 = KIND == 1;
    static constexpr int NPE = kH8 ? 8 : 4;
    static constexpr int m4 = 23, I4m = 29;
    static constexpr int m6 = kI4 ? 35 : 23, I6m = m6 + 6;
    static constexpr int M2 = 23, I2m = 44;
    static constexpr int M5 = 23, I5m = 44, M7 = 80, I7m = 101;
    static constexpr int after_mat = 23 + (kI4 ? 12 : 0) + (kI6 ? 12 : 0) + (kI2 ? 57 : 0) + (kI57 ? 114 : 0);
    static constexpr int khg = after_mat, gamma = after_mat + 1;
    static constexpr int count = after_mat + (kH8 ? 33 : 0);
};

// Device control block: the step counter and the failure flags of
// advance_step / run_simulation, kept on the device so a multi-step graph
// needs no host round trip.
struct Ctrl {
    long long step;                 // SimState::step
    unsigned long long first_inv;   // min inverted element this step (~0ull: none)
    unsigned long long inv_count;   // inverted elements this step
    unsigned int blocks_done;       // k_node completion counter
    int diverged;                   // non-finite seen this step
    int halted;                     // 0, or DJG_E_INVERSION / DJG_E_DIVERGENCE
    int agreed;                     // multi-part: halt_first_inv already a global id
    long long fail_step;            // state.step + 1 of the failing step
    long long halt_first_inv;       // element reported with an inversion halt
    unsigned long long total_inv;   // accumulated inverted elements
    long long inv_steps;            // steps with >= 1 inversion
    unsigned long long asm_first;   // djg_assemble result
    unsigned long long asm_count;
    unsigned int epoch;             // fused step: launches completed (flag stamps)
    int ticket;                     // fused step: next work-list item
    int multipart;                  // 1: totals accumulate the parts' summed counts (k_agree)
    unsigned long long step_inv;    // counted inversions of the last closed step (k_step_status)
};

constexpr unsigned long long kNone = ~0ull;

template <class Real>
struct MatParams {
    Real dI1;     // mu/2 (NH/TI/OT) or c10 (MR): energy_derivatives, material.hpp:266-290
    Real kappa;   // dJ = kappa (J - 1)
    Real eta_a;   // dI4 = eta_a (Ib4 - 1)
    Real eta_b;   // dI6 = eta_b (Ib6 - 1)
    Real dI2;     // c01
    // compact mode / device precompute: what build_element_constants needs
    Real A[6], B[6];  // fibre structure tensors a a^T, b b^T (FibreDirections)
    Real fa[3], fb[3];  // unit fibre directions (TLED invariants)
    Real chk;         // c_hg * kappa (k_hg = chk * cbrt(V0), precompute.hpp:252)
};

// DJG_CHECKS=1 (the _build_checked library, tests/test_gpu_checked.py):
// device-side bounds checks on every gathered node id and every slot
// position; a violation traps the kernel (a CUDA error on the next call).
#ifndef DJG_CHECKS
#define DJG_CHECKS 0
#endif
#if DJG_CHECKS
#define DJG_ASSERT(c) \
    do {              \
        if (!(c)) {   \
            printf("djg check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__); \
            __trap(); \
        }             \
    } while (0)
#else
#define DJG_ASSERT(c) ((void)0)
#endif

template <class Real>
struct ElemArgs {
    long long E;
    long long N;                         // nodes (DJG_CHECKS bounds)
    long long cap;                       // force-slot entries (DJG_CHECKS bounds)
    const int4* conn;                    // NPE/4 planes of int4[E]
    const void* rank;                    // per element: npe ranks (uint8 or uint16) of the element
                                         // in its nodes' CSR rows, packed in one 4/8/16-byte word
    const int* slice_base;               // first slot of each 32-node slice
    int slice_w;                         // > 0: uniform slices, slice_base[s] = 32 slice_w s
    const int4* slot;                    // node windows: NPE/4 planes of int4[E], slot position of
                                         // each element-node (slice_base[n/32] + 32 rank + n%32)
    const void* widx;                    // node windows: per element NPE window indices (uint8 / uint16)
    const int* wdesc;                    // node windows: kWinDesc ints per 128-element tile, or NULL
    const long long* elem_l2g;           // multi-part: global id of each local element (inversions
                                         // are reported in global ids), else NULL
    const unsigned char* counted;        // multi-part: 1 for the elements whose inversions this part
                                         // counts (its own; ghosts are counted by their owner), or NULL
    const typename RT<Real>::Plane* c;   // nplanes planes of Plane[E]
    const Real* ctail;                   // record remainder planes (compact T4): Real[tail_stride]
    long long tail_stride;
    const typename RT<Real>::Node* u[3]; // triple-buffered displacement
    const typename RT<Real>::Node* u_override;
    const typename RT<Real>::Node* X;    // reference coordinates (compact H8, device precompute)
    typename RT<Real>::Node* ef;         // force slots (xyz + pad), sliced CSR order
    Ctrl* ctrl;
    MatParams<Real> mat;
};

template <class Real>
struct NodeArgs {
    long long N;
    long long cap;                       // force-slot entries (DJG_CHECKS bounds)
    const int* row_len;                  // CSR row length per node
    const int* slice_base;               // first slot position of each 32-node slice
    int slice_w;                         // > 0: uniform slices, slice_base[s] = 32 slice_w s
    const typename RT<Real>::Node* ef;   // force slots
    typename RT<Real>::Node* u[3];
    const typename RT<Real>::Node* r_ext;  // NULL: identically zero
    const Real* c1;
    const unsigned char* code;           // 2 bits per DOF kind | massless << 6
    const Real* target;                  // 3N
    const Real* t_total;                 // 3N
    Real c2, c3, dt;
    int policy;                          // 0 abort, 1 skip and report
    Ctrl* ctrl;
    Real* f_out;                         // assemble mode: 3N internal forces
};

// ------------------------------------------------------------------ cbrt

// The reference calls std::cbrt (kinematics.hpp:69), i.e. glibc's cbrtf /
// cbrt, which are NOT correctly rounded (10.7 % of floats in [0.5, 2) differ
// from the correctly rounded cube root) and differ from CUDA's cbrtf. This is
// a restatement of glibc 2.39's algorithm (sysdeps/ieee754/{flt-32,dbl-64}/
// s_cbrt*.c: frexp reduction, a polynomial seed, one rational Halley step in
// double, exponent scaling by 2^(1/3) powers). Evaluated with IEEE double ops
// (no FMA: --fmad=false) it returns the same bits as the host libm; pinned by
// tests/test_cbrt.py against the host for every float in [0.25, 4).
__device__ __forceinline__ double glibc_cbrt_factor(int r) {
    // 2^(r/3) for r = xe % 3 in {-2..2} (selects, no branch)
    const double pos = r == 1 ? 1.2599210498948731648 : 1.5874010519681994748;
    const double neg = r == -1 ? 1.0 / 1.2599210498948731648 : 1.0 / 1.5874010519681994748;
    return r == 0 ? 1.0 : (r > 0 ? pos : neg);
}

// glibc's cbrtf for zero, subnormal, infinite and NaN x (frexpf / ldexpf).
__device__ __noinline__ float ref_cbrt_general(float x) {
    int xe;
    const float xm = frexpf(fabsf(x), &xe);
    if (x == 0.0f || !isfinite(x)) return x + x;
    const float u = float(0.492659620528969547 + (0.697570460207922770 - 0.191502161678719066 * double(xm)) *
                                                     double(xm));
    const float t2 = u * u * u;
    const float ym = float(double(u) * (double(t2) + 2.0 * double(xm)) / (2.0 * double(t2) + double(xm)) *
                           glibc_cbrt_factor(xe % 3));
    return ldexpf(x > 0.0f ? ym : -ym, xe / 3);
}

// Normal x: frexp and ldexp on the exponent field directly -- the same
// values (|ym| lies in [0.5, 1.6) and |xe / 3| <= 42, so the result is normal
// and the exponent addition is exact).
__device__ __forceinline__ float ref_cbrt(float x) {
    const unsigned bits = __float_as_uint(x);
    const unsigned ex = (bits >> 23) & 0xffu;
    if (ex == 0u || ex == 0xffu) return ref_cbrt_general(x);
    const int xe = int(ex) - 126;
    const float xm = __uint_as_float((bits & 0x007fffffu) | 0x3f000000u);
    const float u = float(0.492659620528969547 + (0.697570460207922770 - 0.191502161678719066 * double(xm)) *
                                                     double(xm));
    const float t2 = u * u * u;
    // x in [0.5, 2) (the volume ratio of any sane step): xe = 0 or 1, so
    // xe / 3 = 0 and xe % 3 = xe -- the same factor without the division
    double f;
    int q;
    if (__builtin_expect(unsigned(xe) <= 1u, 1)) {
        f = xe ? 1.2599210498948731648 : 1.0;
        q = 0;
    } else {
        f = glibc_cbrt_factor(xe % 3);
        q = xe / 3;
    }
    const float ym = float(double(u) * (double(t2) + 2.0 * double(xm)) / (2.0 * double(t2) + double(xm)) * f);
    const float sy = x > 0.0f ? ym : -ym;
    return __uint_as_float(__float_as_uint(sy) + (unsigned(q) << 23));
}

__device__ __forceinline__ double ref_cbrt(double x) {
    int xe;
    const double xm = frexp(fabs(x), &xe);
    if (x == 0.0 || !isfinite(x)) return x + x;
    const double u =
        (0.354895765043919860 +
         ((1.50819193781584896 +
           ((-2.11499494167371287 +
             ((2.44693122563534430 + ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) *
                                      xm)) *
              xm)) *
            xm)) *
          xm));
    const double t2 = u * u * u;
    const double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * glibc_cbrt_factor(xe % 3);
    return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

template <class Real>
__global__ void k_cbrt(const Real* __restrict__ in, Real* __restrict__ out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ref_cbrt(in[i]);
}

// ------------------------------------------------------------------ K1

// Force row of element-node a into slot slice_base[n/32] + 32 rank + n%32:
// one 16-byte (f64: 32-byte) store. (Three 4-byte planes move 25 % fewer
// bytes but cost more in scattered L2 write transactions than they save.)
template <class Real>
__device__ __forceinline__ void store_row(const ElemArgs<Real>& A, int pos, Real x, Real y, Real z) {
    DJG_ASSERT(pos >= 0 && pos < A.cap);
    RT<Real>::store_node(A.ef + pos, x, y, z);
}

// Where element_body's rows go: the force slots in HBM (store_row), or -- for
// a Src that declares itself a row sink (the fused box step) -- the Src's own
// storage. Likewise whether an inversion is counted: A.counted, or the Src.
template <class Src, class = void>
struct RowSink : std::false_type {};
template <class Src>
struct RowSink<Src, std::void_t<decltype(Src::kRowSink)>> : std::true_type {};

template <class Real, class Src>
__device__ __forceinline__ void emit_row(const ElemArgs<Real>& A, const Src& src, int pos, Real x, Real y, Real z) {
    if constexpr (RowSink<Src>::value) src.store(pos, x, y, z);
    else store_row(A, pos, x, y, z);
}
template <class Real, class Src>
__device__ __forceinline__ bool counts_inversion(const ElemArgs<Real>& A, const Src& src, long long e) {
    if constexpr (RowSink<Src>::value) return src.count_inv;
    else return !A.counted || A.counted[e];
}

// Ranks of element e in its nodes' CSR rows (RB bytes each), packed in one
// 4 / 8 / 16-byte word per element.
template <int NPE, int RB>
struct RankWord {
    using type = typename std::conditional<NPE * RB == 4, unsigned,
                                           typename std::conditional<NPE * RB == 8, uint2, uint4>::type>::type;
};

template <int NPE, int RB>
__device__ __forceinline__ void decode_ranks(const typename RankWord<NPE, RB>::type w, int (&rk)[NPE]) {
    if constexpr (NPE == 4 && RB == 1) {
#pragma unroll
        for (int a = 0; a < 4; ++a) rk[a] = (w >> (8 * a)) & 0xff;
    } else if constexpr (NPE == 8 && RB == 1) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            rk[a] = (w.x >> (8 * a)) & 0xff;
            rk[4 + a] = (w.y >> (8 * a)) & 0xff;
        }
    } else if constexpr (NPE == 4) {
        rk[0] = w.x & 0xffff; rk[1] = w.x >> 16; rk[2] = w.y & 0xffff; rk[3] = w.y >> 16;
    } else {
        const unsigned v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            rk[2 * q] = v[q] & 0xffff;
            rk[2 * q + 1] = v[q] >> 16;
        }
    }
}

template <int NPE, int RB>
__device__ __forceinline__ void load_ranks(const void* base, long long e, int (&rk)[NPE]) {
    using W = typename RankWord<NPE, RB>::type;
    decode_ranks<NPE, RB>(__ldcs(static_cast<const W*>(base) + e), rk);
}

// Slot of element-node (n, rank k): slice_base[n/32] + 32 k + n%32 -- the
// base computed (uniform slices, w > 0) or loaded.
__device__ __forceinline__ int slice_base_of(const int* __restrict__ slice_base, int w, long long n) {
    return w > 0 ? int(32 * w * (n >> 5)) : __ldg(slice_base + (n >> 5));
}
__device__ __forceinline__ int slot_of(const int* __restrict__ slice_base, int w, int n, int k) {
    return slice_base_of(slice_base, w, n) + 32 * k + (n & 31);
}

// Where element_body takes its streamed per-element inputs from: straight
// from HBM (GlobalSrc), or from a shared-memory stage filled by bulk async
// copies (SmemSrc, k_element_pipe).
template <class Real>
struct GlobalSrc {
    const ElemArgs<Real>& A;
    long long e;
    __device__ __forceinline__ int4 conn(int p) const { return __ldcs(A.conn + (long long)p * A.E + e); }
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const {
        return RT<Real>::load_plane(A.c + (long long)p * A.E + e);
    }
    template <int NPE, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[NPE]) const { load_ranks<NPE, RB>(A.rank, e, rk); }
    __device__ __forceinline__ typename RT<Real>::Node node(int, const typename RT<Real>::Node* __restrict__ u,
                                                            int n) const {
        return RT<Real>::load_node(u + n);
    }
    __device__ __forceinline__ int slot(const int* __restrict__ sb, int, int n, int k) const {
        return slot_of(sb, A.slice_w, n, k);
    }
    __device__ __forceinline__ Real tail(int t) const { return __ldcs(A.ctail + t * A.tail_stride + e); }
    __device__ __forceinline__ typename RT<Real>::Node coord(const ElemArgs<Real>& a, int n) const {
        return RT<Real>::load_node(a.X + n);
    }
};

template <class Real, int TILE>
struct SmemSrc {
    const int4* sconn;                   // [NPE/4][TILE]
    const typename RT<Real>::Plane* srec;  // [planes][TILE]
    const void* srank;                   // [TILE] rank words
    const Real* stail;                   // [NTAIL][TILE] record remainder
    int i;
    int w;                               // ElemArgs::slice_w
    __device__ __forceinline__ typename RT<Real>::Node node(int, const typename RT<Real>::Node* __restrict__ u,
                                                            int n) const {
        return RT<Real>::load_node(u + n);
    }
    __device__ __forceinline__ int4 conn(int p) const { return sconn[p * TILE + i]; }
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const { return srec[p * TILE + i]; }
    template <int NPE, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[NPE]) const {
        using W = typename RankWord<NPE, RB>::type;
        decode_ranks<NPE, RB>(static_cast<const W*>(srank)[i], rk);
    }
    __device__ __forceinline__ int slot(const int* __restrict__ sb, int, int n, int k) const {
        return slot_of(sb, w, n, k);
    }
    __device__ __forceinline__ Real tail(int t) const { return stail[t * TILE + i]; }
    __device__ __forceinline__ typename RT<Real>::Node coord(const ElemArgs<Real>& a, int n) const {
        return RT<Real>::load_node(a.X + n);
    }
};

// Compact record kept in HBM. T4: nothing -- J0 is rebuilt from the node
// coordinates (gathered like the displacements, mostly L1/L2 hits) with
// jacobian0's own sums, det J0 and V0 with det3 / volume0, the invariant
// tensors from J0^-1: all bit-identical to the stored values.
// H8: J0, det J0, V0, pad, then the hourglass data k_hg, gamma (32) (cheap
// to store, costly to rebuild: it needs the coordinates and a cube root).
constexpr int kCompactRecord = 12;
template <int KIND>
constexpr int kCompactLen = KIND == 1 ? kCompactRecord + 33 : 0;

// Storage of a record of LEN Reals: NFULL 16-byte planes [E], and -- only for
// the compact T4 record, whose 9 Reals would leave a padded plane -- NTAIL
// scalar planes [tail_stride] for the remainder.
template <class Real, int LEN, bool TAIL>
struct RecPlanes {
    static constexpr int W = RT<Real>::kPlane;
    static constexpr int NFULL = TAIL ? LEN / W : (LEN + W - 1) / W;
    static constexpr int NTAIL = TAIL ? LEN % W : 0;
};
template <int KIND, bool COMPACT>
constexpr bool kTailRecord = COMPACT && KIND == 0;

// One element: loads, DJ-TLED force, stores of its npe rows into their slots.
// One fibre second-order invariant term: I = g^T M g (Sym6::quadratic_form,
// core.hpp:296-304), Ib = J^-4/3 I (kinematics.hpp:89-101), d = eta (Ib - 1),
// s += (J^-2/3 d) contract_ghat(g, Im), dev += 2 d Ib (djtled_force.hpp:18-24,
// 58-65).
template <class Real>
__device__ __forceinline__ void fibre_quad_term(const Real* M, const Real* Im, const Real g[6], Real j_m23, Real eta,
                                                Real s[6], Real& dev) {
    constexpr int idx[6][6] = {{0, 1, 2, 3, 4, 5},      {1, 6, 7, 8, 9, 10},    {2, 7, 11, 12, 13, 14},
                               {3, 8, 12, 15, 16, 17}, {4, 9, 13, 16, 18, 19}, {5, 10, 14, 17, 19, 20}};
    Real q = Real(0);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        Real row = M[idx[i][i]] * g[i];
#pragma unroll
        for (int j = i + 1; j < 6; ++j) row += Real(2) * M[idx[i][j]] * g[j];
        q += row * g[i];
    }
    const Real Ib = (j_m23 * j_m23) * q;
    const Real d = eta * (Ib - Real(1));
    Real cg[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) cg[k] = g[0] * Im[k];
#pragma unroll
    for (int m = 1; m < 6; ++m)
#pragma unroll
        for (int k = 0; k < 6; ++k) cg[k] = cg[k] + g[m] * Im[6 * m + k];
    const Real w = j_m23 * d;
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = s[k] + w * cg[k];
    dev += Real(2) * d * Ib;
}

// A row source that supplies the whole record of an element (the fused box
// step on a coordinate lattice: one record per tet kind and cell-size class).
template <class S, class = void>
struct SrcLattice : std::false_type {};
template <class S>
struct SrcLattice<S, std::void_t<decltype(S::kLattice)>> : std::bool_constant<S::kLattice> {};

// A row source that supplies a T4 tet's kinematics (Jt, g, det and the
// adjugate) from per-cell edge terms (the fused box step on a lattice).
template <class S, class = void>
struct SrcCellKin : std::false_type {};
template <class S>
struct SrcCellKin<S, std::void_t<decltype(S::kCellKin)>> : std::bool_constant<S::kCellKin> {};

// Compact T4 record, part 1 -- jacobian0 (element.hpp:59-77):
// J0[i][j] = sum_a D[i][a] x_a[j] with D[i] = (-1, e_i), summed from +0 in
// node order; the 0 * x terms cannot change a sum that is never -0, so
// J0[i][j] = (0 + -x_0[j]) + x_{i+1}[j] exactly; then det J0 and volume0
// (element.hpp:80-85).
template <class Node, class Real>
__device__ __forceinline__ void t4_jacobian0(int kind, const Node (&x)[4], Real* c) {
    const Real x0[3] = {Real(0) + -x[0].x, Real(0) + -x[0].y, Real(0) + -x[0].z};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        c[3 * i + 0] = x0[0] + x[i + 1].x;
        c[3 * i + 1] = x0[1] + x[i + 1].y;
        c[3 * i + 2] = x0[2] + x[i + 1].z;
    }
    const Real J0[3][3] = {{c[0], c[1], c[2]}, {c[3], c[4], c[5]}, {c[6], c[7], c[8]}};
    c[9] = em::det3(J0);
    c[10] = em::volume0(kind, c[9]);
}

// Compact record, part 2: the invariant tensors from J0^-1 and V0, the
// precompute's own arithmetic (element.hpp / invariants.hpp).
template <class Real, int KIND, int MODEL>
__device__ __forceinline__ void compact_record_tail(const ElemArgs<Real>& A, Real* c) {
    using L = Layout<KIND, MODEL>;
    const Real J0[3][3] = {{c[0], c[1], c[2]}, {c[3], c[4], c[5]}, {c[6], c[7], c[8]}};
    Real J0i[3][3];
    em::inv3(J0, c[9], J0i);
    em::first_invariant_tensors_fast(J0i, c[10], c + 11, c + 17);
    if constexpr (L::kI4) em::fibre_tensors(J0i, c[10], A.mat.A, c + L::m4, c + L::I4m);
    if constexpr (L::kI6) em::fibre_tensors(J0i, c[10], A.mat.B, c + L::m6, c + L::I6m);
    if constexpr (L::kI2) em::second_invariant_tensors(J0i, c[10], c + 11, c + L::M2, c + L::I2m);
}

template <class Real, int KIND, int MODEL, int RB, bool COMPACT, class Src>
__device__ __forceinline__ void element_body(const ElemArgs<Real>& A, const long long e,
                                             const typename RT<Real>::Node* __restrict__ u, const Src& src) {
    using L = Layout<KIND, MODEL>;
    using T = RT<Real>;
    static_assert(!(COMPACT && L::kI57), "the I57 energy runs on the full record only");
    constexpr int NPE = L::NPE;
    constexpr int NP = (L::count + T::kPlane - 1) / T::kPlane;

    // Connectivity (int32 node ids), 128-bit per 4 nodes.
    int nid[NPE];
#pragma unroll
    for (int p = 0; p < NPE / 4; ++p) {
        const int4 q = src.conn(p);
        nid[4 * p + 0] = q.x; nid[4 * p + 1] = q.y; nid[4 * p + 2] = q.z; nid[4 * p + 3] = q.w;
    }
#pragma unroll
    for (int a = 0; a < NPE; ++a) DJG_ASSERT(nid[a] >= 0 && nid[a] < A.N);
    // Gathered displacements of the element's nodes (issued first: their
    // latency overlaps the record loads and the compact rebuild).
    Real ux[NPE], uy[NPE], uz[NPE];
#pragma unroll
    for (int a = 0; a < NPE; ++a) {
        const typename T::Node v = src.node(a, u, nid[a]);
        ux[a] = v.x; uy[a] = v.y; uz[a] = v.z;
    }

    // Hot constants: the full record from HBM, or (compact) J0 [, det J0, V0,
    // hourglass data] from HBM and the rest rebuilt here with the
    // precompute's own arithmetic. H8: the planes holding only hourglass data
    // (k_hg, gamma: 33 Reals) are loaded just before the hourglass term, so
    // they do not occupy registers through the whole body.
    constexpr int NCR = COMPACT ? kCompactLen<KIND> : L::count;
    using RP = RecPlanes<Real, NCR, kTailRecord<KIND, COMPACT>>;
    constexpr int NC = RP::NFULL * T::kPlane + RP::NTAIL;
    constexpr int KHG = COMPACT ? kCompactRecord : L::khg;  // record index of k_hg (H8)
    constexpr int NPA = L::kH8 ? (KHG + T::kPlane - 1) / T::kPlane : RP::NFULL;  // planes loaded up front
    Real r[NC > 0 ? NC : 1];
#pragma unroll
    for (int p = 0; p < NPA; ++p) {
        const typename T::Plane v = src.plane(p);
        if constexpr (T::kPlane == 4) {
            r[4 * p + 0] = v.x; r[4 * p + 1] = v.y; r[4 * p + 2] = v.z; r[4 * p + 3] = v.w;
        } else {
            r[2 * p + 0] = v.x; r[2 * p + 1] = v.y;
        }
    }
#pragma unroll
    for (int t = 0; t < RP::NTAIL; ++t) r[RP::NFULL * T::kPlane + t] = src.tail(t);
    constexpr int NCU = L::kH8 ? KHG : NC;  // record fields used before the hourglass term
    Real c[COMPACT ? L::count + 1 : (NCU > 0 ? NCU : 1)];
    if constexpr (!COMPACT) {
#pragma unroll
        for (int k = 0; k < NCU; ++k) c[k] = r[k];
    } else {
        if constexpr (KIND == 0 && SrcLattice<Src>::value) {
            src.template lattice_record<L::count>(c);  // the whole record of this tet's lattice class (k_box_step)
        } else {
            if constexpr (KIND == 0) {
                const typename T::Node x[4] = {src.coord(A, nid[0]), src.coord(A, nid[1]), src.coord(A, nid[2]),
                                               src.coord(A, nid[3])};
                t4_jacobian0(KIND, x, c);
            } else {
#pragma unroll
                for (int k = 0; k < 11; ++k) c[k] = r[k];
            }
            compact_record_tail<Real, KIND, MODEL>(A, c);
        }
    }
    // update_jacobian (kinematics.hpp:31-45): Jt = J0 + D U.
    Real Jt[3][3];
    Real g[6];         // g_vector (the cell path has it here; else below)
    Real cof[3][3];    // adjugate entries (cell path)
    Real det;
    constexpr bool kCell = KIND == 0 && SrcCellKin<Src>::value;
    if constexpr (kCell) {
        src.cell_kinematics(Jt, g, cof, det);
    } else if constexpr (KIND == 0) {
        // T4: D[i] = (-1, e_i): du = u_{i+1} - u_0 (the reference's sum
        // 0 - u0 + u_{i+1} + 0 + 0 rounds identically).
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            Jt[i][0] = c[3 * i + 0] + (ux[i + 1] - ux[0]);
            Jt[i][1] = c[3 * i + 1] + (uy[i + 1] - uy[0]);
            Jt[i][2] = c[3 * i + 2] + (uz[i + 1] - uz[0]);
        }
    } else {
        // H8: D[i][a] = sign/8; summing the signed terms first and scaling by
        // the exact power of two 1/8 afterwards gives the same rounding.
        constexpr int S[8][3] = {{-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
                                 {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1}};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            Real sx = S[0][i] > 0 ? ux[0] : -ux[0];
            Real sy = S[0][i] > 0 ? uy[0] : -uy[0];
            Real sz = S[0][i] > 0 ? uz[0] : -uz[0];
#pragma unroll
            for (int a = 1; a < 8; ++a) {
                if (S[a][i] > 0) { sx = sx + ux[a]; sy = sy + uy[a]; sz = sz + uz[a]; }
                else { sx = sx - ux[a]; sy = sy - uy[a]; sz = sz - uz[a]; }
            }
            Jt[i][0] = c[3 * i + 0] + Real(0.125) * sx;
            Jt[i][1] = c[3 * i + 1] + Real(0.125) * sy;
            Jt[i][2] = c[3 * i + 2] + Real(0.125) * sz;
        }
    }

    // det / inversion test / adjugate inverse (core.hpp:187-212).
    if constexpr (!kCell)
        det = Jt[0][0] * (Jt[1][1] * Jt[2][2] - Jt[1][2] * Jt[2][1]) -
              Jt[0][1] * (Jt[1][0] * Jt[2][2] - Jt[1][2] * Jt[2][0]) +
              Jt[0][2] * (Jt[1][0] * Jt[2][1] - Jt[1][1] * Jt[2][0]);

    int sl[NPE];  // slot positions fit in 32 bits (checked at engine creation)
    {
        int rk[NPE];
        src.template ranks<NPE, RB>(rk);
#pragma unroll
        for (int a = 0; a < NPE; ++a) sl[a] = src.slot(A.slice_base, a, nid[a], rk[a]);
    }

    if (!(det > Real(0))) {
        // record_inversion (djtled_force.hpp:107-112) + zeroed rows (:187-191).
        if (counts_inversion(A, src, e)) atomicAdd(&A.ctrl->inv_count, 1ull);
        atomicMin(&A.ctrl->first_inv, (unsigned long long)(A.elem_l2g ? A.elem_l2g[e] : e));
#pragma unroll
        for (int a = 0; a < NPE; ++a) emit_row(A, src, sl[a], Real(0), Real(0), Real(0));
        return;
    }
    const Real s_inv = Real(1) / det;
    Real Ji[3][3];
    if constexpr (kCell) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) Ji[i][j] = cof[i][j] * s_inv;
    } else {
        Ji[0][0] = (Jt[1][1] * Jt[2][2] - Jt[1][2] * Jt[2][1]) * s_inv;
        Ji[0][1] = (Jt[0][2] * Jt[2][1] - Jt[0][1] * Jt[2][2]) * s_inv;
        Ji[0][2] = (Jt[0][1] * Jt[1][2] - Jt[0][2] * Jt[1][1]) * s_inv;
        Ji[1][0] = (Jt[1][2] * Jt[2][0] - Jt[1][0] * Jt[2][2]) * s_inv;
        Ji[1][1] = (Jt[0][0] * Jt[2][2] - Jt[0][2] * Jt[2][0]) * s_inv;
        Ji[1][2] = (Jt[0][2] * Jt[1][0] - Jt[0][0] * Jt[1][2]) * s_inv;
        Ji[2][0] = (Jt[1][0] * Jt[2][1] - Jt[1][1] * Jt[2][0]) * s_inv;
        Ji[2][1] = (Jt[0][1] * Jt[2][0] - Jt[0][0] * Jt[2][1]) * s_inv;
        Ji[2][2] = (Jt[0][0] * Jt[1][1] - Jt[0][1] * Jt[1][0]) * s_inv;
    }

    // volume_ratio, g_vector, invariants (kinematics.hpp:47-103).
    const Real J = det / c[9];
    if constexpr (!kCell) {
        g[0] = Jt[0][0] * Jt[0][0] + Jt[0][1] * Jt[0][1] + Jt[0][2] * Jt[0][2];
        g[1] = Jt[1][0] * Jt[1][0] + Jt[1][1] * Jt[1][1] + Jt[1][2] * Jt[1][2];
        g[2] = Jt[2][0] * Jt[2][0] + Jt[2][1] * Jt[2][1] + Jt[2][2] * Jt[2][2];
        g[3] = Jt[0][0] * Jt[1][0] + Jt[0][1] * Jt[1][1] + Jt[0][2] * Jt[1][2];
        g[4] = Jt[0][0] * Jt[2][0] + Jt[0][1] * Jt[2][1] + Jt[0][2] * Jt[2][2];
        g[5] = Jt[1][0] * Jt[2][0] + Jt[1][1] * Jt[2][1] + Jt[1][2] * Jt[2][2];
    }
    const Real cb = ref_cbrt(J);
    const Real j_m23 = Real(1) / (cb * cb);
    const Real I1 = g[0] * c[11] + g[1] * c[12] + g[2] * c[13] + g[3] * c[14] + g[4] * c[15] + g[5] * c[16];
    const Real Ib1 = j_m23 * I1;

    // energy_derivatives + the Table 3 bracket (djtled_force.hpp:36-82).
    const Real dJ = A.mat.kappa * (J - Real(1));
    Real s[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        // (the lattice table holds dI1 I1m already: the same product, once per class)
        if constexpr (KIND == 0 && SrcLattice<Src>::value) s[k] = c[17 + k];
        else s[k] = A.mat.dI1 * c[17 + k];
    }
    Real dev = A.mat.dI1 * Ib1;
    if constexpr (L::kI4) {
        const Real I4 = g[0] * c[L::m4 + 0] + g[1] * c[L::m4 + 1] + g[2] * c[L::m4 + 2] + g[3] * c[L::m4 + 3] +
                        g[4] * c[L::m4 + 4] + g[5] * c[L::m4 + 5];
        const Real Ib4 = j_m23 * I4;
        const Real dI4 = A.mat.eta_a * (Ib4 - Real(1));
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k] = s[k] + dI4 * c[L::I4m + k];
        dev += dI4 * Ib4;
    }
    if constexpr (L::kI6) {
        const Real I6 = g[0] * c[L::m6 + 0] + g[1] * c[L::m6 + 1] + g[2] * c[L::m6 + 2] + g[3] * c[L::m6 + 3] +
                        g[4] * c[L::m6 + 4] + g[5] * c[L::m6 + 5];
        const Real Ib6 = j_m23 * I6;
        const Real dI6 = A.mat.eta_b * (Ib6 - Real(1));
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k] = s[k] + dI6 * c[L::I6m + k];
        dev += dI6 * Ib6;
    }
    if constexpr (L::kI2) {
        // I2 = g^T M2 g (Sym6::quadratic_form, core.hpp:296-304).
        constexpr int idx[6][6] = {{0, 1, 2, 3, 4, 5},      {1, 6, 7, 8, 9, 10},    {2, 7, 11, 12, 13, 14},
                                   {3, 8, 12, 15, 16, 17}, {4, 9, 13, 16, 18, 19}, {5, 10, 14, 17, 19, 20}};
        Real q = Real(0);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            Real row = c[L::M2 + idx[i][i]] * g[i];
#pragma unroll
            for (int j = i + 1; j < 6; ++j) row += Real(2) * c[L::M2 + idx[i][j]] * g[j];
            q += row * g[i];
        }
        const Real j_m43 = j_m23 * j_m23;
        const Real Ib2 = j_m43 * q;
        // contract_ghat (djtled_force.hpp:18-24)
        Real cg[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) cg[k] = g[0] * c[L::I2m + k];
#pragma unroll
        for (int m = 1; m < 6; ++m)
#pragma unroll
            for (int k = 0; k < 6; ++k) cg[k] = cg[k] + g[m] * c[L::I2m + 6 * m + k];
        const Real w = j_m23 * A.mat.dI2;
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k] = s[k] + w * cg[k];
        dev += Real(2) * A.mat.dI2 * Ib2;
    }
    if constexpr (L::kI57) {
        // need.i5 then need.i7 (djtled_force.hpp:58-65) with the test
        // energy's dI5 = eta5 (Ib5 - 1), dI7 = eta7 (Ib7 - 1).
        fibre_quad_term(c + L::M5, c + L::I5m, g, j_m23, A.mat.eta_a, s, dev);
        fibre_quad_term(c + L::M7, c + L::I7m, g, j_m23, A.mat.eta_b, s, dev);
    }
    const Real cc = (-Real(2) / Real(3) * dev + J * dJ) * c[10];

    // K = j_m23 (Jt^T S) + c Jt^-1
    const Real Sm[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    Real K[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const Real mt = Jt[0][i] * Sm[0][j] + Jt[1][i] * Sm[1][j] + Jt[2][i] * Sm[2][j];
            K[i][j] = j_m23 * mt + cc * Ji[i][j];
        }

    if constexpr (KIND == 0) {
        // T4 rows: f1..f3 = columns of K, f0 = -(f1 + f2 + f3).
        emit_row(A, src, sl[1], K[0][0], K[1][0], K[2][0]);
        emit_row(A, src, sl[2], K[0][1], K[1][1], K[2][1]);
        emit_row(A, src, sl[3], K[0][2], K[1][2], K[2][2]);
        emit_row(A, src, sl[0], Real(-1) * ((K[0][0] + K[0][1]) + K[0][2]), Real(-1) * ((K[1][0] + K[1][1]) + K[1][2]),
                  Real(-1) * ((K[2][0] + K[2][1]) + K[2][2]));
    } else {
        // Hourglass data: the remaining record planes, loaded now.
#pragma unroll
        for (int p = NPA; p < RP::NFULL; ++p) {
            const typename T::Plane v = src.plane(p);
            if constexpr (T::kPlane == 4) {
                r[4 * p + 0] = v.x; r[4 * p + 1] = v.y; r[4 * p + 2] = v.z; r[4 * p + 3] = v.w;
            } else {
                r[2 * p + 0] = v.x; r[2 * p + 1] = v.y;
            }
        }
        const Real khg = r[KHG];
        const Real* gamma = r + KHG + 1;  // gamma[8 m + b]
        // hourglass_force (djtled_force.hpp:86-95): q_m = sum_b gamma_mb u_b
        // (b ascending), then every row b adds k_hg gamma_mb q_m for m = 0..3
        // in order -- each row is finished and stored in turn, same sums.
        Real q[4][3];
        if (khg != Real(0)) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                Real q0 = Real(0), q1 = Real(0), q2 = Real(0);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const Real gm = gamma[8 * m + b];
                    q0 = q0 + gm * ux[b];
                    q1 = q1 + gm * uy[b];
                    q2 = q2 + gm * uz[b];
                }
                q[m][0] = q0; q[m][1] = q1; q[m][2] = q2;
            }
        }
        constexpr int S[8][3] = {{-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
                                 {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1}};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            Real f[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                // D0a K[i][0] + D1a K[i][1] + D2a K[i][2] with D = sign/8.
                Real t = S[a][0] > 0 ? K[i][0] : -K[i][0];
                t = S[a][1] > 0 ? t + K[i][1] : t - K[i][1];
                t = S[a][2] > 0 ? t + K[i][2] : t - K[i][2];
                f[i] = Real(0.125) * t;
            }
            if (khg != Real(0)) {
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const Real kg = khg * gamma[8 * m + a];
                    f[0] = f[0] + kg * q[m][0];
                    f[1] = f[1] + kg * q[m][1];
                    f[2] = f[2] + kg * q[m][2];
                }
            }
            emit_row(A, src, sl[a], f[0], f[1], f[2]);
        }
    }
}

// Select by value: indexing the kernel-parameter array with a runtime value
// would copy the whole parameter block to local memory.
template <class P>
__device__ __forceinline__ P pick3(int i, P a, P b, P c) {
    return i == 0 ? a : (i == 1 ? b : c);
}

// Elements [e0, e1) of the step (one slab).
// Blocks per SM the one-shot kernel's registers are sized for. Left alone,
// ptxas gives the f32 H8 bodies ~170 registers (3 blocks, 12 warps per SM)
// to hoist every record load; capping at 5 blocks (~96 registers) is 10-20 %
// faster for NH / TI / OT (cfg4-sized meshes). The f64 NH / TI / OT bodies
// (~210-250 registers uncapped) run 7-16 % faster capped at 3 blocks. The MR
// bodies spill under a cap and stay uncapped (tools/ab_h8_caps.sh).
#ifndef DJG_K1_MINB_H8
#define DJG_K1_MINB_H8 5
#endif
#ifndef DJG_K1_MINB_H8_MR
#define DJG_K1_MINB_H8_MR 1
#endif
#ifndef DJG_K1_MINB_H8_64
#define DJG_K1_MINB_H8_64 3
#endif
template <class Real, int KIND, int MODEL>
constexpr int kElemMinBlocks = KIND != 1 ? 1
                               : MODEL >= 3 ? DJG_K1_MINB_H8_MR
                               : sizeof(Real) == 8 ? DJG_K1_MINB_H8_64 : DJG_K1_MINB_H8;

template <class Real, int KIND, int MODEL, int RB, bool COMPACT>
__global__ void __launch_bounds__(128, (kElemMinBlocks<Real, KIND, MODEL>)) k_element(const ElemArgs<Real> A, long long e0, long long e1) {
    const long long e = e0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e1) return;
    if (__ldcg(&A.ctrl->halted)) return;
    const int phase = int(__ldcg(&A.ctrl->step) % 3);
    const typename RT<Real>::Node* u = A.u_override ? A.u_override : pick3(phase, A.u[0], A.u[1], A.u[2]);
    element_body<Real, KIND, MODEL, RB, COMPACT>(A, e, u, GlobalSrc<Real>{A, e});
}

// ------------------------------------------------------------------ TLED

// The conventional total Lagrangian path the paper compares against
// (tled_force.hpp): X = I + sum_a u_a B0_a^T, C = X^T X,
// C^-1, invariants from C, second Piola-Kirchhoff stress, F = X S B0 V0.
// Same slots, gather and update as the DJ-TLED step; record per element:
// B0 (npe x 3), V0 [, k_hg, gamma (H8)].
template <int KIND>
struct TledLayout {
    static constexpr int NPE = KIND == 1 ? 8 : 4;
    static constexpr int V0 = 3 * NPE;
    static constexpr int khg = V0 + 1;
    static constexpr int gamma = khg + 1;
    static constexpr int count = KIND == 1 ? gamma + 32 : V0 + 1;
};

template <class Real, int KIND, int MODEL, int RB, class Src>
__device__ __forceinline__ void element_body_tled(const ElemArgs<Real>& A, const long long e,
                                                  const typename RT<Real>::Node* __restrict__ u, const Src& src) {
    using T = RT<Real>;
    using TL = TledLayout<KIND>;
    using L = Layout<KIND, MODEL>;
    constexpr int NPE = TL::NPE;
    constexpr int NP = (TL::count + T::kPlane - 1) / T::kPlane;
    int nid[NPE];
#pragma unroll
    for (int p = 0; p < NPE / 4; ++p) {
        const int4 q = src.conn(p);
        nid[4 * p + 0] = q.x; nid[4 * p + 1] = q.y; nid[4 * p + 2] = q.z; nid[4 * p + 3] = q.w;
    }
#pragma unroll
    for (int a = 0; a < NPE; ++a) DJG_ASSERT(nid[a] >= 0 && nid[a] < A.N);
    Real c[NP * T::kPlane];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const typename T::Plane v = src.plane(p);
        if constexpr (T::kPlane == 4) {
            c[4 * p + 0] = v.x; c[4 * p + 1] = v.y; c[4 * p + 2] = v.z; c[4 * p + 3] = v.w;
        } else {
            c[2 * p + 0] = v.x; c[2 * p + 1] = v.y;
        }
    }
    Real uu[NPE][3];
#pragma unroll
    for (int a = 0; a < NPE; ++a) {
        const typename T::Node v = src.node(a, u, nid[a]);
        uu[a][0] = v.x; uu[a][1] = v.y; uu[a][2] = v.z;
    }
    int sl[NPE];
    {
        int rk[NPE];
        src.template ranks<NPE, RB>(rk);
#pragma unroll
        for (int a = 0; a < NPE; ++a) sl[a] = src.slot(A.slice_base, a, nid[a], rk[a]);
    }
    // deformation_gradient (tled_force.hpp:28-36)
    Real X[3][3] = {{Real(1), Real(0), Real(0)}, {Real(0), Real(1), Real(0)}, {Real(0), Real(0), Real(1)}};
#pragma unroll
    for (int a = 0; a < NPE; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) X[i][j] += uu[a][i] * c[3 * a + j];
    // deformation_state (tled_force.hpp:39-48)
    const Real J = em::det3(X);
    if (!(J > Real(0))) {
        if (counts_inversion(A, src, e)) atomicAdd(&A.ctrl->inv_count, 1ull);
        atomicMin(&A.ctrl->first_inv, (unsigned long long)(A.elem_l2g ? A.elem_l2g[e] : e));
#pragma unroll
        for (int a = 0; a < NPE; ++a) emit_row(A, src, sl[a], Real(0), Real(0), Real(0));
        return;
    }
    Real m[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) m[i][j] = X[0][i] * X[0][j] + X[1][i] * X[1][j] + X[2][i] * X[2][j];
    const Real C[6] = {m[0][0], m[1][1], m[2][2], (m[0][1] + m[1][0]) / 2, (m[0][2] + m[2][0]) / 2,
                       (m[1][2] + m[2][1]) / 2};
    const Real Cf[3][3] = {{C[0], C[3], C[4]}, {C[3], C[1], C[5]}, {C[4], C[5], C[2]}};
    Real ci[3][3];
    em::inv3(Cf, em::det3(Cf), ci);
    const Real Ci[6] = {ci[0][0], ci[1][1], ci[2][2], (ci[0][1] + ci[1][0]) / 2, (ci[0][2] + ci[2][0]) / 2,
                        (ci[1][2] + ci[2][1]) / 2};
    // conventional_invariants (tled_force.hpp:51-94)
    const Real cb = ref_cbrt(J);
    const Real j_m23 = Real(1) / (cb * cb);
    const Real j_m43 = j_m23 * j_m23;
    const Real I1 = C[0] + C[1] + C[2];
    const Real Ib1 = j_m23 * I1;
    // energy_derivatives + second_pk_stress (material.hpp:266-290, tled_force.hpp:101-135)
    const Real dJ = A.mat.kappa * (J - Real(1));
    Real iso[6];
    const Real ident[6] = {Real(1), Real(1), Real(1), Real(0), Real(0), Real(0)};
#pragma unroll
    for (int k = 0; k < 6; ++k) iso[k] = A.mat.dI1 * ident[k];
    Real dev = A.mat.dI1 * Ib1;
    if constexpr (L::kI4) {
        const Real* a = A.mat.fa;
        Real ca[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) ca[i] = Cf[i][0] * a[0] + Cf[i][1] * a[1] + Cf[i][2] * a[2];
        const Real Ib4 = j_m23 * (a[0] * ca[0] + a[1] * ca[1] + a[2] * ca[2]);
        const Real dI4 = A.mat.eta_a * (Ib4 - Real(1));
#pragma unroll
        for (int k = 0; k < 6; ++k) iso[k] = iso[k] + dI4 * A.mat.A[k];
        dev += dI4 * Ib4;
    }
    if constexpr (L::kI6) {
        const Real* b = A.mat.fb;
        Real cbv[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) cbv[i] = Cf[i][0] * b[0] + Cf[i][1] * b[1] + Cf[i][2] * b[2];
        const Real Ib6 = j_m23 * (b[0] * cbv[0] + b[1] * cbv[1] + b[2] * cbv[2]);
        const Real dI6 = A.mat.eta_b * (Ib6 - Real(1));
#pragma unroll
        for (int k = 0; k < 6; ++k) iso[k] = iso[k] + dI6 * A.mat.B[k];
        dev += dI6 * Ib6;
    }
    Real s[6];
    const Real two_jm23 = 2 * j_m23;
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = two_jm23 * iso[k];
    if constexpr (L::kI2) {
        const Real I2 = (I1 * I1 - em::ddot(C, C)) / 2;
        const Real Ib2 = j_m43 * I2;
        const Real ker[6] = {I1 - C[0], I1 - C[1], I1 - C[2], -C[3], -C[4], -C[5]};
        const Real w = 2 * j_m43 * A.mat.dI2;
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k] = s[k] + w * ker[k];
        dev += 2 * A.mat.dI2 * Ib2;
    }
    const Real cc = -Real(2) / Real(3) * dev + J * dJ;
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = s[k] + cc * Ci[k];
    // tled_element_force (tled_force.hpp:147-156): F = X S B0 V0
    const Real Sf[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    Real P[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) P[i][j] = X[i][0] * Sf[0][j] + X[i][1] * Sf[1][j] + X[i][2] * Sf[2][j];
    const Real V0 = c[TL::V0];
    Real f[NPE][3];
#pragma unroll
    for (int a = 0; a < NPE; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            f[a][i] = V0 * (c[3 * a + 0] * P[i][0] + c[3 * a + 1] * P[i][1] + c[3 * a + 2] * P[i][2]);
    if constexpr (KIND == 1) {
        // hourglass_force (djtled_force.hpp:86-95)
        const Real khg = c[TL::khg];
        if (khg != Real(0)) {
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
                Real q0 = Real(0), q1 = Real(0), q2 = Real(0);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const Real gm = c[TL::gamma + 8 * mm + b];
                    q0 = q0 + gm * uu[b][0];
                    q1 = q1 + gm * uu[b][1];
                    q2 = q2 + gm * uu[b][2];
                }
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const Real kg = khg * c[TL::gamma + 8 * mm + b];
                    f[b][0] = f[b][0] + kg * q0;
                    f[b][1] = f[b][1] + kg * q1;
                    f[b][2] = f[b][2] + kg * q2;
                }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < NPE; ++a) emit_row(A, src, sl[a], f[a][0], f[a][1], f[a][2]);
}

template <class Real, int KIND, int MODEL, int RB>
__global__ void __launch_bounds__(128) k_element_tled(const ElemArgs<Real> A, long long e0, long long e1) {
    const long long e = e0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e1) return;
    if (__ldcg(&A.ctrl->halted)) return;
    const int phase = int(__ldcg(&A.ctrl->step) % 3);
    const typename RT<Real>::Node* u = A.u_override ? A.u_override : pick3(phase, A.u[0], A.u[1], A.u[2]);
    element_body_tled<Real, KIND, MODEL, RB>(A, e, u, GlobalSrc<Real>{A, e});
}

// ------------------------------------------------------------------ K1, pipelined

// The per-element streams (connectivity, rank words, record planes) are
// plain contiguous runs of 16-byte rows, so a persistent block can move a
// whole tile of them into shared memory with a handful of bulk async copies
// (cp.async.bulk, TMA unit, completion on an mbarrier) several tiles ahead of
// the threads computing on it. The dependent node gather u[conn[e]] then
// starts from shared memory instead of waiting on an HBM round trip, and the
// bytes in flight per SM no longer depend on registers or resident warps.
// Warp 4 of each block is the producer; warps 0-3 compute one element per
// thread with exactly the arithmetic of k_element / k_element_tled.

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "DJG_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra DJG_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// bytes: multiple of 16; src and dst 16-byte aligned.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

#ifndef DJG_PIPE_TILE
#define DJG_PIPE_TILE 128
#endif
constexpr int kPipeTile = DJG_PIPE_TILE;  // elements per tile = compute threads per block

// Stage layout: connectivity planes, record planes, record tail planes, rank words.
template <class Real, int KIND, int MODEL, int RB, int FORM>  // FORM 0 full, 1 compact, 2 TLED
struct PipeShape {
    using T = RT<Real>;
    static constexpr int NPE = KIND == 1 ? 8 : 4;
    static constexpr int NCP = NPE / 4;
    static constexpr int kRecLen = FORM == 2   ? TledLayout<KIND>::count
                                   : FORM == 1 ? kCompactLen<KIND>
                                               : Layout<KIND, MODEL>::count;
    using RP = RecPlanes<Real, kRecLen, FORM == 1 && kTailRecord<KIND, true>>;
    static constexpr int NRP = RP::NFULL;
    static constexpr int NTAIL = RP::NTAIL;
    static constexpr int kRankBytes = NPE * RB;
    static constexpr int kConnOff = 0, kRecOff = kPipeTile * 16 * NCP, kTailOff = kRecOff + kPipeTile * 16 * NRP;
    static constexpr int kRankOff = kTailOff + kPipeTile * int(sizeof(Real)) * NTAIL;
    static constexpr int kStageBytes = kRankOff + kPipeTile * kRankBytes;
    static constexpr size_t smem_bytes(int stages) { return size_t(stages) * kStageBytes + 2 * 8 * size_t(stages); }
};

// Blocks per SM the register allocation is sized for, per material and
// precision (DJG_PIPE_MINB_T4C{,64}_M<model>, measured on a 10.4M-tet cube,
// tools/ab_models.py): f32 NH 6 (64 registers), TI 5, OT 4, MR 3; f64 NH 4,
// TI 3, OT 2. Tighter caps spill the heavier bodies; looser ones lose latency
// hiding. (f64 MR keeps the full record by default.) The full-record forms
// are left uncapped.
#ifndef DJG_PIPE_MINB_T4C
#define DJG_PIPE_MINB_T4C 6
#endif
#ifndef DJG_PIPE_MINB_OTHER
#define DJG_PIPE_MINB_OTHER 1
#endif
#ifndef DJG_PIPE_MINB_T4C64
#define DJG_PIPE_MINB_T4C64 4
#endif
#ifndef DJG_PIPE_MINB_T4C_M1
#define DJG_PIPE_MINB_T4C_M1 5
#endif
#ifndef DJG_PIPE_MINB_T4C_M2
#define DJG_PIPE_MINB_T4C_M2 4
#endif
#ifndef DJG_PIPE_MINB_T4C_M3
#define DJG_PIPE_MINB_T4C_M3 3
#endif
#ifndef DJG_PIPE_MINB_T4C64_M1
#define DJG_PIPE_MINB_T4C64_M1 3
#endif
#ifndef DJG_PIPE_MINB_T4C64_M2
#define DJG_PIPE_MINB_T4C64_M2 2
#endif
#ifndef DJG_PIPE_MINB_T4C64_M3
#define DJG_PIPE_MINB_T4C64_M3 2
#endif
template <class Real, int MODEL>
constexpr int kPipeMinBlocksT4C =
    sizeof(Real) == 4 ? (MODEL == 1 ? DJG_PIPE_MINB_T4C_M1 : MODEL == 2 ? DJG_PIPE_MINB_T4C_M2
                                                   : MODEL == 3 ? DJG_PIPE_MINB_T4C_M3 : DJG_PIPE_MINB_T4C)
                      : (MODEL == 1 ? DJG_PIPE_MINB_T4C64_M1 : MODEL == 2 ? DJG_PIPE_MINB_T4C64_M2
                                                     : MODEL == 3 ? DJG_PIPE_MINB_T4C64_M3 : DJG_PIPE_MINB_T4C64);
template <class Real, int KIND, int MODEL, int FORM>
#ifndef DJG_PIPE_MINB_H8
#define DJG_PIPE_MINB_H8 3
#endif
constexpr int kPipeMinBlocks = (KIND == 0 && FORM == 1) ? kPipeMinBlocksT4C<Real, MODEL>
                               : (KIND == 1 && FORM == 1 && sizeof(Real) == 4 && MODEL != 3) ? DJG_PIPE_MINB_H8
                                                                                             : DJG_PIPE_MINB_OTHER;
constexpr int kPipeThreads = kPipeTile + 32;  // 4 compute warps + the producer warp

// Persistent blocks; tile `it` of a block (global tile blockIdx + it * grid)
// lives in stage it % STAGES. A dedicated producer warp (warp 4) issues the
// copies of a tile once all four compute warps have released its stage
// (empty barrier), running up to STAGES tiles ahead. (Issuing from thread 0
// of a compute warp instead, or also prefetching the next tile's gathers,
// measured slower.)
template <class Real, int KIND, int MODEL, int RB, int FORM, int STAGES>
__global__ void __launch_bounds__(kPipeThreads, (kPipeMinBlocks<Real, KIND, MODEL, FORM>)) k_element_pipe(const ElemArgs<Real> A, long long e0,
                                                                              long long e1) {
    using PS = PipeShape<Real, KIND, MODEL, RB, FORM>;
    using Plane = typename RT<Real>::Plane;
    using Node = typename RT<Real>::Node;
    static_assert(STAGES >= 2, "pipeline needs at least two stages");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + STAGES * PS::kStageBytes);
    unsigned long long* empty = full + STAGES;
    const int tid = threadIdx.x;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kPipeTile / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (__ldcg(&A.ctrl->halted)) return;
    const long long ntiles = (e1 - e0 + kPipeTile - 1) / kPipeTile;
    const long long G = gridDim.x;
    const long long nmine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    unsigned long long pol = 0;

    // Bulk copies of this block's tile number `it` into stage it % STAGES.
    auto issue = [&](long long it) {
        const int s = int(it % STAGES);
        if (it >= STAGES) mbar_wait(empty + s, unsigned((it / STAGES - 1) & 1));
        const long long eb = e0 + (blockIdx.x + it * G) * kPipeTile;
        const unsigned n = unsigned(min((long long)kPipeTile, e1 - eb));
        const unsigned rbytes = (n * PS::kRankBytes + 15u) & ~15u;  // rank array is padded by 16 bytes
        const unsigned tbytes = (n * unsigned(sizeof(Real)) + 15u) & ~15u;  // tail planes likewise
        mbar_expect_tx(full + s, n * 16u * (PS::NCP + PS::NRP) + tbytes * PS::NTAIL + rbytes);
        unsigned char* st = smem + s * PS::kStageBytes;
#pragma unroll
        for (int p = 0; p < PS::NCP; ++p)
            bulk_load(st + PS::kConnOff + p * kPipeTile * 16, A.conn + (long long)p * A.E + eb, n * 16u, full + s, pol);
#pragma unroll
        for (int p = 0; p < PS::NRP; ++p)
            bulk_load(st + PS::kRecOff + p * kPipeTile * 16, A.c + (long long)p * A.E + eb, n * 16u, full + s, pol);
#pragma unroll
        for (int t = 0; t < PS::NTAIL; ++t)
            bulk_load(st + PS::kTailOff + t * kPipeTile * int(sizeof(Real)), A.ctail + t * A.tail_stride + eb, tbytes,
                      full + s, pol);
        bulk_load(st + PS::kRankOff, static_cast<const unsigned char*>(A.rank) + eb * PS::kRankBytes, rbytes, full + s,
                  pol);
    };
    if (tid >= kPipeTile) {  // producer warp
        if (tid == kPipeTile) {
            pol = l2_evict_first_policy();
            for (long long it = 0; it < nmine; ++it) issue(it);
        }
        return;
    }

    const int phase = int(__ldcg(&A.ctrl->step) % 3);
    const Node* u = A.u_override ? A.u_override : pick3(phase, A.u[0], A.u[1], A.u[2]);
    for (long long it = 0; it < nmine; ++it) {
        const int s = int(it % STAGES);
        mbar_wait(full + s, unsigned((it / STAGES) & 1));
        const long long e = e0 + (blockIdx.x + it * G) * kPipeTile + tid;
        if (e < e1) {
            const unsigned char* st = smem + s * PS::kStageBytes;
            const SmemSrc<Real, kPipeTile> src{reinterpret_cast<const int4*>(st + PS::kConnOff),
                                               reinterpret_cast<const Plane*>(st + PS::kRecOff), st + PS::kRankOff,
                                               reinterpret_cast<const Real*>(st + PS::kTailOff), tid,
                                               A.slice_w};
            if constexpr (FORM == 2) element_body_tled<Real, KIND, MODEL, RB>(A, e, u, src);
            else element_body<Real, KIND, MODEL, RB, FORM == 1>(A, e, u, src);
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(empty + s);
    }
}

// ------------------------------------------------------------------ K1, node windows

// A 128-element tile of a mesh numbered with some locality touches its nodes
// in a few contiguous id runs (the cube: <= 6 runs, <= 96 nodes per T4 tile,
// <= 528 per H8 tile). The engine lists each tile's runs once (kWinDesc ints:
// nruns, window length, then (first node, window offset) per run) and gives
// every element-node its index in the tile's window. The producer warp then
// moves the window's displacements (and, for the compact T4 record, the
// reference coordinates) into the stage with one bulk copy per run, next to
// the slot positions, window indices and record planes of the tile: the
// compute warps read every input from shared memory and only store to HBM,
// so the dependent node gather no longer sits on their critical path.
// Tiles whose nodes do not fit (more than kWinRuns runs or kWinCap nodes)
// are flagged nruns = 0 and stage their connectivity instead (global gather,
// as in k_element_pipe). Arithmetic and slot positions are unchanged:
// bit-identical to k_element / k_element_pipe.
constexpr int kWinDesc = 16;  // ints per tile descriptor
constexpr int kWinRuns = 7;   // runs per tile descriptor
#ifndef DJG_WIN_CAP_T4
#define DJG_WIN_CAP_T4 128
#endif
#ifndef DJG_WIN_CAP_H8
#define DJG_WIN_CAP_H8 576
#endif
template <int KIND>
constexpr int kWinCap = KIND == 1 ? DJG_WIN_CAP_H8 : DJG_WIN_CAP_T4;
template <int KIND>
constexpr int kWinIdxBytes = kWinCap<KIND> <= 256 ? 1 : 2;

template <class Real, int KIND, int MODEL, int FORM>  // FORM 0 full, 1 compact, 2 TLED
struct WinShape {
    using T = RT<Real>;
    using Node = typename T::Node;
    static constexpr int NPE = KIND == 1 ? 8 : 4;
    static constexpr int NCP = NPE / 4;
    static constexpr int LB = kWinIdxBytes<KIND>;
    static constexpr int CAP = kWinCap<KIND>;
    static constexpr int NX = (FORM == 1 && KIND == 0) ? 2 : 1;  // u (+ X for the compact T4 rebuild)
    static constexpr int kRecLen = FORM == 2   ? TledLayout<KIND>::count
                                   : FORM == 1 ? kCompactLen<KIND>
                                               : Layout<KIND, MODEL>::count;
    using RP = RecPlanes<Real, kRecLen, FORM == 1 && kTailRecord<KIND, true>>;
    static constexpr int NRP = RP::NFULL;
    static constexpr int NTAIL = RP::NTAIL;
    static constexpr int kSlotOff = 0;
    static constexpr int kIdxOff = kSlotOff + kPipeTile * 16 * NCP;
    static constexpr int kRecOff = kIdxOff + kPipeTile * NPE * LB;
    static constexpr int kTailOff = kRecOff + kPipeTile * 16 * NRP;
    static constexpr int kWinOff = (kTailOff + kPipeTile * int(sizeof(Real)) * NTAIL + 15) / 16 * 16;
    static constexpr int kWinBytes = CAP * int(sizeof(Node)) * NX > kPipeTile * 16 * NCP
                                         ? CAP * int(sizeof(Node)) * NX
                                         : kPipeTile * 16 * NCP;  // (fallback tiles: connectivity planes)
    static constexpr int kModeOff = kWinOff + kWinBytes;  // the tile's run count (0: global gather)
    static constexpr int kStageBytes = kModeOff + 16;
    static constexpr size_t smem_bytes(int stages) { return size_t(stages) * kStageBytes + 2 * 8 * size_t(stages); }
};

// Inputs of a windowed tile: everything from the stage.
template <class Real, int TILE, int NPE, int LB>
struct WinSrc {
    using Node = typename RT<Real>::Node;
    const int4* sslot;                     // [NPE/4][TILE] slot positions
    const void* sidx;                      // [TILE] window indices
    const typename RT<Real>::Plane* srec;  // [planes][TILE]
    const Real* stail;                     // [NTAIL][TILE]
    const Node* wu;                        // window displacements
    const Node* wx;                        // window coordinates (compact T4)
    int i;
    __device__ __forceinline__ int4 conn(int p) const {
        if constexpr (LB == 1) {
            static_assert(NPE == 4, "uint8 window indices: T4");
            const unsigned w = static_cast<const unsigned*>(sidx)[i];
            return make_int4(int(w & 0xff), int((w >> 8) & 0xff), int((w >> 16) & 0xff), int(w >> 24));
        } else {
            const uint2 q = static_cast<const uint2*>(sidx)[i * (NPE / 4) + p];
            return make_int4(int(q.x & 0xffff), int(q.x >> 16), int(q.y & 0xffff), int(q.y >> 16));
        }
    }
    __device__ __forceinline__ Node node(int, const Node* __restrict__, int h) const { return wu[h]; }
    __device__ __forceinline__ Node coord(const ElemArgs<Real>&, int h) const { return wx[h]; }
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const { return srec[p * TILE + i]; }
    __device__ __forceinline__ Real tail(int t) const { return stail[t * TILE + i]; }
    template <int N, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[N]) const {
#pragma unroll
        for (int a = 0; a < N; ++a) rk[a] = 0;
    }
    __device__ __forceinline__ int slot(const int* __restrict__, int a, int, int) const {
        return reinterpret_cast<const int*>(sslot + (a >> 2) * TILE + i)[a & 3];
    }
};

// Inputs of a tile that did not fit a window: connectivity staged in the
// window region, node rows gathered from global memory.
template <class Real, int TILE>
struct WinGlobalSrc {
    using Node = typename RT<Real>::Node;
    const int4* sslot;
    const int4* sconn;                     // [NPE/4][TILE] node ids
    const typename RT<Real>::Plane* srec;
    const Real* stail;
    int i;
    __device__ __forceinline__ int4 conn(int p) const { return sconn[p * TILE + i]; }
    __device__ __forceinline__ Node node(int, const Node* __restrict__ u, int n) const { return RT<Real>::load_node(u + n); }
    __device__ __forceinline__ Node coord(const ElemArgs<Real>& a, int n) const { return RT<Real>::load_node(a.X + n); }
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const { return srec[p * TILE + i]; }
    __device__ __forceinline__ Real tail(int t) const { return stail[t * TILE + i]; }
    template <int N, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[N]) const {
#pragma unroll
        for (int a = 0; a < N; ++a) rk[a] = 0;
    }
    __device__ __forceinline__ int slot(const int* __restrict__, int a, int, int) const {
        return reinterpret_cast<const int*>(sslot + (a >> 2) * TILE + i)[a & 3];
    }
};

// Persistent blocks over tiles [e0, e1) (e0 on a tile boundary), tile `it` of
// a block in stage it % STAGES: the producer warp (warp 4) reads the tile's
// descriptor, lane 0 posts the stage's byte count and copies the per-element
// streams, lanes r < nruns copy run r of the window; the compute warps run
// the element body on the stage and release it.
template <class Real, int KIND, int MODEL, int FORM, int STAGES>
__global__ void __launch_bounds__(kPipeThreads, (kPipeMinBlocks<Real, KIND, MODEL, FORM>))
    k_element_win(const ElemArgs<Real> A, long long e0, long long e1) {
    using WS = WinShape<Real, KIND, MODEL, FORM>;
    using Plane = typename RT<Real>::Plane;
    using Node = typename RT<Real>::Node;
    static_assert(STAGES >= 2, "pipeline needs at least two stages");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + STAGES * WS::kStageBytes);
    unsigned long long* empty = full + STAGES;
    const int tid = threadIdx.x;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kPipeTile / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (__ldcg(&A.ctrl->halted)) return;
    const long long ntiles = (e1 - e0 + kPipeTile - 1) / kPipeTile;
    const long long G = gridDim.x;
    const long long nmine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    const int phase = int(__ldcg(&A.ctrl->step) % 3);
    const Node* u = A.u_override ? A.u_override : pick3(phase, A.u[0], A.u[1], A.u[2]);

    if (tid >= kPipeTile) {  // producer warp
        const int lane = tid - kPipeTile;
        const unsigned long long pol = l2_evict_first_policy();
        unsigned long long wpol;  // (evict_last measured no better: profiles/r02)
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(wpol));
        // Descriptors are read kWinAhead tiles ahead (registers), so their
        // HBM latency overlaps the empty-barrier waits instead of delaying
        // the tile's copies. Every lane reads the run count and window
        // length, lane r < kWinRuns its run's first node and window offsets
        // (no shuffles: the producer's issue slots are the scarce resource).
        constexpr int kWinAhead = 2;
        struct Desc {
            int nruns, total, rstart, roff, rnext;
        };
        auto desc_of = [&](long long it) {
            Desc d{0, 0, 0, 0, 0};
            if (it < nmine) {
                const int* p = A.wdesc + ((e0 + (blockIdx.x + it * G) * kPipeTile) / kPipeTile) * kWinDesc;
                d.nruns = __ldg(p);
                d.total = __ldg(p + 1);
                if (lane < kWinRuns) {
                    d.rstart = __ldg(p + 2 + 2 * lane);
                    d.roff = __ldg(p + 3 + 2 * lane);
                    d.rnext = lane + 1 < kWinRuns ? __ldg(p + 5 + 2 * lane) : 0;
                }
            }
            return d;
        };
        Desc dq[kWinAhead];
#pragma unroll
        for (int k = 0; k < kWinAhead; ++k) dq[k] = desc_of(k);
        for (long long it = 0; it < nmine; ++it) {
            const int s = int(it % STAGES);
            const Desc dv = dq[0];
#pragma unroll
            for (int k = 0; k + 1 < kWinAhead; ++k) dq[k] = dq[k + 1];
            dq[kWinAhead - 1] = desc_of(it + kWinAhead);
            // all lanes wait (a converged warp: no collective emulation below)
            if (it >= STAGES) mbar_wait(empty + s, unsigned((it / STAGES - 1) & 1));
            const long long eb = e0 + (blockIdx.x + it * G) * kPipeTile;
            const unsigned n = unsigned(min((long long)kPipeTile, e1 - eb));
            const int nruns = dv.nruns, total = dv.total, rstart = dv.rstart, roff = dv.roff, rnext = dv.rnext;
            unsigned char* st = smem + s * WS::kStageBytes;
            if (lane == 0) {
                DJG_ASSERT(nruns >= 0 && nruns <= kWinRuns && total >= 0 && total <= WS::CAP);
                const unsigned ibytes = (n * WS::NPE * WS::LB + 15u) & ~15u;  // index array padded by 16 bytes
                const unsigned tbytes = (n * unsigned(sizeof(Real)) + 15u) & ~15u;
                const unsigned wbytes = nruns > 0 ? unsigned(total) * unsigned(sizeof(Node)) * WS::NX : n * 16u * WS::NCP;
                *reinterpret_cast<int*>(st + WS::kModeOff) = nruns;
                mbar_expect_tx(full + s, n * 16u * (WS::NCP + WS::NRP) + ibytes + tbytes * WS::NTAIL + wbytes);
#pragma unroll
                for (int p = 0; p < WS::NCP; ++p)
                    bulk_load(st + WS::kSlotOff + p * kPipeTile * 16, A.slot + (long long)p * A.E + eb, n * 16u,
                              full + s, pol);
                bulk_load(st + WS::kIdxOff, static_cast<const unsigned char*>(A.widx) + eb * WS::NPE * WS::LB, ibytes,
                          full + s, pol);
#pragma unroll
                for (int p = 0; p < WS::NRP; ++p)
                    bulk_load(st + WS::kRecOff + p * kPipeTile * 16, A.c + (long long)p * A.E + eb, n * 16u, full + s,
                              pol);
#pragma unroll
                for (int t = 0; t < WS::NTAIL; ++t)
                    bulk_load(st + WS::kTailOff + t * kPipeTile * int(sizeof(Real)), A.ctail + t * A.tail_stride + eb,
                              tbytes, full + s, pol);
                if (nruns == 0) {
#pragma unroll
                    for (int p = 0; p < WS::NCP; ++p)
                        bulk_load(st + WS::kWinOff + p * kPipeTile * 16, A.conn + (long long)p * A.E + eb, n * 16u,
                                  full + s, pol);
                }
            }
            __syncwarp();
            if (lane < nruns) {
                const int wend = lane + 1 < nruns ? rnext : total;
                const unsigned bytes = unsigned(wend - roff) * unsigned(sizeof(Node));
                DJG_ASSERT(roff >= 0 && wend <= total && rstart >= 0 && rstart + (wend - roff) <= A.N);
                // node rows are re-read by neighbouring tiles (other cell rows
                // and planes): kept in L2 with the window policy
                bulk_load(st + WS::kWinOff + roff * int(sizeof(Node)), u + rstart, bytes, full + s, wpol);
                if constexpr (WS::NX == 2)
                    bulk_load(st + WS::kWinOff + (WS::CAP + roff) * int(sizeof(Node)), A.X + rstart, bytes, full + s,
                              wpol);
            }
        }
        return;
    }

    for (long long it = 0; it < nmine; ++it) {
        const int s = int(it % STAGES);
        mbar_wait(full + s, unsigned((it / STAGES) & 1));
        const long long e = e0 + (blockIdx.x + it * G) * kPipeTile + tid;
        const unsigned char* st = smem + s * WS::kStageBytes;
        const int mode = *reinterpret_cast<const int*>(st + WS::kModeOff);
        if (e < e1) {
            const int4* sslot = reinterpret_cast<const int4*>(st + WS::kSlotOff);
            const Plane* srec = reinterpret_cast<const Plane*>(st + WS::kRecOff);
            const Real* stail = reinterpret_cast<const Real*>(st + WS::kTailOff);
            if (mode > 0) {
                const Node* wu = reinterpret_cast<const Node*>(st + WS::kWinOff);
                const WinSrc<Real, kPipeTile, WS::NPE, WS::LB> src{sslot, st + WS::kIdxOff, srec, stail, wu,
                                                                     wu + WS::CAP, tid};
                if constexpr (FORM == 2) element_body_tled<Real, KIND, MODEL, 1>(A, e, u, src);
                else element_body<Real, KIND, MODEL, 1, FORM == 1>(A, e, u, src);
            } else {
                const WinGlobalSrc<Real, kPipeTile> src{sslot, reinterpret_cast<const int4*>(st + WS::kWinOff), srec,
                                                        stail, tid};
                if constexpr (FORM == 2) element_body_tled<Real, KIND, MODEL, 1>(A, e, u, src);
                else element_body<Real, KIND, MODEL, 1, FORM == 1>(A, e, u, src);
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(empty + s);
    }
}

// Slot position of every element-node (slice_base[n/32] + 32 rank + n%32),
// in the connectivity's int4 plane layout, for the windowed element kernel.
template <int RB>
__global__ void k_slot_planes(const int4* __restrict__ conn, const void* __restrict__ rank,
                              const int* __restrict__ slice_base, long long E, int npe, int4* __restrict__ out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const unsigned char* r = static_cast<const unsigned char*>(rank) + e * npe * RB;
    for (int p = 0; p < npe / 4; ++p) {
        const int4 q = conn[(long long)p * E + e];
        const int n[4] = {q.x, q.y, q.z, q.w};
        int v[4];
        for (int k = 0; k < 4; ++k) {
            const int a = 4 * p + k;
            const int rk = RB == 1 ? int(r[a]) : int(r[2 * a] | (r[2 * a + 1] << 8));
            v[k] = slice_base[n[k] >> 5] + 32 * rk + (n[k] & 31);
        }
        out[(long long)p * E + e] = make_int4(v[0], v[1], v[2], v[3]);
    }
}

// TledModel::build on the device (tled_force.hpp:167-195).
template <class Real, int KIND>
__global__ void k_precompute_tled(const ElemArgs<Real> A, typename RT<Real>::Plane* planes, unsigned long long* bad) {
    using T = RT<Real>;
    using TL = TledLayout<KIND>;
    constexpr int NPE = TL::NPE;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= A.E) return;
    int nid[NPE];
#pragma unroll
    for (int p = 0; p < NPE / 4; ++p) {
        const int4 q = A.conn[(long long)p * A.E + e];
        nid[4 * p + 0] = q.x; nid[4 * p + 1] = q.y; nid[4 * p + 2] = q.z; nid[4 * p + 3] = q.w;
    }
    Real x[8][3];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        if (a < NPE) {
            const typename T::Node v = T::load_node(A.X + nid[a]);
            x[a][0] = v.x; x[a][1] = v.y; x[a][2] = v.z;
        } else {
            x[a][0] = x[a][1] = x[a][2] = Real(0);
        }
    }
    Real J[3][3], Ji[3][3], det;
    if (!em::jacobian0(KIND, x, J, Ji, det)) {
        atomicMin(bad, (unsigned long long)e);
        return;
    }
    constexpr int NR = (TL::count + T::kPlane - 1) / T::kPlane * T::kPlane;
    Real c[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) c[k] = Real(0);
    em::tled_b0(KIND, Ji, c);
    const Real v0 = em::volume0(KIND, det);
    c[TL::V0] = v0;
    if constexpr (KIND == 1) {
        Real gamma[4][8];
        em::hourglass_vectors(x, Ji, gamma);
        c[TL::khg] = A.mat.chk * ref_cbrt(v0);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int a = 0; a < 8; ++a) c[TL::gamma + 8 * m + a] = gamma[m][a];
    }
#pragma unroll
    for (int p = 0; p < NR / T::kPlane; ++p) {
        Real* dst = reinterpret_cast<Real*>(planes + (long long)p * A.E + e);
#pragma unroll
        for (int k = 0; k < T::kPlane; ++k) dst[k] = c[p * T::kPlane + k];
    }
}

// ------------------------------------------------------------------ K2+K3

// Sums node n's element rows in ascending element order from +0
// (gather_nodal_forces, djtled_force.hpp:116-134). Slot k of the node sits at
// ef[p0 + 32 k]: lane i of a slice reads consecutive 16-byte rows.
#ifndef DJG_GATHER_BATCH
#define DJG_GATHER_BATCH 12
#endif
#ifndef DJG_GATHER_BATCH64
#define DJG_GATHER_BATCH64 6
#endif
template <class Real>
__device__ __forceinline__ void gather_row(const typename RT<Real>::Node* __restrict__ p, int len, Real& sx, Real& sy,
                                           Real& sz) {
    using T = RT<Real>;
    sx = Real(0); sy = Real(0); sz = Real(0);
    int k = 0;
    // Batches of rows loaded together (more loads in flight per thread than
    // the compiler's own pipelining), then folded in order: 12 f32 rows
    // (cfg5 k_node 561 -> 553 us; 16 and 24 no better), 6 f64 rows (cfg5
    // 1071 -> 1057 us; 12 no better).
    constexpr int B = sizeof(Real) == 4 ? DJG_GATHER_BATCH : DJG_GATHER_BATCH64;
    if constexpr (B > 0) {
        for (; k + B <= len; k += B) {
            typename T::Node v[B > 0 ? B : 1];
#pragma unroll
            for (int j = 0; j < B; ++j) v[j] = T::load_stream(p + 32 * (k + j));
#pragma unroll
            for (int j = 0; j < B; ++j) { sx += v[j].x; sy += v[j].y; sz += v[j].z; }
        }
    }
    for (; k < len; ++k) {
        const typename T::Node v = T::load_stream(p + 32 * k);
        sx += v.x; sy += v.y; sz += v.z;
    }
}


// Per-DOF central-difference update (advance_step, solver.hpp:112-141).
template <class Real>
__device__ __forceinline__ Real dof_update(int kind, bool massless, Real c1, Real r, Real f, Real uc, Real up,
                                           Real c2, Real c3, Real t_next, const Real* target, const Real* t_total,
                                           long long dof, bool& nonfinite) {
    if (kind == 1) return Real(0);
    if (kind == 2) {
        const Real s = t_next / t_total[dof];
        return (s >= Real(1) ? Real(1) : s) * target[dof];
    }
    if (massless) return Real(0);
    const Real v = c1 * (r - f) + c2 * uc + c3 * up;
    if (!isfinite(v)) nonfinite = true;
    return v;
}

// One node: gather + (assemble: write f | step: central difference into
// u_next). Returns true if a non-finite displacement was produced.
template <class Real, bool kAssemble>
__device__ __forceinline__ bool node_body(const NodeArgs<Real>& A, const long long n, long long p0, int len,
                                          long long step) {
    using T = RT<Real>;
    Real fx, fy, fz;
    DJG_ASSERT(p0 >= 0 && len >= 0 && (len == 0 || p0 + 32LL * (len - 1) < A.cap));
    gather_row<Real>(A.ef + p0, len, fx, fy, fz);
    if constexpr (kAssemble) {
        A.f_out[3 * n + 0] = fx;
        A.f_out[3 * n + 1] = fy;
        A.f_out[3 * n + 2] = fz;
        return false;
    } else {
        const int ph = int(step % 3);
        const typename T::Node uc = T::load_node(pick3(ph, A.u[0], A.u[1], A.u[2]) + n);
        const typename T::Node up = T::load_node(pick3(ph, A.u[2], A.u[0], A.u[1]) + n);
        typename T::Node* unxt = pick3(ph, A.u[1], A.u[2], A.u[0]);
        typename T::Node r;
        if (A.r_ext) r = T::load_node(A.r_ext + n);
        else { r.x = Real(0); r.y = Real(0); r.z = Real(0); }
        const int code = A.code[n];
        const bool massless = (code >> 6) & 1;
        const Real c1 = A.c1[n];
        const Real t_next = A.dt * Real(step + 1);
        bool nf = false;
        const Real vx = dof_update<Real>(code & 3, massless, c1, r.x, fx, uc.x, up.x, A.c2, A.c3, t_next,
                                         A.target, A.t_total, 3 * n + 0, nf);
        const Real vy = dof_update<Real>((code >> 2) & 3, massless, c1, r.y, fy, uc.y, up.y, A.c2, A.c3, t_next,
                                         A.target, A.t_total, 3 * n + 1, nf);
        const Real vz = dof_update<Real>((code >> 4) & 3, massless, c1, r.z, fz, uc.z, up.z, A.c2, A.c3, t_next,
                                         A.target, A.t_total, 3 * n + 2, nf);
        T::store_node(unxt + n, vx, vy, vz);
        return nf;
    }
}

// Closes a step (advance_step's tail, solver.hpp:143-152): called by the last
// CTA to finish, after every other CTA's writes are visible.
template <bool kAssemble>
__device__ __forceinline__ void close_step(Ctrl* ctrl, long long step, int policy) {
    __threadfence();
    const unsigned long long cnt = atomicAdd(&ctrl->inv_count, 0ull);
    const unsigned long long first = atomicAdd(&ctrl->first_inv, 0ull);
    if (kAssemble) {
        ctrl->asm_first = (first != kNone && policy == 0) ? first : kNone;
        ctrl->asm_count = cnt;
    } else {
        const int div = atomicOr(&ctrl->diverged, 0);
        if (!ctrl->multipart) {
            ctrl->total_inv += cnt;
            if (cnt > 0) ctrl->inv_steps += 1;
        }
        ctrl->step_inv = cnt;
        if (first != kNone && policy == 0) {
            ctrl->halted = 4;  // DJG_E_INVERSION: state stays at the last good step
            ctrl->halt_first_inv = (long long)first;
            ctrl->fail_step = step + 1;
        } else if (div) {
            ctrl->halted = 5;  // DJG_E_DIVERGENCE
            ctrl->fail_step = step + 1;
        } else {
            ctrl->step = step + 1;
        }
    }
    ctrl->inv_count = 0;
    ctrl->first_inv = kNone;
    ctrl->diverged = 0;
}

// Whole-mesh gather + update (the default single-slab step): one thread per
// node, the last block to finish closes the step. Written out in full rather
// than through node_body/close_step: this form compiles to 38 registers
// (6 blocks/SM) instead of 44, which the latency-bound gather needs.
template <class Real, bool kAssemble>
__global__ void __launch_bounds__(256) k_node(const NodeArgs<Real> A) {
    using T = RT<Real>;
    Ctrl* ctrl = A.ctrl;
    if (*(volatile const int*)&ctrl->halted && !kAssemble) return;
    __shared__ int s_nonfinite;
    if (threadIdx.x == 0) s_nonfinite = 0;
    __syncthreads();
    const long long step = ctrl->step;
    const bool inverted = ctrl->first_inv != kNone;
    const bool skip = inverted && A.policy == 0;  // Abort: no gather, no update (djtled_force.hpp:202-208)
    // Grid-stride over nodes: the launch may size the grid to the resident
    // blocks (one barrier + completion count per block, no tail wave).
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < A.N && !skip;
         n += (long long)gridDim.x * blockDim.x) {
        Real fx, fy, fz;
        const long long p0 = (long long)slice_base_of(A.slice_base, A.slice_w, n) + (n & 31);
        DJG_ASSERT(A.row_len[n] == 0 || p0 + 32LL * (A.row_len[n] - 1) < A.cap);
        gather_row<Real>(A.ef + p0, A.row_len[n], fx, fy, fz);
        if constexpr (kAssemble) {
            A.f_out[3 * n + 0] = fx;
            A.f_out[3 * n + 1] = fy;
            A.f_out[3 * n + 2] = fz;
        } else {
            const int ph = int(step % 3);
            const typename T::Node* ucur = ph == 0 ? A.u[0] : (ph == 1 ? A.u[1] : A.u[2]);
            const typename T::Node* uprv = ph == 0 ? A.u[2] : (ph == 1 ? A.u[0] : A.u[1]);
            typename T::Node* unxt = ph == 0 ? A.u[1] : (ph == 1 ? A.u[2] : A.u[0]);
            const typename T::Node uc = T::load_node(ucur + n);
            const typename T::Node up = T::load_node(uprv + n);
            typename T::Node r;
            if (A.r_ext) r = T::load_node(A.r_ext + n);
            else { r.x = Real(0); r.y = Real(0); r.z = Real(0); }
            const int code = A.code[n];
            const bool massless = (code >> 6) & 1;
            const Real c1 = A.c1[n];
            const Real t_next = A.dt * Real(step + 1);
            bool nf = false;
            const Real vx = dof_update<Real>(code & 3, massless, c1, r.x, fx, uc.x, up.x, A.c2, A.c3, t_next,
                                             A.target, A.t_total, 3 * n + 0, nf);
            const Real vy = dof_update<Real>((code >> 2) & 3, massless, c1, r.y, fy, uc.y, up.y, A.c2, A.c3, t_next,
                                             A.target, A.t_total, 3 * n + 1, nf);
            const Real vz = dof_update<Real>((code >> 4) & 3, massless, c1, r.z, fz, uc.z, up.z, A.c2, A.c3, t_next,
                                             A.target, A.t_total, 3 * n + 2, nf);
            T::store_node(unxt + n, vx, vy, vz);
            if (nf) s_nonfinite = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (s_nonfinite) atomicOr(&ctrl->diverged, 1);
    __threadfence();
    const unsigned int done = atomicAdd(&ctrl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    // Last block: close the step (advance_step's tail, solver.hpp:143-152).
    __threadfence();
    const unsigned long long cnt = atomicAdd(&ctrl->inv_count, 0ull);
    const unsigned long long first = atomicAdd(&ctrl->first_inv, 0ull);
    if (kAssemble) {
        ctrl->asm_first = (first != kNone && A.policy == 0) ? first : kNone;
        ctrl->asm_count = cnt;
    } else {
        const int div = atomicOr(&ctrl->diverged, 0);
        if (!ctrl->multipart) {
            ctrl->total_inv += cnt;
            if (cnt > 0) ctrl->inv_steps += 1;
        }
        ctrl->step_inv = cnt;
        if (skip) {
            ctrl->halted = 4;  // DJG_E_INVERSION
            ctrl->halt_first_inv = (long long)first;
            ctrl->fail_step = step + 1;
        } else if (div) {
            ctrl->halted = 5;  // DJG_E_DIVERGENCE
            ctrl->fail_step = step + 1;
        } else {
            ctrl->step = step + 1;
        }
    }
    ctrl->inv_count = 0;
    ctrl->first_inv = kNone;
    ctrl->diverged = 0;
    __threadfence();
    ctrl->blocks_done = 0;
}

// ------------------------------------------------------------------ fused box step
//
// One kernel per explicit step for a generated box of T4 cells
// (generate_box: lexicographic nodes, six Kuhn tets per cell in cell order),
// with no force slots in HBM. Block = a column tile of BX x BY owned nodes
// and a segment of BZ node layers; it streams cell layer by cell layer:
//   1. the node rows (u, X) of the two node layers a cell layer spans are in
//      a 3-layer shared ring (the next layer's rows go in with cp.async while
//      the current one is computed);
//   2. every tet of the cell layer that touches the tile's nodes -- the
//      tile's (BX+1) x (BY+1) cell footprint, ~10 % of them also computed by a
//      neighbouring tile -- runs element_body with its four rows written to
//      shared memory instead of HBM;
//   3. each owned node folds the rows of the tets around it in ascending
//      element id from +0 (the four cells below it in id order, each cell's
//      tets in order, then the four cells above: the order of its CSR row),
//      carrying the partial sum of the layer below in a register, then runs
//      the central-difference update (dof_update) and stores u_next.
// The last block closes the step (close_step). Rows, sums and update are
// those of k_element + k_node: bit-identical; what disappears is the 16-byte
// slot row per element-node written and read back through HBM (6.4 GB per
// cfg5 step). Inversions are counted by the tile that owns the cell (the
// one owning node (ci+1, cj+1)) in the segment that owns its layer.
#ifndef DJG_BOX_UNROLL_T
#define DJG_BOX_UNROLL_T 6  // tets of a cell per unrolled iteration (lattice table, cfg5: 1: 1.28 ms, 2: 1.27, 3: 1.28, 6: 1.22)
#endif
constexpr int kBoxUnrollT = DJG_BOX_UNROLL_T;
#ifndef DJG_BOX_MINB
#define DJG_BOX_MINB 2
#endif
struct BoxArgs {
    int nx, ny, nz;   // cells per axis
    int tiles_x, tiles_y;
    // node layers [lay0, lay1) updated by this launch (the whole box: 0,
    // nz + 1); close: the launch's last block closes the step
    int lay0, lay1, close;
    // coordinate lattice (k_box_step<..., LAT = true>): record fields 9.. of
    // tet t of a cell with axis classes (cx, cy, cz) are lat[((cz * lncy + cy)
    // * lncx + cx) * 6 + t] (plane-padded); its J0 is made of the classes'
    // interval lengths ld[cx], ld[lncx + cy], ld[lncx + lncy + cz]; lcls =
    // the class of every cell index along x, then y, then z
    const void* lat;   // RT<Real>::Plane[]
    const int* lcls;
    const void* ld;    // Real[]
    int lncx, lncy, lncz, _pad;
};

// H8 corner signs (element.hpp:17-20) as a compile-time function for device code.
__device__ __forceinline__ constexpr int kBoxCornerSignDev(int a, int i) {
    constexpr int s[8][3] = {{-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
                             {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1}};
    return s[a][i];
}

// Corner code (dx + 2 dy + 4 dz) of local node a of Kuhn tet t
// (generate_box's axis orders with the odd-permutation swap, mesh.hpp:228-258).
__device__ __constant__ signed char kTetCorner[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7}, {0, 3, 2, 7},
                                                        {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 6, 4, 7}};

// Stage offset (dy * SX + dx, bit 7 = dz) of local node a of Kuhn tet t,
// four per tet packed in a word.
template <int SX>
__device__ __forceinline__ unsigned tet_stage_offsets(int t) {
    constexpr int C[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 6, 4, 7}};
    static_assert(SX + 1 < 128, "stage row too long for the packed offsets");
    auto pack = [](int t2) {
        unsigned w = 0;
        for (int a = 0; a < 4; ++a) {
            const int cr = C[t2][a];
            w |= unsigned(((cr >> 1) & 1) * SX + (cr & 1) + ((cr >> 2) << 7)) << (8 * a);
        }
        return w;
    };
    switch (t) {
        case 0: return pack(0);
        case 1: return pack(1);
        case 2: return pack(2);
        case 3: return pack(3);
        case 4: return pack(4);
        default: return pack(5);
    }
}

// J0 of Kuhn tet t on a lattice cell with interval lengths d: node 0 is
// corner 0, so row i (node i + 1 at corner cr) is d_j where cr has bit j,
// else (0 + -x) + x = +0 -- t4_jacobian0's values (k_lattice_verify checks
// them on every tet).
template <class Real>
__device__ __forceinline__ void lattice_j0(int t, const Real (&d)[3], Real* c) {
    constexpr int C[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 6, 4, 7}};
    int cr[3];
    switch (t) {
        case 0: cr[0] = C[0][1]; cr[1] = C[0][2]; break;
        case 1: cr[0] = C[1][1]; cr[1] = C[1][2]; break;
        case 2: cr[0] = C[2][1]; cr[1] = C[2][2]; break;
        case 3: cr[0] = C[3][1]; cr[1] = C[3][2]; break;
        case 4: cr[0] = C[4][1]; cr[1] = C[4][2]; break;
        default: cr[0] = C[5][1]; cr[1] = C[5][2]; break;
    }
    cr[2] = 7;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) c[3 * i + j] = ((cr[i] >> j) & 1) ? d[j] : Real(0);
}

#ifndef DJG_BOX_EDGES
#define DJG_BOX_EDGES 1
#endif

// Corner code of local node a of Kuhn tet t (a compile-time constant once
// the tet loop is unrolled).
__device__ __forceinline__ int box_tet_corner(int t, int a) {
    constexpr int C[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 6, 4, 7}};
    switch (t) {
        case 0: return C[0][a];
        case 1: return C[1][a];
        case 2: return C[2][a];
        case 3: return C[3][a];
        case 4: return C[4][a];
        default: return C[5][a];
    }
}

// The terms of one Jt row that the tets of a lattice cell share: the row E
// of the edge from corner 0 to corner c (J0's d-masked row + u_c - u_0,
// update_jacobian's sums), its g-vector norm, its dot product with the
// diagonal row D (corner 7), and its products with D as the det minors /
// adjugate entries take them (each in element_body's operand order, so
// every value is the one the tet would compute itself).
template <class Real>
struct EdgeKin {
    Real E[3], N, P, m0, m1, m2, n0, n1, n2;
};
template <class Real>
__device__ __forceinline__ EdgeKin<Real> edge_kin(int c, const Real (&d)[3], const typename RT<Real>::Node& uc,
                                                  const typename RT<Real>::Node& u0, const Real (&D)[3]) {
    EdgeKin<Real> k;
    k.E[0] = ((c & 1) ? d[0] : Real(0)) + (uc.x - u0.x);
    k.E[1] = ((c & 2) ? d[1] : Real(0)) + (uc.y - u0.y);
    k.E[2] = ((c & 4) ? d[2] : Real(0)) + (uc.z - u0.z);
    k.N = k.E[0] * k.E[0] + k.E[1] * k.E[1] + k.E[2] * k.E[2];
    k.P = k.E[0] * D[0] + k.E[1] * D[1] + k.E[2] * D[2];
    k.m0 = k.E[1] * D[2] - k.E[2] * D[1];  // as row 1: J11 J22 - J12 J21
    k.m1 = k.E[0] * D[2] - k.E[2] * D[0];  //           J10 J22 - J12 J20 (as row 0: J00 J22 - J02 J20)
    k.m2 = k.E[0] * D[1] - k.E[1] * D[0];  //           J10 J21 - J11 J20
    k.n0 = k.E[2] * D[1] - k.E[1] * D[2];  // as row 0: J02 J21 - J01 J22
    k.n1 = k.E[2] * D[0] - k.E[0] * D[2];  // as row 1: J12 J20 - J10 J22
    k.n2 = k.E[1] * D[0] - k.E[0] * D[1];  // as row 0: J01 J20 - J00 J21
    return k;
}

template <class Real, bool LAT = false, bool ROW0 = false>
struct BoxSrc {
    using Node = typename RT<Real>::Node;
    static constexpr bool kRowSink = true;
    static constexpr bool kLattice = LAT;
    static constexpr bool kCellKin = LAT && !ROW0 && DJG_BOX_EDGES;
    EdgeKin<Real> e0, e1;  // kCellKin: the tet's rows 0 and 1
    Real D[3], ND;         // kCellKin: row 2 (the diagonal) and its norm
    __device__ __forceinline__ void cell_kinematics(Real (&Jt)[3][3], Real (&g)[6], Real (&cof)[3][3], Real& det) const {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            Jt[0][j] = e0.E[j];
            Jt[1][j] = e1.E[j];
            Jt[2][j] = D[j];
        }
        g[0] = e0.N;
        g[1] = e1.N;
        g[2] = ND;
        g[3] = e0.E[0] * e1.E[0] + e0.E[1] * e1.E[1] + e0.E[2] * e1.E[2];
        g[4] = e0.P;
        g[5] = e1.P;
        det = e0.E[0] * e1.m0 - e0.E[1] * e1.m1 + e0.E[2] * e1.m2;
        cof[0][0] = e1.m0;
        cof[0][1] = e0.n0;
        cof[0][2] = e0.E[1] * e1.E[2] - e0.E[2] * e1.E[1];
        cof[1][0] = e1.n1;
        cof[1][1] = e0.m1;
        cof[1][2] = e0.E[2] * e1.E[0] - e0.E[0] * e1.E[2];
        cof[2][0] = e1.m2;
        cof[2][1] = e0.n2;
        cof[2][2] = e0.E[0] * e1.E[1] - e0.E[1] * e1.E[0];
    }
    const typename RT<Real>::Plane* rc;  // TLED: the record planes (A.c) when not on the lattice
    long long E, e;                      // TLED: plane stride, this tet's element id
    const Node* su;    // stage u (all ring slots)
    const Node* sx;    // stage X (LAT: unused)
    const typename RT<Real>::Plane* lrec;  // LAT: this tet's record (DJ: fields 9..; TLED: all)
    Real d[3];           // LAT: the cell's interval lengths
    int t;               // LAT: the tet (a compile-time constant once the tet loop is unrolled)
    template <int NREC>
    __device__ __forceinline__ void lattice_record(Real* c) const {
        constexpr int KP = RT<Real>::kPlane;
        lattice_j0(t, d, c);
#pragma unroll
        for (int q = 0; q < (NREC - 9 + KP - 1) / KP; ++q) {
            const typename RT<Real>::Plane v = __ldg(lrec + q);
#pragma unroll
            for (int k = 0; k < KP; ++k)
                if (9 + KP * q + k < NREC) c[9 + KP * q + k] = plane_at(v, k);
        }
    }
    Real* rows;        // [footprint cell][t][a][3]
    int h[4];          // stage indices of the tet's nodes
    int row0;          // first row of this tet
    bool count_inv;
    __device__ __forceinline__ int4 conn(int) const { return make_int4(h[0], h[1], h[2], h[3]); }
    __device__ __forceinline__ Node node(int, const Node* __restrict__, int k) const { return su[k]; }
    __device__ __forceinline__ Node coord(const ElemArgs<Real>&, int k) const { return sx[k]; }
    // TLED (ROW0): the tet's B0 / V0 record -- the lattice table's entry or
    // the precomputed planes in HBM
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const {
        if constexpr (ROW0) {
            if constexpr (LAT) return __ldg(lrec + p);
            else return RT<Real>::load_plane(rc + (long long)p * E + e);
        } else {
            return typename RT<Real>::Plane{};
        }
    }
    __device__ __forceinline__ Real tail(int) const { return Real(0); }
    template <int N, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[N]) const {
#pragma unroll
        for (int a = 0; a < N; ++a) rk[a] = 0;
    }
    int ntet;          // tets per footprint layer: 9 planes [column j][xyz][tet] of K (ROW0: 12, rows 0..3)
    __device__ __forceinline__ int slot(const int* __restrict__, int a, int, int) const { return row0 + a; }
    // T4 rows 1..3 are the columns of K (element_body); row 0 is not kept --
    // the fold recomputes it from the columns with the same operations.
    __device__ __forceinline__ void store(int pos, Real x, Real y, Real z) const {
        const int tet = pos >> 2, a = pos & 3;
        if constexpr (ROW0) {
            rows[(3 * a + 0) * ntet + tet] = x;
            rows[(3 * a + 1) * ntet + tet] = y;
            rows[(3 * a + 2) * ntet + tet] = z;
        } else {
            if (a == 0) return;
            rows[(3 * (a - 1) + 0) * ntet + tet] = x;  // consecutive tets -> consecutive words: no bank conflicts
            rows[(3 * (a - 1) + 1) * ntet + tet] = y;
            rows[(3 * (a - 1) + 2) * ntet + tet] = z;
        }
    }
};

// The Kuhn tets of a cell holding corner C, as (tet, local node) in
// ascending tet order (the inverse of kTetCorner), at compile time.
template <int C, int NCELL, bool ROW0 = false, class Real>
__device__ __forceinline__ void corner_rows(const Real* __restrict__ rows, int ntet, int c, Real& fx, Real& fy,
                                            Real& fz) {
    constexpr int n = (C == 0 || C == 7) ? 6 : 2;
    constexpr int T0[8][6] = {{0, 1, 2, 3, 4, 5}, {0, 1}, {2, 3}, {0, 2}, {4, 5}, {1, 4}, {3, 5}, {0, 1, 2, 3, 4, 5}};
    constexpr int A0[8][6] = {{0, 0, 0, 0, 0, 0}, {1, 2}, {2, 1}, {2, 1}, {1, 2}, {1, 2}, {2, 1}, {3, 3, 3, 3, 3, 3}};
#pragma unroll
    for (int m = 0; m < n; ++m) {
        const int tet = T0[C][m] * NCELL + c, a = A0[C][m];
        if constexpr (ROW0) {  // TLED: all four rows kept
            fx += rows[(3 * a + 0) * ntet + tet];
            fy += rows[(3 * a + 1) * ntet + tet];
            fz += rows[(3 * a + 2) * ntet + tet];
        } else if (a == 0) {  // f0 = -(f1 + f2 + f3), element_body's expression (djtled_force.hpp:73-77)
            const Real* k = rows + tet;
            fx += Real(-1) * ((k[0 * ntet] + k[3 * ntet]) + k[6 * ntet]);
            fy += Real(-1) * ((k[1 * ntet] + k[4 * ntet]) + k[7 * ntet]);
            fz += Real(-1) * ((k[2 * ntet] + k[5 * ntet]) + k[8 * ntet]);
        } else {
            fx += rows[(3 * (a - 1) + 0) * ntet + tet];
            fy += rows[(3 * (a - 1) + 1) * ntet + tet];
            fz += rows[(3 * (a - 1) + 2) * ntet + tet];
        }
    }
}

template <int BX, int BY>
struct BoxShape {
    static constexpr int SX = BX + 2, SY = BY + 2;  // stage nodes per layer (footprint + 1 halo node each side)
    static constexpr int CX = BX + 1, CY = BY + 1;  // footprint cells per layer
    static constexpr int kStageNodes = SX * SY;
    static constexpr size_t kRowFloats = size_t(CX) * CY * 6 * 9;  // K per tet (TLED: 12, rows 0..3)
    // one thread per footprint cell (its six tets in turn: every thread the
    // same work per layer), the first BX * BY of them also one owned node each
    static constexpr int kThreads = (CX * CY + 31) / 32 * 32;
    // the ring holds u, and X unless the records come from the lattice table
    // or the TLED planes
    template <class Real, bool LAT = false, bool TLED = false>
    static constexpr size_t smem_bytes() {
        return (LAT || TLED ? 1 : 2) * 3 * size_t(kStageNodes) * sizeof(typename RT<Real>::Node) +
               kRowFloats / 9 * (TLED ? 12 : 9) * sizeof(Real);
    }
};

// Planes of a T4 record in the lattice table (DJ: fields 9.., I1m pre-multiplied by dI1; TLED: B0 / V0).
template <class Real, int MODEL>
constexpr int kLatPlanes = (Layout<0, MODEL>::count - 9 + RT<Real>::kPlane - 1) / RT<Real>::kPlane;
template <class Real>
constexpr int kTledPlanes = (TledLayout<0>::count + RT<Real>::kPlane - 1) / RT<Real>::kPlane;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
template <class Node>
__device__ __forceinline__ void cp_async_node(Node* dst, const Node* src) {
#pragma unroll
    for (int k = 0; k < int(sizeof(Node) / 16); ++k)
        cp_async16(reinterpret_cast<char*>(dst) + 16 * k, reinterpret_cast<const char*>(src) + 16 * k);
}
#ifndef DJG_BOX_MINB64
#define DJG_BOX_MINB64 1  // f64: 156 KB of shared memory per block
#endif

template <class Real, int MODEL, int BX, int BY, bool LAT, bool TLED = false>
__global__ void __launch_bounds__(BoxShape<BX, BY>::kThreads, sizeof(Real) == 4 ? DJG_BOX_MINB : DJG_BOX_MINB64)
    k_box_step(const ElemArgs<Real> A, const NodeArgs<Real> NA, const BoxArgs B) {
    using T = RT<Real>;
    using Node = typename T::Node;
    using BS = BoxShape<BX, BY>;
    constexpr int NT = BS::kThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    Node* su = reinterpret_cast<Node*>(smem);
    Node* sx = su + 3 * BS::kStageNodes;
    constexpr bool kXRing = !LAT && !TLED;  // coordinates staged (per-tet DJ record rebuild)
    Real* rows = reinterpret_cast<Real*>(su + (kXRing ? 2 : 1) * 3 * BS::kStageNodes);
    constexpr int NQ = TLED ? kTledPlanes<Real> : kLatPlanes<Real, MODEL>;
    using Plane = typename T::Plane;
    const Plane* lat = static_cast<const Plane*>(B.lat);
    const Real* ld = static_cast<const Real*>(B.ld);
    __shared__ int s_nonfinite;
    Ctrl* ctrl = A.ctrl;
    if (*(volatile const int*)&ctrl->halted) return;
    const int tid = threadIdx.x;
    if (tid == 0) s_nonfinite = 0;
    const int nx = B.nx, ny = B.ny, nz = B.nz;
    int i0 = 0, j0 = 0, k0 = 0, k1 = 0;  // the current piece: column tile at (i0, j0), node layers [k0, k1)
    const long long step = ctrl->step;
    const int ph = int(step % 3);
    const Node* ucur = pick3(ph, NA.u[0], NA.u[1], NA.u[2]);
    const Node* uprv = pick3(ph, NA.u[2], NA.u[0], NA.u[1]);
    Node* unxt = pick3(ph, NA.u[1], NA.u[2], NA.u[0]);
    auto gid = [&](int i, int j, int k) { return (long long)i + (long long)(nx + 1) * (j + (long long)(ny + 1) * k); };
    // node layer k into ring slot k % 3 (cp.async; out-of-box rows are left stale and never read)
    auto load_layer = [&](int k) {
        if (k > nz) return;
        const int slot = k % 3;
        for (int q = tid; q < BS::kStageNodes; q += NT) {
            const int gi = i0 - 1 + q % BS::SX, gj = j0 - 1 + q / BS::SX;
            if (gi < 0 || gi > nx || gj < 0 || gj > ny) continue;
            const long long n = gid(gi, gj, k);
            cp_async_node(su + slot * BS::kStageNodes + q, ucur + n);
            if constexpr (kXRing) cp_async_node(sx + slot * BS::kStageNodes + q, A.X + n);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // owned node of this thread (one per column position) and footprint
    // cell (one per thread), relative to the tile
    int oi = 0, oj = 0, cb = 0, mci = 0, mcj = 0;
    bool own = false, hx0 = false, hx1 = false, hy0 = false, hy1 = false, my_cell = false;
    Real px = Real(0), py = Real(0), pz = Real(0);  // partial sum of the node one layer up (cells below it)

    // fold the rows of the cell layer around node (oi, oj): its four cells in
    // id order (the node is their corner 3, 2, 1, 0 at height dz), each
    // cell's tets in order
    constexpr int NCELL = BS::CX * BS::CY, NTET = NCELL * 6;  // rows: tet t of footprint cell c is t * NCELL + c
    auto fold_below = [&](Real& fx, Real& fy, Real& fz) {  // node at the top (dz = 1) of the cells
        if (hy0 && hx0) corner_rows<7, NCELL, TLED>(rows, NTET, cb, fx, fy, fz);
        if (hy0 && hx1) corner_rows<6, NCELL, TLED>(rows, NTET, cb + 1, fx, fy, fz);
        if (hy1 && hx0) corner_rows<5, NCELL, TLED>(rows, NTET, cb + BS::CX, fx, fy, fz);
        if (hy1 && hx1) corner_rows<4, NCELL, TLED>(rows, NTET, cb + BS::CX + 1, fx, fy, fz);
    };
    auto fold_above = [&](Real& fx, Real& fy, Real& fz) {  // node at the bottom (dz = 0)
        if (hy0 && hx0) corner_rows<3, NCELL, TLED>(rows, NTET, cb, fx, fy, fz);
        if (hy0 && hx1) corner_rows<2, NCELL, TLED>(rows, NTET, cb + 1, fx, fy, fz);
        if (hy1 && hx0) corner_rows<1, NCELL, TLED>(rows, NTET, cb + BS::CX, fx, fy, fz);
        if (hy1 && hx1) corner_rows<0, NCELL, TLED>(rows, NTET, cb + BS::CX + 1, fx, fy, fz);
    };
    // the update's per-node operands, loaded a cell layer ahead of their use
    // (their HBM latency then overlaps the layer's tets, not the barrier)
    struct NodeOps {
        typename T::Node up;
        int code;
        Real c1;
    };
    auto node_ops = [&](int k) {
        const long long n = gid(oi, oj, k);
        return NodeOps{T::load_node(uprv + n), int(NA.code[n]), NA.c1[n]};
    };
    auto update = [&](int k, const NodeOps& ops, Real fx, Real fy, Real fz) {
        const long long n = gid(oi, oj, k);
        const typename T::Node uc = su[(k % 3) * BS::kStageNodes + (oj - j0 + 1) * BS::SX + (oi - i0 + 1)];
        const typename T::Node up = ops.up;
        typename T::Node r;
        if (NA.r_ext) r = T::load_node(NA.r_ext + n);
        else { r.x = Real(0); r.y = Real(0); r.z = Real(0); }
        const int code = ops.code;
        const bool massless = (code >> 6) & 1;
        const Real c1 = ops.c1;
        const Real t_next = NA.dt * Real(step + 1);
        bool nf = false;
        const Real vx = dof_update<Real>(code & 3, massless, c1, r.x, fx, uc.x, up.x, NA.c2, NA.c3, t_next, NA.target,
                                         NA.t_total, 3 * n + 0, nf);
        const Real vy = dof_update<Real>((code >> 2) & 3, massless, c1, r.y, fy, uc.y, up.y, NA.c2, NA.c3, t_next,
                                         NA.target, NA.t_total, 3 * n + 1, nf);
        const Real vz = dof_update<Real>((code >> 4) & 3, massless, c1, r.z, fz, uc.z, up.z, NA.c2, NA.c3, t_next,
                                         NA.target, NA.t_total, 3 * n + 2, nf);
        T::store_node(unxt + n, vx, vy, vz);
        if (nf) s_nonfinite = 1;
    };

    const int mcy = tid / BS::CX, mcx = tid - mcy * BS::CX;
    const bool my_count = mcx < BX && mcy < BY;  // the tile owning node (ci + 1, cj + 1) counts its inversions
    const int mbase = mcy * BS::SX + mcx;

    // Persistent blocks: the column-layers (every column tile x every node
    // layer, columns in order) are split evenly over the grid; a block walks
    // its range as one or two column pieces, each starting with one extra
    // cell layer below it (the partial sums of its first node layer).
    const long long L = B.lay1 - B.lay0, W = (long long)B.tiles_x * B.tiles_y * L;
    const long long w_end = W * (blockIdx.x + 1) / gridDim.x;
    for (long long w = W * blockIdx.x / gridDim.x; w < w_end;) {
        const long long col = w / L;
        k0 = B.lay0 + int(w - col * L);
        k1 = int(min((long long)B.lay1, (long long)k0 + (w_end - w)));
        w += k1 - k0;
        i0 = int(col % B.tiles_x) * BX;
        j0 = int(col / B.tiles_x) * BY;
        oi = i0 + tid % BX;
        oj = j0 + tid / BX;
        own = tid < BX * BY && oi <= nx && oj <= ny;
        cb = (oj - j0) * BS::CX + (oi - i0);  // footprint cell (oi - 1, oj - 1)
        hx0 = oi >= 1; hx1 = oi < nx; hy0 = oj >= 1; hy1 = oj < ny;
        mci = i0 - 1 + mcx;
        mcj = j0 - 1 + mcy;
        my_cell = tid < NCELL && mci >= 0 && mci < nx && mcj >= 0 && mcj < ny;
        int lxy = 0;  // LAT: the cell's (cy * lncx + cx) and x / y interval lengths
        Real ldx = Real(0), ldy = Real(0);
        if constexpr (LAT) {
            if (my_cell) {
                const int cx = __ldg(B.lcls + mci), cy = __ldg(B.lcls + nx + mcj);
                lxy = cy * B.lncx + cx;
                ldx = __ldg(ld + cx);
                ldy = __ldg(ld + B.lncx + cy);
            }
        }
        px = Real(0); py = Real(0); pz = Real(0);
        const int kc0 = max(k0 - 1, 0), kc1 = min(k1 - 1, nz - 1);  // cell layers this piece computes
        load_layer(kc0);
        load_layer(kc0 + 1);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (int kc = kc0; kc <= kc1; ++kc) {
            load_layer(kc + 2);  // ring slot (kc + 2) % 3 held layer kc - 1, released by the last barrier
            // 2. the cell layer's tets around the tile: this thread's cell, its
            // six tets in order (a warp shares t: uniform corner offsets;
            // consecutive cells write consecutive row words)
            NodeOps ops{};
            if (own && kc >= k0) ops = node_ops(kc);
            if (my_cell) {
                const int hb0 = (kc % 3) * BS::kStageNodes + mbase, hb1 = ((kc + 1) % 3) * BS::kStageNodes + mbase;
                const bool count = my_count && kc >= k0;
                const long long ebase = ((long long)mci + (long long)nx * (mcj + (long long)ny * kc)) * 6;
                const Plane* lcell = nullptr;
                Real ldz = Real(0);
                if constexpr (LAT) {
                    const int cz = __ldg(B.lcls + nx + ny + kc);
                    lcell = lat + size_t(cz * B.lncy * B.lncx + lxy) * 6 * NQ;
                    ldz = __ldg(ld + B.lncx + B.lncy + cz);
                }
                // the cell path (kCellKin): tets in the order 0, 1, 4, 5, 3, 2, so
                // that each tet's row 1 is the previous tet's row 0 (the edges
                // to corners 3, 1, 5, 4, 6, 2) and its terms carry over; the
                // diagonal's (corner 7) serve all six
                constexpr bool kCell = BoxSrc<Real, LAT, TLED>::kCellKin;
                static_assert(!kCell || kBoxUnrollT == 6, "the cell path needs the tet loop unrolled");
                constexpr int kOrder[6] = {0, 1, 4, 5, 3, 2};
                typename T::Node cu0{}, cu7{};
                Real Dg[3] = {Real(0), Real(0), Real(0)}, NDg = Real(0);
                EdgeKin<Real> prev{};
                const Real dcell[3] = {ldx, ldy, ldz};
                if constexpr (kCell) {
                    cu0 = su[hb0];
                    cu7 = su[hb1 + BS::SX + 1];
                    Dg[0] = dcell[0] + (cu7.x - cu0.x);
                    Dg[1] = dcell[1] + (cu7.y - cu0.y);
                    Dg[2] = dcell[2] + (cu7.z - cu0.z);
                    NDg = Dg[0] * Dg[0] + Dg[1] * Dg[1] + Dg[2] * Dg[2];
                }
                auto corner_u = [&](int cr) {
                    return su[((cr >> 2) ? hb1 : hb0) + ((cr >> 1) & 1) * BS::SX + (cr & 1)];
                };
    #pragma unroll kBoxUnrollT
                for (int q = 0; q < 6; ++q) {
                    const int t = kCell ? kOrder[q] : q;
                    BoxSrc<Real, LAT, TLED> src;
                    if constexpr (kCell) {
                        const int c1 = box_tet_corner(t, 1), c2 = box_tet_corner(t, 2);
                        src.e1 = q == 0 ? edge_kin<Real>(c2, dcell, corner_u(c2), cu0, Dg) : prev;
                        src.e0 = edge_kin<Real>(c1, dcell, corner_u(c1), cu0, Dg);
                        src.D[0] = Dg[0]; src.D[1] = Dg[1]; src.D[2] = Dg[2];
                        src.ND = NDg;
                        prev = src.e0;
                    }
                    src.rc = A.c;
                    src.E = A.E;
                    src.e = ebase + t;
                    src.su = su;
                    src.sx = sx;
                    src.lrec = LAT ? lcell + t * NQ : nullptr;
                    src.d[0] = ldx; src.d[1] = ldy; src.d[2] = ldz;
                    src.t = t;
                    src.rows = rows;
                    src.ntet = NTET;
                    src.row0 = (t * NCELL + tid) * 4;
                    src.count_inv = count;
                        // the tet's four stage offsets, packed per tet (bit 7: upper layer)
                    const unsigned pk = tet_stage_offsets<BS::SX>(t);
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        const unsigned v = (pk >> (8 * a)) & 0xffu;
                        src.h[a] = ((v & 0x80u) ? hb1 : hb0) + int(v & 0x7fu);
                    }
                    if constexpr (TLED) element_body_tled<Real, 0, MODEL, 1>(A, ebase + t, nullptr, src);
                    else element_body<Real, 0, MODEL, 1, true>(A, ebase + t, nullptr, src);
                }
            }
            __syncthreads();
            // 3. finish node layer kc, start node layer kc + 1
            if (own) {
                if (kc >= k0) {
                    Real fx = px, fy = py, fz = pz;
                    fold_above(fx, fy, fz);
                    update(kc, ops, fx, fy, fz);
                }
                if (kc + 1 < k1) {
                    px = Real(0); py = Real(0); pz = Real(0);
                    fold_below(px, py, pz);
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        }
        // the top node layer has no cells above it
        if (own && k1 - 1 == nz && nz >= k0 && nz > kc1) update(nz, node_ops(nz), px, py, pz);
        __syncthreads();  // (the next piece's loads reuse the ring)
    }
    if (tid != 0) return;
    if (s_nonfinite) atomicOr(&ctrl->diverged, 1);
    __threadfence();
    const unsigned int done = atomicAdd(&ctrl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    if (B.close) close_step<false>(ctrl, step, NA.policy);
    __threadfence();
    ctrl->blocks_done = 0;
}

// Lattice table of the fused T4 step: for every axis-class triple, the
// record of each tet of a representative cell (rep[cx], rep[lncx + cy],
// rep[lncx + lncy + cz]: the first cell index of each class), rebuilt by
// element_body's own compact arithmetic.
template <class Node>
__device__ __forceinline__ void box_tet_coords(const Node* __restrict__ X, const BoxArgs& B, int ci, int cj, int ck,
                                               int t, Node (&x)[4]) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int cr = kTetCorner[t][a];
        x[a] = X[(long long)(ci + (cr & 1)) +
                 (long long)(B.nx + 1) * ((cj + ((cr >> 1) & 1)) + (long long)(B.ny + 1) * (ck + (cr >> 2)))];
    }
}

template <class Real, int MODEL>
__global__ void k_lattice_table(const ElemArgs<Real> A, const BoxArgs B, const int* __restrict__ rep,
                                typename RT<Real>::Plane* __restrict__ lat) {
    constexpr int NQ = kLatPlanes<Real, MODEL>, KP = RT<Real>::kPlane;
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= (long long)B.lncx * B.lncy * B.lncz * 6) return;
    const int t = int(q % 6);
    const long long comb = q / 6;
    const int cx = int(comb % B.lncx), cy = int(comb / B.lncx % B.lncy), cz = int(comb / B.lncx / B.lncy);
    typename RT<Real>::Node x[4];
    box_tet_coords(A.X, B, rep[cx], rep[B.lncx + cy], rep[B.lncx + B.lncy + cz], t, x);
    Real c[9 + NQ * KP];
#pragma unroll
    for (int k = 0; k < 9 + NQ * KP; ++k) c[k] = Real(0);
    t4_jacobian0(0, x, c);
    compact_record_tail<Real, 0, MODEL>(A, c);
#pragma unroll
    for (int k = 0; k < 6; ++k) c[17 + k] = A.mat.dI1 * c[17 + k];  // element_body's first s term
    Real* f = reinterpret_cast<Real*>(lat + q * NQ);
#pragma unroll
    for (int k = 0; k < NQ * KP; ++k) f[k] = c[9 + k];
}

// Every tet of the box against its class's table record, bit for bit (+0
// and -0 distinct); `bad` counts the mismatches. The fused step reads the
// table only when there are none: the table is exact by check, not by an
// argument about the coordinates.
template <class Real, int MODEL>
__global__ void k_lattice_verify(const ElemArgs<Real> A, const BoxArgs B, const typename RT<Real>::Plane* __restrict__ lat,
                                 unsigned long long* bad) {
    constexpr int NQ = kLatPlanes<Real, MODEL>, KP = RT<Real>::kPlane, NREC = Layout<0, MODEL>::count;
    const Real* ld = static_cast<const Real*>(B.ld);
    const long long ncell = (long long)B.nx * B.ny * B.nz;
    unsigned long long mism = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ncell * 6;
         e += (long long)gridDim.x * blockDim.x) {
        const int t = int(e % 6);
        const long long cell = e / 6;
        const int ci = int(cell % B.nx), cj = int(cell / B.nx % B.ny), ck = int(cell / B.nx / B.ny);
        typename RT<Real>::Node x[4];
        box_tet_coords(A.X, B, ci, cj, ck, t, x);
        Real c[9 + NQ * KP];
#pragma unroll
        for (int k = 0; k < 9 + NQ * KP; ++k) c[k] = Real(0);
        t4_jacobian0(0, x, c);
        compact_record_tail<Real, 0, MODEL>(A, c);
#pragma unroll
        for (int k = 0; k < 6; ++k) c[17 + k] = A.mat.dI1 * c[17 + k];  // as k_lattice_table
        const int cx = B.lcls[ci], cy = B.lcls[B.nx + cj], cz = B.lcls[B.nx + B.ny + ck];
        const long long comb = ((long long)cz * B.lncy + cy) * B.lncx + cx;
        const Real* want = reinterpret_cast<const Real*>(lat + (comb * 6 + t) * NQ);
        Real j0[9];
        const Real d[3] = {ld[cx], ld[B.lncx + cy], ld[B.lncx + B.lncy + cz]};
        lattice_j0(t, d, j0);
        bool same = true;
#pragma unroll
        for (int k = 0; k < 9; ++k) same = same && same_bits(c[k], j0[k]);
#pragma unroll
        for (int k = 9; k < NREC; ++k) same = same && same_bits(c[k], want[k - 9]);
        mism += same ? 0 : 1;
    }
    if (mism) atomicAdd(bad, mism);
}

// TLED on a lattice: the B0 / V0 record of tet t of a representative cell
// per class triple, copied from the precomputed planes (A.c); then every
// tet's planes against its class's entry, bit for bit.
template <class Real>
__global__ void k_lattice_table_rec(const ElemArgs<Real> A, const BoxArgs B, const int* __restrict__ rep,
                                    typename RT<Real>::Plane* __restrict__ lat) {
    constexpr int NQ = kTledPlanes<Real>;
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= (long long)B.lncx * B.lncy * B.lncz * 6) return;
    const int t = int(q % 6);
    const long long comb = q / 6;
    const int cx = int(comb % B.lncx), cy = int(comb / B.lncx % B.lncy), cz = int(comb / B.lncx / B.lncy);
    const long long e =
        (rep[cx] + (long long)B.nx * (rep[B.lncx + cy] + (long long)B.ny * rep[B.lncx + B.lncy + cz])) * 6 + t;
#pragma unroll
    for (int p = 0; p < NQ; ++p) lat[q * NQ + p] = A.c[(long long)p * A.E + e];
}

template <class Real>
__global__ void k_lattice_verify_rec(const ElemArgs<Real> A, const BoxArgs B,
                                     const typename RT<Real>::Plane* __restrict__ lat, unsigned long long* bad) {
    constexpr int NQ = kTledPlanes<Real>, KP = RT<Real>::kPlane, NREC = TledLayout<0>::count;
    const long long ncell = (long long)B.nx * B.ny * B.nz;
    unsigned long long mism = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ncell * 6;
         e += (long long)gridDim.x * blockDim.x) {
        const int t = int(e % 6);
        const long long cell = e / 6;
        const int ci = int(cell % B.nx), cj = int(cell / B.nx % B.ny), ck = int(cell / B.nx / B.ny);
        const long long comb =
            ((long long)B.lcls[B.nx + B.ny + ck] * B.lncy + B.lcls[B.nx + cj]) * B.lncx + B.lcls[ci];
        bool same = true;
#pragma unroll
        for (int p = 0; p < NQ; ++p) {
            const typename RT<Real>::Plane g = A.c[(long long)p * A.E + e], w = lat[(comb * 6 + t) * NQ + p];
#pragma unroll
            for (int k = 0; k < KP; ++k)
                if (KP * p + k < NREC) same = same && same_bits(plane_at(g, k), plane_at(w, k));
        }
        mism += same ? 0 : 1;
    }
    if (mism) atomicAdd(bad, mism);
}

// The same fused step for a generated box of H8 cells (one hexahedron per
// cell, corners in kBoxCornerSign order): a thread per footprint cell runs
// element_body on its hex -- compact record planes streamed from HBM, node
// rows from the stage -- and keeps its eight rows in shared memory; a node
// folds the row of each of its eight cells (corner order below) in cell-id
// order.
template <class Real>
struct BoxSrcH8 {
    using Node = typename RT<Real>::Node;
    static constexpr bool kRowSink = true;
    const Node* su;
    float* rows;       // planes [a][xyz][cell]
    const typename RT<Real>::Plane* rec;  // this element's record: plane p at rec[p * E]
    long long E;
    int h[8];
    int cell, ncell;
    bool count_inv;
    __device__ __forceinline__ int4 conn(int p) const { return make_int4(h[4 * p], h[4 * p + 1], h[4 * p + 2], h[4 * p + 3]); }
    __device__ __forceinline__ Node node(int, const Node* __restrict__, int k) const { return su[k]; }
    __device__ __forceinline__ Node coord(const ElemArgs<Real>&, int) const { return Node{}; }
    __device__ __forceinline__ typename RT<Real>::Plane plane(int p) const { return RT<Real>::load_plane(rec + p * E); }
    __device__ __forceinline__ Real tail(int) const { return Real(0); }
    template <int N, int RB>
    __device__ __forceinline__ void ranks(int (&rk)[N]) const {
#pragma unroll
        for (int a = 0; a < N; ++a) rk[a] = 0;
    }
    __device__ __forceinline__ int slot(const int* __restrict__, int a, int, int) const { return a; }
    __device__ __forceinline__ void store(int a, Real x, Real y, Real z) const {
        rows[(3 * a + 0) * ncell + cell] = x;
        rows[(3 * a + 1) * ncell + cell] = y;
        rows[(3 * a + 2) * ncell + cell] = z;
    }
};

template <int BX, int BY>
struct BoxShapeH8 {
    static constexpr int SX = BX + 2, SY = BY + 2, CX = BX + 1, CY = BY + 1;
    static constexpr int kStageNodes = SX * SY;
    static constexpr int kThreads = (CX * CY + 31) / 32 * 32;
    template <class Real>
    static constexpr size_t smem_bytes() {
        return 3 * size_t(kStageNodes) * sizeof(typename RT<Real>::Node) + size_t(CX) * CY * 24 * sizeof(float);
    }
};

#ifndef DJG_BOXH8_MINB
#define DJG_BOXH8_MINB 2
#endif
template <class Real, int MODEL, int BX, int BY>
__global__ void __launch_bounds__(BoxShapeH8<BX, BY>::kThreads, DJG_BOXH8_MINB)
    k_box_step_h8(const ElemArgs<Real> A, const NodeArgs<Real> NA, const BoxArgs B) {
    static_assert(sizeof(Real) == 4, "the fused box step keeps float rows");
    using T = RT<Real>;
    using Node = typename T::Node;
    using BS = BoxShapeH8<BX, BY>;
    constexpr int NT = BS::kThreads, NCELL = BS::CX * BS::CY;
    extern __shared__ __align__(128) unsigned char smem[];
    Node* su = reinterpret_cast<Node*>(smem);
    float* rows = reinterpret_cast<float*>(su + 3 * BS::kStageNodes);
    __shared__ int s_nonfinite;
    Ctrl* ctrl = A.ctrl;
    if (*(volatile const int*)&ctrl->halted) return;
    const int tid = threadIdx.x;
    if (tid == 0) s_nonfinite = 0;
    const int nx = B.nx, ny = B.ny, nz = B.nz;
    int i0 = 0, j0 = 0, k0 = 0, k1 = 0;
    const long long step = ctrl->step;
    const int ph = int(step % 3);
    const Node* ucur = pick3(ph, NA.u[0], NA.u[1], NA.u[2]);
    const Node* uprv = pick3(ph, NA.u[2], NA.u[0], NA.u[1]);
    Node* unxt = pick3(ph, NA.u[1], NA.u[2], NA.u[0]);
    auto gid = [&](int i, int j, int k) { return (long long)i + (long long)(nx + 1) * (j + (long long)(ny + 1) * k); };
    auto load_layer = [&](int k) {
        if (k > nz) return;
        const int slot = k % 3;
        for (int q = tid; q < BS::kStageNodes; q += NT) {
            const int gi = i0 - 1 + q % BS::SX, gj = j0 - 1 + q / BS::SX;
            if (gi < 0 || gi > nx || gj < 0 || gj > ny) continue;
            cp_async16(su + slot * BS::kStageNodes + q, ucur + gid(gi, gj, k));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int oi = 0, oj = 0, cb = 0, mci = 0, mcj = 0;
    bool own = false, hx0 = false, hx1 = false, hy0 = false, hy1 = false, my_cell = false;
    Real px = Real(0), py = Real(0), pz = Real(0);
    auto row = [&](int a, int c, Real& fx, Real& fy, Real& fz) {
        fx += rows[(3 * a + 0) * NCELL + c];
        fy += rows[(3 * a + 1) * NCELL + c];
        fz += rows[(3 * a + 2) * NCELL + c];
    };
    // the node is corner (dx, dy, dz) of cell (oi - dx, oj - dy): local node
    // a of kBoxCornerSign: (1,1,dz) -> 2 / 6, (0,1,dz) -> 3 / 7, (1,0,dz) -> 1 / 5, (0,0,dz) -> 0 / 4
    auto fold_below = [&](Real& fx, Real& fy, Real& fz) {
        if (hy0 && hx0) row(6, cb, fx, fy, fz);
        if (hy0 && hx1) row(7, cb + 1, fx, fy, fz);
        if (hy1 && hx0) row(5, cb + BS::CX, fx, fy, fz);
        if (hy1 && hx1) row(4, cb + BS::CX + 1, fx, fy, fz);
    };
    auto fold_above = [&](Real& fx, Real& fy, Real& fz) {
        if (hy0 && hx0) row(2, cb, fx, fy, fz);
        if (hy0 && hx1) row(3, cb + 1, fx, fy, fz);
        if (hy1 && hx0) row(1, cb + BS::CX, fx, fy, fz);
        if (hy1 && hx1) row(0, cb + BS::CX + 1, fx, fy, fz);
    };
    auto update = [&](int k, Real fx, Real fy, Real fz) {
        const long long n = gid(oi, oj, k);
        const typename T::Node uc = su[(k % 3) * BS::kStageNodes + (oj - j0 + 1) * BS::SX + (oi - i0 + 1)];
        const typename T::Node up = T::load_node(uprv + n);
        typename T::Node r;
        if (NA.r_ext) r = T::load_node(NA.r_ext + n);
        else { r.x = Real(0); r.y = Real(0); r.z = Real(0); }
        const int code = NA.code[n];
        const bool massless = (code >> 6) & 1;
        const Real c1 = NA.c1[n];
        const Real t_next = NA.dt * Real(step + 1);
        bool nf = false;
        const Real vx = dof_update<Real>(code & 3, massless, c1, r.x, fx, uc.x, up.x, NA.c2, NA.c3, t_next, NA.target,
                                         NA.t_total, 3 * n + 0, nf);
        const Real vy = dof_update<Real>((code >> 2) & 3, massless, c1, r.y, fy, uc.y, up.y, NA.c2, NA.c3, t_next,
                                         NA.target, NA.t_total, 3 * n + 1, nf);
        const Real vz = dof_update<Real>((code >> 4) & 3, massless, c1, r.z, fz, uc.z, up.z, NA.c2, NA.c3, t_next,
                                         NA.target, NA.t_total, 3 * n + 2, nf);
        T::store_node(unxt + n, vx, vy, vz);
        if (nf) s_nonfinite = 1;
    };
    const int mcy = tid / BS::CX, mcx = tid - mcy * BS::CX;
    const bool my_count = mcx < BX && mcy < BY;
    const int mbase = mcy * BS::SX + mcx;
    const long long L = B.lay1 - B.lay0, W = (long long)B.tiles_x * B.tiles_y * L;
    const long long w_end = W * (blockIdx.x + 1) / gridDim.x;
    for (long long w = W * blockIdx.x / gridDim.x; w < w_end;) {
        const long long col = w / L;
        k0 = B.lay0 + int(w - col * L);
        k1 = int(min((long long)B.lay1, (long long)k0 + (w_end - w)));
        w += k1 - k0;
        i0 = int(col % B.tiles_x) * BX;
        j0 = int(col / B.tiles_x) * BY;
        oi = i0 + tid % BX;
        oj = j0 + tid / BX;
        own = tid < BX * BY && oi <= nx && oj <= ny;
        cb = (oj - j0) * BS::CX + (oi - i0);
        hx0 = oi >= 1; hx1 = oi < nx; hy0 = oj >= 1; hy1 = oj < ny;
        mci = i0 - 1 + mcx;
        mcj = j0 - 1 + mcy;
        my_cell = tid < NCELL && mci >= 0 && mci < nx && mcj >= 0 && mcj < ny;
        px = Real(0); py = Real(0); pz = Real(0);
        const int kc0 = max(k0 - 1, 0), kc1 = min(k1 - 1, nz - 1);
        load_layer(kc0);
        load_layer(kc0 + 1);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (int kc = kc0; kc <= kc1; ++kc) {
            load_layer(kc + 2);
            if (my_cell) {
                const int slot0 = (kc % 3) * BS::kStageNodes, slot1 = ((kc + 1) % 3) * BS::kStageNodes;
                const long long e = (long long)mci + (long long)nx * (mcj + (long long)ny * kc);
                BoxSrcH8<Real> src;
                src.su = su;
                src.rows = rows;
                src.rec = A.c + e;
                src.E = A.E;
                src.cell = tid;
                src.ncell = NCELL;
                src.count_inv = my_count && kc >= k0;
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    const int dx = (kBoxCornerSignDev(a, 0) + 1) / 2, dy = (kBoxCornerSignDev(a, 1) + 1) / 2,
                              dz = (kBoxCornerSignDev(a, 2) + 1) / 2;
                    src.h[a] = (dz ? slot1 : slot0) + mbase + dy * BS::SX + dx;
                }
                element_body<Real, 1, MODEL, 1, true>(A, e, nullptr, src);
            }
            __syncthreads();
            if (own) {
                if (kc >= k0) {
                    Real fx = px, fy = py, fz = pz;
                    fold_above(fx, fy, fz);
                    update(kc, fx, fy, fz);
                }
                if (kc + 1 < k1) {
                    px = Real(0); py = Real(0); pz = Real(0);
                    fold_below(px, py, pz);
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        }
        if (own && k1 - 1 == nz && nz >= k0 && nz > kc1) update(nz, px, py, pz);
        __syncthreads();
    }
    if (tid != 0) return;
    if (s_nonfinite) atomicOr(&ctrl->diverged, 1);
    __threadfence();
    const unsigned int done = atomicAdd(&ctrl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    if (B.close) close_step<false>(ctrl, step, NA.policy);
    __threadfence();
    ctrl->blocks_done = 0;
}

// ------------------------------------------------------------------ slab step

// A step runs as S slabs: k_element over elements [e0, e1), then k_node_slices
// over the 32-node slices whose last element lies in that slab. The slab's
// force rows (~32 MB) are read back while still in L2 and their lines are
// then discarded (discard.global.L2), so the element->node exchange mostly
// never reaches HBM. Kernel boundaries order the two phases; no device-side
// waiting. Each node sums its slots in ascending element order, so the
// result is independent of S (bit-identical to S = 1, the plain two-kernel
// step).
__device__ __forceinline__ void l2_discard(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <class Real, bool kAssemble>
__global__ void __launch_bounds__(256) k_node_slices(const NodeArgs<Real> A, const int* __restrict__ slices,
                                                      int nslices, int discard, int close) {
    Ctrl* ctrl = A.ctrl;
    if (__ldcg(&ctrl->halted) && !kAssemble) return;
    __shared__ int s_nonfinite;
    if (threadIdx.x == 0) s_nonfinite = 0;
    __syncthreads();
    const long long step = __ldcg(&ctrl->step);
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w < nslices) {
        const int sl = slices[w];
        const long long n = 32ll * sl + lane;
        const long long b0 = A.slice_base[sl], b1 = A.slice_base[sl + 1];
        if (n < A.N && node_body<Real, kAssemble>(A, n, b0 + lane, A.row_len[n], step)) s_nonfinite = 1;
        __syncwarp();
        if (discard) {
            // the slice's rows: 32 * width slots, 128-byte aligned
            const char* lo = reinterpret_cast<const char*>(A.ef + b0);
            const char* hi = reinterpret_cast<const char*>(A.ef + b1);
            for (const char* q = lo + 128 * lane; q < hi; q += 128 * 32) l2_discard(q);
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (s_nonfinite) atomicOr(&ctrl->diverged, 1);
    if (!close) return;
    // The last slab's kernel closes the step once all its blocks are done
    // (every earlier slab kernel finished before it, in stream order).
    __threadfence();
    const unsigned int done = atomicAdd(&ctrl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    close_step<kAssemble>(ctrl, step, A.policy);
    __threadfence();
    ctrl->blocks_done = 0;
}

// ------------------------------------------------------------------ halo

// Multi-GPU step: after the local step, owners send the new
// displacement of nodes other parts reference; receivers overwrite their
// ghost copies. Both read the phase from the control block, so they follow
// the device-side buffer rotation.
template <class Real>
__global__ void k_halo_pack(const Ctrl* ctrl, typename RT<Real>::Node* u0, typename RT<Real>::Node* u1,
                            typename RT<Real>::Node* u2, const int* __restrict__ idx, long long n,
                            typename RT<Real>::Node* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const typename RT<Real>::Node* u = pick3(int(__ldcg(&ctrl->step) % 3), u0, u1, u2);
    out[i] = u[idx[i]];
}

template <class Real>
__global__ void k_halo_unpack(const Ctrl* ctrl, typename RT<Real>::Node* u0, typename RT<Real>::Node* u1,
                              typename RT<Real>::Node* u2, const int* __restrict__ idx, long long n,
                              const typename RT<Real>::Node* __restrict__ in) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    typename RT<Real>::Node* u = pick3(int(__ldcg(&ctrl->step) % 3), u0, u1, u2);
    u[idx[i]] = in[i];
}

// Failure agreement across parts. status[0]: 2 inversion (Abort), 1
// divergence, 0 none (inversion outranks divergence, as assemble runs before
// the update in advance_step); status[1]: -(global id of the first inverted
// element) or INT64_MIN. Reduced with MAX over parts, then k_agree applies the
// global outcome: parts that did advance roll back one step (their previous
// two buffers are intact), so every part halts at the same state.
// status[2]: the inversions this part counted in the step (its own elements
// only), summed over parts; k_agree accumulates the sum into every part's
// totals, so all parts report the global count of the single-GPU run.
__global__ void k_step_status(Ctrl* ctrl, const long long* __restrict__ elem_l2g, long long* status) {
    const int h = ctrl->halted;
    const long long none = -0x7fffffffffffffffll - 1;
    status[0] = h == 4 ? 2 : (h == 5 ? 1 : 0);
    (void)elem_l2g;  // inversions are recorded in global ids already (ElemArgs::elem_l2g)
    if (h != 4 || ctrl->halt_first_inv < 0) status[1] = none;
    else status[1] = -ctrl->halt_first_inv;
    status[2] = (long long)ctrl->step_inv;
    ctrl->step_inv = 0;  // (a halted part runs no more steps: it contributes 0 from now on)
}

__device__ __forceinline__ void accumulate_counts(Ctrl* ctrl, long long global_count) {
    if (!ctrl->multipart) return;
    ctrl->total_inv += (unsigned long long)global_count;
    if (global_count > 0) ctrl->inv_steps += 1;
}

__global__ void k_agree(Ctrl* ctrl, const long long* __restrict__ reduced) {
    const long long code = reduced[0];
    if (ctrl->agreed) return;
    accumulate_counts(ctrl, reduced[2]);
    if (code == 0) return;
    if (ctrl->halted == 0) {
        ctrl->step -= 1;  // this part advanced; another one failed the same step
        ctrl->fail_step = ctrl->step + 1;
    }
    ctrl->halted = code == 2 ? 4 : 5;
    ctrl->halt_first_inv = code == 2 ? -reduced[1] : -1;
    ctrl->agreed = 1;  // later status/agree rounds (halted engine) are no-ops
}

// ------------------------------------------------------------------ peer-memory multi-GPU step
//
// The halo exchange and the failure agreement without NCCL: the node kernel
// of each part stores the new displacement of every owned node another part
// references straight into that part's displacement buffer (NVLink peer
// memory, mapped with CUDA IPC), and its last block posts the step's status
// and epoch into every part's mailbox (system-scope release). A one-warp
// kernel then waits for all parts' epoch (acquire) and applies the same
// agreement as k_agree. No staging buffers, no pack / unpack, no collective
// launches: compute and transfer are one kernel.
constexpr int kMaxParts = 64;

struct Mailbox {
    unsigned long long flag[kMaxParts];  // last epoch each part closed
    long long status[2][kMaxParts][3];   // by epoch parity: {code, -global first inverted, counted inversions}
};

template <class Real>
struct PeerArgs {
    const int* dest_off;                      // [num_owned + 1] halo destinations per owned node
    const int2* dest;                         // (peer part, peer-local node)
    typename RT<Real>::Node* const* peer_u;   // [nparts * 3] every part's displacement buffers
    Mailbox* const* peer_mail;                // [nparts] every part's mailbox (own included)
    int nparts, part;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class Real>
__global__ void __launch_bounds__(256) k_node_peer(const NodeArgs<Real> A, const PeerArgs<Real> P) {
    using T = RT<Real>;
    Ctrl* ctrl = A.ctrl;
    if (*(volatile const int*)&ctrl->halted) return;
    __shared__ int s_nonfinite;
    if (threadIdx.x == 0) s_nonfinite = 0;
    __syncthreads();
    const long long step = ctrl->step;
    const int phn = int((step + 1) % 3);
    typename T::Node* unxt = pick3(phn, A.u[0], A.u[1], A.u[2]);
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < A.N;
         n += (long long)gridDim.x * blockDim.x) {
        if (node_body<Real, false>(A, n, (long long)slice_base_of(A.slice_base, A.slice_w, n) + (n & 31), A.row_len[n],
                                   step))
            s_nonfinite = 1;
        const int d0 = P.dest_off[n], d1 = P.dest_off[n + 1];
        if (d0 < d1) {
            const typename T::Node v = unxt[n];  // written just above by this thread
            for (int d = d0; d < d1; ++d) {
                const int2 q = P.dest[d];
                T::store_node(P.peer_u[3 * q.x + phn] + q.y, v.x, v.y, v.z);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (s_nonfinite) atomicOr(&ctrl->diverged, 1);
    __threadfence_system();  // this block's peer stores, visible to the peers before the epoch
    const unsigned int done = atomicAdd(&ctrl->blocks_done, 1u);
    if (done != gridDim.x - 1) return;
    __threadfence_system();
    close_step<false>(ctrl, step, A.policy);
    const unsigned long long epoch = ++ctrl->epoch;
    const long long code = ctrl->halted == 4 ? 2 : (ctrl->halted == 5 ? 1 : 0);
    const long long first = code == 2 ? -ctrl->halt_first_inv : (-0x7fffffffffffffffll - 1);
    const long long counted = (long long)ctrl->step_inv;
    ctrl->step_inv = 0;
    for (int q = 0; q < P.nparts; ++q) {
        Mailbox* m = P.peer_mail[q];
        m->status[epoch & 1][P.part][0] = code;
        m->status[epoch & 1][P.part][1] = first;
        m->status[epoch & 1][P.part][2] = counted;
    }
    __threadfence_system();
    for (int q = 0; q < P.nparts; ++q) st_release_sys(&P.peer_mail[q]->flag[P.part], epoch);
    ctrl->blocks_done = 0;
}

// Waits until every part closed this part's last epoch, then agrees on the
// outcome exactly like k_agree (all parts halt at the same state).
// The wait is bounded by `timeout_ns` (%globaltimer): a part that never
// posts (dead or stuck rank) halts this one with DJG_E_PEER (6) instead of
// leaving a kernel spinning on the GPU.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_wait_agree(Ctrl* ctrl, const Mailbox* __restrict__ own, int nparts, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    if (ctrl->agreed) return;  // halted and agreed in an earlier step: nothing ran since
    const unsigned long long epoch = ctrl->epoch;
    if (epoch == 0) return;
    const unsigned long long t0 = global_ns();
    for (int q = 0; q < nparts; ++q)
        while (ld_acquire_sys(&own->flag[q]) < epoch) {
            if (global_ns() - t0 > timeout_ns) {
                ctrl->halted = 6;  // DJG_E_PEER
                ctrl->fail_step = ctrl->step + 1;
                ctrl->agreed = 1;
                return;
            }
            __nanosleep(256);
        }
    long long code = 0, first = -0x7fffffffffffffffll - 1, counted = 0;
    for (int q = 0; q < nparts; ++q) {
        code = max(code, own->status[epoch & 1][q][0]);
        first = max(first, own->status[epoch & 1][q][1]);
        counted += own->status[epoch & 1][q][2];
    }
    accumulate_counts(ctrl, counted);
    if (code == 0) return;
    if (ctrl->halted == 0) {
        ctrl->step -= 1;  // this part advanced; another one failed the same step
        ctrl->fail_step = ctrl->step + 1;
    }
    ctrl->halted = code == 2 ? 4 : 5;
    ctrl->halt_first_inv = code == 2 ? -first : -1;
    ctrl->agreed = 1;
}

// ------------------------------------------------------------------ precompute

// build_element_constants on the device: the record of every
// element from the reference coordinates, through the same element_math
// functions as the host builder, written straight into the constant planes
// (the first `nrec` Reals of the record: everything, or the compact part).
// bad[0] collects the smallest element with det J0 <= 0 (MeshError).
template <class Real, int KIND, int MODEL>
__global__ void k_precompute(const ElemArgs<Real> A, int nrec, int nfull, typename RT<Real>::Plane* planes,
                             Real* tail, unsigned long long* bad) {
    using L = Layout<KIND, MODEL>;
    using T = RT<Real>;
    constexpr int NPE = L::NPE;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= A.E) return;
    int nid[NPE];
#pragma unroll
    for (int p = 0; p < NPE / 4; ++p) {
        const int4 q = A.conn[(long long)p * A.E + e];
        nid[4 * p + 0] = q.x; nid[4 * p + 1] = q.y; nid[4 * p + 2] = q.z; nid[4 * p + 3] = q.w;
    }
    Real x[8][3];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        if (a < NPE) {
            const typename T::Node v = T::load_node(A.X + nid[a]);
            x[a][0] = v.x; x[a][1] = v.y; x[a][2] = v.z;
        } else {
            x[a][0] = x[a][1] = x[a][2] = Real(0);
        }
    }
    Real c[L::count + 1];
    Real J[3][3], Ji[3][3], det;
    if (!em::jacobian0(KIND, x, J, Ji, det)) {
        atomicMin(bad, (unsigned long long)e);
        return;
    }
    const Real v0 = em::volume0(KIND, det);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) c[3 * i + j] = J[i][j];
    c[9] = det;
    c[10] = v0;
    c[L::count] = Real(0);
    {
        em::first_invariant_tensors(Ji, v0, c + 11, c + 17);
        if constexpr (L::kI4) em::fibre_tensors(Ji, v0, A.mat.A, c + L::m4, c + L::I4m);
        if constexpr (L::kI6) em::fibre_tensors(Ji, v0, A.mat.B, c + L::m6, c + L::I6m);
        if constexpr (L::kI2) em::second_invariant_tensors(Ji, v0, c + 11, c + L::M2, c + L::I2m);
        if constexpr (L::kH8) {
            Real gamma[4][8];
            em::hourglass_vectors(x, Ji, gamma);
            c[L::khg] = A.mat.chk * ref_cbrt(v0);
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int a = 0; a < 8; ++a) c[L::gamma + 8 * m + a] = gamma[m][a];
        }
    }
    // compact record: T4 J0; H8 J0, det, V0, pad, k_hg, gamma (kCompactLen)
    const bool compact = nrec < L::count;
    constexpr int W = T::kPlane;
    for (int f = 0; f < nfull * W + (compact && KIND == 0 ? nrec - nfull * W : 0); ++f) {
        int src = f;
        if (compact && KIND == 1 && f >= kCompactRecord) src = L::khg + (f - kCompactRecord);
        const Real v = (f < nrec && src < L::count && !(compact && KIND == 1 && f == 11)) ? c[src] : Real(0);
        if (f < nfull * W) reinterpret_cast<Real*>(planes + (long long)(f / W) * A.E + e)[f % W] = v;
        else tail[(long long)(f - nfull * W) * A.tail_stride + e] = v;
    }
}

// ------------------------------------------------------------------ setup

// AoS record chunk -> plane layout: plane p of element e holds record Reals
// [kPlane*p, kPlane*p + kPlane).
// nrec < nconst: the compact record (J0, det, V0, pad [, k_hg, gamma from
// canonical offset hg_src]).
template <class Real>
__global__ void k_transpose_consts(const Real* __restrict__ aos, int nconst, int nrec, int hg_src, long long e0,
                                   long long ne, long long E, int nplanes, Real* __restrict__ planes,
                                   Real* __restrict__ tail, long long tail_stride, int ntail) {
    constexpr int W = RT<Real>::kPlane;
    const int nslots = nplanes + ntail;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne * nslots) return;
    const long long e = i / nslots;
    const int p = int(i % nslots);
    const bool compact = nrec < nconst;
    // compact H8 maps record field f >= 12 to canonical field hg_src + f - 12
    auto field = [&](int f) {
        int src = f;
        if (compact && hg_src >= 0 && f >= kCompactRecord) src = hg_src + (f - kCompactRecord);
        const bool pad = f >= nrec || (compact && hg_src >= 0 && f == 11) || src >= nconst;
        return pad ? Real(0) : aos[e * nconst + src];
    };
    if (p < nplanes) {
        Real* dst = planes + ((long long)p * E + e0 + e) * W;
#pragma unroll
        for (int k = 0; k < W; ++k) dst[k] = field(p * W + k);
    } else {
        tail[(long long)(p - nplanes) * tail_stride + e0 + e] = field(nplanes * W + (p - nplanes));
    }
}

// ------------------------------------------------------------------ layout on the device
//
// NodeElementAdjacency::build (mesh.hpp:299-320) and the engine's slot layout
// built on the GPU (DJG_FLAG_DEVICE_PRECOMPUTE without a caller CSR): count
// pairs per node, exclusive scan -> row offsets, stable radix sort of the
// pair index p = e * npe + a by node (stable: each row keeps ascending
// element order, exactly the host counting sort's order), rank of a pair =
// its sorted position - the row offset. Integer work, identical results.

__global__ void k_count_nodes(const int* __restrict__ conn, long long P, long long N, int* __restrict__ cnt,
                              int* __restrict__ bad) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int n = conn[p];
    if (n < 0 || n >= N) {
        atomicOr(bad, 1);
        return;
    }
    atomicAdd(cnt + n, 1);
}

__global__ void k_iota(int* __restrict__ v, long long P) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) v[p] = int(p);
}

__global__ void k_ranks_from_sorted(const int* __restrict__ keys, const int* __restrict__ vals,
                                    const int* __restrict__ off, long long P, int* __restrict__ rank_of_pair) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < P) rank_of_pair[vals[q]] = int(q - off[keys[q]]);
}

// 32 x the widest row of each 32-node slice (the slice's slot rows).
__global__ void k_slice_caps(const int* __restrict__ len, long long N, long long* __restrict__ cap) {
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long S = (N + 31) / 32;
    if (s > S) return;
    int w = 0;
    if (s < S)
        for (long long n = 32 * s; n < 32 * s + 32 && n < N; ++n) w = max(w, len[n]);
    cap[s] = 32ll * w;
}

__global__ void k_narrow_i64(const long long* __restrict__ in, long long n, int* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = int(in[i]);
}

__global__ void k_pack_ranks(const int* __restrict__ rank_of_pair, long long P, int rb, unsigned char* __restrict__ out) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int k = rank_of_pair[p];
    out[p * rb] = (unsigned char)(k & 0xff);
    if (rb == 2) out[p * rb + 1] = (unsigned char)(k >> 8);
}

__global__ void k_conn_planes(const int* __restrict__ conn, long long E, int npe, int* __restrict__ planes) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    for (int q = 0; q < npe / 4; ++q)
        for (int k = 0; k < 4; ++k) planes[((long long)q * E + e) * 4 + k] = conn[e * npe + 4 * q + k];
}

// V0 (element.hpp:59-85) and characteristic_length (precompute.hpp:303-319)
// of every element from the reference coordinates.
template <class Real, int KIND>
__global__ void k_volume_length(const ElemArgs<Real> A, Real* __restrict__ v0_out, Real* __restrict__ len_out) {
    using T = RT<Real>;
    constexpr int NPE = KIND == 1 ? 8 : 4;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= A.E) return;
    Real x[8][3];
#pragma unroll
    for (int q = 0; q < NPE / 4; ++q) {
        const int4 c = A.conn[(long long)q * A.E + e];
        const int id[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const typename T::Node v = T::load_node(A.X + id[k]);
            x[4 * q + k][0] = v.x; x[4 * q + k][1] = v.y; x[4 * q + k][2] = v.z;
        }
    }
#pragma unroll
    for (int a = NPE; a < 8; ++a) x[a][0] = x[a][1] = x[a][2] = Real(0);
    Real J[3][3], Ji[3][3], det;
    Real v0 = Real(0);
    if (em::jacobian0(KIND, x, J, Ji, det)) v0 = em::volume0(KIND, det);
    v0_out[e] = v0;
    len_out[e] = em::char_length(KIND, x, v0);
}

// lump_mass (precompute.hpp:275-287): every node sums rho V0 / npe of its
// elements in ascending element order (its sorted CSR row), from +0.
template <class Real>
__global__ void k_lump_mass(const int* __restrict__ pairs, const int* __restrict__ off, long long N, int npe,
                            const Real* __restrict__ v0, Real rho, Real* __restrict__ mass) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    Real acc = Real(0);
    for (int q = off[n]; q < off[n + 1]; ++q) acc += rho * v0[pairs[q] / npe] / Real(npe);
    mass[n] = acc;
}

// djg_advance_host: the largest node id each element chunk reads (so a chunk
// can start once that prefix of u_curr has been uploaded).
template <int NPE>
__global__ void k_chunk_maxnode(const int4* __restrict__ conn, long long E, long long chunk, int* __restrict__ out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int m = -1;
    if (e < E) {
#pragma unroll
        for (int p = 0; p < NPE / 4; ++p) {
            const int4 q = conn[(long long)p * E + e];
            m = max(m, max(max(q.x, q.y), max(q.z, q.w)));
        }
    }
    // a warp may straddle two chunks: reduce per chunk id
    const long long c = e < E ? e / chunk : -1;
    const long long c0 = __shfl_sync(0xffffffffu, c, 0);
    const bool uniform = __all_sync(0xffffffffu, c == c0);
    if (uniform) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && c0 >= 0) atomicMax(out + c0, m);
    } else if (c >= 0) {
        atomicMax(out + c, m);
    }
}

// Packs flat Real[3N] into padded nodes and back.
template <class Real>
__global__ void k_pack_nodes(const Real* __restrict__ flat, long long N, typename RT<Real>::Node* __restrict__ out) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    if (flat) RT<Real>::store_node(out + n, flat[3 * n], flat[3 * n + 1], flat[3 * n + 2]);
    else RT<Real>::store_node(out + n, Real(0), Real(0), Real(0));
}

template <class Real>
__global__ void k_unpack_nodes(const typename RT<Real>::Node* __restrict__ in, long long N, Real* __restrict__ flat) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const typename RT<Real>::Node v = in[n];
    flat[3 * n] = v.x;
    flat[3 * n + 1] = v.y;
    flat[3 * n + 2] = v.z;
}

}  // namespace djg
