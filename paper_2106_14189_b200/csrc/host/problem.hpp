// Host-side problem preparation for the B200 DJ-TLED engine.
//
// Everything here runs once before the step loop: mesh generation, the
// node->element adjacency, the per-element hot constants, lumped masses, the
// stable time step, boundary conditions and update coefficients. The
// arithmetic is written to follow the reference operation by operation (the
// file:line next to each function), because the device step consumes these
// Reals and parity with the reference starts here: the same inputs must come
// out bit-identical. Compile without -ffast-math and with -ffp-contract=off.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "djg_types.h"
#include "../common/box_mesh.hpp"
#include "../common/element_math.hpp"

namespace djg {

// Error types with the reference's meaning (core.hpp:28-57).
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct MeshError : std::runtime_error {
    MeshError(const std::string& what, long element = -1)
        : std::runtime_error(element < 0 ? what : "element " + std::to_string(element) + ": " + what),
          element_(element) {}
    long element() const { return element_; }
    long element_;
};
struct SimulationError : std::runtime_error {
    enum class Kind { ElementInversion, Divergence };
    SimulationError(Kind kind, const std::string& what, long index)
        : std::runtime_error(what), kind_(kind), index_(index) {}
    Kind kind() const { return kind_; }
    long index() const { return index_; }
    Kind kind_;
    long index_;
};

inline int npe_of(int kind) { return kind == DJG_T4 ? 4 : 8; }

// Number of Reals in the canonical hot-field record (djg.h).
inline int const_count(int kind, int model) {
    int n = 23;
    if (model == DJG_TI || model == DJG_OT) n += 12;
    if (model == DJG_OT) n += 12;
    if (model == DJG_MR) n += 21 + 36;
    if (model == DJG_I57) n += 2 * (21 + 36);
    if (kind == DJG_H8) n += 33;
    return n;
}

// Field offsets inside the canonical record.
struct ConstLayout {
    int J0 = 0, det = 9, V0 = 10, m1 = 11, I1m = 17;
    int m4 = -1, I4m = -1, m6 = -1, I6m = -1, M2 = -1, I2m = -1, M5 = -1, I5m = -1, M7 = -1, I7m = -1;
    int khg = -1, gamma = -1;
    int count = 23;
    ConstLayout(int kind, int model) {
        int o = 23;
        if (model == DJG_TI || model == DJG_OT) { m4 = o; I4m = o + 6; o += 12; }
        if (model == DJG_OT) { m6 = o; I6m = o + 6; o += 12; }
        if (model == DJG_MR) { M2 = o; I2m = o + 21; o += 57; }
        if (model == DJG_I57) { M5 = o; I5m = o + 21; M7 = o + 57; I7m = o + 78; o += 114; }
        if (kind == DJG_H8) { khg = o; gamma = o + 1; o += 33; }
        count = o;
    }
};

// Shape derivatives at the single integration point, d[i][a] = dh_a/dxi_i
// (element.hpp:31-47). H8 corner signs follow element.hpp:17-20.
inline constexpr int kCornerSign[8][3] = {
    {-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
    {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1},
};

template <class Real>
struct Shape {
    int kind, n;
    Real d[3][8];
    explicit Shape(int k) : kind(k), n(npe_of(k)) {
        for (int i = 0; i < 3; ++i)
            for (int a = 0; a < 8; ++a) d[i][a] = Real(0);
        if (k == DJG_T4) {
            for (int i = 0; i < 3; ++i) {
                d[i][0] = Real(-1);
                d[i][i + 1] = Real(1);
            }
        } else {
            for (int a = 0; a < 8; ++a)
                for (int i = 0; i < 3; ++i) d[i][a] = Real(kCornerSign[a][i]) / Real(8);
        }
    }
};

template <class Real>
struct V3 {
    Real x, y, z;
};

// Symmetric 3x3 in (xx,yy,zz,xy,xz,yz) order (core.hpp:214-228).
template <class Real>
struct Sym {
    Real v[6];
};

// outer(v) (core.hpp:240-251): the fibre structure tensor of a unit fibre.
// (Every other tensor operation of the precompute lives in
// common/element_math.hpp, shared with the device.)
template <class Real>
inline Sym<Real> outer(const V3<Real>& v) {
    return {{v.x * v.x, v.y * v.y, v.z * v.z, v.x * v.y, v.x * v.z, v.y * v.z}};
}

// ---------------------------------------------------------------- material

// Material<Real> (material.hpp:140-230) restricted to what precompute and the
// step need.
template <class Real>
struct Material {
    int model = DJG_NH;
    Real mu = 0, kappa = 0, rho = 0, eta_a = 0, eta_b = 0, c10 = 0, c01 = 0;
    V3<Real> fa{0, 0, 0}, fb{0, 0, 0};

    static Material from(const djg_material_params& p) {
        Material m;
        m.model = p.model;
        m.mu = Real(p.mu); m.kappa = Real(p.kappa); m.rho = Real(p.rho);
        m.eta_a = Real(p.eta_a); m.eta_b = Real(p.eta_b);
        m.c10 = Real(p.c10); m.c01 = Real(p.c01);
        m.fa = {Real(p.fibre_a[0]), Real(p.fibre_a[1]), Real(p.fibre_a[2])};
        m.fb = {Real(p.fibre_b[0]), Real(p.fibre_b[1]), Real(p.fibre_b[2])};
        m.validate();
        return m;
    }

    static Real norm(const V3<Real>& v) { return std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }

    void validate() const {  // material.hpp:187-207
        if (model < DJG_NH || model > DJG_I57) throw ConfigError("unknown material model");
        if (!(kappa > Real(0))) throw ConfigError("bulk modulus must be positive");
        if (!(rho > Real(0))) throw ConfigError("density must be positive");
        if (model == DJG_MR) {
            if (c10 < Real(0) || c01 < Real(0)) throw ConfigError("Mooney-Rivlin coefficients must be >= 0");
            if (!(c10 + c01 > Real(0))) throw ConfigError("Mooney-Rivlin coefficients must not both vanish");
            return;
        }
        if (model == DJG_I57) {  // test_forces.cpp:248-260: both fibre families
            if (eta_a < Real(0) || eta_b < Real(0)) throw ConfigError("fibre stiffnesses eta5 / eta7 must be >= 0");
            if (!(norm(fa) > Real(0)) || !(norm(fb) > Real(0))) throw ConfigError("fibre directions a and b must be nonzero");
        }
        if (model == DJG_OT) {
            if (eta_b < Real(0)) throw ConfigError("fibre stiffness eta_b must be >= 0");
            if (!(norm(fb) > Real(0))) throw ConfigError("fibre direction b must be nonzero");
        }
        if (model == DJG_OT || model == DJG_TI) {
            if (eta_a < Real(0)) throw ConfigError("fibre stiffness eta_a must be >= 0");
            if (!(norm(fa) > Real(0))) throw ConfigError("fibre direction a must be nonzero");
        }
        if (!(mu > Real(0))) throw ConfigError("shear modulus must be positive");
    }

    bool needs_i4() const { return model == DJG_TI || model == DJG_OT; }
    bool needs_i6() const { return model == DJG_OT; }
    bool needs_i2() const { return model == DJG_MR; }
    bool needs_i57() const { return model == DJG_I57; }
    bool needs_fibre_a() const { return needs_i4() || needs_i57(); }  // InvariantSet::any_fibre_a
    bool needs_fibre_b() const { return needs_i6() || needs_i57(); }

    Real shear_modulus() const { return model == DJG_MR ? 2 * (c10 + c01) : mu; }

    // FibreDirections::from normalisation (precompute.hpp:22-39).
    static V3<Real> unit(const V3<Real>& v) {
        const Real n = norm(v);
        const Real s = Real(1) / n;
        return {s * v.x, s * v.y, s * v.z};
    }
};

// dilatational_wave_speed (material.hpp:117-120)
template <class Real>
inline Real wave_speed(const Material<Real>& m) {
    return std::sqrt((m.kappa + Real(4) / Real(3) * m.shear_modulus()) / m.rho);
}

// ---------------------------------------------------------------- mesh

template <class Real>
struct Mesh {
    int kind = DJG_T4;
    std::vector<Real> nodes;      // 3N
    std::vector<int32_t> conn;    // npe*E
    int32_t box_div[3] = {0, 0, 0};  // generate_box divisions (0: not a generated box)
    int npe() const { return npe_of(kind); }
    int64_t num_nodes() const { return int64_t(nodes.size() / 3); }
    int64_t num_elements() const { return int64_t(conn.size()) / npe(); }
    V3<Real> node(int64_t n) const { return {nodes[3 * n], nodes[3 * n + 1], nodes[3 * n + 2]}; }
};

// generate_box (mesh.hpp:208-264): lexicographic nodes, H8 cells in corner
// order, T4 six-tet split along the (0,0,0)-(1,1,1) diagonal, odd axis orders
// swapping the middle pair. The per-node and per-cell pieces are separate
// so a part of the box can be generated without the rest (build_box_part).
template <class Real>
inline Real box_coord(const double extent, int64_t i, int64_t n) {
    return Real(extent) * Real(int(i)) / Real(int(n));
}

inline void check_box(const double extent[3], const int32_t div[3]) {
    for (int i = 0; i < 3; ++i) {
        if (!(extent[i] > 0)) throw ConfigError("box extent must be positive");
        if (div[i] < 1) throw ConfigError("box divisions must be >= 1");
    }
}

template <class Real>
inline Mesh<Real> generate_box(const double extent_in[3], const int32_t div[3], int kind) {
    for (int i = 0; i < 3; ++i)
        if (!(Real(extent_in[i]) > Real(0))) throw ConfigError("box extent must be positive");
    check_box(extent_in, div);
    const int64_t nx = div[0], ny = div[1], nz = div[2];
    Mesh<Real> m;
    m.kind = kind;
    for (int i = 0; i < 3; ++i) m.box_div[i] = div[i];
    m.nodes.resize(size_t(3 * (nx + 1) * (ny + 1) * (nz + 1)));
    size_t w = 0;
    for (int64_t k = 0; k <= nz; ++k)
        for (int64_t j = 0; j <= ny; ++j)
            for (int64_t i = 0; i <= nx; ++i) {
                m.nodes[w++] = box_coord<Real>(extent_in[0], i, nx);
                m.nodes[w++] = box_coord<Real>(extent_in[1], j, ny);
                m.nodes[w++] = box_coord<Real>(extent_in[2], k, nz);
            }
    const int64_t cells = nx * ny * nz;
    const int per = kind == DJG_H8 ? 8 : 24;
    m.conn.resize(size_t(cells * per));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < cells; ++c) box_cell_conn(kind, div, c, m.conn.data() + c * per);
    return m;
}

// validate_mesh (mesh.hpp:75-92).
template <class Real>
inline void validate_mesh(const Mesh<Real>& m) {
    const int npe = m.npe();
    const int64_t n = m.num_nodes();
    if (m.conn.size() % size_t(npe) != 0)
        throw MeshError("connectivity length not a multiple of nodes per element");
    const int64_t E = m.num_elements();
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < npe; ++a) {
            const int32_t c = m.conn[size_t(e * npe + a)];
            if (c < 0 || c >= n) throw MeshError("connectivity index " + std::to_string(c) + " out of range", long(e));
        }
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t e = 0; e < E; ++e) {
        Real x[8][3] = {};
        for (int a = 0; a < npe; ++a) {
            const V3<Real> p = m.node(m.conn[size_t(e * npe + a)]);
            x[a][0] = p.x;
            x[a][1] = p.y;
            x[a][2] = p.z;
        }
        Real J[3][3], Ji[3][3], det;
        if (!em::jacobian0(m.kind, x, J, Ji, det) || !(em::volume0(m.kind, det) > Real(0)))
            bad = std::max<int64_t>(bad, E - e);
    }
    if (bad >= 0) throw MeshError("non-positive reference Jacobian determinant", long(E - bad));
}

// NodeElementAdjacency::build (mesh.hpp:299-320): counting sort over elements
// in ascending order, so each node's row lists its elements ascending.
struct Adjacency {
    std::vector<int64_t> offsets;  // N+1
    std::vector<int64_t> elem;     // npe*E
    std::vector<int32_t> local;    // npe*E
};

inline Adjacency build_adjacency(const std::vector<int32_t>& conn, int64_t n, int npe) {
    Adjacency adj;
    std::vector<int64_t> count(size_t(n), 0);
    for (int32_t idx : conn) ++count[size_t(idx)];
    adj.offsets.assign(size_t(n) + 1, 0);
    for (int64_t i = 0; i < n; ++i) adj.offsets[size_t(i + 1)] = adj.offsets[size_t(i)] + count[size_t(i)];
    adj.elem.resize(conn.size());
    adj.local.resize(conn.size());
    std::vector<int64_t> cursor(adj.offsets.begin(), adj.offsets.end() - 1);
    const int64_t E = int64_t(conn.size()) / npe;
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < npe; ++a) {
            const int64_t p = cursor[size_t(conn[size_t(e * npe + a)])]++;
            adj.elem[size_t(p)] = e;
            adj.local[size_t(p)] = a;
        }
    return adj;
}

// ---------------------------------------------------------------- precompute

// The hot-field record of build_element_constants (precompute.hpp:206-255),
// through the arithmetic shared with the device (common/element_math.hpp).
template <class Real>
inline bool element_record(const V3<Real>* x, const Shape<Real>& D, const Material<Real>& mat,
                           const V3<Real>& fa_unit, const V3<Real>& fb_unit, Real c_hg,
                           const ConstLayout& L, Real* out) {
    Real xa[8][3];
    for (int a = 0; a < D.n; ++a) {
        xa[a][0] = x[a].x;
        xa[a][1] = x[a].y;
        xa[a][2] = x[a].z;
    }
    for (int a = D.n; a < 8; ++a) xa[a][0] = xa[a][1] = xa[a][2] = Real(0);
    Real J[3][3], Ji[3][3], det;
    if (!em::jacobian0(D.kind, xa, J, Ji, det)) return false;
    const Real v0 = em::volume0(D.kind, det);
    if (!(v0 > Real(0))) return false;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out[L.J0 + 3 * r + c] = J[r][c];
    out[L.det] = det;
    out[L.V0] = v0;
    em::first_invariant_tensors(Ji, v0, out + L.m1, out + L.I1m);
    if (mat.needs_i2()) em::second_invariant_tensors(Ji, v0, out + L.m1, out + L.M2, out + L.I2m);
    if (mat.needs_i4()) {
        const Sym<Real> A = outer(fa_unit);
        em::fibre_tensors(Ji, v0, A.v, out + L.m4, out + L.I4m);
    }
    if (mat.needs_i6()) {
        const Sym<Real> B = outer(fb_unit);
        em::fibre_tensors(Ji, v0, B.v, out + L.m6, out + L.I6m);
    }
    if (mat.needs_i57()) {  // precompute.hpp:237-240, 245-248
        const Sym<Real> A = outer(fa_unit), B = outer(fb_unit);
        const Real a[3] = {fa_unit.x, fa_unit.y, fa_unit.z}, b[3] = {fb_unit.x, fb_unit.y, fb_unit.z};
        em::fibre_second_tensors(Ji, v0, a, A.v, out + L.M5, out + L.I5m);
        em::fibre_second_tensors(Ji, v0, b, B.v, out + L.M7, out + L.I7m);
    }
    if (D.kind == DJG_H8) {
        Real gamma[4][8];
        em::hourglass_vectors(xa, Ji, gamma);
        out[L.khg] = c_hg * mat.kappa * std::cbrt(v0);
        for (int m = 0; m < 4; ++m)
            for (int a = 0; a < 8; ++a) out[L.gamma + 8 * m + a] = gamma[m][a];
    }
    return true;
}

// Characteristic length (precompute.hpp:303-319) and critical dt (:323-331).
template <class Real>
inline Real tri_area(V3<Real> a, V3<Real> b, V3<Real> c) {
    const V3<Real> u{b.x - a.x, b.y - a.y, b.z - a.z}, v{c.x - a.x, c.y - a.y, c.z - a.z};
    const V3<Real> w{u.y * v.z - u.z * v.y, u.z * v.x - u.x * v.z, u.x * v.y - u.y * v.x};
    return std::sqrt(w.x * w.x + w.y * w.y + w.z * w.z) / 2;
}

template <class Real>
inline Real char_length(const V3<Real>* x, int kind, Real v0) {
    Real a_max = 0;
    if (kind == DJG_T4) {
        static constexpr int f[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        for (auto& t : f) a_max = std::max(a_max, tri_area(x[t[0]], x[t[1]], x[t[2]]));
        return 3 * v0 / a_max;
    }
    static constexpr int f[6][4] = {{0, 3, 2, 1}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
    for (auto& q : f)
        a_max = std::max(a_max, tri_area(x[q[0]], x[q[1]], x[q[2]]) + tri_area(x[q[0]], x[q[2]], x[q[3]]));
    return v0 / a_max;
}

// ---------------------------------------------------------------- problem

template <class Real>
struct Problem {
    Mesh<Real> mesh;
    Material<Real> mat;
    Adjacency adj;
    int nconst = 0;
    std::vector<Real> consts;          // E*nconst
    std::vector<Real> mass;            // N
    std::vector<Real> c1;              // N
    std::vector<uint8_t> massless;     // N
    std::vector<uint8_t> dof_kind;     // 3N
    std::vector<Real> dof_target;      // 3N
    std::vector<Real> dof_t_total;     // 3N
    Real dt = 0, crit_dt = 0, alpha = 0, c2 = 0, c3 = 0, ramp_t_total = 0, c_wave = 0;
    Real c_hg = 0;
    int policy = DJG_ABORT;
};

template <class Real>
inline void bounding_box(const Mesh<Real>& m, Real lo[3], Real hi[3]) {
    for (int i = 0; i < 3; ++i) {
        lo[i] = std::numeric_limits<Real>::max();
        hi[i] = std::numeric_limits<Real>::lowest();
    }
    const int64_t n = m.num_nodes();
    for (int64_t k = 0; k < n; ++k)
        for (int i = 0; i < 3; ++i) {
            lo[i] = std::min(lo[i], m.nodes[size_t(3 * k + i)]);
            hi[i] = std::max(hi[i], m.nodes[size_t(3 * k + i)]);
        }
}

// select_plane_nodes (config.hpp:31-42)
template <class Real>
inline std::vector<int32_t> plane_nodes(const Mesh<Real>& m, int axis, bool is_max, const Real lo[3], const Real hi[3]) {
    const Real value = is_max ? hi[axis] : lo[axis];
    const Real extent = hi[axis] - lo[axis];
    const Real eps = Real(1e-9) * (extent > Real(0) ? extent : Real(1));
    std::vector<int32_t> out;
    const int64_t n = m.num_nodes();
    for (int64_t k = 0; k < n; ++k)
        if (std::abs(m.nodes[size_t(3 * k + axis)] - value) <= eps) out.push_back(int32_t(k));
    return out;
}

template <class Real>
inline Problem<Real> build_problem(const djg_scenario_spec& s, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    if (s.kind != DJG_T4 && s.kind != DJG_H8) throw ConfigError("unknown element kind");
    Problem<Real> P;
    P.policy = s.policy;
    if (s.nodes == nullptr) {
        P.mesh = generate_box<Real>(s.extent, s.divisions, s.kind);
    } else {
        if (s.num_nodes < 0 || s.num_elements < 0 || (s.num_elements > 0 && !s.conn))
            throw ConfigError("explicit mesh needs nodes and connectivity");
        P.mesh.kind = s.kind;
        P.mesh.nodes.resize(size_t(3 * s.num_nodes));
        for (int64_t i = 0; i < 3 * s.num_nodes; ++i) P.mesh.nodes[size_t(i)] = Real(s.nodes[i]);
        P.mesh.conn.assign(s.conn, s.conn + s.num_elements * npe_of(s.kind));
    }
    validate_mesh(P.mesh);
    P.mat = Material<Real>::from(s.material);
    const int npe = P.mesh.npe();
    const int64_t N = P.mesh.num_nodes(), E = P.mesh.num_elements();
    const ConstLayout L(s.kind, P.mat.model);
    P.nconst = L.count;

    // DjModel::build -> build_constants (djtled_force.hpp:145-157, precompute.hpp:258-272)
    V3<Real> fa{0, 0, 0}, fb{0, 0, 0};
    if (P.mat.needs_fibre_a()) fa = Material<Real>::unit(P.mat.fa);
    if (P.mat.needs_fibre_b()) fb = Material<Real>::unit(P.mat.fb);
    const Real c_hg = Real(s.c_hg);
    P.c_hg = c_hg;
    const Shape<Real> D(s.kind);
    P.consts.assign(size_t(E) * size_t(L.count), Real(0));
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t e = 0; e < E; ++e) {
        V3<Real> x[8];
        for (int a = 0; a < npe; ++a) x[a] = P.mesh.node(P.mesh.conn[size_t(e * npe + a)]);
        if (!element_record(x, D, P.mat, fa, fb, c_hg, L, P.consts.data() + size_t(e) * L.count))
            bad = std::max<int64_t>(bad, E - e);
    }
    if (bad >= 0) throw MeshError("non-positive reference Jacobian determinant", long(E - bad));

    P.adj = build_adjacency(P.mesh.conn, N, npe);

    // lump_mass (precompute.hpp:275-287): each node sums the shares of its
    // elements in ascending element order -- the order of the reference's
    // serial element loop -- so the CSR row gives the same bits in parallel.
    P.mass.assign(size_t(N), Real(0));
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        Real acc = Real(0);
        for (int64_t p = P.adj.offsets[size_t(n)]; p < P.adj.offsets[size_t(n + 1)]; ++p) {
            const int64_t e = P.adj.elem[size_t(p)];
            acc += P.mat.rho * P.consts[size_t(e) * L.count + L.V0] / Real(npe);
        }
        P.mass[size_t(n)] = acc;
    }

    // critical_dt (precompute.hpp:323-331); min is order independent.
    P.c_wave = wave_speed(P.mat);
    Real l_min = std::numeric_limits<Real>::max();
#pragma omp parallel
    {
        Real local = std::numeric_limits<Real>::max();
#pragma omp for schedule(static) nowait
        for (int64_t e = 0; e < E; ++e) {
            V3<Real> x[8];
            for (int a = 0; a < npe; ++a) x[a] = P.mesh.node(P.mesh.conn[size_t(e * npe + a)]);
            local = std::min(local, char_length(x, s.kind, P.consts[size_t(e) * L.count + L.V0]));
        }
#pragma omp critical
        l_min = std::min(l_min, local);
    }
    if (!(l_min > Real(0))) throw MeshError("degenerate element with zero characteristic length");
    P.crit_dt = l_min / P.c_wave;
    P.dt = s.dt > 0 ? Real(s.dt) : Real(s.safety) * P.crit_dt;
    if (!(P.dt > Real(0))) throw ConfigError("time step must be positive");

    // relaxation_alpha (solver.hpp:330-339)
    Real lo[3], hi[3];
    bounding_box(P.mesh, lo, hi);
    if (s.alpha_mode == 0) {
        const Real mu = P.mat.shear_modulus();
        const Real e_mod = 9 * P.mat.kappa * mu / (3 * P.mat.kappa + mu);
        const Real c_bar = std::sqrt(e_mod / P.mat.rho);
        const Real l = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
        if (!(l > Real(0))) throw ConfigError("mesh has zero extent");
        P.alpha = Real(M_PI) * c_bar / l;
    } else {
        P.alpha = Real(s.alpha);
    }

    // Boundary conditions -> DofConstraints (solver.hpp:18-33, mesh.hpp:55-70).
    P.dof_kind.assign(size_t(3 * N), uint8_t(DJG_FREE));
    P.dof_target.assign(size_t(3 * N), Real(0));
    P.dof_t_total.assign(size_t(3 * N), Real(1));
    auto claim = [&](int64_t node, int axis) -> uint8_t& {
        if (node < 0 || node >= N) throw ConfigError("boundary condition references invalid node");
        if (axis < 0 || axis > 2) throw ConfigError("boundary condition axis out of range");
        uint8_t& k = P.dof_kind[size_t(3 * node + axis)];
        if (k != DJG_FREE)
            throw ConfigError("node " + std::to_string(node) + " axis " + std::to_string(axis) +
                              " appears in more than one boundary condition");
        return k;
    };
    auto prescribe = [&](int64_t node, int axis, Real target, Real t_total) {
        if (!(t_total > Real(0))) throw ConfigError("ramp duration must be positive");
        claim(node, axis) = DJG_PRESCRIBED;
        P.dof_target[size_t(3 * node + axis)] = target;
        P.dof_t_total[size_t(3 * node + axis)] = t_total;
    };
    if (s.bc_mode == 1) {
        const auto bottom = plane_nodes(P.mesh, 2, false, lo, hi);
        const auto top = plane_nodes(P.mesh, 2, true, lo, hi);
        for (int32_t n : bottom) {
            if (s.fix_all_axes) {
                claim(n, 0) = DJG_FIXED;
                claim(n, 1) = DJG_FIXED;
            }
            claim(n, 2) = DJG_FIXED;
        }
        if (top.empty()) throw ConfigError("prescribe rule selects no nodes");
        P.ramp_t_total = P.dt * Real(s.ramp_steps);
        for (int32_t n : top) prescribe(n, 2, Real(s.target), P.ramp_t_total);
    } else if (s.bc_mode == 2) {
        for (int64_t i = 0; i < s.n_fixed; ++i) claim(s.fixed_node[i], s.fixed_axis[i]) = DJG_FIXED;
        for (int64_t i = 0; i < s.n_prescribed; ++i)
            prescribe(s.presc_node[i], s.presc_axis[i], Real(s.presc_target[i]), Real(s.presc_t_total[i]));
    } else if (s.bc_mode != 0) {
        throw ConfigError("unknown boundary condition mode");
    }

    // UpdateCoeffs::build (solver.hpp:70-86)
    const Real denom = Real(1) + P.alpha * P.dt / 2;
    P.c2 = Real(2) / denom;
    P.c3 = -(Real(1) - P.alpha * P.dt / 2) / denom;
    P.c1.assign(size_t(N), Real(0));
    P.massless.assign(size_t(N), 0);
    for (int64_t n = 0; n < N; ++n) {
        if (P.mass[size_t(n)] > Real(0))
            P.c1[size_t(n)] = P.dt * P.dt / (P.mass[size_t(n)] * denom);
        else
            P.massless[size_t(n)] = 1;
    }
    return P;
}

}  // namespace djg

// ---------------------------------------------------------------- partition
//
// Multi-GPU decomposition. Elements are split by recursive
// coordinate bisection of their centroids (ties broken by element id, so the
// result is reproducible); a node is owned by the part of its lowest-id
// element. Part p computes every element touching a node it owns (its own
// plus "ghost" elements), in ascending global element id, so the gather of an
// owned node sums exactly the same rows in exactly the same order as on one
// GPU: results are bit-identical for any part count. After each step, owners
// send the displacement of nodes other parts reference (halo).

namespace djg {

template <class Real>
inline std::vector<int32_t> rcb_parts(const Mesh<Real>& m, int nparts) {
    const int64_t E = m.num_elements();
    const int npe = m.npe();
    std::vector<double> c(size_t(3 * E));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
        for (int i = 0; i < 3; ++i) {
            double s = 0;
            for (int a = 0; a < npe; ++a) s += double(m.nodes[size_t(3 * m.conn[size_t(e * npe + a)] + i)]);
            c[size_t(3 * e + i)] = s / npe;
        }
    std::vector<int64_t> idx(static_cast<size_t>(E));
    for (int64_t e = 0; e < E; ++e) idx[size_t(e)] = e;
    std::vector<int32_t> part(static_cast<size_t>(E), 0);
    struct Job {
        int64_t lo, hi;
        int p0, np;
    };
    std::vector<Job> stack{{0, E, 0, nparts}};
    while (!stack.empty()) {
        const Job j = stack.back();
        stack.pop_back();
        if (j.np <= 1 || j.hi - j.lo <= 1) {
            for (int64_t q = j.lo; q < j.hi; ++q) part[size_t(idx[size_t(q)])] = j.p0;
            continue;
        }
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int64_t q = j.lo; q < j.hi; ++q)
            for (int i = 0; i < 3; ++i) {
                lo[i] = std::min(lo[i], c[size_t(3 * idx[size_t(q)] + i)]);
                hi[i] = std::max(hi[i], c[size_t(3 * idx[size_t(q)] + i)]);
            }
        int ax = 0;
        for (int i = 1; i < 3; ++i)
            if (hi[i] - lo[i] > hi[ax] - lo[ax]) ax = i;
        const int nl = j.np / 2;
        const int64_t mid = j.lo + (j.hi - j.lo) * nl / j.np;
        // strict total order (coordinate, id): the split set is unique
        std::nth_element(idx.begin() + j.lo, idx.begin() + mid, idx.begin() + j.hi, [&](int64_t a, int64_t b) {
            const double ca = c[size_t(3 * a + ax)], cb = c[size_t(3 * b + ax)];
            return ca < cb || (ca == cb && a < b);
        });
        stack.push_back({mid, j.hi, j.p0 + nl, j.np - nl});
        stack.push_back({j.lo, mid, j.p0, nl});
    }
    return part;
}

struct Halo {
    std::vector<int32_t> neighbors;    // ascending part ids
    std::vector<int64_t> send_off;     // per neighbor, into send_nodes
    std::vector<int64_t> recv_off;     // per neighbor, into recv_nodes
    std::vector<int32_t> send_nodes;   // local ids of owned nodes, ascending global id per neighbor
    std::vector<int32_t> recv_nodes;   // local ids of ghost nodes, ascending global id per neighbor
};

// Local problem of one part: same layout as Problem, renumbered. Owned nodes
// come first (ascending global id), ghost nodes after (ascending global id);
// local elements ascend in global id.
template <class Real>
struct PartProblem {
    Problem<Real> local;
    int nparts = 1, part = 0;
    int64_t num_owned = 0, global_nodes = 0, global_elements = 0, owned_elements = 0;
    int64_t interior_elements = 0;  // local elements [0, interior) reference no ghost node
    std::vector<int64_t> node_l2g, elem_l2g;
    std::vector<uint8_t> elem_owned;  // per local element: 1 if assigned to this part (it reports the
                                      // element's inversions; other parts hold it as a ghost)
    Halo halo;
};

// Graph partitioning of the element dual graph (elements adjacent when they
// share a face: 3 nodes for T4, 4 for H8) with METIS k-way
// (METIS_PartMeshDual from the CUDA toolkit's libmetis_static.a, idx_t =
// int64). Fixed options and seed: the same mesh gives the same partition on
// every rank and every run.
extern "C" {
int METIS_SetDefaultOptions(int64_t* options);
int METIS_PartMeshDual(int64_t* ne, int64_t* nn, int64_t* eptr, int64_t* eind, int64_t* vwgt, int64_t* vsize,
                       int64_t* ncommon, int64_t* nparts, void* tpwgts, int64_t* options, int64_t* objval,
                       int64_t* epart, int64_t* npart);
}

enum PartMethod { kPartRcb = 0, kPartMetis = 1, kPartBox = 2 };

// Box partition (generated boxes only): recursive bisection of the CELL grid
// -- the longest axis (in cells; ties to the lower axis) split at
// cells * floor(np/2) / np -- so all elements of a cell share a part and every
// part is a block of cells. It needs no coordinates and no global mesh: a
// rank can build its part alone (build_box_part).
struct CellBlock {
    int64_t lo[3], hi[3];  // [lo, hi) cells per axis
};

inline std::vector<CellBlock> box_blocks(const int32_t div[3], int nparts) {
    std::vector<CellBlock> out(static_cast<size_t>(nparts));
    struct Job {
        CellBlock b;
        int p0, np;
    };
    std::vector<Job> stack{{{{0, 0, 0}, {div[0], div[1], div[2]}}, 0, nparts}};
    while (!stack.empty()) {
        Job j = stack.back();
        stack.pop_back();
        if (j.np == 1) {
            out[size_t(j.p0)] = j.b;
            continue;
        }
        int ax = 0;
        for (int i = 1; i < 3; ++i)
            if (j.b.hi[i] - j.b.lo[i] > j.b.hi[ax] - j.b.lo[ax]) ax = i;
        const int nl = j.np / 2;
        const int64_t len = j.b.hi[ax] - j.b.lo[ax];
        if (len < 2) throw ConfigError("box too small for the requested part count");
        const int64_t cut = j.b.lo[ax] + std::max<int64_t>(1, std::min<int64_t>(len - 1, len * nl / j.np));
        Job a = j, b = j;
        a.b.hi[ax] = cut;
        a.np = nl;
        b.b.lo[ax] = cut;
        b.p0 = j.p0 + nl;
        b.np = j.np - nl;
        stack.push_back(b);
        stack.push_back(a);
    }
    return out;
}

inline int box_part_of_cell(const std::vector<CellBlock>& blocks, int64_t ci, int64_t cj, int64_t ck) {
    for (size_t p = 0; p < blocks.size(); ++p) {
        const CellBlock& b = blocks[p];
        if (ci >= b.lo[0] && ci < b.hi[0] && cj >= b.lo[1] && cj < b.hi[1] && ck >= b.lo[2] && ck < b.hi[2])
            return int(p);
    }
    return 0;
}

template <class Real>
inline std::vector<int32_t> metis_parts(const Mesh<Real>& m, int nparts) {
    const int64_t E = m.num_elements(), N = m.num_nodes();
    const int npe = m.npe();
    std::vector<int32_t> part(static_cast<size_t>(E), 0);
    if (nparts <= 1 || E <= 1) return part;
    std::vector<int64_t> eptr(static_cast<size_t>(E + 1)), eind(m.conn.begin(), m.conn.end());
    for (int64_t e = 0; e <= E; ++e) eptr[size_t(e)] = e * npe;
    int64_t options[40];
    METIS_SetDefaultOptions(options);
    options[8] = 1;  // METIS_OPTION_SEED
    int64_t ne = E, nn = N, ncommon = m.kind == DJG_T4 ? 3 : 4, np = nparts, objval = 0;
    std::vector<int64_t> epart(static_cast<size_t>(E)), npart(static_cast<size_t>(N));
    const int rc = METIS_PartMeshDual(&ne, &nn, eptr.data(), eind.data(), nullptr, nullptr, &ncommon, &np, nullptr,
                                      options, &objval, epart.data(), npart.data());
    if (rc != 1) throw ConfigError("METIS_PartMeshDual failed (" + std::to_string(rc) + ")");
    for (int64_t e = 0; e < E; ++e) part[size_t(e)] = int32_t(epart[size_t(e)]);
    return part;
}

template <class Real>
inline std::vector<int32_t> box_parts(const Mesh<Real>& m, int nparts) {
    if (m.box_div[0] < 1) throw ConfigError("the box partition needs a generated box mesh");
    const auto blocks = box_blocks(m.box_div, nparts);
    const int64_t E = m.num_elements(), nx = m.box_div[0], ny = m.box_div[1];
    const int per_cell = m.kind == DJG_T4 ? 6 : 1;
    std::vector<int32_t> part(static_cast<size_t>(E));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const int64_t c = e / per_cell;
        part[size_t(e)] = box_part_of_cell(blocks, c % nx, (c / nx) % ny, c / (nx * ny));
    }
    return part;
}

template <class Real>
inline std::vector<int32_t> element_parts(const Mesh<Real>& m, int nparts, int method) {
    if (method == kPartRcb) return rcb_parts(m, nparts);
    if (method == kPartMetis) return metis_parts(m, nparts);
    if (method == kPartBox) return box_parts(m, nparts);
    throw ConfigError("unknown partition method");
}

// Adjacency of a part's local mesh with every node's row in ascending GLOBAL
// element id (local element ids are interior-first), so an owned node sums
// its rows in the single-GPU order.
inline Adjacency local_adjacency(const std::vector<int32_t>& conn, int64_t Nl, int npe,
                                 const std::vector<int64_t>& elem_l2g) {
    Adjacency adj = build_adjacency(conn, Nl, npe);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t q = 0; q < Nl; ++q) {
        const int64_t b = adj.offsets[size_t(q)], t = adj.offsets[size_t(q + 1)];
        std::vector<std::pair<int64_t, int64_t>> row;
        row.reserve(size_t(t - b));
        for (int64_t p = b; p < t; ++p) row.emplace_back(elem_l2g[size_t(adj.elem[size_t(p)])], p);
        std::sort(row.begin(), row.end());
        std::vector<int64_t> el(size_t(t - b));
        std::vector<int32_t> lo(size_t(t - b));
        for (int64_t k = 0; k < t - b; ++k) {
            el[size_t(k)] = adj.elem[size_t(row[size_t(k)].second)];
            lo[size_t(k)] = adj.local[size_t(row[size_t(k)].second)];
        }
        std::copy(el.begin(), el.end(), adj.elem.begin() + b);
        std::copy(lo.begin(), lo.end(), adj.local.begin() + b);
    }
    return adj;
}

template <class Real>
inline PartProblem<Real> build_part(const Problem<Real>& P, int nparts, int part, int method = kPartRcb) {
    if (nparts < 1 || part < 0 || part >= nparts) throw ConfigError("invalid part index");
    const Mesh<Real>& m = P.mesh;
    const int npe = m.npe();
    const int64_t N = m.num_nodes(), E = m.num_elements();
    const std::vector<int32_t> epart = element_parts(m, nparts, method);
    // owner of a node: part of its lowest-id element (first in its CSR row)
    std::vector<int32_t> owner(static_cast<size_t>(N), 0);  // isolated nodes: part 0
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n)
        if (P.adj.offsets[size_t(n + 1)] > P.adj.offsets[size_t(n)])
            owner[size_t(n)] = epart[size_t(P.adj.elem[size_t(P.adj.offsets[size_t(n)])])];
    // elements computed by this part: any node owned here
    PartProblem<Real> R;
    R.nparts = nparts;
    R.part = part;
    R.global_nodes = N;
    R.global_elements = E;
    std::vector<uint8_t> elocal(static_cast<size_t>(E), 0);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < npe; ++a)
            if (owner[size_t(m.conn[size_t(e * npe + a)])] == part) elocal[size_t(e)] = 1;
    for (int64_t e = 0; e < E; ++e)
        if (elocal[size_t(e)]) {
            R.elem_l2g.push_back(e);
            if (epart[size_t(e)] == part) ++R.owned_elements;
        }
    // local nodes: owned (ascending), then ghosts (ascending)
    std::vector<uint8_t> nlocal(static_cast<size_t>(N), 0);
    for (int64_t e : R.elem_l2g)
        for (int a = 0; a < npe; ++a) nlocal[size_t(m.conn[size_t(e * npe + a)])] = 1;
    for (int64_t n = 0; n < N; ++n)
        if (owner[size_t(n)] == part && (nlocal[size_t(n)] || P.adj.offsets[size_t(n + 1)] == P.adj.offsets[size_t(n)]))
            R.node_l2g.push_back(n);
    R.num_owned = int64_t(R.node_l2g.size());
    for (int64_t n = 0; n < N; ++n)
        if (nlocal[size_t(n)] && owner[size_t(n)] != part) R.node_l2g.push_back(n);
    std::vector<int32_t> g2l(static_cast<size_t>(N), -1);
    for (size_t q = 0; q < R.node_l2g.size(); ++q) g2l[size_t(R.node_l2g[q])] = int32_t(q);
    // Local element order: interior elements (no ghost node) first, then the
    // boundary elements, each ascending in global id -- so a step can compute
    // the interior while the halo is in flight. Each node's CSR row is still
    // sorted by global element id below: the summation order is unchanged.
    {
        std::vector<int64_t> interior, boundary;
        for (int64_t e : R.elem_l2g) {
            bool ghost = false;
            for (int a = 0; a < npe; ++a) ghost |= g2l[size_t(m.conn[size_t(e * npe + a)])] >= R.num_owned;
            (ghost ? boundary : interior).push_back(e);
        }
        R.interior_elements = int64_t(interior.size());
        R.elem_l2g = std::move(interior);
        R.elem_l2g.insert(R.elem_l2g.end(), boundary.begin(), boundary.end());
        R.elem_owned.resize(R.elem_l2g.size());
        for (size_t q = 0; q < R.elem_l2g.size(); ++q) R.elem_owned[q] = epart[size_t(R.elem_l2g[q])] == part;
    }
    // local problem arrays
    Problem<Real>& L = R.local;
    L.mat = P.mat;
    L.nconst = P.nconst;
    L.dt = P.dt;
    L.crit_dt = P.crit_dt;
    L.alpha = P.alpha;
    L.c2 = P.c2;
    L.c3 = P.c3;
    L.ramp_t_total = P.ramp_t_total;
    L.c_wave = P.c_wave;
    L.c_hg = P.c_hg;
    L.policy = P.policy;
    L.mesh.kind = m.kind;
    const int64_t Nl = int64_t(R.node_l2g.size()), El = int64_t(R.elem_l2g.size());
    L.mesh.nodes.resize(size_t(3 * Nl));
    L.mass.resize(size_t(Nl));
    L.c1.resize(size_t(Nl));
    L.massless.resize(size_t(Nl));
    L.dof_kind.resize(size_t(3 * Nl));
    L.dof_target.resize(size_t(3 * Nl));
    L.dof_t_total.resize(size_t(3 * Nl));
    for (int64_t q = 0; q < Nl; ++q) {
        const int64_t n = R.node_l2g[size_t(q)];
        for (int i = 0; i < 3; ++i) {
            L.mesh.nodes[size_t(3 * q + i)] = m.nodes[size_t(3 * n + i)];
            L.dof_kind[size_t(3 * q + i)] = P.dof_kind[size_t(3 * n + i)];
            L.dof_target[size_t(3 * q + i)] = P.dof_target[size_t(3 * n + i)];
            L.dof_t_total[size_t(3 * q + i)] = P.dof_t_total[size_t(3 * n + i)];
        }
        L.mass[size_t(q)] = P.mass[size_t(n)];
        L.c1[size_t(q)] = P.c1[size_t(n)];
        L.massless[size_t(q)] = P.massless[size_t(n)];
    }
    L.mesh.conn.resize(size_t(El * npe));
    L.consts.resize(size_t(El) * size_t(P.nconst));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < El; ++q) {
        const int64_t e = R.elem_l2g[size_t(q)];
        for (int a = 0; a < npe; ++a) L.mesh.conn[size_t(q * npe + a)] = g2l[size_t(m.conn[size_t(e * npe + a)])];
        std::copy(P.consts.begin() + e * P.nconst, P.consts.begin() + (e + 1) * P.nconst,
                  L.consts.begin() + q * P.nconst);
    }
    L.adj = local_adjacency(L.mesh.conn, Nl, npe, R.elem_l2g);
    // halo: parts referencing each node (as a local node of theirs)
    // recv: my ghosts, from their owners
    std::vector<std::vector<int32_t>> recv(static_cast<size_t>(nparts)), send(static_cast<size_t>(nparts));
    for (int64_t q = R.num_owned; q < Nl; ++q) recv[size_t(owner[size_t(R.node_l2g[size_t(q)])])].push_back(int32_t(q));
    // send: my owned nodes that another part's elements touch
    for (int64_t q = 0; q < R.num_owned; ++q) {
        const int64_t n = R.node_l2g[size_t(q)];
        std::vector<int32_t> parts;
        for (int64_t p = P.adj.offsets[size_t(n)]; p < P.adj.offsets[size_t(n + 1)]; ++p) {
            const int64_t e = P.adj.elem[size_t(p)];
            for (int a = 0; a < npe; ++a) {
                const int32_t o = owner[size_t(m.conn[size_t(e * npe + a)])];
                if (o != part) parts.push_back(o);
            }
        }
        std::sort(parts.begin(), parts.end());
        parts.erase(std::unique(parts.begin(), parts.end()), parts.end());
        for (int32_t o : parts) send[size_t(o)].push_back(int32_t(q));
    }
    R.halo.send_off.push_back(0);
    R.halo.recv_off.push_back(0);
    for (int q = 0; q < nparts; ++q) {
        if (q == part || (send[size_t(q)].empty() && recv[size_t(q)].empty())) continue;
        R.halo.neighbors.push_back(q);
        R.halo.send_nodes.insert(R.halo.send_nodes.end(), send[size_t(q)].begin(), send[size_t(q)].end());
        R.halo.recv_nodes.insert(R.halo.recv_nodes.end(), recv[size_t(q)].begin(), recv[size_t(q)].end());
        R.halo.send_off.push_back(int64_t(R.halo.send_nodes.size()));
        R.halo.recv_off.push_back(int64_t(R.halo.recv_nodes.size()));
    }
    return R;
}


// ---------------------------------------------------------------- part-local build
//
// One part of a generated box, built without the global mesh or the global
// problem (multi-GPU setup at scale: each rank builds only its part, SURVEY
// §8(e)). With the box partition (box_blocks) everything the global path
// derives from the whole mesh has a closed form here: the lowest-id element
// of node (i, j, k) lies in cell (max(i-1,0), max(j-1,0), max(k-1,0)), so a
// node's owner is that cell's part; the elements touching an owned node lie
// in the part's cell block grown by one cell on its low sides. The result is
// identical to build_part(build_problem(spec), nparts, part, kPartBox) on
// every owned node and local element (tests/test_partition.py) except the
// time-step data, which needs the GLOBAL minimum characteristic length:
// build_box_part returns this part's minimum, the caller reduces it over the
// parts (MIN is exact) and finish_box_part completes dt, alpha, the BCs and
// the update coefficients.
template <class Real>
inline PartProblem<Real> build_box_part(const djg_scenario_spec& s, int nparts, int part, Real& local_lmin) {
    if (s.nodes != nullptr) throw ConfigError("the part-local build needs a generated box (no explicit mesh)");
    if (s.kind != DJG_T4 && s.kind != DJG_H8) throw ConfigError("unknown element kind");
    if (nparts < 1 || part < 0 || part >= nparts) throw ConfigError("invalid part index");
    if (s.bc_mode != 0 && s.bc_mode != 1) throw ConfigError("the part-local build supports the plane BCs (bc_mode 0 / 1)");
    check_box(s.extent, s.divisions);
    for (int i = 0; i < 3; ++i)
        if (!(Real(s.extent[i]) > Real(0))) throw ConfigError("box extent must be positive");
    const int kind = s.kind, npe = npe_of(kind), per_cell = kind == DJG_T4 ? 6 : 1;
    const int32_t* div = s.divisions;
    const int64_t nx = div[0], ny = div[1], nz = div[2];
    const int64_t N = (nx + 1) * (ny + 1) * (nz + 1), cells = nx * ny * nz;
    if (int64_t(npe) * cells * per_cell > INT32_MAX || N > INT32_MAX) throw ConfigError("box too large for int32 ids");
    const auto blocks = box_blocks(div, nparts);
    const CellBlock& B = blocks[size_t(part)];
    auto node_ijk = [&](int64_t n, int64_t& i, int64_t& j, int64_t& k) {
        i = n % (nx + 1);
        j = (n / (nx + 1)) % (ny + 1);
        k = n / ((nx + 1) * (ny + 1));
    };
    auto owner = [&](int64_t n) {
        int64_t i, j, k;
        node_ijk(n, i, j, k);
        return box_part_of_cell(blocks, std::max<int64_t>(i - 1, 0), std::max<int64_t>(j - 1, 0),
                                std::max<int64_t>(k - 1, 0));
    };
    // owned node ranges per axis (inclusive): max(i-1, 0) in [lo, hi)
    int64_t a0[3], a1[3];
    for (int ax = 0; ax < 3; ++ax) {
        a0[ax] = B.lo[ax] == 0 ? 0 : B.lo[ax] + 1;
        a1[ax] = B.hi[ax];
    }
    PartProblem<Real> R;
    R.nparts = nparts;
    R.part = part;
    R.global_nodes = N;
    R.global_elements = cells * per_cell;
    for (int64_t k = a0[2]; k <= a1[2]; ++k)
        for (int64_t j = a0[1]; j <= a1[1]; ++j)
            for (int64_t i = a0[0]; i <= a1[0]; ++i) R.node_l2g.push_back(i + (nx + 1) * (j + (ny + 1) * k));
    R.num_owned = int64_t(R.node_l2g.size());
    auto is_owned = [&](int64_t n) {
        int64_t i, j, k;
        node_ijk(n, i, j, k);
        return i >= a0[0] && i <= a1[0] && j >= a0[1] && j <= a1[1] && k >= a0[2] && k <= a1[2];
    };
    // candidate cells: the part's block grown by one cell on the low sides
    int64_t c0[3], c1[3];
    for (int ax = 0; ax < 3; ++ax) {
        c0[ax] = std::max<int64_t>(a0[ax] - 1, 0);
        c1[ax] = std::min<int64_t>(a1[ax], int64_t(div[ax]) - 1);
    }
    std::vector<int64_t> interior, boundary;  // global element ids, ascending
    std::vector<int32_t> gconn;               // global connectivity of the local elements, by global id
    std::vector<int64_t> order;               // global ids in ascending order (parallel to gconn)
    std::vector<int32_t> ghosts;
    {
        // one cell layer (ck) per work item, concatenated in ck order: the
        // element ids stay ascending
        const int64_t nk = c1[2] - c0[2] + 1;
        struct Layer {
            std::vector<int64_t> interior, boundary, order;
            std::vector<int32_t> gconn, ghosts;
        };
        std::vector<Layer> layers(static_cast<size_t>(std::max<int64_t>(nk, 0)));
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t l = 0; l < nk; ++l) {
            const int64_t ck = c0[2] + l;
            Layer& Ly = layers[size_t(l)];
            int32_t cc[24];
            for (int64_t cj = c0[1]; cj <= c1[1]; ++cj)
                for (int64_t ci = c0[0]; ci <= c1[0]; ++ci) {
                    const int64_t c = ci + nx * (cj + ny * ck);
                    box_cell_conn(kind, div, c, cc);
                    for (int t = 0; t < per_cell; ++t) {
                        bool touches = false, ghost = false;
                        for (int a = 0; a < npe; ++a) {
                            const bool o = is_owned(cc[t * npe + a]);
                            touches |= o;
                            ghost |= !o;
                        }
                        if (!touches) continue;
                        const int64_t e = c * per_cell + t;
                        Ly.order.push_back(e);
                        Ly.gconn.insert(Ly.gconn.end(), cc + t * npe, cc + (t + 1) * npe);
                        (ghost ? Ly.boundary : Ly.interior).push_back(e);
                        if (ghost)
                            for (int a = 0; a < npe; ++a)
                                if (!is_owned(cc[t * npe + a])) Ly.ghosts.push_back(cc[t * npe + a]);
                    }
                }
        }
        size_t ni = 0, nb = 0, no = 0, ng = 0;
        for (const Layer& Ly : layers) {
            ni += Ly.interior.size();
            nb += Ly.boundary.size();
            no += Ly.order.size();
            ng += Ly.ghosts.size();
        }
        interior.reserve(ni);
        boundary.reserve(nb);
        order.reserve(no);
        gconn.reserve(no * size_t(npe));
        ghosts.reserve(ng);
        for (Layer& Ly : layers) {
            interior.insert(interior.end(), Ly.interior.begin(), Ly.interior.end());
            boundary.insert(boundary.end(), Ly.boundary.begin(), Ly.boundary.end());
            order.insert(order.end(), Ly.order.begin(), Ly.order.end());
            gconn.insert(gconn.end(), Ly.gconn.begin(), Ly.gconn.end());
            ghosts.insert(ghosts.end(), Ly.ghosts.begin(), Ly.ghosts.end());
            Ly = Layer{};
        }
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    R.node_l2g.insert(R.node_l2g.end(), ghosts.begin(), ghosts.end());
    R.interior_elements = int64_t(interior.size());
    R.elem_l2g = std::move(interior);
    R.elem_l2g.insert(R.elem_l2g.end(), boundary.begin(), boundary.end());
    const int64_t Nl = int64_t(R.node_l2g.size()), El = int64_t(R.elem_l2g.size());
    R.elem_owned.resize(size_t(El));
    for (int64_t q = 0; q < El; ++q) {
        const int64_t c = R.elem_l2g[size_t(q)] / per_cell;
        R.elem_owned[size_t(q)] = box_part_of_cell(blocks, c % nx, (c / nx) % ny, c / (nx * ny)) == part;
        R.owned_elements += R.elem_owned[size_t(q)];
    }
    // global -> local node ids: owned nodes form a block; ghosts by search
    const int64_t bx = a1[0] - a0[0] + 1, by = a1[1] - a0[1] + 1;
    auto g2l = [&](int64_t n) -> int32_t {
        int64_t i, j, k;
        node_ijk(n, i, j, k);
        if (is_owned(n)) return int32_t((i - a0[0]) + bx * ((j - a0[1]) + by * (k - a0[2])));
        return int32_t(R.num_owned + (std::lower_bound(ghosts.begin(), ghosts.end(), int32_t(n)) - ghosts.begin()));
    };
    // local problem
    Problem<Real>& L = R.local;
    L.policy = s.policy;
    L.mat = Material<Real>::from(s.material);
    L.mesh.kind = kind;
    L.mesh.nodes.resize(size_t(3 * Nl));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < Nl; ++q) {
        int64_t i, j, k;
        node_ijk(R.node_l2g[size_t(q)], i, j, k);
        L.mesh.nodes[size_t(3 * q + 0)] = box_coord<Real>(s.extent[0], i, nx);
        L.mesh.nodes[size_t(3 * q + 1)] = box_coord<Real>(s.extent[1], j, ny);
        L.mesh.nodes[size_t(3 * q + 2)] = box_coord<Real>(s.extent[2], k, nz);
    }
    L.mesh.conn.resize(size_t(El * npe));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < El; ++q) {
        const int64_t pos = std::lower_bound(order.begin(), order.end(), R.elem_l2g[size_t(q)]) - order.begin();
        for (int a = 0; a < npe; ++a) L.mesh.conn[size_t(q * npe + a)] = g2l(gconn[size_t(pos * npe + a)]);
    }
    std::vector<int32_t>().swap(gconn);  // (peak host memory: the global-id copies go before the records)
    std::vector<int64_t>().swap(order);
    const ConstLayout CL(kind, L.mat.model);
    L.nconst = CL.count;
    V3<Real> fa{0, 0, 0}, fb{0, 0, 0};
    if (L.mat.needs_fibre_a()) fa = Material<Real>::unit(L.mat.fa);
    if (L.mat.needs_fibre_b()) fb = Material<Real>::unit(L.mat.fb);
    L.c_hg = Real(s.c_hg);
    const Shape<Real> D(kind);
    L.consts.assign(size_t(El) * size_t(CL.count), Real(0));
    int64_t bad = -1;
    Real lmin = std::numeric_limits<Real>::max();
#pragma omp parallel reduction(max : bad)
    {
        Real lm = std::numeric_limits<Real>::max();
#pragma omp for schedule(static) nowait
        for (int64_t q = 0; q < El; ++q) {
            V3<Real> x[8];
            for (int a = 0; a < npe; ++a) x[a] = L.mesh.node(L.mesh.conn[size_t(q * npe + a)]);
            Real* rec = L.consts.data() + size_t(q) * CL.count;
            if (!element_record(x, D, L.mat, fa, fb, L.c_hg, CL, rec)) {
                bad = std::max<int64_t>(bad, R.global_elements - R.elem_l2g[size_t(q)]);
                continue;
            }
            lm = std::min(lm, char_length(x, kind, rec[CL.V0]));
        }
#pragma omp critical
        lmin = std::min(lmin, lm);
    }
    if (bad >= 0) throw MeshError("non-positive reference Jacobian determinant", long(R.global_elements - bad));
    local_lmin = lmin;
    L.adj = local_adjacency(L.mesh.conn, Nl, npe, R.elem_l2g);
    // lump_mass: owned nodes hold all their elements (ascending global id);
    // ghost masses are partial and never used (only owned nodes are updated)
    L.mass.assign(size_t(Nl), Real(0));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < Nl; ++q) {
        Real acc = Real(0);
        for (int64_t p = L.adj.offsets[size_t(q)]; p < L.adj.offsets[size_t(q + 1)]; ++p)
            acc += L.mat.rho * L.consts[size_t(L.adj.elem[size_t(p)]) * CL.count + CL.V0] / Real(npe);
        L.mass[size_t(q)] = acc;
    }
    // halo: recv = my ghosts grouped by owner; send = my owned nodes that
    // another part's elements touch (the elements around the node)
    std::vector<std::vector<int32_t>> recv(static_cast<size_t>(nparts)), send(static_cast<size_t>(nparts));
    for (int64_t q = R.num_owned; q < Nl; ++q) recv[size_t(owner(R.node_l2g[size_t(q)]))].push_back(int32_t(q));
    std::vector<std::vector<int32_t>> need(static_cast<size_t>(R.num_owned));
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t q = 0; q < R.num_owned; ++q) {
        const int64_t n = R.node_l2g[size_t(q)];
        int64_t i, j, k;
        node_ijk(n, i, j, k);
        // interior of the owned block: every neighbour is owned here
        if (i > a0[0] && i < a1[0] && j > a0[1] && j < a1[1] && k > a0[2] && k < a1[2]) continue;
        int32_t cc[24];
        std::vector<int32_t> parts;
        for (int64_t ck = std::max<int64_t>(k - 1, 0); ck <= std::min<int64_t>(k, nz - 1); ++ck)
            for (int64_t cj = std::max<int64_t>(j - 1, 0); cj <= std::min<int64_t>(j, ny - 1); ++cj)
                for (int64_t ci = std::max<int64_t>(i - 1, 0); ci <= std::min<int64_t>(i, nx - 1); ++ci) {
                    box_cell_conn(kind, div, ci + nx * (cj + ny * ck), cc);
                    for (int t = 0; t < per_cell; ++t) {
                        const int32_t* ec = cc + t * npe;
                        if (std::find(ec, ec + npe, int32_t(n)) == ec + npe) continue;
                        for (int a = 0; a < npe; ++a) {
                            const int o = owner(ec[a]);
                            if (o != part) parts.push_back(o);
                        }
                    }
                }
        std::sort(parts.begin(), parts.end());
        parts.erase(std::unique(parts.begin(), parts.end()), parts.end());
        need[size_t(q)] = std::move(parts);
    }
    for (int64_t q = 0; q < R.num_owned; ++q)
        for (int32_t o : need[size_t(q)]) send[size_t(o)].push_back(int32_t(q));
    R.halo.send_off.push_back(0);
    R.halo.recv_off.push_back(0);
    for (int q = 0; q < nparts; ++q) {
        if (q == part || (send[size_t(q)].empty() && recv[size_t(q)].empty())) continue;
        R.halo.neighbors.push_back(q);
        R.halo.send_nodes.insert(R.halo.send_nodes.end(), send[size_t(q)].begin(), send[size_t(q)].end());
        R.halo.recv_nodes.insert(R.halo.recv_nodes.end(), recv[size_t(q)].begin(), recv[size_t(q)].end());
        R.halo.send_off.push_back(int64_t(R.halo.send_nodes.size()));
        R.halo.recv_off.push_back(int64_t(R.halo.recv_nodes.size()));
    }
    return R;
}

// Time-step data of a part-local box (build_problem's, from the GLOBAL
// minimum characteristic length `lmin`): critical dt, dt, relaxation alpha
// (the box's bounding box: its coordinates at 0 and at the last division),
// the zmin / zmax plane BCs (the same predicate as plane_nodes) and the
// update coefficients.
template <class Real>
inline void finish_box_part(PartProblem<Real>& R, const djg_scenario_spec& s, Real lmin) {
    Problem<Real>& P = R.local;
    if (!(lmin > Real(0))) throw MeshError("degenerate element with zero characteristic length");
    P.c_wave = wave_speed(P.mat);
    P.crit_dt = lmin / P.c_wave;
    P.dt = s.dt > 0 ? Real(s.dt) : Real(s.safety) * P.crit_dt;
    if (!(P.dt > Real(0))) throw ConfigError("time step must be positive");
    Real lo[3], hi[3];
    for (int ax = 0; ax < 3; ++ax) {
        lo[ax] = box_coord<Real>(s.extent[ax], 0, s.divisions[ax]);
        hi[ax] = box_coord<Real>(s.extent[ax], s.divisions[ax], s.divisions[ax]);
    }
    if (s.alpha_mode == 0) {
        const Real mu = P.mat.shear_modulus();
        const Real e_mod = 9 * P.mat.kappa * mu / (3 * P.mat.kappa + mu);
        const Real c_bar = std::sqrt(e_mod / P.mat.rho);
        const Real l = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
        if (!(l > Real(0))) throw ConfigError("mesh has zero extent");
        P.alpha = Real(M_PI) * c_bar / l;
    } else {
        P.alpha = Real(s.alpha);
    }
    const int64_t Nl = P.mesh.num_nodes();
    P.dof_kind.assign(size_t(3 * Nl), uint8_t(DJG_FREE));
    P.dof_target.assign(size_t(3 * Nl), Real(0));
    P.dof_t_total.assign(size_t(3 * Nl), Real(1));
    P.ramp_t_total = 0;
    if (s.bc_mode == 1) {
        const auto bottom = plane_nodes(P.mesh, 2, false, lo, hi);
        const auto top = plane_nodes(P.mesh, 2, true, lo, hi);
        for (int32_t n : bottom) {
            if (s.fix_all_axes) {
                P.dof_kind[size_t(3 * n + 0)] = DJG_FIXED;
                P.dof_kind[size_t(3 * n + 1)] = DJG_FIXED;
            }
            P.dof_kind[size_t(3 * n + 2)] = DJG_FIXED;
        }
        P.ramp_t_total = P.dt * Real(s.ramp_steps);
        if (!(P.ramp_t_total > Real(0))) throw ConfigError("ramp duration must be positive");
        for (int32_t n : top) {
            if (P.dof_kind[size_t(3 * n + 2)] != DJG_FREE)
                throw ConfigError("node axis 2 appears in more than one boundary condition");
            P.dof_kind[size_t(3 * n + 2)] = DJG_PRESCRIBED;
            P.dof_target[size_t(3 * n + 2)] = Real(s.target);
            P.dof_t_total[size_t(3 * n + 2)] = P.ramp_t_total;
        }
    }
    const Real denom = Real(1) + P.alpha * P.dt / 2;
    P.c2 = Real(2) / denom;
    P.c3 = -(Real(1) - P.alpha * P.dt / 2) / denom;
    P.c1.assign(size_t(Nl), Real(0));
    P.massless.assign(size_t(Nl), 0);
    for (int64_t n = 0; n < Nl; ++n) {
        if (P.mass[size_t(n)] > Real(0))
            P.c1[size_t(n)] = P.dt * P.dt / (P.mass[size_t(n)] * denom);
        else
            P.massless[size_t(n)] = 1;
    }
}

}  // namespace djg
