// Element-level precompute arithmetic shared by the host builder (g++,
// -ffp-contract=off) and the device kernels (nvcc, --fmad=false): one source
// for every operation, so a record built on the host, built on the device,
// or rebuilt in registers by the compact force kernel is the same bits.
// Each function follows the reference expression order (file:line under
// /root/reference/proj/include/djtled/).
#pragma once

#include <cmath>

#if defined(__CUDACC__)
#define DJG_HD __host__ __device__ __forceinline__
#define DJG_UNROLL _Pragma("unroll")
#else
#define DJG_HD inline
#define DJG_UNROLL
#endif

namespace djg {
namespace em {

// Correctly rounded square root in the argument's precision on both sides.
DJG_HD float sqrt_rn(float x) { return std::sqrt(x); }
DJG_HD double sqrt_rn(double x) { return std::sqrt(x); }

// H8 natural corner signs (element.hpp:17-20).
DJG_HD int corner_sign(int a, int i) {
    // a: bits (x, y) follow the counter-clockwise face order, z = a >= 4
    const int sx[8] = {-1, +1, +1, -1, -1, +1, +1, -1};
    const int sy[8] = {-1, -1, +1, +1, -1, -1, +1, +1};
    return i == 0 ? sx[a] : (i == 1 ? sy[a] : (a < 4 ? -1 : 1));
}

// shape_derivatives (element.hpp:31-47): d[i][a] = dh_a / dxi_i.
template <class R>
DJG_HD R shape_d(int kind, int i, int a) {
    if (kind == 0) return a == 0 ? R(-1) : (a == i + 1 ? R(1) : R(0));
    return R(corner_sign(a, i)) / R(8);
}

// det (core.hpp:187-192)
template <class R>
DJG_HD R det3(const R a[3][3]) {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

// inverse via adjugate (core.hpp:198-212)
template <class R>
DJG_HD void inv3(const R a[3][3], R d, R r[3][3]) {
    const R s = R(1) / d;
    r[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) * s;
    r[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) * s;
    r[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) * s;
    r[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) * s;
    r[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) * s;
    r[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) * s;
    r[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) * s;
    r[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) * s;
    r[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) * s;
}

// Q^T S Q for symmetric S in (xx,yy,zz,xy,xz,yz) order (core.hpp:259-271).
template <class R>
DJG_HD void congruence(const R q[3][3], const R s[6], R out[6]) {
    const R sf[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    R sq[3][3];
    DJG_UNROLL
    for (int i = 0; i < 3; ++i)
        DJG_UNROLL
        for (int j = 0; j < 3; ++j) sq[i][j] = sf[i][0] * q[0][j] + sf[i][1] * q[1][j] + sf[i][2] * q[2][j];
    out[0] = q[0][0] * sq[0][0] + q[1][0] * sq[1][0] + q[2][0] * sq[2][0];
    out[1] = q[0][1] * sq[0][1] + q[1][1] * sq[1][1] + q[2][1] * sq[2][1];
    out[2] = q[0][2] * sq[0][2] + q[1][2] * sq[1][2] + q[2][2] * sq[2][2];
    out[3] = q[0][0] * sq[0][1] + q[1][0] * sq[1][1] + q[2][0] * sq[2][1];
    out[4] = q[0][0] * sq[0][2] + q[1][0] * sq[1][2] + q[2][0] * sq[2][2];
    out[5] = q[0][1] * sq[0][2] + q[1][1] * sq[1][2] + q[2][1] * sq[2][2];
}

// Frobenius product of symmetric matrices (core.hpp:277-280).
template <class R>
DJG_HD R ddot(const R a[6], const R b[6]) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + 2 * (a[3] * b[3] + a[4] * b[4] + a[5] * b[5]);
}

// G_k = outer / sym_outer of the columns of J0inv (precompute.hpp:45-50; core.hpp:240-251).
template <class R>
DJG_HD void g_matrix(const R ji[3][3], int k, R g[6]) {
    if (k < 3) {
        const R x = ji[0][k], y = ji[1][k], z = ji[2][k];
        g[0] = x * x; g[1] = y * y; g[2] = z * z; g[3] = x * y; g[4] = x * z; g[5] = y * z;
        return;
    }
    const int p = k == 5 ? 1 : 0, q = k == 3 ? 1 : 2;
    const R ux = ji[0][p], uy = ji[1][p], uz = ji[2][p];
    const R vx = ji[0][q], vy = ji[1][q], vz = ji[2][q];
    g[0] = 2 * ux * vx; g[1] = 2 * uy * vy; g[2] = 2 * uz * vz;
    g[3] = ux * vy + uy * vx; g[4] = ux * vz + uz * vx; g[5] = uy * vz + uz * vy;
}

template <class R>
DJG_HD R trace6(const R g[6]) { return g[0] + g[1] + g[2]; }

// m1[k] = tr(G_k) and I1m = 2 V0 J0inv^T J0inv (precompute.hpp:52-58, 97-101, 224-225).
template <class R>
DJG_HD void first_invariant_tensors(const R ji[3][3], R v0, R m1[6], R i1m[6]) {
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {
        R g[6];
        g_matrix(ji, k, g);
        m1[k] = trace6(g);
    }
    const R ident[6] = {R(1), R(1), R(1), R(0), R(0), R(0)};
    R t[6];
    congruence(ji, ident, t);
    const R two_v0 = 2 * v0;
    DJG_UNROLL
    for (int c = 0; c < 6; ++c) i1m[c] = two_v0 * t[c];
}

// Same tensors with I1m taken from m1: I1m_ij = 2 V0 (q_i . q_j) (the
// congruence with the identity) and m1 = tr(G_k) evaluate the same products
// in the same order, the off-diagonal traces carrying an exact factor 2, so
// I1m = (2V0 m1[0..2], V0 m1[3..5]) bit for bit (up to the sign of an exact
// zero). Used by the compact force kernel, where it saves ~80 operations.
template <class R>
DJG_HD void first_invariant_tensors_fast(const R ji[3][3], R v0, R m1[6], R i1m[6]) {
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {
        R g[6];
        g_matrix(ji, k, g);
        m1[k] = trace6(g);
    }
    const R two_v0 = 2 * v0;
    DJG_UNROLL
    for (int c = 0; c < 3; ++c) i1m[c] = two_v0 * m1[c];
    DJG_UNROLL
    for (int c = 3; c < 6; ++c) i1m[c] = v0 * m1[c];
}

// Fibre family: m[k] = tr(S G_k), Im = 2 V0 J0inv^T S J0inv (precompute.hpp:60-65, 97-101).
template <class R>
DJG_HD void fibre_tensors(const R ji[3][3], R v0, const R S[6], R m[6], R im[6]) {
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {
        R g[6];
        g_matrix(ji, k, g);
        m[k] = ddot(S, g);
    }
    R t[6];
    congruence(ji, S, t);
    const R two_v0 = 2 * v0;
    DJG_UNROLL
    for (int c = 0; c < 6; ++c) im[c] = two_v0 * t[c];
}

// M2 = (m1 m1^T - W) / 2 packed upper (precompute.hpp:67-84) and
// I2m_k = 2 V0 J0inv^T (tr(G_k) I - G_k) J0inv (precompute.hpp:104-115).
template <class R>
DJG_HD void second_invariant_tensors(const R ji[3][3], R v0, const R m1[6], R m2[21], R i2m[36]) {
    int w = 0;
    DJG_UNROLL
    for (int p = 0; p < 6; ++p) {
        R gp[6];
        g_matrix(ji, p, gp);
        DJG_UNROLL
        for (int q = p; q < 6; ++q) {
            R gq[6];
            g_matrix(ji, q, gq);
            m2[w++] = (m1[p] * m1[q] - ddot(gp, gq)) / 2;
        }
    }
    const R two_v0 = 2 * v0;
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {
        R g[6];
        g_matrix(ji, k, g);
        const R tr = trace6(g);
        const R ker[6] = {tr - g[0], tr - g[1], tr - g[2], -g[3], -g[4], -g[5]};
        R t[6];
        congruence(ji, ker, t);
        DJG_UNROLL
        for (int c = 0; c < 6; ++c) i2m[6 * k + c] = two_v0 * t[c];
    }
}

// Fibre second-order family for a unit fibre s, S = s s^T (precompute.hpp:
// 86-95, 117-131): M[p][q] = (G_p s) . (G_q s) packed upper, and
// Im_k = 2 V0 J0inv^T (S G_k + G_k S) J0inv. Used by I5 (a, A) and I7 (b, B).
template <class R>
DJG_HD void fibre_second_tensors(const R ji[3][3], R v0, const R s[3], const R S[6], R m[21], R im[36]) {
    R gs[6][3];
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {  // mul(G_k.full(), s)
        R g[6];
        g_matrix(ji, k, g);
        gs[k][0] = g[0] * s[0] + g[3] * s[1] + g[4] * s[2];
        gs[k][1] = g[3] * s[0] + g[1] * s[1] + g[5] * s[2];
        gs[k][2] = g[4] * s[0] + g[5] * s[1] + g[2] * s[2];
    }
    int w = 0;
    DJG_UNROLL
    for (int p = 0; p < 6; ++p)
        DJG_UNROLL
        for (int q = p; q < 6; ++q) m[w++] = gs[p][0] * gs[q][0] + gs[p][1] * gs[q][1] + gs[p][2] * gs[q][2];
    const R sf[3][3] = {{S[0], S[3], S[4]}, {S[3], S[1], S[5]}, {S[4], S[5], S[2]}};
    const R two_v0 = 2 * v0;
    DJG_UNROLL
    for (int k = 0; k < 6; ++k) {
        R g[6];
        g_matrix(ji, k, g);
        const R gf[3][3] = {{g[0], g[3], g[4]}, {g[3], g[1], g[5]}, {g[4], g[5], g[2]}};
        R sg[3][3];  // mul(S.full(), G_k.full())
        DJG_UNROLL
        for (int i = 0; i < 3; ++i)
            DJG_UNROLL
            for (int j = 0; j < 3; ++j) sg[i][j] = sf[i][0] * gf[0][j] + sf[i][1] * gf[1][j] + sf[i][2] * gf[2][j];
        const R ker[6] = {2 * sg[0][0], 2 * sg[1][1], 2 * sg[2][2],
                          sg[0][1] + sg[1][0], sg[0][2] + sg[2][0], sg[1][2] + sg[2][1]};
        R t[6];
        congruence(ji, ker, t);
        DJG_UNROLL
        for (int c = 0; c < 6; ++c) im[6 * k + c] = two_v0 * t[c];
    }
}

// Hourglass shape vectors (precompute.hpp:136-165).
template <class R>
DJG_HD void hourglass_vectors(const R x[8][3], const R ji[3][3], R gamma[4][8]) {
    R b[3][8];
    DJG_UNROLL
    for (int j = 0; j < 3; ++j)
        DJG_UNROLL
        for (int a = 0; a < 8; ++a)
            b[j][a] = ji[j][0] * shape_d<R>(1, 0, a) + ji[j][1] * shape_d<R>(1, 1, a) + ji[j][2] * shape_d<R>(1, 2, a);
    DJG_UNROLL
    for (int m = 0; m < 4; ++m) {
        R base[8];
        DJG_UNROLL
        for (int a = 0; a < 8; ++a) {
            const int xi = corner_sign(a, 0), eta = corner_sign(a, 1), zeta = corner_sign(a, 2);
            base[a] = R(m == 0 ? eta * zeta : (m == 1 ? xi * zeta : (m == 2 ? xi * eta : xi * eta * zeta)));
        }
        R hx[3] = {R(0), R(0), R(0)};
        DJG_UNROLL
        for (int j = 0; j < 3; ++j)
            DJG_UNROLL
            for (int a = 0; a < 8; ++a) hx[j] += base[a] * x[a][j];
        DJG_UNROLL
        for (int a = 0; a < 8; ++a) gamma[m][a] = base[a] - (hx[0] * b[0][a] + hx[1] * b[1][a] + hx[2] * b[2][a]);
    }
}

// jacobian0 (element.hpp:59-77): J = D X; false if det <= 0.
template <class R>
DJG_HD bool jacobian0(int kind, const R x[8][3], R J[3][3], R Ji[3][3], R& det) {
    const int n = kind == 0 ? 4 : 8;
    DJG_UNROLL
    for (int i = 0; i < 3; ++i) {
        R r0 = R(0), r1 = R(0), r2 = R(0);
        DJG_UNROLL
        for (int a = 0; a < n; ++a) {
            const R d = shape_d<R>(kind, i, a);
            r0 = r0 + d * x[a][0];
            r1 = r1 + d * x[a][1];
            r2 = r2 + d * x[a][2];
        }
        J[i][0] = r0;
        J[i][1] = r1;
        J[i][2] = r2;
    }
    det = det3(J);
    if (!(det > R(0))) return false;
    inv3(J, det, Ji);
    return true;
}

// volume0 (element.hpp:80-85)
template <class R>
DJG_HD R volume0(int kind, R det) {
    return kind == 0 ? det / R(6) : R(8) * det;
}

// triangle_area / characteristic_length (precompute.hpp:290-319): the largest
// face area (H8: quads as two triangles), l = 3 V0 / a_max (T4), V0 / a_max (H8).
template <class R>
DJG_HD R tri_area(const R a[3], const R b[3], const R c[3]) {
    const R u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const R w[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    return sqrt_rn(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]) / 2;
}

template <class R>
DJG_HD R char_length(int kind, const R x[8][3], R v0) {
    R a_max = 0;
    if (kind == 0) {
        constexpr int f[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        DJG_UNROLL
        for (int t = 0; t < 4; ++t) {
            const R a = tri_area(x[f[t][0]], x[f[t][1]], x[f[t][2]]);
            a_max = a_max < a ? a : a_max;  // std::max(a_max, a)
        }
        return 3 * v0 / a_max;
    }
    constexpr int f[6][4] = {{0, 3, 2, 1}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
    DJG_UNROLL
    for (int q = 0; q < 6; ++q) {
        const R a = tri_area(x[f[q][0]], x[f[q][1]], x[f[q][2]]) + tri_area(x[f[q][0]], x[f[q][2]], x[f[q][3]]);
        a_max = a_max < a ? a : a_max;
    }
    return v0 / a_max;
}

// TledModel::build record (tled_force.hpp:176-192): B0[a][j] = dh_a/dx_j at the
// reference configuration, V0 -> out[3*npe], out[3*npe + 1] (the hourglass
// data, H8, is appended by the caller exactly as for the DJ record).
template <class R>
DJG_HD void tled_b0(int kind, const R ji[3][3], R* b0) {
    const int n = kind == 0 ? 4 : 8;
    DJG_UNROLL
    for (int a = 0; a < n; ++a)
        DJG_UNROLL
        for (int j = 0; j < 3; ++j)
            b0[3 * a + j] = ji[j][0] * shape_d<R>(kind, 0, a) + ji[j][1] * shape_d<R>(kind, 1, a) +
                            ji[j][2] * shape_d<R>(kind, 2, a);
}

// unit fibre direction (FibreDirections::normalise, precompute.hpp:35-39)
template <class R>
DJG_HD void unit3(const R a[3], R u[3]) {
    const R n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const R s = R(1) / n;
    u[0] = s * a[0];
    u[1] = s * a[1];
    u[2] = s * a[2];
}

// FibreDirections::from: S = a' a'^T with a' = a / |a| (precompute.hpp:22-39).
template <class R>
DJG_HD void fibre_structure(const R a[3], R S[6]) {
    const R n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const R s = R(1) / n;
    const R x = s * a[0], y = s * a[1], z = s * a[2];
    S[0] = x * x; S[1] = y * y; S[2] = z * z; S[3] = x * y; S[4] = x * z; S[5] = y * z;
}

}  // namespace em
}  // namespace djg
