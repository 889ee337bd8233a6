/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Included twice by
 * djtled_oracle.c with R = float / double and FN() adding a _f / _d suffix.
 *
 * A plain-C restatement of the reference algorithm for the hot path and the
 * host steps that produce its inputs. Every function cites the reference
 * file:line it restates (paths under /root/reference/proj/include/djtled/).
 * Expressions keep the reference's evaluation order so results are
 * bit-identical to the reference (pinned by tests/test_oracle.py against
 * oracle/_ref and tests/golden/).
 */

/* ---------------------------------------------------------------- algebra */

/* det (core.hpp:187-192) */
static R FN(det3)(const R a[3][3]) {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
           a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

/* inverse via adjugate (core.hpp:198-212) */
static void FN(inv3)(const R a[3][3], R d, R r[3][3]) {
    const R s = (R)1 / d;
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

/* Q^T S Q for symmetric S in (xx,yy,zz,xy,xz,yz) order (core.hpp:259-271) */
static void FN(congruence)(const R q[3][3], const R s[6], R out[6]) {
    const R sf[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    R sq[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sq[i][j] = sf[i][0] * q[0][j] + sf[i][1] * q[1][j] + sf[i][2] * q[2][j];
    out[0] = q[0][0] * sq[0][0] + q[1][0] * sq[1][0] + q[2][0] * sq[2][0];
    out[1] = q[0][1] * sq[0][1] + q[1][1] * sq[1][1] + q[2][1] * sq[2][1];
    out[2] = q[0][2] * sq[0][2] + q[1][2] * sq[1][2] + q[2][2] * sq[2][2];
    out[3] = q[0][0] * sq[0][1] + q[1][0] * sq[1][1] + q[2][0] * sq[2][1];
    out[4] = q[0][0] * sq[0][2] + q[1][0] * sq[1][2] + q[2][0] * sq[2][2];
    out[5] = q[0][1] * sq[0][2] + q[1][1] * sq[1][2] + q[2][1] * sq[2][2];
}

/* Frobenius product of symmetric matrices (core.hpp:277-280) */
static R FN(ddot)(const R a[6], const R b[6]) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + 2 * (a[3] * b[3] + a[4] * b[4] + a[5] * b[5]);
}

/* Sym6::quadratic_form g^T M g over the packed upper triangle (core.hpp:296-304) */
static R FN(quadform)(const R* p, const R g[6]) {
    R q = 0;
    for (int i = 0; i < 6; ++i) {
        R row = p[sym6_index(i, i)] * g[i];
        for (int j = i + 1; j < 6; ++j) row += 2 * p[sym6_index(i, j)] * g[j];
        q += row * g[i];
    }
    return q;
}

/* ---------------------------------------------------------------- element */

/* shape_derivatives (element.hpp:31-47) */
static void FN(shape)(int kind, R d[3][8]) {
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 8; ++a) d[i][a] = 0;
    if (kind == DJG_T4) {
        for (int i = 0; i < 3; ++i) {
            d[i][0] = -1;
            d[i][i + 1] = 1;
        }
    } else {
        for (int a = 0; a < 8; ++a)
            for (int i = 0; i < 3; ++i) d[i][a] = (R)corner_sign[a][i] / (R)8;
    }
}

/* jacobian0 (element.hpp:59-77): J = D X; returns 0 if det <= 0 */
static int FN(jacobian0)(const R x[8][3], const R d[3][8], int n, R J[3][3], R Jinv[3][3], R* det) {
    for (int i = 0; i < 3; ++i) {
        R r0 = 0, r1 = 0, r2 = 0;
        for (int a = 0; a < n; ++a) {
            r0 = r0 + d[i][a] * x[a][0];
            r1 = r1 + d[i][a] * x[a][1];
            r2 = r2 + d[i][a] * x[a][2];
        }
        J[i][0] = r0;
        J[i][1] = r1;
        J[i][2] = r2;
    }
    *det = FN(det3)(J);
    if (!(*det > 0)) return 0;
    FN(inv3)(J, *det, Jinv);
    return 1;
}

/* hourglass_vectors (precompute.hpp:136-165) */
static void FN(hourglass_vectors)(const R x[8][3], const R d[3][8], const R jinv[3][3], R gamma[4][8]) {
    R base[4][8], b[3][8];
    for (int a = 0; a < 8; ++a) {
        const int xi = corner_sign[a][0], eta = corner_sign[a][1], zeta = corner_sign[a][2];
        base[0][a] = (R)(eta * zeta);
        base[1][a] = (R)(xi * zeta);
        base[2][a] = (R)(xi * eta);
        base[3][a] = (R)(xi * eta * zeta);
    }
    for (int j = 0; j < 3; ++j)
        for (int a = 0; a < 8; ++a) b[j][a] = jinv[j][0] * d[0][a] + jinv[j][1] * d[1][a] + jinv[j][2] * d[2][a];
    for (int m = 0; m < 4; ++m) {
        R hx[3] = {0, 0, 0};
        for (int j = 0; j < 3; ++j)
            for (int a = 0; a < 8; ++a) hx[j] += base[m][a] * x[a][j];
        for (int a = 0; a < 8; ++a) gamma[m][a] = base[m][a] - (hx[0] * b[0][a] + hx[1] * b[1][a] + hx[2] * b[2][a]);
    }
}

/* Unit fibre (FibreDirections::normalise, precompute.hpp:35-39) into u and
 * A = a a^T */
static void FN(fibre_tensor)(const double v[3], R A[6], R u[3]) {
    const R a0 = (R)v[0], a1 = (R)v[1], a2 = (R)v[2];
    const R n = SQRT(a0 * a0 + a1 * a1 + a2 * a2);
    const R s = (R)1 / n;
    const R u0 = s * a0, u1 = s * a1, u2 = s * a2;
    u[0] = u0; u[1] = u1; u[2] = u2;
    A[0] = u0 * u0; A[1] = u1 * u1; A[2] = u2 * u2;
    A[3] = u0 * u1; A[4] = u0 * u2; A[5] = u1 * u2;
}

/* trace_matrix(G, s) (precompute.hpp:86-95): M[p][q] = (G_p s) . (G_q s),
 * packed upper; second_order_tensors(J0inv, V0, G, S) (precompute.hpp:
 * 117-131): 2 V0 J0inv^T (S G_k + G_k S) J0inv. The I5 (a) / I7 (b) blocks. */
static void FN(fibre_second_order)(R G[6][6], const R Ji[3][3], R two_v0, const R u[3], const R S[6], R* M,
                                   R* Im) {
    R gs[6][3];
    for (int k = 0; k < 6; ++k) {
        const R* g = G[k]; /* full(): [[xx,xy,xz],[xy,yy,yz],[xz,yz,zz]] */
        gs[k][0] = g[0] * u[0] + g[3] * u[1] + g[4] * u[2];
        gs[k][1] = g[3] * u[0] + g[1] * u[1] + g[5] * u[2];
        gs[k][2] = g[4] * u[0] + g[5] * u[1] + g[2] * u[2];
    }
    for (int p = 0; p < 6; ++p)
        for (int q = p; q < 6; ++q) M[sym6_index(p, q)] = gs[p][0] * gs[q][0] + gs[p][1] * gs[q][1] + gs[p][2] * gs[q][2];
    const R Sf[3][3] = {{S[0], S[3], S[4]}, {S[3], S[1], S[5]}, {S[4], S[5], S[2]}};
    for (int k = 0; k < 6; ++k) {
        const R* g = G[k];
        const R Gf[3][3] = {{g[0], g[3], g[4]}, {g[3], g[1], g[5]}, {g[4], g[5], g[2]}};
        R P[3][3]; /* mul(S.full(), G_k.full()) */
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) P[i][j] = Sf[i][0] * Gf[0][j] + Sf[i][1] * Gf[1][j] + Sf[i][2] * Gf[2][j];
        const R ker[6] = {2 * P[0][0], 2 * P[1][1], 2 * P[2][2], P[0][1] + P[1][0], P[0][2] + P[2][0], P[1][2] + P[2][1]};
        R t[6];
        FN(congruence)(Ji, ker, t);
        for (int c = 0; c < 6; ++c) Im[6 * k + c] = two_v0 * t[c];
    }
}

/* build_element_constants hot fields (precompute.hpp:206-255) into the
 * canonical record of include/djg.h. Returns 0 on a bad element. */
static int FN(element_record)(const R x[8][3], int kind, int model, R c_hg, R kappa, const R A[6], const R B[6],
                              const R a[3], const R b[3], R* out) {
    layout_t L = layout_of(kind, model);
    R d[3][8], J[3][3], Ji[3][3], det;
    FN(shape)(kind, d);
    if (!FN(jacobian0)(x, d, kind == DJG_T4 ? 4 : 8, J, Ji, &det)) return 0;
    const R v0 = kind == DJG_T4 ? det / (R)6 : (R)8 * det; /* volume0, element.hpp:80-85 */
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) out[3 * i + j] = J[i][j];
    out[9] = det;
    out[10] = v0;
    /* G_k = outer / sym_outer of J0inv columns (precompute.hpp:45-50) */
    const R q[3][3] = {{Ji[0][0], Ji[1][0], Ji[2][0]}, {Ji[0][1], Ji[1][1], Ji[2][1]}, {Ji[0][2], Ji[1][2], Ji[2][2]}};
    R G[6][6];
    for (int k = 0; k < 3; ++k) {
        const R* v = q[k];
        G[k][0] = v[0] * v[0]; G[k][1] = v[1] * v[1]; G[k][2] = v[2] * v[2];
        G[k][3] = v[0] * v[1]; G[k][4] = v[0] * v[2]; G[k][5] = v[1] * v[2];
    }
    static const int pairs[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int p = 0; p < 3; ++p) {
        const R* u = q[pairs[p][0]];
        const R* v = q[pairs[p][1]];
        R* g = G[3 + p];
        g[0] = 2 * u[0] * v[0]; g[1] = 2 * u[1] * v[1]; g[2] = 2 * u[2] * v[2];
        g[3] = u[0] * v[1] + u[1] * v[0]; g[4] = u[0] * v[2] + u[2] * v[0]; g[5] = u[1] * v[2] + u[2] * v[1];
    }
    R m1[6];
    for (int k = 0; k < 6; ++k) m1[k] = out[11 + k] = G[k][0] + G[k][1] + G[k][2];
    const R two_v0 = 2 * v0;
    const R ident[6] = {1, 1, 1, 0, 0, 0};
    R t[6];
    FN(congruence)(Ji, ident, t);
    for (int k = 0; k < 6; ++k) out[17 + k] = two_v0 * t[k];
    if (model == DJG_MR) {
        for (int p = 0; p < 6; ++p)
            for (int qq = p; qq < 6; ++qq) out[L.M2 + sym6_index(p, qq)] = (m1[p] * m1[qq] - FN(ddot)(G[p], G[qq])) / 2;
        for (int k = 0; k < 6; ++k) {
            const R tr = G[k][0] + G[k][1] + G[k][2];
            const R ker[6] = {tr - G[k][0], tr - G[k][1], tr - G[k][2], -G[k][3], -G[k][4], -G[k][5]};
            FN(congruence)(Ji, ker, t);
            for (int c = 0; c < 6; ++c) out[L.I2m + 6 * k + c] = two_v0 * t[c];
        }
    }
    if (model == DJG_TI || model == DJG_OT) {
        for (int k = 0; k < 6; ++k) out[L.m4 + k] = FN(ddot)(A, G[k]);
        FN(congruence)(Ji, A, t);
        for (int c = 0; c < 6; ++c) out[L.I4m + c] = two_v0 * t[c];
    }
    if (model == DJG_OT) {
        for (int k = 0; k < 6; ++k) out[L.m6 + k] = FN(ddot)(B, G[k]);
        FN(congruence)(Ji, B, t);
        for (int c = 0; c < 6; ++c) out[L.I6m + c] = two_v0 * t[c];
    }
    if (model == DJG_I57) {
        FN(fibre_second_order)(G, Ji, two_v0, a, A, out + L.M5, out + L.I5m);
        FN(fibre_second_order)(G, Ji, two_v0, b, B, out + L.M7, out + L.I7m);
    }
    if (kind == DJG_H8) {
        R gamma[4][8];
        FN(hourglass_vectors)(x, d, Ji, gamma);
        out[L.khg] = c_hg * kappa * CBRT(v0);
        for (int m = 0; m < 4; ++m)
            for (int a = 0; a < 8; ++a) out[L.gamma + 8 * m + a] = gamma[m][a];
    }
    return 1;
}

/* Material scalars in Real (material.hpp:140-290) */
typedef struct {
    int model;
    R mu, kappa, rho, eta_a, eta_b, c10, c01;
} FN(mat_t);

static FN(mat_t) FN(mat_of)(const djg_material_params* p) {
    FN(mat_t) m;
    m.model = p->model;
    m.mu = (R)p->mu; m.kappa = (R)p->kappa; m.rho = (R)p->rho;
    m.eta_a = (R)p->eta_a; m.eta_b = (R)p->eta_b; m.c10 = (R)p->c10; m.c01 = (R)p->c01;
    return m;
}

static R FN(shear_modulus)(const FN(mat_t)* m) { return m->model == DJG_MR ? 2 * (m->c10 + m->c01) : m->mu; }

/* One element's DJ-TLED nodal forces from its record and displacements:
 * update_kinematics (kinematics.hpp:31-115) -> energy_derivatives
 * (material.hpp:266-290) -> element_force (djtled_force.hpp:36-82) ->
 * hourglass_force (djtled_force.hpp:86-95). Returns 0 on inversion. */
static int FN(element_force)(int kind, const FN(mat_t)* mat, const R* rec, const R u[8][3], R f[8][3]) {
    layout_t L = layout_of(kind, mat->model);
    const int n = kind == DJG_T4 ? 4 : 8;
    R d[3][8];
    FN(shape)(kind, d);
    /* update_jacobian: Jt = J0 + D U */
    R Jt[3][3];
    for (int i = 0; i < 3; ++i) {
        R du0 = 0, du1 = 0, du2 = 0;
        for (int a = 0; a < n; ++a) {
            du0 = du0 + d[i][a] * u[a][0];
            du1 = du1 + d[i][a] * u[a][1];
            du2 = du2 + d[i][a] * u[a][2];
        }
        Jt[i][0] = rec[3 * i + 0] + du0;
        Jt[i][1] = rec[3 * i + 1] + du1;
        Jt[i][2] = rec[3 * i + 2] + du2;
    }
    const R detJt = FN(det3)(Jt);
    if (!(detJt > 0)) return 0;
    R Ji[3][3];
    FN(inv3)(Jt, detJt, Ji);
    const R J = detJt / rec[9]; /* volume_ratio */
    /* g_vector: (r0.r0, r1.r1, r2.r2, r0.r1, r0.r2, r1.r2) of Jt rows */
    R g[6];
    g[0] = Jt[0][0] * Jt[0][0] + Jt[0][1] * Jt[0][1] + Jt[0][2] * Jt[0][2];
    g[1] = Jt[1][0] * Jt[1][0] + Jt[1][1] * Jt[1][1] + Jt[1][2] * Jt[1][2];
    g[2] = Jt[2][0] * Jt[2][0] + Jt[2][1] * Jt[2][1] + Jt[2][2] * Jt[2][2];
    g[3] = Jt[0][0] * Jt[1][0] + Jt[0][1] * Jt[1][1] + Jt[0][2] * Jt[1][2];
    g[4] = Jt[0][0] * Jt[2][0] + Jt[0][1] * Jt[2][1] + Jt[0][2] * Jt[2][2];
    g[5] = Jt[1][0] * Jt[2][0] + Jt[1][1] * Jt[2][1] + Jt[1][2] * Jt[2][2];
    /* invariants (kinematics.hpp:60-103) */
    const R cb = CBRT(J);
    const R j_m23 = (R)1 / (cb * cb);
    const R j_m43 = j_m23 * j_m23;
    const R* m1 = rec + 11;
    const R I1 = g[0] * m1[0] + g[1] * m1[1] + g[2] * m1[2] + g[3] * m1[3] + g[4] * m1[4] + g[5] * m1[5];
    const R Ib1 = j_m23 * I1;
    /* energy_derivatives + element_force bracket */
    const R dJ = mat->kappa * (J - 1);
    R s[6], dev;
    const R* I1m = rec + 17;
    R dI1 = mat->model == DJG_MR ? mat->c10 : mat->mu / 2;
    for (int k = 0; k < 6; ++k) s[k] = dI1 * I1m[k];
    dev = dI1 * Ib1;
    if (mat->model == DJG_TI || mat->model == DJG_OT) {
        const R* m4 = rec + L.m4;
        const R I4 = g[0] * m4[0] + g[1] * m4[1] + g[2] * m4[2] + g[3] * m4[3] + g[4] * m4[4] + g[5] * m4[5];
        const R Ib4 = j_m23 * I4;
        const R dI4 = mat->eta_a * (Ib4 - 1);
        for (int k = 0; k < 6; ++k) s[k] = s[k] + dI4 * rec[L.I4m + k];
        dev += dI4 * Ib4;
    }
    if (mat->model == DJG_OT) {
        const R* m6 = rec + L.m6;
        const R I6 = g[0] * m6[0] + g[1] * m6[1] + g[2] * m6[2] + g[3] * m6[3] + g[4] * m6[4] + g[5] * m6[5];
        const R Ib6 = j_m23 * I6;
        const R dI6 = mat->eta_b * (Ib6 - 1);
        for (int k = 0; k < 6; ++k) s[k] = s[k] + dI6 * rec[L.I6m + k];
        dev += dI6 * Ib6;
    }
    if (mat->model == DJG_MR) {
        const R I2 = FN(quadform)(rec + L.M2, g);
        const R Ib2 = j_m43 * I2;
        const R dI2 = mat->c01;
        /* contract_ghat (djtled_force.hpp:18-24): g0*M0, then + gk*Mk */
        R cg[6];
        const R* I2m = rec + L.I2m;
        for (int c = 0; c < 6; ++c) cg[c] = g[0] * I2m[c];
        for (int k = 1; k < 6; ++k)
            for (int c = 0; c < 6; ++c) cg[c] = cg[c] + g[k] * I2m[6 * k + c];
        const R w = j_m23 * dI2;
        for (int k = 0; k < 6; ++k) s[k] = s[k] + w * cg[k];
        dev += 2 * dI2 * Ib2;
    }
    if (mat->model == DJG_I57) {
        /* need.i5, need.i7 (kinematics.hpp:89-101; djtled_force.hpp:58-65)
         * with the derivatives of test_forces.cpp:262-268 */
        const int Mo[2] = {L.M5, L.M7}, Io[2] = {L.I5m, L.I7m};
        const R eta[2] = {mat->eta_a, mat->eta_b};
        for (int f = 0; f < 2; ++f) {
            const R I = FN(quadform)(rec + Mo[f], g);
            const R Ib = j_m43 * I;
            const R dI = eta[f] * (Ib - 1);
            R cg[6];
            const R* Im = rec + Io[f];
            for (int c = 0; c < 6; ++c) cg[c] = g[0] * Im[c];
            for (int k = 1; k < 6; ++k)
                for (int c = 0; c < 6; ++c) cg[c] = cg[c] + g[k] * Im[6 * k + c];
            const R w = j_m23 * dI;
            for (int k = 0; k < 6; ++k) s[k] = s[k] + w * cg[k];
            dev += 2 * dI * Ib;
        }
    }
    const R c = (-(R)2 / (R)3 * dev + J * dJ) * rec[10];
    /* K = j_m23 (Jt^T S) + c Jt^-1 */
    const R S[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    R K[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const R mt = Jt[0][i] * S[0][j] + Jt[1][i] * S[1][j] + Jt[2][i] * S[2][j];
            K[i][j] = j_m23 * mt + c * Ji[i][j];
        }
    if (kind == DJG_T4) {
        for (int i = 0; i < 3; ++i) {
            f[1][i] = K[i][0];
            f[2][i] = K[i][1];
            f[3][i] = K[i][2];
            f[0][i] = (R)(-1) * ((f[1][i] + f[2][i]) + f[3][i]);
        }
    } else {
        for (int a = 0; a < 8; ++a)
            for (int i = 0; i < 3; ++i) f[a][i] = d[0][a] * K[i][0] + d[1][a] * K[i][1] + d[2][a] * K[i][2];
        /* hourglass_force (djtled_force.hpp:86-95) */
        const R k = rec[L.khg];
        if (k != (R)0) {
            const R* gam = rec + L.gamma;
            for (int m = 0; m < 4; ++m) {
                R q0 = 0, q1 = 0, q2 = 0;
                for (int b = 0; b < 8; ++b) {
                    q0 = q0 + gam[8 * m + b] * u[b][0];
                    q1 = q1 + gam[8 * m + b] * u[b][1];
                    q2 = q2 + gam[8 * m + b] * u[b][2];
                }
                for (int b = 0; b < 8; ++b) {
                    const R kg = k * gam[8 * m + b];
                    f[b][0] = f[b][0] + kg * q0;
                    f[b][1] = f[b][1] + kg * q1;
                    f[b][2] = f[b][2] + kg * q2;
                }
            }
        }
    }
    return 1;
}

/* ---------------------------------------------------------------- problem */

typedef struct {
    int kind, npe, nconst, policy;
    int64_t N, E;
    FN(mat_t) mat;
    R* nodes;        /* 3N */
    int32_t* conn;   /* npe*E */
    int64_t* off;    /* N+1 */
    int64_t* celem;  /* npe*E */
    int32_t* cloc;   /* npe*E */
    R* consts;       /* E*nconst */
    R* mass;         /* N */
    R* c1;           /* N */
    uint8_t* massless;
    uint8_t* kindv;  /* 3N */
    R* target;       /* 3N */
    R* t_total;      /* 3N */
    R dt, crit, alpha, c2, c3, ramp_t_total, c_wave;
} FN(prob_t);

static void FN(prob_free)(FN(prob_t)* P) {
    free(P->nodes); free(P->conn); free(P->off); free(P->celem); free(P->cloc); free(P->consts);
    free(P->mass); free(P->c1); free(P->massless); free(P->kindv); free(P->target); free(P->t_total);
    memset(P, 0, sizeof(*P));
}

static void FN(gather_x)(const FN(prob_t)* P, int64_t e, R x[8][3]) {
    for (int a = 0; a < P->npe; ++a) {
        const int32_t n = P->conn[e * P->npe + a];
        x[a][0] = P->nodes[3 * n]; x[a][1] = P->nodes[3 * n + 1]; x[a][2] = P->nodes[3 * n + 2];
    }
}

static R FN(tri_area)(const R* a, const R* b, const R* c) {
    const R u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
    const R v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
    const R w0 = u1 * v2 - u2 * v1, w1 = u2 * v0 - u0 * v2, w2 = u0 * v1 - u1 * v0;
    return SQRT(w0 * w0 + w1 * w1 + w2 * w2) / 2;
}

/* characteristic_length (precompute.hpp:303-319) */
static R FN(char_length)(const R x[8][3], int kind, R v0) {
    R a_max = 0;
    if (kind == DJG_T4) {
        static const int f[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        for (int i = 0; i < 4; ++i) {
            const R ar = FN(tri_area)(x[f[i][0]], x[f[i][1]], x[f[i][2]]);
            a_max = a_max < ar ? ar : a_max; /* std::max */
        }
        return 3 * v0 / a_max;
    }
    static const int f[6][4] = {{0, 3, 2, 1}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
    for (int i = 0; i < 6; ++i) {
        const R ar = FN(tri_area)(x[f[i][0]], x[f[i][1]], x[f[i][2]]) + FN(tri_area)(x[f[i][0]], x[f[i][2]], x[f[i][3]]);
        a_max = a_max < ar ? ar : a_max;
    }
    return v0 / a_max;
}

/* Builds the scenario: generate_box (mesh.hpp:208-264), DjModel constants,
 * NodeElementAdjacency (mesh.hpp:299-320), lump_mass (precompute.hpp:275-287),
 * critical_dt (:323-331), relaxation_alpha (solver.hpp:330-339), box BCs
 * (config.hpp:31-42, bench.hpp:386-411), DofConstraints (solver.hpp:18-33),
 * UpdateCoeffs (solver.hpp:70-86). Returns 0 or an error code. */
static int FN(prob_build)(const djg_scenario_spec* s, FN(prob_t)* P) {
    memset(P, 0, sizeof(*P));
    P->kind = s->kind;
    P->npe = s->kind == DJG_T4 ? 4 : 8;
    P->policy = s->policy;
    P->mat = FN(mat_of)(&s->material);
    P->nconst = layout_of(s->kind, s->material.model).count;
    if (!s->nodes) {
        const R ex[3] = {(R)s->extent[0], (R)s->extent[1], (R)s->extent[2]};
        const int64_t nx = s->divisions[0], ny = s->divisions[1], nz = s->divisions[2];
        if (!(ex[0] > 0 && ex[1] > 0 && ex[2] > 0) || nx < 1 || ny < 1 || nz < 1) return DJG_E_CONFIG;
        P->N = (nx + 1) * (ny + 1) * (nz + 1);
        P->nodes = (R*)malloc(sizeof(R) * 3 * P->N);
        int64_t w = 0;
        for (int64_t k = 0; k <= nz; ++k)
            for (int64_t j = 0; j <= ny; ++j)
                for (int64_t i = 0; i <= nx; ++i) {
                    P->nodes[w++] = ex[0] * (R)(int)i / (R)(int)nx;
                    P->nodes[w++] = ex[1] * (R)(int)j / (R)(int)ny;
                    P->nodes[w++] = ex[2] * (R)(int)k / (R)(int)nz;
                }
        const int64_t cells = nx * ny * nz;
        P->E = cells * (s->kind == DJG_H8 ? 1 : 6);
        P->conn = (int32_t*)malloc(sizeof(int32_t) * P->npe * P->E);
        static const int orders[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        int64_t e = 0;
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t i = 0; i < nx; ++i) {
                    int32_t cor[2][2][2];
                    for (int dz = 0; dz < 2; ++dz)
                        for (int dy = 0; dy < 2; ++dy)
                            for (int dx = 0; dx < 2; ++dx)
                                cor[dx][dy][dz] = (int32_t)((i + dx) + (nx + 1) * ((j + dy) + (ny + 1) * (k + dz)));
                    if (s->kind == DJG_H8) {
                        for (int a = 0; a < 8; ++a)
                            P->conn[e * 8 + a] =
                                cor[(corner_sign[a][0] + 1) / 2][(corner_sign[a][1] + 1) / 2][(corner_sign[a][2] + 1) / 2];
                        ++e;
                        continue;
                    }
                    for (int t = 0; t < 6; ++t) {
                        int st[3] = {0, 0, 0};
                        int32_t path[4];
                        path[0] = cor[0][0][0];
                        for (int q = 0; q < 3; ++q) {
                            st[orders[t][q]] = 1;
                            path[q + 1] = cor[st[0]][st[1]][st[2]];
                        }
                        const int o0 = orders[t][0], o1 = orders[t][1];
                        if ((o0 == 0 && o1 == 2) || (o0 == 1 && o1 == 0) || (o0 == 2 && o1 == 1)) {
                            const int32_t tmp = path[1];
                            path[1] = path[2];
                            path[2] = tmp;
                        }
                        for (int a = 0; a < 4; ++a) P->conn[e * 4 + a] = path[a];
                        ++e;
                    }
                }
    } else {
        P->N = s->num_nodes;
        P->E = s->num_elements;
        P->nodes = (R*)malloc(sizeof(R) * 3 * (P->N > 0 ? P->N : 1));
        for (int64_t i = 0; i < 3 * P->N; ++i) P->nodes[i] = (R)s->nodes[i];
        P->conn = (int32_t*)malloc(sizeof(int32_t) * P->npe * (P->E > 0 ? P->E : 1));
        memcpy(P->conn, s->conn, sizeof(int32_t) * P->npe * P->E);
        for (int64_t i = 0; i < P->npe * P->E; ++i)
            if (P->conn[i] < 0 || P->conn[i] >= P->N) return DJG_E_CONFIG;
    }
    const int64_t N = P->N, E = P->E;
    const int npe = P->npe, nc = P->nconst;
    /* constants */
    R A[6] = {0}, B[6] = {0}, ua[3] = {0}, ub[3] = {0};
    const int mdl = s->material.model;
    if (mdl == DJG_TI || mdl == DJG_OT || mdl == DJG_I57) FN(fibre_tensor)(s->material.fibre_a, A, ua);
    if (mdl == DJG_OT || mdl == DJG_I57) FN(fibre_tensor)(s->material.fibre_b, B, ub);
    P->consts = (R*)calloc((size_t)(E > 0 ? E : 1) * nc, sizeof(R));
    int bad = 0;
    const R c_hg = (R)s->c_hg;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t e = 0; e < E; ++e) {
        R x[8][3];
        FN(gather_x)(P, e, x);
        if (!FN(element_record)(x, P->kind, mdl, c_hg, P->mat.kappa, A, B, ua, ub, P->consts + e * nc)) bad = 1;
    }
    if (bad) return DJG_E_CONFIG;
    /* adjacency: counting sort in ascending element order */
    P->off = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
    P->celem = (int64_t*)malloc(sizeof(int64_t) * (npe * E > 0 ? npe * E : 1));
    P->cloc = (int32_t*)malloc(sizeof(int32_t) * (npe * E > 0 ? npe * E : 1));
    for (int64_t i = 0; i < npe * E; ++i) P->off[P->conn[i] + 1]++;
    for (int64_t i = 0; i < N; ++i) P->off[i + 1] += P->off[i];
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (N > 0 ? N : 1));
    memcpy(cur, P->off, sizeof(int64_t) * N);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < npe; ++a) {
            const int64_t p = cur[P->conn[e * npe + a]]++;
            P->celem[p] = e;
            P->cloc[p] = a;
        }
    free(cur);
    /* lump_mass: serial element loop, += share */
    P->mass = (R*)calloc((size_t)(N > 0 ? N : 1), sizeof(R));
    for (int64_t e = 0; e < E; ++e) {
        const R share = P->mat.rho * P->consts[e * nc + 10] / (R)npe;
        for (int a = 0; a < npe; ++a) P->mass[P->conn[e * npe + a]] += share;
    }
    /* critical_dt with the dilatational wave speed (material.hpp:117-120) */
    P->c_wave = SQRT((P->mat.kappa + (R)4 / (R)3 * FN(shear_modulus)(&P->mat)) / P->mat.rho);
    R l_min = RMAX;
    for (int64_t e = 0; e < E; ++e) {
        R x[8][3];
        FN(gather_x)(P, e, x);
        const R l = FN(char_length)(x, P->kind, P->consts[e * nc + 10]);
        l_min = l < l_min ? l : l_min; /* std::min */
    }
    P->crit = l_min / P->c_wave;
    P->dt = s->dt > 0 ? (R)s->dt : (R)s->safety * P->crit;
    /* bounding box */
    R lo[3] = {RMAX, RMAX, RMAX}, hi[3] = {-RMAX, -RMAX, -RMAX};
    for (int64_t n = 0; n < N; ++n)
        for (int i = 0; i < 3; ++i) {
            const R v = P->nodes[3 * n + i];
            lo[i] = v < lo[i] ? v : lo[i];
            hi[i] = hi[i] < v ? v : hi[i];
        }
    if (s->alpha_mode == 0) {
        const R mu = FN(shear_modulus)(&P->mat);
        const R e_mod = 9 * P->mat.kappa * mu / (3 * P->mat.kappa + mu);
        const R c_bar = SQRT(e_mod / P->mat.rho);
        R l = hi[0] - lo[0];
        if (l < hi[1] - lo[1]) l = hi[1] - lo[1];
        if (l < hi[2] - lo[2]) l = hi[2] - lo[2];
        P->alpha = (R)M_PI * c_bar / l;
    } else {
        P->alpha = (R)s->alpha;
    }
    /* DofConstraints */
    P->kindv = (uint8_t*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), 1);
    P->target = (R*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), sizeof(R));
    P->t_total = (R*)malloc(sizeof(R) * (3 * N > 0 ? 3 * N : 1));
    for (int64_t i = 0; i < 3 * N; ++i) P->t_total[i] = 1;
    if (s->bc_mode == 1) {
        /* select_plane_nodes (config.hpp:31-42) on zmin / zmax */
        const R ext = hi[2] - lo[2];
        const R eps = (R)1e-9 * (ext > 0 ? ext : (R)1);
        P->ramp_t_total = P->dt * (R)s->ramp_steps;
        for (int64_t n = 0; n < N; ++n) {
            const R z = P->nodes[3 * n + 2];
            if (FABS(z - lo[2]) <= eps) {
                if (s->fix_all_axes) {
                    P->kindv[3 * n + 0] = DJG_FIXED;
                    P->kindv[3 * n + 1] = DJG_FIXED;
                }
                P->kindv[3 * n + 2] = DJG_FIXED;
            }
        }
        for (int64_t n = 0; n < N; ++n) {
            const R z = P->nodes[3 * n + 2];
            if (FABS(z - hi[2]) <= eps) {
                if (P->kindv[3 * n + 2] != DJG_FREE) return DJG_E_CONFIG;
                P->kindv[3 * n + 2] = DJG_PRESCRIBED;
                P->target[3 * n + 2] = (R)s->target;
                P->t_total[3 * n + 2] = P->ramp_t_total;
            }
        }
    } else if (s->bc_mode == 2) {
        for (int64_t i = 0; i < s->n_fixed; ++i) {
            const int64_t dof = 3 * (int64_t)s->fixed_node[i] + s->fixed_axis[i];
            if (P->kindv[dof] != DJG_FREE) return DJG_E_CONFIG;
            P->kindv[dof] = DJG_FIXED;
        }
        for (int64_t i = 0; i < s->n_prescribed; ++i) {
            const int64_t dof = 3 * (int64_t)s->presc_node[i] + s->presc_axis[i];
            if (P->kindv[dof] != DJG_FREE) return DJG_E_CONFIG;
            P->kindv[dof] = DJG_PRESCRIBED;
            P->target[dof] = (R)s->presc_target[i];
            P->t_total[dof] = (R)s->presc_t_total[i];
        }
    }
    /* UpdateCoeffs */
    const R denom = (R)1 + P->alpha * P->dt / 2;
    P->c2 = (R)2 / denom;
    P->c3 = -((R)1 - P->alpha * P->dt / 2) / denom;
    P->c1 = (R*)calloc((size_t)(N > 0 ? N : 1), sizeof(R));
    P->massless = (uint8_t*)calloc((size_t)(N > 0 ? N : 1), 1);
    for (int64_t n = 0; n < N; ++n) {
        if (P->mass[n] > 0)
            P->c1[n] = P->dt * P->dt / (P->mass[n] * denom);
        else
            P->massless[n] = 1;
    }
    return 0;
}

/* assemble_internal (djtled_force.hpp:163-209): element stage into elem_f,
 * min inverted element, then the ascending-order CSR gather
 * (djtled_force.hpp:116-134). Returns first inverted element or -1. */
static int64_t FN(assemble)(const FN(prob_t)* P, const R* u, R* elem_f, R* f, int64_t* inv_count) {
    const int64_t E = P->E, N = P->N;
    const int npe = P->npe, nc = P->nconst;
    int64_t first = -1, cnt = 0;
#pragma omp parallel
    {
        int64_t lfirst = -1, lcnt = 0;
#pragma omp for schedule(static)
        for (int64_t e = 0; e < E; ++e) {
            R ue[8][3], fe[8][3];
            for (int a = 0; a < npe; ++a) {
                const int32_t n = P->conn[e * npe + a];
                ue[a][0] = u[3 * n]; ue[a][1] = u[3 * n + 1]; ue[a][2] = u[3 * n + 2];
            }
            R* dst = elem_f + e * npe * 3;
            if (!FN(element_force)(P->kind, &P->mat, P->consts + e * nc, (const R(*)[3])ue, fe)) {
                ++lcnt;
                if (lfirst < 0 || e < lfirst) lfirst = e;
                for (int i = 0; i < npe * 3; ++i) dst[i] = 0;
                continue;
            }
            for (int a = 0; a < npe; ++a)
                for (int i = 0; i < 3; ++i) dst[a * 3 + i] = fe[a][i];
        }
#pragma omp critical
        {
            cnt += lcnt;
            if (lfirst >= 0 && (first < 0 || lfirst < first)) first = lfirst;
        }
    }
    *inv_count = cnt;
    if (first >= 0 && P->policy == DJG_ABORT) return first;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        R sx = 0, sy = 0, sz = 0;
        for (int64_t p = P->off[n]; p < P->off[n + 1]; ++p) {
            const R* src = elem_f + (P->celem[p] * npe + P->cloc[p]) * 3;
            sx += src[0];
            sy += src[1];
            sz += src[2];
        }
        f[3 * n] = sx;
        f[3 * n + 1] = sy;
        f[3 * n + 2] = sz;
    }
    return P->policy == DJG_ABORT ? -1 : -1;
}

/* advance_step loop (solver.hpp:98-153) with run_simulation's failure
 * semantics (solver.hpp:225-239); explicit step count. */
static int FN(run)(const FN(prob_t)* P, int64_t steps, const R* u0, const R* up0, const R* r_ext, R* u_out, R* up_out,
                   djg_report* rep) {
    const int64_t N = P->N;
    R* uc = (R*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), sizeof(R));
    R* up = (R*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), sizeof(R));
    R* un = (R*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), sizeof(R));
    R* f = (R*)calloc((size_t)(3 * N > 0 ? 3 * N : 1), sizeof(R));
    R* ef = (R*)calloc((size_t)(P->E * P->npe * 3 > 0 ? P->E * P->npe * 3 : 1), sizeof(R));
    if (u0) memcpy(uc, u0, sizeof(R) * 3 * N);
    if (up0) memcpy(up, up0, sizeof(R) * 3 * N);
    djg_report r;
    memset(&r, 0, sizeof(r));
    r.first_inverted = -1;
    r.fail_step = -1;
    int64_t step = 0;
    for (int64_t s = 0; s < steps; ++s) {
        int64_t cnt = 0;
        const int64_t first = FN(assemble)(P, uc, ef, f, &cnt);
        r.inverted_count += cnt;
        if (cnt > 0) r.inverted_steps++;
        if (first >= 0) {
            r.first_inverted = first;
            r.fail_step = step + 1;
            r.status = DJG_E_INVERSION;
            break;
        }
        const R t_next = P->dt * (R)(step + 1);
        int nonfinite = 0;
#pragma omp parallel for schedule(static) reduction(| : nonfinite)
        for (int64_t n = 0; n < N; ++n) {
            for (int i = 0; i < 3; ++i) {
                const int64_t dof = 3 * n + i;
                if (P->kindv[dof] == DJG_FIXED) {
                    un[dof] = 0;
                } else if (P->kindv[dof] == DJG_PRESCRIBED) {
                    const R sr = t_next / P->t_total[dof];
                    un[dof] = (sr >= (R)1 ? (R)1 : sr) * P->target[dof];
                } else if (P->massless[n]) {
                    un[dof] = 0;
                } else {
                    const R rx = r_ext ? r_ext[dof] : (R)0;
                    const R v = P->c1[n] * (rx - f[dof]) + P->c2 * uc[dof] + P->c3 * up[dof];
                    un[dof] = v;
                    if (!isfinite(v)) nonfinite = 1;
                }
            }
        }
        if (nonfinite) {
            r.diverged = 1;
            r.fail_step = step + 1;
            r.status = DJG_E_DIVERGENCE;
            break;
        }
        R* t = up;
        up = uc;
        uc = un;
        un = t;
        ++step;
        ++r.steps_done;
    }
    r.step = step;
    if (u_out) memcpy(u_out, uc, sizeof(R) * 3 * N);
    if (up_out) memcpy(up_out, up, sizeof(R) * 3 * N);
    if (rep) *rep = r;
    free(uc); free(up); free(un); free(f); free(ef);
    return r.status;
}
