/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle (plain-C restatement of the
 * reference algorithm, see djo_impl.h). Built into oracle/_build/libdjoracle.so
 * by oracle/Makefile. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product never does.
 *
 * Pinned: tests/test_oracle.py checks it bit-for-bit against the reference
 * itself (oracle/_ref/libdjref.so, built from the unmodified reference
 * headers) and against the committed fixtures in tests/golden/.
 */
#define _GNU_SOURCE
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "djg_types.h"

/* H8 corner signs (element.hpp:17-20) */
static const int corner_sign[8][3] = {
    {-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
    {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1},
};

/* Sym6::index (core.hpp:287-290) */
static int sym6_index(int i, int j) {
    if (i > j) {
        const int t = i;
        i = j;
        j = t;
    }
    return i * 6 - i * (i + 1) / 2 + j;
}

/* Offsets of the canonical hot-field record (include/djg.h). */
typedef struct {
    int m4, I4m, m6, I6m, M2, I2m, M5, I5m, M7, I7m, khg, gamma, count;
} layout_t;

static layout_t layout_of(int kind, int model) {
    layout_t L = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 23};
    int o = 23;
    if (model == DJG_TI || model == DJG_OT) { L.m4 = o; L.I4m = o + 6; o += 12; }
    if (model == DJG_OT) { L.m6 = o; L.I6m = o + 6; o += 12; }
    if (model == DJG_MR) { L.M2 = o; L.I2m = o + 21; o += 57; }
    if (model == DJG_I57) { L.M5 = o; L.I5m = o + 21; L.M7 = o + 57; L.I7m = o + 78; o += 114; }
    if (kind == DJG_H8) { L.khg = o; L.gamma = o + 1; o += 33; }
    L.count = o;
    return L;
}

#define R float
#define FN(x) x##_f
#define SQRT sqrtf
#define CBRT cbrtf
#define FABS fabsf
#define RMAX FLT_MAX
#include "djo_impl.h"
#undef R
#undef FN
#undef SQRT
#undef CBRT
#undef FABS
#undef RMAX

#define R double
#define FN(x) x##_d
#define SQRT sqrt
#define CBRT cbrt
#define FABS fabs
#define RMAX DBL_MAX
#include "djo_impl.h"

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

#define EXPORT_IMAGE(S)                                                                           \
    static void image_out_##S(const prob_t_##S* P, const djg_image_ptrs* o, djg_image_scalars* sc) { \
        const int64_t N = P->N, E = P->E;                                                         \
        if (sc) {                                                                                 \
            sc->num_nodes = N;                                                                    \
            sc->num_elements = E;                                                                 \
            sc->npe = P->npe;                                                                     \
            sc->nconst = P->nconst;                                                               \
            sc->dt = P->dt;                                                                       \
            sc->critical_dt = P->crit;                                                            \
            sc->alpha = P->alpha;                                                                 \
            sc->c2 = P->c2;                                                                       \
            sc->c3 = P->c3;                                                                       \
            sc->ramp_t_total = P->ramp_t_total;                                                   \
            sc->wave_speed = P->c_wave;                                                           \
        }                                                                                         \
        if (!o) return;                                                                           \
        const size_t rs = sizeof(P->dt);                                                          \
        if (o->nodes) memcpy(o->nodes, P->nodes, rs * 3 * N);                                     \
        if (o->conn) memcpy(o->conn, P->conn, sizeof(int32_t) * P->npe * E);                      \
        if (o->csr_offsets) memcpy(o->csr_offsets, P->off, sizeof(int64_t) * (N + 1));            \
        if (o->csr_elem) memcpy(o->csr_elem, P->celem, sizeof(int64_t) * P->npe * E);             \
        if (o->csr_local) memcpy(o->csr_local, P->cloc, sizeof(int32_t) * P->npe * E);            \
        if (o->consts) memcpy(o->consts, P->consts, rs * P->nconst * E);                          \
        if (o->mass) memcpy(o->mass, P->mass, rs * N);                                            \
        if (o->c1) memcpy(o->c1, P->c1, rs * N);                                                  \
        if (o->massless) memcpy(o->massless, P->massless, N);                                     \
        if (o->dof_kind) memcpy(o->dof_kind, P->kindv, 3 * N);                                    \
        if (o->dof_target) memcpy(o->dof_target, P->target, rs * 3 * N);                          \
        if (o->dof_t_total) memcpy(o->dof_t_total, P->t_total, rs * 3 * N);                       \
    }

EXPORT_IMAGE(f)
EXPORT_IMAGE(d)

int djo_image(const djg_scenario_spec* s, int32_t threads, const djg_image_ptrs* o, djg_image_scalars* sc) {
    set_threads(threads);
    int rc;
    if (s->precision == 4) {
        prob_t_f P;
        rc = prob_build_f(s, &P);
        if (!rc) image_out_f(&P, o, sc);
        prob_free_f(&P);
    } else {
        prob_t_d P;
        rc = prob_build_d(s, &P);
        if (!rc) image_out_d(&P, o, sc);
        prob_free_d(&P);
    }
    return rc;
}

int djo_run(const djg_scenario_spec* s, int64_t steps, int32_t threads, const void* u0, const void* up0,
            const void* r_ext, void* u_out, void* up_out, djg_report* rep) {
    set_threads(threads);
    int rc;
    if (s->precision == 4) {
        prob_t_f P;
        rc = prob_build_f(s, &P);
        if (!rc) rc = run_f(&P, steps, (const float*)u0, (const float*)up0, (const float*)r_ext, (float*)u_out,
                            (float*)up_out, rep);
        prob_free_f(&P);
    } else {
        prob_t_d P;
        rc = prob_build_d(s, &P);
        if (!rc) rc = run_d(&P, steps, (const double*)u0, (const double*)up0, (const double*)r_ext, (double*)u_out,
                            (double*)up_out, rep);
        prob_free_d(&P);
    }
    return rc;
}

int djo_assemble(const djg_scenario_spec* s, int32_t threads, const void* u, void* f, djg_assemble_stats* st) {
    set_threads(threads);
    int rc;
    int64_t first = -1, cnt = 0;
    if (s->precision == 4) {
        prob_t_f P;
        rc = prob_build_f(s, &P);
        if (!rc) {
            float* ef = (float*)calloc((size_t)(P.E * P.npe * 3 + 1), sizeof(float));
            first = assemble_f(&P, (const float*)u, ef, (float*)f, &cnt);
            free(ef);
        }
        prob_free_f(&P);
    } else {
        prob_t_d P;
        rc = prob_build_d(s, &P);
        if (!rc) {
            double* ef = (double*)calloc((size_t)(P.E * P.npe * 3 + 1), sizeof(double));
            first = assemble_d(&P, (const double*)u, ef, (double*)f, &cnt);
            free(ef);
        }
        prob_free_d(&P);
    }
    if (st) {
        st->first_inverted = first;
        st->inverted_count = cnt;
    }
    if (rc) return rc;
    return first >= 0 ? DJG_E_INVERSION : 0;
}

/* Single-element force from a canonical record and element displacements
 * (npe x 3 Reals). Returns DJG_E_INVERSION for an inverted state. */
int djo_element_force_rec(int32_t precision, int32_t kind, const djg_material_params* m, const void* rec,
                          const void* u, void* f) {
    const int npe = kind == DJG_T4 ? 4 : 8;
    if (precision == 4) {
        mat_t_f mat = mat_of_f(m);
        float ue[8][3] = {{0}}, fe[8][3];
        memcpy(ue, u, sizeof(float) * 3 * npe);
        if (!element_force_f(kind, &mat, (const float*)rec, (const float(*)[3])ue, fe)) return DJG_E_INVERSION;
        memcpy(f, fe, sizeof(float) * 3 * npe);
    } else {
        mat_t_d mat = mat_of_d(m);
        double ue[8][3] = {{0}}, fe[8][3];
        memcpy(ue, u, sizeof(double) * 3 * npe);
        if (!element_force_d(kind, &mat, (const double*)rec, (const double(*)[3])ue, fe)) return DJG_E_INVERSION;
        memcpy(f, fe, sizeof(double) * 3 * npe);
    }
    return 0;
}

/* Canonical record of one element from its coordinates (npe x 3 doubles). */
int djo_element_record(int32_t precision, int32_t kind, const djg_material_params* m, double c_hg,
                       const double* coords, void* rec) {
    const int npe = kind == DJG_T4 ? 4 : 8;
    const int fa = m->model == DJG_TI || m->model == DJG_OT || m->model == DJG_I57;
    const int fb = m->model == DJG_OT || m->model == DJG_I57;
    if (precision == 4) {
        float x[8][3] = {{0}}, A[6] = {0}, B[6] = {0}, ua[3] = {0}, ub[3] = {0};
        for (int a = 0; a < npe; ++a)
            for (int i = 0; i < 3; ++i) x[a][i] = (float)coords[3 * a + i];
        if (fa) fibre_tensor_f(m->fibre_a, A, ua);
        if (fb) fibre_tensor_f(m->fibre_b, B, ub);
        return element_record_f((const float(*)[3])x, kind, m->model, (float)c_hg, (float)m->kappa, A, B, ua, ub,
                                (float*)rec)
                   ? 0
                   : DJG_E_CONFIG;
    }
    double x[8][3] = {{0}}, A[6] = {0}, B[6] = {0}, ua[3] = {0}, ub[3] = {0};
    for (int a = 0; a < npe; ++a)
        for (int i = 0; i < 3; ++i) x[a][i] = coords[3 * a + i];
    if (fa) fibre_tensor_d(m->fibre_a, A, ua);
    if (fb) fibre_tensor_d(m->fibre_b, B, ub);
    return element_record_d((const double(*)[3])x, kind, m->model, c_hg, m->kappa, A, B, ua, ub, (double*)rec)
               ? 0
               : DJG_E_CONFIG;
}

int djo_const_count(int32_t kind, int32_t model) { return layout_of(kind, model).count; }

/* Host libm cube root over an array (what the reference's std::cbrt calls),
 * and the same algorithm restated (glibc 2.39 s_cbrtf.c / s_cbrt.c). */
void djo_libm_cbrt(int32_t precision, const void* in, void* out, int64_t n) {
    if (precision == 4) {
        for (int64_t i = 0; i < n; ++i) ((float*)out)[i] = cbrtf(((const float*)in)[i]);
    } else {
        for (int64_t i = 0; i < n; ++i) ((double*)out)[i] = cbrt(((const double*)in)[i]);
    }
}

static const double cbrt_factor[5] = {1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648, 1.0,
                                      1.2599210498948731648, 1.5874010519681994748};

void djo_restated_cbrt(int32_t precision, const void* in, void* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        int xe;
        if (precision == 4) {
            const float x = ((const float*)in)[i];
            const float xm = frexpf(fabsf(x), &xe);
            if (x == 0.0f || !isfinite(x)) { ((float*)out)[i] = x + x; continue; }
            const float u = (float)(0.492659620528969547 + (0.697570460207922770 - 0.191502161678719066 * xm) * xm);
            const float t2 = u * u * u;
            const float ym = (float)(u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * cbrt_factor[2 + xe % 3]);
            ((float*)out)[i] = ldexpf(x > 0.0f ? ym : -ym, xe / 3);
        } else {
            const double x = ((const double*)in)[i];
            const double xm = frexp(fabs(x), &xe);
            if (x == 0.0 || !isfinite(x)) { ((double*)out)[i] = x + x; continue; }
            const double u = (0.354895765043919860 +
                              ((1.50819193781584896 +
                                ((-2.11499494167371287 +
                                  ((2.44693122563534430 +
                                    ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) *
                                     xm)) * xm)) * xm)) * xm));
            const double t2 = u * u * u;
            const double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * cbrt_factor[2 + xe % 3];
            ((double*)out)[i] = ldexp(x > 0.0 ? ym : -ym, xe / 3);
        }
    }
}
