// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// A thin C-ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include/djtled/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libdjref.so. It drives the reference's own public API
// (generate_box, DjEngine/TledEngine, lump_mass, critical_dt,
// relaxation_alpha, DofConstraints, UpdateCoeffs, advance_step) on the same
// djg_scenario_spec the product builder and the C restatement consume, so the
// three can be compared bit for bit. It is the oracle's own oracle and the
// CPU baseline of bench.py (`cpu_baseline.kind = "reference"`).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "djtled/bench.hpp"
#include "djtled/solver.hpp"
#include "djg_types.h"

using namespace djtled;

namespace {

thread_local std::string g_err;

template <class Real>
Material<Real> make_material(const djg_material_params& p) {
    const Vec3<Real> a{Real(p.fibre_a[0]), Real(p.fibre_a[1]), Real(p.fibre_a[2])};
    const Vec3<Real> b{Real(p.fibre_b[0]), Real(p.fibre_b[1]), Real(p.fibre_b[2])};
    switch (p.model) {
        case DJG_NH: return Material<Real>::neo_hookean(Real(p.mu), Real(p.kappa), Real(p.rho));
        case DJG_TI: return Material<Real>::transverse_isotropic(Real(p.mu), Real(p.eta_a), Real(p.kappa), Real(p.rho), a);
        case DJG_OT:
            return Material<Real>::orthotropic(Real(p.mu), Real(p.eta_a), Real(p.eta_b), Real(p.kappa), Real(p.rho), a, b);
        case DJG_MR: return Material<Real>::mooney_rivlin(Real(p.c10), Real(p.c01), Real(p.kappa), Real(p.rho));
        // DJG_I57 has no reference Material: the neo-Hookean part carries mu,
        // kappa and rho; element_impl supplies the I5 / I7 need set,
        // fibres and derivatives of test_forces.cpp:248-271.
        case DJG_I57: return Material<Real>::neo_hookean(Real(p.mu), Real(p.kappa), Real(p.rho));
    }
    throw ConfigError("unknown material model");
}

template <class Real>
struct RefProblem {
    Mesh<Real> mesh;
    Material<Real> mat;
    std::unique_ptr<DjEngine<Real>> dj;
    std::unique_ptr<TledEngine<Real>> tled;
    std::vector<Real> mass;
    DofConstraints<Real> bc;
    Real dt = 0, crit = 0, alpha = 0, ramp_t_total = 0, c_wave = 0;
    InversionPolicy policy = InversionPolicy::Abort;

    // engine 0: DJ-TLED only; 1: also TLED; 2: TLED only (the DJ model is
    // built for lump_mass / critical_dt, which take its constants, then freed).
    RefProblem(const djg_scenario_spec& s, int engine, int build_threads = 1) {
        const ElementKind kind = s.kind == DJG_T4 ? ElementKind::T4 : ElementKind::H8;
        if (!s.nodes) {
            mesh = generate_box<Real>({Real(s.extent[0]), Real(s.extent[1]), Real(s.extent[2])},
                                      {s.divisions[0], s.divisions[1], s.divisions[2]}, kind);
        } else {
            mesh.kind = kind;
            for (int64_t n = 0; n < s.num_nodes; ++n)
                mesh.nodes.push_back({Real(s.nodes[3 * n]), Real(s.nodes[3 * n + 1]), Real(s.nodes[3 * n + 2])});
            mesh.conn.assign(s.conn, s.conn + s.num_elements * mesh.npe());
            validate_mesh(mesh);
        }
        mat = make_material<Real>(s.material);
        const Real c_hg = Real(s.c_hg);
        dj = std::make_unique<DjEngine<Real>>(mesh, mat, c_hg, build_threads);
        if (engine == 1) tled = std::make_unique<TledEngine<Real>>(mesh, mat, c_hg, build_threads);
        mass = lump_mass(mesh, mat.rho, dj->model().elems);
        c_wave = dilatational_wave_speed(mat);
        crit = critical_dt(mesh, dj->model().elems, c_wave);
        if (engine == 2) {
            dj.reset();
            tled = std::make_unique<TledEngine<Real>>(mesh, mat, c_hg, build_threads);
        }
        dt = s.dt > 0 ? Real(s.dt) : Real(s.safety) * crit;
        alpha = s.alpha_mode == 0 ? relaxation_alpha(mat, mesh) : Real(s.alpha);
        policy = s.policy == DJG_ABORT ? InversionPolicy::Abort : InversionPolicy::SkipAndReport;
        BoundaryConditions<Real> bcs;
        if (s.bc_mode == 1) {
            for (int n : select_plane_nodes(mesh, Plane::ZMin)) {
                if (s.fix_all_axes) {
                    bcs.fixed.emplace_back(n, 0);
                    bcs.fixed.emplace_back(n, 1);
                }
                bcs.fixed.emplace_back(n, 2);
            }
            PrescribedRamp<Real> ramp;
            ramp.nodes = select_plane_nodes(mesh, Plane::ZMax);
            ramp.axis = 2;
            ramp.target = Real(s.target);
            ramp_t_total = dt * Real(s.ramp_steps);
            ramp.t_total = ramp_t_total;
            bcs.prescribed.push_back(ramp);
        } else if (s.bc_mode == 2) {
            for (int64_t i = 0; i < s.n_fixed; ++i) bcs.fixed.emplace_back(s.fixed_node[i], s.fixed_axis[i]);
            for (int64_t i = 0; i < s.n_prescribed; ++i) {
                PrescribedRamp<Real> r;
                r.nodes = {s.presc_node[i]};
                r.axis = s.presc_axis[i];
                r.target = Real(s.presc_target[i]);
                r.t_total = Real(s.presc_t_total[i]);
                bcs.prescribed.push_back(r);
            }
        }
        bc = DofConstraints<Real>::build(bcs, mesh.num_nodes());
    }
};

template <class Real>
int image_impl(const djg_scenario_spec& s, const djg_image_ptrs* o, djg_image_scalars* sc) {
    RefProblem<Real> P(s, 0);
    const auto& mesh = P.mesh;
    const long N = mesh.num_nodes(), E = mesh.num_elements();
    const int npe = mesh.npe();
    const auto& elems = P.dj->model().elems;
    const auto coeffs = UpdateCoeffs<Real>::build(P.mass, P.dt, P.alpha);
    if (sc) {
        sc->num_nodes = N;
        sc->num_elements = E;
        sc->npe = npe;
        sc->dt = double(P.dt);
        sc->critical_dt = double(P.crit);
        sc->alpha = double(P.alpha);
        sc->c2 = double(coeffs.c2);
        sc->c3 = double(coeffs.c3);
        sc->ramp_t_total = double(P.ramp_t_total);
        sc->wave_speed = double(P.c_wave);
    }
    if (!o) return 0;
    if (o->nodes) {
        Real* d = static_cast<Real*>(o->nodes);
        for (long n = 0; n < N; ++n)
            for (int i = 0; i < 3; ++i) d[3 * n + i] = mesh.nodes[size_t(n)][i];
    }
    if (o->conn) std::memcpy(o->conn, mesh.conn.data(), mesh.conn.size() * sizeof(int));
    const auto adj = NodeElementAdjacency::build(mesh);
    if (o->csr_offsets)
        for (size_t i = 0; i < adj.offsets.size(); ++i) o->csr_offsets[i] = adj.offsets[i];
    for (size_t i = 0; i < adj.pairs.size(); ++i) {
        if (o->csr_elem) o->csr_elem[i] = adj.pairs[i].first;
        if (o->csr_local) o->csr_local[i] = adj.pairs[i].second;
    }
    if (o->consts) {
        // Canonical record order of include/djg.h.
        const auto need = P.mat.needs();
        Real* d = static_cast<Real*>(o->consts);
        size_t w = 0;
        for (long e = 0; e < E; ++e) {
            const auto& ec = elems[size_t(e)];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) d[w++] = ec.J0.m[i][j];
            d[w++] = ec.det_J0;
            d[w++] = ec.V0;
            for (int k = 0; k < 6; ++k) d[w++] = ec.m1[k];
            const Real i1[6] = {ec.I1m.xx, ec.I1m.yy, ec.I1m.zz, ec.I1m.xy, ec.I1m.xz, ec.I1m.yz};
            for (Real v : i1) d[w++] = v;
            if (need.i4) {
                for (int k = 0; k < 6; ++k) d[w++] = ec.m4[k];
                const Real t[6] = {ec.I4m.xx, ec.I4m.yy, ec.I4m.zz, ec.I4m.xy, ec.I4m.xz, ec.I4m.yz};
                for (Real v : t) d[w++] = v;
            }
            if (need.i6) {
                for (int k = 0; k < 6; ++k) d[w++] = ec.m6[k];
                const Real t[6] = {ec.I6m.xx, ec.I6m.yy, ec.I6m.zz, ec.I6m.xy, ec.I6m.xz, ec.I6m.yz};
                for (Real v : t) d[w++] = v;
            }
            if (need.i2) {
                for (int k = 0; k < 21; ++k) d[w++] = ec.M2.p[size_t(k)];
                for (int k = 0; k < 6; ++k) {
                    const auto& t = ec.I2m[size_t(k)];
                    const Real v6[6] = {t.xx, t.yy, t.zz, t.xy, t.xz, t.yz};
                    for (Real v : v6) d[w++] = v;
                }
            }
            if (mesh.kind == ElementKind::H8) {
                d[w++] = ec.k_hg;
                for (int m = 0; m < 4; ++m)
                    for (int a = 0; a < 8; ++a) d[w++] = ec.hg_gamma[size_t(m)][size_t(a)];
            }
        }
        if (sc) sc->nconst = int32_t(w / size_t(E > 0 ? E : 1));
    }
    auto put = [](void* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    put(o->mass, P.mass);
    put(o->c1, coeffs.c1);
    put(o->massless, coeffs.massless);
    put(o->dof_kind, P.bc.kind);
    put(o->dof_target, P.bc.target);
    put(o->dof_t_total, P.bc.t_total);
    return 0;
}

// Explicit step count loop over the reference's advance_step with
// run_simulation's failure semantics (solver.hpp:225-239).
template <class Real, class Engine>
int run_loop(RefProblem<Real>& P, Engine& eng, int64_t steps, int threads, const Real* u0, const Real* up0,
             Real* u_out, Real* up_out, djg_report* rep, double* seconds, int64_t untimed = 0) {
    const long ndof = P.mesh.num_dofs();
    auto state = SimState<Real>::rest(ndof);
    if (u0) std::memcpy(state.u_curr.data(), u0, size_t(ndof) * sizeof(Real));
    if (up0) std::memcpy(state.u_prev.data(), up0, size_t(ndof) * sizeof(Real));
    const auto coeffs = UpdateCoeffs<Real>::build(P.mass, P.dt, P.alpha);
    std::vector<Real> scratch(static_cast<size_t>(ndof), Real(0));
    djg_report r{};
    r.first_inverted = -1;
    r.fail_step = -1;
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t s = 0; s < steps; ++s) {
        if (s == untimed) t0 = std::chrono::steady_clock::now();
        const StepOutcome oc = advance_step(state, eng, coeffs, P.bc, P.dt, threads, P.policy, scratch);
        r.inverted_count += oc.inverted_count;
        if (oc.inverted_count > 0) ++r.inverted_steps;
        if (!oc.ok) {
            r.fail_step = state.step + 1;
            if (oc.diverged) {
                r.diverged = 1;
                r.status = DJG_E_DIVERGENCE;
            } else {
                r.first_inverted = oc.inverted_element;
                r.status = DJG_E_INVERSION;
            }
            break;
        }
        ++r.steps_done;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    r.step = state.step;
    if (u_out) std::memcpy(u_out, state.u_curr.data(), size_t(ndof) * sizeof(Real));
    if (up_out) std::memcpy(up_out, state.u_prev.data(), size_t(ndof) * sizeof(Real));
    if (rep) *rep = r;
    return r.status;
}

template <class Real>
int run_impl(const djg_scenario_spec& s, int64_t steps, int threads, int engine, const void* u0, const void* up0,
             void* u_out, void* up_out, djg_report* rep, double* seconds) {
    RefProblem<Real> P(s, engine);
    auto* a = static_cast<const Real*>(u0);
    auto* b = static_cast<const Real*>(up0);
    auto* c = static_cast<Real*>(u_out);
    auto* d = static_cast<Real*>(up_out);
    if (engine == 1) return run_loop(P, *P.tled, steps, threads, a, b, c, d, rep, seconds);
    return run_loop(P, *P.dj, steps, threads, a, b, c, d, rep, seconds);
}

template <class Real>
int assemble_impl(const djg_scenario_spec& s, int threads, int engine, const void* u, void* f,
                  djg_assemble_stats* st) {
    RefProblem<Real> P(s, engine);
    const long ndof = P.mesh.num_dofs();
    std::vector<Real> uu(static_cast<const Real*>(u), static_cast<const Real*>(u) + ndof), ff(size_t(ndof), Real(0));
    AssembleStats a = engine == 1 ? P.tled->assemble(uu, ff, threads, P.policy) : P.dj->assemble(uu, ff, threads, P.policy);
    if (st) {
        st->first_inverted = a.first_inverted;
        st->inverted_count = a.inverted_count;
    }
    if (a.ok()) std::memcpy(f, ff.data(), size_t(ndof) * sizeof(Real));
    return a.ok() ? 0 : DJG_E_INVERSION;
}

// Single-element DJ (engine 0) or TLED (engine 1) force, the library-level
// chain of tests/test_forces.cpp:29-57 (+ hourglass for H8 like assemble).
template <class Real>
int element_impl(int kind_i, const djg_material_params& mp, double c_hg, const double* x, const double* u, double* f,
                 int engine) {
    const ElementKind kind = kind_i == DJG_T4 ? ElementKind::T4 : ElementKind::H8;
    const auto D = shape_derivatives<Real>(kind);
    const auto mat = make_material<Real>(mp);
    Vec3<Real> coords[8], ue[8];
    for (int a = 0; a < D.n; ++a) {
        coords[a] = {Real(x[3 * a]), Real(x[3 * a + 1]), Real(x[3 * a + 2])};
        ue[a] = {Real(u[3 * a]), Real(u[3 * a + 1]), Real(u[3 * a + 2])};
    }
    ElementForces<Real> ef;
    const bool i57 = mp.model == DJG_I57;
    auto need = mat.needs();
    FibreDirections<Real> fib;
    const FibreDirections<Real>* fp = nullptr;
    if (i57) {  // test_forces.cpp:253-257
        if (engine != 0) throw ConfigError("I57 has no TLED form");
        need.i5 = need.i7 = true;
        const Vec3<Real> a{Real(mp.fibre_a[0]), Real(mp.fibre_a[1]), Real(mp.fibre_a[2])};
        const Vec3<Real> b{Real(mp.fibre_b[0]), Real(mp.fibre_b[1]), Real(mp.fibre_b[2])};
        fib = FibreDirections<Real>::from(a, &b);
        fp = &fib;
    } else if (need.any_fibre_a() || need.any_fibre_b()) {
        fib = mat.fibres();
        fp = &fib;
    }
    if (engine == 0) {
        const auto ec = build_element_constants(coords, D, need, fp, mat.kappa, Real(c_hg));
        ElementKinematics<Real> kin;
        if (!update_kinematics(ec, ue, D, need, kin)) return DJG_E_INVERSION;
        EnergyDerivatives<Real> dv = energy_derivatives(mat, kin.inv);
        if (i57) {  // test_forces.cpp:262-268, in Real
            dv.dI5 = Real(mp.eta_a) * (kin.inv.Ib5 - 1);
            dv.dI7 = Real(mp.eta_b) * (kin.inv.Ib7 - 1);
        }
        ef = element_force(ec, kin, dv, need, D);
        if (ec.has_hourglass) hourglass_force(ec.hg_gamma, ec.k_hg, ue, ef);
    } else {
        const auto j0 = jacobian0(coords, D);
        TledElementConstants<Real> tc;
        tc.V0 = volume0(j0, D.kind);
        for (int a = 0; a < D.n; ++a)
            for (int j = 0; j < 3; ++j)
                tc.B0[a][j] = j0.Jinv.m[j][0] * D.d[0][a] + j0.Jinv.m[j][1] * D.d[1][a] + j0.Jinv.m[j][2] * D.d[2][a];
        DeformationState<Real> st;
        if (!deformation_state(deformation_gradient(ue, tc, D.n), st)) return DJG_E_INVERSION;
        const auto inv = conventional_invariants(st, fp, need);
        const auto S = second_pk_stress(energy_derivatives(mat, inv), need, st, inv, fp);
        ef = tled_element_force(st.X, S, tc, D.n);
        if (kind == ElementKind::H8) {
            tc.hg_gamma = hourglass_vectors(coords, D, j0.Jinv);
            tc.k_hg = Real(c_hg) * mat.kappa * std::cbrt(tc.V0);
            hourglass_force(tc.hg_gamma, tc.k_hg, ue, ef);
        }
    }
    for (int a = 0; a < D.n; ++a)
        for (int i = 0; i < 3; ++i) f[3 * a + i] = double(ef.f[size_t(a)][i]);
    return 0;
}

// bench::detail::time_steps protocol (bench.hpp:42-97) on the scenario:
// warmup untimed steps, then mean seconds per timed step.
template <class Real>
double time_impl(const djg_scenario_spec& s, int64_t warmup, int64_t steps, int threads, int engine) {
    RefProblem<Real> P(s, engine);
    double secs = 0;
    djg_report r{};
    const Real* none = nullptr;
    Real* out = nullptr;
    if (engine == 1)
        run_loop(P, *P.tled, warmup + steps, threads, none, none, out, out, &r, &secs, warmup);
    else
        run_loop(P, *P.dj, warmup + steps, threads, none, none, out, out, &r, &secs, warmup);
    if (r.status != 0) throw SimulationError(SimulationError::Kind::Divergence, "timed run failed", r.fail_step);
    return steps > 0 ? secs / double(steps) : 0.0;
}

// The SURVEY §8(d) CPU protocol on ONE built problem (cfg5 takes tens of
// seconds to build): engine 0 (DjEngine) or 2 (TledEngine, built with
// build_threads like the DjEngine), then for each i: warmup[i] untimed +
// steps[i] timed advance_step calls with threads[i] threads, from rest.
// secs[i] = mean seconds per timed step; *build_s = problem build time.
template <class Real>
int protocol_impl(const djg_scenario_spec& s, int engine, int build_threads, int n, const int32_t* threads,
                  const int64_t* warmup, const int64_t* steps, double* secs, double* build_s) {
    const auto t0 = std::chrono::steady_clock::now();
    RefProblem<Real> P(s, engine == 0 ? 0 : 2, build_threads);
    *build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const Real* none = nullptr;
    Real* out = nullptr;
    for (int i = 0; i < n; ++i) {
        djg_report r{};
        double sec = 0;
        if (engine == 0)
            run_loop(P, *P.dj, warmup[i] + steps[i], threads[i], none, none, out, out, &r, &sec, warmup[i]);
        else
            run_loop(P, *P.tled, warmup[i] + steps[i], threads[i], none, none, out, out, &r, &sec, warmup[i]);
        if (r.status != 0) throw SimulationError(SimulationError::Kind::Divergence, "timed run failed", r.fail_step);
        secs[i] = steps[i] > 0 ? sec / double(steps[i]) : 0.0;
    }
    return 0;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const SimulationError& e) {
        g_err = e.what();
        return e.kind() == SimulationError::Kind::Divergence ? DJG_E_DIVERGENCE : DJG_E_INVERSION;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DJG_E_CONFIG;
    }
}

}  // namespace

extern "C" {

const char* djref_error(void) { return g_err.c_str(); }

int djref_image(const djg_scenario_spec* s, const djg_image_ptrs* o, djg_image_scalars* sc) {
    return guarded([&] { return s->precision == 4 ? image_impl<float>(*s, o, sc) : image_impl<double>(*s, o, sc); });
}

int djref_run(const djg_scenario_spec* s, int64_t steps, int32_t threads, int32_t engine, const void* u0,
              const void* up0, void* u_out, void* up_out, djg_report* rep, double* seconds) {
    return guarded([&] {
        return s->precision == 4 ? run_impl<float>(*s, steps, threads, engine, u0, up0, u_out, up_out, rep, seconds)
                                 : run_impl<double>(*s, steps, threads, engine, u0, up0, u_out, up_out, rep, seconds);
    });
}

int djref_assemble(const djg_scenario_spec* s, int32_t threads, int32_t engine, const void* u, void* f,
                   djg_assemble_stats* st) {
    return guarded([&] {
        return s->precision == 4 ? assemble_impl<float>(*s, threads, engine, u, f, st)
                                 : assemble_impl<double>(*s, threads, engine, u, f, st);
    });
}

int djref_element_force(int32_t precision, int32_t kind, const djg_material_params* m, double c_hg,
                        const double* coords, const double* u, double* f, int32_t engine) {
    return guarded([&] {
        return precision == 4 ? element_impl<float>(kind, *m, c_hg, coords, u, f, engine)
                              : element_impl<double>(kind, *m, c_hg, coords, u, f, engine);
    });
}

double djref_time_steps(const djg_scenario_spec* s, int64_t warmup, int64_t steps, int32_t threads, int32_t engine) {
    double r = -1;
    guarded([&] {
        r = s->precision == 4 ? time_impl<float>(*s, warmup, steps, threads, engine)
                              : time_impl<double>(*s, warmup, steps, threads, engine);
        return 0;
    });
    return r;
}

int djref_time_protocol(const djg_scenario_spec* s, int32_t engine, int32_t build_threads, int32_t n,
                        const int32_t* threads, const int64_t* warmup, const int64_t* steps, double* secs,
                        double* build_s) {
    return guarded([&] {
        return s->precision == 4 ? protocol_impl<float>(*s, engine, build_threads, n, threads, warmup, steps, secs, build_s)
                                 : protocol_impl<double>(*s, engine, build_threads, n, threads, warmup, steps, secs, build_s);
    });
}

int djref_max_threads(void) { return hardware_threads(); }

}  // extern "C"
