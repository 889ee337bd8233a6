// djg.hpp — header-only C++ layer over libdjg's C-ABI that mirrors the
// reference's solver API (/root/reference/proj/include/djtled/solver.hpp),
// so a caller of the reference swaps engines without touching its loop:
//
//   djtled::DjEngine<Real> eng(mesh, material);          // solver.hpp:264
//   djg::GpuDjEngine<Real> eng(mesh, material);          // this header
//
// * GpuDjEngine satisfies the reference's duck-typed Engine concept
//   (assemble(u, f, threads, policy) -> .ok()/.first_inverted/.inverted_count),
//   so the reference's own advance_step / run_simulation accept it unchanged
//   (per-step state round trip over PCIe).
// * djg::run_simulation(engine, node_mass, bc, params) is the device-resident
//   run loop (solver.hpp:205-258): state stays in HBM, one launch graph per
//   32 steps, failures reported like SimulationError.
//
// The mesh / material / constraint / params arguments are duck-typed: the
// reference's Mesh<Real>, Material<Real>, DofConstraints<Real> and
// RunParams<Real> work as they are (C++20).
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "djg.h"

namespace djg {

// Status != DJG_OK from the library (ConfigError / CUDA failures).
class Error : public std::runtime_error {
public:
    Error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
    int status() const { return status_; }

private:
    int status_;
};

// SimulationError (core.hpp:44-57): kind + inverted element id or failing step.
class SimulationError : public std::runtime_error {
public:
    enum class Kind { ElementInversion, Divergence };
    SimulationError(Kind kind, const std::string& what, long index)
        : std::runtime_error(what), kind_(kind), index_(index) {}
    Kind kind() const { return kind_; }
    long index() const { return index_; }

private:
    Kind kind_;
    long index_;
};

// AssembleStats (djtled_force.hpp:99-103). Converts to any stats type with
// the same two fields, so `const djtled::AssembleStats s = engine.assemble(...)`
// inside the reference's advance_step (solver.hpp:104) compiles unchanged.
struct AssembleStats {
    long first_inverted = -1;
    long inverted_count = 0;
    bool ok() const { return first_inverted < 0; }

    template <class T>
        requires requires(T t) {
            t.first_inverted = 0;
            t.inverted_count = 0;
        }
    operator T() const {
        T t{};
        t.first_inverted = first_inverted;
        t.inverted_count = inverted_count;
        return t;
    }
};

namespace detail {

inline void check(int rc, djg_engine* eng) {
    if (rc == DJG_OK || rc == DJG_E_INVERSION || rc == DJG_E_DIVERGENCE) return;
    throw Error(rc, eng ? djg_last_error(eng) : djg_create_error());
}

template <class V>
double comp(const V& v, int i) {
    if constexpr (requires { v.x; }) {
        return double(i == 0 ? v.x : (i == 1 ? v.y : v.z));
    } else {
        return double(v[i]);
    }
}

template <class MaterialT>
djg_material_params material_params(const MaterialT& m) {
    djg_material_params p{};
    p.model = static_cast<int32_t>(m.model);  // NH, TI, OT, MR in both enums
    p.mu = double(m.mu);
    p.kappa = double(m.kappa);
    p.rho = double(m.rho);
    p.eta_a = double(m.eta_a);
    p.eta_b = double(m.eta_b);
    p.c10 = double(m.c10);
    p.c01 = double(m.c01);
    for (int i = 0; i < 3; ++i) {
        p.fibre_a[i] = comp(m.fibre_a, i);
        p.fibre_b[i] = comp(m.fibre_b, i);
    }
    return p;
}

}  // namespace detail

template <class Real>
class GpuDjEngine {
public:
    // DjEngine(mesh, material, c_hg, build_threads) (solver.hpp:264-267).
    template <class MeshT, class MaterialT>
    GpuDjEngine(const MeshT& mesh, const MaterialT& material, Real c_hg = Real(0.1), int build_threads = 0,
                int device = 0, uint32_t flags = 0) {
        std::vector<Real> xyz;
        xyz.reserve(mesh.nodes.size() * 3);
        for (const auto& p : mesh.nodes)
            for (int i = 0; i < 3; ++i) xyz.push_back(Real(detail::comp(p, i)));
        djg_mesh_desc d{};
        d.precision = int32_t(sizeof(Real));
        d.kind = static_cast<int32_t>(mesh.kind);  // T4 = 0, H8 = 1 in both enums
        d.num_nodes = int64_t(mesh.nodes.size());
        d.num_elements = int64_t(mesh.conn.size()) / (d.kind == DJG_T4 ? 4 : 8);
        d.nodes = xyz.data();
        d.conn = reinterpret_cast<const int32_t*>(mesh.conn.data());
        d.material = detail::material_params(material);
        d.c_hg = double(c_hg);
        d.inversion_policy = DJG_ABORT;
        d.device = device;
        d.flags = flags;
        d.threads = build_threads;
        static_assert(sizeof(mesh.conn[0]) == 4, "connectivity must be 32-bit");
        const int rc = djg_create_from_mesh(&d, &eng_);
        if (rc != DJG_OK) throw Error(rc, djg_create_error());
        num_dofs_ = 3 * d.num_nodes;
    }

    GpuDjEngine(const GpuDjEngine&) = delete;
    GpuDjEngine& operator=(const GpuDjEngine&) = delete;
    GpuDjEngine(GpuDjEngine&& o) noexcept : eng_(std::exchange(o.eng_, nullptr)), num_dofs_(o.num_dofs_) {}
    ~GpuDjEngine() {
        if (eng_) djg_destroy(eng_);
    }

    // lump_mass(mesh, material.rho, elems) (precompute.hpp:275-287) computed on
    // the device -- engines built with DJG_FLAG_DEVICE_PRECOMPUTE. Bit-identical.
    std::vector<Real> lump_mass() const {
        std::vector<Real> m(size_t(num_dofs_ / 3));
        detail::check(djg_lump_mass(eng_, m.data()), eng_);
        return m;
    }
    // critical_dt(mesh, elems, wave_speed) (precompute.hpp:323-331): the minimum
    // characteristic length from the device over wave_speed, in Real.
    Real critical_dt(Real wave_speed) const {
        double l = 0;
        detail::check(djg_min_char_length(eng_, &l), eng_);
        return Real(l) / wave_speed;
    }

    // Engine::assemble (solver.hpp:269-272): internal forces at u. Under Abort
    // with an inverted element f is left untouched, like assemble_internal.
    template <class Policy>
    AssembleStats assemble(const std::vector<Real>& u, std::vector<Real>& f, int /*threads*/, Policy policy) {
        set_policy(static_cast<int>(policy));
        f.resize(u.size());
        djg_assemble_stats st{};
        detail::check(djg_assemble(eng_, u.data(), f.data(), &st), eng_);
        return {long(st.first_inverted), long(st.inverted_count)};
    }
    AssembleStats assemble(const std::vector<Real>& u, std::vector<Real>& f, int threads = 1) {
        return assemble(u, f, threads, DJG_ABORT);
    }

    // UpdateCoeffs::build(node_mass, dt, alpha) + DofConstraints.
    template <class DofT>
    void configure(const std::vector<Real>& node_mass, const DofT& bc, Real dt, Real alpha) {
        djg_step_desc s{};
        s.node_mass = node_mass.data();
        s.dof_kind = bc.kind.empty() ? nullptr : reinterpret_cast<const uint8_t*>(bc.kind.data());
        s.dof_target = bc.target.empty() ? nullptr : bc.target.data();
        s.dof_t_total = bc.t_total.empty() ? nullptr : bc.t_total.data();
        s.dt = double(dt);
        s.alpha = double(alpha);
        detail::check(djg_configure_step(eng_, &s), eng_);
    }

    void set_policy(int policy) {
        if (policy != policy_) {
            detail::check(djg_set_policy(eng_, policy), eng_);
            policy_ = policy;
        }
    }

    void set_state(const std::vector<Real>* u_curr, const std::vector<Real>* u_prev, long step) {
        detail::check(djg_set_state(eng_, u_curr ? u_curr->data() : nullptr, u_prev ? u_prev->data() : nullptr, step),
                      eng_);
    }

    void set_external(const std::vector<Real>* r_ext) {
        detail::check(djg_set_external(eng_, r_ext ? r_ext->data() : nullptr), eng_);
    }

    // nsteps x advance_step on the device; returns the report (no throw).
    djg_report step(long nsteps) {
        djg_report r{};
        detail::check(djg_step(eng_, nsteps, &r), eng_);
        return r;
    }

    long get_state(std::vector<Real>& u_curr, std::vector<Real>& u_prev) {
        u_curr.resize(size_t(num_dofs_));
        u_prev.resize(size_t(num_dofs_));
        int64_t step = 0;
        detail::check(djg_get_state(eng_, u_curr.data(), u_prev.data(), &step), eng_);
        return long(step);
    }

    djg_engine* handle() { return eng_; }
    long num_dofs() const { return long(num_dofs_); }
    static constexpr const char* name() { return "djtled-b200"; }

private:
    djg_engine* eng_ = nullptr;
    int64_t num_dofs_ = 0;
    int policy_ = DJG_ABORT;
};

// TledEngine(mesh, material, c_hg, build_threads) (solver.hpp:287-300): the
// conventional total Lagrangian element forces (tled_force.hpp) on the device,
// with the same slots, gather, update and run loop; its record (B0, V0, and
// for H8 the hourglass data) is built on the GPU.
template <class Real>
class GpuTledEngine : public GpuDjEngine<Real> {
public:
    template <class MeshT, class MaterialT>
    GpuTledEngine(const MeshT& mesh, const MaterialT& material, Real c_hg = Real(0.1), int build_threads = 0,
                  int device = 0, uint32_t flags = 0)
        : GpuDjEngine<Real>(mesh, material, c_hg, build_threads, device, flags | DJG_FLAG_TLED) {}
    static constexpr const char* name() { return "tled-b200"; }
};

// SimState / RunResult (solver.hpp:41-57, 193-200).
template <class Real>
struct SimState {
    std::vector<Real> u_curr, u_prev;
    Real t = 0;
    long step = 0;
};

template <class Real>
struct RunResult {
    SimState<Real> state;
    long steps = 0;
    double wall_seconds = 0;
    double mean_step_seconds = 0;
    long inverted_steps = 0;
};

// advance_step (solver.hpp:98-153) on a host SimState through the GPU engine
// (djg_advance_host): one step with the engine's configured coefficients,
// constraints and dt. On success the state rotates (u_prev <- u_curr <- new,
// step + 1, t = dt * step); on failure it is unchanged and the report says why.
template <class Real>
djg_report advance_step(GpuDjEngine<Real>& engine, SimState<Real>& state, Real dt) {
    std::vector<Real> next(state.u_curr.size());
    djg_report r{};
    const int rc = djg_advance_host(engine.handle(), state.u_curr.data(), state.u_prev.data(), state.step, next.data(),
                                    &r);
    if (rc != DJG_OK && rc != DJG_E_INVERSION && rc != DJG_E_DIVERGENCE)
        throw Error(rc, djg_last_error(engine.handle()));
    if (rc == DJG_OK) {
        state.u_prev.swap(state.u_curr);
        state.u_curr.swap(next);
        state.step = long(r.step);
        state.t = dt * Real(state.step);
    }
    return r;
}

// run_simulation (solver.hpp:205-258) with the state resident on the B200.
// `hook(step, t, max_abs_u, seconds_per_step)` is called every
// p.report_stride steps and at the end, like the reference's progress hook.
template <class Real, class DofT, class ParamsT>
RunResult<Real> run_simulation(GpuDjEngine<Real>& engine, const std::vector<Real>& node_mass, const DofT& bc,
                               const ParamsT& p,
                               const std::function<void(long, Real, Real, double)>& hook = {},
                               const SimState<Real>* initial = nullptr) {
    if (!(p.dt > Real(0))) throw Error(DJG_E_CONFIG, "time step must be positive");
    if (p.t_end < Real(0)) throw Error(DJG_E_CONFIG, "t_end must be >= 0");
    const long num_steps = long(std::ceil(double(p.t_end) / double(p.dt) - 1e-9));
    engine.configure(node_mass, bc, p.dt, p.alpha);
    engine.set_policy(static_cast<int>(p.on_inversion));
    if (initial) engine.set_state(&initial->u_curr, &initial->u_prev, initial->step);
    else engine.set_state(nullptr, nullptr, 0);
    RunResult<Real> result;
    const long stride = (hook && p.report_stride > 0) ? long(p.report_stride) : num_steps;
    const auto t0 = std::chrono::steady_clock::now();
    auto last = t0;
    long done = 0;
    while (done < num_steps) {
        const long n = std::min(stride > 0 ? stride : num_steps, num_steps - done);
        const djg_report r = engine.step(n);
        done += r.steps_done;
        result.inverted_steps += long(r.inverted_steps);
        if (r.status == DJG_E_DIVERGENCE)
            throw SimulationError(SimulationError::Kind::Divergence,
                                  "solution diverged at step " + std::to_string(r.fail_step) + "; reduce the time step",
                                  long(r.fail_step));
        if (r.status == DJG_E_INVERSION)
            throw SimulationError(SimulationError::Kind::ElementInversion,
                                  "element " + std::to_string(r.first_inverted) + " inverted at step " +
                                      std::to_string(r.fail_step),
                                  long(r.first_inverted));
        if (hook && p.report_stride > 0) {
            std::vector<Real> u, up;
            const long step = engine.get_state(u, up);
            Real mx = 0;
            for (Real v : u) mx = std::max(mx, std::abs(v));
            const auto now = std::chrono::steady_clock::now();
            hook(step, p.dt * Real(step), mx, std::chrono::duration<double>(now - last).count() / double(n));
            last = now;
        }
    }
    result.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    result.state.step = engine.get_state(result.state.u_curr, result.state.u_prev);
    result.state.t = p.dt * Real(result.state.step);
    result.steps = result.state.step;
    result.mean_step_seconds = num_steps > 0 ? result.wall_seconds / double(num_steps) : 0;
    return result;
}

}  // namespace djg
