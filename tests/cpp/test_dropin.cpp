// TEST INFRASTRUCTURE: proves the drop-in boundary from the reference side.
// Compiled against the UNMODIFIED reference headers plus include/djg.hpp and
// linked to libdjg.so (tests/cpp/Makefile). Three runs of the same problem:
//   cpu  : djtled::DjEngine + djtled::run_simulation           (reference)
//   seam : djg::GpuDjEngine + djtled::run_simulation           (reference loop,
//          GPU forces through the Engine::assemble seam)
//   gpu  : djg::GpuDjEngine + djg::run_simulation              (device resident)
// and the reference's failure semantics through both loops.
#include <cstdio>
#include <cstdlib>

#include "djg.hpp"
#include "djtled/bench.hpp"
#include "djtled/solver.hpp"

using namespace djtled;

static int g_fail = 0;
#define EXPECT(cond, ...)                       \
    do {                                        \
        if (!(cond)) {                          \
            std::printf("FAIL: " __VA_ARGS__);  \
            std::printf("\n");                  \
            ++g_fail;                           \
        }                                       \
    } while (0)

template <class Real>
double rel_err(const std::vector<Real>& a, const std::vector<Real>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::abs(double(a[i]) - double(b[i])));
        den = std::max(den, std::abs(double(b[i])));
    }
    return den > 0 ? num / den : num;
}

template <class Real>
void compare_runs(ElementKind kind, MaterialModel model, int div, long steps, double tol) {
    const auto mesh = generate_box<Real>({1, 1, 1}, {div, div, div}, kind);
    const auto mat = bench_material<Real>(model);
    DjEngine<Real> cpu(mesh, mat);
    djg::GpuDjEngine<Real> gpu(mesh, mat);
    const auto mass = lump_mass(mesh, mat.rho, cpu.model().elems);
    BoundaryConditions<Real> bcs;
    for (int n : select_plane_nodes(mesh, Plane::ZMin))
        for (int a = 0; a < 3; ++a) bcs.fixed.emplace_back(n, a);
    RunParams<Real> p;
    p.dt = Real(0.5) * critical_dt(mesh, cpu.model().elems, dilatational_wave_speed(mat));
    p.t_end = p.dt * Real(steps);
    p.alpha = relaxation_alpha(mat, mesh);
    PrescribedRamp<Real> ramp;
    ramp.nodes = select_plane_nodes(mesh, Plane::ZMax);
    ramp.axis = 2;
    ramp.target = Real(-0.2);
    ramp.t_total = p.t_end;
    bcs.prescribed.push_back(ramp);
    const auto bc = DofConstraints<Real>::build(bcs, mesh.num_nodes());

    const auto r_cpu = djtled::run_simulation(cpu, mass, bc, p);
    const auto r_seam = djtled::run_simulation(gpu, mass, bc, p);
    const auto r_gpu = djg::run_simulation(gpu, mass, bc, p);
    const double e_seam = rel_err(r_seam.state.u_curr, r_cpu.state.u_curr);
    const double e_gpu = rel_err(r_gpu.state.u_curr, r_cpu.state.u_curr);
    // the same run as a host loop of djg::advance_step (djg_advance_host)
    djg::SimState<Real> hs;
    hs.u_curr.assign(size_t(mesh.num_dofs()), Real(0));
    hs.u_prev = hs.u_curr;
    for (long k = 0; k < r_cpu.steps; ++k) {
        const djg_report rr = djg::advance_step(gpu, hs, p.dt);
        EXPECT(rr.status == DJG_OK, "host-state step failed");
    }
    const double e_host = rel_err(hs.u_curr, r_cpu.state.u_curr);
    EXPECT(e_host <= tol, "host-state loop differs: %.3e", e_host);
    std::printf("%s-%s d=%d f%zu steps=%ld: seam %.3e  device %.3e  (max|u| %.4f)\n", to_string(kind),
                to_string(model), div, 8 * sizeof(Real), r_cpu.steps, e_seam, e_gpu,
                [&] { double m = 0; for (Real v : r_cpu.state.u_curr) m = std::max(m, std::abs(double(v))); return m; }());
    EXPECT(r_cpu.steps == r_seam.steps && r_cpu.steps == r_gpu.steps, "step counts differ");
    EXPECT(e_seam <= tol, "seam run differs: %.3e", e_seam);
    EXPECT(e_gpu <= tol, "device run differs: %.3e", e_gpu);
    EXPECT(std::abs(double(r_gpu.state.t) - double(r_cpu.state.t)) == 0.0, "final time differs");
}

template <class Real>
void inversion_semantics() {
    // tests/test_solver.cpp:214-241
    const auto mesh = generate_box<Real>({Real(0.1), Real(0.1), Real(0.1)}, {1, 1, 1}, ElementKind::T4);
    const auto mat = bench_material<Real>(MaterialModel::NeoHookean);
    DjEngine<Real> cpu(mesh, mat);
    djg::GpuDjEngine<Real> gpu(mesh, mat);
    const auto mass = lump_mass(mesh, mat.rho, cpu.model().elems);
    BoundaryConditions<Real> bcs;
    for (int n : select_plane_nodes(mesh, Plane::ZMin))
        for (int a = 0; a < 3; ++a) bcs.fixed.emplace_back(n, a);
    PrescribedRamp<Real> ramp;
    ramp.nodes = select_plane_nodes(mesh, Plane::ZMax);
    ramp.axis = 2;
    ramp.target = Real(-0.5);
    ramp.t_total = Real(1e-4);
    bcs.prescribed.push_back(ramp);
    const auto bc = DofConstraints<Real>::build(bcs, mesh.num_nodes());
    RunParams<Real> p;
    p.dt = Real(1e-4);
    p.t_end = Real(0.01);
    p.alpha = 0;
    long cpu_index = -2, seam_index = -3, gpu_index = -4;
    try { djtled::run_simulation(cpu, mass, bc, p); } catch (const djtled::SimulationError& e) { cpu_index = e.index(); }
    try { djtled::run_simulation(gpu, mass, bc, p); } catch (const djtled::SimulationError& e) { seam_index = e.index(); }
    try {
        djg::run_simulation(gpu, mass, bc, p);
    } catch (const djg::SimulationError& e) {
        EXPECT(e.kind() == djg::SimulationError::Kind::ElementInversion, "wrong failure kind");
        gpu_index = e.index();
    }
    std::printf("inversion f%zu: cpu element %ld, seam %ld, device %ld\n", 8 * sizeof(Real), cpu_index, seam_index,
                gpu_index);
    EXPECT(cpu_index >= 0 && cpu_index == seam_index && cpu_index == gpu_index, "inverted element ids differ");
    // Skip-and-report keeps going (or diverges), never aborts on inversion.
    p.on_inversion = InversionPolicy::SkipAndReport;
    long inv_steps = -1;
    try {
        inv_steps = djg::run_simulation(gpu, mass, bc, p).inverted_steps;
    } catch (const djg::SimulationError& e) {
        EXPECT(e.kind() == djg::SimulationError::Kind::Divergence, "report policy aborted on inversion");
        inv_steps = 1;
    }
    EXPECT(inv_steps > 0, "no inverted steps reported");
}

// djg::GpuTledEngine in place of djtled::TledEngine, both
// loops, bit-identical.
template <class Real>
void tled_dropin(ElementKind kind, MaterialModel model, int div, long steps) {
    const auto mesh = generate_box<Real>({1, 1, 1}, {div, div, div}, kind);
    const auto mat = bench_material<Real>(model);
    DjEngine<Real> dj(mesh, mat);
    TledEngine<Real> cpu(mesh, mat);
    djg::GpuTledEngine<Real> gpu(mesh, mat);
    const auto mass = lump_mass(mesh, mat.rho, dj.model().elems);
    BoundaryConditions<Real> bcs;
    for (int n : select_plane_nodes(mesh, Plane::ZMin))
        for (int a = 0; a < 3; ++a) bcs.fixed.emplace_back(n, a);
    RunParams<Real> p;
    p.dt = Real(0.5) * critical_dt(mesh, dj.model().elems, dilatational_wave_speed(mat));
    p.t_end = p.dt * Real(steps);
    p.alpha = relaxation_alpha(mat, mesh);
    PrescribedRamp<Real> ramp;
    ramp.nodes = select_plane_nodes(mesh, Plane::ZMax);
    ramp.axis = 2;
    ramp.target = Real(-0.2);
    ramp.t_total = p.t_end;
    bcs.prescribed.push_back(ramp);
    const auto bc = DofConstraints<Real>::build(bcs, mesh.num_nodes());
    const auto r_cpu = djtled::run_simulation(cpu, mass, bc, p);
    const auto r_seam = djtled::run_simulation(gpu, mass, bc, p);
    const auto r_gpu = djg::run_simulation(gpu, mass, bc, p);
    const double e_seam = rel_err(r_seam.state.u_curr, r_cpu.state.u_curr);
    const double e_gpu = rel_err(r_gpu.state.u_curr, r_cpu.state.u_curr);
    std::printf("TLED %s-%s f%zu steps=%ld: seam %.3e  device %.3e\n", to_string(kind), to_string(model),
                8 * sizeof(Real), r_cpu.steps, e_seam, e_gpu);
    EXPECT(e_seam == 0.0 && e_gpu == 0.0, "TLED drop-in differs: %.3e %.3e", e_seam, e_gpu);
}

// the precompute on the device (records, adjacency, slot
// ranks, lump_mass, characteristic lengths) == the reference's host functions.
template <class Real>
void device_precompute(ElementKind kind, MaterialModel model, int div, long steps) {
    const auto mesh = generate_box<Real>({1, 1, 1}, {div, div + 1, div + 2}, kind);
    const auto mat = bench_material<Real>(model);
    DjEngine<Real> cpu(mesh, mat);
    djg::GpuDjEngine<Real> gpu(mesh, mat, Real(0.1), 0, 0, DJG_FLAG_DEVICE_PRECOMPUTE);
    const auto mass = lump_mass(mesh, mat.rho, cpu.model().elems);
    const auto gmass = gpu.lump_mass();
    EXPECT(gmass == mass, "device lump_mass differs from lump_mass");
    const Real c = dilatational_wave_speed(mat);
    const Real dt_cpu = critical_dt(mesh, cpu.model().elems, c);
    EXPECT(gpu.critical_dt(c) == dt_cpu, "device critical_dt differs: %.9g vs %.9g", double(gpu.critical_dt(c)),
           double(dt_cpu));
    BoundaryConditions<Real> bcs;
    for (int n : select_plane_nodes(mesh, Plane::ZMin))
        for (int a = 0; a < 3; ++a) bcs.fixed.emplace_back(n, a);
    RunParams<Real> p;
    p.dt = Real(0.5) * gpu.critical_dt(c);
    p.t_end = p.dt * Real(steps);
    p.alpha = relaxation_alpha(mat, mesh);
    PrescribedRamp<Real> ramp;
    ramp.nodes = select_plane_nodes(mesh, Plane::ZMax);
    ramp.axis = 2;
    ramp.target = Real(-0.2);
    ramp.t_total = p.t_end;
    bcs.prescribed.push_back(ramp);
    const auto bc = DofConstraints<Real>::build(bcs, mesh.num_nodes());
    const auto r_cpu = djtled::run_simulation(cpu, mass, bc, p);
    const auto r_gpu = djg::run_simulation(gpu, gmass, bc, p);
    const double e = rel_err(r_gpu.state.u_curr, r_cpu.state.u_curr);
    std::printf("device precompute %s-%s f%zu: mass %s, dt %s, run %.3e\n", to_string(kind), to_string(model),
                8 * sizeof(Real), gmass == mass ? "equal" : "DIFFER", gpu.critical_dt(c) == dt_cpu ? "equal" : "DIFFER",
                e);
    EXPECT(e == 0.0, "device-precompute run differs: %.3e", e);
}

int main() {
    // Bit-identical to the reference: tolerance 0.
    compare_runs<float>(ElementKind::T4, MaterialModel::NeoHookean, 6, 300, 0.0);
    compare_runs<float>(ElementKind::H8, MaterialModel::TransverseIsotropic, 5, 300, 0.0);
    compare_runs<double>(ElementKind::T4, MaterialModel::MooneyRivlin, 4, 200, 0.0);
    compare_runs<double>(ElementKind::H8, MaterialModel::NeoHookean, 5, 200, 0.0);
    compare_runs<float>(ElementKind::T4, MaterialModel::Orthotropic, 5, 200, 0.0);
    inversion_semantics<double>();
    inversion_semantics<float>();
    tled_dropin<float>(ElementKind::T4, MaterialModel::NeoHookean, 5, 200);
    tled_dropin<double>(ElementKind::H8, MaterialModel::TransverseIsotropic, 4, 150);
    device_precompute<float>(ElementKind::T4, MaterialModel::NeoHookean, 5, 200);
    device_precompute<double>(ElementKind::T4, MaterialModel::TransverseIsotropic, 4, 150);
    device_precompute<float>(ElementKind::H8, MaterialModel::Orthotropic, 4, 150);
    device_precompute<double>(ElementKind::H8, MaterialModel::MooneyRivlin, 3, 100);
    std::printf(g_fail ? "FAILED (%d)\n" : "PASS\n", g_fail);
    return g_fail ? 1 : 0;
}
