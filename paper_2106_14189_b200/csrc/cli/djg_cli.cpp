// djg: command-line front end of the B200 engine with the reference CLI's
// subcommands, options, config files, reports and exit codes
// (tools/djtled_main.cpp): `run`, `compare`, `bench` -- the element forces,
// gather and update on the GPU (libdjg.so), everything else host-side.
//
//   djg run <config> [--precision single|double] [--threads N]
//                    [--on-inversion abort|report] [--strict-stability] [--device N]
//   djg compare <config> ...      DJ-TLED and TLED on identical inputs
//   djg bench <config> ...        both engines over the [bench] ladder
//   djg convert <in> <out> [--precision ...]   text <-> binary mesh (".djgmesh")
//
// Exit codes (djtled_main.cpp:13-20): 0 ok, 1 internal (also CUDA failures),
// 2 config / parse / mesh error, 3 unstable dt with --strict-stability,
// 4 element inversion, 5 divergence.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <omp.h>

#include "djg.h"
#include "djg_host.h"
#include "meshio.hpp"

namespace djg::cli {
namespace {

enum ExitCode : int { kOk = 0, kInternal = 1, kConfig = 2, kStability = 3, kInversion = 4, kDivergence = 5 };

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Options {
    std::string config_path;
    std::string precision = "double";
    int threads = -1;
    std::string on_inversion;
    bool strict_stability = false;
    int device = 0;
};

template <class Real>
RunConfig<Real> load_config(const Options& o) {
    std::ifstream in(o.config_path);
    if (!in) throw ConfigError("cannot open config file '" + o.config_path + "'");
    RunConfig<Real> cfg = parse_config<Real>(in);
    if (o.threads >= 1) cfg.threads = o.threads;
    if (o.on_inversion == "abort") cfg.on_inversion = DJG_ABORT;
    else if (o.on_inversion == "report") cfg.on_inversion = DJG_SKIP_AND_REPORT;
    return cfg;
}

std::string config_dir(const std::string& path) {
    const size_t slash = path.find_last_of('/');
    return slash == std::string::npos ? std::string(".") : path.substr(0, slash);
}

int hardware_threads() { return std::max(1, omp_get_max_threads()); }

// Owns a built scenario (host problem) and the arrays its spec points to.
struct Scenario {
    djg_scenario* sc = nullptr;
    djg_image_scalars s{};
    ~Scenario() {
        if (sc) djg_scenario_free(sc);
    }
};

struct EngineHandle {
    djg_engine* eng = nullptr;
    ~EngineHandle() {
        if (eng) djg_destroy(eng);
    }
};

void build_scenario(const djg_scenario_spec& spec, int threads, Scenario& out) {
    if (djg_scenario_build(&spec, threads, &out.sc) != DJG_OK) throw ConfigError(djg_scenario_error());
    djg_scenario_scalars(out.sc, &out.s);
}

void create_engine(const Scenario& sc, int device, uint32_t flags, EngineHandle& out) {
    djg_desc d;
    djg_scenario_desc(sc.sc, device, &d);
    d.flags = flags;
    const int rc = djg_create(&d, &out.eng);
    if (rc == DJG_E_CUDA) throw CudaFailure(djg_create_error());
    if (rc != DJG_OK) throw ConfigError(djg_create_error());
}

template <class Real>
djg_material_params material_params(const RunConfig<Real>& c) {
    djg_material_params m{};
    m.model = c.model;
    m.mu = double(c.mu);
    m.kappa = double(c.kappa);
    m.rho = double(c.rho);
    m.eta_a = double(c.eta_a);
    m.eta_b = double(c.eta_b);
    m.c10 = double(c.c10);
    m.c01 = double(c.c01);
    for (int i = 0; i < 3; ++i) {
        m.fibre_a[i] = double(c.fibre_a[i]);
        m.fibre_b[i] = double(c.fibre_b[i]);
    }
    return m;
}

// prepare (djtled_main.cpp:72-87) + build_bcs (config.hpp:483-502).
template <class Real>
struct Prepared {
    Mesh<Real> mesh;
    std::vector<double> nodes;
    std::vector<int32_t> fixed_node, fixed_axis, presc_node, presc_axis;
    std::vector<double> presc_target, presc_t_total;
    djg_scenario_spec spec{};
    Scenario sc;
    int threads = 1;
    double precompute_s = 0;
};

template <class Real>
void prepare(const RunConfig<Real>& cfg, const std::string& base_dir, Prepared<Real>& p) {
    const auto t0 = std::chrono::steady_clock::now();
    p.threads = cfg.threads > 0 ? cfg.threads : hardware_threads();
    omp_set_num_threads(p.threads);
    p.mesh = build_mesh(cfg, base_dir);
    Real lo[3], hi[3];
    bounding_box(p.mesh, lo, hi);
    for (const auto& f : cfg.fixes) {
        const int axis = int(f.plane) / 2;
        for (int32_t n : plane_nodes(p.mesh, axis, int(f.plane) % 2 == 1, lo, hi))
            for (int a = 0; a < 3; ++a)
                if (f.axes[a]) {
                    p.fixed_node.push_back(n);
                    p.fixed_axis.push_back(a);
                }
    }
    for (const auto& r : cfg.prescribes) {
        const auto nodes = plane_nodes(p.mesh, int(r.plane) / 2, int(r.plane) % 2 == 1, lo, hi);
        if (nodes.empty()) throw ConfigError("prescribe rule selects no nodes");
        for (int32_t n : nodes) {
            p.presc_node.push_back(n);
            p.presc_axis.push_back(r.axis);
            p.presc_target.push_back(double(r.target));
            p.presc_t_total.push_back(double(r.t_total));
        }
    }
    p.nodes.assign(p.mesh.nodes.begin(), p.mesh.nodes.end());
    djg_scenario_spec& s = p.spec;
    s.precision = int32_t(sizeof(Real));
    s.kind = p.mesh.kind;
    s.num_nodes = p.mesh.num_nodes();
    s.num_elements = p.mesh.num_elements();
    s.nodes = p.nodes.data();
    s.conn = p.mesh.conn.data();
    s.material = material_params(cfg);
    s.c_hg = 0.1;  // DjModel default (precompute.hpp:204)
    s.bc_mode = 2;
    s.n_fixed = int64_t(p.fixed_node.size());
    s.fixed_node = p.fixed_node.data();
    s.fixed_axis = p.fixed_axis.data();
    s.n_prescribed = int64_t(p.presc_node.size());
    s.presc_node = p.presc_node.data();
    s.presc_axis = p.presc_axis.data();
    s.presc_target = p.presc_target.data();
    s.presc_t_total = p.presc_t_total.data();
    s.dt = cfg.dt_auto ? 0.0 : double(cfg.dt);
    s.safety = double(cfg.safety);
    s.alpha_mode = cfg.alpha_relax ? 0 : 1;
    s.alpha = double(cfg.alpha);
    s.policy = cfg.on_inversion;
    build_scenario(s, p.threads, p.sc);
    p.precompute_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int check_stability(const Scenario& sc, bool strict) {
    if (sc.s.dt > sc.s.critical_dt) {
        std::cerr << "warning: dt = " << sc.s.dt << " s exceeds the stability bound " << sc.s.critical_dt << " s"
                  << std::endl;
        if (strict) {
            std::cerr << "error: refusing to run an unstable configuration (--strict-stability)" << std::endl;
            return kStability;
        }
    }
    return kOk;
}

struct SimFailure : std::runtime_error {
    SimFailure(int code, const std::string& what) : std::runtime_error(what), code(code) {}
    int code;
};

template <class Real>
struct RunOutcome {
    std::vector<Real> u;
    long steps = 0;
    double wall_seconds = 0, mean_step_seconds = 0;
    long inverted_steps = 0;
};

// run_simulation (solver.hpp:205-258) on the device: from rest for
// ceil(t_end / dt - 1e-9) steps, progress every frame_stride steps.
template <class Real>
RunOutcome<Real> execute(const Prepared<Real>& p, const RunConfig<Real>& cfg, int device, uint32_t flags) {
    EngineHandle h;
    create_engine(p.sc, device, flags, h);
    const Real dt = Real(p.sc.s.dt);
    const long num_steps = long(std::ceil(double(cfg.t_end) / double(dt) - 1e-9));
    RunOutcome<Real> r;
    const int64_t ndof = 3 * p.mesh.num_nodes();
    r.u.assign(size_t(ndof), Real(0));
    if (djg_set_state(h.eng, nullptr, nullptr, 0) != DJG_OK) throw CudaFailure(djg_last_error(h.eng));
    djg_report rep{};
    const auto t0 = std::chrono::steady_clock::now();
    auto last = t0;
    long done = 0, last_step = 0;
    while (done < num_steps) {
        long chunk = num_steps - done;
        if (cfg.frame_stride > 0) chunk = std::min(chunk, cfg.frame_stride - done % cfg.frame_stride);
        const int rc = djg_step(h.eng, chunk, &rep);
        r.inverted_steps = rep.inverted_steps;
        if (rc == DJG_E_DIVERGENCE)
            throw SimFailure(kDivergence, "solution diverged at step " + std::to_string(rep.fail_step) +
                                              "; reduce the time step");
        if (rc == DJG_E_INVERSION)
            throw SimFailure(kInversion, "element " + std::to_string(rep.first_inverted) + " inverted at step " +
                                             std::to_string(rep.fail_step));
        if (rc == DJG_E_CUDA) throw CudaFailure(djg_last_error(h.eng));
        if (rc != DJG_OK) throw ConfigError(djg_last_error(h.eng));
        done += chunk;
        if (cfg.frame_stride > 0) {
            int64_t step = 0;
            djg_get_state(h.eng, r.u.data(), nullptr, &step);
            Real m = 0;
            for (Real v : r.u) m = std::max(m, std::abs(v));
            const auto now = std::chrono::steady_clock::now();
            const long span = long(step) - last_step;
            const double sps = span > 0 ? std::chrono::duration<double>(now - last).count() / double(span) : 0.0;
            last = now;
            last_step = long(step);
            std::cerr << "  step " << step << "  t=" << dt * Real(step) << " s  max|u|=" << m << " m  " << sps * 1e6
                      << " us/step" << std::endl;
        }
    }
    const auto t1 = std::chrono::steady_clock::now();
    int64_t step = 0;
    if (djg_get_state(h.eng, r.u.data(), nullptr, &step) != DJG_OK) throw CudaFailure(djg_last_error(h.eng));
    r.steps = long(step);
    r.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    r.mean_step_seconds = num_steps > 0 ? r.wall_seconds / double(num_steps) : 0.0;
    return r;
}

std::string with_suffix(const std::string& path, const std::string& suffix) {
    const size_t dot = path.find_last_of('.');
    if (dot == std::string::npos || path.find('/', dot) != std::string::npos) return path + suffix;
    return path.substr(0, dot) + suffix + path.substr(dot);
}

void emit_report(const std::string& text, const std::string& path) {
    if (!path.empty()) {
        std::ofstream out(path);
        if (!out) throw ConfigError("cannot open report file '" + path + "'");
        out << text;
    }
    std::cout << text;
}

template <class Real>
int cmd_run(const Options& o) {
    const auto cfg = load_config<Real>(o);
    if (cfg.engine == Engine::Both) throw ConfigError("engine = both is only valid for 'compare'");
    Prepared<Real> p;
    prepare(cfg, config_dir(o.config_path), p);
    if (const int rc = check_stability(p.sc, o.strict_stability); rc != kOk) return rc;
    std::cerr << "running " << engine_name(cfg.engine) << " on the GPU: " << p.mesh.num_nodes() << " nodes, "
              << p.mesh.num_elements() << " " << kind_name(p.mesh.kind) << " elements, dt=" << Real(p.sc.s.dt) << " s"
              << std::endl;
    const auto r = execute(p, cfg, o.device, cfg.engine == Engine::Tled ? DJG_FLAG_TLED : 0u);
    Real max_disp = 0;
    for (Real v : r.u) max_disp = std::max(max_disp, std::abs(v));
    if (!cfg.field_path.empty()) write_field(cfg.field_path, p.mesh, r.u);
    std::ostringstream rep;
    rep << std::setprecision(12);
    rep << "djtled run report\n";
    rep << "engine " << engine_name(cfg.engine) << "\n";
    rep << "nodes " << p.mesh.num_nodes() << "\n";
    rep << "elements " << p.mesh.num_elements() << "\n";
    rep << "steps " << r.steps << "\n";
    rep << "dt " << Real(p.sc.s.dt) << "\n";
    rep << "dt_critical " << Real(p.sc.s.critical_dt) << "\n";
    rep << "alpha " << Real(p.sc.s.alpha) << "\n";
    rep << "threads " << p.threads << "\n";
    rep << "precompute_s " << p.precompute_s << "\n";
    rep << "wall_total_s " << r.wall_seconds << "\n";
    rep << "mean_step_us " << r.mean_step_seconds * 1e6 << "\n";
    rep << "max_disp " << max_disp << "\n";
    if (r.inverted_steps > 0) rep << "inverted_steps " << r.inverted_steps << "\n";
    emit_report(rep.str(), cfg.report_path);
    return kOk;
}

// rmse / nre / histogram (metrics.hpp:11-62).
template <class Real>
Real rmse(const std::vector<Real>& a, const std::vector<Real>& b) {
    if (a.size() != b.size()) throw ConfigError("rmse: field lengths differ");
    if (a.empty()) throw ConfigError("rmse: empty fields");
    double acc = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double d = double(a[i]) - double(b[i]);
        acc += d * d;
    }
    return Real(std::sqrt(acc / double(a.size())));
}

template <class Real>
std::pair<Real, std::vector<long>> nre_histogram(const std::vector<Real>& a, const std::vector<Real>& b, int buckets) {
    const auto [lo, hi] = std::minmax_element(b.begin(), b.end());
    const Real range = *hi - *lo;
    if (!(range > Real(0))) throw ConfigError("nre: reference field is uniform, range is zero");
    std::vector<Real> v(a.size());
    for (size_t i = 0; i < a.size(); ++i) v[i] = std::abs(a[i] - b[i]) / range;
    std::vector<long> counts(size_t(buckets), 0);
    Real vmax = 0;
    for (Real x : v) vmax = std::max(vmax, x);
    if (vmax <= Real(0)) {
        counts[0] = long(v.size());
        return {Real(0), counts};
    }
    const Real width = vmax / Real(buckets);
    for (Real x : v) {
        int k = int(x / width);
        if (k >= buckets) k = buckets - 1;
        ++counts[size_t(k)];
    }
    return {width, counts};
}

template <class Real>
int cmd_compare(const Options& o) {
    const auto cfg = load_config<Real>(o);
    if (cfg.engine != Engine::Both) throw ConfigError("compare requires engine = both");
    Prepared<Real> p;
    prepare(cfg, config_dir(o.config_path), p);
    if (const int rc = check_stability(p.sc, o.strict_stability); rc != kOk) return rc;
    std::cerr << "comparing engines on the GPU: " << p.mesh.num_nodes() << " nodes, " << p.mesh.num_elements() << " "
              << kind_name(p.mesh.kind) << " elements, dt=" << Real(p.sc.s.dt) << " s" << std::endl;
    const auto r_dj = execute(p, cfg, o.device, 0u);
    const auto r_tled = execute(p, cfg, o.device, DJG_FLAG_TLED);
    const Real field_rmse = rmse(r_dj.u, r_tled.u);
    const double ratio = r_dj.mean_step_seconds / std::max(r_tled.mean_step_seconds, 1e-300);
    std::string dj_field, tled_field;
    if (!cfg.field_path.empty()) {
        dj_field = with_suffix(cfg.field_path, "_djtled");
        tled_field = with_suffix(cfg.field_path, "_tled");
        write_field(dj_field, p.mesh, r_dj.u);
        write_field(tled_field, p.mesh, r_tled.u);
    }
    std::ostringstream rep;
    rep << std::setprecision(12);
    rep << "djtled compare report\n";
    rep << "nodes " << p.mesh.num_nodes() << "\n";
    rep << "elements " << p.mesh.num_elements() << "\n";
    rep << "dofs " << 3 * p.mesh.num_nodes() << "\n";
    rep << "steps " << r_dj.steps << "\n";
    rep << "dt " << Real(p.sc.s.dt) << "\n";
    rep << "precompute_s " << p.precompute_s << "\n";
    rep << "rmse " << field_rmse << "\n";
    rep << "wall_total_s_djtled " << r_dj.wall_seconds << "\n";
    rep << "wall_total_s_tled " << r_tled.wall_seconds << "\n";
    rep << "mean_step_us_djtled " << r_dj.mean_step_seconds * 1e6 << "\n";
    rep << "mean_step_us_tled " << r_tled.mean_step_seconds * 1e6 << "\n";
    rep << "ratio " << ratio << "\n";
    const auto [umin, umax] = std::minmax_element(r_tled.u.begin(), r_tled.u.end());
    if (*umax > *umin) {
        const auto [width, counts] = nre_histogram(r_dj.u, r_tled.u, 20);
        rep << "nre_histogram buckets " << counts.size() << " width " << width << "\n";
        for (size_t b = 0; b < counts.size(); ++b) rep << "nre_bucket " << b << " " << counts[b] << "\n";
    } else {
        rep << "nre_histogram undefined (uniform reference field)\n";
    }
    if (!dj_field.empty()) rep << "field_djtled " << dj_field << "\nfield_tled " << tled_field << "\n";
    emit_report(rep.str(), cfg.report_path);
    return kOk;
}

// run_bench / time_steps (bench.hpp:42-132): each engine on the bench box,
// zmin fixed along z, zmax ramped +1 % of the height over warmup + steps,
// alpha 10, dt 0.4 of the stability bound (the reference forms
// 0.4 * l_min / c; here 0.4 * (l_min / c) -- timing only); timed region =
// `steps` device steps after `warmup`, synchronised, wall clock.
template <class Real>
double time_engine(const Scenario& sc, int device, uint32_t flags, long warmup, long steps) {
    EngineHandle h;
    create_engine(sc, device, flags, h);
    djg_report rep{};
    if (warmup > 0 && djg_step(h.eng, warmup, &rep) != DJG_OK)
        throw SimFailure(kDivergence, "bench run failed");
    const auto t0 = std::chrono::steady_clock::now();
    if (djg_step(h.eng, steps, &rep) != DJG_OK) throw SimFailure(kDivergence, "bench run failed");
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / double(steps);
}

template <class Real>
int cmd_bench(const Options& o) {
    const auto cfg = load_config<Real>(o);
    BenchSpec<Real> b = cfg.bench;
    if (o.threads >= 1) b.threads = {o.threads};
    struct Row {
        long dofs;
        int kind, model;
        bool dj;
        int threads;
        double us, ratio;
    };
    std::vector<Row> rows;
    for (int div : b.divisions)
        for (int kind : b.kinds) {
            const double ex[3] = {double(b.extent), double(b.extent), double(b.extent)};
            const int32_t dv[3] = {div, div, div};
            const Mesh<Real> mesh = generate_box<Real>(ex, dv, kind);
            Real lo[3], hi[3];
            bounding_box(mesh, lo, hi);
            for (int model : b.models) {
                djg_scenario_spec s{};
                s.precision = int32_t(sizeof(Real));
                s.kind = kind;
                for (int i = 0; i < 3; ++i) {
                    s.divisions[i] = div;
                    s.extent[i] = double(b.extent);
                }
                djg_bench_material(model, &s.material);
                s.c_hg = 0.1;
                s.bc_mode = 1;
                s.fix_all_axes = 0;
                s.target = double((hi[2] - lo[2]) * Real(0.01));
                s.ramp_steps = b.warmup + b.steps;
                s.dt = 0.0;
                s.safety = 0.4;
                s.alpha_mode = 1;
                s.alpha = 10.0;
                s.policy = DJG_ABORT;
                for (int threads : b.threads) {
                    const int t = threads > 0 ? threads : hardware_threads();
                    std::cerr << "bench: div=" << div << " kind=" << kind_name(kind) << " material=" << model_name(model)
                              << " threads=" << t << "..." << std::endl;
                    Scenario sc;
                    build_scenario(s, t, sc);
                    const double us_dj = time_engine<Real>(sc, o.device, 0u, b.warmup, b.steps);
                    const double us_tled = time_engine<Real>(sc, o.device, DJG_FLAG_TLED, b.warmup, b.steps);
                    const double ratio = us_dj / us_tled;
                    rows.push_back({long(3 * mesh.num_nodes()), kind, model, true, t, us_dj, ratio});
                    rows.push_back({long(3 * mesh.num_nodes()), kind, model, false, t, us_tled, ratio});
                }
            }
        }
    std::ostringstream csv;
    csv << "dofs,kind,material,engine,threads,mean_step_us,ratio\n";
    csv << std::setprecision(6) << std::fixed;
    for (const auto& r : rows)
        csv << r.dofs << "," << kind_name(r.kind) << "," << model_name(r.model) << "," << (r.dj ? "djtled" : "tled")
            << "," << r.threads << "," << r.us << "," << r.ratio << "\n";
    std::ofstream out(b.csv_path);
    if (!out) throw ConfigError("cannot open CSV output '" + b.csv_path + "'");
    out << csv.str();
    std::cout << csv.str();
    long max_dofs = 0;
    for (const auto& r : rows) max_dofs = std::max(max_dofs, r.dofs);
    std::cerr << "achievable step rates at " << max_dofs << " DOFs:" << std::endl;
    for (const auto& r : rows)
        if (r.dofs == max_dofs && r.dj)
            std::cerr << "  " << kind_name(r.kind) << " " << model_name(r.model) << " threads=" << r.threads << ": "
                      << 1e6 / r.us << " steps/s" << std::endl;
    return kOk;
}

template <class Real>
int cmd_convert(const std::string& in_path, const std::string& out_path) {
    RunConfig<Real> cfg;
    cfg.mesh_file = in_path;
    const Mesh<Real> m = build_mesh(cfg, "");
    if (ends_with(out_path, ".djgmesh")) save_binary_mesh(m, out_path);
    else save_text_mesh(m, out_path);
    std::cerr << "wrote " << out_path << ": " << m.num_nodes() << " nodes, " << m.num_elements() << " "
              << kind_name(m.kind) << " elements" << std::endl;
    return kOk;
}

template <class F>
int guarded(const F& f) {
    try {
        return f();
    } catch (const ParseError& e) {
        std::cerr << "parse error: " << e.what() << std::endl;
        return kConfig;
    } catch (const ConfigError& e) {
        std::cerr << "config error: " << e.what() << std::endl;
        return kConfig;
    } catch (const MeshError& e) {
        std::cerr << "mesh error: " << e.what() << std::endl;
        return kConfig;
    } catch (const SimFailure& e) {
        std::cerr << "simulation error: " << e.what() << std::endl;
        return e.code;
    } catch (const CudaFailure& e) {
        std::cerr << "error: CUDA: " << e.what() << std::endl;
        return kInternal;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << std::endl;
        return kInternal;
    }
}

void usage() {
    std::cerr << "usage: djg run|compare|bench <config> [--precision single|double] [--threads N]\n"
                 "           [--on-inversion abort|report] [--strict-stability] [--device N]\n"
                 "       djg convert <in.mesh|in.djgmesh> <out.mesh|out.djgmesh> [--precision single|double]\n";
}

}  // namespace
}  // namespace djg::cli

int main(int argc, char** argv) {
    using namespace djg::cli;
    if (argc < 2) {
        usage();
        return kInternal;
    }
    const std::string cmd = argv[1];
    Options o;
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&](const char* name) -> std::string {
            if (i + 1 >= argc) {
                std::cerr << name << " needs a value" << std::endl;
                std::exit(kInternal);
            }
            return argv[++i];
        };
        if (a == "--precision") {
            o.precision = value("--precision");
            if (o.precision != "single" && o.precision != "double") {
                std::cerr << "--precision: single or double" << std::endl;
                return kInternal;
            }
        } else if (a == "--threads") {
            o.threads = std::atoi(value("--threads").c_str());
        } else if (a == "--on-inversion") {
            o.on_inversion = value("--on-inversion");
            if (o.on_inversion != "abort" && o.on_inversion != "report") {
                std::cerr << "--on-inversion: abort or report" << std::endl;
                return kInternal;
            }
        } else if (a == "--strict-stability") {
            o.strict_stability = true;
        } else if (a == "--device") {
            o.device = std::atoi(value("--device").c_str());
        } else if (a == "--engine") {
            if (value("--engine") != "gpu") {
                std::cerr << "--engine: this tool runs the gpu engine" << std::endl;
                return kInternal;
            }
        } else if (!a.empty() && a[0] == '-') {
            std::cerr << "unknown option " << a << std::endl;
            usage();
            return kInternal;
        } else {
            pos.push_back(a);
        }
    }
    const bool single = o.precision == "single";
    if (cmd == "convert") {
        if (pos.size() != 2) {
            usage();
            return kInternal;
        }
        return guarded([&] { return single ? cmd_convert<float>(pos[0], pos[1]) : cmd_convert<double>(pos[0], pos[1]); });
    }
    if (pos.size() != 1 || (cmd != "run" && cmd != "compare" && cmd != "bench")) {
        usage();
        return kInternal;
    }
    o.config_path = pos[0];
    if (cmd == "run") return guarded([&] { return single ? cmd_run<float>(o) : cmd_run<double>(o); });
    if (cmd == "compare") return guarded([&] { return single ? cmd_compare<float>(o) : cmd_compare<double>(o); });
    return guarded([&] { return single ? cmd_bench<float>(o) : cmd_bench<double>(o); });
}
