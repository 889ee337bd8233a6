// C-ABI over the host problem builder (include/djg_host.h).
#include <cstring>
#include <memory>
#include <string>
#include <variant>

#include "djg_host.h"
#include "problem.hpp"

namespace {

thread_local std::string g_error;

template <class Real>
void copy_out(const djg::Problem<Real>& P, const djg_image_ptrs& o) {
    auto put = [](void* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    put(o.nodes, P.mesh.nodes);
    put(o.conn, P.mesh.conn);
    put(o.csr_offsets, P.adj.offsets);
    put(o.csr_elem, P.adj.elem);
    put(o.csr_local, P.adj.local);
    put(o.consts, P.consts);
    put(o.mass, P.mass);
    put(o.c1, P.c1);
    put(o.massless, P.massless);
    put(o.dof_kind, P.dof_kind);
    put(o.dof_target, P.dof_target);
    put(o.dof_t_total, P.dof_t_total);
}

template <class Real>
void scalars_of(const djg::Problem<Real>& P, djg_image_scalars& s) {
    s.num_nodes = P.mesh.num_nodes();
    s.num_elements = P.mesh.num_elements();
    s.npe = P.mesh.npe();
    s.nconst = P.nconst;
    s.dt = double(P.dt);
    s.critical_dt = double(P.crit_dt);
    s.alpha = double(P.alpha);
    s.c2 = double(P.c2);
    s.c3 = double(P.c3);
    s.ramp_t_total = double(P.ramp_t_total);
    s.wave_speed = double(P.c_wave);
}

template <class Real>
void desc_of(const djg::Problem<Real>& P, int32_t device, djg_desc& d) {
    std::memset(&d, 0, sizeof(d));
    d.precision = int32_t(sizeof(Real));
    d.kind = P.mesh.kind;
    d.num_nodes = P.mesh.num_nodes();
    d.num_elements = P.mesh.num_elements();
    d.conn = P.mesh.conn.data();
    d.consts = P.consts.data();
    d.nconst = P.nconst;
    d.inversion_policy = P.policy;
    d.csr_offsets = P.adj.offsets.data();
    d.csr_elem = P.adj.elem.data();
    d.csr_local = P.adj.local.data();
    d.dof_kind = P.dof_kind.data();
    d.dof_target = P.dof_target.data();
    d.dof_t_total = P.dof_t_total.data();
    d.c1 = P.c1.data();
    d.massless = P.massless.data();
    d.c2 = double(P.c2);
    d.c3 = double(P.c3);
    d.dt = double(P.dt);
    d.material.model = P.mat.model;
    d.material.mu = double(P.mat.mu);
    d.material.kappa = double(P.mat.kappa);
    d.material.rho = double(P.mat.rho);
    d.material.eta_a = double(P.mat.eta_a);
    d.material.eta_b = double(P.mat.eta_b);
    d.material.c10 = double(P.mat.c10);
    d.material.c01 = double(P.mat.c01);
    for (int i = 0; i < 3; ++i) {
        d.material.fibre_a[i] = double(i == 0 ? P.mat.fa.x : (i == 1 ? P.mat.fa.y : P.mat.fa.z));
        d.material.fibre_b[i] = double(i == 0 ? P.mat.fb.x : (i == 1 ? P.mat.fb.y : P.mat.fb.z));
    }
    d.device = device;
    d.nodes = P.mesh.nodes.data();
    d.c_hg = double(P.c_hg);
}

// DjEngine(mesh, material, c_hg) precompute (djtled_force.hpp:145-157) for
// djg_create_from_mesh: hot-constant records + adjacency, then djg_create.
template <class Real>
int create_from_mesh(const djg_mesh_desc& m, djg_engine** out) {
    djg::Mesh<Real> mesh;
    mesh.kind = m.kind;
    const Real* xn = static_cast<const Real*>(m.nodes);
    if (!xn || !m.conn || m.num_nodes < 1 || m.num_elements < 1) throw djg::ConfigError("mesh needs nodes and elements");
    mesh.nodes.assign(xn, xn + 3 * m.num_nodes);
    mesh.conn.assign(m.conn, m.conn + m.num_elements * djg::npe_of(m.kind));
#ifdef _OPENMP
    if (m.threads > 0) omp_set_num_threads(m.threads);
#endif
    const int npe = mesh.npe();
    const int64_t E = mesh.num_elements();
    const bool on_device = (m.flags & DJG_FLAG_DEVICE_PRECOMPUTE) != 0;
    const auto mat = djg::Material<Real>::from(m.material);
    const djg::ConstLayout L(m.kind, mat.model);
    std::vector<Real> consts;
    if (on_device) {
        // the engine checks the connectivity, builds the records and rejects
        // inverted elements on the GPU
    } else {
        djg::validate_mesh(mesh);
        const djg::Shape<Real> D(m.kind);
        djg::V3<Real> fa{0, 0, 0}, fb{0, 0, 0};
        if (mat.needs_fibre_a()) fa = djg::Material<Real>::unit(mat.fa);
        if (mat.needs_fibre_b()) fb = djg::Material<Real>::unit(mat.fb);
        consts.assign(size_t(E) * size_t(L.count), Real(0));
        const Real c_hg = Real(m.c_hg);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < E; ++e) {
            djg::V3<Real> x[8];
            for (int a = 0; a < npe; ++a) x[a] = mesh.node(mesh.conn[size_t(e * npe + a)]);
            djg::element_record(x, D, mat, fa, fb, c_hg, L, consts.data() + size_t(e) * L.count);
        }
    }
    // With device precompute (and no slabs) the engine builds the adjacency
    // on the GPU as well.
    const bool device_csr = on_device && !(m.flags & DJG_FLAG_SLABS);
    djg::Adjacency adj;
    if (!device_csr) adj = djg::build_adjacency(mesh.conn, mesh.num_nodes(), npe);
    djg_desc d;
    std::memset(&d, 0, sizeof(d));
    d.precision = int32_t(sizeof(Real));
    d.kind = m.kind;
    d.num_nodes = mesh.num_nodes();
    d.num_elements = E;
    d.conn = mesh.conn.data();
    d.consts = on_device ? nullptr : consts.data();
    d.nconst = L.count;
    d.inversion_policy = m.inversion_policy;
    d.csr_offsets = device_csr ? nullptr : adj.offsets.data();
    d.csr_elem = device_csr ? nullptr : adj.elem.data();
    d.csr_local = device_csr ? nullptr : adj.local.data();
    d.material = m.material;
    d.device = m.device;
    d.flags = m.flags;
    d.nodes = mesh.nodes.data();
    d.c_hg = m.c_hg;
    return djg_create(&d, out);
}

}  // namespace

extern "C" void djg_internal_set_create_error(const char* msg);

struct djg_scenario {
    std::variant<djg::Problem<float>, djg::Problem<double>> p;
};

struct djg_partition {
    std::variant<djg::PartProblem<float>, djg::PartProblem<double>> p;
    djg_scenario_spec spec{};  // part-local build: the box spec (its pointers are not kept)
};

extern "C" {

void djg_bench_material(int32_t model, djg_material_params* m) {
    // bench_material (bench.hpp:12-25): mu 6567, kappa 326210, rho 1060,
    // fibres along x (and y), eta = 2 mu, MR c10 = mu/2, c01 = 3000.
    std::memset(m, 0, sizeof(*m));
    m->model = model;
    m->mu = 6567.0;
    m->kappa = 326210.0;
    m->rho = 1060.0;
    m->fibre_a[0] = 1.0;
    m->fibre_b[1] = 1.0;
    if (model == DJG_TI || model == DJG_OT) m->eta_a = 2 * 6567.0;
    if (model == DJG_OT) m->eta_b = 2 * 6567.0;
    if (model == DJG_MR) {
        m->mu = 0.0;
        m->c10 = 6567.0 / 2;
        m->c01 = 3000.0;
    }
    if (model == DJG_I57) {  // test_forces.cpp:251 ratios (eta5 800, eta7 650 over mu 500)
        m->eta_a = 1.6 * 6567.0;
        m->eta_b = 1.3 * 6567.0;
        m->fibre_a[1] = 1.0;
        m->fibre_b[2] = 1.0;
    }
}

void djg_spec_default_box(djg_scenario_spec* s, int32_t precision, int32_t kind, int32_t model,
                          int32_t divisions, int64_t ramp_steps) {
    std::memset(s, 0, sizeof(*s));
    s->precision = precision;
    s->kind = kind;
    for (int i = 0; i < 3; ++i) {
        s->divisions[i] = divisions;
        s->extent[i] = 1.0;
    }
    djg_bench_material(model, &s->material);
    s->c_hg = 0.1;
    s->bc_mode = 1;
    s->fix_all_axes = 1;
    s->target = -0.2;
    s->ramp_steps = ramp_steps;
    s->safety = 0.5;
    s->alpha_mode = 0;
    s->policy = DJG_ABORT;
}

const char* djg_scenario_error(void) { return g_error.c_str(); }

int djg_scenario_build(const djg_scenario_spec* spec, int32_t threads, djg_scenario** out) {
    if (!spec || !out) {
        g_error = "null argument";
        return DJG_E_CONFIG;
    }
    *out = nullptr;
    try {
        auto sc = std::make_unique<djg_scenario>();
        if (spec->precision == 4)
            sc->p = djg::build_problem<float>(*spec, threads);
        else if (spec->precision == 8)
            sc->p = djg::build_problem<double>(*spec, threads);
        else
            throw djg::ConfigError("precision must be 4 or 8");
        *out = sc.release();
        return DJG_OK;
    } catch (const djg::ConfigError& e) {
        g_error = e.what();
    } catch (const djg::MeshError& e) {
        g_error = e.what();
    } catch (const std::exception& e) {
        g_error = e.what();
        return DJG_E_INTERNAL;
    }
    return DJG_E_CONFIG;
}

void djg_scenario_free(djg_scenario* sc) { delete sc; }

int djg_create_from_mesh(const djg_mesh_desc* m, djg_engine** out) {
    if (!m || !out) return DJG_E_CONFIG;
    *out = nullptr;
    try {
        if (m->precision == 4) return create_from_mesh<float>(*m, out);
        if (m->precision == 8) return create_from_mesh<double>(*m, out);
        throw djg::ConfigError("precision must be 4 or 8");
    } catch (const djg::ConfigError& e) {
        djg_internal_set_create_error(e.what());
    } catch (const djg::MeshError& e) {
        djg_internal_set_create_error(e.what());
    } catch (const std::exception& e) {
        djg_internal_set_create_error(e.what());
        return DJG_E_INTERNAL;
    }
    return DJG_E_CONFIG;
}

int djg_scenario_scalars(const djg_scenario* sc, djg_image_scalars* out) {
    if (!sc || !out) return DJG_E_CONFIG;
    std::visit([&](const auto& P) { scalars_of(P, *out); }, sc->p);
    return DJG_OK;
}

int djg_scenario_image(const djg_scenario* sc, const djg_image_ptrs* out) {
    if (!sc || !out) return DJG_E_CONFIG;
    std::visit([&](const auto& P) { copy_out(P, *out); }, sc->p);
    return DJG_OK;
}

int djg_scenario_desc(const djg_scenario* sc, int32_t device, djg_desc* out) {
    if (!sc || !out) return DJG_E_CONFIG;
    std::visit([&](const auto& P) { desc_of(P, device, *out); }, sc->p);
    return DJG_OK;
}

int djg_partition_build(const djg_scenario* sc, int32_t nparts, int32_t part, djg_partition** out) {
    return djg_partition_build_method(sc, nparts, part, DJG_PART_RCB, out);
}

int djg_partition_build_method(const djg_scenario* sc, int32_t nparts, int32_t part, int32_t method,
                               djg_partition** out) {
    if (!sc || !out) return DJG_E_CONFIG;
    *out = nullptr;
    try {
        auto pp = std::make_unique<djg_partition>();
        std::visit(
            [&](const auto& P) {
                using R = typename std::decay_t<decltype(P.consts)>::value_type;
                pp->p = djg::build_part<R>(P, nparts, part, method);
            },
            sc->p);
        *out = pp.release();
        return DJG_OK;
    } catch (const std::exception& e) {
        g_error = e.what();
        return DJG_E_CONFIG;
    }
}

int djg_partition_build_box(const djg_scenario_spec* spec, int32_t nparts, int32_t part, djg_partition** out,
                            double* local_min_length) {
    if (!spec || !out) return DJG_E_CONFIG;
    *out = nullptr;
    try {
        auto pp = std::make_unique<djg_partition>();
        double lmin = 0;
        if (spec->precision == 4) {
            float l = 0;
            pp->p = djg::build_box_part<float>(*spec, nparts, part, l);
            lmin = l;
        } else if (spec->precision == 8) {
            double l = 0;
            pp->p = djg::build_box_part<double>(*spec, nparts, part, l);
            lmin = l;
        } else {
            throw djg::ConfigError("precision must be 4 or 8");
        }
        pp->spec = *spec;
        if (local_min_length) *local_min_length = lmin;
        *out = pp.release();
        return DJG_OK;
    } catch (const std::exception& e) {
        g_error = e.what();
        return DJG_E_CONFIG;
    }
}

int djg_partition_finish(djg_partition* p, double global_min_length) {
    if (!p) return DJG_E_CONFIG;
    try {
        std::visit(
            [&](auto& R) {
                using Real = typename std::decay_t<decltype(R.local.consts)>::value_type;
                djg::finish_box_part<Real>(R, p->spec, Real(global_min_length));
            },
            p->p);
        return DJG_OK;
    } catch (const std::exception& e) {
        g_error = e.what();
        return DJG_E_CONFIG;
    }
}

void djg_partition_free(djg_partition* p) { delete p; }

int djg_partition_get_info(const djg_partition* p, djg_partition_info* o) {
    if (!p || !o) return DJG_E_CONFIG;
    std::visit(
        [&](const auto& R) {
            std::memset(o, 0, sizeof(*o));
            o->nparts = R.nparts;
            o->part = R.part;
            o->num_neighbors = int32_t(R.halo.neighbors.size());
            o->num_nodes = int64_t(R.node_l2g.size());
            o->num_owned = R.num_owned;
            o->num_elements = int64_t(R.elem_l2g.size());
            o->owned_elements = R.owned_elements;
            o->interior_elements = R.interior_elements;
            o->send_total = int64_t(R.halo.send_nodes.size());
            o->recv_total = int64_t(R.halo.recv_nodes.size());
            o->global_nodes = R.global_nodes;
            o->global_elements = R.global_elements;
        },
        p->p);
    return DJG_OK;
}

int djg_partition_image(const djg_partition* p, const djg_image_ptrs* out) {
    if (!p || !out) return DJG_E_CONFIG;
    std::visit([&](const auto& R) { copy_out(R.local, *out); }, p->p);
    return DJG_OK;
}

int djg_partition_desc(const djg_partition* p, int32_t device, djg_desc* out) {
    if (!p || !out) return DJG_E_CONFIG;
    std::visit([&](const auto& R) { desc_of(R.local, device, *out); }, p->p);
    return DJG_OK;
}

int djg_partition_halo(const djg_partition* p, int32_t* nb, int64_t* so, int64_t* ro, int32_t* sn, int32_t* rn) {
    if (!p) return DJG_E_CONFIG;
    std::visit(
        [&](const auto& R) {
            auto put = [](auto* dst, const auto& v) {
                if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
            };
            put(nb, R.halo.neighbors);
            put(so, R.halo.send_off);
            put(ro, R.halo.recv_off);
            put(sn, R.halo.send_nodes);
            put(rn, R.halo.recv_nodes);
        },
        p->p);
    return DJG_OK;
}

int djg_partition_maps(const djg_partition* p, int64_t* node_l2g, int64_t* elem_l2g) {
    if (!p) return DJG_E_CONFIG;
    std::visit(
        [&](const auto& R) {
            if (node_l2g) std::memcpy(node_l2g, R.node_l2g.data(), R.node_l2g.size() * sizeof(int64_t));
            if (elem_l2g) std::memcpy(elem_l2g, R.elem_l2g.data(), R.elem_l2g.size() * sizeof(int64_t));
        },
        p->p);
    return DJG_OK;
}

int djg_partition_owned_elements(const djg_partition* p, uint8_t* owned) {
    if (!p || !owned) return DJG_E_CONFIG;
    std::visit([&](const auto& R) { std::memcpy(owned, R.elem_owned.data(), R.elem_owned.size()); }, p->p);
    return DJG_OK;
}

int djg_element_parts(const djg_scenario* sc, int32_t nparts, int32_t* part) {
    return djg_element_parts_method(sc, nparts, DJG_PART_RCB, part);
}

int djg_element_parts_method(const djg_scenario* sc, int32_t nparts, int32_t method, int32_t* part) {
    if (!sc || !part || nparts < 1) return DJG_E_CONFIG;
    try {
        std::visit(
            [&](const auto& P) {
                const auto v = djg::element_parts(P.mesh, nparts, method);
                std::memcpy(part, v.data(), v.size() * sizeof(int32_t));
            },
            sc->p);
    } catch (const std::exception& e) {
        g_error = e.what();
        return DJG_E_CONFIG;
    }
    return DJG_OK;
}

}  // extern "C"
