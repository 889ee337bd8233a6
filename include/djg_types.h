/*
 * djg_types.h — plain-C data types shared by the DJ-TLED B200 engine C-ABI
 * (djg.h), the host-side scenario builder (djg_host.h) and the CPU checkers
 * under oracle/.
 *
 * Every type here restates a reference type as a flat C struct so it can
 * cross an FFI boundary (ctypes / cgo / JNI) without C++ templates:
 *
 *   djg_material_params  <- djtled::Material<Real>           (material.hpp:140-230)
 *   djg_scenario_spec    <- mesh + BoundaryConditions + RunParams inputs of
 *                           cmd_run / bench::detail::time_steps
 *                           (mesh.hpp:41-71,208-264; solver.hpp:183-191;
 *                            config.hpp:31-42,484-502; bench.hpp:42-97)
 *   djg_report           <- StepOutcome / RunResult / SimulationError
 *                           (solver.hpp:89-94,193-200,229-239; core.hpp:44-57)
 *   djg_assemble_stats   <- AssembleStats (djtled_force.hpp:99-103)
 *
 * All floating-point inputs are passed as double and converted to the
 * engine's Real (float or double) exactly once, the way the reference
 * converts its config values (config.hpp parse_config -> Real).
 */
#ifndef DJG_TYPES_H
#define DJG_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ElementKind (element.hpp:9) */
enum djg_element_kind { DJG_T4 = 0, DJG_H8 = 1 };

/* MaterialModel (material.hpp:9), plus DJG_I57: the fifth/seventh-invariant
 * energy the reference drives its I5 / I7 force terms with
 * (test_forces.cpp:248-271; djtled_force.hpp:58-65, kinematics.hpp:89-101,
 * precompute.hpp:237-248):
 *   psi = mu/2 (Ib1 - 3) + eta5/2 (Ib5 - 1)^2 + eta7/2 (Ib7 - 1)^2 + kappa/2 (J - 1)^2,
 * eta5 / eta7 carried in eta_a / eta_b, fibre families a and b. No named
 * reference Material selects i5 / i7 (material.hpp:93-99), so this model has
 * no reference engine counterpart; its element terms are pinned against the
 * reference's element_force with these derivatives (oracle/ref_driver.cpp). */
enum djg_material_model { DJG_NH = 0, DJG_TI = 1, DJG_OT = 2, DJG_MR = 3, DJG_I57 = 4 };

/* InversionPolicy (djtled_force.hpp:97) */
enum djg_inversion_policy { DJG_ABORT = 0, DJG_SKIP_AND_REPORT = 1 };

/* DofConstraints kinds (solver.hpp:13) */
enum djg_dof_kind { DJG_FREE = 0, DJG_FIXED = 1, DJG_PRESCRIBED = 2 };

/* Return codes. 0 is success; the non-zero values mirror the CLI's exit
 * codes (djtled_main.cpp:13-20) so a caller can forward them unchanged. */
enum djg_status {
    DJG_OK = 0,
    DJG_E_INTERNAL = 1,   /* kInternal */
    DJG_E_CONFIG = 2,     /* kConfig: ConfigError / MeshError / bad descriptor */
    DJG_E_CUDA = 3,       /* CUDA runtime failure (no reference analogue) */
    DJG_E_INVERSION = 4,  /* kInversion: SimulationError::ElementInversion */
    DJG_E_DIVERGENCE = 5, /* kDivergence: SimulationError::Divergence */
    DJG_E_PEER = 6        /* peer-memory step: a part did not post its step within the
                             wait limit (DJG_PEER_TIMEOUT_MS, default 10000); no reference
                             analogue -- the engine halts instead of hanging the GPU */
};

/* Material<Real> (material.hpp:140-230). Only the fields of `model` are read. */
typedef struct djg_material_params {
    int32_t model;      /* djg_material_model */
    int32_t _pad;
    double mu;          /* NH/TI/OT shear modulus [Pa] */
    double kappa;       /* bulk modulus [Pa] */
    double rho;         /* density [kg/m^3] */
    double eta_a;       /* TI/OT fibre stiffness a [Pa] */
    double eta_b;       /* OT fibre stiffness b [Pa] */
    double c10, c01;    /* MR coefficients [Pa] */
    double fibre_a[3];  /* TI/OT fibre direction (normalised by the builder) */
    double fibre_b[3];  /* OT second fibre direction */
} djg_material_params;

/* One simulation problem. With nodes == NULL the mesh is the structured box
 * generate_box(extent, divisions, kind) (mesh.hpp:208-264); otherwise the
 * caller's mesh (validated like validate_mesh, mesh.hpp:75-92). */
typedef struct djg_scenario_spec {
    int32_t precision;     /* sizeof(Real): 4 or 8 */
    int32_t kind;          /* djg_element_kind */
    int32_t divisions[3];  /* box only */
    int32_t _pad0;
    double extent[3];      /* box only [m] */
    int64_t num_nodes;     /* explicit mesh only */
    int64_t num_elements;  /* explicit mesh only */
    const double* nodes;   /* 3*num_nodes, converted to Real */
    const int32_t* conn;   /* npe*num_elements */

    djg_material_params material;
    double c_hg;           /* hourglass coefficient (precompute.hpp:204, default 0.1) */

    /* Boundary conditions: 0 none; 1 box preset = zmin face fixed (all axes
     * when fix_all_axes, else z only), zmax face prescribed along z to
     * `target`, ramped over t_total = dt * Real(ramp_steps) (the bench and
     * SURVEY §8(d) loading, bench.hpp:52-72); 2 explicit lists below. */
    int32_t bc_mode;
    int32_t fix_all_axes;
    double target;
    int64_t ramp_steps;
    int64_t n_fixed;
    const int32_t* fixed_node;
    const int32_t* fixed_axis;
    int64_t n_prescribed;
    const int32_t* presc_node;
    const int32_t* presc_axis;
    const double* presc_target;
    const double* presc_t_total;

    /* Time step: dt = Real(dt) when dt > 0, else Real(safety) * critical_dt
     * (precompute.hpp:323-331, material.hpp:117-120). */
    double dt;
    double safety;
    /* Damping: alpha_mode 0 -> relaxation_alpha (solver.hpp:330-339),
     * 1 -> Real(alpha). */
    int32_t alpha_mode;
    int32_t policy;        /* djg_inversion_policy */
    double alpha;
} djg_scenario_spec;

/* Caller-owned output arrays for a fully built scenario ("image"). Any
 * pointer may be NULL. Real arrays use the scenario's precision. */
typedef struct djg_image_ptrs {
    void* nodes;            /* 3N Real, reference coordinates */
    int32_t* conn;          /* npe*E */
    int64_t* csr_offsets;   /* N+1   NodeElementAdjacency::offsets (mesh.hpp:300) */
    int64_t* csr_elem;      /* npe*E NodeElementAdjacency::pairs.first  */
    int32_t* csr_local;     /* npe*E NodeElementAdjacency::pairs.second */
    void* consts;           /* E*nconst Real, canonical hot-field record (djg.h) */
    void* mass;             /* N Real  lump_mass (precompute.hpp:275-287) */
    void* c1;               /* N Real  UpdateCoeffs::c1 (solver.hpp:66) */
    uint8_t* massless;      /* N       UpdateCoeffs::massless */
    uint8_t* dof_kind;      /* 3N      DofConstraints::kind (solver.hpp:14) */
    void* dof_target;       /* 3N Real */
    void* dof_t_total;      /* 3N Real */
} djg_image_ptrs;

/* Scalars of a built scenario, each a Real value widened to double. */
typedef struct djg_image_scalars {
    int64_t num_nodes;
    int64_t num_elements;
    int32_t npe;
    int32_t nconst;
    double dt;
    double critical_dt;
    double alpha;
    double c2, c3;
    double ramp_t_total;   /* box preset ramp duration */
    double wave_speed;
} djg_image_scalars;

/* Outcome of a multi-step call: StepOutcome + RunResult + the
 * SimulationError payload (solver.hpp:89-94,193-200,229-239). */
typedef struct djg_report {
    int64_t steps_done;       /* steps completed by this call */
    int64_t step;             /* state.step after the call */
    int64_t first_inverted;   /* min inverted element of the failing step (Abort), -1 */
    int64_t inverted_count;   /* inverted elements summed over the call's steps */
    int64_t inverted_steps;   /* steps that saw >= 1 inverted element (RunResult::inverted_steps) */
    int64_t fail_step;        /* state.step + 1 of the failing step, -1 */
    int32_t diverged;         /* 1 if the divergence detector fired */
    int32_t status;           /* djg_status */
} djg_report;

/* AssembleStats (djtled_force.hpp:99-103) */
typedef struct djg_assemble_stats {
    int64_t first_inverted;   /* -1 unless an inversion occurred under Abort */
    int64_t inverted_count;
} djg_assemble_stats;

#ifdef __cplusplus
}
#endif

#endif /* DJG_TYPES_H */
