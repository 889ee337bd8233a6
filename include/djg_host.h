/*
 * djg_host.h — C-ABI of the host-side problem builder (also in libdjg.so).
 *
 * It runs the reference's host pipeline ahead of the step loop, in native
 * C++, so a caller without the reference can produce an engine descriptor:
 *
 *   generate_box / caller mesh + validate_mesh   mesh.hpp:75-92, 208-264
 *   NodeElementAdjacency::build                  mesh.hpp:299-320 (bit-exact)
 *   DjModel::build -> build_element_constants    djtled_force.hpp:145-157,
 *                                                precompute.hpp:206-255
 *   lump_mass, critical_dt                       precompute.hpp:275-331
 *   select_plane_nodes + BoundaryConditions      config.hpp:31-42, 484-502
 *   DofConstraints::build, UpdateCoeffs::build   solver.hpp:18-33, 70-86
 *   relaxation_alpha                             solver.hpp:330-339
 *
 * The arithmetic follows the reference operation by operation, so every
 * Real it produces is bit-identical to the reference's (checked by
 * tests/test_host_parity.py against oracle/_ref and the golden fixtures).
 */
#ifndef DJG_HOST_H
#define DJG_HOST_H

#include "djg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct djg_scenario djg_scenario;

/* Fills `spec` with the SURVEY §8(d) defaults for a box: extent 1 m,
 * bench_material(model) parameters (bench.hpp:12-25), c_hg 0.1, zmin fixed
 * in all axes, zmax prescribed to -0.2 m, dt = 0.5 critical_dt,
 * alpha = relaxation_alpha, Abort policy. */
void djg_spec_default_box(djg_scenario_spec* spec, int32_t precision, int32_t kind,
                          int32_t model, int32_t divisions, int64_t ramp_steps);

/* bench_material (bench.hpp:12-25) parameters for `model`. */
void djg_bench_material(int32_t model, djg_material_params* out);

/* Builds the whole problem. Returns DJG_E_CONFIG (message in
 * djg_scenario_error()) on a ConfigError / MeshError condition. */
int djg_scenario_build(const djg_scenario_spec* spec, int32_t threads, djg_scenario** out);
void djg_scenario_free(djg_scenario* sc);
const char* djg_scenario_error(void);

int djg_scenario_scalars(const djg_scenario* sc, djg_image_scalars* out);
/* Copies the built arrays into caller buffers (NULL pointers skipped). */
int djg_scenario_image(const djg_scenario* sc, const djg_image_ptrs* out);
/* Engine descriptor whose pointers alias the scenario's arrays (valid while
 * the scenario lives). */
int djg_scenario_desc(const djg_scenario* sc, int32_t device, djg_desc* out);

#ifdef __cplusplus
}
#endif

#endif /* DJG_HOST_H */
