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

/*
 * Multi-GPU decomposition; no reference analogue (the
 * reference is single-process). Part `part` of `nparts` of a built scenario:
 * recursive coordinate bisection of element centroids; a node belongs to the
 * part of its lowest-id element; a part computes every element touching its
 * nodes (ghost elements included) in ascending global element id, so owned
 * nodes are bit-identical to the single-GPU step. Local node numbering: owned
 * nodes first, then ghost nodes, each ascending in global id.
 */
typedef struct djg_partition djg_partition;

typedef struct djg_partition_info {
    int32_t nparts, part;
    int32_t num_neighbors, _pad;
    int64_t num_nodes;        /* local nodes (owned + ghost) */
    int64_t num_owned;        /* owned nodes: local ids [0, num_owned) */
    int64_t num_elements;     /* local elements (owned + ghost) */
    int64_t owned_elements;   /* elements assigned to this part */
    int64_t send_total, recv_total;
    int64_t global_nodes, global_elements;
    int64_t interior_elements;  /* local elements [0, interior) reference no ghost node */
} djg_partition_info;

/* Partition methods: recursive coordinate bisection of element centroids
 * (default; fast, reproducible), METIS k-way on the element dual graph
 * (faces shared; METIS_PartMeshDual, fixed seed: reproducible), or -- for
 * generated boxes -- recursive bisection of the cell grid (every part a
 * block of cells; the partition the part-local build uses). */
enum djg_partition_method { DJG_PART_RCB = 0, DJG_PART_METIS = 1, DJG_PART_BOX = 2 };
int djg_partition_build(const djg_scenario* sc, int32_t nparts, int32_t part, djg_partition** out);
int djg_partition_build_method(const djg_scenario* sc, int32_t nparts, int32_t part, int32_t method,
                               djg_partition** out);
/* Part-local build of a generated box (spec->nodes == NULL, plane BCs):
 * part `part` of the DJG_PART_BOX partition built without the global mesh or
 * problem -- the same local problem djg_partition_build_method(...,
 * DJG_PART_BOX) extracts from the global one, for every owned node and local
 * element. Two steps, because dt needs the global minimum characteristic
 * length: build returns this part's minimum in *local_min_length; the caller
 * reduces it over the parts (MIN) and passes it to djg_partition_finish,
 * which completes dt, alpha, the BCs and the update coefficients. */
int djg_partition_build_box(const djg_scenario_spec* spec, int32_t nparts, int32_t part, djg_partition** out,
                            double* local_min_length);
int djg_partition_finish(djg_partition* p, double global_min_length);
void djg_partition_free(djg_partition* p);
int djg_partition_get_info(const djg_partition* p, djg_partition_info* out);
/* Local problem arrays (same layout as djg_scenario_image, local ids). */
int djg_partition_image(const djg_partition* p, const djg_image_ptrs* out);
/* Engine descriptor of the local problem (pointers alias the partition). */
int djg_partition_desc(const djg_partition* p, int32_t device, djg_desc* out);
/* Halo lists: neighbors[num_neighbors]; send_off/recv_off[num_neighbors+1];
 * send_nodes[send_total] (owned local ids), recv_nodes[recv_total] (ghost
 * local ids), each neighbor's block ascending in global node id. */
int djg_partition_halo(const djg_partition* p, int32_t* neighbors, int64_t* send_off, int64_t* recv_off,
                       int32_t* send_nodes, int32_t* recv_nodes);
/* Local -> global ids: node_l2g[num_nodes], elem_l2g[num_elements]. */
int djg_partition_maps(const djg_partition* p, int64_t* node_l2g, int64_t* elem_l2g);
/* Per local element: 1 if the partitioner assigned it to this part (it
 * reports that element's inversions, djg_set_counted_elements), 0 for the
 * ghost copies of other parts' elements. */
int djg_partition_owned_elements(const djg_partition* p, uint8_t* owned);
/* Element -> part assignment of the whole scenario (E entries). */
int djg_element_parts(const djg_scenario* sc, int32_t nparts, int32_t* part);
int djg_element_parts_method(const djg_scenario* sc, int32_t nparts, int32_t method, int32_t* part);

#ifdef __cplusplus
}
#endif

#endif /* DJG_HOST_H */
