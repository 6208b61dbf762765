/* CPU oracle API for the GMCP contact hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Two libraries export exactly these symbols and are loaded side by side by
 * the tests (ctypes, RTLD_LOCAL):
 *   oracle/libgmcp_oracle.so   -- oracle/gmcp_oracle.c, a plain-C restatement
 *                                 of the reference algorithm (cites file:line);
 *   oracle/_ref/libgmcp_ref.so -- oracle/ref_capi.cpp, the UNMODIFIED reference
 *                                 headers (/root/reference/proj/include) built
 *                                 against oracle/eigen_shim; used to pin the
 *                                 restatement and to generate tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * either of them; the product library never links them.
 *
 * Conventions: positions/gradients are flat 3N arrays (xyz per vertex) like the
 * reference's VecX; every function returns a GMCP_* status and fills out-params;
 * orc_last_error() returns the thread-local message of the last failure.
 */
#ifndef GMCP_ORACLE_API_H
#define GMCP_ORACLE_API_H

#include "../include/gmcp_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_pairs orc_pairs;
typedef struct orc_state orc_state;

const char* orc_last_error(void);
int orc_is_reference(void); /* 1 for the compiled reference, 0 for the restatement */

/* barrier.hpp:25-46 */
int orc_resolve_barrier_params(gmcp_barrier_params* p, double mean_slave_edge);
/* contact_sampling.hpp:257-263 */
int orc_mean_edge_length(const gmcp_surface* s, const double* x, double* out);
/* barrier.hpp:55-66 -> out = {B, B', B''} */
int orc_barrier(double g, double eps, double* out);

/* contact_sampling.hpp:281-340. which: 0 tris, 1 edges, 2 verts (feature ids) */
int orc_build_candidate_pairs(const gmcp_surface* slave, const gmcp_surface* master,
                              const double* x, double r, int use_tree, orc_pairs** out);
int orc_pairs_from_csr(int32_t n_slave_tris, const int64_t* tri_off, const int32_t* tri_ids,
                       const int64_t* edge_off, const int32_t* edge_ids, const int64_t* vert_off,
                       const int32_t* vert_ids, orc_pairs** out);
int64_t orc_pairs_size(const orc_pairs* p, int which);
int32_t orc_pairs_slave_tris(const orc_pairs* p);
void orc_pairs_copy(const orc_pairs* p, int which, int64_t* offsets, int32_t* ids);
void orc_pairs_free(orc_pairs* p);

/* contact_sampling.hpp:382-487 */
int orc_build_contact_state(const gmcp_surface* slave, const gmcp_surface* master,
                            const orc_pairs* pairs, const double* x, int64_t n_dof,
                            const gmcp_barrier_params* params, const double* eps_reference,
                            orc_state** out);
/* hand-built states (test_contact.cpp:69-83) */
int orc_state_from_samples(const gmcp_samples* s, const double* ref_x, int64_t n_dof,
                           orc_state** out);
int64_t orc_state_size(const orc_state* st);
void orc_state_copy(const orc_state* st, gmcp_samples* out);
void orc_state_free(orc_state* st);

/* contact_sampling.hpp:350-372 */
int orc_sample_gap(const orc_state* st, int64_t i, const double* x, double* g);
/* contact_energy.hpp:26-73: per sample g, nv, ids[6], dg[6][3] (unused slots 0) */
int orc_kinematics(const orc_state* st, const double* x, double* g, int32_t* nv, int32_t* ids,
                   double* dg);
/* contact_energy.hpp:95-108 */
int orc_try_contact_energy(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                           double* energy, double* min_gap, int32_t* feasible);
/* contact_energy.hpp:110-123; bad = first offending sample on GMCP_ERR_INFEASIBLE */
int orc_contact_energy(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                       double* energy, int64_t* bad);
/* contact_energy.hpp:126-142 (grad is accumulated into, never cleared) */
int orc_add_contact_gradient(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                             double* grad, double* energy, int64_t* bad);
/* contact_energy.hpp:146-179. The Gauss-Newton triplets are summed per 3x3
 * block (setFromTriplets semantics) and returned sorted by (row, col). Call
 * with null block arrays first to learn n_blocks. n_triplets = scalar
 * triplets the reference emits. */
int orc_add_contact_gradient_hessian(const orc_state* st, const gmcp_barrier_params* p,
                                     const double* x, double* grad, double* energy,
                                     int64_t* bad, int64_t* n_blocks, int32_t* brow,
                                     int32_t* bcol, double* bval, int64_t* n_triplets);
/* contact_energy.hpp:184-193 */
int orc_step_filter(const orc_state* st, const double* x, const double* dx, double* alpha);
/* contact_energy.hpp:198-213; n_dof = length of dx */
int orc_displacement_cap(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                         const double* dx, int64_t n_dof, double* alpha);
/* contact_energy.hpp:225-242; out may be null to count */
int orc_pressure_field(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                       int64_t* n, gmcp_pressure_record* out);
/* contact_energy.hpp:253-276 -> out[12] = face, edge, point, total */
int orc_force_summary(const orc_state* st, const gmcp_barrier_params* p, const double* x,
                      double* out);

/* CPU baseline timing: best-of-reps seconds of one assembly call
 * (add_contact_gradient_hessian) over the state, excluding marshalling. */
int orc_time_assembly(const orc_state* st, const gmcp_barrier_params* p, const double* x, int32_t reps,
                      double* best_seconds, int64_t* n_triplets);

/* ---- dual-mesh embedding (embedding.hpp) -------------------------------- */
/* embedding.hpp:26-84: nearest host triangle per point (lowest index on ties),
 * plane barycentrics and signed normal offset. host: n_hv vertices (3 doubles
 * each), n_ht triangles (local ids). use_tree selects the reference's AABB
 * tree (reference library only; the restatement always scans). On a
 * degenerate host triangle returns GMCP_ERR_DEGENERATE with *bad = index. */
int orc_embed_in_surface(const double* points, int64_t n_points, const double* host_v, int64_t n_hv,
                         const int32_t* host_t, int64_t n_ht, int32_t use_tree, int32_t* tri, double* bary,
                         double* offset, int64_t* bad);
/* embedding.hpp:87-106: reconstruct; GMCP_ERR_DEGENERATE with *bad = host
 * triangle of the first embedded vertex whose triangle degenerated. */
int orc_apply_embedding(const int32_t* tri, const double* bary, const double* offset, int64_t n,
                        const int32_t* host_t, int64_t n_ht, const double* host_x, int64_t n_hv, double* out,
                        int64_t* bad);

#ifdef __cplusplus
}
#endif

#endif
