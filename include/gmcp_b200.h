/* GMCP B200 C-ABI: the drop-in boundary for the reference's per-Newton-
 * iteration contact pipeline (proj/include/gmcp/, a header-only C++ library
 * with no FFI of its own). Every entry point is extern "C" with
 * plain pointers and sizes. The C++ drop-in layer include/gmcp/b200.hpp keeps
 * the reference signatures on top of it and rethrows the reference exceptions.
 *
 * Model: one gmcp_ctx per GPU, bound to one CUDA stream. The context holds
 * device copies of the contact surfaces, positions x, step dx, the frozen
 * sample set and the assembled contact Hessian. Calls are synchronous (they
 * return after the stream work finished) unless noted; a context is not
 * thread-safe; independent contexts may be driven from different threads.
 * There is no CPU fallback: without a CUDA device every call returns
 * GMCP_ERR_CUDA.
 *
 * Reference interface each entry point replaces (file:line under
 * /root/reference/proj/include/gmcp/):
 *   gmcp_broadphase            build_candidate_pairs      contact_sampling.hpp:281-340
 *   gmcp_build_samples         build_contact_state        contact_sampling.hpp:382-487
 *   gmcp_try_energy            try_contact_energy         contact_energy.hpp:95-108
 *   gmcp_energy                contact_energy             contact_energy.hpp:110-123
 *   gmcp_gradient              add_contact_gradient       contact_energy.hpp:126-142
 *   gmcp_gradient_hessian      add_contact_gradient_hessian contact_energy.hpp:146-179
 *   gmcp_add_gradient          add_contact_gradient (x, grad in one call)  :126-142
 *   gmcp_add_gradient_hessian  add_contact_gradient_hessian (one call)     :146-179
 *   gmcp_step_filter           step_filter                contact_energy.hpp:184-193
 *   gmcp_displacement_cap      displacement_cap           contact_energy.hpp:198-213
 *   gmcp_pressure_field        contact_pressure_field     contact_energy.hpp:225-242
 *   gmcp_force_summary         contact_force_summary      contact_energy.hpp:253-276
 *   gmcp_kinematics            sample_kinematics          contact_energy.hpp:26-73
 *   gmcp_resolve_barrier_params resolve_barrier_params    barrier.hpp:25-46
 */
#ifndef GMCP_B200_H
#define GMCP_B200_H

#include "gmcp_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmcp_ctx gmcp_ctx;

/* ---- context -------------------------------------------------------------- */
int gmcp_ctx_create(int device, gmcp_ctx** out);
void gmcp_ctx_destroy(gmcp_ctx* ctx);
const char* gmcp_last_error(void);       /* thread-local message of the last failure */
int gmcp_device_count(int* n);
/* Number of kernels this library launched on ctx since creation (evidence for
 * bench.py's gpu_launches). */
int64_t gmcp_launch_count(const gmcp_ctx* ctx);

/* ---- inputs (host buffers, copied to the device) ------------------------------ */
int gmcp_resolve_barrier_params(gmcp_barrier_params* p, double mean_slave_edge);
int gmcp_set_params(gmcp_ctx* ctx, const gmcp_barrier_params* p); /* resolved params */
int gmcp_set_surfaces(gmcp_ctx* ctx, const gmcp_surface* slave, const gmcp_surface* master);
/* x: flat 3N positions. n_dof fixes N for the context (may change). */
int gmcp_set_positions(gmcp_ctx* ctx, const double* x, int64_t n_dof);
int gmcp_set_step(gmcp_ctx* ctx, const double* dx, int64_t n_dof);
/* Batched independent scenes (no reference equivalent -- the
 * reference runs one scene per System): scene[v] is the scene of vertex v
 * (n_vertices = N, scenes numbered 0..S-1, S <= 2^20), or NULL for one scene.
 * The broadphase then pairs a slave triangle only with master triangles of
 * its own scene (scene taken from the triangle's first vertex), so a packed
 * batch yields exactly the concatenation of the per-scene candidate sets and
 * samples. Every later stage is per sample / per vertex and needs no change. */
int gmcp_set_vertex_scenes(gmcp_ctx* ctx, const int32_t* scene, int64_t n_vertices);
/* Device-resident fast path: the context's own x / dx buffers (3N doubles,
 * valid after gmcp_set_positions / gmcp_set_step sized them). */
double* gmcp_positions_device(gmcp_ctx* ctx);
double* gmcp_step_device(gmcp_ctx* ctx);

/* ---- broadphase + sampler (per rebuild) ---------------------------------------- */
/* Candidate master tris/edges/verts per slave triangle at the current x,
 * inflated-AABB overlap with radius r. counts = {tris, edges, verts}. */
int gmcp_broadphase(gmcp_ctx* ctx, double r, int64_t* counts);
/* which: 0 tris, 1 edges, 2 verts; offsets has n_slave_tris+1 entries. */
int gmcp_download_pairs(gmcp_ctx* ctx, int which, int64_t* offsets, int32_t* ids);
int gmcp_upload_pairs(gmcp_ctx* ctx, const int64_t* tri_off, const int32_t* tri_ids,
                      const int64_t* edge_off, const int32_t* edge_ids, const int64_t* vert_off,
                      const int32_t* vert_ids);
/* Samples the current pair set at the current x (build_contact_state).
 * eps_reference (host, 3N, nullable) anchors the support radii. */
int gmcp_build_samples(gmcp_ctx* ctx, const double* eps_reference, int64_t* n_samples);
/* Replace the frozen sample set (e.g. hand-built states, oracle inputs). */
int gmcp_upload_samples(gmcp_ctx* ctx, const gmcp_samples* s);
int64_t gmcp_num_samples(const gmcp_ctx* ctx);
int gmcp_download_samples(gmcp_ctx* ctx, gmcp_samples* out);

/* ---- per Newton iteration (at the context's current x / dx) --------------------- */
int gmcp_try_energy(gmcp_ctx* ctx, double* energy, double* min_gap, int32_t* feasible);
/* On a non-positive gap: GMCP_ERR_INFEASIBLE with *bad = lowest offending index. */
int gmcp_energy(gmcp_ctx* ctx, double* energy, int64_t* bad);
/* grad (host, 3N) is accumulated into, never cleared; may be null to keep the
 * gradient on the device only. */
int gmcp_gradient(gmcp_ctx* ctx, double* grad, double* energy, int64_t* bad);
/* Gradient plus the Gauss-Newton Hessian assembled into the context's BCSR
 * (3x3 blocks, rows = all N vertices, columns sorted). */
int gmcp_gradient_hessian(gmcp_ctx* ctx, double* grad, double* energy, int64_t* bad);
/* One call with the reference signature add_contact_gradient[_hessian](state,
 * params, x, grad[, H]) (contact_energy.hpp:126-179): positions x (host, 3N)
 * become the context's positions, grad (host, 3N, may be null) is accumulated
 * into, the Hessian stays in the context's BCSR. Transfers overlap the
 * assembly (grad goes up during K7 and comes down while the Hessian blocks are
 * gathered); one synchronisation. On GMCP_ERR_INFEASIBLE / _DEGENERATE grad is
 * unchanged. */
int gmcp_add_gradient(gmcp_ctx* ctx, const double* x, int64_t n_dof, double* grad, double* energy,
                      int64_t* bad);
int gmcp_add_gradient_hessian(gmcp_ctx* ctx, const double* x, int64_t n_dof, double* grad,
                              double* energy, int64_t* bad);
/* BCSR download: rowptr has N+1 entries; call with null arrays to get nnzb. */
int gmcp_download_hessian(gmcp_ctx* ctx, int64_t* nnzb, int32_t* rowptr, int32_t* cols,
                          double* vals);
int gmcp_step_filter(gmcp_ctx* ctx, double* alpha);
int gmcp_displacement_cap(gmcp_ctx* ctx, double* alpha);
/* out may be null to count face samples. */
int gmcp_pressure_field(gmcp_ctx* ctx, int64_t* n, gmcp_pressure_record* out);
int gmcp_force_summary(gmcp_ctx* ctx, double* out12);
/* Per-sample gap, vertex count, ids[6], dg[6][3] (parity / debugging). */
int gmcp_kinematics(gmcp_ctx* ctx, double* g, int32_t* nv, int32_t* ids, double* dg);

/* ---- timing helpers for the benchmark (device events on the ctx stream) ------- */
/* Runs the assembly pass (energy + gradient + Hessian blocks) `reps` times
 * back to back on device-resident data and returns the mean milliseconds per
 * pass of the whole pass and of its dominant kernel. */
int gmcp_time_assembly(gmcp_ctx* ctx, int reps, int flush_l2, double* ms_pass, double* ms_kernel);

/* ---- dual-mesh embedding (embedding.hpp:26-106) ------------ */
/* embed_in_surface: each point binds to the host triangle with the smallest
 * point-triangle distance (lowest index on ties; LBVH branch and bound, equal
 * to the reference's tree and brute-force results) and stores unclamped plane
 * barycentrics (3 per point) and the signed offset along the triangle normal.
 * host: n_host_vertices xyz, n_host_tris local-id triangles. A zero-area host
 * triangle returns GMCP_ERR_DEGENERATE with *bad = its index. */
int gmcp_embed_in_surface(gmcp_ctx* ctx, const double* points, int64_t n_points, const double* host_vertices,
                          int64_t n_host_vertices, const int32_t* host_tris, int64_t n_host_tris, int32_t* tri,
                          double* bary, double* offset, int64_t* bad);
/* apply_embedding: reconstruct the embedded points from deformed host
 * positions. A host triangle that degenerated returns GMCP_ERR_DEGENERATE
 * with *bad = that triangle (of the first embedded point using it). */
int gmcp_apply_embedding(gmcp_ctx* ctx, const int32_t* tri, const double* bary, const double* offset, int64_t n,
                         const int32_t* host_tris, int64_t n_host_tris, const double* host_positions,
                         int64_t n_host_vertices, double* out, int64_t* bad);

#ifdef __cplusplus
}
#endif

#endif /* GMCP_B200_H */
