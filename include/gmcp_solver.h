/* GMCP B200 quasi-static solver C-ABI: the device-resident replacement of
 * gmcp::System (proj/include/gmcp/solver.hpp:63-376). Bodies are linear-
 * elastic tet meshes (elasticity.hpp), Dirichlet dofs are eliminated by
 * masking, contact pairs run the GMCP pipeline of include/gmcp_b200.h, and
 * the Newton direction comes from a block-Jacobi preconditioned CG on the
 * 3x3 BCSR Hessian instead of the reference's SimplicialLDLT
 * (solver.hpp:325-375).
 *
 *   gmcp_system_add_body          System::add_body            solver.hpp:73-91
 *   gmcp_system_fix_dofs          System::fix_dof / fix_vertex solver.hpp:97-105
 *   gmcp_system_set_external_force System::f_ext              solver.hpp:69
 *   gmcp_system_add_contact_pair  System::add_contact_pair    solver.hpp:110-121
 *                                 (surfaces + params resolved by the caller)
 *   gmcp_system_solve             System::solve               solver.hpp:125-228
 */
#ifndef GMCP_SOLVER_H
#define GMCP_SOLVER_H

#include "gmcp_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmcp_system gmcp_system;

/* SolverSettings (solver.hpp:35-42) + the Krylov controls that replace LDL^T. */
typedef struct {
  int32_t load_steps;        /* 10 */
  int32_t max_newton_iters;  /* 200 */
  double newton_tol;         /* <= 0: derived from loads (solver.hpp:256-269) */
  int32_t max_line_search;   /* 40 */
  double pcg_tol;            /* relative residual ||r||_2 / ||b||_2, e.g. 1e-10 */
  int32_t pcg_max_iters;     /* e.g. 20000 */
} gmcp_solver_settings;

/* StepStats (solver.hpp:44-53) + PCG iterations. */
typedef struct {
  int32_t step, newton_iters, rebuilds, backtracks;
  int64_t pcg_iters;
  double residual, energy, min_gap;
  int32_t energy_monotone;
} gmcp_step_stats;

/* RunStats (solver.hpp:55-61). residual is set when a solve fails. */
typedef struct {
  int64_t total_newton_iters, total_rebuilds, total_pcg_iters;
  double newton_tol_used, wall_seconds, residual;
} gmcp_run_stats;

/* StepCallback (solver.hpp:123): stats and the host copy of x after each load step. */
typedef void (*gmcp_step_callback)(const gmcp_step_stats* stats, const double* x, int64_t n_dof, void* user);

const char* gmcp_system_last_error(void);
int gmcp_system_create(int device, gmcp_system** out);
void gmcp_system_destroy(gmcp_system* sys);
int gmcp_system_add_body(gmcp_system* sys, const double* verts, int64_t n_verts, const int32_t* tets,
                         int64_t n_tets, double youngs, double poisson, int32_t* vertex_offset);
int gmcp_system_fix_dofs(gmcp_system* sys, int64_t n, const int64_t* dofs, const double* targets);
int gmcp_system_set_external_force(gmcp_system* sys, const double* f_ext, int64_t n_dof);
int gmcp_system_add_contact_pair(gmcp_system* sys, const gmcp_surface* slave, const gmcp_surface* master,
                                 const gmcp_barrier_params* resolved, int32_t* pair_id);
/* On failure returns GMCP_ERR_SOLVER / GMCP_ERR_CONFIG like the reference's
 * SolverError / ConfigError; out->residual carries SolverError::residual. */
int gmcp_system_solve(gmcp_system* sys, const gmcp_solver_settings* settings, gmcp_step_callback cb,
                      void* user, gmcp_run_stats* out);
/* Benchmark hook: runs the solve from the current state and stops after
 * n_iters Newton iterations (SURVEY.md 8d "Newton steps/s"), returning the
 * wall milliseconds of each full iteration (assembly, residual, PCG to
 * tolerance, filter + cap, every line-search trial, rebuild check) and its
 * PCG iteration count. */
int gmcp_system_time_newton(gmcp_system* sys, const gmcp_solver_settings* settings, int32_t n_iters,
                            double* ms_per_iter, int64_t* pcg_per_iter, int32_t* n_done);
/* PCG measurement (no reference counterpart): device ms and iterations of
 * the PCG chunk graphs since the last gmcp_system_time_newton started (CUDA
 * events on the solve stream), and the merged operand's shape (rows, 3x3
 * blocks). */
int gmcp_system_pcg_stats(const gmcp_system* sys, double* ev_ms, int64_t* ev_iters, int64_t* n_rows,
                          int64_t* nnzb);
/* Preconditioner of the single-system PCG after a solve: vertex-pair 6x6
 * block-Jacobi on/off, two-level coarse space on/off, its aggregate count and
 * padded coarse dimension (runtime switches GMCP_PAIR_JACOBI, GMCP_COARSE,
 * GMCP_COARSE_AGGS; both default on). */
int gmcp_system_precond_info(gmcp_system* sys, int32_t* pair_jacobi, int32_t* coarse, int32_t* n_aggregates,
                             int32_t* n_coarse_padded);
/* Standalone Newton linear solve: replaces solve_descent (solver.hpp:325-375)
 * under the reference's own CPU System. The matrix is an AoS BCSR of 3x3
 * blocks over n_vertices (rowptr[n_vertices + 1], ascending columns per row,
 * vals[9 nnzb] row-major blocks): H = the assembled elastic + contact Hessian
 * over all dofs; fixed[3 n_vertices] (or NULL) marks Dirichlet dofs, which are
 * eliminated as P H P + I - P with the rhs masked (solver.hpp:271-277, 331-341).
 * positions[3 n_vertices] (or NULL) enable the two-level preconditioner's
 * geometric aggregates. Solves H dx = rhs with the device PCG to pcg_tol and
 * accepts as the reference accepts its LDL^T solve (||H dx - rhs||_inf <= 1e-6
 * ||rhs||_inf); otherwise retries with the diagonal shifted by 1e-8 x the mean
 * free diagonal entry (*regularized = 1), and returns GMCP_ERR_SOLVER if that
 * fails too (the reference's SolverError). Use a system handle with no bodies
 * and no contact pairs. */
int gmcp_system_linear_solve(gmcp_system* sys, int64_t n_vertices, const int32_t* rowptr, const int32_t* cols,
                             const double* vals, const uint8_t* fixed, const double* positions, const double* rhs,
                             double pcg_tol, int32_t max_iters, double* dx, int32_t* iterations,
                             double* residual_inf_rel, int32_t* regularized);
/* PCG operand storage: *stored_blocks = 3x3 blocks the SpMV streams from the
 * symmetric-half copy (blocks on and above the diagonal, once each; 0 when
 * the SpMV reads the full merged BCSR: batched scenes, GMCP_HALF_SPMV=0). */
int gmcp_system_operand_info(gmcp_system* sys, int64_t* stored_blocks);
int gmcp_system_positions(gmcp_system* sys, double* x, int64_t n_dof);
int gmcp_system_set_positions(gmcp_system* sys, const double* x, int64_t n_dof);
int64_t gmcp_system_num_samples(gmcp_system* sys, int32_t pair);
int gmcp_system_pair_force_summary(gmcp_system* sys, int32_t pair, double* out12);
int gmcp_system_pair_pressure(gmcp_system* sys, int32_t pair, int64_t* n, gmcp_pressure_record* out);
int64_t gmcp_system_launch_count(const gmcp_system* sys);
/* Batched independent scenes (gmcp_system_set_vertex_scenes):
 * the StepStats of every scene for every completed load step of the last
 * solve, out[step * n_scenes + scene] (pass out = null to query n_steps);
 * residual / energy / min_gap / backtracks / rebuilds / newton_iters are the
 * scene's own (pcg_iters is 0: the per-scene CTA PCG runs all scenes at once). */
int gmcp_system_scene_step_stats(gmcp_system* sys, int32_t* n_steps, gmcp_step_stats* out);
/* Sample offsets of each scene inside a pair's packed sample set after the
 * last batched solve ([n_scenes + 1]; the pressure records of scene s are the
 * records whose sample index lies in [soff[s], soff[s+1])). */
int gmcp_system_pair_scene_offsets(gmcp_system* sys, int32_t pair, int64_t* soff);
/* Linear-solve parity (solver.hpp:349-356: the reference accepts a solve iff
 * ||M s - rhs||_inf <= 1e-6 ||rhs||_inf). After every PCG solve the residual
 * of the masked Newton system is RECOMPUTED (not PCG's recursive residual);
 * a solve is accepted only if it converged and passes the reference's
 * inf-norm test, else it is retried regularized like the reference. Returns
 * the maxima of ||H dx - rhs||_2/||rhs||_2 and of the inf-norm ratio over the
 * solves since the last reset, and their count. */
int gmcp_system_linear_stats(gmcp_system* sys, int32_t reset, double* max_rel2, double* max_relinf,
                             int64_t* n_solves);
/* Inspection: when on, every solve copies its linear system to the host (the
 * operand as one AoS BCSR with all sources summed, Dirichlet mask, gradient
 * (rhs = -mask .* grad), solution dx, diagonal shift); the last one is read
 * back with gmcp_system_captured_linear_system (pass null arrays to query
 * nnzb; rowptr has n_vertices + 1 entries, vectors n_dof). */
int gmcp_system_capture_linear_system(gmcp_system* sys, int32_t on);
int gmcp_system_captured_linear_system(gmcp_system* sys, int64_t* nnzb, int32_t* rowptr, int32_t* cols, double* vals,
                                       double* mask, double* grad, double* dx, double* shift);

/* Batched independent scenes. scene[v] numbers the scenes
 * 0, 1, ... over contiguous vertex ranges (no body spans two scenes); NULL
 * clears. gmcp_system_solve then runs every scene with its own residual
 * tolerance (derived from that scene's loads and bodies), step filter, cap,
 * line search and convergence; the linear solve is one PCG over the active
 * scenes. gmcp_run_stats.total_newton_iters then counts scene-Newton-
 * iterations (sum over scenes); per-step newton_iters counts loop passes. */
int gmcp_system_set_vertex_scenes(gmcp_system* sys, const int32_t* scene, int64_t n_vertices);
/* Batched gmcp_system_time_newton: scenes iterated in each timed loop pass. */
int gmcp_system_timed_active_scenes(const gmcp_system* sys, int64_t* out, int32_t n);
/* Newton iterations per scene of the last batched solve (out[n_scenes]). */
int gmcp_system_scene_newton_iters(const gmcp_system* sys, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif
