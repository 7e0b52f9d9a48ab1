/*
 * pf_b200.h — C-ABI of the B200-native staggered phase-field fracture hot path.
 *
 * This library replaces the inner solves of the reference's load-step entry point
 *   phasefrac.schemes.staggered_step(disc, state, scheme, bc_increments, params, config,
 *                                    pinned_d_nodes)            (schemes.py:332-392)
 * and the helpers it and its caller use:
 *   solve_momentum        (schemes.py:192-239)   -> pf_solve_momentum
 *   solve_evolution       (schemes.py:242-313)   -> pf_solve_evolution
 *   evolution_residual_norm (schemes.py:316-329) -> pf_evolution_residual_norm
 *   reaction_force        (assembly.py:315-326)  -> pf_reaction_force
 *   internal_force        (assembly.py:161-171)  -> pf_internal_force
 *   assemble_momentum     (assembly.py:174-198)  -> pf_momentum_tangent_apply (matrix-free K_uu x)
 *   assemble_evolution    (assembly.py:201-247)  -> pf_evolution_residual / pf_evolution_tangent_apply
 *   refresh_gp_from_displacement (assembly.py:260-269) -> pf_refresh_gp
 *   softening_gate / extra_stiffness / update_active_energy (schemes.py:96-176)
 *                                                -> pf_softening_gate / pf_extra_stiffness /
 *                                                   pf_update_active_energy
 *   factor_solve(.., "cg") / check_spd (linsolve.py:44-77) -> device Jacobi-PCG with the
 *                                                   curvature SPD predicate (inside the solves)
 *
 * The reference has no FFI: its seam is a Python signature.  The Python
 * drop-in (paper_2209_07969_b200.schemes.staggered_step) binds these entry points with ctypes;
 * INTEGRATION.md shows the binding.  Plain pointers and sizes only; all host arrays are
 * C-contiguous float64 / int64 in the reference's own layouts:
 *   u        [2*n_nodes]   interleaved (ux, uy) per node      (assembly.py:132-134)
 *   d, d_prev[n_nodes]
 *   GP arrays[n_elems*4]   (n_elems, 4) row-major, GP order (-,-),(+,-),(+,+),(-,+)
 *   DOF index = 2*node + component                          (assembly.py:272-276)
 *
 * Every function returns a pf_status; on failure pf_last_error() describes it.  State after a
 * convergence error is unspecified, as in the reference (SURVEY.md §8(b) "Errors").
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PF_OK = 0,
  PF_ERR_INVALID = 1,          /* -> ValueError                                   */
  PF_ERR_INDEX = 2,            /* -> IndexError (apply_dirichlet, assembly.py:292) */
  PF_ERR_CONV_MOMENTUM = 3,    /* -> ConvergenceError (schemes.py:227-231)        */
  PF_ERR_CONV_EVOLUTION = 4,   /* -> ConvergenceError (schemes.py:287-291)        */
  PF_ERR_CONV_STAGGERED = 5,   /* -> ConvergenceError (schemes.py:366-370)        */
  PF_ERR_SINGULAR = 6,         /* -> SingularSystemError (linsolve.py:52-53)      */
  PF_ERR_CUDA = 7,             /* device / driver failure                          */
  PF_ERR_NCCL = 8              /* collective failure (row-strip decomposition)     */
} pf_status;

typedef enum { PF_ST = 0, PF_S1 = 1, PF_S2 = 2, PF_S3 = 3 } pf_scheme; /* schemes.py:33-37 */

/* Structured row-compact Q4 mesh with uniform rectangular cells hx x hy.
 * Node (i, j) exists iff node_lo[j] <= i < node_hi[j]; its id is node_start[j] + i - node_lo[j].
 * Cell (i, j) exists iff elem_lo[j] <= i < elem_hi[j]; its id is elem_start[j] + i - elem_lo[j];
 * its nodes are (i,j), (i+1,j), (i+1,j+1), (i,j+1) (CCW, meshing.py:116) except that cells of
 * row notch_row use the duplicate of (c, notch_row) for bottom corners with notch_lo <= c <
 * notch_hi; that duplicate's id is dup_start + c - notch_lo (meshing.py:126-138).
 * This covers build_notched_square (meshing.py:90-151) and build_lshape_mesh (:159-215). */
typedef struct {
  int32_t nx, ny;              /* bounding cell grid                                 */
  double hx, hy;               /* uniform cell size                                  */
  const int32_t* node_lo;      /* [ny+1] */
  const int32_t* node_hi;      /* [ny+1] */
  const int64_t* node_start;   /* [ny+1] */
  const int32_t* elem_lo;      /* [ny]   */
  const int32_t* elem_hi;      /* [ny]   */
  const int64_t* elem_start;   /* [ny]   */
  int32_t notch_row;           /* -1 when there is no slit */
  int32_t notch_lo, notch_hi;
  int64_t dup_start;
  int64_t n_nodes, n_elems;
} pf_mesh;

/* MaterialParams (material.py:31-96) after __post_init__ derivation. */
typedef struct {
  double mu, lam, bulk_k, g_c, length_l, eta, c_w, gamma;
  int32_t at2;                 /* 1 = AT2, 0 = AT1 */
} pf_material;

/* SolverConfig (schemes.py:40-54). */
typedef struct {
  double tol_nr, tol_st, d_cap, res_floor;
  int32_t max_nr, max_stag;
  double cg_rtol;              /* 1e-12, linsolve.py:51 */
  int32_t cg_maxiter_factor;   /* 20,    linsolve.py:51 */
} pf_config;

/* StaggeredStats (schemes.py:57-68) plus device counters. */
typedef struct {
  int32_t n_stag, n_nr_u, n_nr_d, spd_fallbacks;
  double final_rd_ratio, final_ru_ratio, wall_u, wall_d;
  int32_t n_hist;              /* entries written to the residual-history buffer */
  int64_t cg_iters_u, cg_iters_d;          /* PCG iterations executed              */
  double cg_dofiters_u, cg_dofiters_d;     /* sum over PCG iterations of free DOFs */
  double kernel_ms_u, kernel_ms_d;         /* CUDA-event time inside the PCG kernels */
  int32_t cg_launches_u, cg_launches_d;
  int32_t launches;                        /* all kernels launched by this call    */
  double step_ms;                          /* CUDA-event time of the whole call    */
} pf_stats;

typedef struct pf_handle pf_handle;

/* lifecycle ------------------------------------------------------------------------------ */
pf_status pf_create(const pf_mesh* mesh, const pf_material* mat, const pf_config* cfg,
                    int device, pf_handle** out);
void pf_destroy(pf_handle* h);
const char* pf_last_error(const pf_handle* h);
const char* pf_version(void);

/* state mirror (SolverState, schemes.py:71-87; GaussPointState, assembly.py:46-72).
 * Any pointer may be NULL to skip that array. */
pf_status pf_set_state(pf_handle* h, const double* u, const double* d, const double* d_prev,
                       const double* tr_eps_plus, const double* dev_dot_dev,
                       const double* psi_plus, const double* psi_max);
pf_status pf_get_state(pf_handle* h, double* u, double* d, double* d_prev,
                       double* tr_eps_plus, double* dev_dot_dev, double* psi_plus,
                       double* psi_max);
/* Device-side state construction: the zero state of SolverState.zeros
 * (schemes.py:80-87) and d = d_prev = 1 at every node within `radius` of one of the
 * n_segments pre-crack segments (segments[4k..4k+3] = ax, ay, bx, by; configs.precrack_nodes),
 * node (i, j) at (i hx, j hy) with the last column / row at x_last / y_last (np.linspace).
 * No host state arrays are needed (config 5: 8.6 GB of zero GP arrays otherwise).
 * Single-GPU handles only. */
pf_status pf_init_state(pf_handle* h, const double* segments, int64_t n_segments,
                        double radius, double x_last, double y_last);
/* gp.strain [n_elems*4*4] Voigt (xx,yy,zz,xy) and gp.tr_eps [n_elems*4] recomputed from u
 * (refresh_gp_from_displacement, assembly.py:260-269). */
pf_status pf_get_gp_strain(pf_handle* h, double* strain, double* tr_eps);
/* Discretization.interp_nodal (assembly.py:148-150): the nodal scalar field field[n_nodes]
 * interpolated at the 4 Gauss points of every cell, out[n_elems*4] (reference GP order). */
pf_status pf_interp_nodal(pf_handle* h, const double* field, double* out);
/* Page-locked host buffers (cudaHostAlloc): state arrays in them move by direct DMA in
 * pf_set_state / pf_get_state / pf_get_gp_strain (other host pointers go through the handle's
 * pinned staging buffer). */
pf_status pf_host_alloc(int64_t bytes, void** out);
void pf_host_free(void* p);

/* hot path: one load step (schemes.py:332-392).
 * Boundary pairs: pair k covers bc_dofs[bc_offsets[k] .. bc_offsets[k+1]) with increment
 * bc_incs[k].  pins: pinned phase-field nodes (may be NULL / 0).  hist receives
 * residual_history (capacity hist_cap). */
pf_status pf_staggered_step(pf_handle* h, int scheme, const int64_t* bc_dofs,
                            const int64_t* bc_offsets, const double* bc_incs, int32_t n_bc,
                            const int64_t* pins, int64_t n_pins, pf_stats* out, double* hist,
                            int32_t hist_cap);

/* inner solvers exposed for solver-level parity (r0 in/out: NaN = "not yet set", like the
 * reference's _StepContext, schemes.py:179-185). */
pf_status pf_solve_momentum(pf_handle* h, const int64_t* bc_dofs, const int64_t* bc_offsets,
                            const double* bc_incs, int32_t n_bc, double* r0_u,
                            int32_t* n_nr, double* last_ratio);
pf_status pf_solve_evolution(pf_handle* h, int scheme, const int64_t* pins, int64_t n_pins,
                             double* r0_d, int32_t* n_nr, int32_t* spd_fallbacks);
pf_status pf_evolution_residual_norm(pf_handle* h, const int64_t* pins, int64_t n_pins,
                                     double* out);
/* commit at step acceptance: psi_max = max(psi_max, psi_plus); d_prev = d (schemes.py:390-391) */
pf_status pf_commit_step(pf_handle* h);

/* operators at the handle's current state (kernel-level parity) */
pf_status pf_internal_force(pf_handle* h, double* f_out);
pf_status pf_reaction_force(pf_handle* h, const int64_t* nodes, int64_t n, int component,
                            double* out);
pf_status pf_momentum_tangent_apply(pf_handle* h, const double* x, double* y, double* diag);
pf_status pf_evolution_residual(pf_handle* h, double* r_out);
pf_status pf_evolution_tangent_apply(pf_handle* h, int scheme, const double* x, double* y,
                                     double* diag);
pf_status pf_refresh_gp(pf_handle* h);
pf_status pf_softening_gate(pf_handle* h, uint8_t* gate_out);
pf_status pf_extra_stiffness(pf_handle* h, int scheme, double* extra_out);
pf_status pf_update_active_energy(pf_handle* h, int scheme, const double* delta_d_nodal);

/* row-strip decomposition ---------------------------------------------
 * Each rank owns a contiguous range of node rows of the global mesh; its handle is created on
 * the LOCAL row-compact sub-mesh (owned rows plus one ghost row per neighbour, plus the slit
 * duplicates when it owns the slit row; paper_2209_07969_b200/strips.py builds it).  Owned
 * nodes: [own_lo, own_hi) and [dup_lo, n_nodes); owned cells: [cell_lo, cell_hi).  Halo rows
 * are contiguous local ranges.  comm_kind 0 = NCCL (nccl_id from pf_nccl_unique_id on rank 0,
 * broadcast by the caller); 1 = in-process host emulation (host_group from
 * pf_host_group_create, one host thread per strip, all strips on the same GPU — tests). */
typedef struct {
  int32_t rank, nranks;
  int64_t own_lo, own_hi, dup_lo, cell_lo, cell_hi;
  int64_t send_lo_start, send_lo_count, recv_lo_start, recv_lo_count;
  int64_t send_hi_start, send_hi_count, recv_hi_start, recv_hi_count;
  int32_t comm_kind;
  unsigned char nccl_id[128];
  void* host_group;
} pf_strip;

pf_status pf_nccl_unique_id(unsigned char out[128]);
pf_status pf_host_group_create(int32_t nranks, void** out);
void pf_host_group_destroy(void* group);
pf_status pf_create_strip(const pf_mesh* local_mesh, const pf_material* mat, const pf_config* cfg,
                          int device, const pf_strip* strip, pf_handle** out);

/* device-resident benchmarking helpers */
/* n_iter PCG iterations of the momentum (physics 0) or phase-field (1) operator at the current
 * state with the stopping test disabled (rtol 0): per-iteration cost at any mesh size without
 * solving to convergence; physics 2 = the multigrid-preconditioned momentum PCG (including its
 * per-solve hierarchy setup), 3 = the scalar phase-field multigrid PCG (pf_mgs.cuh, including
 * its hierarchy setup).  ms_out = CUDA-event time of the PCG launch. */
pf_status pf_bench_cg(pf_handle* h, int physics, int64_t n_iter, double* ms_out,
                      int64_t* iters_out);
pf_status pf_device_info(pf_handle* h, int32_t* cg_grid, int32_t* sm_count, int64_t* l2_bytes);
/* Benchmark helper (not on the solve path): average device time of one fine-level multigrid
 * march, re-launched `reps` times on the current hierarchy / state with CUDA events (kernels of
 * the conditional solve graph cannot be event-timed individually).  which: 0 / 1 / 2 momentum
 * fine residual, smoothing, PCG-direction march; 10 / 11 / 12 the same for the scalar
 * phase-field hierarchy.  bytes_out: algorithmic bytes per launch. */
pf_status pf_bench_mg_kernel(pf_handle* h, int which, int reps, double* ms_out,
                             double* bytes_out);
/* Multigrid hierarchy of the momentum PCG (replaces the Jacobi preconditioner M = D^-1 of
 * linsolve.py:49 by a Galerkin V-cycle; same system, same stopping test): level count, first
 * level of the single-CTA tail kernel (n_levels: none), dense coarsest solve, hierarchy builds
 * so far; omega (optional, [n_levels]) builds the hierarchy at the current state and returns
 * the damped-Jacobi weights 4 / (3 lambda_max(D^-1 A_l)).  n_levels = 0: this handle solves
 * with Jacobi PCG (PFB200_MG=0, strips, meshes that do not agglomerate). */
pf_status pf_mg_info(pf_handle* h, int32_t* n_levels, int32_t* n_grid, int32_t* dense,
                     int64_t* setups, double* omega);
/* Linear solver of each Newton system on this handle (all solve the reference's CG system of
 * linsolve.py:48-54 to the same stopping test).  momentum: 0 two-barrier Jacobi PCG (k_cg),
 * 1 single-reduction Jacobi PCG (k_cg_sr), 2 multigrid PCG.  phase_field (solves without the
 * SPD probe; probe solves always run k_cg): 0 k_cg, 1 k_cg_sr (matrix-free march), 2 k_cg_st
 * (assembled stencil, L2-resident meshes), 3 multigrid PCG on the two-component packing
 * (PFB200_MG_EVO=packed), 4 native scalar multigrid PCG (pf_mgs.cuh). */
pf_status pf_solver_kinds(pf_handle* h, int32_t* momentum, int32_t* phase_field);
pf_status pf_flush_l2(pf_handle* h);
pf_status pf_synchronize(pf_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* PF_B200_H */
