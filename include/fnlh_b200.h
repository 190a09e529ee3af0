/*
 * fnlh_b200.h -- C ABI of the B200-native FNLH implicit pseudo-time hot path.
 *
 * Plain pointers and sizes only.  Host-buffer entry points take the reference's
 * layouts: BlockVec node-major AoS v[i*b+m] (core.hpp:62-91), complex values as
 * interleaved (re, im) doubles (std::complex<double>), Bsr row-major b x b blocks in
 * CSR order with ascending columns and the diagonal included (sparse.hpp:136-157).
 * Every function returns 0 on success or a status code mirroring the reference
 * exception taxonomy (core.hpp:22-56); fnlh_last_error*() give the message and the
 * node / stage payload of FactorizationError / DivergenceError.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj/src).  INTEGRATION.md shows the reference-side binding.
 */
#ifndef FNLH_B200_H
#define FNLH_B200_H

#ifdef __cplusplus
extern "C" {
#endif

enum fnlh_status {
    FNLH_OK = 0,
    FNLH_CONFIG = 1,        /* ConfigError */
    FNLH_STATE = 2,         /* StateError */
    FNLH_SHAPE = 3,         /* ShapeError */
    FNLH_UNSUPPORTED = 4,   /* UnsupportedCaseError */
    FNLH_FACTORIZATION = 5, /* FactorizationError(node) */
    FNLH_DIVERGENCE = 6,    /* DivergenceError(stage, field) */
    FNLH_CUDA = 7,          /* device / runtime failure */
    FNLH_NONCONVERGENCE = 8 /* NonConvergenceError (core.hpp:54-56): the URANS oracle's period cap */
};

typedef struct fnlh_pattern fnlh_pattern;
typedef struct fnlh_disc fnlh_disc;
typedef struct fnlh_solver fnlh_solver;
typedef struct fnlh_sector_dual fnlh_sector_dual;

/* LinearSolveReport (sparse.hpp:231-236) */
typedef struct {
    int iterations;
    double initial_residual;
    double final_residual;
    int converged;
} fnlh_linear_report;

const char* fnlh_last_error(void);
int fnlh_last_error_node(void);
int fnlh_last_error_stage(void);
int fnlh_device_count(void);
/* make `device` current for the calling host thread (one process per GPU: the local rank) */
int fnlh_set_device(int device);
/* Boundary-state pow (disc_euler.cpp:179-180,187).  0: glibc's pow restated bit for bit
   (its tables located in the libm this process loaded and the restatement checked against
   ::pow on a fixed sample at first use, csrc/libm_pow.cuh) -- the device then rounds every
   boundary state as the reference does; 1: correctly rounded (tables absent, the check
   failed, or FNLH_POW=cr in the environment).  fnlh_pow evaluates the selected routine on
   the host (for tests). */
int fnlh_pow_mode(void);
const char* fnlh_pow_mode_info(void);
double fnlh_pow(double x, double y);
/* number of CUDA kernels this library has launched (monotonic) */
long long fnlh_launch_count(void);
/* Guard builds only (-DFNLH_GUARD, a measurement variant of the library): every device
   buffer carries 4 KiB guard zones of 0xFF bytes on both sides (the reference's
   CountedBuffer canaries, sparse.hpp:40-100); *bad_bytes = guard bytes overwritten so far
   (live buffers and freed ones), *blocks = live guarded buffers.  Product builds return
   FNLH_UNSUPPORTED. */
int fnlh_guard_check(long long* bad_bytes, long long* blocks);

/* ---- L1: block-sparse LA --------------------------------------------------- */

/* BlockSparsityPattern + make_pattern/validate (sparse.hpp:106-134, sparse.cpp:42-117);
   partition may be NULL (single partition).  Computes the ILU(0) level schedule of the
   given ordering. */
int fnlh_pattern_create(int b, int rows, const int* row_ptr, const int* col_idx, const int* partition,
                        fnlh_pattern** out);
void fnlh_pattern_destroy(fnlh_pattern* p);
int fnlh_pattern_levels(const fnlh_pattern* p, int* fwd_levels, int* bwd_levels);

/* The system matrix, in the two forms the reference builds:
     is_complex = 0: real Bsr<real> values A (nnzb*b*b doubles)             (mean-flow A5)
     is_complex = 1, A_complex != 0: Bsr<cplx> values (nnzb*b*b*2 doubles)
     is_complex = 1, A_complex == 0: real A5 + per-node diagonal shift i*shift_im[i]
                                     (build_lhs_harmonic -> shift_diagonal, rk.cpp:32-39,
                                     sparse.cpp:157-171), never materialized.            */

/* Ilu<S>::factorize (sparse.cpp:187-257); outputs in the reference's Ilu layout
   (any output may be NULL). */
int fnlh_ilu_factorize(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                       double* vals, double* diag_lu, int* diag_piv, double* diag_inv);
/* factorize + Ilu<S>::apply (sparse.cpp:259-291) */
int fnlh_ilu_apply(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                   const double* rhs, double* x);
/* Bsr<S>::matvec (sparse.hpp:259-270) */
int fnlh_matvec(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                const double* x, double* y);
/* factorize + smoothed_solve<S, Ilu<S>> (sparse.hpp:295-331) */
int fnlh_smoothed_solve(const fnlh_pattern* p, int is_complex, const double* A, int A_complex,
                        const double* shift_im, const double* rhs, double tol_rel, int max_iter, double* x,
                        fnlh_linear_report* rep);

/* ---- L1, persistent operator handles (the drop-in at the reference's call sites) ----
   The reference builds A5 once per outer iteration and, per harmonic worker, factorizes
   once per harmonic (driver.cpp:213-216: build_lhs_harmonic + Ilu::factorize) and then
   solves once per RK stage with the same factors (rk.cpp:82-85: smoothed_solve).  These
   handles keep that structure on the device: the LHS is uploaded once, each worker's
   factors stay resident in its own workspace, and a stage solve moves only rhs and x.

   fnlh_lhs    the shared real LHS (J / A5: Bsr<real>, sparse.hpp:136-157) on a pattern,
               resident in HBM in the layouts the kernels read (2-colour SELL-32, or BSR +
               sliced copy).  fnlh_lhs_upload replaces the values (reference BSR layout,
               nnzb*b*b doubles).  Replaces the Bsr<real> A5 of driver.cpp:67,179-181.
   fnlh_prec   one worker's Ilu<S> workspace (sparse.cpp:187-257; the per-worker Ilu of
               driver.cpp:117) on an fnlh_lhs: fnlh_prec_factorize factorizes A (real,
               shift_im NULL) or the harmonic operator A + i diag(shift_im) (complex; the
               reference's build_lhs_harmonic -> shift_diagonal -> factorize, rk.cpp:32-39,
               sparse.cpp:157-171), the complex matrix never materialized.
   fnlh_richardson  smoothed_solve<S, Ilu<S>> (sparse.hpp:295-331) on the prec's operator
               and factors: host rhs / x (BlockVec layout, complex interleaved), x0 = 0.
   *_bytes     device bytes held, for the reference's LHS accounting
               (detail::lhs_alloc_register / lhs_alloc_release, sparse.hpp:34-37).
   Handles are not shared between concurrent calls except the read-only fnlh_lhs, which
   any number of precs (host threads) may use at once. */
typedef struct fnlh_lhs fnlh_lhs;
typedef struct fnlh_prec fnlh_prec;
int fnlh_lhs_create(const fnlh_pattern* p, fnlh_lhs** out);
int fnlh_lhs_upload(fnlh_lhs* A, const double* vals);
int fnlh_lhs_bytes(const fnlh_lhs* A, long long* bytes);
void fnlh_lhs_destroy(fnlh_lhs* A);
int fnlh_prec_create(const fnlh_lhs* A, int is_complex, fnlh_prec** out);
int fnlh_prec_factorize(fnlh_prec* f, const double* shift_im);
int fnlh_prec_bytes(const fnlh_prec* f, long long* bytes);
void fnlh_prec_destroy(fnlh_prec* f);
int fnlh_richardson(fnlh_prec* f, const double* rhs, double tol_rel, int max_iter, double* x, fnlh_linear_report* rep);

/* 2-colour fast path (rb.cuh): *n0 = size of colour 0 when the pattern is a colour-major
   2-colour ordering with one partition, else -1.  fnlh_set_red_black(0) forces the general
   level-scheduled kernels everywhere.  fnlh_set_rb_sweep selects the 2-colour sweep:
     0 (default) iterates bitwise those of smoothed_solve (sparse.hpp:295-331): L_ik =
       A_ik inv(U_kk) rebuilt per block in the reference's operation order; the colour-1
       residual of sweep s is fused with the colour-1 forward substitution of sweep s+1
       (2 kernels per sweep);
     1 the same arithmetic as three kernels per sweep (K_F, K_B, K_R);
     2 one pass over A per sweep, L_ik r_k applied as A_ik (U_kk^{-1} r_k): the same
       preconditioner, iterates equal to rounding, not bitwise;
     3 mode 0's arithmetic (bitwise) with edge-parallel kernels: one thread per (row,
       off-diagonal block) forms the block products, the row's sums are then taken in the
       reference's order from shared memory (at most 6 off-diagonal blocks per row);
     4 mode 0's kernels and arithmetic (bitwise, the same norms) with lane-warp CTAs for a
       batch of P > 1 systems sharing A: a CTA is one 32-row slice for up to 4 systems, one
       warp each, so the systems' loads of the shared A blocks meet in L1;
     5 lane-warp CTAs whose slice of A sits in shared memory for both passes of all their
       systems and whose inv(U_kk) columns stream through a per-thread cp.async ring one
       edge ahead (complex batches, P > 1; bitwise, the same norms);
     6 as 5 without the ring (inv(U_kk) through L1).
   Modes 3-6 are measured variants: every one is slower than mode 0. */
int fnlh_pattern_is_red_black(fnlh_pattern* p, int* n0);
/* compact factors of the 2-colour ILU(0): pivot LU + piv for every row, inv(U_kk) for colour 0 */
int fnlh_rb_factorize(fnlh_pattern* p, int is_complex, const double* A, const double* shift_im, double* diag_lu,
                      int* diag_piv, double* inv0);
void fnlh_set_red_black(int enable);
int fnlh_set_rb_sweep(int mode);

/* ---- L2/L3: the 3D edge-based discretization ---------------------------------
   Node-centred median-dual mesh (paper_2404_01407_b200/mesh.py builds one):
   faces a->b with area-weighted normals fn (outward on inlet/outlet faces), slip
   walls via the per-node closure source -p*closure_i.  b = 5 (Euler) or 6 (Euler +
   SA-like scalar).  Replaces Discretization (disc.hpp:42-106) for the BASELINE 3D
   configurations; on a line mesh it is the reference nozzle (disc_euler.cpp). */
typedef struct {
    int n, nf, b;
    const int *fa, *fb, *fbc, *ford;      /* nf each; fb = -1 and fbc in {0 inlet, 1 outlet} on boundary faces */
    const double *fn, *farea, *fnh;       /* 3*nf, nf, 3*nf */
    const double *fvis, *vol, *closure;   /* nf, n, 3*n */
    const double* mu;                     /* n (b = 6 eddy viscosity) */
    const int *nf_ptr, *nf_idx, *bflag;   /* node->face CSR ascending (mesh.cpp:44-59), n */
    double gamma, gas_constant, p0, T0, p_out, nt_in, forcing_scale;
} fnlh_mesh_desc;

int fnlh_disc_create(const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx, const int* partition,
                     fnlh_disc** out);
void fnlh_disc_destroy(fnlh_disc* d);
/* Discretization::residual (disc_euler.cpp:56-85): mode 0 Steady, 1 Perturbation (wref = reference) */
int fnlh_disc_residual(fnlh_disc* d, const double* W, const double* wref, int order, int mode, const double* forcing,
                       int nforcing, int need_vis, double* inv, double* vis);
/* Discretization::assemble_jacobian / assemble_diag_blocks (disc.cpp:25-130); J or P may be NULL */
int fnlh_disc_fd_jacobian(fnlh_disc* d, const double* W, double* J, double* P);
/* linearized_residual (residual_ops.cpp:63-102); complex arrays as (re,im) pairs */
int fnlh_disc_linearized_residual(fnlh_disc* d, const double* mean, const double* what, double omega,
                                  const double* forcing, int nforcing, int order, int need_vis, double* inv,
                                  double* vis);
/* deterministic_flux (residual_ops.cpp:113-161); amps nh*n*b complex */
int fnlh_disc_deterministic_flux(fnlh_disc* d, const double* mean, int nh, const double* omega, const double* amps,
                                 double* df);

/* ---- L4/L5: the outer FNLH iteration (driver.hpp:83-126) ------------------- */
typedef struct { /* SchemeConfig (driver.hpp:22-42) */
    int implicit;
    double sigma_cfl;
    double eps_relax;
    double linear_tol;
    int linear_max_iter;
    double target_drop_orders;
    int max_outer_iters;
    int workers; /* harmonics in flight (driver.cpp:246-265): on the 2-colour path min(workers,
                    N_h, 8) lanes, each with its own complex ILU workspace, share one read of A5
                    per batched sweep; > 1 also gives the reference's worker semantics (every
                    harmonic runs, successful ones commit, the first error by index rethrown) */
} fnlh_scheme;

typedef struct { /* ConvergenceEntry (driver.hpp:50-58); resid_h returned separately */
    int iter;
    double resid_mean;
    double rz;
    int has_rz;
    double seconds; /* cumulative device time */
} fnlh_entry;

int fnlh_solver_create(const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx, const int* partition,
                       const fnlh_scheme* s, int nh, const int* index, const double* omega, const double* forcing,
                       int nforcing, const double* mean0, fnlh_solver** out);
void fnlh_solver_destroy(fnlh_solver* s);
/* FAS multigrid, explicit scheme only (SchemeConfig::mg_levels, driver.hpp:24; the levels of
   build_hierarchy, multigrid.cpp:129-140, driver.cpp:104-131): append a coarse level below
   the current coarsest -- its mesh and block pattern, parent[i] = its node agglomerating node
   i of the current coarsest level, and its boundary forcing (nh x nforcing complex pairs).
   Every level then runs the V-cycle of multigrid.cpp:184-214 (coarse levels first order, DF
   on the finest level only).  ConfigError on an implicit solver. */
int fnlh_solver_add_level(fnlh_solver* s, const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx,
                          const int* parent, const double* forcing, int nforcing);
int fnlh_solver_levels(const fnlh_solver* s);
/* FnlhSolver::outer_iteration (driver.cpp:157-333) */
int fnlh_solver_outer_iteration(fnlh_solver* s, fnlh_entry* e, double* resid_h);
/* the same on host buffers: set_state(mean_in, amps_in) + outer_iteration + get_state into
   (mean_out, amps_out), with the transfers overlapped with the step (the harmonic fields
   go up while the Jacobian is assembled and come back while DF and the mean step run);
   in and out may alias; pinned host buffers give asynchronous copies */
int fnlh_solver_outer_iteration_host(fnlh_solver* s, const double* mean_in, const double* amps_in, double* mean_out,
                                     double* amps_out, fnlh_entry* e, double* resid_h);
/* outer_iteration in two halves, for harmonic sharding across GPUs (the
   reference's harmonic workers, driver.cpp:246-265, one rank per GPU):
   phase_harmonics: transform/FD Jacobian/A5/mean ILU, then the RK steps of the harmonics
     with owned[h] != 0 (owned NULL: all); h_norm[h] (nh doubles) receives their stage-1
     norms.  The caller then makes every harmonic field current on every rank (e.g. one
     broadcast per harmonic from its owner, fnlh_solver_copy_amps to stage it) and
   phase_mean: DF from all fields, the mean RK step and the monitor entry, given every
     harmonic's stage-1 norm and its linear reports (nrep[h] of them, concatenated in
     harmonic order).  fnlh_solver_outer_iteration == phase_harmonics(NULL) + phase_mean. */
int fnlh_solver_phase_harmonics(fnlh_solver* s, const int* owned, double* h_norm);
/* CUDA graphs (default on; FNLH_GRAPHS=0 in the environment turns them off at load): the
   launch sequences of the outer iteration without a host synchronization inside -- the
   five stages of each RK step on the 2-colour and explicit paths, and each harmonic
   batch's factorizations + stages -- are captured once per call site and replayed; the
   per-step synchronization that reads the error words stays outside, so results and
   error semantics are those of the launch-by-launch path.  0 disables (A/B, tests). */
void fnlh_set_graphs(int enable);
/* the harmonic whose error the last phase_harmonics returned (the first failing one by
   index, driver.cpp:262-264), or -1 when it succeeded or failed before the harmonics; lets
   a sharded caller rethrow the lowest failing harmonic's error on every rank */
int fnlh_solver_failed_harmonic(const fnlh_solver* s, int* h);
/* deterministic_flux split over its quadrature points (residual_ops.cpp:145-160), so ranks
   can share the nq residual evaluations and still sum them in the reference's k order:
     df_points       nq (4 l_max + 2, or 1 when every frequency is 0)
     df_terms        R(W(t_k)) for k in [k0, k1) into terms_dev ((k1-k0) * N*b doubles,
                     device), from the solver's current mean and harmonic fields
     df_accumulate   acc_dev += terms in order (first != 0: acc starts as terms[0], the
                     reference's sum from k = 0); chained over consecutive ranges it equals
                     the single-device sum bit for bit
     set_external_df the next phase_mean takes DF = acc/nq - R(mean) from acc_dev (N*b
                     doubles, device) instead of evaluating the quadrature itself
   Each call synchronizes before it returns (the caller's collectives see finished data). */
int fnlh_solver_df_points(fnlh_solver* s, int* nq);
int fnlh_solver_df_terms(fnlh_solver* s, int k0, int k1, void* terms_dev);
int fnlh_solver_df_accumulate(fnlh_solver* s, const void* terms_dev, int count, void* acc_dev, int first);
int fnlh_solver_set_external_df(fnlh_solver* s, const void* acc_dev);
/* linear reports of harmonic h from the last phase_harmonics (count in *n, at most max copied) */
int fnlh_solver_harmonic_reports(const fnlh_solver* s, int h, fnlh_linear_report* out, int max, int* n);
int fnlh_solver_phase_mean(fnlh_solver* s, const double* h_norm, const int* nrep, const fnlh_linear_report* reps,
                           fnlh_entry* e, double* resid_h);
/* copy harmonic h's field (N*b complex, device) to (to_dev = 1) or from (0) caller device memory */
int fnlh_solver_copy_amps(fnlh_solver* s, int h, void* dev, int to_dev);
/* FnlhSolver::run_to_convergence (driver.cpp:335-379): *reason 0 target-drop, 1 cap, 2 divergence */
int fnlh_solver_run(fnlh_solver* s, int* reason, int* n_entries, fnlh_entry* entries, int max_entries);
int fnlh_solver_get_state(const fnlh_solver* s, double* mean, double* amps);
int fnlh_solver_set_state(fnlh_solver* s, const double* mean, const double* amps);
int fnlh_solver_get_df(const fnlh_solver* s, double* df);
int fnlh_solver_num_reports(const fnlh_solver* s);
int fnlh_solver_get_reports(const fnlh_solver* s, fnlh_linear_report* out);
/* LHS value bytes (A5 + real ILU + one complex ILU workspace): independent of nh */
double fnlh_solver_lhs_bytes(const fnlh_solver* s);
/* time `sweeps` Richardson sweeps (smoothed_solve, sparse.hpp:315-329) of harmonic h's system at
   the current mean; *ms = device time of the loop */
int fnlh_solver_time_sweeps(fnlh_solver* s, int h, int sweeps, double* ms);
/* the batched sweep of harmonics [0, P) (P <= lanes), device ms for the whole loop */
int fnlh_solver_time_sweeps_batch(fnlh_solver* s, int P, int sweeps, double* ms);
int fnlh_solver_lanes(const fnlh_solver* s);
/* [red_black (0/1), n0 (colour 0 rows), SELL doubles incl. padding, nnzb] */
int fnlh_solver_info(const fnlh_solver* s, double* out);
/* counters (7 doubles): [sweeps, block-row updates, last outer iteration device ms, and its
   split: J + A5 + mean ILU, harmonic RK steps (+ exchange), DF, mean RK step (ms)] */
int fnlh_solver_counters(const fnlh_solver* s, double* out);

/* ---- time-accurate reference solver (SPEC oracle_urans; declared by oracle.hpp:28-52,
   `unsteady_solve`, which the reference does not implement) -------------------------------
   Classical 4-stage explicit time-accurate integration of V dQ/dt = -R(W, t) at a global
   stable step (cfl * min_i V_i / sum_f lambda_f at the steady state, then shrunk so a period
   is a whole number of steps and of samples), from `steady` (N*b, primitive; NULL = the
   solver's current mean) under the periodic boundary forcing
   sum_l 2 Re(forcing_l e^{i omega_l t}) in perturbation mode referenced to `steady`
   (order 2, the FNLH residual itself), marched period by period until the period-to-period
   relative L2 change of the state is below periodic_tol (after at least min_periods), then
   one period sampled uniformly into samples (samples_per_period * N*b doubles; the count is
   raised to 4 l_max + 2 when smaller and returned in info[0]).
   info (5 doubles): [samples, steps per period, dt, periods marched, last relative change].
   NonConvergenceError when max_periods pass first (the last period is still sampled). */
int fnlh_solver_unsteady(fnlh_solver* s, const double* steady, int samples_per_period, double cfl,
                         double periodic_tol, int max_periods, int min_periods, double* samples, double* info);

/* ---- device mesh preprocessing (csrc/meshgen.cu) ----------------
   Median-dual geometry of a structured ci x cj x ck sector (hex cells, or each hex split
   into 6 Kuhn tets), periodic in j or not.  Xu: unwrapped node coordinates
   [(ci+1)(cj+1)(ck+1)][3], node (i, j, k) at ((i (cj+1) + j)(ck+1) + k); mesh nodes are
   (i, j mod nj, k) with nj = cj (periodic) or cj + 1.  Produces the unique edges (ea < eb,
   ascending), their summed dual-face normals en [ne][3] and the node volumes [n],
   bitwise equal to paper_2404_01407_b200/mesh.py::_sector_dual_host.  No reference
   counterpart: the reference's meshes are the quasi-1D nozzle's (mesh.cpp). */
int fnlh_sector_dual_create(int ci, int cj, int ck, int periodic_j, int tets, const double* Xu, long long* n_edges,
                            fnlh_sector_dual** out);
int fnlh_sector_dual_get(const fnlh_sector_dual* h, long long* ea, long long* eb, double* en, double* vol);
void fnlh_sector_dual_destroy(fnlh_sector_dual* h);
/* make_pattern (sparse.cpp:91-117) on the device: block-CSR pattern of `rows` rows from the
   diagonal and both directions of every edge (ea[k], eb[k]), columns sorted and unique per
   row.  row_ptr [rows+1], col_idx [capacity rows + 2 n_edges], diag_idx [rows]; *nnzb =
   entries written.  ShapeError on an endpoint outside [0, rows). */
int fnlh_make_pattern(int rows, long long n_edges, const int* ea, const int* eb, int* row_ptr, int* col_idx,
                      int* diag_idx, long long* nnzb);
/* Reverse Cuthill-McKee ordering of the graph of a CSR pattern (row_ptr [n+1], col_idx with
   the diagonal in every row or in none), on the device: perm[position] = node.  Each
   component is seeded by the first unvisited node of `starts` (NULL: nodes by ascending
   degree, stable); with starts = np.argsort(degree) it equals
   scipy.sparse.csgraph.reverse_cuthill_mckee(graph, symmetric_mode=True) (the ordering step
   of the configurations' mesh generator).  Degrees must be <= 255. */
int fnlh_rcm(int n, const int* row_ptr, const int* col_idx, const int* starts, int* perm);
/* Greedy colouring of the graph of a CSR pattern (Jones-Plassmann rounds on the device):
   colour[i] in [0, *ncolours), no two neighbours share a colour, at most 64 colours.
   Deterministic for a given seed (node priorities from splitmix64(seed + i)); equal to
   mesh.py::greedy_colouring.  Meshes without a structural colouring get a colour-major
   ordering from it (each colour one ILU(0) level: the level-scheduled path's levels). */
int fnlh_greedy_colour(int n, const int* row_ptr, const int* col_idx, unsigned long long seed, int* colour,
                       int* ncolours);
/* Mesh::build_adjacency (mesh.cpp:44-59) and the derived arrays of mesh.py::from_faces on
   the device: per face (fa, fb = -1 on boundary faces, fn [nf][3]) the area, unit normal
   and viscous weight area / |x_fb - x_fa| (0 on boundary faces or without coords); per
   node its faces in ascending order (nf_ptr [n+1], nf_idx [capacity 2 nf]), the closure
   sum_f (+-fn_f) accumulated from 0.0 in face order, and the boundary flag. */
int fnlh_mesh_derive(int n, int nf, const int* fa, const int* fb, const double* fn, const double* coords,
                     double* farea, double* fnh, double* fvis, int* nf_ptr, int* nf_idx, double* closure, int* bflag);

/* ---- work-unit normalization (workunit.cpp:11-46 restated; host) ---------------------
   T_ref: best of 3 timings of the fixed 256 x 256, 60-sweep Jacobi stencil on one host
   core (measured once per process); WU = workers x seconds / T_ref. */
double fnlh_normalization_kernel_seconds(void);
double fnlh_work_units(int workers, double seconds, double t_ref);

#ifdef __cplusplus
}
#endif
#endif
