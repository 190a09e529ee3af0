/*
 * fnlh_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C CPU restatement of the FNLH implicit pseudo-time hot path of the
 * reference (/root/reference/proj/src, C++20).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Every function cites the reference file:line it restates.  Generic layers
 * (dense blocks, ILU(0), Richardson, RK(5,3), linearized residual, DF, outer
 * iteration) follow the reference operation by operation so that, compiled with
 * gcc -O2 -ffp-contract=off (no -march), they are bitwise identical to the
 * reference compiled the same way (pinned by tests/test_oracle_pin.py against
 * oracle/_ref/libfnlh_ref.so, which is the reference itself).
 *
 * The 3D edge-based Euler discretization (b = 5, or 6 with an SA-like scalar) has
 * no reference counterpart; it is the reference's quasi-1D JST nozzle
 * (disc_euler.cpp) restated on node-centred median-dual faces with face normals.
 * On a 1D line mesh with normals (A,0,0) it reduces to the reference nozzle
 * (pinned bitwise for first-order quantities, 1e-13 for order 2).
 */
#ifndef FNLH_ORACLE_H
#define FNLH_ORACLE_H

#include <complex.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double _Complex ocplx;

/* error codes mirror the reference exception taxonomy (core.hpp:22-56) */
enum {
    OR_OK = 0,
    OR_CONFIG = 1,
    OR_STATE = 2,
    OR_SHAPE = 3,
    OR_UNSUPPORTED = 4,
    OR_FACTORIZATION = 5,
    OR_DIVERGENCE = 6
};

typedef struct {
    int code;
    int node;
    int stage;
    char msg[256];
} or_error;

const or_error* or_last_error(void);
/* boundary-state pow: 0 glibc (the reference's libm, default), 1 correctly rounded (the device's) */
void or_set_pow_mode(int cr);
double or_cr_pow(double x, double y);

/* BlockSparsityPattern (sparse.hpp:106-121) */
typedef struct {
    int b, rows, nnzb;
    const int* row_ptr;   /* rows+1 */
    const int* col_idx;   /* nnzb, ascending per row, diagonal included */
    const int* diag_idx;  /* rows */
    const int* partition; /* rows */
} or_pattern;

/* Ilu<S> storage (sparse.hpp:180-205) */
typedef struct {
    double* vals;     /* nnzb*b*b */
    double* diag_lu;  /* rows*b*b */
    int* diag_piv;    /* rows*b */
    double* diag_inv; /* rows*b*b */
} or_ilu_d;

typedef struct {
    ocplx* vals;
    ocplx* diag_lu;
    int* diag_piv;
    ocplx* diag_inv;
} or_ilu_z;

typedef struct {
    int iterations;
    double initial_residual;
    double final_residual;
    int converged;
} or_linear_report;

/* ---- dense + sparse LA (dense.hpp, sparse.hpp/.cpp) ---- */
int or_block_lu_factor_d(int b, double* A, int* piv, int node, double* cond);
int or_block_lu_factor_z(int b, ocplx* A, int* piv, int node, double* cond);
void or_block_lu_solve_d(int b, const double* LU, const int* piv, const double* rhs, double* x);
void or_block_lu_solve_z(int b, const ocplx* LU, const int* piv, const ocplx* rhs, ocplx* x);

int or_ilu_factorize_d(const or_pattern* p, const double* A, or_ilu_d* f);
int or_ilu_factorize_z(const or_pattern* p, const ocplx* A, or_ilu_z* f);
void or_ilu_apply_d(const or_pattern* p, const or_ilu_d* f, const double* rhs, double* x);
void or_ilu_apply_z(const or_pattern* p, const or_ilu_z* f, const ocplx* rhs, ocplx* x);
void or_matvec_d(const or_pattern* p, const double* A, const double* x, double* y);
void or_matvec_z(const or_pattern* p, const ocplx* A, const ocplx* x, ocplx* y);
int or_smoothed_solve_d(const or_pattern* p, const double* A, const double* rhs, const or_ilu_d* f,
                        double tol_rel, int max_iter, double* x, or_linear_report* rep);
int or_smoothed_solve_z(const or_pattern* p, const ocplx* A, const ocplx* rhs, const or_ilu_z* f,
                        double tol_rel, int max_iter, ocplx* x, or_linear_report* rep);
/* build_lhs_mean (rk.cpp:5-30): mode 0 explicit, 1 implicit */
int or_build_lhs_mean(const or_pattern* p, const double* J, int implicit, double sigma_cfl,
                      double eps_relax, int stage_k, double* A);
/* shift_diagonal (sparse.cpp:157-171) */
void or_shift_diagonal(const or_pattern* p, const double* A, const ocplx* s, ocplx* out);

/* ---- 3D edge-based Euler discretization (restates disc_euler.cpp / disc.cpp) ---- */
typedef struct {
    int n, nf, b;              /* b = 5 (Euler) or 6 (Euler + SA-like scalar) */
    const int* fa;             /* nf: first node (interior node for boundary faces) */
    const int* fb;             /* nf: second node, -1 on a boundary face */
    const int* fbc;            /* nf: -1 interior, 0 inlet (west), 1 outlet (east) */
    const int* ford;           /* nf: global boundary ordinal (forcing slot) */
    const double* fn;          /* 3*nf area-weighted normal, a->b (outward on boundary) */
    const double* farea;       /* nf |n| */
    const double* fnh;         /* 3*nf unit normal */
    const double* fvis;        /* nf viscous geometric factor |n|/|x_b-x_a| (b=6) */
    const double* vol;         /* n */
    const double* closure;     /* 3*n: sum of incident outward normals (slip-wall closure) */
    const double* mu;          /* n: frozen eddy viscosity (b=6) */
    const int* nf_ptr;         /* n+1 node->face CSR (ascending face index) */
    const int* nf_idx;
    const int* bflag;          /* n: node carries an inlet/outlet face */
    double gamma, gas_constant;
    double p0, T0, p_out;      /* inlet total pressure/temperature, outlet static pressure */
    double nt_in;              /* inlet SA-like scalar (b=6) */
    double forcing_scale;      /* Discretization::forcing_scale */
} or_mesh;

int or_prim_to_cons(int b, int n, double gamma, const double* W, double* Q);
/* 1 when the interior faces are exactly (i, i+1), i = 0..n-2: the order-2 terms then use the
   reference's 1D stencil verbatim (disc_euler.cpp:113-119,145-157) */
int or_mesh_is_line(const or_mesh* m);
int or_cons_to_prim(int b, int n, double gamma, const double* Q, double* W);
int or_transform_jacobian(int b, int n, double gamma, const double* W, double* M);

/* residual (disc_euler.cpp:56-85); mode 0 Steady, 1 Perturbation (wref used) */
int or_residual(const or_mesh* m, const double* W, const double* wref, int order, int mode,
                const double* forcing, int nforcing, int need_vis, double* inv, double* vis);
/* fd_jacobian (disc.cpp:37-130): J (nnzb*b*b) and/or P (n*b*b), either may be NULL */
int or_fd_jacobian(const or_mesh* m, const or_pattern* p, const double* W, double* J, double* P);
/* linearized_residual (residual_ops.cpp:63-102) */
int or_linearized_residual(const or_mesh* m, const double* mean, const double* M,
                           const ocplx* what, double omega, const ocplx* forcing, int nforcing,
                           int order, int need_vis, ocplx* inv, ocplx* vis);
/* deterministic_flux (residual_ops.cpp:113-161); amps nh*n*b */
int or_deterministic_flux(const or_mesh* m, const double* mean, int nh, const int* index,
                          const double* omega, const ocplx* amps, double* df);

/* ---- outer FNLH iteration (driver.cpp:157-333) ---- */
typedef struct {
    int implicit;          /* 1 implicit (ILU-Richardson), 0 explicit single grid */
    double sigma_cfl;      /* <= 0: mode default (2 / 50) */
    double eps_relax;
    double linear_tol;
    int linear_max_iter;
    double target_drop_orders;
    int max_outer_iters;
} or_scheme;

typedef struct {
    int iter;
    double resid_mean;
    double rz;
    int has_rz;
    double stage1_norm_mean;
} or_entry;

typedef struct or_solver or_solver;

or_solver* or_solver_create(const or_mesh* m, const or_pattern* p, const or_scheme* s, int nh,
                            const int* index, const double* omega, const ocplx* forcing,
                            int nforcing, const double* mean0);
void or_solver_destroy(or_solver* s);
int or_solver_outer_iteration(or_solver* s, or_entry* e, double* resid_h);
int or_solver_phase_harmonics(or_solver* s, const int* owned, double* hnorm_out);
/* harmonic whose error the last phase_harmonics returned (-1: none / before the harmonics) */
int or_solver_failed_harmonic(const or_solver* s);
/* deterministic_flux split over quadrature points (the restatement of fnlh_solver_df_*) */
int or_solver_df_points(const or_solver* s);
int or_solver_df_terms(or_solver* s, int k0, int k1, double* terms);
void or_solver_df_accumulate(const or_solver* s, const double* terms, int count, double* acc, int first);
void or_solver_set_external_df(or_solver* s, const double* acc);
/* harmonic worker threads (SchemeConfig::workers, driver.cpp:246-265), process-wide */
void or_set_workers(int w);
/* append a coarse multigrid level (explicit scheme): parent maps the current coarsest
   level's nodes to this level's; forcing is nh * nforcing complex */
int or_solver_add_level(or_solver* s, const or_mesh* m, const or_pattern* p, const int* parent, const ocplx* forcing,
                        int nforcing);
int or_solver_harmonic_reports(const or_solver* s, int h, or_linear_report* out, int max);
int or_solver_phase_mean(or_solver* s, const double* hnorm, const int* nrep, const or_linear_report* reps,
                         or_entry* e, double* resid_h);
void or_solver_get_state(const or_solver* s, double* mean, ocplx* amps);
void or_solver_set_state(or_solver* s, const double* mean, const ocplx* amps);
int or_solver_num_reports(const or_solver* s);
void or_solver_get_reports(const or_solver* s, or_linear_report* out);
const double* or_solver_df(const or_solver* s);
/* run_to_convergence (driver.cpp:335-379): returns termination 0 target-drop, 1 cap, 2 divergence */
int or_solver_run(or_solver* s, int* n_entries, or_entry* entries, int max_entries);

#ifdef __cplusplus
}
#endif
#endif
