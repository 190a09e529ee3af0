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
    FNLH_CUDA = 7           /* device / runtime failure */
};

typedef struct fnlh_pattern fnlh_pattern;
typedef struct fnlh_disc fnlh_disc;
typedef struct fnlh_solver fnlh_solver;

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

#ifdef __cplusplus
}
#endif
#endif
