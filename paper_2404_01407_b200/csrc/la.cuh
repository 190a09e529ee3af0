// la.cuh -- device block-sparse LA: pattern with ILU level schedules, ILU(0)
// factorization / substitution, shifted matvec-residual, deterministic norms,
// preconditioned Richardson (smoothed_solve).  Restates sparse.hpp/.cpp.
#pragma once

#include <vector>

#include "common.cuh"

namespace fnlh {

struct LinearSolveReport {  // sparse.hpp:231-236
    int iterations = 0;
    double initial_residual = 0.0;
    double final_residual = 0.0;
    int converged = 0;
};

// BlockSparsityPattern (sparse.hpp:106-121) resident in HBM, plus the ILU(0) level
// schedule of its ordering: fwd level of row i = 1 + max over same-partition k < i in
// row i; bwd level likewise over j > i.  Rows of one level are independent, so the
// device executes the reference's sequential natural-order loops level by level
// with identical per-row arithmetic.  A colour-major ordering has (#colours) levels.
struct DevicePattern {
    int b = 0, rows = 0, nnzb = 0;
    int *row_ptr = nullptr, *col_idx = nullptr, *diag_idx = nullptr, *part = nullptr;
    int* fwd_rows = nullptr;  // rows grouped by forward level, ascending within a level
    int* bwd_rows = nullptr;
    std::vector<int> fwd_ptr, bwd_ptr;  // host level offsets
    std::vector<int> h_row_ptr, h_col_idx, h_diag_idx, h_part;
    int max_deg = 0;
    bool single_partition = true;

    DevicePattern(int b, int rows, const int* row_ptr, const int* col_idx, const int* partition);
    ~DevicePattern();
    DevicePattern(const DevicePattern&) = delete;
    DevicePattern& operator=(const DevicePattern&) = delete;
    int fwd_levels() const { return static_cast<int>(fwd_ptr.size()) - 1; }
    int bwd_levels() const { return static_cast<int>(bwd_ptr.size()) - 1; }
};

// Ilu<S> storage (sparse.hpp:180-205): vals nnzb*b*b, diag_lu / diag_inv rows*b*b, piv rows*b
template <class S>
struct DeviceIlu {
    const DevicePattern* p = nullptr;
    S* vals = nullptr;
    S* diag_lu = nullptr;
    int* diag_piv = nullptr;
    S* diag_inv = nullptr;
    explicit DeviceIlu(const DevicePattern* pat);
    ~DeviceIlu();
    DeviceIlu(const DeviceIlu&) = delete;
    DeviceIlu& operator=(const DeviceIlu&) = delete;
    std::size_t bytes() const;
};

// A system matrix as the reference sees it: either a stored S-valued BSR, or a real
// BSR (the shared LHS A5) plus a per-node complex diagonal shift s_i*I
// (build_lhs_harmonic, rk.cpp:32-39) applied on the fly.
template <class S>
struct SystemView {
    const DevicePattern* p = nullptr;
    const double* real_vals = nullptr;  // used when vals == nullptr
    const S* vals = nullptr;
    const double* shift_im = nullptr;   // per node Im(s_i) (Re(s_i) = 0), complex systems only
};

// Scratch for reductions and the Richardson loop, one per stream.
struct Workspace {
    cudaStream_t stream = nullptr;
    double* partials = nullptr;  // reduction partials
    double* scalars = nullptr;   // device scalars
    double* h_scalars = nullptr; // pinned mirror
    int* status = nullptr;       // device status words [code, node]
    int* h_status = nullptr;
    void* vec[4] = {nullptr, nullptr, nullptr, nullptr};  // r, z, ax, spare (len * sizeof(cplx))
    std::size_t vec_len = 0;
    int n_partials = 0;
    explicit Workspace(std::size_t max_len);
    ~Workspace();
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
};

// one system of a batched level-scheduled solve (harmonic lanes on the general path)
constexpr int kMaxLanes = 8;
template <class S>
struct LaneSystem {
    const DeviceIlu<S>* f;
    const double* shift;  // Im of the per-node diagonal shift (complex systems), or nullptr
    const S* rhs;
    S* x;
    S* z;
    S* r;
};
struct LaneReport {
    LinearSolveReport rep;
    int diverged = 0;  // a non-finite residual norm (DivergenceError at rep.iterations)
};
// P smoothed_solves on systems sharing the real A (A_real, the pattern's BSR layout) with
// per-lane shifts and factors; host stopping rule per lane after each sweep
template <class S>
void smoothed_solve_batch(const DevicePattern& p, const double* A_real, const LaneSystem<S>* sys, int P,
                          double tol_rel, int max_iter, LaneReport* reps, Workspace& ws);

// status codes (mirror core.hpp:22-56)
enum Status : int { kOk = 0, kConfig = 1, kState = 2, kShape = 3, kUnsupported = 4, kFactorization = 5,
                    kDivergence = 6, kCuda = 7 };

// --- operations (all asynchronous on ws.stream unless they return host values) -------
template <class S>
void ilu_factorize(const SystemView<S>& A, DeviceIlu<S>& f, Workspace& ws);
// the same, enqueued only: status[1] receives the first near-singular pivot row (0x7fffffff when clean)
template <class S>
void ilu_factorize_async(const SystemView<S>& A, DeviceIlu<S>& f, int* status, cudaStream_t st);  // throws FactorizationError
template <class S>
void ilu_apply(const DeviceIlu<S>& f, const S* rhs, S* x, Workspace& ws, S* x_accum = nullptr);
template <class S>
void residual_norm(const SystemView<S>& A, const S* rhs, const S* x, S* r, double* d_norm2, Workspace& ws);
template <class S>
void matvec(const SystemView<S>& A, const S* x, S* y, Workspace& ws);
template <class S>
void norm2_sq(const S* x, std::size_t len, double* d_out, Workspace& ws);
// the same on a given stream with caller partials (>= 592 doubles)
template <class S>
void norm2_sq_on(const S* x, std::size_t len, double* d_out, double* partials, cudaStream_t st);
template <class S>
LinearSolveReport smoothed_solve(const SystemView<S>& A, const S* rhs, const DeviceIlu<S>& f, double tol_rel,
                                 int max_iter, S* x, Workspace& ws);
// explicit block-Jacobi: x = P^{-1} rhs per node (BlockDiagLU::solve, dense.hpp:170-175)
template <class S>
void block_diag_solve(int b, int n, const S* lu, const int* piv, const S* rhs, S* x, cudaStream_t st);
template <class S>
void block_diag_factor(int b, int n, S* blocks, int* piv, int* status, cudaStream_t st);

}  // namespace fnlh
