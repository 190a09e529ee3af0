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

    // Sliced-ELL storage of the ILU factor values (DeviceIlu), so that the threads of a
    // level kernel (one row each) read their rows' blocks coalesced: the rows of one
    // forward level are cut into slices of 32 (rows of a level ordered by descending
    // lower-entry count, stable), and slot s (the s-th lower entry, ascending column)
    // element k of the row in lane l sits at lbase + (s*b*b + k)*32 with lbase = slice
    // offset + l.  Upper entries likewise over the backward levels, slots in descending
    // column order (the backward loop's order); diagonal entries and the pivot LUs /
    // pivots over backward-level slices too.  ent[e] = element-0 offset of CSR entry e
    // (element stride 32), used by the factorization; host unpacking uses h_ent / h_dpos.
    long long* ent = nullptr;
    long long* lbase = nullptr;
    long long* ubase = nullptr;
    int *lcolb = nullptr, *ucolb = nullptr, *nlow = nullptr, *nup = nullptr;
    int *lcols = nullptr, *ucols = nullptr;
    int* dpos = nullptr;  // slice*32 + lane of row i in the pivot (diag_lu / diag_piv) layout
    int *blk_e = nullptr, *blk_row = nullptr;  // per block position (sell_elems / b^2): CSR entry, row; -1 = padding
    long long sell_elems = 0;  // elements of DeviceIlu::vals
    int n_dslices = 0;         // slices of the pivot layout
    std::vector<long long> h_ent;
    std::vector<int> h_dpos;
    // Sliced-ELL copy of a real BSR on this pattern (the matvec operand A5, sell_from_bsr):
    // slices of 32 consecutive rows, slot s = the row's s-th entry, element pairs of a block
    // as 16-byte words, lane-minor: row i (lane l) slot s pair q at mbase[i] + (s*pairs + q)*64
    // (doubles), mbase = slice offset + 2l; columns at mcols[mcolb[i] + 32 s]
    long long* mbase = nullptr;
    int *mcolb = nullptr, *mcols = nullptr, *mblk_e = nullptr;
    long long msell_doubles = 0;
    // the factorization's (k, j) lookups, precomputed: for row i, lower entry ek and each
    // later entry ej, the sliced offset of U_kj = entry (col ek, col ej) or -1, at
    // kj[kjo[i] + ...] in loop order (the reference's find, sparse.cpp:42-48, done once)
    long long *kjo = nullptr, *kj = nullptr;

    DevicePattern(int b, int rows, const int* row_ptr, const int* col_idx, const int* partition);
    ~DevicePattern();
    DevicePattern(const DevicePattern&) = delete;
    DevicePattern& operator=(const DevicePattern&) = delete;
    int fwd_levels() const { return static_cast<int>(fwd_ptr.size()) - 1; }
    int bwd_levels() const { return static_cast<int>(bwd_ptr.size()) - 1; }
};

// Ilu<S> storage (sparse.hpp:180-205) in the pattern's sliced layout: vals (sell_elems),
// diag_lu / diag_piv over n_dslices*32 rows, diag_inv rows*b*b (row-major, gathered by the
// factorization only)
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
    // the reference layout (Ilu<S>: vals nnzb*b*b, diag_lu rows*b*b, diag_piv rows*b, diag_inv
    // rows*b*b); any pointer may be null
    void download(S* vals_out, S* diag_lu_out, int* diag_piv_out, S* diag_inv_out) const;
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
    const double* real_sell = nullptr;  // optional sliced copy of real_vals (sell_from_bsr): matvec operand
};

// real BSR (pattern layout) -> the pattern's sliced matvec layout (msell_doubles)
void sell_from_bsr(const DevicePattern& p, const double* bsr, double* sell, cudaStream_t st);

// Scratch for reductions and the Richardson loop, one per stream.
struct Workspace {
    cudaStream_t stream = nullptr;
    double* partials = nullptr;  // reduction partials
    double* scalars = nullptr;   // device scalars
    double* h_scalars = nullptr; // pinned mirror
    int* status = nullptr;       // device status words [code, node]
    int* h_status = nullptr;
    int* h_flags = nullptr;             // pinned: lanes' active flags after a sweep, two slots
    cudaEvent_t flag_ev[2] = {nullptr, nullptr};
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
// per-lane shifts and factors; device-side stopping rule per lane after each sweep (one host synchronization per solve)
template <class S>
void smoothed_solve_batch(const DevicePattern& p, const double* A_real, const LaneSystem<S>* sys, int P,
                          double tol_rel, int max_iter, LaneReport* reps, Workspace& ws,
                          const double* A_sell = nullptr);

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
