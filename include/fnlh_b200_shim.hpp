// fnlh_b200_shim.hpp -- the reference-side C++ binding of the C ABI:
// compiled into the reference next to its sparse.hpp, it adapts the reference's own types
// (BlockSparsityPattern, Bsr<S>, BlockVec<S>, LinearSolveReport; sparse.hpp:106-236,
// core.hpp:62-92) to include/fnlh_b200.h and rethrows the C ABI's status codes as the
// reference's exception types (core.hpp:22-56).  Header-only; link libfnlh_b200.so.
//
// Replaces, at the call sites of FnlhSolver::outer_iteration (driver.cpp:179-181,215-216;
// rk.cpp:84-85):
//   smoothed_solve(A, rhs, ilu, tol, max_iter, x)    (sparse.hpp:295-331)
//     -> smoothed_solve_b200(pattern, A, tol, max_iter, rhs, x)            real systems
//     -> smoothed_solve_b200(pattern, A5, shift_im, tol, max_iter, rhs, x) harmonic systems:
//        the shared real A5 plus the per-node i omega V_i / (Gamma alpha_5) shift, the
//        complex workspace (build_lhs_harmonic + its Ilu) never materialized
//   Ilu<S>::factorize (sparse.cpp:187-257)           -> ilu_factorize_b200(...)
#pragma once

#include <complex>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "fnlh_b200.h"
#include "sparse.hpp"

namespace fnlh {

inline void rethrow_b200(int st) {
    if (st == FNLH_OK) return;
    const std::string msg = fnlh_last_error();
    switch (st) {
        case FNLH_CONFIG: throw ConfigError(msg);
        case FNLH_STATE: throw StateError(msg);
        case FNLH_SHAPE: throw ShapeError(msg);
        case FNLH_UNSUPPORTED: throw UnsupportedCaseError(msg);
        case FNLH_FACTORIZATION: throw FactorizationError(msg, fnlh_last_error_node());
        case FNLH_DIVERGENCE: throw DivergenceError(msg, fnlh_last_error_stage(), "linear");
        case FNLH_NONCONVERGENCE: throw NonConvergenceError(msg);
        default: throw std::runtime_error("fnlh_b200: " + msg);
    }
}

// one device pattern per reference PatternPtr (the reference shares one across J, A5 and
// every workspace, driver.cpp:67)
struct PatternB200 {
    fnlh_pattern* h = nullptr;
    explicit PatternB200(const BlockSparsityPattern& p) {
        rethrow_b200(fnlh_pattern_create(p.b, p.rows, p.row_ptr.data(), p.col_idx.data(),
                                         p.partition.empty() ? nullptr : p.partition.data(), &h));
    }
    ~PatternB200() { fnlh_pattern_destroy(h); }
    PatternB200(const PatternB200&) = delete;
    PatternB200& operator=(const PatternB200&) = delete;
};

inline LinearSolveReport report_b200(const fnlh_linear_report& r) {
    LinearSolveReport out;
    out.iterations = r.iterations;
    out.initial_residual = r.initial_residual;
    out.final_residual = r.final_residual;
    out.converged = r.converged != 0;
    return out;
}

// smoothed_solve with the reference's ILU(0) preconditioner on a real system
inline LinearSolveReport smoothed_solve_b200(const PatternB200& p, const Bsr<real>& A, real tol_rel, int max_iter,
                                             const BlockVec<real>& rhs, BlockVec<real>& x) {
    x = BlockVec<real>(rhs.b, rhs.nodes());
    fnlh_linear_report r{};
    rethrow_b200(fnlh_smoothed_solve(p.h, 0, A.vals.data(), 0, nullptr, rhs.v.data(), tol_rel, max_iter,
                                     x.v.data(), &r));
    return report_b200(r);
}

// the same on a harmonic system: A5 (real) + i * shift_im[i] on every diagonal entry
inline LinearSolveReport smoothed_solve_b200(const PatternB200& p, const Bsr<real>& A5,
                                             std::span<const real> shift_im, real tol_rel, int max_iter,
                                             const BlockVec<cplx>& rhs, BlockVec<cplx>& x) {
    if (static_cast<int>(shift_im.size()) != rhs.nodes()) throw ShapeError("smoothed_solve_b200: shift size");
    x = BlockVec<cplx>(rhs.b, rhs.nodes());
    fnlh_linear_report r{};
    rethrow_b200(fnlh_smoothed_solve(p.h, 1, A5.vals.data(), 0, shift_im.data(),
                                     reinterpret_cast<const double*>(rhs.v.data()), tol_rel, max_iter,
                                     reinterpret_cast<double*>(x.v.data()), &r));
    return report_b200(r);
}

// Ilu<S>::factorize on the device, factors returned in the reference's layout
// (vals nnzb*b*b, diag_lu rows*b*b, diag_piv rows*b, diag_inv rows*b*b)
template <class S>
inline void ilu_factorize_b200(const PatternB200& p, const Bsr<S>& A, S* vals, S* diag_lu, int* diag_piv,
                               S* diag_inv) {
    constexpr int cx = std::is_same_v<S, cplx> ? 1 : 0;
    rethrow_b200(fnlh_ilu_factorize(p.h, cx, reinterpret_cast<const double*>(A.vals.data()), cx, nullptr,
                                    reinterpret_cast<double*>(vals), reinterpret_cast<double*>(diag_lu), diag_piv,
                                    reinterpret_cast<double*>(diag_inv)));
}

}  // namespace fnlh
