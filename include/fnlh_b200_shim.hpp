// fnlh_b200_shim.hpp -- the reference-side C++ binding of the C ABI:
// compiled into the reference next to its sparse.hpp, it adapts the reference's own types
// (BlockSparsityPattern, Bsr<S>, BlockVec<S>, LinearSolveReport; sparse.hpp:106-236,
// core.hpp:62-92) to include/fnlh_b200.h and rethrows the C ABI's status codes as the
// reference's exception types (core.hpp:22-56).  Header-only; link libfnlh_b200.so.
//
// Persistent handles (the drop-in at the call sites; device memory reported through the
// reference's own LHS accounting, detail::lhs_alloc_register/release, sparse.hpp:34-37):
//   driver.cpp:179-181  A5 = build_lhs_mean(J, ...)       -> LhsB200 a5(p, A5)  (or a5.upload(A5))
//   driver.cpp:213-216  build_lhs_harmonic(A5, mesh, omega, rk, 5, w.mat); w.ilu.factorize(w.mat)
//                                                        -> w.dev.factorize(harmonic_shift_b200(mesh, omega, rk, 5))
//   driver.cpp:180-181  ilu.factorize(A5) (mean)          -> mean_dev.factorize()
//   rk.cpp:82-85        smoothed_solve(*s.lhs, rhs, *s.ilu, tol, max_iter, x)
//                                                        -> smoothed_solve_b200(w.dev, rhs, tol, max_iter, x)
// so a stage solve moves only rhs and x; the worker's factors stay resident on the device.
//
// One-shot forms (upload + factorize + solve per call, for validation and small cases):
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
#include "mesh.hpp"
#include "rk.hpp"
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

// ---- persistent handles ------------------------------------------------------------

// the shared real LHS resident on the device (the Bsr<real> A5 of driver.cpp:67,179-181)
class LhsB200 {
public:
    LhsB200(const PatternB200& p, const Bsr<real>& A5) {
        rethrow_b200(fnlh_lhs_create(p.h, &h_));
        long long bytes = 0;
        rethrow_b200(fnlh_lhs_bytes(h_, &bytes));
        registered_ = static_cast<std::size_t>(bytes);
        detail::lhs_alloc_register(registered_);
        upload(A5);
    }
    // new values on the same pattern (once per outer iteration)
    void upload(const Bsr<real>& A5) { rethrow_b200(fnlh_lhs_upload(h_, A5.vals.data())); }
    ~LhsB200() {
        detail::lhs_alloc_release(registered_);
        fnlh_lhs_destroy(h_);
    }
    LhsB200(const LhsB200&) = delete;
    LhsB200& operator=(const LhsB200&) = delete;
    fnlh_lhs* handle() const { return h_; }

private:
    fnlh_lhs* h_ = nullptr;
    std::size_t registered_ = 0;
};

// one worker's Ilu<S> (driver.cpp:117) on the device: Ilu<real> for the mean flow, Ilu<cplx>
// for a harmonic, whose operator is A5 + i diag(shift) (build_lhs_harmonic, never materialized)
template <class S>
class IluB200 {
public:
    explicit IluB200(const LhsB200& A) {
        rethrow_b200(fnlh_prec_create(A.handle(), std::is_same_v<S, cplx> ? 1 : 0, &h_));
        long long bytes = 0;
        rethrow_b200(fnlh_prec_bytes(h_, &bytes));
        registered_ = static_cast<std::size_t>(bytes);
        detail::lhs_alloc_register(registered_);
    }
    // Ilu<real>::factorize(A5)
    void factorize() {
        static_assert(!std::is_same_v<S, cplx>, "a harmonic workspace factorizes A5 + i diag(shift)");
        rethrow_b200(fnlh_prec_factorize(h_, nullptr));
    }
    // build_lhs_harmonic + Ilu<cplx>::factorize (driver.cpp:213-216)
    void factorize(std::span<const real> shift_im) {
        static_assert(std::is_same_v<S, cplx>, "the shifted operator is complex");
        rethrow_b200(fnlh_prec_factorize(h_, shift_im.data()));
    }
    ~IluB200() {
        detail::lhs_alloc_release(registered_);
        fnlh_prec_destroy(h_);
    }
    IluB200(const IluB200&) = delete;
    IluB200& operator=(const IluB200&) = delete;
    fnlh_prec* handle() const { return h_; }

private:
    fnlh_prec* h_ = nullptr;
    std::size_t registered_ = 0;
};

// the diagonal term of build_lhs_harmonic (rk.cpp:32-39): s_i = omega V_i / (Gamma alpha_k)
inline std::vector<real> harmonic_shift_b200(const Mesh& mesh, real omega, const RKConfig& config, int stage_k) {
    if (stage_k < 1 || stage_k > 5) throw ConfigError("stage index must be in 1..5");
    const real ga = config.gamma_factor() * config.alpha[stage_k - 1];
    std::vector<real> s(mesh.num_nodes());
    for (int i = 0; i < mesh.num_nodes(); ++i) s[i] = omega * mesh.volume[i] / ga;
    return s;
}

// the stage solve of rk_step (rk.cpp:82-85) on the worker's resident factors
template <class S>
inline LinearSolveReport smoothed_solve_b200(IluB200<S>& f, const BlockVec<S>& rhs, real tol_rel, int max_iter,
                                             BlockVec<S>& x) {
    x = BlockVec<S>(rhs.b, rhs.nodes());
    fnlh_linear_report r{};
    rethrow_b200(fnlh_richardson(f.handle(), reinterpret_cast<const double*>(rhs.v.data()), tol_rel, max_iter,
                                 reinterpret_cast<double*>(x.v.data()), &r));
    return report_b200(r);
}

}  // namespace fnlh
