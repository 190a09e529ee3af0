// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Thin extern "C" wrappers around the UNMODIFIED reference (/root/reference/proj/src),
// compiled together with the reference sources by oracle/Makefile into
// oracle/_ref/libfnlh_ref.so.  Nothing here re-implements reference arithmetic: every
// call forwards to the reference's own classes (Ilu, Bsr, smoothed_solve,
// build_lhs_mean, the nozzle Discretization, linearized_residual,
// deterministic_flux, FnlhSolver).  Used to pin the C restatement (fnlh_oracle.c)
// and, on the GPU box (the .so travels with the snapshot), to check the CUDA path
// directly against the reference.
#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "case.hpp"
#include "core.hpp"
#include "dense.hpp"
#include "disc.hpp"
#include "driver.hpp"
#include "mesh.hpp"
#include "residual_ops.hpp"
#include "rk.hpp"
#include "sparse.hpp"
#include "state.hpp"

using namespace fnlh;

namespace {

thread_local std::string g_msg;
thread_local int g_node = -1, g_stage = -1;

template <class F>
int guarded(F&& f) {
    g_node = -1;
    g_stage = -1;
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_msg = e.what();
        return 1;
    } catch (const StateError& e) {
        g_msg = e.what();
        return 2;
    } catch (const ShapeError& e) {
        g_msg = e.what();
        return 3;
    } catch (const UnsupportedCaseError& e) {
        g_msg = e.what();
        return 4;
    } catch (const FactorizationError& e) {
        g_msg = e.what();
        g_node = e.node;
        return 5;
    } catch (const DivergenceError& e) {
        g_msg = e.what();
        g_stage = e.stage;
        return 6;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 99;
    }
}

PatternPtr pattern_from_csr(int b, int rows, const int* row_ptr, const int* col_idx, const int* part) {
    auto p = std::make_shared<BlockSparsityPattern>();
    p->b = b;
    p->rows = rows;
    p->row_ptr.assign(row_ptr, row_ptr + rows + 1);
    p->col_idx.assign(col_idx, col_idx + row_ptr[rows]);
    p->diag_idx.assign(rows, -1);
    for (int i = 0; i < rows; ++i)
        for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
            if (col_idx[e] == i) p->diag_idx[i] = e;
    if (part)
        p->partition.assign(part, part + rows);
    else
        p->partition.assign(rows, 0);
    p->validate();
    return p;
}

template <class S>
Bsr<S> bsr_from(PatternPtr p, const S* vals) {
    Bsr<S> A(p);
    const std::size_t n = static_cast<std::size_t>(p->nnzb()) * p->b * p->b;
    std::copy(vals, vals + n, A.vals.data());
    return A;
}

template <class S>
BlockVec<S> vec_from(int b, int n, const S* v) {
    BlockVec<S> x(b, n);
    std::copy(v, v + static_cast<std::size_t>(b) * n, x.v.data());
    return x;
}

template <class S>
void ilu_export(const Ilu<S>& f, S* vals, S* diag_lu, int* diag_piv, S* diag_inv) {
    if (vals) std::copy(f.vals.data(), f.vals.data() + f.vals.size(), vals);
    if (diag_lu) std::copy(f.diag_lu.begin(), f.diag_lu.end(), diag_lu);
    if (diag_piv) std::copy(f.diag_piv.begin(), f.diag_piv.end(), diag_piv);
    if (diag_inv) std::copy(f.diag_inv.begin(), f.diag_inv.end(), diag_inv);
}

struct Nozzle {
    CaseConfig cfg;
    Mesh mesh;
    std::unique_ptr<Discretization> disc;
    PatternPtr pattern;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }
int ref_last_error_node(void) { return g_node; }
int ref_last_error_stage(void) { return g_stage; }

// ---- generic sparse LA (sparse.hpp/.cpp) ----------------------------------

#define REF_LA(SUF, S)                                                                                    \
    int ref_ilu_factorize_##SUF(int b, int rows, const int* row_ptr, const int* col_idx, const int* part,  \
                                const S* A, S* vals, S* diag_lu, int* diag_piv, S* diag_inv) {            \
        return guarded([&] {                                                                              \
            auto p = pattern_from_csr(b, rows, row_ptr, col_idx, part);                                   \
            Bsr<S> M = bsr_from<S>(p, A);                                                                 \
            Ilu<S> f;                                                                                     \
            f.factorize(M);                                                                               \
            ilu_export(f, vals, diag_lu, diag_piv, diag_inv);                                             \
        });                                                                                               \
    }                                                                                                     \
    int ref_ilu_apply_##SUF(int b, int rows, const int* row_ptr, const int* col_idx, const int* part,      \
                            const S* A, const S* rhs, S* x) {                                             \
        return guarded([&] {                                                                              \
            auto p = pattern_from_csr(b, rows, row_ptr, col_idx, part);                                   \
            Bsr<S> M = bsr_from<S>(p, A);                                                                 \
            Ilu<S> f;                                                                                     \
            f.factorize(M);                                                                               \
            BlockVec<S> r = vec_from<S>(b, rows, rhs), y;                                                 \
            f.apply(r, y);                                                                                \
            std::copy(y.v.begin(), y.v.end(), x);                                                         \
        });                                                                                               \
    }                                                                                                     \
    int ref_matvec_##SUF(int b, int rows, const int* row_ptr, const int* col_idx, const S* A, const S* x, \
                         S* y) {                                                                          \
        return guarded([&] {                                                                              \
            auto p = pattern_from_csr(b, rows, row_ptr, col_idx, nullptr);                                \
            Bsr<S> M = bsr_from<S>(p, A);                                                                 \
            BlockVec<S> xv = vec_from<S>(b, rows, x), yv;                                                 \
            M.matvec(xv, yv);                                                                             \
            std::copy(yv.v.begin(), yv.v.end(), y);                                                       \
        });                                                                                               \
    }                                                                                                     \
    /* factorize once, then smoothed_solve; trace (max_iter*len, optional) gets every iterate */          \
    int ref_smoothed_solve_##SUF(int b, int rows, const int* row_ptr, const int* col_idx, const int* part, \
                                 const S* A, const S* rhs, double tol, int max_iter, S* x, int* iters,     \
                                 double* r0, double* r1, int* converged, S* trace) {                      \
        return guarded([&] {                                                                              \
            auto p = pattern_from_csr(b, rows, row_ptr, col_idx, part);                                   \
            Bsr<S> M = bsr_from<S>(p, A);                                                                 \
            Ilu<S> f;                                                                                     \
            f.factorize(M);                                                                               \
            BlockVec<S> r = vec_from<S>(b, rows, rhs), xv;                                                \
            std::vector<BlockVec<S>> tr;                                                                  \
            LinearSolveReport rep = smoothed_solve(M, r, f, tol, max_iter, xv, trace ? &tr : nullptr);    \
            std::copy(xv.v.begin(), xv.v.end(), x);                                                       \
            *iters = rep.iterations;                                                                      \
            *r0 = rep.initial_residual;                                                                   \
            *r1 = rep.final_residual;                                                                     \
            *converged = rep.converged ? 1 : 0;                                                           \
            if (trace)                                                                                    \
                for (std::size_t k = 0; k < tr.size(); ++k)                                               \
                    std::copy(tr[k].v.begin(), tr[k].v.end(), trace + k * xv.v.size());                   \
        });                                                                                               \
    }                                                                                                     \
    /* CPU baseline: factorize once, then time `sweeps` smoothed_solve iterations */                      \
    double ref_time_sweeps_##SUF(int b, int rows, const int* row_ptr, const int* col_idx, const S* A,     \
                                 const S* rhs, int sweeps, double* factor_seconds) {                      \
        double out = -1.0;                                                                                \
        guarded([&] {                                                                                     \
            auto p = pattern_from_csr(b, rows, row_ptr, col_idx, nullptr);                                \
            Bsr<S> M = bsr_from<S>(p, A);                                                                 \
            Ilu<S> f;                                                                                     \
            auto t0 = std::chrono::steady_clock::now();                                                   \
            f.factorize(M);                                                                               \
            auto t1 = std::chrono::steady_clock::now();                                                   \
            if (factor_seconds) *factor_seconds = std::chrono::duration<double>(t1 - t0).count();         \
            BlockVec<S> r = vec_from<S>(b, rows, rhs), xv;                                                \
            auto t2 = std::chrono::steady_clock::now();                                                   \
            smoothed_solve(M, r, f, 1e-300, sweeps, xv);                                                  \
            auto t3 = std::chrono::steady_clock::now();                                                   \
            out = std::chrono::duration<double>(t3 - t2).count();                                         \
        });                                                                                               \
        return out;                                                                                       \
    }

REF_LA(d, double)
REF_LA(z, std::complex<double>)

int ref_block_lu_factor_z(int b, std::complex<double>* A, int* piv, double* cond) {
    return guarded([&] { *cond = block_lu_factor(b, A, piv, 0); });
}
void ref_block_lu_solve_z(int b, const std::complex<double>* LU, const int* piv, const std::complex<double>* rhs,
                          std::complex<double>* x) {
    block_lu_solve(b, LU, piv, rhs, x);
}
void ref_cdiv(const std::complex<double>* a, const std::complex<double>* b, std::complex<double>* out, int n) {
    for (int k = 0; k < n; ++k) out[k] = a[k] / b[k];
}

// build_lhs_mean (rk.cpp:5-30) and shift_diagonal (sparse.cpp:157-171)
int ref_build_lhs_mean(int b, int rows, const int* row_ptr, const int* col_idx, const double* J, int implicit,
                       double sigma, double eps, int stage, double* A) {
    return guarded([&] {
        auto p = pattern_from_csr(b, rows, row_ptr, col_idx, nullptr);
        Bsr<real> Jm = bsr_from<real>(p, J);
        RKConfig rk;
        rk.mode = implicit ? RkMode::Implicit : RkMode::Explicit;
        rk.sigma_cfl = sigma;
        rk.eps_relax = eps;
        Bsr<real> out = build_lhs_mean(Jm, rk, stage);
        std::copy(out.vals.data(), out.vals.data() + out.vals.size(), A);
    });
}

// ---- full-size harmonic workers (bench.py --impl reference) ----------------------
// The objects one reference harmonic worker holds (driver.cpp:117, 213-216): the shared
// real LHS A5 on its pattern, the worker's complex workspace filled by shift_diagonal
// (sparse.cpp:157-171, as build_lhs_harmonic does, rk.cpp:32-39), its Ilu<cplx>
// (sparse.cpp:187-257), and smoothed_solve (sparse.hpp:295-331) on them.  Several
// workers may run concurrently from host threads (distinct workers, shared read-only A5).
struct RefLhs {
    PatternPtr p;
    Bsr<real> A5;
};
struct RefWorker {
    const RefLhs* lhs;
    Bsr<cplx> M;
    Ilu<cplx> f;
    BlockVec<cplx> rhs, x;
};

void* ref_lhs_create(int b, int rows, const int* row_ptr, const int* col_idx, const double* A5) {
    RefLhs* out = nullptr;
    guarded([&] {
        auto h = std::make_unique<RefLhs>();
        h->p = pattern_from_csr(b, rows, row_ptr, col_idx, nullptr);
        h->A5 = bsr_from<real>(h->p, A5);
        out = h.release();
    });
    return out;
}
void ref_lhs_destroy(void* h) { delete static_cast<RefLhs*>(h); }

// shift_diagonal(A5, i shift) into the worker's workspace, then Ilu::factorize (timed)
void* ref_hworker_create(void* lhs, const double* shift_im, const std::complex<double>* rhs, double* factor_seconds) {
    RefWorker* out = nullptr;
    guarded([&] {
        auto w = std::make_unique<RefWorker>();
        w->lhs = static_cast<const RefLhs*>(lhs);
        const int n = w->lhs->A5.rows(), b = w->lhs->A5.b();
        std::vector<cplx> s(n);
        for (int i = 0; i < n; ++i) s[i] = cplx(0.0, shift_im[i]);
        shift_diagonal(w->lhs->A5, s, w->M);
        const auto t0 = std::chrono::steady_clock::now();
        w->f.factorize(w->M);
        const auto t1 = std::chrono::steady_clock::now();
        if (factor_seconds) *factor_seconds = std::chrono::duration<double>(t1 - t0).count();
        w->rhs = vec_from<cplx>(b, n, rhs);
        out = w.release();
    });
    return out;
}
void ref_hworker_destroy(void* h) { delete static_cast<RefWorker*>(h); }

// one smoothed_solve of `sweeps` iterations from x = 0 (tol 1e-300: every sweep runs)
int ref_hworker_sweeps(void* h, int sweeps, double* seconds, double* final_residual) {
    return guarded([&] {
        RefWorker* w = static_cast<RefWorker*>(h);
        const auto t0 = std::chrono::steady_clock::now();
        const LinearSolveReport rep = smoothed_solve(w->M, w->rhs, w->f, 1e-300, sweeps, w->x);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (final_residual) *final_residual = rep.final_residual;
    });
}

// ---- pattern / adjacency builders (sparse.cpp:91-117, mesh.cpp:44-59) ----------

// make_pattern on an edge list; col_idx capacity rows + 2 ne; returns nnzb in *nnz
int ref_make_pattern(int b, int rows, long long ne, const int* ea, const int* eb, int* row_ptr, int* col_idx,
                     int* diag_idx, long long* nnz) {
    return guarded([&] {
        std::vector<std::pair<int, int>> edges(ne);
        for (long long k = 0; k < ne; ++k) edges[k] = {ea[k], eb[k]};
        PatternPtr p = make_pattern(b, rows, edges, {});
        std::copy(p->row_ptr.begin(), p->row_ptr.end(), row_ptr);
        std::copy(p->col_idx.begin(), p->col_idx.end(), col_idx);
        std::copy(p->diag_idx.begin(), p->diag_idx.end(), diag_idx);
        *nnz = static_cast<long long>(p->col_idx.size());
    });
}

// Mesh::build_adjacency on a face list (fb = -1: boundary face)
int ref_build_adjacency(int n, int nf, const int* fa, const int* fb, int* nf_ptr, int* nf_idx) {
    return guarded([&] {
        Mesh m;
        m.volume.assign(n, 1.0);
        m.faces.resize(nf);
        for (int f = 0; f < nf; ++f) {
            m.faces[f].a = fa[f];
            m.faces[f].b = fb[f];
            m.faces[f].boundary = fb[f] < 0 ? kBoundaryWest : kInterior;
        }
        m.build_adjacency();
        std::copy(m.node_face_ptr.begin(), m.node_face_ptr.end(), nf_ptr);
        std::copy(m.node_face_idx.begin(), m.node_face_idx.end(), nf_idx);
    });
}

// ---- nozzle case (the reference's own quasi-1D Euler discretization) ----------

void* ref_nozzle_create(const char* case_text) {
    Nozzle* z = nullptr;
    int st = guarded([&] {
        auto nz = std::make_unique<Nozzle>();
        nz->cfg = parse_case_text(case_text);
        nz->mesh = build_mesh(nz->cfg);
        nz->disc = make_discretization(nz->cfg, nz->mesh);
        nz->pattern = build_pattern(nz->mesh, nz->cfg.block_size());
        z = nz.release();
    });
    return st ? nullptr : z;
}

void ref_nozzle_destroy(void* h) { delete static_cast<Nozzle*>(h); }

// sizes: [n, nfaces, b, nnzb, n_harmonics]
void ref_nozzle_sizes(void* h, int* out) {
    auto* z = static_cast<Nozzle*>(h);
    out[0] = z->mesh.num_nodes();
    out[1] = static_cast<int>(z->mesh.faces.size());
    out[2] = z->cfg.block_size();
    out[3] = z->pattern->nnzb();
    out[4] = z->cfg.harmonics.count();
}

// faces (a, b, boundary, ordinal) + area; volumes; node->face CSR; pattern CSR
void ref_nozzle_mesh(void* h, int* fa, int* fb, int* fbc, int* ford, double* area, double* vol, int* nf_ptr,
                     int* nf_idx, int* row_ptr, int* col_idx) {
    auto* z = static_cast<Nozzle*>(h);
    const Mesh& m = z->mesh;
    for (std::size_t f = 0; f < m.faces.size(); ++f) {
        fa[f] = m.faces[f].a;
        fb[f] = m.faces[f].b;
        fbc[f] = m.faces[f].boundary;
        ford[f] = m.faces[f].boundary_ordinal;
        area[f] = m.faces[f].area;
    }
    std::copy(m.volume.begin(), m.volume.end(), vol);
    std::copy(m.node_face_ptr.begin(), m.node_face_ptr.end(), nf_ptr);
    std::copy(m.node_face_idx.begin(), m.node_face_idx.end(), nf_idx);
    std::copy(z->pattern->row_ptr.begin(), z->pattern->row_ptr.end(), row_ptr);
    std::copy(z->pattern->col_idx.begin(), z->pattern->col_idx.end(), col_idx);
}

// case scalars: [gamma, R, p0, T0, p_out, forcing_scale]
void ref_nozzle_case(void* h, double* out) {
    auto* z = static_cast<Nozzle*>(h);
    out[0] = z->cfg.gas.gamma;
    out[1] = z->cfg.gas.gas_constant;
    out[2] = z->cfg.inlet_total_pressure;
    out[3] = z->cfg.inlet_total_temperature;
    out[4] = z->cfg.outlet_static_pressure;
    out[5] = z->disc->forcing_scale();
}

int ref_nozzle_initial_mean(void* h, double* W) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        PrimitiveState w = nozzle_steady_reference(z->cfg);
        std::copy(w.v.begin(), w.v.end(), W);
    });
}

// harmonic list: omega, index and forcing (3 complex per harmonic)
void ref_nozzle_harmonics(void* h, double* omega, int* index, std::complex<double>* forcing) {
    auto* z = static_cast<Nozzle*>(h);
    for (int l = 0; l < z->cfg.harmonics.count(); ++l) {
        const Harmonic& hm = z->cfg.harmonics.harmonics[l];
        omega[l] = hm.omega;
        index[l] = hm.index;
        std::vector<cplx> f = z->disc->harmonic_forcing(hm);
        std::copy(f.begin(), f.end(), forcing + 3 * l);
    }
}

int ref_nozzle_residual(void* h, const double* W, const double* wref, int order, int mode, const double* forcing,
                        int nforcing, int need_vis, double* inv, double* vis) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        const int n = z->mesh.num_nodes(), b = 3;
        if (wref) z->disc->set_perturbation_reference(vec_from<real>(b, n, wref));
        BlockVec<real> iv, vv;
        z->disc->residual(vec_from<real>(b, n, W), order, mode ? BcMode::Perturbation : BcMode::Steady,
                          std::span<const real>(forcing, forcing ? nforcing : 0), need_vis != 0, iv, vv);
        std::copy(iv.v.begin(), iv.v.end(), inv);
        if (need_vis && vis) std::copy(vv.v.begin(), vv.v.end(), vis);
    });
}

int ref_nozzle_jacobian(void* h, const double* W, double* J) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        Bsr<real> Jm(z->pattern);
        z->disc->assemble_jacobian(vec_from<real>(3, z->mesh.num_nodes(), W), Jm);
        std::copy(Jm.vals.data(), Jm.vals.data() + Jm.vals.size(), J);
    });
}

int ref_nozzle_diag_blocks(void* h, const double* W, double* P) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        BlockDiag<real> D = z->disc->assemble_diag_blocks(vec_from<real>(3, z->mesh.num_nodes(), W));
        std::copy(D.blocks.begin(), D.blocks.end(), P);
    });
}

int ref_nozzle_linres(void* h, const double* mean, const std::complex<double>* what, double omega,
                      const std::complex<double>* forcing, int nforcing, int order, int need_vis,
                      std::complex<double>* inv, std::complex<double>* vis) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        const int n = z->mesh.num_nodes(), b = 3;
        PrimitiveState mv = vec_from<real>(b, n, mean);
        z->disc->set_perturbation_reference(mv);
        BlockDiag<real> M = transform_jacobian(mv, z->cfg.gas);
        BlockVec<cplx> iv, vv;
        linearized_residual(*z->disc, mv, M, vec_from<cplx>(b, n, what), omega,
                            std::span<const cplx>(forcing, nforcing), order, need_vis != 0, iv, vv);
        std::copy(iv.v.begin(), iv.v.end(), inv);
        if (need_vis && vis) std::copy(vv.v.begin(), vv.v.end(), vis);
    });
}

int ref_nozzle_df(void* h, const double* mean, int nh, const int* index, const double* omega,
                  const std::complex<double>* amps, double* df) {
    auto* z = static_cast<Nozzle*>(h);
    return guarded([&] {
        const int n = z->mesh.num_nodes(), b = 3;
        std::vector<HarmonicField> hs(nh);
        for (int l = 0; l < nh; ++l) {
            hs[l].index = index[l];
            hs[l].omega = omega[l];
            hs[l].amp = vec_from<cplx>(b, n, amps + static_cast<std::size_t>(l) * n * b);
        }
        BlockVec<real> d = deterministic_flux(*z->disc, vec_from<real>(b, n, mean), hs);
        std::copy(d.v.begin(), d.v.end(), df);
    });
}

// ---- full FnlhSolver (driver.hpp/.cpp) -------------------------------------

void* ref_solver_create(const char* case_text, int implicit, double sigma, double eps, double tol, int max_iter,
                        double drop_orders, int max_outer, int mg_levels) {
    FnlhSolver* s = nullptr;
    guarded([&] {
        SchemeConfig sc;
        sc.mode = implicit ? RkMode::Implicit : RkMode::Explicit;
        sc.sigma_cfl = sigma;
        sc.eps_relax = eps;
        sc.linear_tol = tol;
        sc.linear_max_iter = max_iter;
        sc.target_drop_orders = drop_orders;
        sc.max_outer_iters = max_outer;
        sc.mg_levels = mg_levels;
        s = new FnlhSolver(parse_case_text(case_text), sc);
    });
    return s;
}

void ref_solver_destroy(void* h) { delete static_cast<FnlhSolver*>(h); }

// entry: [iter, resid_mean, rz, has_rz] + resid_h[nh]
int ref_solver_outer(void* h, double* entry, double* resid_h) {
    auto* s = static_cast<FnlhSolver*>(h);
    return guarded([&] {
        ConvergenceEntry e = s->outer_iteration();
        entry[0] = e.iter;
        entry[1] = e.resid_mean;
        entry[2] = e.rz;
        entry[3] = e.has_rz ? 1.0 : 0.0;
        for (std::size_t k = 0; k < e.resid_h.size(); ++k) resid_h[k] = e.resid_h[k];
    });
}

void ref_solver_state(void* h, double* mean, std::complex<double>* amps) {
    auto* s = static_cast<FnlhSolver*>(h);
    std::copy(s->mean().v.begin(), s->mean().v.end(), mean);
    std::size_t off = 0;
    for (const HarmonicField& f : s->harmonics()) {
        std::copy(f.amp.v.begin(), f.amp.v.end(), amps + off);
        off += f.amp.v.size();
    }
}

void ref_solver_df(void* h, double* df) {
    auto* s = static_cast<FnlhSolver*>(h);
    std::copy(s->deterministic_flux_vector().v.begin(), s->deterministic_flux_vector().v.end(), df);
}

// run_to_convergence: returns reason (0 target-drop, 1 cap, 2 divergence) or -1 on an escaped error;
// hist rows of [iter, resid_mean, rz]; reports rows of [iterations, r0, r1, converged]
int ref_solver_run(void* h, int* n_hist, double* hist, int max_hist, int* n_rep, double* reps, int max_rep,
                   double* peak_lhs_bytes) {
    auto* s = static_cast<FnlhSolver*>(h);
    int reason = -1;
    int st = guarded([&] {
        lhs_alloc_reset();
        SolveOutcome out = s->run_to_convergence();
        reason = static_cast<int>(out.reason);
        *n_hist = static_cast<int>(out.history.size());
        for (int k = 0; k < *n_hist && k < max_hist; ++k) {
            hist[3 * k + 0] = out.history[k].iter;
            hist[3 * k + 1] = out.history[k].resid_mean;
            hist[3 * k + 2] = out.history[k].rz;
        }
        *n_rep = static_cast<int>(out.linear_reports.size());
        for (int k = 0; k < *n_rep && k < max_rep; ++k) {
            reps[4 * k + 0] = out.linear_reports[k].iterations;
            reps[4 * k + 1] = out.linear_reports[k].initial_residual;
            reps[4 * k + 2] = out.linear_reports[k].final_residual;
            reps[4 * k + 3] = out.linear_reports[k].converged ? 1.0 : 0.0;
        }
        *peak_lhs_bytes = static_cast<double>(out.peak_lhs_bytes);
    });
    return st ? -1 : reason;
}

}  // extern "C"
