// capi_la.cu -- extern "C" entry points for the L1 block-sparse LA (include/fnlh_b200.h).
#include <memory>
#include <string>
#include <vector>

#include "fnlh_b200.h"
#include "capi_util.hpp"
#include "la.cuh"
#include "rb.cuh"
#include "capi_types.hpp"

using namespace fnlh;


namespace {

template <class S>
struct HostSystem {
    DeviceBuffer<double> real_vals, sell;
    DeviceBuffer<S> vals;
    DeviceBuffer<double> shift;
    SystemView<S> view;
    HostSystem(const DevicePattern* p, const double* A, int A_complex, const double* shift_im) {
        const std::size_t n = (std::size_t)p->nnzb * p->b * p->b;
        view.p = p;
        if (A_complex) {
            vals.upload(reinterpret_cast<const S*>(A), n);
            view.vals = vals.ptr;
        } else {
            real_vals.upload(A, n);
            view.real_vals = real_vals.ptr;
            sell.alloc(std::max<long long>(p->msell_doubles, 1));  // the matvec operand, as the solver keeps A5
            sell_from_bsr(*p, real_vals.ptr, sell.ptr, nullptr);
            FNLH_CUDA(cudaDeviceSynchronize());
            view.real_sell = sell.ptr;
            if (shift_im) {
                shift.upload(shift_im, p->rows);
                view.shift_im = shift.ptr;
            }
        }
    }
};

template <class S>
int factorize_impl(const fnlh_pattern* p, const double* A, int A_complex, const double* shift_im, double* vals,
                   double* diag_lu, int* diag_piv, double* diag_inv) {
    const DevicePattern* dp = p->p.get();
    HostSystem<S> sys(dp, A, A_complex, shift_im);
    Workspace ws(1);
    DeviceIlu<S> f(dp);
    ilu_factorize(sys.view, f, ws);
    f.download(reinterpret_cast<S*>(vals), reinterpret_cast<S*>(diag_lu), diag_piv, reinterpret_cast<S*>(diag_inv));
    return 0;
}

template <class S>
int apply_impl(const fnlh_pattern* p, const double* A, int A_complex, const double* shift_im, const double* rhs,
               double* x) {
    const DevicePattern* dp = p->p.get();
    const std::size_t len = (std::size_t)dp->rows * dp->b;
    HostSystem<S> sys(dp, A, A_complex, shift_im);
    Workspace ws(len);
    DeviceIlu<S> f(dp);
    ilu_factorize(sys.view, f, ws);
    DeviceBuffer<S> r, z;
    r.upload(reinterpret_cast<const S*>(rhs), len);
    z.alloc(len);
    ilu_apply(f, r.ptr, z.ptr, ws);
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    download(reinterpret_cast<S*>(x), z.ptr, len);
    return 0;
}

template <class S>
int matvec_impl(const fnlh_pattern* p, const double* A, int A_complex, const double* shift_im, const double* x,
                double* y) {
    const DevicePattern* dp = p->p.get();
    const std::size_t len = (std::size_t)dp->rows * dp->b;
    HostSystem<S> sys(dp, A, A_complex, shift_im);
    Workspace ws(len);
    DeviceBuffer<S> xv, yv;
    xv.upload(reinterpret_cast<const S*>(x), len);
    yv.alloc(len);
    matvec(sys.view, xv.ptr, yv.ptr, ws);
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    download(reinterpret_cast<S*>(y), yv.ptr, len);
    return 0;
}

template <class S>
int solve_rb(const fnlh_pattern* p, const double* A, const double* shift_im, const double* rhs, double tol, int max_iter,
             double* x, fnlh_linear_report* rep) {
    const DevicePattern* dp = p->p.get();
    const std::size_t len = (std::size_t)dp->rows * dp->b;
    Workspace ws(len);
    DeviceBuffer<double> a, sh;
    a.upload(A, (std::size_t)dp->nnzb * dp->b * dp->b);
    if (shift_im) sh.upload(shift_im, dp->rows);
    RbSystem sys(dp, p->n0);
    sys.load(a.ptr, ws.stream);
    RbIlu<S> f(dp, p->n0);
    rb_factorize<S>(sys, shift_im ? sh.ptr : nullptr, f, ws);
    DeviceBuffer<S> b, xv, z, r;
    DeviceBuffer<RbControl> ctl(1);
    b.upload(reinterpret_cast<const S*>(rhs), len);
    xv.alloc(len);
    z.alloc(len);
    r.alloc(len);
    rb_smoothed_solve<S>(sys, shift_im ? sh.ptr : nullptr, f, b.ptr, tol, max_iter, xv.ptr, z.ptr, r.ptr, ctl.ptr, ws);
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    RbControl h;
    download(&h, ctl.ptr, 1);
    download(reinterpret_cast<S*>(x), xv.ptr, len);
    if (h.status == 6) throw DivergenceError("non-finite iterate in smoothed_solve", h.iterations, "linear");
    if (rep) *rep = fnlh_linear_report{h.iterations, h.initial_residual, h.final_residual, h.converged};
    return 0;
}

template <class S>
int rb_factor_impl(fnlh_pattern* p, const double* A, const double* shift_im, double* diag_lu, int* diag_piv,
                   double* inv0) {
    const DevicePattern* dp = p->p.get();
    Workspace ws(1);
    DeviceBuffer<double> a, sh;
    a.upload(A, (std::size_t)dp->nnzb * dp->b * dp->b);
    if (shift_im) sh.upload(shift_im, dp->rows);
    RbSystem sys(dp, p->n0);
    sys.load(a.ptr, ws.stream);
    RbIlu<S> f(dp, p->n0);
    rb_factorize<S>(sys, shift_im ? sh.ptr : nullptr, f, ws);
    const int b = dp->b, bb = b * b;
    if (diag_lu) {  // packed [slice][k][lane] -> row-major rows*b*b
        std::vector<S> pk(f.packed_rows() * bb);
        download(pk.data(), f.diag_lu, pk.size());
        S* out = reinterpret_cast<S*>(diag_lu);
        for (int i = 0; i < dp->rows; ++i)
            for (int k = 0; k < bb; ++k) out[(std::size_t)i * bb + k] = pk[f.packed_base(i, bb) + 32 * k];
    }
    if (diag_piv) {
        std::vector<int> pk(f.packed_rows() * b);
        download(pk.data(), f.diag_piv, pk.size());
        for (int i = 0; i < dp->rows; ++i)
            for (int k = 0; k < b; ++k) diag_piv[(std::size_t)i * b + k] = pk[f.packed_base(i, b) + 32 * k];
    }
    if (inv0) {  // slice-major on the device (rb_uoff); the C ABI returns row-major blocks per node
        std::vector<S> dv((std::size_t)32 * ((p->n0 + 31) / 32) * bb);
        download(dv.data(), f.inv0, dv.size());
        S* out = reinterpret_cast<S*>(inv0);
        for (int k = 0; k < p->n0; ++k)
            for (int m = 0; m < b; ++m)
                for (int c = 0; c < b; ++c) out[(std::size_t)k * bb + m * b + c] = dv[rb_uoff(b, k, m, c)];
    }
    return 0;
}

template <class S>
int solve_impl(const fnlh_pattern* p, const double* A, int A_complex, const double* shift_im, const double* rhs,
               double tol, int max_iter, double* x, fnlh_linear_report* rep) {
    const DevicePattern* dp = p->p.get();
    const std::size_t len = (std::size_t)dp->rows * dp->b;
    HostSystem<S> sys(dp, A, A_complex, shift_im);
    Workspace ws(len);
    DeviceIlu<S> f(dp);
    ilu_factorize(sys.view, f, ws);
    DeviceBuffer<S> b, xv;
    b.upload(reinterpret_cast<const S*>(rhs), len);
    xv.alloc(len);
    LinearSolveReport r = smoothed_solve(sys.view, b.ptr, f, tol, max_iter, xv.ptr, ws);
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    download(reinterpret_cast<S*>(x), xv.ptr, len);
    if (rep) *rep = fnlh_linear_report{r.iterations, r.initial_residual, r.final_residual, r.converged};
    return 0;
}

}  // namespace

extern "C" {

int fnlh_pattern_create(int b, int rows, const int* row_ptr, const int* col_idx, const int* partition,
                        fnlh_pattern** out) {
    return guarded([&] {
        auto h = std::make_unique<fnlh_pattern>();
        h->p = std::make_unique<DevicePattern>(b, rows, row_ptr, col_idx, partition);
        h->rb = rb_eligible(*h->p, &h->n0) ? 1 : 0;
        *out = h.release();
    });
}

void fnlh_pattern_destroy(fnlh_pattern* p) { delete p; }

int fnlh_pattern_levels(const fnlh_pattern* p, int* fwd, int* bwd) {
    *fwd = p->p->fwd_levels();
    *bwd = p->p->bwd_levels();
    return 0;
}

int fnlh_ilu_factorize(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                       double* vals, double* diag_lu, int* diag_piv, double* diag_inv) {
    return guarded([&] {
        if (is_complex)
            factorize_impl<cplx>(p, A, A_complex, shift_im, vals, diag_lu, diag_piv, diag_inv);
        else
            factorize_impl<double>(p, A, 0, nullptr, vals, diag_lu, diag_piv, diag_inv);
    });
}

int fnlh_ilu_apply(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                   const double* rhs, double* x) {
    return guarded([&] {
        if (is_complex)
            apply_impl<cplx>(p, A, A_complex, shift_im, rhs, x);
        else
            apply_impl<double>(p, A, 0, nullptr, rhs, x);
    });
}

int fnlh_matvec(const fnlh_pattern* p, int is_complex, const double* A, int A_complex, const double* shift_im,
                const double* x, double* y) {
    return guarded([&] {
        if (is_complex)
            matvec_impl<cplx>(p, A, A_complex, shift_im, x, y);
        else
            matvec_impl<double>(p, A, 0, nullptr, x, y);
    });
}

int fnlh_smoothed_solve(const fnlh_pattern* p, int is_complex, const double* A, int A_complex,
                        const double* shift_im, const double* rhs, double tol_rel, int max_iter, double* x,
                        fnlh_linear_report* rep) {
    return guarded([&] {
        if (!A_complex && p->use_rb()) {  // the 2-colour fused path (rb.cuh)
            if (is_complex)
                solve_rb<cplx>(p, A, shift_im, rhs, tol_rel, max_iter, x, rep);
            else
                solve_rb<double>(p, A, nullptr, rhs, tol_rel, max_iter, x, rep);
            return;
        }
        if (is_complex)
            solve_impl<cplx>(p, A, A_complex, shift_im, rhs, tol_rel, max_iter, x, rep);
        else
            solve_impl<double>(p, A, 0, nullptr, rhs, tol_rel, max_iter, x, rep);
    });
}

int fnlh_pattern_is_red_black(fnlh_pattern* p, int* n0) {
    return guarded([&] {
        *n0 = -1;
        if (p->rb == 1) *n0 = p->n0;
    });
}

int fnlh_rb_factorize(fnlh_pattern* p, int is_complex, const double* A, const double* shift_im, double* diag_lu,
                      int* diag_piv, double* inv0) {
    return guarded([&] {
        if (p->rb != 1) throw ShapeError("pattern is not a 2-colour colour-major ordering with one partition");
        if (is_complex)
            rb_factor_impl<cplx>(p, A, shift_im, diag_lu, diag_piv, inv0);
        else
            rb_factor_impl<double>(p, A, nullptr, diag_lu, diag_piv, inv0);
    });
}

void fnlh_set_red_black(int enable) { fnlh::rb_enabled() = enable != 0; }

int fnlh_set_rb_sweep(int mode) {
    return guarded([&] {
        if (mode < 0 || mode > 6) throw ConfigError("fnlh_set_rb_sweep: mode must be 0..6");
        fnlh::rb_sweep_mode() = mode;
    });
}

}  // extern "C"
