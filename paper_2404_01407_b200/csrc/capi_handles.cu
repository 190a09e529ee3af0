// capi_handles.cu -- persistent operator handles of the C ABI (include/fnlh_b200.h,
// "persistent operator handles"): the shared real LHS resident in HBM (fnlh_lhs), one
// worker's ILU(0) workspace on it (fnlh_prec), and smoothed_solve on those factors
// (fnlh_richardson).  The structure of the reference's outer iteration: A5 once per outer
// iteration (driver.cpp:179-181), factorize once per harmonic (driver.cpp:213-216), solve
// once per RK stage (rk.cpp:82-85) -- each call moves only what the reference's call
// reads or writes.
#include <vector>

#include "fnlh_b200.h"
#include "capi_types.hpp"
#include "capi_util.hpp"

using namespace fnlh;

struct fnlh_lhs {
    const fnlh_pattern* pat = nullptr;
    bool rb = false;
    DeviceBuffer<double> bsr;      // reference BSR layout: upload target, factorization source (general path)
    DeviceBuffer<double> sell;     // general path: sliced matvec operand (sell_from_bsr)
    std::unique_ptr<RbSystem> rbs; // 2-colour path: SELL-32 copy, the only resident form
    std::size_t bytes() const { return rb ? rbs->bytes() : bsr.bytes() + sell.bytes(); }
};

struct fnlh_prec {
    const fnlh_lhs* A = nullptr;
    int cx = 0;
    std::unique_ptr<Workspace> ws;
    DeviceBuffer<double> shift;    // rows: the imaginary diagonal shift of the harmonic operator
    bool shifted = false;
    bool factored = false;
    std::unique_ptr<RbIlu<double>> rbd;
    std::unique_ptr<RbIlu<cplx>> rbz;
    std::unique_ptr<DeviceIlu<double>> gd;
    std::unique_ptr<DeviceIlu<cplx>> gz;
    DeviceBuffer<cplx> rhs, x, z, r;  // len complex (real systems use the first len doubles)
    DeviceBuffer<RbControl> ctl;
    DeviceBuffer<double> parts;       // this workspace's norm partials (precs on one lhs run concurrently)
    std::size_t bytes() const {
        return (rbd ? rbd->bytes() : 0) + (rbz ? rbz->bytes() : 0) + (gd ? gd->bytes() : 0) + (gz ? gz->bytes() : 0) +
               shift.bytes();
    }
};

namespace {

template <class S>
SystemView<S> general_view(const fnlh_prec* f) {
    SystemView<S> v;
    v.p = f->A->pat->p.get();
    v.real_vals = f->A->bsr.ptr;
    v.real_sell = f->A->sell.ptr;
    v.shift_im = f->shifted ? f->shift.ptr : nullptr;
    return v;
}

template <class S>
void factorize_prec(fnlh_prec* f) {
    if (f->A->rb) {
        RbIlu<S>& ilu = *([&]() -> RbIlu<S>* {
            if constexpr (sizeof(S) == sizeof(cplx)) return f->rbz.get(); else return f->rbd.get();
        }());
        rb_factorize<S>(*f->A->rbs, f->shifted ? f->shift.ptr : nullptr, ilu, *f->ws);
    } else {
        DeviceIlu<S>& ilu = *([&]() -> DeviceIlu<S>* {
            if constexpr (sizeof(S) == sizeof(cplx)) return f->gz.get(); else return f->gd.get();
        }());
        ilu_factorize<S>(general_view<S>(f), ilu, *f->ws);
    }
    FNLH_CUDA(cudaStreamSynchronize(f->ws->stream));
}

template <class S>
void richardson_prec(fnlh_prec* f, const double* rhs, double tol, int max_iter, double* x, fnlh_linear_report* rep) {
    const DevicePattern* dp = f->A->pat->p.get();
    const std::size_t len = (std::size_t)dp->rows * dp->b;
    cudaStream_t st = f->ws->stream;
    S* b = reinterpret_cast<S*>(f->rhs.ptr);
    S* xv = reinterpret_cast<S*>(f->x.ptr);
    FNLH_CUDA(cudaMemcpyAsync(b, rhs, len * sizeof(S), cudaMemcpyHostToDevice, st));
    LinearSolveReport out;
    if (f->A->rb) {
        const RbIlu<S>& ilu = *([&]() -> const RbIlu<S>* {
            if constexpr (sizeof(S) == sizeof(cplx)) return f->rbz.get(); else return f->rbd.get();
        }());
        const RbMember<S> m{&ilu, f->shifted ? f->shift.ptr : nullptr, b, xv, reinterpret_cast<S*>(f->z.ptr),
                            reinterpret_cast<S*>(f->r.ptr), f->ctl.ptr, f->parts.ptr};
        rb_smoothed_solve_batch<S>(*f->A->rbs, &m, 1, tol, max_iter, st);
        RbControl h;
        FNLH_CUDA(cudaMemcpyAsync(&h, f->ctl.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaMemcpyAsync(x, xv, len * sizeof(S), cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        if (h.status == 6) throw DivergenceError("non-finite iterate in smoothed_solve", h.iterations, "linear");
        out = LinearSolveReport{h.iterations, h.initial_residual, h.final_residual, h.converged != 0};
    } else {
        const DeviceIlu<S>& ilu = *([&]() -> const DeviceIlu<S>* {
            if constexpr (sizeof(S) == sizeof(cplx)) return f->gz.get(); else return f->gd.get();
        }());
        out = smoothed_solve<S>(general_view<S>(f), b, ilu, tol, max_iter, xv, *f->ws);
        FNLH_CUDA(cudaMemcpyAsync(x, xv, len * sizeof(S), cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
    }
    if (rep) *rep = fnlh_linear_report{out.iterations, out.initial_residual, out.final_residual, out.converged};
}

}  // namespace

extern "C" {

int fnlh_lhs_create(const fnlh_pattern* p, fnlh_lhs** out) {
    return guarded([&] {
        if (!p || !out) throw ConfigError("fnlh_lhs_create: null argument");
        auto h = std::make_unique<fnlh_lhs>();
        h->pat = p;
        h->rb = p->use_rb();
        const DevicePattern* dp = p->p.get();
        if (h->rb) {
            h->rbs = std::make_unique<RbSystem>(dp, p->n0);
        } else {
            h->bsr.alloc((std::size_t)dp->nnzb * dp->b * dp->b);
            h->sell.alloc(std::max<long long>(dp->msell_doubles, 1));
        }
        *out = h.release();
    });
}

int fnlh_lhs_upload(fnlh_lhs* A, const double* vals) {
    return guarded([&] {
        if (!A || !vals) throw ConfigError("fnlh_lhs_upload: null argument");
        const DevicePattern* dp = A->pat->p.get();
        const std::size_t n = (std::size_t)dp->nnzb * dp->b * dp->b;
        if (A->rb) {  // staged through a transient BSR buffer into the SELL-32 copy
            DeviceBuffer<double> tmp;
            tmp.upload(vals, n);
            A->rbs->load(tmp.ptr, nullptr);
            FNLH_CUDA(cudaStreamSynchronize(nullptr));
        } else {
            FNLH_CUDA(cudaMemcpy(A->bsr.ptr, vals, n * sizeof(double), cudaMemcpyHostToDevice));
            sell_from_bsr(*dp, A->bsr.ptr, A->sell.ptr, nullptr);
            FNLH_CUDA(cudaStreamSynchronize(nullptr));
        }
    });
}

int fnlh_lhs_bytes(const fnlh_lhs* A, long long* bytes) {
    return guarded([&] { *bytes = static_cast<long long>(A->bytes()); });
}

void fnlh_lhs_destroy(fnlh_lhs* A) { delete A; }

int fnlh_prec_create(const fnlh_lhs* A, int is_complex, fnlh_prec** out) {
    return guarded([&] {
        if (!A || !out) throw ConfigError("fnlh_prec_create: null argument");
        auto f = std::make_unique<fnlh_prec>();
        f->A = A;
        f->cx = is_complex ? 1 : 0;
        const DevicePattern* dp = A->pat->p.get();
        const std::size_t len = (std::size_t)dp->rows * dp->b;
        f->ws = std::make_unique<Workspace>(len);
        if (A->rb) {
            if (f->cx)
                f->rbz = std::make_unique<RbIlu<cplx>>(dp, A->pat->n0);
            else
                f->rbd = std::make_unique<RbIlu<double>>(dp, A->pat->n0);
        } else {
            if (f->cx)
                f->gz = std::make_unique<DeviceIlu<cplx>>(dp);
            else
                f->gd = std::make_unique<DeviceIlu<double>>(dp);
        }
        f->shift.alloc(dp->rows);
        f->rhs.alloc(len);
        f->x.alloc(len);
        f->z.alloc(len);
        f->r.alloc(len);
        f->ctl.alloc(1);
        if (A->rb) f->parts.alloc(A->rbs->partials_len());
        legacy_sync();
        *out = f.release();
    });
}

int fnlh_prec_factorize(fnlh_prec* f, const double* shift_im) {
    return guarded([&] {
        if (!f) throw ConfigError("fnlh_prec_factorize: null handle");
        if (shift_im && !f->cx) throw ConfigError("fnlh_prec_factorize: a shifted operator needs a complex workspace");
        f->factored = false;
        f->shifted = shift_im != nullptr;
        if (shift_im) {
            FNLH_CUDA(cudaMemcpyAsync(f->shift.ptr, shift_im, f->shift.bytes(), cudaMemcpyHostToDevice, f->ws->stream));
        }
        if (f->cx)
            factorize_prec<cplx>(f);
        else
            factorize_prec<double>(f);
        f->factored = true;
    });
}

int fnlh_prec_bytes(const fnlh_prec* f, long long* bytes) {
    return guarded([&] { *bytes = static_cast<long long>(f->bytes()); });
}

void fnlh_prec_destroy(fnlh_prec* f) { delete f; }

int fnlh_richardson(fnlh_prec* f, const double* rhs, double tol_rel, int max_iter, double* x, fnlh_linear_report* rep) {
    return guarded([&] {
        if (!f || !rhs || !x) throw ConfigError("fnlh_richardson: null argument");
        if (!f->factored) throw StateError("fnlh_richardson: the workspace holds no factorization");
        if (f->cx)
            richardson_prec<cplx>(f, rhs, tol_rel, max_iter, x, rep);
        else
            richardson_prec<double>(f, rhs, tol_rel, max_iter, x, rep);
    });
}

}  // extern "C"
