// disc.cuh -- the 3D edge-based discretization resident on the device: residual
// (disc_euler.cpp:56-85), FD Jacobian (disc.cpp:37-130), linearized residual
// (residual_ops.cpp:63-102), deterministic flux (residual_ops.cpp:113-161), and the
// RK stage / update kernels (rk.cpp:41-99, driver.cpp:32-46,274-280).
#pragma once

#include <complex>
#include <memory>
#include <vector>

#include "capi_util.hpp"
#include "euler.cuh"
#include "la.cuh"

namespace fnlh {

struct MeshArrays {  // host-side description (include/fnlh_b200.h fnlh_disc_create)
    int n = 0, nf = 0, b = 5;
    const int *fa, *fb, *fbc, *ford;
    const double *fn, *farea, *fnh, *fvis, *vol, *closure, *mu;
    const int *nf_ptr, *nf_idx, *bflag;
    double gamma, gas_constant, p0, T0, p_out, nt_in, forcing_scale;
};

// where fd_jacobian may write A5 = J/ga (+ J_ii inv_es/ga on the diagonal) directly
// (build_lhs_mean fused, rk.cpp:5-30): the BSR layout (sell_map null) or the 2-colour SELL
// copy (sell_map = per-CSR-entry element offsets); `bytes` of vals are zeroed first
struct A5Target {
    double* vals;
    const long long* sell_map;
    double ga, inv_es;
    std::size_t bytes;
};

class DeviceDisc {
public:
    DeviceDisc(const MeshArrays& m, const DevicePattern* pattern);
    ~DeviceDisc();
    DeviceDisc(const DeviceDisc&) = delete;
    DeviceDisc& operator=(const DeviceDisc&) = delete;
    int n() const { return view_.n; }
    int b() const { return view_.b; }
    int nf() const { return view_.nf; }
    const MeshDev& view() const { return view_; }
    const DevicePattern* pattern() const { return pat_; }
    std::size_t len() const { return (std::size_t)view_.n * view_.b; }

    // device error word: (key << 4) | code, ~0 when clean
    unsigned long long* err() const { return cur_err_ ? cur_err_ : err_.ptr; }
    // route error records of subsequent launches to another device word (nullptr: the default)
    void redirect_err(unsigned long long* p) { cur_err_ = p; }
    void reset_err(cudaStream_t st);
    // 0 or the reference status code of the first recorded error (synchronizes)
    int read_err(cudaStream_t st, long long* key = nullptr);
    void raise_if_err(cudaStream_t st, const char* what);

    // residual(W, order, mode, forcing, need_vis) -> inv, vis (async);
    // skip_if_zero: device scalar; when it holds 0.0 the evaluation is skipped (delta == 0)
    void residual(const double* W, const double* wref, int order, int mode, const double* forcing, int nforcing,
                  bool need_vis, double* inv, double* vis, cudaStream_t st, const double* skip_if_zero = nullptr);
    // J (pattern layout) and/or P (n*b*b); validates W and the diagonal blocks (throws)
    void fd_jacobian(const double* W, double* J, double* P, cudaStream_t st, const A5Target* a5 = nullptr);
    // transform_jacobian validation (state.cpp:82-94): throws StateError on an inadmissible mean
    void validate(const double* W, cudaStream_t st);
    // linearized_residual (mean is the perturbation reference); complex vectors as cplx
    void linearized_residual(const double* mean, const cplx* what, double omega, const cplx* forcing, int nforcing,
                             int order, bool need_vis, cplx* inv, cplx* vis, cudaStream_t st);
    // deterministic_flux; amps: nh device pointers; omega/index host.  deferred: enqueue
    // only (no host synchronization); errors stay in err() for the caller to read
    // side: extra streams; with scratch contexts 1.. they evaluate quadrature points concurrently
    void deterministic_flux(const double* mean, const std::vector<const cplx*>& amps,
                            const std::vector<double>& omega, double* df, cudaStream_t st, bool deferred = false,
                            const std::vector<cudaStream_t>& side = {});

    // deterministic_flux in pieces, for quadrature points split across ranks
    // (residual_ops.cpp:145-160): the number of points; the residuals R(W(t_k)) of points
    // [k0, k1) into terms (k1-k0 vectors); their in-order sum into acc (first: acc = terms[0],
    // the k = 0 start of the reference's sum); DF = acc / nq - R(mean) with the zero-amplitude
    // rule.  Chaining df_accumulate over consecutive ranges in k order reproduces
    // deterministic_flux bit for bit.  Errors throw (df_terms, df_finish synchronize).
    int df_points(const std::vector<double>& omega);
    void df_terms(const double* mean, const std::vector<const cplx*>& amps, const std::vector<double>& omega,
                  int k0, int k1, double* terms, cudaStream_t st);
    void df_accumulate(const double* terms, int count, double* acc, bool first, cudaStream_t st);
    void df_finish(const double* mean, const std::vector<const cplx*>& amps, const std::vector<double>& omega,
                   const double* acc, double* df, cudaStream_t st, bool deferred);

    const int* df_active() const { return df_flag_.ptr; }  // set by the last deterministic_flux
    // scratch contexts: the residual / linearized-residual temporaries of context k, so k
    // independent evaluations can run concurrently on k streams (harmonic lanes)
    void ensure_contexts(int k);
    void use_context(int k) { cur_ = k; }
    int contexts() const { return static_cast<int>(ctx_.size()); }
private:
    struct Scratch {
        DeviceBuffer<double> nu, lap, flux, vflux, scal, fwork, rec;
        DeviceBuffer<unsigned long long> umax;
        DeviceBuffer<double> real[6];  // linres / DF temporaries (len each)
    };
    std::vector<std::unique_ptr<Scratch>> ctx_;
    int cur_ = 0;
    Scratch& C() const { return *ctx_[cur_]; }
    void alloc_scratch(Scratch& c);
    MeshDev view_{};
    const DevicePattern* pat_;
    DeviceBuffer<int> fa_, fb_, fbc_, ford_, nf_ptr_, nf_idx_, nf_code_, bflag_, e_ab_, e_ba_;
    DeviceBuffer<double> fn_, farea_, fnh_, fvis_, vol_, closure_, mu_;
    DeviceBuffer<double> fgeo_;    // interior face records of the packed order-2 residual
    DeviceBuffer<double> powtab_;  // glibc's pow tables (libm_pow.cuh), empty: correctly rounded pow
    DeviceBuffer<double> qscale_;
    DeviceBuffer<unsigned long long> err_;
    unsigned long long* cur_err_ = nullptr;
    int nf_int_ = -1;              // boundary faces are the tail [nf_int_, nf) (else -1)
    int nbn_ = 0;                  // nodes with boundary faces
    DeviceBuffer<int> bnodes_;
    DeviceBuffer<double> fdpart_;  // FD Jacobian diagonal partial sums (split kernels)
    DeviceBuffer<double> fddiag_;  // J_ii when fd_jacobian writes A5
    DeviceBuffer<unsigned long long> umax_;  // FD Jacobian scales
    DeviceBuffer<int> df_flag_;   // any nonzero amplitude (residual_ops.cpp:133-141)
    DeviceBuffer<cplx> df_ph_;    // quadrature phases e^{i omega_h t_k}, cached per omega set
    std::vector<double> df_omega_;
    std::vector<cudaEvent_t> df_ev_;
    std::vector<double> h_nfpad_;
};

// HarmonicSpec::base_frequency / max_multiple (case.cpp:10-44): base = 0, lmax = 0 without
// positive frequencies; ConfigError when incommensurate
void base_frequency(const std::vector<double>& omega, double& base, int& lmax);

// --- RK stage / update kernels (rk.cpp:41-99) ---------------------------------
template <class S>
void stage_blend(double beta, const S* vis_fresh, S* vis_blend, std::size_t len, cudaStream_t st);
template <class S>
void stage_rhs(const S* inv, const S* vis_blend, S* rhs, std::size_t len, cudaStream_t st);
// rhs = -((inv + vis_blend) - f): the FAS-forced stage right-hand side (coarse levels)
template <class S>
void stage_rhs_forced(const S* inv, const S* vis_blend, const S* f, S* rhs, std::size_t len, cudaStream_t st);
template <class S>
void scale(S* x, double a, std::size_t len, cudaStream_t st);
template <class S>
void add_inplace(S* x, const S* y, std::size_t len, cudaStream_t st);
// harmonic update out = base + M(mean)^{-1} x (driver.cpp:32-46)
void apply_harmonic(int b, int n, double gamma, const double* mean, const cplx* base, const cplx* x, cplx* out,
                    cudaStream_t st);
// mean update out = prim(cons(base) + x) (driver.cpp:274-280); status -> err word (code 2)
void apply_mean(int b, int n, double gamma, const double* base, const double* x, double* out,
                unsigned long long* err, cudaStream_t st);
// all_finite (core.hpp:127-132) -> err word code 6 when a value is not finite
template <class S>
void check_finite(const S* x, std::size_t len, unsigned long long* err, cudaStream_t st);

}  // namespace fnlh
