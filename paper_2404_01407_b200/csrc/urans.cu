// urans.cu -- the time-accurate reference solver of SPEC oracle_urans (`unsteady_solve`,
// declared by oracle.hpp:28-52 and never implemented by the reference): classical 4-stage
// explicit integration of V dQ/dt = -R(W, t) with the FNLH residual itself (order 2,
// perturbation-mode boundaries referenced to the steady state, disc_euler.cpp:195-230),
// so amplitude comparisons isolate the harmonic-method error (SPEC: "Oracle spatial
// discretization is IDENTICAL to the FNLH residual discretization").
#include <algorithm>
#include <cmath>

#include "solver.cuh"

namespace fnlh {

namespace {

constexpr int kT = 256;
constexpr int kMaxH = 64;
inline int nb(long long n) { return static_cast<int>((n + kT - 1) / kT); }

// sum over the node's faces of lambda_f = (|u_bar . n_hat| + c_bar) |n| (the dissipation
// coefficient of the face flux, disc_euler.cpp:128-132; arithmetic-mean primitives, the
// node's own state on a boundary face), divided by the node volume
template <int B>
__global__ void k_rate(MeshDev m, const double* __restrict__ W, double* __restrict__ rate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    const double* wi = W + (size_t)i * B;
    double s = 0.0;
    for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
        const int f = m.nf_idx[e];
        const int code = m.nf_code[e];
        const double* wj = code == kBoundaryFace ? wi : W + (size_t)(code >= 0 ? code : -code - 1) * B;
        const double rho = 0.5 * (wi[0] + wj[0]);
        const double u = 0.5 * (wi[1] + wj[1]), v = 0.5 * (wi[2] + wj[2]), w = 0.5 * (wi[3] + wj[3]);
        const double p = 0.5 * (wi[4] + wj[4]);
        const double* nh = m.fnh + 3 * (size_t)f;
        s += (fabs(u * nh[0] + v * nh[1] + w * nh[2]) + sqrt(m.gamma * p / rho)) * m.farea[f];
    }
    rate[i] = s / m.vol[i];
}

// boundary forcing at time t: F_k = sum_l 2 Re(f_lk e^{i omega_l t}) = sum_l (2cos) f.re - (2sin) f.im
struct Phase {
    double c[kMaxH], s[kMaxH];
};
__global__ void k_time_forcing(const cplx* __restrict__ f, int nh, int nf, Phase ph, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nf) return;
    double acc = 0.0;
    for (int l = 0; l < nh; ++l) {
        const cplx z = f[(size_t)l * nf + k];
        acc += ph.c[l] * z.re - ph.s[l] * z.im;
    }
    out[k] = acc;
}

// stage: R = inv (+ vis); acc (+)= wk R; x = a R / V  (a = -dt/2, -dt/2, -dt)
__global__ void k_stage(std::size_t len, int b, const double* __restrict__ vol, const double* __restrict__ inv,
                        const double* __restrict__ vis, double a, double wk, int first, double* __restrict__ acc,
                        double* __restrict__ x) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    const double r = vis ? inv[t] + vis[t] : inv[t];
    acc[t] = first ? wk * r : acc[t] + wk * r;
    if (x) x[t] = a * r / vol[t / b];
}
// final: x = a acc / V (a = -dt/6)
__global__ void k_final(std::size_t len, int b, const double* __restrict__ vol, const double* __restrict__ acc,
                        double a, double* __restrict__ x) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    x[t] = a * acc[t] / vol[t / b];
}
__global__ void k_diff(std::size_t len, const double* __restrict__ a, const double* __restrict__ b,
                       double* __restrict__ out) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t < len) out[t] = a[t] - b[t];
}

}  // namespace

void DeviceSolver::unsteady_solve(const double* steady_host, int samples_per_period, double cfl, double periodic_tol,
                                  int max_periods, int min_periods, double* samples_host, double* info) {
    if (!(cfl > 0.0) || !(periodic_tol > 0.0) || max_periods < 1 || min_periods < 1 || samples_per_period < 1)
        throw ConfigError("unsteady_solve: cfl, periodic_tol > 0; max_periods, min_periods, samples >= 1");
    if (nh_ > kMaxH) throw ConfigError("unsteady_solve: at most 64 harmonics");
    double base;
    int lmax;
    base_frequency(omega_, base, lmax);
    if (lmax == 0) throw ConfigError("unsteady_solve: needs time-periodic forcing (a positive frequency)");
    cudaStream_t st = ws_->stream;
    DeviceDisc& d = *disc_;
    const MeshDev& m = d.view();
    const int n = d.n(), b = d.b();
    const std::size_t L = d.len();
    const double period = 2.0 * std::acos(-1.0) / base;
    const int S = std::max(samples_per_period, 4 * lmax + 2);

    DeviceBuffer<double> steady(L), w0(L), w(L), wst(L), prev(L), inv(L), vis(L), acc(L), x(L), forc(std::max(nforcing_, 1)),
        rate(n), parts(592), nrm(2);  // norm2_sq_on: >= 592 partials
    if (steady_host)
        FNLH_CUDA(cudaMemcpyAsync(steady.ptr, steady_host, L * sizeof(double), cudaMemcpyHostToDevice, st));
    else
        FNLH_CUDA(cudaMemcpyAsync(steady.ptr, mean_.ptr, L * sizeof(double), cudaMemcpyDeviceToDevice, st));
    d.validate(steady.ptr, st);

    // global stable step, then a whole number of samples and steps per period
    if (b == 5) {
        ::fnlh::note_launch();
        k_rate<5><<<nb(n), kT, 0, st>>>(m, steady.ptr, rate.ptr);
    } else if (b == 6) {
        ::fnlh::note_launch();
        k_rate<6><<<nb(n), kT, 0, st>>>(m, steady.ptr, rate.ptr);
    } else {
        throw ShapeError("unsteady_solve: block size 5 or 6");
    }
    std::vector<double> hr(n);
    FNLH_CUDA(cudaMemcpyAsync(hr.data(), rate.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    FNLH_CUDA(cudaStreamSynchronize(st));
    const double rmax = *std::max_element(hr.begin(), hr.end());
    if (!(rmax > 0.0) || !std::isfinite(rmax)) throw StateError("unsteady_solve: no finite spectral radius");
    const double dt_stable = cfl / rmax;
    const long long per = (long long)std::ceil(period / (S * dt_stable));
    const long long steps = (long long)S * std::max(1LL, per);
    const double dt = period / (double)steps;

    auto forcing_at = [&](double t) {
        Phase ph{};
        for (int l = 0; l < nh_; ++l) {
            ph.c[l] = 2.0 * std::cos(omega_[l] * t);
            ph.s[l] = 2.0 * std::sin(omega_[l] * t);
        }
        if (nforcing_) { ::fnlh::note_launch(); k_time_forcing<<<nb(nforcing_), kT, 0, st>>>(forcing_.ptr, nh_, nforcing_, ph, forc.ptr); }
    };
    const int order = 2;
    const bool need_vis = b == 6;
    auto R = [&](const double* W, double t) {
        forcing_at(t);
        d.residual(W, steady.ptr, order, 1, forc.ptr, nforcing_, need_vis, inv.ptr, vis.ptr, st);
    };
    const int g = nb((long long)L);
    // one classical RK4 step from w at time t (w0 = copy of the step's start state)
    auto step = [&](double t) {
        FNLH_CUDA(cudaMemcpyAsync(w0.ptr, w.ptr, L * sizeof(double), cudaMemcpyDeviceToDevice, st));
        const double a[3] = {-0.5 * dt, -0.5 * dt, -dt}, tc[4] = {t, t + 0.5 * dt, t + 0.5 * dt, t + dt};
        const double wk[4] = {1.0, 2.0, 2.0, 1.0};
        const double* cur = w0.ptr;
        for (int k = 0; k < 4; ++k) {
            R(cur, tc[k]);
            { ::fnlh::note_launch(); k_stage<<<g, kT, 0, st>>>(L, b, d.view().vol, inv.ptr, need_vis ? vis.ptr : nullptr, k < 3 ? a[k] : 0.0,
                                                          wk[k], k == 0, acc.ptr, k < 3 ? x.ptr : nullptr); }
            if (k < 3) {
                apply_mean(b, n, m.gamma, w0.ptr, x.ptr, wst.ptr, d.err(), st);  // prim(cons(w0) + x)
                cur = wst.ptr;
            }
        }
        { ::fnlh::note_launch(); k_final<<<g, kT, 0, st>>>(L, b, d.view().vol, acc.ptr, -dt / 6.0, x.ptr); }
        apply_mean(b, n, m.gamma, w0.ptr, x.ptr, w.ptr, d.err(), st);
    };
    auto rel_change = [&]() {
        { ::fnlh::note_launch(); k_diff<<<g, kT, 0, st>>>(L, w.ptr, prev.ptr, x.ptr); }
        norm2_sq_on<double>(x.ptr, L, nrm.ptr, parts.ptr, st);
        norm2_sq_on<double>(w.ptr, L, nrm.ptr + 1, parts.ptr, st);
        double h[2];
        FNLH_CUDA(cudaMemcpyAsync(h, nrm.ptr, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        return std::sqrt(h[0]) / std::sqrt(h[1]);
    };

    d.reset_err(st);
    FNLH_CUDA(cudaMemcpyAsync(w.ptr, steady.ptr, L * sizeof(double), cudaMemcpyDeviceToDevice, st));
    double t = 0.0, change = 1.0;
    int periods = 0;
    bool periodic = false;
    while (periods < max_periods) {
        FNLH_CUDA(cudaMemcpyAsync(prev.ptr, w.ptr, L * sizeof(double), cudaMemcpyDeviceToDevice, st));
        for (long long s = 0; s < steps; ++s) {
            step(t);
            t = period * periods + dt * (double)(s + 1);
        }
        ++periods;
        t = period * periods;
        d.raise_if_err(st, "unsteady_solve");
        change = rel_change();
        if (!std::isfinite(change)) throw DivergenceError("unsteady_solve: non-finite state", periods, "urans");
        if (periods >= min_periods && change < periodic_tol) {
            periodic = true;
            break;
        }
    }
    // one more period sampled uniformly: t_k = k T / S from the period start
    const long long every = steps / S;
    for (long long s = 0; s < steps; ++s) {
        if (s % every == 0)
            FNLH_CUDA(cudaMemcpyAsync(samples_host + (std::size_t)(s / every) * L, w.ptr, L * sizeof(double),
                                      cudaMemcpyDeviceToHost, st));
        step(t);
        t = period * periods + dt * (double)(s + 1);
    }
    FNLH_CUDA(cudaStreamSynchronize(st));
    d.raise_if_err(st, "unsteady_solve");
    if (info) {
        info[0] = S;
        info[1] = (double)steps;
        info[2] = dt;
        info[3] = periods;
        info[4] = change;
    }
    if (!periodic)
        throw NonConvergenceError("unsteady_solve: no periodic state after " + std::to_string(max_periods) +
                                  " periods (relative change " + std::to_string(change) + ")");
}

}  // namespace fnlh
