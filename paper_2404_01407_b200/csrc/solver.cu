// solver.cu -- host orchestration of the FNLH outer iteration on the device
// (driver.cpp:157-379, rk.cpp:41-99), calling the sm_100a kernels of la.cu / disc.cu.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <type_traits>

#include "solver.cuh"

namespace fnlh {

namespace {

constexpr double kAlpha[5] = {1.0 / 4.0, 1.0 / 6.0, 3.0 / 8.0, 1.0 / 2.0, 1.0};   // rk.hpp:27
constexpr double kBeta[5] = {1.0, 0.0, 14.0 / 25.0, 0.0, 11.0 / 25.0};           // rk.hpp:28
constexpr int kT = 128;
inline int nb(long long n) { return static_cast<int>((n + kT - 1) / kT); }

__global__ void k_shift(const double* __restrict__ vol, int n, double omega, double ga, double* __restrict__ s) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) s[i] = omega * vol[i] / ga;  // rk.cpp:37 shift = i omega V / ga
}

// shifted_blocks (driver.cpp:48-59): P + i omega V I (not divided by Gamma alpha)
__global__ void k_shifted_blocks(const double* __restrict__ P, const double* __restrict__ vol, int b, int n,
                                 double omega, cplx* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const cplx s = mk(0.0, omega * vol[i]);
    for (int k = 0; k < b * b; ++k) {
        cplx v = mk(P[(size_t)i * b * b + k], 0.0);
        if (k / b == k % b) v = v + s;
        out[(size_t)i * b * b + k] = v;
    }
}

// --- FAS multigrid transfers (multigrid.cpp:142-182), one thread per node -----------
__device__ __forceinline__ double div_real(double a, double v) { return a / v; }
__device__ __forceinline__ cplx div_real(cplx a, double v) { return mk(a.re / v, a.im / v); }

// restrict_state: volume-weighted mean over the children, summed in ascending fine order
template <class S>
__global__ void k_restrict_state(const int* __restrict__ cptr, const int* __restrict__ cidx,
                                 const double* __restrict__ vol, int b, int nc, const S* __restrict__ wf,
                                 S* __restrict__ wc) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nc) return;
    S acc[6];
    for (int m = 0; m < b; ++m) acc[m] = zero<S>();
    double v = 0.0;
    for (int q = cptr[p]; q < cptr[p + 1]; ++q) {
        const int i = cidx[q];
        const double vi = vol[i];
        v += vi;
        for (int m = 0; m < b; ++m) acc[m] += vi * wf[(std::size_t)i * b + m];
    }
    for (int m = 0; m < b; ++m) wc[(std::size_t)p * b + m] = div_real(acc[m], v);
}

// restrict_residual of (r_f - F_f) and fas_forcing: rstar (= R_c(w_c0) on entry) -= sum
template <class S>
__global__ void k_restrict_fas(const int* __restrict__ cptr, const int* __restrict__ cidx, int b, int nc,
                               const S* __restrict__ rf, const S* __restrict__ ff, S* __restrict__ rstar) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nc) return;
    S acc[6];
    for (int m = 0; m < b; ++m) acc[m] = zero<S>();
    for (int q = cptr[p]; q < cptr[p + 1]; ++q) {
        const std::size_t i = (std::size_t)cidx[q] * b;
        for (int m = 0; m < b; ++m) {
            S t = rf[i + m];
            if (ff) t -= ff[i + m];
            acc[m] += t;
        }
    }
    for (int m = 0; m < b; ++m) rstar[(std::size_t)p * b + m] -= acc[m];
}

// prolong_add of the coarse correction (injection): w_i += (w_c - w_c0)[parent_i]
template <class S>
__global__ void k_prolong(const int* __restrict__ parent, int b, int n, const S* __restrict__ wc,
                          const S* __restrict__ wc0, S* __restrict__ w) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t pc = (std::size_t)parent[i] * b;
    for (int m = 0; m < b; ++m) {
        const S dlt = wc[pc + m] - wc0[pc + m];
        w[(std::size_t)i * b + m] += dlt;
    }
}

}  // namespace

void harmonic_shift(const double* vol, int n, double omega, double ga, double* s, cudaStream_t st) {
    { ::fnlh::note_launch(); k_shift<<<nb(n), kT, 0, st>>>(vol, n, omega, ga, s); }
}

void shifted_blocks(const double* P, const double* vol, int b, int n, double omega, cplx* out, cudaStream_t st) {
    { ::fnlh::note_launch(); k_shifted_blocks<<<nb(n), kT, 0, st>>>(P, vol, b, n, omega, out); }
}

std::atomic<int>& graphs_enabled() {
    static std::atomic<int> on{[] {
        const char* e = std::getenv("FNLH_GRAPHS");
        return e ? std::atoi(e) : 1;
    }()};
    return on;
}

template <class F>
void DeviceSolver::captured(const std::string& key, F&& body) {
    cudaStream_t st = ws_->stream;
    GraphEntry& g = graphs_[key];
    if (!graphs_enabled() || g.failed || g.calls++ == 0) {
        body();
        return;
    }
    if (!g.exec) {
        const long long l0 = tl_launches;
        FNLH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        cudaGraph_t graph = nullptr;
        bool ok = true;
        try {
            body();
        } catch (...) {
            ok = false;
        }
        const cudaError_t e = cudaStreamEndCapture(st, &graph);
        if (!ok || e != cudaSuccess || !graph ||
            cudaGraphInstantiate(&g.exec, graph, cudaGraphInstantiateFlagAutoFreeOnLaunch) != cudaSuccess) {
            (void)cudaGetLastError();
            if (graph) cudaGraphDestroy(graph);
            g.exec = nullptr;
            g.failed = true;  // a host synchronization inside: launch by launch from now on
            launch_count().fetch_sub(tl_launches - l0);
            tl_launches = l0;
            body();
            return;
        }
        cudaGraphDestroy(graph);
        g.launches = tl_launches - l0;
        launch_count().fetch_sub(g.launches);  // counted when the graph runs
        tl_launches = l0;
    }
    FNLH_CUDA(cudaGraphLaunch(g.exec, st));
    launch_count().fetch_add(g.launches);
}

DeviceSolver::DeviceSolver(const MeshArrays& mesh, const int* row_ptr, const int* col_idx, const int* partition,
                           const SchemeConfig& scheme, int nh, const int* index, const double* omega,
                           const double* forcing_pairs, int nforcing, const double* mean0)
    : sch_(scheme), nh_(nh), nforcing_(nforcing) {
    if (sch_.max_outer_iters < 0) throw ConfigError("max_outer_iters must be >= 0");
    sigma_ = sch_.sigma_cfl > 0.0 ? sch_.sigma_cfl : (sch_.implicit ? 50.0 : 2.0);  // driver.hpp:33-41
    index_.assign(index, index + nh);
    omega_.assign(omega, omega + nh);
    for (double w : omega_)
        if (w < 0.0) throw ConfigError("harmonic frequency must be >= 0");
    pat_ = std::make_unique<DevicePattern>(mesh.b, mesh.n, row_ptr, col_idx, partition);
    disc_ = std::make_unique<DeviceDisc>(mesh, pat_.get());
    const std::size_t len = (std::size_t)mesh.n * mesh.b;
    ws_ = std::make_unique<Workspace>(len);
    mean_.upload(mean0, len);
    df_.alloc(len);
    FNLH_CUDA(cudaMemset(df_.ptr, 0, len * sizeof(double)));
    amps_.alloc(std::max<std::size_t>((std::size_t)nh * len, 1));
    FNLH_CUDA(cudaMemset(amps_.ptr, 0, amps_.bytes()));
    forcing_.alloc(std::max<std::size_t>((std::size_t)nh * nforcing, 1));
    if (nh * nforcing)
        FNLH_CUDA(cudaMemcpy(forcing_.ptr, forcing_pairs, (std::size_t)nh * nforcing * sizeof(cplx),
                             cudaMemcpyHostToDevice));
    legacy_sync();  // the memsets and uploads above complete before any work stream runs
    if (sch_.implicit) {

        int n0 = 0;
        if (rb_enabled() && rb_eligible(*pat_, &n0)) {
            rbA_ = std::make_unique<RbSystem>(pat_.get(), n0);
            rb_mean_ = std::make_unique<RbIlu<double>>(pat_.get(), n0);
            rb_h_ = std::make_unique<RbIlu<cplx>>(pat_.get(), n0);  // ONE workspace reused by every harmonic
            ctl_.alloc(5);
            rb_z_.alloc(len);
            rb_r_.alloc(len);
        } else {
            A5_.alloc((std::size_t)pat_->nnzb * mesh.b * mesh.b);  // BSR A5 (the 2-colour path keeps only its SELL copy)
            A5s_.alloc(std::max<long long>(pat_->msell_doubles, 1));  // sliced copy: the matvec operand (la.cuh)
            ilu_mean_ = std::make_unique<DeviceIlu<double>>(pat_.get());
            ilu_h_ = std::make_unique<DeviceIlu<cplx>>(pat_.get());  // ONE workspace reused by every harmonic
        }
        shift_.alloc(mesh.n);
    } else {
        P_.alloc((std::size_t)mesh.n * mesh.b * mesh.b);
        PLU_.alloc((std::size_t)mesh.n * mesh.b * mesh.b);
        Ppiv_.alloc(len);
        pclu_.alloc((std::size_t)mesh.n * mesh.b * mesh.b);
        pcpiv_.alloc(len);
    }
    for (auto& v : rk_) v.alloc(len);
    stage_err_.alloc(11);
    fac_status_.alloc(2);
    if (sch_.workers < 1) throw ConfigError("workers must be >= 1");
    const int P = std::min(std::min(sch_.workers, nh_), kMaxBatch);
    if (sch_.implicit && P >= 2) {  // harmonics in flight: one workspace per lane
        rb_h_.reset();
        ilu_h_.reset();
        for (int m = 0; m < P; ++m) {
            auto ln = std::make_unique<HarmonicLane>();
            if (rbA_) {
                ln->f = std::make_unique<RbIlu<cplx>>(pat_.get(), rbA_->n0());
                ln->parts.alloc(rbA_->partials_len());
            } else {
                ln->gf = std::make_unique<DeviceIlu<cplx>>(pat_.get());
            }
            ln->shift.alloc(mesh.n);
            for (auto& v : ln->v) v.alloc(len);
            ln->ctl.alloc(5);
            ln->err.alloc(10);
            ln->fac.alloc(2);
            ln->norm.alloc(1);
            ln->nparts.alloc(1024);
            FNLH_CUDA(cudaStreamCreateWithFlags(&ln->stream, cudaStreamNonBlocking));
            FNLH_CUDA(cudaEventCreateWithFlags(&ln->done, cudaEventDisableTiming));
            lanes_.push_back(std::move(ln));
        }
    }
    FNLH_CUDA(cudaEventCreate(&ev0_));
    FNLH_CUDA(cudaEventCreate(&ev1_));
    for (auto& e : evp_) FNLH_CUDA(cudaEventCreate(&e));
    FNLH_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    FNLH_CUDA(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming));
    FNLH_CUDA(cudaEventCreateWithFlags(&ev_h_, cudaEventDisableTiming));
    FNLH_CUDA(cudaEventCreateWithFlags(&ev_stage_, cudaEventDisableTiming));
    if (!lanes_.empty()) disc_->ensure_contexts(static_cast<int>(lanes_.size()));
}

DeviceSolver::~DeviceSolver() {
    for (auto& kv : graphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    cudaEventDestroy(ev0_);
    cudaEventDestroy(ev1_);
    for (auto& e : evp_) cudaEventDestroy(e);
    cudaEventDestroy(ev_in_);
    cudaEventDestroy(ev_h_);
    cudaEventDestroy(ev_stage_);
    cudaStreamDestroy(cs_);
}

std::size_t DeviceSolver::lhs_bytes() const {
    std::size_t s = 0;
    if (sch_.implicit && rbA_) {
        s = A5_.bytes() + rbA_->bytes() + rb_mean_->bytes();
        if (lanes_.empty())
            s += rb_h_->bytes();
        else
            for (const auto& ln : lanes_) s += ln->f->bytes();
    } else if (sch_.implicit) {
        s = A5_.bytes() + A5s_.bytes() + ilu_mean_->bytes();
        if (lanes_.empty())
            s += ilu_h_->bytes();
        else
            for (const auto& ln : lanes_) s += ln->gf->bytes();
    }
    else {
        s = P_.bytes() + PLU_.bytes() + pclu_.bytes();
        for (const auto& c : mg_) s += c->P.bytes() + c->PLU.bytes() + c->pclu.bytes();
    }
    return s;
}

void DeviceSolver::check_step(const unsigned long long* errs, const RbControl* ctls,
                              const LinearSolveReport* host_rep, const bool* have_host, const std::string& field,
                              RkStepResult& res, const int* host_div) {
    for (int k = 1; k <= 5; ++k) {
        const unsigned long long ee = errs[k - 1], ea = errs[5 + k - 1];
        if (ee != ~0ull) {
            const int code = (int)(ee & 15ull);
            if (code == 2) throw DivergenceError("residual evaluation failed: inadmissible boundary state", k, field);
            if (code == 4) throw UnsupportedCaseError("supersonic boundary state");
            throw std::runtime_error("device error during residual evaluation");
        }
        if (sch_.implicit) {
            LinearSolveReport rep;
            if (have_host && have_host[k - 1]) {
                rep = host_rep[k - 1];
                if (host_div && host_div[k - 1])
                    throw DivergenceError("non-finite iterate in smoothed_solve", rep.iterations, "linear");
            } else {
                const RbControl& c = ctls[k - 1];
                if (c.status == 6) throw DivergenceError("non-finite iterate in smoothed_solve", c.iterations, "linear");
                rep.iterations = c.iterations;
                rep.initial_residual = c.initial_residual;
                rep.final_residual = c.final_residual;
                rep.converged = c.converged;
            }
            sweeps += rep.iterations;
            row_updates += (long long)rep.iterations * disc_->n();
            res.linear_reports.push_back(rep);
        }
        if (ea != ~0ull) {
            if ((int)(ea & 15ull) == 2) throw DivergenceError("update left the admissible set", k, field);
            throw DivergenceError("non-finite stage state", k, field);
        }
    }
}

template <class S>
void DeviceSolver::rb_solve_async(const double* shift, const RbIlu<S>& f, const S* rhs, S* x, RbControl* ctl) {
    rb_smoothed_solve<S>(*rbA_, shift, f, rhs, sch_.linear_tol, sch_.linear_max_iter, x,
                         reinterpret_cast<S*>(rb_z_.ptr), reinterpret_cast<S*>(rb_r_.ptr), ctl, *ws_);
}

// rk_step (rk.cpp:41-99), enqueued without host round trips: residual-evaluation and
// update errors land in per-stage device words, the fused solver's reports in per-stage
// control blocks, the stage-1 norm on the device; one synchronization at the end turns
// them into the reference's exceptions in stage order.  `solve` returns the report when
// the solver is host-driven (general path) and false when it is deferred (ctl[k-1]).
template <class S, class Eval, class Apply, class Solve>
RkStepResult DeviceSolver::rk_step(S* state, Eval&& eval, Apply&& apply, Solve&& solve, const S* pdiag_lu,
                                   const int* pdiag_piv, const std::string& field, const int* fac_status,
                                   bool check_df, int level, const S* mg_forcing) {
    cudaStream_t st = ws_->stream;
    DeviceDisc* d = lv_disc(level);
    const std::size_t len = d->len();
    S* state0 = reinterpret_cast<S*>(rk_[0].ptr);
    S* inv = reinterpret_cast<S*>(rk_[1].ptr);
    S* vis_fresh = reinterpret_cast<S*>(rk_[2].ptr);
    S* vis_blend = reinterpret_cast<S*>(rk_[3].ptr);
    S* rhs = reinterpret_cast<S*>(rk_[4].ptr);
    S* x = reinterpret_cast<S*>(rk_[5].ptr);
    S* stage = reinterpret_cast<S*>(rk_[6].ptr);
    RkStepResult res;
    LinearSolveReport host_rep[5];
    bool have_host[5] = {false, false, false, false, false};
    const double gfac = sch_.implicit ? 1.0 / sch_.eps_relax : sigma_;  // rk.hpp:34
    auto stages = [&] {
    res = RkStepResult{};
    for (int k = 0; k < 5; ++k) have_host[k] = false;
    FNLH_CUDA(cudaMemcpyAsync(state0, state, len * sizeof(S), cudaMemcpyDeviceToDevice, st));
    FNLH_CUDA(cudaMemcpyAsync(stage, state, len * sizeof(S), cudaMemcpyDeviceToDevice, st));
    FNLH_CUDA(cudaMemsetAsync(vis_blend, 0, len * sizeof(S), st));
    FNLH_CUDA(cudaMemsetAsync(vis_fresh, 0, len * sizeof(S), st));
    FNLH_CUDA(cudaMemsetAsync(stage_err_.ptr, 0xff, 10 * sizeof(unsigned long long), st));
    for (int k = 1; k <= 5; ++k) {
        const double beta = kBeta[k - 1];
        const bool fresh = beta != 0.0;
        d->redirect_err(stage_err_.ptr + (k - 1));
        eval(stage, fresh, inv, vis_fresh);
        d->redirect_err(nullptr);
        if (fresh) {
            ++res.viscous_evaluations;
            stage_blend<S>(beta, vis_fresh, vis_blend, len, st);
        }
        if (mg_forcing)  // FAS forcing R* on coarse levels (multigrid.cpp:184-214)
            stage_rhs_forced<S>(inv, vis_blend, mg_forcing, rhs, len, st);
        else
            stage_rhs<S>(inv, vis_blend, rhs, len, st);
        if (k == 1) norm2_sq<S>(rhs, len, ws_->scalars + 8, *ws_);
        if (!sch_.implicit) {
            block_diag_solve<S>(d->b(), d->n(), pdiag_lu, pdiag_piv, rhs, x, st);
            scale<S>(x, gfac * kAlpha[k - 1], len, st);
        } else {
            scale<S>(rhs, kAlpha[k - 1], len, st);
            LinearSolveReport rep;
            if (solve(rhs, x, k, rep)) {
                host_rep[k - 1] = rep;
                have_host[k - 1] = true;
            }
        }
        d->redirect_err(stage_err_.ptr + 5 + (k - 1));
        apply(state0, x, stage);
        check_finite<S>(stage, len, d->err(), st);
        d->redirect_err(nullptr);
    }
    };
    // the general path's solves are host-driven (a synchronization per solve): no graph
    if ((sch_.implicit && rbA_) || !sch_.implicit)
        captured("rk:" + field + ":" + std::to_string(level) + ":" + std::to_string((std::uintptr_t)state) +
                     (mg_forcing ? ":fas" : "") + ":" + std::to_string(rb_sweep_mode().load()),
                 stages);
    else
        stages();
    unsigned long long errs[11];
    RbControl ctls[5];
    int fac[2] = {0, 0x7fffffff};
    FNLH_CUDA(cudaMemcpyAsync(errs, stage_err_.ptr, sizeof errs, cudaMemcpyDeviceToHost, st));
    if (fac_status) FNLH_CUDA(cudaMemcpyAsync(fac, fac_status, sizeof fac, cudaMemcpyDeviceToHost, st));
    int df_active = 0;
    if (check_df && disc_->df_active())
        FNLH_CUDA(cudaMemcpyAsync(&df_active, disc_->df_active(), sizeof(int), cudaMemcpyDeviceToHost, st));
    if (rbA_ && sch_.implicit) FNLH_CUDA(cudaMemcpyAsync(ctls, ctl_.ptr, sizeof ctls, cudaMemcpyDeviceToHost, st));
    FNLH_CUDA(cudaMemcpyAsync(ws_->h_scalars + 8, ws_->scalars + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
    FNLH_CUDA(cudaStreamSynchronize(st));
    res.stage1_residual_norm = std::sqrt(ws_->h_scalars[8]);
    // errors raised before the step in the reference: the factorization, then DF
    if (fac[1] != 0x7fffffff) throw FactorizationError("near-singular ILU pivot block", fac[1]);
    if (check_df && df_active && errs[10] != ~0ull) {
        const int code = (int)(errs[10] & 15ull);
        if (code == 2) throw StateError("deterministic_flux: inadmissible state");
        if (code == 4) throw UnsupportedCaseError("deterministic_flux: supersonic boundary state");
        throw std::runtime_error("deterministic_flux: device error " + std::to_string(code));
    }
    check_step(errs, ctls, host_rep, have_host, field, res);
    FNLH_CUDA(cudaMemcpyAsync(state, stage, len * sizeof(S), cudaMemcpyDeviceToDevice, st));
    return res;
}

void DeviceSolver::add_level(const MeshArrays& mesh, const int* row_ptr, const int* col_idx, const int* parent,
                             const double* forcing_pairs, int nforcing) {
    if (sch_.implicit) throw ConfigError("multigrid is available for the explicit scheme only");
    DeviceDisc* fine = lv_disc(levels() - 1);
    const int nf = fine->n(), nc = mesh.n;
    if (mesh.b != disc_->b()) throw ShapeError("add_level: block size differs from the finest level");
    // children lists of the coarse nodes in ascending fine order (the reference's loops)
    std::vector<int> cptr(nc + 1, 0), cidx(nf);
    for (int i = 0; i < nf; ++i) {
        if (parent[i] < 0 || parent[i] >= nc) throw ShapeError("add_level: parent index out of range");
        ++cptr[parent[i] + 1];
    }
    for (int p = 0; p < nc; ++p) {
        if (cptr[p + 1] == 0) throw ShapeError("add_level: coarse node without children");
        cptr[p + 1] += cptr[p];
    }
    {
        std::vector<int> fill(cptr.begin(), cptr.end() - 1);
        for (int i = 0; i < nf; ++i) cidx[fill[parent[i]]++] = i;
    }
    auto L = std::make_unique<MgLevel>();
    L->pat = std::make_unique<DevicePattern>(mesh.b, mesh.n, row_ptr, col_idx, nullptr);
    L->disc = std::make_unique<DeviceDisc>(mesh, L->pat.get());
    L->parent.upload(parent, nf);
    L->cptr.upload(cptr.data(), cptr.size());
    L->cidx.upload(cidx.data(), cidx.size());
    L->nforcing = nforcing;
    L->forcing.alloc(std::max<std::size_t>((std::size_t)nh_ * nforcing, 1));
    if (nh_ * nforcing)
        FNLH_CUDA(cudaMemcpy(L->forcing.ptr, forcing_pairs, (std::size_t)nh_ * nforcing * sizeof(cplx),
                             cudaMemcpyHostToDevice));
    legacy_sync();
    const std::size_t len = (std::size_t)nc * mesh.b, bb = (std::size_t)nc * mesh.b * mesh.b;
    L->mean.alloc(len);
    L->P.alloc(bb);
    L->PLU.alloc(bb);
    L->pclu.alloc(bb);
    L->Ppiv.alloc(len);
    L->pcpiv.alloc(len);
    L->wc0.alloc(len);
    L->wc.alloc(len);
    L->rstar.alloc(len);
    mg_.push_back(std::move(L));
}

// coarse means (driver.cpp:168-171) and their transform_jacobian validation (:172-176);
// mg_diag_blocks: assemble_diag_blocks + LU per coarse level (:183-186)
void DeviceSolver::mg_means() {
    cudaStream_t st = ws_->stream;
    for (int l = 1; l < levels(); ++l) {
        MgLevel& c = *mg_[l - 1];
        const int nc = c.disc->n();
        ::fnlh::note_launch();
        k_restrict_state<double><<<nb(nc), kT, 0, st>>>(c.cptr.ptr, c.cidx.ptr, lv_disc(l - 1)->view().vol, c.disc->b(),
                                                         nc, lv_mean(l - 1), c.mean.ptr);
    }
    for (int l = 1; l < levels(); ++l) mg_[l - 1]->disc->validate(mg_[l - 1]->mean.ptr, st);
}

void DeviceSolver::mg_diag_blocks() {
    cudaStream_t st = ws_->stream;
    for (int l = 1; l < levels(); ++l) {
        MgLevel& c = *mg_[l - 1];
        const int nc = c.disc->n(), b = c.disc->b();
        c.disc->fd_jacobian(c.mean.ptr, nullptr, c.P.ptr, st);
        FNLH_CUDA(cudaMemcpyAsync(c.PLU.ptr, c.P.ptr, c.P.bytes(), cudaMemcpyDeviceToDevice, st));
        const int init[2] = {0, 0x7fffffff};
        FNLH_CUDA(cudaMemcpyAsync(ws_->status, init, sizeof init, cudaMemcpyHostToDevice, st));
        block_diag_factor<double>(b, nc, c.PLU.ptr, c.Ppiv.ptr, ws_->status, st);
        FNLH_CUDA(cudaMemcpyAsync(ws_->h_status, ws_->status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        if (ws_->h_status[1] != 0x7fffffff) throw FactorizationError("singular pivot block", ws_->h_status[1]);
    }
}

// LevelOps::full_residual (driver.cpp:230-236 harmonic, 300-306 mean): out = inv + vis
// (+ DF on the finest mean level); raises the evaluation's own error
template <class S>
void DeviceSolver::mg_full_residual(int h, int l, const S* state, S* out, S* vis) {
    cudaStream_t st = ws_->stream;
    DeviceDisc* d = lv_disc(l);
    const int order = l == 0 ? 2 : 1;
    if constexpr (std::is_same<S, cplx>::value) {
        d->linearized_residual(lv_mean(l), state, omega_[h], lv_forcing(l, h), lv_nforcing(l), order, true, out, vis,
                               st);
        add_inplace<cplx>(out, vis, d->len(), st);
    } else {
        d->residual(state, nullptr, order, 0, nullptr, 0, true, out, vis, st);
        add_inplace<double>(out, vis, d->len(), st);
        if (l == 0) add_inplace<double>(out, df_.ptr, d->len(), st);
    }
    d->raise_if_err(st, "full_residual");
}

// vcycle_level (multigrid.cpp:184-214): pre-smoothing RK step with the FAS forcing, then
// restriction, the coarse problem, and the injected correction
template <class S>
RkStepResult DeviceSolver::mg_vcycle(int h, int l, S* w, const S* forcing, const std::string& field) {
    cudaStream_t st = ws_->stream;
    DeviceDisc* d = lv_disc(l);
    const int n = d->n(), b = d->b();
    const double gamma = d->view().gamma;
    const int order = l == 0 ? 2 : 1;
    const double* mean = lv_mean(l);
    auto none = [&](const S*, S*, int, LinearSolveReport&) { return true; };
    RkStepResult res;
    if constexpr (std::is_same<S, cplx>::value) {
        const double omega = omega_[h];
        const cplx* hf = lv_forcing(l, h);
        const int nfl = lv_nforcing(l);
        auto eval = [&](const cplx* state, bool need_vis, cplx* inv, cplx* vis) {
            d->linearized_residual(mean, state, omega, hf, nfl, order, need_vis, inv, vis, st);
        };
        auto apply = [&](const cplx* base, const cplx* x, cplx* out) {
            apply_harmonic(b, n, gamma, mean, base, x, out, st);
        };
        res = rk_step<cplx>(w, eval, apply, none, l == 0 ? pclu_.ptr : mg_[l - 1]->pclu.ptr,
                            l == 0 ? pcpiv_.ptr : mg_[l - 1]->pcpiv.ptr, field, nullptr, false, l, forcing);
    } else {
        auto eval = [&](const double* state, bool need_vis, double* inv, double* vis) {
            d->residual(state, nullptr, order, 0, nullptr, 0, need_vis, inv, vis, st);
            if (l == 0) add_inplace<double>(inv, df_.ptr, d->len(), st);  // DF on the finest level only
        };
        auto apply = [&](const double* base, const double* x, double* out) {
            apply_mean(b, n, gamma, base, x, out, d->err(), st);
        };
        res = rk_step<double>(w, eval, apply, none, l == 0 ? PLU_.ptr : mg_[l - 1]->PLU.ptr,
                              l == 0 ? Ppiv_.ptr : mg_[l - 1]->Ppiv.ptr, field, nullptr, l == 0, l, forcing);
    }
    if (l + 1 >= levels()) return res;
    MgLevel& c = *mg_[l];
    const int nc = c.disc->n();
    S* wc0 = reinterpret_cast<S*>(c.wc0.ptr);
    S* wc = reinterpret_cast<S*>(c.wc.ptr);
    S* rstar = reinterpret_cast<S*>(c.rstar.ptr);
    S* rf = reinterpret_cast<S*>(rk_[1].ptr);  // the RK scratch is free between steps
    S* vf = reinterpret_cast<S*>(rk_[2].ptr);
    { ::fnlh::note_launch(); k_restrict_state<S><<<nb(nc), kT, 0, st>>>(c.cptr.ptr, c.cidx.ptr, d->view().vol, b, nc, w, wc0); }
    mg_full_residual<S>(h, l, w, rf, vf);
    mg_full_residual<S>(h, l + 1, wc0, rstar, vf);
    { ::fnlh::note_launch(); k_restrict_fas<S><<<nb(nc), kT, 0, st>>>(c.cptr.ptr, c.cidx.ptr, b, nc, rf, forcing, rstar); }
    FNLH_CUDA(cudaMemcpyAsync(wc, wc0, (std::size_t)nc * b * sizeof(S), cudaMemcpyDeviceToDevice, st));
    mg_vcycle<S>(h, l + 1, wc, rstar, field);
    { ::fnlh::note_launch(); k_prolong<S><<<nb(n), kT, 0, st>>>(c.parent.ptr, b, n, wc, wc0, w); }
    d->reset_err(st);
    check_finite<S>(w, d->len(), d->err(), st);
    if (d->read_err(st)) {
        d->reset_err(st);
        throw DivergenceError("non-finite state after coarse-grid correction", 0, field);
    }
    return res;
}

void DeviceSolver::harmonic_batch(const int* hs, int P, std::vector<double>& h_norm,
                                  std::vector<std::vector<LinearSolveReport>>& h_reps,
                                  std::vector<std::exception_ptr>& herr) {
    cudaStream_t st = ws_->stream;
    const int n = disc_->n(), b = disc_->b();
    const std::size_t len = disc_->len();
    const double gamma = disc_->view().gamma;
    const double ga5 = (1.0 / sch_.eps_relax) * kAlpha[4];
    std::vector<std::exception_ptr> early(P);  // level-scheduled path: factorization errors
    LaneReport lrep[kMaxBatch][5];
    int ldiv[kMaxBatch][5] = {};
    LinearSolveReport hrep[kMaxBatch][5];
    auto batch = [&] {
    FNLH_CUDA(cudaEventRecord(ev_stage_, st));
    for (int m = 0; m < P; ++m) {  // build_lhs_harmonic + factorize per lane (driver.cpp:213-216)
        HarmonicLane& ln = *lanes_[m];
        const int h = hs[m];
        const cplx* amp = amps_.ptr + (std::size_t)h * len;
        if (rbA_) {  // the lanes' factorizations are independent: one per lane stream
            cudaStream_t sm = ln.stream;
            FNLH_CUDA(cudaStreamWaitEvent(sm, ev_stage_, 0));
            harmonic_shift(disc_->view().vol, n, omega_[h], ga5, ln.shift.ptr, sm);
            rb_factorize_async<cplx>(*rbA_, ln.shift.ptr, *ln.f, ln.fac.ptr, sm);
            FNLH_CUDA(cudaEventRecord(ln.done, sm));
            FNLH_CUDA(cudaStreamWaitEvent(st, ln.done, 0));
        } else {  // likewise on the level-scheduled path (the status is checked after the step)
            cudaStream_t sm = ln.stream;
            FNLH_CUDA(cudaStreamWaitEvent(sm, ev_stage_, 0));
            harmonic_shift(disc_->view().vol, n, omega_[h], ga5, ln.shift.ptr, sm);
            SystemView<cplx> Ah;
            Ah.p = pat_.get();
            Ah.real_vals = A5_.ptr;
            Ah.real_sell = A5s_.ptr;
            Ah.shift_im = ln.shift.ptr;
            ilu_factorize_async<cplx>(Ah, *ln.gf, ln.fac.ptr, sm);
            FNLH_CUDA(cudaEventRecord(ln.done, sm));
            FNLH_CUDA(cudaStreamWaitEvent(st, ln.done, 0));
        }
        FNLH_CUDA(cudaMemcpyAsync(ln.v[0].ptr, amp, len * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        FNLH_CUDA(cudaMemcpyAsync(ln.v[6].ptr, amp, len * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        FNLH_CUDA(cudaMemsetAsync(ln.v[2].ptr, 0, len * sizeof(cplx), st));
        FNLH_CUDA(cudaMemsetAsync(ln.v[3].ptr, 0, len * sizeof(cplx), st));
        FNLH_CUDA(cudaMemsetAsync(ln.err.ptr, 0xff, 10 * sizeof(unsigned long long), st));
    }
    RbMember<cplx> mem[kMaxBatch];
    for (int k = 1; k <= 5; ++k) {  // rk_step (rk.cpp:41-99), the lanes interleaved stage by stage
        const double beta = kBeta[k - 1];
        const bool fresh = beta != 0.0;
        // the lanes' stage evaluations are independent: each runs on its own stream with its
        // own residual scratch (DeviceDisc context m), joined before the batched solve
        FNLH_CUDA(cudaEventRecord(ev_stage_, st));
        for (int m = 0; m < P; ++m) {
            if (early[m]) continue;
            HarmonicLane& ln = *lanes_[m];
            const int h = hs[m];
            cudaStream_t sm = ln.stream;
            FNLH_CUDA(cudaStreamWaitEvent(sm, ev_stage_, 0));
            disc_->use_context(m);
            disc_->redirect_err(ln.err.ptr + (k - 1));
            disc_->linearized_residual(mean_.ptr, ln.v[6].ptr, omega_[h], forcing_.ptr + (std::size_t)h * nforcing_,
                                       nforcing_, 2, fresh, ln.v[1].ptr, ln.v[2].ptr, sm);
            disc_->redirect_err(nullptr);
            disc_->use_context(0);
            if (fresh) stage_blend<cplx>(beta, ln.v[2].ptr, ln.v[3].ptr, len, sm);
            stage_rhs<cplx>(ln.v[1].ptr, ln.v[3].ptr, ln.v[4].ptr, len, sm);
            if (k == 1) norm2_sq_on<cplx>(ln.v[4].ptr, len, ln.norm.ptr, ln.nparts.ptr, sm);
            scale<cplx>(ln.v[4].ptr, kAlpha[k - 1], len, sm);
            FNLH_CUDA(cudaEventRecord(ln.done, sm));
            FNLH_CUDA(cudaStreamWaitEvent(st, ln.done, 0));
            if (rbA_)
                mem[m] = RbMember<cplx>{ln.f.get(), ln.shift.ptr, ln.v[4].ptr, ln.v[5].ptr,
                                        ln.v[7].ptr, ln.v[8].ptr, ln.ctl.ptr + (k - 1), ln.parts.ptr};
        }
        if (rbA_) {
            rb_smoothed_solve_batch<cplx>(*rbA_, mem, P, sch_.linear_tol, sch_.linear_max_iter, st);
        } else {  // level-scheduled lanes: one launch per level for every live lane
            LaneSystem<cplx> sys[kMaxBatch];
            LaneReport out[kMaxBatch];
            int live[kMaxBatch], nl = 0;
            for (int m = 0; m < P; ++m)
                if (!early[m]) {
                    HarmonicLane& ln = *lanes_[m];
                    sys[nl] = LaneSystem<cplx>{ln.gf.get(), ln.shift.ptr, ln.v[4].ptr, ln.v[5].ptr, ln.v[7].ptr,
                                               ln.v[8].ptr};
                    live[nl++] = m;
                }
            if (nl) smoothed_solve_batch<cplx>(*pat_, A5_.ptr, sys, nl, sch_.linear_tol, sch_.linear_max_iter, out, *ws_, A5s_.ptr);
            for (int q = 0; q < nl; ++q) {
                lrep[live[q]][k - 1] = out[q];
                hrep[live[q]][k - 1] = out[q].rep;
                ldiv[live[q]][k - 1] = out[q].diverged;
            }
        }
        for (int m = 0; m < P; ++m) {
            if (early[m]) continue;
            HarmonicLane& ln = *lanes_[m];
            disc_->redirect_err(ln.err.ptr + 5 + (k - 1));
            apply_harmonic(b, n, gamma, mean_.ptr, ln.v[0].ptr, ln.v[5].ptr, ln.v[6].ptr, st);
            check_finite<cplx>(ln.v[6].ptr, len, disc_->err(), st);
            disc_->redirect_err(nullptr);
        }
    }
    };
    if (rbA_) {  // factorizations + five stages of P lanes: one graph per batch of harmonics
        std::string key = "batch:" + std::to_string(rb_sweep_mode().load());
        for (int m = 0; m < P; ++m) key += ":" + std::to_string(hs[m]);
        captured(key, batch);
    } else {  // level-scheduled lanes synchronize per solve
        batch();
    }
    struct Rec {
        unsigned long long errs[10];
        RbControl ctls[5];
        int fac[2];
        double norm;
    };
    std::vector<Rec> rec(P);
    for (int m = 0; m < P; ++m) {
        HarmonicLane& ln = *lanes_[m];
        FNLH_CUDA(cudaMemcpyAsync(rec[m].errs, ln.err.ptr, sizeof rec[m].errs, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaMemcpyAsync(rec[m].ctls, ln.ctl.ptr, sizeof rec[m].ctls, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaMemcpyAsync(rec[m].fac, ln.fac.ptr, sizeof rec[m].fac, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaMemcpyAsync(&rec[m].norm, ln.norm.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    FNLH_CUDA(cudaStreamSynchronize(st));
    for (int m = 0; m < P; ++m) {  // each lane as its own worker: commit or capture (driver.cpp:248-262)
        const int h = hs[m];
        if (early[m]) {
            herr[h] = early[m];
            continue;
        }
        try {
            if (rec[m].fac[1] != 0x7fffffff) throw FactorizationError("near-singular ILU pivot block", rec[m].fac[1]);
            RkStepResult res;
            res.stage1_residual_norm = std::sqrt(rec[m].norm);
            const bool all[5] = {true, true, true, true, true};
            check_step(rec[m].errs, rec[m].ctls, rbA_ ? nullptr : hrep[m], rbA_ ? nullptr : all,
                       "harmonic-" + std::to_string(index_[h]), res, rbA_ ? nullptr : ldiv[m]);
            FNLH_CUDA(cudaMemcpyAsync(amps_.ptr + (std::size_t)h * len, lanes_[m]->v[6].ptr, len * sizeof(cplx),
                                      cudaMemcpyDeviceToDevice, st));
            h_norm[h] = res.stage1_residual_norm;
            h_reps[h] = std::move(res.linear_reports);
        } catch (...) {
            herr[h] = std::current_exception();
        }
    }
}

ConvergenceEntry DeviceSolver::outer_iteration() {
    phase_harmonics(nullptr);
    return phase_mean(h_norm_, h_reps_);
}

// FD Jacobian straight into A5 (build_lhs_mean fused into the column kernel): the SELL copy
// of the 2-colour path, else the BSR A5
void DeviceSolver::assemble_a5(cudaStream_t st) {
    const double ga5 = (1.0 / sch_.eps_relax) * kAlpha[4];
    const double inv_es = 1.0 / (sch_.eps_relax * sigma_);
    A5Target t{};
    t.ga = ga5;
    t.inv_es = inv_es;
    if (rbA_) {
        t.vals = rbA_->vals_mut();
        t.sell_map = rbA_->sell_map();
        t.bytes = rbA_->bytes();
    } else {
        t.vals = A5_.ptr;
        t.sell_map = nullptr;
        t.bytes = A5_.bytes();
    }
    disc_->fd_jacobian(mean_.ptr, nullptr, nullptr, st, &t);
    if (!rbA_) sell_from_bsr(*pat_, A5_.ptr, A5s_.ptr, st);
}

ConvergenceEntry DeviceSolver::outer_iteration_host(const double* mean_in, const cplx* amps_in, double* mean_out,
                                                    cplx* amps_out) {
    cudaStream_t st = ws_->stream;
    const std::size_t len = disc_->len();
    FNLH_CUDA(cudaStreamSynchronize(cs_));
    FNLH_CUDA(cudaMemcpyAsync(mean_.ptr, mean_in, len * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nh_) {
        FNLH_CUDA(cudaMemcpyAsync(amps_.ptr, amps_in, (std::size_t)nh_ * len * sizeof(cplx), cudaMemcpyHostToDevice,
                                  cs_));
        FNLH_CUDA(cudaEventRecord(ev_in_, cs_));
    }
    struct Reset {
        DeviceSolver* s;
        ~Reset() {
            s->wait_amps_ = false;
            s->amps_download_ = nullptr;
            cudaStreamSynchronize(s->cs_);
        }
    } reset{this};
    wait_amps_ = nh_ > 0;
    amps_download_ = amps_out;
    phase_harmonics(nullptr);
    ConvergenceEntry e = phase_mean(h_norm_, h_reps_);
    FNLH_CUDA(cudaMemcpyAsync(mean_out, mean_.ptr, len * sizeof(double), cudaMemcpyDeviceToHost, st));
    FNLH_CUDA(cudaStreamSynchronize(st));
    FNLH_CUDA(cudaStreamSynchronize(cs_));
    return e;
}

void DeviceSolver::phase_harmonics(const int* owned) {
    cudaStream_t st = ws_->stream;
    FNLH_CUDA(cudaEventRecord(ev0_, st));
    ++iter_;
    failed_h_ = -1;
    const int n = disc_->n(), b = disc_->b();
    const std::size_t len = disc_->len();
    const double gamma = disc_->view().gamma;
    disc_->validate(mean_.ptr, st);  // transform_jacobian / MLU.factor (driver.cpp:172-176)

    const bool implicit = sch_.implicit != 0;
    const double ga5 = (implicit ? 1.0 / sch_.eps_relax : sigma_) * kAlpha[4];
    if (implicit) {
        assemble_a5(st);  // J and build_lhs_mean (rk.cpp:5-30) in one pass
        if (rbA_) {
            rb_factorize<double>(*rbA_, nullptr, *rb_mean_, *ws_);
        } else {
            SystemView<double> Am;
            Am.p = pat_.get();
            Am.real_vals = A5_.ptr;
            Am.real_sell = A5s_.ptr;
            ilu_factorize<double>(Am, *ilu_mean_, *ws_);
        }
    } else {
        if (!mg_.empty()) mg_means();
        disc_->fd_jacobian(mean_.ptr, nullptr, P_.ptr, st);  // assemble_diag_blocks (disc.cpp:31-35)
        FNLH_CUDA(cudaMemcpyAsync(PLU_.ptr, P_.ptr, P_.bytes(), cudaMemcpyDeviceToDevice, st));
        const int init[2] = {0, 0x7fffffff};
        FNLH_CUDA(cudaMemcpyAsync(ws_->status, init, sizeof init, cudaMemcpyHostToDevice, st));
        block_diag_factor<double>(b, n, PLU_.ptr, Ppiv_.ptr, ws_->status, st);
        FNLH_CUDA(cudaMemcpyAsync(ws_->h_status, ws_->status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        if (ws_->h_status[1] != 0x7fffffff) throw FactorizationError("singular pivot block", ws_->h_status[1]);
        if (!mg_.empty()) mg_diag_blocks();
    }

    FNLH_CUDA(cudaEventRecord(evp_[0], st));  // phase marks: J + A5 + mean ILU done
    if (wait_amps_) FNLH_CUDA(cudaStreamWaitEvent(st, ev_in_, 0));  // harmonic fields uploaded
    std::vector<double>& h_norm = h_norm_;
    std::vector<std::vector<LinearSolveReport>>& h_reps = h_reps_;
    h_norm.assign(nh_, 0.0);
    h_reps.assign(nh_, {});
    std::vector<std::exception_ptr> herr(nh_);
    const bool parallel = sch_.workers > 1 && nh_ > 1;  // driver.cpp:246-265
    std::vector<int> mine;  // harmonics this solver relaxes (all, or this rank's shard)
    for (int h = 0; h < nh_; ++h)
        if (!owned || owned[h]) mine.push_back(h);
    if (!lanes_.empty()) {
        const int P = static_cast<int>(lanes_.size());
        for (std::size_t q = 0; q < mine.size(); q += P)
            harmonic_batch(mine.data() + q, std::min<int>(P, (int)(mine.size() - q)), h_norm, h_reps, herr);
    } else {
        for (int h : mine) {
            try {
                cplx* amp = amps_.ptr + (std::size_t)h * len;
                const double omega = omega_[h];
                const std::string name = "harmonic-" + std::to_string(index_[h]);
                const cplx* forcing = forcing_.ptr + (std::size_t)h * nforcing_;
                auto eval = [&](const cplx* state, bool need_vis, cplx* inv, cplx* vis) {
                    disc_->linearized_residual(mean_.ptr, state, omega, forcing, nforcing_, 2, need_vis, inv, vis, st);
                };
                auto apply = [&](const cplx* base, const cplx* x, cplx* out) {
                    apply_harmonic(b, n, gamma, mean_.ptr, base, x, out, st);
                };
                RkStepResult step;
                if (implicit) {
                    harmonic_shift(disc_->view().vol, n, omega, ga5, shift_.ptr, st);
                    SystemView<cplx> Ah;
                    Ah.p = pat_.get();
                    Ah.real_vals = A5_.ptr;
                    Ah.real_sell = A5s_.ptr;
                    Ah.shift_im = shift_.ptr;
                    if (rbA_) {
                        rb_factorize_async<cplx>(*rbA_, shift_.ptr, *rb_h_, fac_status_.ptr, st);
                        auto solve = [&](const cplx* rhs, cplx* x, int k, LinearSolveReport&) {
                            rb_solve_async<cplx>(shift_.ptr, *rb_h_, rhs, x, ctl_.ptr + (k - 1));
                            return false;
                        };
                        step = rk_step<cplx>(amp, eval, apply, solve, nullptr, nullptr, name, fac_status_.ptr);
                    } else {
                        ilu_factorize<cplx>(Ah, *ilu_h_, *ws_);
                        auto solve = [&](const cplx* rhs, cplx* x, int, LinearSolveReport& rep) {
                            rep = smoothed_solve<cplx>(Ah, rhs, *ilu_h_, sch_.linear_tol, sch_.linear_max_iter, x, *ws_);
                            return true;
                        };
                        step = rk_step<cplx>(amp, eval, apply, solve, nullptr, nullptr, name);
                    }
                } else {
                    shifted_blocks(P_.ptr, disc_->view().vol, b, n, omega, pclu_.ptr, st);
                    const int init[2] = {0, 0x7fffffff};
                    FNLH_CUDA(cudaMemcpyAsync(ws_->status, init, sizeof init, cudaMemcpyHostToDevice, st));
                    block_diag_factor<cplx>(b, n, pclu_.ptr, pcpiv_.ptr, ws_->status, st);
                    FNLH_CUDA(cudaMemcpyAsync(ws_->h_status, ws_->status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
                    FNLH_CUDA(cudaStreamSynchronize(st));
                    if (ws_->h_status[1] != 0x7fffffff) throw FactorizationError("singular pivot block", ws_->h_status[1]);
                    for (int l = 1; l < levels(); ++l) {  // shifted_blocks per level (driver.cpp:224-229)
                        MgLevel& c = *mg_[l - 1];
                        const int nc = c.disc->n();
                        shifted_blocks(c.P.ptr, c.disc->view().vol, b, nc, omega, c.pclu.ptr, st);
                        FNLH_CUDA(cudaMemcpyAsync(ws_->status, init, sizeof init, cudaMemcpyHostToDevice, st));
                        block_diag_factor<cplx>(b, nc, c.pclu.ptr, c.pcpiv.ptr, ws_->status, st);
                        FNLH_CUDA(cudaMemcpyAsync(ws_->h_status, ws_->status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
                        FNLH_CUDA(cudaStreamSynchronize(st));
                        if (ws_->h_status[1] != 0x7fffffff)
                            throw FactorizationError("singular pivot block", ws_->h_status[1]);
                    }
                    if (!mg_.empty()) {
                        step = mg_vcycle<cplx>(h, 0, amp, nullptr, name);
                    } else {
                        auto none = [&](const cplx*, cplx*, int, LinearSolveReport&) { return true; };
                        step = rk_step<cplx>(amp, eval, apply, none, pclu_.ptr, pcpiv_.ptr, name);
                    }
                }
                h_norm[h] = step.stage1_residual_norm;
                h_reps[h] = std::move(step.linear_reports);
            } catch (...) {
                if (!parallel) {
                    failed_h_ = h;
                    throw;
                }
                herr[h] = std::current_exception();
            }
        }
    }
    for (int h = 0; h < nh_; ++h)
        if (herr[h]) {
            failed_h_ = h;
            std::rethrow_exception(herr[h]);
        }
    if (amps_download_ && nh_) {  // updated harmonic fields home while DF and the mean step run
        FNLH_CUDA(cudaEventRecord(ev_h_, st));
        FNLH_CUDA(cudaStreamWaitEvent(cs_, ev_h_, 0));
        FNLH_CUDA(cudaMemcpyAsync(amps_download_, amps_.ptr, (std::size_t)nh_ * len * sizeof(cplx),
                                  cudaMemcpyDeviceToHost, cs_));
    }
}

int DeviceSolver::df_points() { return disc_->df_points(omega_); }

void DeviceSolver::df_terms(int k0, int k1, double* terms) {
    const std::size_t len = disc_->len();
    std::vector<const cplx*> amps;
    for (int h = 0; h < nh_; ++h) amps.push_back(amps_.ptr + (std::size_t)h * len);
    disc_->df_terms(mean_.ptr, amps, omega_, k0, k1, terms, ws_->stream);
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
}

void DeviceSolver::df_accumulate(const double* terms, int count, double* acc, bool first) {
    disc_->df_accumulate(terms, count, acc, first, ws_->stream);
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
}

ConvergenceEntry DeviceSolver::phase_mean(const std::vector<double>& h_norm,
                                          const std::vector<std::vector<LinearSolveReport>>& h_reps) {
    cudaStream_t st = ws_->stream;
    const int n = disc_->n(), b = disc_->b();
    const std::size_t len = disc_->len();
    const double gamma = disc_->view().gamma;
    const bool implicit = sch_.implicit != 0;
    if ((int)h_norm.size() != nh_ || (int)h_reps.size() != nh_) throw ShapeError("phase_mean: one entry per harmonic");
    // deterministic flux from the fresh harmonic fields (driver.cpp:268-271)
    FNLH_CUDA(cudaEventRecord(evp_[1], st));  // harmonics done (and exchanged, when sharded)
    std::vector<const cplx*> amps;
    for (int h = 0; h < nh_; ++h) amps.push_back(amps_.ptr + (std::size_t)h * len);
    FNLH_CUDA(cudaMemsetAsync(stage_err_.ptr + 10, 0xff, sizeof(unsigned long long), st));
    disc_->redirect_err(stage_err_.ptr + 10);
    std::vector<cudaStream_t> side;  // the lanes' streams take quadrature points concurrently
    for (std::size_t m = 1; m < lanes_.size(); ++m) side.push_back(lanes_[m]->stream);
    if (ext_df_acc_) {  // the quadrature sum chained across ranks (df_terms / df_accumulate)
        disc_->df_finish(mean_.ptr, amps, omega_, ext_df_acc_, df_.ptr, st, /*deferred=*/true);
        ext_df_acc_ = nullptr;
    } else {
        disc_->deterministic_flux(mean_.ptr, amps, omega_, df_.ptr, st, /*deferred=*/true, side);
    }
    disc_->redirect_err(nullptr);

    FNLH_CUDA(cudaEventRecord(evp_[2], st));  // DF done
    // mean update including DF (driver.cpp:273-296)
    auto mean_eval = [&](const double* state, bool need_vis, double* inv, double* vis) {
        disc_->residual(state, nullptr, 2, 0, nullptr, 0, need_vis, inv, vis, st);
        add_inplace<double>(inv, df_.ptr, len, st);
    };
    auto mean_apply = [&](const double* base, const double* x, double* out) {
        apply_mean(b, n, gamma, base, x, out, disc_->err(), st);
    };
    RkStepResult mstep;
    if (implicit && rbA_) {
        auto solve = [&](const double* rhs, double* x, int k, LinearSolveReport&) {
            rb_solve_async<double>(nullptr, *rb_mean_, rhs, x, ctl_.ptr + (k - 1));
            return false;
        };
        mstep = rk_step<double>(mean_.ptr, mean_eval, mean_apply, solve, nullptr, nullptr, "mean", nullptr, true);
    } else if (implicit) {
        SystemView<double> Am;
        Am.p = pat_.get();
        Am.real_vals = A5_.ptr;
        Am.real_sell = A5s_.ptr;
        auto solve = [&](const double* rhs, double* x, int, LinearSolveReport& rep) {
            rep = smoothed_solve<double>(Am, rhs, *ilu_mean_, sch_.linear_tol, sch_.linear_max_iter, x, *ws_);
            return true;
        };
        mstep = rk_step<double>(mean_.ptr, mean_eval, mean_apply, solve, nullptr, nullptr, "mean", nullptr, true);
    } else if (!mg_.empty()) {  // FAS V-cycle of the mean (driver.cpp:297-311)
        mstep = mg_vcycle<double>(-1, 0, mean_.ptr, nullptr, "mean");
    } else {
        auto none = [&](const double*, double*, int, LinearSolveReport&) { return true; };
        mstep = rk_step<double>(mean_.ptr, mean_eval, mean_apply, none, PLU_.ptr, Ppiv_.ptr, "mean", nullptr, true);
    }
    for (const auto& hr : h_reps)
        for (const auto& r : hr) reports_.push_back(r);
    for (auto& r : mstep.linear_reports) reports_.push_back(r);

    FNLH_CUDA(cudaEventRecord(ev1_, st));
    FNLH_CUDA(cudaEventSynchronize(ev1_));
    FNLH_CUDA(cudaEventElapsedTime(&last_iteration_ms, ev0_, ev1_));
    {
        cudaEvent_t marks[5] = {ev0_, evp_[0], evp_[1], evp_[2], ev1_};
        for (int k = 0; k < 4; ++k) FNLH_CUDA(cudaEventElapsedTime(&phase_ms[k], marks[k], marks[k + 1]));
    }
    cum_seconds_ += last_iteration_ms * 1e-3;

    ConvergenceEntry e;  // driver.cpp:315-332
    e.iter = iter_;
    e.resid_mean = mstep.stage1_residual_norm / std::sqrt((double)n * b);
    e.resid_h.resize(nh_);
    double acc = 0.0;
    for (int h = 0; h < nh_; ++h) {
        e.resid_h[h] = h_norm[h] / std::sqrt((double)n * b);
        acc += e.resid_h[h] * e.resid_h[h];
    }
    e.has_rz = nh_ > 0;
    e.rz = nh_ > 0 ? std::sqrt(acc / nh_) : 0.0;
    e.seconds = cum_seconds_;
    return e;
}

void DeviceSolver::copy_amps(int h, void* dev, bool to_dev) {
    if (h < 0 || h >= nh_) throw ShapeError("copy_amps: harmonic index out of range");
    const std::size_t bytes = disc_->len() * sizeof(cplx);
    cplx* a = amps_.ptr + (std::size_t)h * disc_->len();
    FNLH_CUDA(cudaMemcpyAsync(to_dev ? dev : (void*)a, to_dev ? (const void*)a : dev, bytes, cudaMemcpyDeviceToDevice,
                              ws_->stream));
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
}

double DeviceSolver::time_harmonic_sweeps(int h, int nsweeps) {
    if (!sch_.implicit) throw ConfigError("time_harmonic_sweeps: implicit scheme only");
    cudaStream_t st = ws_->stream;
    const int n = disc_->n(), b = disc_->b();
    const std::size_t len = disc_->len();
    const double ga5 = (1.0 / sch_.eps_relax) * kAlpha[4];
    assemble_a5(st);
    harmonic_shift(disc_->view().vol, n, omega_[h], ga5, shift_.ptr, st);
    SystemView<cplx> Ah;
    Ah.p = pat_.get();
    Ah.real_vals = A5_.ptr;
    Ah.real_sell = A5s_.ptr;
    Ah.shift_im = shift_.ptr;
    RbIlu<cplx>* fh = rb_h_ ? rb_h_.get() : (lanes_.empty() ? nullptr : lanes_[0]->f.get());
    DeviceIlu<cplx>* gh = ilu_h_ ? ilu_h_.get() : (lanes_.empty() ? nullptr : lanes_[0]->gf.get());
    if (rbA_) {
        rb_factorize<cplx>(*rbA_, shift_.ptr, *fh, *ws_);
    } else {
        ilu_factorize<cplx>(Ah, *gh, *ws_);
    }
    // rhs: the harmonic's current linearized residual direction (any nonzero vector works)
    cplx* rhs = rk_[4].ptr;
    cplx* x = rk_[5].ptr;
    disc_->linearized_residual(mean_.ptr, amps_.ptr + (std::size_t)h * len, omega_[h],
                               forcing_.ptr + (std::size_t)h * nforcing_, nforcing_, 2, false, rhs, nullptr, st);
    FNLH_CUDA(cudaStreamSynchronize(st));
    FNLH_CUDA(cudaEventRecord(ev0_, st));
    if (rbA_)
        rb_smoothed_solve<cplx>(*rbA_, shift_.ptr, *fh, rhs, 1e-300, nsweeps, x, rb_z_.ptr, rb_r_.ptr, ctl_.ptr,
                                *ws_);
    else
        smoothed_solve<cplx>(Ah, rhs, *gh, 1e-300, nsweeps, x, *ws_);
    FNLH_CUDA(cudaEventRecord(ev1_, st));
    FNLH_CUDA(cudaEventSynchronize(ev1_));
    float ms = 0.0f;
    FNLH_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    return ms;
}

double DeviceSolver::time_harmonic_sweeps_batch(int P, int nsweeps) {
    if (lanes_.empty() || P < 1 || P > (int)lanes_.size() || P > nh_)
        throw ConfigError("time_harmonic_sweeps_batch: needs workers >= P harmonic lanes");
    cudaStream_t st = ws_->stream;
    const int n = disc_->n(), b = disc_->b();
    const std::size_t len = disc_->len();
    const double ga5 = (1.0 / sch_.eps_relax) * kAlpha[4];
    assemble_a5(st);
    RbMember<cplx> mem[kMaxBatch];
    LaneSystem<cplx> sys[kMaxBatch];
    for (int m = 0; m < P; ++m) {
        HarmonicLane& ln = *lanes_[m];
        harmonic_shift(disc_->view().vol, n, omega_[m], ga5, ln.shift.ptr, st);
        if (rbA_) {
            rb_factorize<cplx>(*rbA_, ln.shift.ptr, *ln.f, *ws_);
        } else {
            SystemView<cplx> Ah;
            Ah.p = pat_.get();
            Ah.real_vals = A5_.ptr;
            Ah.real_sell = A5s_.ptr;
            Ah.shift_im = ln.shift.ptr;
            ilu_factorize<cplx>(Ah, *ln.gf, *ws_);
        }
        disc_->linearized_residual(mean_.ptr, amps_.ptr + (std::size_t)m * len, omega_[m],
                                   forcing_.ptr + (std::size_t)m * nforcing_, nforcing_, 2, false, ln.v[4].ptr, nullptr,
                                   st);
        if (rbA_)
            mem[m] = RbMember<cplx>{ln.f.get(), ln.shift.ptr, ln.v[4].ptr, ln.v[5].ptr, ln.v[7].ptr, ln.v[8].ptr,
                                    ln.ctl.ptr, ln.parts.ptr};
        else
            sys[m] = LaneSystem<cplx>{ln.gf.get(), ln.shift.ptr, ln.v[4].ptr, ln.v[5].ptr, ln.v[7].ptr, ln.v[8].ptr};
    }
    FNLH_CUDA(cudaStreamSynchronize(st));
    FNLH_CUDA(cudaEventRecord(ev0_, st));
    if (rbA_) {
        rb_smoothed_solve_batch<cplx>(*rbA_, mem, P, 1e-300, nsweeps, st);
    } else {
        LaneReport out[kMaxBatch];
        smoothed_solve_batch<cplx>(*pat_, A5_.ptr, sys, P, 1e-300, nsweeps, out, *ws_, A5s_.ptr);
    }
    FNLH_CUDA(cudaEventRecord(ev1_, st));
    FNLH_CUDA(cudaEventSynchronize(ev1_));
    float ms = 0.0f;
    FNLH_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    return ms;
}

int DeviceSolver::run_to_convergence(std::vector<ConvergenceEntry>& history) {  // driver.cpp:335-379
    const double drop = std::pow(10.0, -sch_.target_drop_orders);
    double r1_mean = -1.0, r1_rz = -1.0, floor_ = 0.0;
    for (int it = 0; it < sch_.max_outer_iters; ++it) {
        ConvergenceEntry e;
        try {
            e = outer_iteration();
        } catch (const DivergenceError&) {
            return 2;
        }
        history.push_back(e);
        if (it == 0) {
            r1_mean = e.resid_mean;
            r1_rz = e.has_rz ? e.rz : 0.0;
            floor_ = 1e-16 * std::max(r1_mean, r1_rz);
        }
        const bool mean_ok = e.resid_mean <= std::max(r1_mean * drop, floor_);
        const bool rz_ok = !e.has_rz || e.rz <= std::max(r1_rz * drop, floor_);
        if (mean_ok && rz_ok) return 0;
    }
    return 1;
}

void DeviceSolver::get_state(double* mean, double* amps_pairs) const {
    const std::size_t len = disc_->len();
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
    if (mean) download(mean, mean_.ptr, len);
    if (amps_pairs && nh_) download(reinterpret_cast<cplx*>(amps_pairs), amps_.ptr, (std::size_t)nh_ * len);
}

void DeviceSolver::set_state(const double* mean, const double* amps_pairs) {
    const std::size_t len = disc_->len();
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
    if (mean) FNLH_CUDA(cudaMemcpy(mean_.ptr, mean, len * sizeof(double), cudaMemcpyHostToDevice));
    if (amps_pairs && nh_)
        FNLH_CUDA(cudaMemcpy(amps_.ptr, amps_pairs, (std::size_t)nh_ * len * sizeof(cplx), cudaMemcpyHostToDevice));
    legacy_sync();
}

void DeviceSolver::get_df(double* df) const {
    FNLH_CUDA(cudaStreamSynchronize(ws_->stream));
    download(df, df_.ptr, disc_->len());
}

}  // namespace fnlh
