// solver.cuh -- the FNLH outer iteration resident on one B200 (driver.cpp:157-333):
// FD Jacobian -> A5 -> real ILU; per harmonic: complex ILU of A5 + i omega V / (Gamma
// alpha_5) in ONE reused workspace, rk_step with the linearized residual; DF; mean
// rk_step.  Host code is the reference's orchestration; every array stays in HBM.
#pragma once

#include <exception>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "disc.cuh"
#include "la.cuh"
#include "rb.cuh"

namespace fnlh {

struct SchemeConfig {  // driver.hpp:22-42
    int implicit = 1;
    double sigma_cfl = -1.0;
    double eps_relax = 0.6;
    double linear_tol = 1e-2;
    int linear_max_iter = 10;
    double target_drop_orders = 8.0;
    int max_outer_iters = 2000;
    int workers = 1;  // harmonics in flight (driver.cpp:246-265); >1: all run, first error rethrown
};

// one harmonic in flight on the device (a reference harmonic worker, driver.cpp:246-265):
// its complex ILU workspace, shift and RK vectors; the batched sweep serves up to
// kMaxBatch lanes from one read of the shared A5
struct HarmonicLane {
    std::unique_ptr<RbIlu<cplx>> f;           // 2-colour path
    std::unique_ptr<DeviceIlu<cplx>> gf;      // level-scheduled path
    DeviceBuffer<double> shift;
    DeviceBuffer<cplx> v[9];  // state0, inv, vis_fresh, vis_blend, rhs, x, stage, z, r
    DeviceBuffer<RbControl> ctl;             // one per RK stage
    DeviceBuffer<unsigned long long> err;    // [0,5) eval, [5,10) apply
    DeviceBuffer<int> fac;                   // factorization status
    DeviceBuffer<double> parts, norm;        // norm partials, stage-1 ||rhs||^2
    DeviceBuffer<double> nparts;             // partials of the lane's own ||rhs|| reduction
    cudaStream_t stream = nullptr;           // the lane's stage evaluations run here concurrently
    cudaEvent_t done = nullptr;
    ~HarmonicLane() {
        if (done) cudaEventDestroy(done);
        if (stream) cudaStreamDestroy(stream);
    }
};

// a coarse multigrid level (multigrid.hpp:26-32; the explicit scheme only, driver.cpp:101-131):
// its discretization on the agglomerated mesh, the parent map from the next finer level and
// the children lists of its own nodes (ascending fine index: the reference's summation
// order), its boundary forcing, the per-level mean / diagonal blocks, and the V-cycle
// vectors that live across the recursion (complex-sized, reinterpreted for the mean)
struct MgLevel {
    std::unique_ptr<DevicePattern> pat;
    std::unique_ptr<DeviceDisc> disc;
    DeviceBuffer<int> parent, cptr, cidx;
    DeviceBuffer<cplx> forcing;  // nh x nforcing
    int nforcing = 0;
    DeviceBuffer<double> mean, P, PLU;
    DeviceBuffer<int> Ppiv, pcpiv;
    DeviceBuffer<cplx> pclu;
    DeviceBuffer<cplx> wc0, wc, rstar;
};

struct ConvergenceEntry {  // driver.hpp:50-58
    int iter = 0;
    double resid_mean = 0.0;
    std::vector<double> resid_h;
    double rz = 0.0;
    int has_rz = 0;
    double seconds = 0.0;  // cumulative device time of outer iterations
};

struct RkStepResult {  // rk.hpp:68-72
    double stage1_residual_norm = 0.0;
    int viscous_evaluations = 0;
    std::vector<LinearSolveReport> linear_reports;
};

// CUDA graphs for the launch sequences of the outer iteration that contain no host
// synchronization: the five stages of an RK step (residual / linearized residual, stage
// arithmetic, the device-gated Richardson sweeps) and a harmonic batch's factorizations +
// stages.  Captured once per call site (key), replayed every outer iteration; the host
// synchronization that reads the step's error words stays outside.  fnlh_set_graphs(0)
// (or FNLH_GRAPHS=0) enqueues the same work launch by launch.
std::atomic<int>& graphs_enabled();

class DeviceSolver {
public:
    DeviceSolver(const MeshArrays& mesh, const int* row_ptr, const int* col_idx, const int* partition,
                 const SchemeConfig& scheme, int nh, const int* index, const double* omega,
                 const double* forcing_pairs, int nforcing, const double* mean0);
    ~DeviceSolver();

    ConvergenceEntry outer_iteration();  // phase_harmonics(all) + phase_mean
    // outer_iteration on host buffers (the reference-facing call): the mean is uploaded
    // first, the harmonic fields on a copy stream while the Jacobian / A5 / mean ILU run,
    // and the updated harmonic fields go back on the copy stream while DF and the mean
    // step run; in/out may alias
    ConvergenceEntry outer_iteration_host(const double* mean_in, const cplx* amps_in, double* mean_out,
                                          cplx* amps_out);
    // the two halves of outer_iteration, split where harmonic sharding exchanges the
    // harmonic fields: J, A5, mean ILU and the owned harmonics' RK steps
    // (owned: nh flags, nullptr = all) ...
    void phase_harmonics(const int* owned);
    // harmonic whose error the last phase_harmonics rethrew (-1: none, or an error before the harmonics)
    int failed_harmonic() const { return failed_h_; }
    // deterministic_flux split over quadrature points (shard.py: ranks chain the in-order sum,
    // residual_ops.cpp:145-160): the point count; R(W(t_k)) for k in [k0, k1) into device
    // `terms`; their in-order sum into device `acc`; and acc as the DF source of the next
    // phase_mean.  All synchronize before returning.
    int df_points();
    void df_terms(int k0, int k1, double* terms);
    void df_accumulate(const double* terms, int count, double* acc, bool first);
    void set_external_df(const double* acc) { ext_df_acc_ = acc; }
    const std::vector<double>& last_h_norm() const { return h_norm_; }
    const std::vector<std::vector<LinearSolveReport>>& last_h_reports() const { return h_reps_; }
    // ... then DF from every harmonic field, the mean RK step and the monitor, given every
    // harmonic's stage-1 norm and reports (in harmonic order)
    ConvergenceEntry phase_mean(const std::vector<double>& h_norm, const std::vector<std::vector<LinearSolveReport>>& h_reps);
    // copy harmonic h's field to / from device memory owned by the caller (exchange buffers)
    void copy_amps(int h, void* dev, bool to_dev);
    int run_to_convergence(std::vector<ConvergenceEntry>& history);  // 0 target, 1 cap, 2 divergence
    // append a coarse level below the current coarsest (explicit scheme): its mesh and
    // pattern, parent[n of the current coarsest] -> its nodes, its boundary forcing
    void add_level(const MeshArrays& mesh, const int* row_ptr, const int* col_idx, const int* parent,
                   const double* forcing_pairs, int nforcing);
    int levels() const { return 1 + static_cast<int>(mg_.size()); }

    void get_state(double* mean, double* amps_pairs) const;
    void set_state(const double* mean, const double* amps_pairs);
    void get_df(double* df) const;
    const std::vector<LinearSolveReport>& reports() const { return reports_; }
    std::size_t lhs_bytes() const;  // LHS value storage (A5 + real ILU + one complex ILU workspace per lane)
    int lanes() const { return lanes_.empty() ? 1 : (int)lanes_.size(); }
    // time `sweeps` batched Richardson sweeps of harmonics [0, P) (P <= lanes())
    double time_harmonic_sweeps_batch(int P, int sweeps);
    // time-accurate reference solver (SPEC oracle_urans; oracle.hpp:28-52; urans.cu):
    // include/fnlh_b200.h fnlh_solver_unsteady
    void unsteady_solve(const double* steady_host, int samples_per_period, double cfl, double periodic_tol,
                        int max_periods, int min_periods, double* samples_host, double* info);
    int n() const { return disc_->n(); }
    int b() const { return disc_->b(); }
    int nh() const { return nh_; }
    double sigma() const { return sigma_; }
    cudaStream_t stream() const { return ws_->stream; }
    // time `sweeps` Richardson sweeps of harmonic h's system at the current mean (factorizes
    // it first); returns device ms for the whole loop (bench.py roofline leg)
    double time_harmonic_sweeps(int h, int sweeps);
    // counters for the bench: total sweeps and block-row updates performed
    long long sweeps = 0, row_updates = 0;
    float last_iteration_ms = 0.0f;
    // last outer iteration split: J + A5 + mean ILU, harmonics, DF, mean RK (device ms)
    float phase_ms[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    bool red_black() const { return rbA_ != nullptr; }
    void info(double* out) const {
        out[0] = rbA_ ? 1.0 : 0.0;
        out[1] = rbA_ ? rbA_->n0() : -1.0;
        out[2] = rbA_ ? (double)rbA_->layout().total_vals : 0.0;
        out[3] = pat_->nnzb;
    }

private:
    template <class S, class Eval, class Apply, class Solve>
    RkStepResult rk_step(S* state, Eval&& eval, Apply&& apply, Solve&& solve, const S* pdiag_lu, const int* pdiag_piv,
                         const std::string& field, const int* fac_status = nullptr, bool check_df = false,
                         int level = 0, const S* mg_forcing = nullptr);
    // the FAS V-cycle from level l (multigrid.cpp:184-214); h = harmonic position, -1 = mean
    template <class S>
    RkStepResult mg_vcycle(int h, int l, S* w, const S* forcing, const std::string& field);
    template <class S>
    void mg_full_residual(int h, int l, const S* state, S* out, S* vis);
    DeviceDisc* lv_disc(int l) const { return l == 0 ? disc_.get() : mg_[l - 1]->disc.get(); }
    double* lv_mean(int l) const { return l == 0 ? mean_.ptr : mg_[l - 1]->mean.ptr; }
    const cplx* lv_forcing(int l, int h) const {
        return l == 0 ? forcing_.ptr + (std::size_t)h * nforcing_ : mg_[l - 1]->forcing.ptr + (std::size_t)h * mg_[l - 1]->nforcing;
    }
    int lv_nforcing(int l) const { return l == 0 ? nforcing_ : mg_[l - 1]->nforcing; }
    void mg_means();        // coarse means and their validation
    void mg_diag_blocks();  // P and its LU per coarse level
    std::vector<std::unique_ptr<MgLevel>> mg_;
    template <class S>
    void rb_solve_async(const double* shift, const RbIlu<S>& f, const S* rhs, S* x, RbControl* ctl);
    // device records of one RK step -> the reference's exceptions (stage order) + reports
    void check_step(const unsigned long long* errs, const RbControl* ctls, const LinearSolveReport* host_rep,
                    const bool* have_host, const std::string& field, RkStepResult& res,
                    const int* host_div = nullptr);
    // rk_step of harmonics hs[0..P) interleaved stage by stage, one batched sweep per stage
    void assemble_a5(cudaStream_t st);
    void harmonic_batch(const int* hs, int P, std::vector<double>& h_norm,
                        std::vector<std::vector<LinearSolveReport>>& h_reps, std::vector<std::exception_ptr>& herr);
    std::vector<double> h_norm_;
    std::vector<std::vector<LinearSolveReport>> h_reps_;

    SchemeConfig sch_;
    double sigma_ = 50.0;
    int nh_ = 0, nforcing_ = 0;
    std::vector<int> index_;
    std::vector<double> omega_;
    std::unique_ptr<DevicePattern> pat_;
    std::unique_ptr<DeviceDisc> disc_;
    std::unique_ptr<Workspace> ws_;
    DeviceBuffer<double> mean_, df_, A5_, A5s_, P_, PLU_, shift_;
    DeviceBuffer<int> Ppiv_, pcpiv_;
    DeviceBuffer<cplx> amps_, forcing_, pclu_;
    std::unique_ptr<DeviceIlu<double>> ilu_mean_;
    std::unique_ptr<DeviceIlu<cplx>> ilu_h_;
    std::unique_ptr<RbSystem> rbA_;  // 2-colour fast path (rb.cuh), null when not eligible
    std::unique_ptr<RbIlu<double>> rb_mean_;
    std::unique_ptr<RbIlu<cplx>> rb_h_;
    DeviceBuffer<RbControl> ctl_;                 // one per RK stage
    DeviceBuffer<unsigned long long> stage_err_;  // [0,5) eval, [5,10) apply, [10] deterministic flux
    DeviceBuffer<int> fac_status_;                // harmonic factorization status (deferred check)
    DeviceBuffer<cplx> rb_z_, rb_r_;
    DeviceBuffer<cplx> rk_[7];  // state0, inv, vis_fresh, vis_blend, rhs, x, stage (complex or reinterpreted real)
    std::vector<std::unique_ptr<HarmonicLane>> lanes_;  // batched harmonic path (workers > 1), else empty
    std::vector<LinearSolveReport> reports_;
    int iter_ = 0;
    int failed_h_ = -1;
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;  // kernels in the graph (the library's launch counter on replay)
        bool failed = false;     // not capturable: run launch by launch
        int calls = 0;           // the first call runs launch by launch (lazy set-up happens there)
    };
    std::unordered_map<std::string, GraphEntry> graphs_;
    // run `body` (enqueues on ws_->stream, forks/joins other streams through events) as the
    // graph cached under `key`, capturing it on first use
    template <class F>
    void captured(const std::string& key, F&& body);
    const double* ext_df_acc_ = nullptr;
    double cum_seconds_ = 0.0;
    cudaEvent_t ev0_, ev1_, evp_[3];
    cudaStream_t cs_ = nullptr;          // copy stream of outer_iteration_host
    cudaEvent_t ev_in_ = nullptr, ev_h_ = nullptr, ev_stage_ = nullptr;
    bool wait_amps_ = false;             // phase_harmonics waits on ev_in_ before the harmonics
    cplx* amps_download_ = nullptr;      // host destination of the harmonic fields (or null)
};

void harmonic_shift(const double* vol, int n, double omega, double ga, double* shift_im, cudaStream_t st);
void shifted_blocks(const double* P, const double* vol, int b, int n, double omega, cplx* out, cudaStream_t st);

}  // namespace fnlh
