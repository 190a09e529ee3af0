// capi_solver.cu -- extern "C" entry points for the discretization and the outer
// FNLH iteration (include/fnlh_b200.h).
#include <memory>
#include <vector>

#include "fnlh_b200.h"
#include "capi_util.hpp"
#include "solver.cuh"

using namespace fnlh;

struct fnlh_disc {
    std::unique_ptr<DevicePattern> pat;
    std::unique_ptr<DeviceDisc> disc;
    std::unique_ptr<Workspace> ws;
};

struct fnlh_solver {
    std::unique_ptr<DeviceSolver> s;
};

namespace {
MeshArrays arrays(const fnlh_mesh_desc* m) {
    MeshArrays a;
    a.n = m->n;
    a.nf = m->nf;
    a.b = m->b;
    a.fa = m->fa;
    a.fb = m->fb;
    a.fbc = m->fbc;
    a.ford = m->ford;
    a.fn = m->fn;
    a.farea = m->farea;
    a.fnh = m->fnh;
    a.fvis = m->fvis;
    a.vol = m->vol;
    a.closure = m->closure;
    a.mu = m->mu;
    a.nf_ptr = m->nf_ptr;
    a.nf_idx = m->nf_idx;
    a.bflag = m->bflag;
    a.gamma = m->gamma;
    a.gas_constant = m->gas_constant;
    a.p0 = m->p0;
    a.T0 = m->T0;
    a.p_out = m->p_out;
    a.nt_in = m->nt_in;
    a.forcing_scale = m->forcing_scale;
    return a;
}
}  // namespace

extern "C" {

int fnlh_disc_create(const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx, const int* partition,
                     fnlh_disc** out) {
    return guarded([&] {
        auto d = std::make_unique<fnlh_disc>();
        d->pat = std::make_unique<DevicePattern>(m->b, m->n, row_ptr, col_idx, partition);
        d->disc = std::make_unique<DeviceDisc>(arrays(m), d->pat.get());
        d->ws = std::make_unique<Workspace>((std::size_t)m->n * m->b);
        *out = d.release();
    });
}

void fnlh_disc_destroy(fnlh_disc* d) { delete d; }

int fnlh_disc_residual(fnlh_disc* d, const double* W, const double* wref, int order, int mode, const double* forcing,
                       int nforcing, int need_vis, double* inv, double* vis) {
    return guarded([&] {
        const std::size_t len = d->disc->len();
        cudaStream_t st = d->ws->stream;
        DeviceBuffer<double> w, wr, f, iv(len), vv(len);
        w.upload(W, len);
        if (wref) wr.upload(wref, len);
        if (forcing && nforcing) f.upload(forcing, nforcing);
        d->disc->reset_err(st);
        d->disc->residual(w.ptr, wref ? wr.ptr : nullptr, order, mode, f.ptr, forcing ? nforcing : 0, need_vis != 0,
                          iv.ptr, vv.ptr, st);
        d->disc->raise_if_err(st, "residual");
        download(inv, iv.ptr, len);
        if (need_vis && vis) download(vis, vv.ptr, len);
    });
}

int fnlh_disc_fd_jacobian(fnlh_disc* d, const double* W, double* J, double* P) {
    return guarded([&] {
        const std::size_t len = d->disc->len();
        const int b = d->disc->b();
        cudaStream_t st = d->ws->stream;
        DeviceBuffer<double> w, Jd, Pd;
        w.upload(W, len);
        if (J) Jd.alloc((std::size_t)d->pat->nnzb * b * b);
        if (P) Pd.alloc((std::size_t)d->disc->n() * b * b);
        d->disc->reset_err(st);
        d->disc->fd_jacobian(w.ptr, J ? Jd.ptr : nullptr, P ? Pd.ptr : nullptr, st);
        FNLH_CUDA(cudaStreamSynchronize(st));
        if (J) download(J, Jd.ptr, Jd.n);
        if (P) download(P, Pd.ptr, Pd.n);
    });
}

int fnlh_disc_linearized_residual(fnlh_disc* d, const double* mean, const double* what, double omega,
                                  const double* forcing, int nforcing, int order, int need_vis, double* inv,
                                  double* vis) {
    return guarded([&] {
        const std::size_t len = d->disc->len();
        cudaStream_t st = d->ws->stream;
        DeviceBuffer<double> mv;
        DeviceBuffer<cplx> wv, f, iv(len), vv(len);
        mv.upload(mean, len);
        wv.upload(reinterpret_cast<const cplx*>(what), len);
        if (nforcing) f.upload(reinterpret_cast<const cplx*>(forcing), nforcing);
        d->disc->reset_err(st);
        d->disc->linearized_residual(mv.ptr, wv.ptr, omega, f.ptr, nforcing, order, need_vis != 0, iv.ptr, vv.ptr, st);
        d->disc->raise_if_err(st, "linearized_residual");
        download(reinterpret_cast<cplx*>(inv), iv.ptr, len);
        if (need_vis && vis) download(reinterpret_cast<cplx*>(vis), vv.ptr, len);
    });
}

int fnlh_disc_deterministic_flux(fnlh_disc* d, const double* mean, int nh, const double* omega, const double* amps,
                                 double* df) {
    return guarded([&] {
        const std::size_t len = d->disc->len();
        cudaStream_t st = d->ws->stream;
        DeviceBuffer<double> mv, dfv(len);
        DeviceBuffer<cplx> av;
        mv.upload(mean, len);
        av.upload(reinterpret_cast<const cplx*>(amps), (std::size_t)nh * len);
        std::vector<const cplx*> ptrs;
        for (int h = 0; h < nh; ++h) ptrs.push_back(av.ptr + (std::size_t)h * len);
        d->disc->reset_err(st);
        d->disc->deterministic_flux(mv.ptr, ptrs, std::vector<double>(omega, omega + nh), dfv.ptr, st);
        FNLH_CUDA(cudaStreamSynchronize(st));
        download(df, dfv.ptr, len);
    });
}

int fnlh_solver_create(const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx, const int* partition,
                       const fnlh_scheme* s, int nh, const int* index, const double* omega, const double* forcing,
                       int nforcing, const double* mean0, fnlh_solver** out) {
    return guarded([&] {
        SchemeConfig sc;
        sc.implicit = s->implicit;
        sc.sigma_cfl = s->sigma_cfl;
        sc.eps_relax = s->eps_relax;
        sc.linear_tol = s->linear_tol;
        sc.linear_max_iter = s->linear_max_iter;
        sc.target_drop_orders = s->target_drop_orders;
        sc.max_outer_iters = s->max_outer_iters;
        sc.workers = s->workers;
        auto h = std::make_unique<fnlh_solver>();
        h->s = std::make_unique<DeviceSolver>(arrays(m), row_ptr, col_idx, partition, sc, nh, index, omega, forcing,
                                              nforcing, mean0);
        *out = h.release();
    });
}

void fnlh_solver_destroy(fnlh_solver* s) { delete s; }

int fnlh_solver_add_level(fnlh_solver* s, const fnlh_mesh_desc* m, const int* row_ptr, const int* col_idx,
                          const int* parent, const double* forcing, int nforcing) {
    return guarded([&] { s->s->add_level(arrays(m), row_ptr, col_idx, parent, forcing, nforcing); });
}

int fnlh_solver_levels(const fnlh_solver* s) { return s->s->levels(); }

int fnlh_solver_outer_iteration(fnlh_solver* s, fnlh_entry* e, double* resid_h) {
    return guarded([&] {
        ConvergenceEntry c = s->s->outer_iteration();
        *e = fnlh_entry{c.iter, c.resid_mean, c.rz, c.has_rz, c.seconds};
        if (resid_h)
            for (std::size_t k = 0; k < c.resid_h.size(); ++k) resid_h[k] = c.resid_h[k];
    });
}

int fnlh_solver_outer_iteration_host(fnlh_solver* s, const double* mean_in, const double* amps_in, double* mean_out,
                                     double* amps_out, fnlh_entry* e, double* resid_h) {
    return guarded([&] {
        ConvergenceEntry c = s->s->outer_iteration_host(mean_in, reinterpret_cast<const cplx*>(amps_in), mean_out,
                                                        reinterpret_cast<cplx*>(amps_out));
        *e = fnlh_entry{c.iter, c.resid_mean, c.rz, c.has_rz, c.seconds};
        if (resid_h)
            for (std::size_t k = 0; k < c.resid_h.size(); ++k) resid_h[k] = c.resid_h[k];
    });
}

int fnlh_solver_phase_harmonics(fnlh_solver* s, const int* owned, double* h_norm) {
    return guarded([&] {
        s->s->phase_harmonics(owned);
        const auto& hn = s->s->last_h_norm();
        if (h_norm)
            for (std::size_t h = 0; h < hn.size(); ++h) h_norm[h] = hn[h];
    });
}

void fnlh_set_graphs(int enable) { fnlh::graphs_enabled() = enable != 0; }

int fnlh_solver_df_points(fnlh_solver* s, int* nq) {
    return guarded([&] { *nq = s->s->df_points(); });
}

int fnlh_solver_df_terms(fnlh_solver* s, int k0, int k1, void* terms_dev) {
    return guarded([&] { s->s->df_terms(k0, k1, static_cast<double*>(terms_dev)); });
}

int fnlh_solver_df_accumulate(fnlh_solver* s, const void* terms_dev, int count, void* acc_dev, int first) {
    return guarded([&] {
        s->s->df_accumulate(static_cast<const double*>(terms_dev), count, static_cast<double*>(acc_dev), first != 0);
    });
}

int fnlh_solver_set_external_df(fnlh_solver* s, const void* acc_dev) {
    return guarded([&] { s->s->set_external_df(static_cast<const double*>(acc_dev)); });
}

int fnlh_solver_failed_harmonic(const fnlh_solver* s, int* h) {
    return guarded([&] { *h = s->s->failed_harmonic(); });
}

int fnlh_solver_harmonic_reports(const fnlh_solver* s, int h, fnlh_linear_report* out, int max, int* n) {
    return guarded([&] {
        const auto& hr = s->s->last_h_reports();
        if (h < 0 || h >= (int)hr.size()) throw ShapeError("harmonic_reports: index out of range");
        *n = (int)hr[h].size();
        for (int k = 0; k < *n && k < max; ++k) {
            const LinearSolveReport& r = hr[h][k];
            out[k] = fnlh_linear_report{r.iterations, r.initial_residual, r.final_residual, r.converged ? 1 : 0};
        }
    });
}

int fnlh_solver_phase_mean(fnlh_solver* s, const double* h_norm, const int* nrep, const fnlh_linear_report* reps,
                           fnlh_entry* e, double* resid_h) {
    return guarded([&] {
        const int nh = s->s->nh();
        std::vector<double> hn(h_norm, h_norm + nh);
        std::vector<std::vector<LinearSolveReport>> hr(nh);
        std::size_t q = 0;
        for (int h = 0; h < nh; ++h)
            for (int k = 0; k < nrep[h]; ++k, ++q) {
                LinearSolveReport r;
                r.iterations = reps[q].iterations;
                r.initial_residual = reps[q].initial_residual;
                r.final_residual = reps[q].final_residual;
                r.converged = reps[q].converged != 0;
                hr[h].push_back(r);
            }
        ConvergenceEntry c = s->s->phase_mean(hn, hr);
        *e = fnlh_entry{c.iter, c.resid_mean, c.rz, c.has_rz, c.seconds};
        if (resid_h)
            for (std::size_t k = 0; k < c.resid_h.size(); ++k) resid_h[k] = c.resid_h[k];
    });
}

int fnlh_solver_copy_amps(fnlh_solver* s, int h, void* dev, int to_dev) {
    return guarded([&] { s->s->copy_amps(h, dev, to_dev != 0); });
}

int fnlh_solver_run(fnlh_solver* s, int* reason, int* n_entries, fnlh_entry* entries, int max_entries) {
    return guarded([&] {
        std::vector<ConvergenceEntry> hist;
        *reason = s->s->run_to_convergence(hist);
        *n_entries = static_cast<int>(hist.size());
        for (int k = 0; k < *n_entries && k < max_entries; ++k)
            entries[k] = fnlh_entry{hist[k].iter, hist[k].resid_mean, hist[k].rz, hist[k].has_rz, hist[k].seconds};
    });
}

int fnlh_solver_get_state(const fnlh_solver* s, double* mean, double* amps) {
    return guarded([&] { s->s->get_state(mean, amps); });
}

int fnlh_solver_set_state(fnlh_solver* s, const double* mean, const double* amps) {
    return guarded([&] { s->s->set_state(mean, amps); });
}

int fnlh_solver_get_df(const fnlh_solver* s, double* df) {
    return guarded([&] { s->s->get_df(df); });
}

int fnlh_solver_unsteady(fnlh_solver* s, const double* steady, int samples_per_period, double cfl,
                         double periodic_tol, int max_periods, int min_periods, double* samples, double* info) {
    return guarded([&] {
        s->s->unsteady_solve(steady, samples_per_period, cfl, periodic_tol, max_periods, min_periods, samples, info);
    });
}

int fnlh_solver_num_reports(const fnlh_solver* s) { return static_cast<int>(s->s->reports().size()); }

int fnlh_solver_get_reports(const fnlh_solver* s, fnlh_linear_report* out) {
    const auto& r = s->s->reports();
    for (std::size_t k = 0; k < r.size(); ++k)
        out[k] = fnlh_linear_report{r[k].iterations, r[k].initial_residual, r[k].final_residual, r[k].converged};
    return 0;
}

int fnlh_solver_time_sweeps(fnlh_solver* s, int h, int sweeps, double* ms) {
    return guarded([&] { *ms = s->s->time_harmonic_sweeps(h, sweeps); });
}

int fnlh_solver_time_sweeps_batch(fnlh_solver* s, int P, int sweeps, double* ms) {
    return guarded([&] { *ms = s->s->time_harmonic_sweeps_batch(P, sweeps); });
}

int fnlh_solver_lanes(const fnlh_solver* s) { return s->s->lanes(); }

double fnlh_solver_lhs_bytes(const fnlh_solver* s) { return static_cast<double>(s->s->lhs_bytes()); }

int fnlh_solver_info(const fnlh_solver* s, double* out) {
    return guarded([&] { s->s->info(out); });
}

int fnlh_solver_counters(const fnlh_solver* s, double* out) {
    out[0] = static_cast<double>(s->s->sweeps);
    out[1] = static_cast<double>(s->s->row_updates);
    out[2] = s->s->last_iteration_ms;
    for (int k = 0; k < 4; ++k) out[3 + k] = s->s->phase_ms[k];
    return 0;
}

}  // extern "C"
