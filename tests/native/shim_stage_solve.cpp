// shim_stage_solve.cpp -- a reference-typed unit using the drop-in at the reference's call
// sites (include/fnlh_b200_shim.hpp) next to the reference's own path, on the same
// reference objects.  TEST INFRASTRUCTURE: built by oracle/Makefile against the reference
// headers and oracle/_ref/libfnlh_ref.so (the unmodified reference), run by
// tests/test_gpu_shim.py on the GPU.
//
// For a 2-colour (colour-major) and a general (level-scheduled) pattern, b = 5:
//   reference: A5 (Bsr<real>) -> build_lhs_harmonic-equivalent shift_diagonal -> Ilu<cplx>
//              factorize once -> smoothed_solve per RK stage (driver.cpp:213-216, rk.cpp:82-85);
//              Ilu<real> factorize + smoothed_solve for the mean flow (driver.cpp:180-181)
//   drop-in:   LhsB200 (A5 uploaded once) -> IluB200<cplx>::factorize(harmonic_shift_b200)
//              once -> smoothed_solve_b200 per stage; IluB200<real> for the mean
// and checks: iterates bitwise equal, iteration counts and convergence flags equal, norms
// within 1e-14, the device bytes registered with the reference's LHS accounting
// (lhs_alloc_stats) while the handles live and released after, and that a stage solve
// launches only sweep kernels (no upload, no refactorization).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "fnlh_b200_shim.hpp"

using namespace fnlh;

namespace {

int failures = 0;
#define CHECK(cond, ...)                    \
    do {                                    \
        if (!(cond)) {                      \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");              \
            ++failures;                     \
        }                                   \
    } while (0)

// nx*ny*nz grid; coloured: 2-colour colour-major order; else natural order plus one diagonal
// edge per cell face pair (not 2-colourable: the general level-scheduled path)
PatternPtr grid_pattern(int nx, int ny, int nz, bool coloured, std::vector<int>& order_out) {
    const int n = nx * ny * nz;
    std::vector<int> rank(n);
    int c0 = 0;
    for (int i = 0; i < n; ++i) {
        const int x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
        if ((x + y + z) % 2 == 0) ++c0;
    }
    int a = 0, bb = c0;
    for (int i = 0; i < n; ++i) {
        const int x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
        rank[i] = !coloured ? i : ((x + y + z) % 2 == 0 ? a++ : bb++);
    }
    std::vector<std::pair<int, int>> edges;
    for (int i = 0; i < n; ++i) {
        const int x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
        if (x + 1 < nx) edges.push_back({rank[i], rank[i + 1]});
        if (y + 1 < ny) edges.push_back({rank[i], rank[i + nx]});
        if (z + 1 < nz) edges.push_back({rank[i], rank[i + nx * ny]});
        if (!coloured && x + 1 < nx && y + 1 < ny) edges.push_back({rank[i], rank[i + 1 + nx]});
    }
    order_out = rank;
    return make_pattern(5, n, edges, {});
}

void fill(Bsr<real>& A, std::mt19937_64& g) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const auto& p = *A.pattern;
    const int b = p.b;
    for (int i = 0; i < p.rows; ++i)
        for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
            real* blk = A.block(e);
            const bool diag = p.col_idx[e] == i;
            for (int r = 0; r < b; ++r)
                for (int c = 0; c < b; ++c) blk[r * b + c] = (diag ? (r == c ? 8.0 : 0.0) : 0.0) + 0.3 * u(g);
        }
}

template <class S>
BlockVec<S> random_vec(int b, int n, std::mt19937_64& g) {
    std::normal_distribution<double> d;
    BlockVec<S> v(b, n);
    for (auto& x : v.v) {
        if constexpr (std::is_same_v<S, cplx>)
            x = cplx(d(g), d(g));
        else
            x = d(g);
    }
    return v;
}

template <class S>
void compare(const char* what, const LinearSolveReport& rr, const BlockVec<S>& xr, const LinearSolveReport& rd,
             const BlockVec<S>& xd) {
    bool same = xr.v.size() == xd.v.size();
    for (std::size_t k = 0; same && k < xr.v.size(); ++k) same = xr.v[k] == xd.v[k];
    CHECK(same, "%s: iterates differ", what);
    CHECK(rr.iterations == rd.iterations && rr.converged == rd.converged, "%s: iterations %d/%d converged %d/%d",
          what, rr.iterations, rd.iterations, int(rr.converged), int(rd.converged));
    CHECK(std::abs(rr.initial_residual - rd.initial_residual) <= 1e-14 * rr.initial_residual &&
              std::abs(rr.final_residual - rd.final_residual) <= 1e-14 * rr.final_residual,
          "%s: norms %.17g/%.17g %.17g/%.17g", what, rr.initial_residual, rd.initial_residual, rr.final_residual,
          rd.final_residual);
}

void run(bool coloured) {
    const char* tag = coloured ? "2-colour" : "general";
    std::vector<int> order;
    PatternPtr pat = grid_pattern(12, 10, 8, coloured, order);
    const int n = pat->rows, b = pat->b;
    std::mt19937_64 g(coloured ? 11 : 13);
    Bsr<real> A5(pat);
    fill(A5, g);
    Mesh mesh;
    mesh.volume.resize(n);
    std::uniform_real_distribution<double> uv(0.5, 2.0);
    for (auto& v : mesh.volume) v = uv(g);
    RKConfig rk;  // implicit, eps_relax 0.6: Gamma alpha_5 = 1/0.6
    const real omega = 2.0 * 3.14159265358979323846 * 3.0;
    const real tol = 1e-3;
    const int max_iter = 6;

    // the reference: the complex workspace materialized, factorized once, solved per stage
    const std::vector<real> shift = harmonic_shift_b200(mesh, omega, rk, 5);
    std::vector<cplx> s(n);
    for (int i = 0; i < n; ++i) s[i] = cplx(0.0, shift[i]);
    Bsr<cplx> M;
    shift_diagonal(A5, s, M);
    Ilu<cplx> ilu;
    ilu.factorize(M);
    Ilu<real> ilu_mean;
    ilu_mean.factorize(A5);

    const LhsAllocStats before = lhs_alloc_stats();
    long long stage_launches = 0, oneshot_launches = 0;
    {
        PatternB200 p(*pat);
        LhsB200 a5(p, A5);                 // uploaded once
        IluB200<cplx> worker(a5);          // one harmonic worker's workspace
        IluB200<real> mean(a5);
        long long lb = 0, pb = 0, mb = 0;
        fnlh_lhs_bytes(a5.handle(), &lb);
        fnlh_prec_bytes(worker.handle(), &pb);
        fnlh_prec_bytes(mean.handle(), &mb);
        const LhsAllocStats live = lhs_alloc_stats();
        CHECK(live.live_bytes - before.live_bytes == static_cast<std::size_t>(lb + pb + mb) && lb > 0 && pb > 0,
              "%s: LHS accounting %zu vs %lld", tag, live.live_bytes - before.live_bytes, lb + pb + mb);
        worker.factorize(shift);           // driver.cpp:213-216, once per harmonic
        mean.factorize();
        for (int k = 1; k <= 5; ++k) {     // rk.cpp:82-85, once per stage
            const BlockVec<cplx> rhs = random_vec<cplx>(b, n, g);
            BlockVec<cplx> xr, xd;
            const LinearSolveReport rr = smoothed_solve(M, rhs, ilu, tol, max_iter, xr);
            const long long l0 = fnlh_launch_count();
            const LinearSolveReport rd = smoothed_solve_b200(worker, rhs, tol, max_iter, xd);
            stage_launches = fnlh_launch_count() - l0;
            char what[64];
            std::snprintf(what, sizeof what, "%s harmonic stage %d", tag, k);
            compare(what, rr, xr, rd, xd);
            if (k == 5) {  // the one-shot form re-uploads and refactorizes per call
                BlockVec<cplx> xo;
                const long long l1 = fnlh_launch_count();
                smoothed_solve_b200(p, A5, std::span<const real>(shift), tol, max_iter, rhs, xo);
                oneshot_launches = fnlh_launch_count() - l1;
                compare("one-shot", rr, xr, rd, xo);
            }
        }
        const BlockVec<real> rhs = random_vec<real>(b, n, g);
        BlockVec<real> xr, xd;
        const LinearSolveReport rr = smoothed_solve(A5, rhs, ilu_mean, tol, max_iter, xr);
        const LinearSolveReport rd = smoothed_solve_b200(mean, rhs, tol, max_iter, xd);
        compare(coloured ? "2-colour mean" : "general mean", rr, xr, rd, xd);
    }
    const LhsAllocStats after = lhs_alloc_stats();
    CHECK(after.live_bytes == before.live_bytes, "%s: LHS bytes not released", tag);
    CHECK(stage_launches > 0 && stage_launches < oneshot_launches,
          "%s: a stage solve launched %lld kernels, the one-shot form %lld", tag, stage_launches, oneshot_launches);
    std::printf("%s: n=%d nnzb=%d stage solve %lld launches (one-shot %lld)\n", tag, n, pat->nnzb(),
                stage_launches, oneshot_launches);
}

}  // namespace

int main() {
    try {
        run(true);
        run(false);
    } catch (const std::exception& e) {
        std::printf("FAIL: exception %s\n", e.what());
        return 2;
    }
    std::printf(failures ? "FAILED %d\n" : "OK\n", failures);
    return failures ? 1 : 0;
}
