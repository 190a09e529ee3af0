// euler.cuh -- per-face / per-node physics of the 3D edge-based Euler discretization
// (b = 5, or 6 with the SA-like scalar), device side.  Operation order follows
// disc_euler.cpp / state.cpp exactly (see oracle/fnlh_oracle.c for the CPU
// restatement it is checked against); compiled with --fmad=false.
#pragma once

#include "common.cuh"
#include "libm_pow.cuh"

namespace fnlh {

// device view of the mesh + case (mirrors oracle or_mesh)
struct MeshDev {
    int n, nf, b;
    const int* __restrict__ fa;
    const int* __restrict__ fb;
    const int* __restrict__ fbc;
    const int* __restrict__ ford;
    const double* __restrict__ fn;
    const double* __restrict__ farea;
    const double* __restrict__ fnh;
    const double* __restrict__ fvis;
    const double* __restrict__ vol;
    const double* __restrict__ closure;
    const double* __restrict__ mu;
    const int* __restrict__ nf_ptr;
    const int* __restrict__ nf_idx;
    const int* __restrict__ bflag;
    double gamma, gas_constant, p0, T0, p_out, nt_in, forcing_scale;
    // per node-face incidence e (parallel to nf_idx): kBoundaryFace for a boundary face, else
    // the other endpoint j as j (this node is fa: the face flux adds) or -(j + 1) (this node
    // is fb: it subtracts) -- the gathers need no random reads of fa / fb / fbc
    const int* __restrict__ nf_code;
    // glibc's pow tables (libm_pow.cuh) or nullptr: the correctly rounded pow
    const double* __restrict__ powtab;
    // 1: the interior faces are exactly (i, i+1) -- the reference's line mesh, whose order-2
    // terms use its 1D stencil verbatim (disc_euler.cpp:113-119,145-157)
    int line;
};

constexpr int kBoundaryFace = -2147483647 - 1;

constexpr double kKappa2 = 0.5;        // disc_euler.cpp:15
constexpr double kKappa4 = 1.0 / 32.0; // disc_euler.cpp:16

// euler_prim_to_cons (state.cpp:14-19), 3D + SA-like scalar
template <int B>
__device__ __forceinline__ void prim_to_cons(const double* w, double g, double* q) {
    const double rho = w[0], u = w[1], v = w[2], ww = w[3], p = w[4];
    q[0] = rho;
    q[1] = rho * u;
    q[2] = rho * v;
    q[3] = rho * ww;
    q[4] = p / (g - 1.0) + 0.5 * rho * u * u + 0.5 * rho * v * v + 0.5 * rho * ww * ww;
    if constexpr (B == 6) q[5] = rho * w[5];
}

// euler_cons_to_prim (state.cpp:21-30); returns kState (2) on an inadmissible state
template <int B>
__device__ __forceinline__ int cons_to_prim(const double* q, double g, double* w) {
    const double rho = q[0];
    if (!(rho > 0.0)) return 2;
    const double u = q[1] / rho, v = q[2] / rho, ww = q[3] / rho;
    const double p = (g - 1.0) * (q[4] - 0.5 * rho * u * u - 0.5 * rho * v * v - 0.5 * rho * ww * ww);
    if (!(p > 0.0)) return 2;
    w[0] = rho;
    w[1] = u;
    w[2] = v;
    w[3] = ww;
    w[4] = p;
    if constexpr (B == 6) w[5] = q[5] / rho;
    return 0;
}

// euler_validate (state.cpp:7-12)
template <int B>
__device__ __forceinline__ bool admissible(const double* w) {
    if (!(w[0] > 0.0) || !(w[4] > 0.0)) return false;
#pragma unroll
    for (int k = 0; k < B; ++k)
        if (!isfinite(w[k])) return false;
    return true;
}

// phys_flux (disc_euler.cpp:105-111) as F(w).n
template <int B>
__device__ __forceinline__ void phys_flux(const double* w, double g, const double* n, double* out) {
    const double rho = w[0], u = w[1], v = w[2], ww = w[3], p = w[4];
    const double rhoE = p / (g - 1.0) + 0.5 * rho * u * u + 0.5 * rho * v * v + 0.5 * rho * ww * ww;
    const double H = rhoE + p;
    const double nx = n[0], ny = n[1], nz = n[2];
    out[0] = rho * u * nx + rho * v * ny + rho * ww * nz;
    out[1] = (rho * u * u + p) * nx + rho * v * u * ny + rho * ww * u * nz;
    out[2] = rho * u * v * nx + (rho * v * v + p) * ny + rho * ww * v * nz;
    out[3] = rho * u * ww * nx + rho * v * ww * ny + (rho * ww * ww + p) * nz;
    out[4] = u * H * nx + v * H * ny + ww * H * nz;
    if constexpr (B == 6) out[5] = rho * u * w[5] * nx + rho * v * w[5] * ny + rho * ww * w[5] * nz;
}

struct BState {
    double w[6];
    double un;
    double vt[3];
};

// steady_inlet_state (disc_euler.cpp:161-182) along the inward normal; 0 ok, 2 State, 4 Unsupported
__device__ __forceinline__ int steady_inlet(const MeshDev& m, const double* wint, const double* nh, BState& s) {
    const double g = m.gamma, R = m.gas_constant;
    const double gp = 0.5 * (g - 1.0);
    const double c_int = sqrt(g * wint[4] / wint[0]);
    const double un_in = -(wint[1] * nh[0] + wint[2] * nh[1] + wint[3] * nh[2]);
    const double jm = un_in - c_int / gp;
    const double c0sq = g * R * m.T0;
    const double qa = gp * gp + gp;
    const double qb = -2.0 * gp * gp * jm;
    const double qc = gp * gp * jm * jm - c0sq;
    const double disc = qb * qb - 4.0 * qa * qc;
    if (disc < 0.0) return 2;
    const double ub = (-qb + sqrt(disc)) / (2.0 * qa);
    const double cb = gp * (ub - jm);
    if (!(cb > 0.0)) return 2;
    if (fabs(ub) >= cb) return 4;
    const double tb = cb * cb / (g * R);
    const double pb = m.p0 * bc_pow(m.powtab, tb / m.T0, g / (g - 1.0));
    s.w[0] = pb / (R * tb);
    s.w[1] = ub * -nh[0];
    s.w[2] = ub * -nh[1];
    s.w[3] = ub * -nh[2];
    s.w[4] = pb;
    s.w[5] = m.nt_in;
    s.un = ub;
    return 0;
}

// steady_outlet_state (disc_euler.cpp:184-193) along the outward normal
template <int B>
__device__ __forceinline__ int steady_outlet(const MeshDev& m, const double* wint, const double* nh, BState& s) {
    const double g = m.gamma;
    const double pb = m.p_out;
    const double rhob = wint[0] * bc_pow(m.powtab, pb / wint[4], 1.0 / g);
    const double cb = sqrt(g * pb / rhob);
    const double c_int = sqrt(g * wint[4] / wint[0]);
    const double un = wint[1] * nh[0] + wint[2] * nh[1] + wint[3] * nh[2];
    const double ubn = un + 2.0 / (g - 1.0) * (c_int - cb);
    if (fabs(ubn) >= cb) return 4;
#pragma unroll
    for (int d = 0; d < 3; ++d) s.vt[d] = wint[1 + d] - un * nh[d];
    s.w[0] = rhob;
#pragma unroll
    for (int d = 0; d < 3; ++d) s.w[1 + d] = s.vt[d] + ubn * nh[d];
    s.w[4] = pb;
    if constexpr (B == 6) s.w[5] = wint[5];
    s.un = ubn;
    return 0;
}

// boundary_state (disc_euler.cpp:195-230); mode 0 Steady, 1 Perturbation
template <int B>
__device__ __forceinline__ int boundary_state(const MeshDev& m, int f, const double* wint, const double* wref,
                                              int mode, const double* forcing, int nforcing, double* wb) {
    const double* nh = m.fnh + 3 * (size_t)f;
    const bool west = m.fbc[f] == 0;
    int st;
    if (mode == 0) {
        BState s;
        st = west ? steady_inlet(m, wint, nh, s) : steady_outlet<B>(m, wint, nh, s);
        if (st) return st;
#pragma unroll
        for (int k = 0; k < B; ++k) wb[k] = s.w[k];
        return 0;
    }
    BState br;
    st = west ? steady_inlet(m, wref, nh, br) : steady_outlet<B>(m, wref, nh, br);
    if (st) return st;
    const double g = m.gamma;
    const double cbar = sqrt(g * br.w[4] / br.w[0]);
    const double rc = br.w[0] * cbar;
    const double drho = wint[0] - wref[0];
    double du[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) du[d] = wint[1 + d] - wref[1 + d];
    const double dp = wint[4] - wref[4];
    const int o = m.ford[f];
    auto fval = [&](int k) { return (3 * o + k) < nforcing ? forcing[3 * o + k] : 0.0; };
    double c_entropy, c_plus, c_minus, du_n;
    if (west) {
        du_n = -(du[0] * nh[0] + du[1] * nh[1] + du[2] * nh[2]);
        c_minus = dp - rc * du_n;
        c_entropy = fval(0);
        c_plus = 2.0 * fval(1);
    } else {
        du_n = du[0] * nh[0] + du[1] * nh[1] + du[2] * nh[2];
        c_entropy = drho - dp / (cbar * cbar);
        c_plus = dp + rc * du_n;
        c_minus = 2.0 * fval(2);
    }
    const double dpb = 0.5 * (c_plus + c_minus);
    const double dub = (c_plus - c_minus) / (2.0 * rc);
    const double drhob = c_entropy + dpb / (cbar * cbar);
    wb[0] = br.w[0] + drhob;
    if (west) {
#pragma unroll
        for (int d = 0; d < 3; ++d) wb[1 + d] = (br.un + dub) * -nh[d];
    } else {
#pragma unroll
        for (int d = 0; d < 3; ++d) wb[1 + d] = (br.vt[d] + (du[d] - du_n * nh[d])) + (br.un + dub) * nh[d];
    }
    wb[4] = br.w[4] + dpb;
    if constexpr (B == 6) wb[5] = west ? br.w[5] : br.w[5] + (wint[5] - wref[5]);
    return 0;
}

// boundary_face_flux (disc_euler.cpp:232-239)
template <int B>
__device__ __forceinline__ int boundary_face_flux(const MeshDev& m, int f, const double* wint, const double* wref,
                                                  int mode, const double* forcing, int nforcing, double* out) {
    double wb[6];
    const int st = boundary_state<B>(m, f, wint, wref, mode, forcing, nforcing, wb);
    if (st) return st;
    phys_flux<B>(wb, m.gamma, m.fn + 3 * (size_t)f, out);
    return 0;
}

// interior_face_flux (disc_euler.cpp:121-159); order 2 takes the node pre-pass values.
// The core takes the face geometry by value (n, nh, area: global or register copies).
template <int B>
__device__ __forceinline__ void interior_flux_core(double g, const double* n, const double* nh, double area,
                                                   const double* wa, const double* wc, int order, double nua,
                                                   double nub, bool trunc, const double* lapa, const double* lapc,
                                                   double* out, bool line = false) {
    double fa[6], fb[6], qa[6], qb[6];
    phys_flux<B>(wa, g, n, fa);
    phys_flux<B>(wc, g, n, fb);
    const double rho = 0.5 * (wa[0] + wc[0]);
    const double u = 0.5 * (wa[1] + wc[1]);
    const double v = 0.5 * (wa[2] + wc[2]);
    const double ww = 0.5 * (wa[3] + wc[3]);
    const double p = 0.5 * (wa[4] + wc[4]);
    const double cs = sqrt(g * p / rho);
    const double lam = (fabs(u * nh[0] + v * nh[1] + ww * nh[2]) + cs) * area;
    prim_to_cons<B>(wa, g, qa);
    prim_to_cons<B>(wc, g, qb);
#pragma unroll
    for (int k = 0; k < B; ++k) out[k] = 0.5 * (fa[k] + fb[k]);
    if (order == 1) {
#pragma unroll
        for (int k = 0; k < B; ++k) out[k] -= 0.5 * lam * (qb[k] - qa[k]);
        return;
    }
    const double s2 = kKappa2 * (nua > nub ? nua : nub);
    double s4 = kKappa4 - s2;
    if (!(s4 > 0.0)) s4 = 0.0;
    if (trunc) s4 = 0.0;
    if (line) {  // lapa = Q(a-1), lapc = Q(b+1): the 1D 4th difference (disc_euler.cpp:150-155)
#pragma unroll
        for (int k = 0; k < B; ++k) {
            double d = s2 * lam * (qb[k] - qa[k]);
            if (s4 > 0.0) d -= s4 * lam * (lapc[k] - 3.0 * qb[k] + 3.0 * qa[k] - lapa[k]);
            out[k] -= d;
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
        double d = s2 * lam * (qb[k] - qa[k]);
        if (s4 > 0.0) d -= s4 * lam * (lapc[k] - lapa[k]);
        out[k] -= d;
    }
}

template <int B>
__device__ __forceinline__ void interior_face_flux(const MeshDev& m, int f, const double* wa, const double* wc,
                                                   int order, double nua, double nub, bool trunc,
                                                   const double* lapa, const double* lapc, double* out,
                                                   bool line = false) {
    interior_flux_core<B>(m.gamma, m.fn + 3 * (size_t)f, m.fnh + 3 * (size_t)f, m.farea[f], wa, wc, order, nua, nub,
                          trunc, lapa, lapc, out, line);
}

// SA-like viscous flux (b = 6 only)
template <int B>
__device__ __forceinline__ void viscous_face_flux(const MeshDev& m, int f, const double* wa, const double* wc,
                                                  double mua, double muc, double* out) {
    const double k = 0.5 * (mua + muc) * m.fvis[f];
    out[0] = 0.0;
    out[1] = -k * (wc[1] - wa[1]);
    out[2] = -k * (wc[2] - wa[2]);
    out[3] = -k * (wc[3] - wa[3]);
    out[4] = 0.0;
    if constexpr (B == 6) out[5] = -k * (wc[5] - wa[5]);
}

// node_source (disc_euler.cpp:95-100): slip-wall closure -p * sum(outward normals)
template <int B>
__device__ __forceinline__ void node_source(const MeshDev& m, int i, double p, double* out) {
#pragma unroll
    for (int k = 0; k < B; ++k) out[k] = 0.0;
    out[1] = -p * m.closure[3 * (size_t)i + 0];
    out[2] = -p * m.closure[3 * (size_t)i + 1];
    out[3] = -p * m.closure[3 * (size_t)i + 2];
}

}  // namespace fnlh
