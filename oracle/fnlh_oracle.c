/*
 * fnlh_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 * CPU restatement of the reference FNLH hot path; see fnlh_oracle.h.
 * Build: gcc -std=gnu11 -O2 -ffp-contract=off -fPIC -shared (no -march), see oracle/Makefile.
 */
#include "fnlh_oracle.h"

#include <pthread.h>
#include "cr_pow.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread or_error g_err; /* per thread: harmonic workers copy theirs out */
static int g_cr_pow = 0; /* 0: glibc pow (reference), 1: correctly rounded (device) */

void or_set_pow_mode(int cr) { g_cr_pow = cr; }
double or_cr_pow(double x, double y) { return cr_pow(x, y); }
static inline double bc_pow(double x, double y) { return g_cr_pow ? cr_pow(x, y) : pow(x, y); }

const or_error* or_last_error(void) { return &g_err; }

static int or_fail(int code, int node, int stage, const char* msg) {
    g_err.code = code;
    g_err.node = node;
    g_err.stage = stage;
    snprintf(g_err.msg, sizeof g_err.msg, "%s", msg);
    return code;
}

/* ---------------------------------------------------------------------------
 * Generic block LA, real and complex (dense.hpp, sparse.hpp/.cpp)
 * ------------------------------------------------------------------------- */
#define S double
#define SUF d
#define ILU_T or_ilu_d
#define ABS(x) fabs(x)
#define SQR(x) ((x) * (x))
#define FINITE(x) isfinite(x)
#include "la_tmpl.inc"
#undef S
#undef SUF
#undef ILU_T
#undef ABS
#undef SQR
#undef FINITE

static inline double cnorm_sq(ocplx z) { return creal(z) * creal(z) + cimag(z) * cimag(z); }
static inline int cfinite(ocplx z) { return isfinite(creal(z)) && isfinite(cimag(z)); }

#define S ocplx
#define SUF z
#define ILU_T or_ilu_z
#define ABS(x) cabs(x)
/* std::norm(complex) = re*re + im*im (core.hpp:106-110) */
#define SQR(x) cnorm_sq(x)
#define FINITE(x) cfinite(x)
#include "la_tmpl.inc"
#undef S
#undef SUF
#undef ILU_T
#undef ABS
#undef SQR
#undef FINITE

/* build_lhs_mean (rk.cpp:5-30) with RKConfig alpha (rk.hpp:27) and gamma_factor (rk.hpp:34) */
static const double kAlpha[5] = {1.0 / 4.0, 1.0 / 6.0, 3.0 / 8.0, 1.0 / 2.0, 1.0};
static const double kBeta[5] = {1.0, 0.0, 14.0 / 25.0, 0.0, 11.0 / 25.0};

static double gamma_factor(int implicit, double sigma_cfl, double eps_relax) {
    return implicit ? 1.0 / eps_relax : sigma_cfl;
}

int or_build_lhs_mean(const or_pattern* p, const double* J, int implicit, double sigma_cfl,
                      double eps_relax, int stage_k, double* A) {
    if (stage_k < 1 || stage_k > 5) return or_fail(OR_CONFIG, -1, -1, "stage index must be in 1..5");
    const double ga = gamma_factor(implicit, sigma_cfl, eps_relax) * kAlpha[stage_k - 1];
    const size_t bb = (size_t)p->b * p->b;
    if (!implicit) {
        memset(A, 0, (size_t)p->nnzb * bb * sizeof(double));
        for (int i = 0; i < p->rows; ++i) {
            const double* pp = J + (size_t)p->diag_idx[i] * bb;
            double* d = A + (size_t)p->diag_idx[i] * bb;
            for (size_t k = 0; k < bb; ++k) d[k] = pp[k] / ga;
        }
        return OR_OK;
    }
    const double inv_es = 1.0 / (eps_relax * sigma_cfl);
    for (size_t k = 0; k < (size_t)p->nnzb * bb; ++k) A[k] = J[k] / ga;
    for (int i = 0; i < p->rows; ++i) {
        const double* pp = J + (size_t)p->diag_idx[i] * bb;
        double* d = A + (size_t)p->diag_idx[i] * bb;
        for (size_t k = 0; k < bb; ++k) d[k] += pp[k] * inv_es / ga;
    }
    return OR_OK;
}

/* shift_diagonal (sparse.cpp:157-171) */
void or_shift_diagonal(const or_pattern* p, const double* A, const ocplx* s, ocplx* out) {
    const int bs = p->b;
    const size_t bb = (size_t)bs * bs;
    const size_t total = (size_t)p->nnzb * bb;
    for (size_t k = 0; k < total; ++k) out[k] = CMPLX(A[k], 0.0);
    for (int i = 0; i < p->rows; ++i) {
        ocplx* d = out + (size_t)p->diag_idx[i] * bb;
        for (int m = 0; m < bs; ++m) d[(size_t)m * bs + m] += s[i];
    }
}

/* ---------------------------------------------------------------------------
 * State conversions (state.cpp:14-44, generalized to 3D + SA-like scalar)
 * W = (rho, u, v, w, p[, nt]);  Q = (rho, rho u, rho v, rho w, rho E[, rho nt])
 * ------------------------------------------------------------------------- */
static int euler_validate(int b, const double* w) { /* state.cpp:7-12 */
    if (!(w[0] > 0.0) || !(w[4] > 0.0)) return or_fail(OR_STATE, -1, -1, "inadmissible Euler state");
    for (int m = 0; m < b; ++m)
        if (!isfinite(w[m])) return or_fail(OR_STATE, -1, -1, "inadmissible Euler state");
    return OR_OK;
}

static inline void e_prim_to_cons(int b, const double* w, double g, double* q) { /* state.cpp:14-19 */
    const double rho = w[0], u = w[1], v = w[2], ww = w[3], p = w[4];
    q[0] = rho;
    q[1] = rho * u;
    q[2] = rho * v;
    q[3] = rho * ww;
    q[4] = p / (g - 1.0) + 0.5 * rho * u * u + 0.5 * rho * v * v + 0.5 * rho * ww * ww;
    if (b == 6) q[5] = rho * w[5];
}

static inline int e_cons_to_prim(int b, const double* q, double g, double* w) { /* state.cpp:21-30 */
    const double rho = q[0];
    if (!(rho > 0.0)) return or_fail(OR_STATE, -1, -1, "conservative state with nonpositive density");
    const double u = q[1] / rho, v = q[2] / rho, ww = q[3] / rho;
    const double p = (g - 1.0) * (q[4] - 0.5 * rho * u * u - 0.5 * rho * v * v - 0.5 * rho * ww * ww);
    if (!(p > 0.0)) return or_fail(OR_STATE, -1, -1, "conservative state with nonpositive pressure");
    w[0] = rho;
    w[1] = u;
    w[2] = v;
    w[3] = ww;
    w[4] = p;
    if (b == 6) w[5] = q[5] / rho;
    return OR_OK;
}

int or_prim_to_cons(int b, int n, double gamma, const double* W, double* Q) { /* state.cpp:59-71 */
    for (int i = 0; i < n; ++i) {
        int st = euler_validate(b, W + (size_t)i * b);
        if (st) return st;
        e_prim_to_cons(b, W + (size_t)i * b, gamma, Q + (size_t)i * b);
    }
    return OR_OK;
}

int or_cons_to_prim(int b, int n, double gamma, const double* Q, double* W) { /* state.cpp:73-80 */
    for (int i = 0; i < n; ++i) {
        int st = e_cons_to_prim(b, Q + (size_t)i * b, gamma, W + (size_t)i * b);
        if (st) return st;
    }
    return OR_OK;
}

/* euler_transform_jacobian (state.cpp:32-44): row-major M = dQ/dW */
int or_transform_jacobian(int b, int n, double gamma, const double* W, double* M) {
    for (int i = 0; i < n; ++i) {
        const double* w = W + (size_t)i * b;
        int st = euler_validate(b, w);
        if (st) return st;
        double* Mi = M + (size_t)i * b * b;
        memset(Mi, 0, sizeof(double) * b * b);
        const double rho = w[0], u = w[1], v = w[2], ww = w[3];
        Mi[0 * b + 0] = 1.0;
        Mi[1 * b + 0] = u;
        Mi[1 * b + 1] = rho;
        Mi[2 * b + 0] = v;
        Mi[2 * b + 2] = rho;
        Mi[3 * b + 0] = ww;
        Mi[3 * b + 3] = rho;
        Mi[4 * b + 0] = 0.5 * u * u + 0.5 * v * v + 0.5 * ww * ww;
        Mi[4 * b + 1] = rho * u;
        Mi[4 * b + 2] = rho * v;
        Mi[4 * b + 3] = rho * ww;
        Mi[4 * b + 4] = 1.0 / (gamma - 1.0);
        if (b == 6) {
            Mi[5 * b + 0] = w[5];
            Mi[5 * b + 5] = rho;
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * 3D edge-based Euler discretization (restates disc_euler.cpp)
 * ------------------------------------------------------------------------- */
static const double kKappa2 = 0.5;        /* disc_euler.cpp:15 */
static const double kKappa4 = 1.0 / 32.0; /* disc_euler.cpp:16 */

/* phys_flux (disc_euler.cpp:105-111) as F(w).n */
static inline void phys_flux(int b, const double* w, double g, const double* n, double* out) {
    const double rho = w[0], u = w[1], v = w[2], ww = w[3], p = w[4];
    const double rhoE = p / (g - 1.0) + 0.5 * rho * u * u + 0.5 * rho * v * v + 0.5 * rho * ww * ww;
    const double H = rhoE + p;
    const double nx = n[0], ny = n[1], nz = n[2];
    out[0] = rho * u * nx + rho * v * ny + rho * ww * nz;
    out[1] = (rho * u * u + p) * nx + rho * v * u * ny + rho * ww * u * nz;
    out[2] = rho * u * v * nx + (rho * v * v + p) * ny + rho * ww * v * nz;
    out[3] = rho * u * ww * nx + rho * v * ww * ny + (rho * ww * ww + p) * nz;
    out[4] = u * H * nx + v * H * ny + ww * H * nz;
    if (b == 6) out[5] = rho * u * w[5] * nx + rho * v * w[5] * ny + rho * ww * w[5] * nz;
}

typedef struct {
    double w[6];   /* boundary primitive state */
    double un;     /* scalar normal speed (inlet: inward, outlet: outward) */
    double vt[3];  /* outlet tangential velocity */
} bstate;

/* steady_inlet_state (disc_euler.cpp:161-182) along the inward face normal */
static int steady_inlet(const or_mesh* m, const double* wint, const double* nh, bstate* s) {
    const double g = m->gamma, R = m->gas_constant;
    const double gp = 0.5 * (g - 1.0);
    const double c_int = sqrt(g * wint[4] / wint[0]);
    const double un_in = -(wint[1] * nh[0] + wint[2] * nh[1] + wint[3] * nh[2]);
    const double jm = un_in - c_int / gp;
    const double c0sq = g * R * m->T0;
    const double qa = gp * gp + gp;
    const double qb = -2.0 * gp * gp * jm;
    const double qc = gp * gp * jm * jm - c0sq;
    const double disc = qb * qb - 4.0 * qa * qc;
    if (disc < 0.0) return or_fail(OR_STATE, -1, -1, "inlet characteristic reconstruction failed");
    const double ub = (-qb + sqrt(disc)) / (2.0 * qa);
    const double cb = gp * (ub - jm);
    if (!(cb > 0.0)) return or_fail(OR_STATE, -1, -1, "inlet boundary state has nonpositive sound speed");
    if (fabs(ub) >= cb) return or_fail(OR_UNSUPPORTED, -1, -1, "supersonic inlet boundary state");
    const double tb = cb * cb / (g * R);
    const double pb = m->p0 * bc_pow(tb / m->T0, g / (g - 1.0));
    s->w[0] = pb / (R * tb);
    s->w[1] = ub * -nh[0];
    s->w[2] = ub * -nh[1];
    s->w[3] = ub * -nh[2];
    s->w[4] = pb;
    s->w[5] = m->nt_in;
    s->un = ub;
    return OR_OK;
}

/* steady_outlet_state (disc_euler.cpp:184-193) along the outward face normal */
static int steady_outlet(const or_mesh* m, const double* wint, const double* nh, bstate* s) {
    const double g = m->gamma;
    const double pb = m->p_out;
    const double rhob = wint[0] * bc_pow(pb / wint[4], 1.0 / g);
    const double cb = sqrt(g * pb / rhob);
    const double c_int = sqrt(g * wint[4] / wint[0]);
    const double un = wint[1] * nh[0] + wint[2] * nh[1] + wint[3] * nh[2];
    const double ubn = un + 2.0 / (g - 1.0) * (c_int - cb);
    if (fabs(ubn) >= cb) return or_fail(OR_UNSUPPORTED, -1, -1, "supersonic outlet boundary state");
    for (int d = 0; d < 3; ++d) s->vt[d] = wint[1 + d] - un * nh[d];
    s->w[0] = rhob;
    for (int d = 0; d < 3; ++d) s->w[1 + d] = s->vt[d] + ubn * nh[d];
    s->w[4] = pb;
    s->w[5] = wint[5 < m->b ? 5 : 0];
    s->un = ubn;
    return OR_OK;
}

/* boundary_state (disc_euler.cpp:195-230) */
static int boundary_state(const or_mesh* m, int f, const double* W, const double* wref, int mode,
                          const double* forcing, int nforcing, double* wb) {
    const int b = m->b;
    const int a = m->fa[f];
    const double* wint = W + (size_t)a * b;
    const double* nh = m->fnh + 3 * (size_t)f;
    const int west = m->fbc[f] == 0;
    bstate s;
    int st;
    if (mode == 0) {
        st = west ? steady_inlet(m, wint, nh, &s) : steady_outlet(m, wint, nh, &s);
        if (st) return st;
        for (int k = 0; k < b; ++k) wb[k] = s.w[k];
        return OR_OK;
    }
    const double* wr = wref + (size_t)a * b;
    bstate br;
    st = west ? steady_inlet(m, wr, nh, &br) : steady_outlet(m, wr, nh, &br);
    if (st) return st;
    const double g = m->gamma;
    const double cbar = sqrt(g * br.w[4] / br.w[0]);
    const double rc = br.w[0] * cbar;
    const double drho = wint[0] - wr[0];
    double du[3];
    for (int d = 0; d < 3; ++d) du[d] = wint[1 + d] - wr[1 + d];
    const double dp = wint[4] - wr[4];
    const int o = m->ford[f];
#define FVAL(k) ((3 * o + (k)) < nforcing ? forcing[3 * o + (k)] : 0.0)
    double c_entropy, c_plus, c_minus, du_n;
    if (west) {
        du_n = -(du[0] * nh[0] + du[1] * nh[1] + du[2] * nh[2]);
        c_minus = dp - rc * du_n;
        c_entropy = FVAL(0);
        c_plus = 2.0 * FVAL(1);
    } else {
        du_n = du[0] * nh[0] + du[1] * nh[1] + du[2] * nh[2];
        c_entropy = drho - dp / (cbar * cbar);
        c_plus = dp + rc * du_n;
        c_minus = 2.0 * FVAL(2);
    }
#undef FVAL
    const double dpb = 0.5 * (c_plus + c_minus);
    const double dub = (c_plus - c_minus) / (2.0 * rc);
    const double drhob = c_entropy + dpb / (cbar * cbar);
    wb[0] = br.w[0] + drhob;
    if (west) {
        for (int d = 0; d < 3; ++d) wb[1 + d] = (br.un + dub) * -nh[d];
    } else {
        for (int d = 0; d < 3; ++d) wb[1 + d] = (br.vt[d] + (du[d] - du_n * nh[d])) + (br.un + dub) * nh[d];
    }
    wb[4] = br.w[4] + dpb;
    if (b == 6) wb[5] = west ? br.w[5] : br.w[5] + (wint[5] - wr[5]);
    return OR_OK;
}

/* boundary_face_flux (disc_euler.cpp:232-239); the normal is outward */
static int boundary_face_flux(const or_mesh* m, int f, const double* W, const double* wref, int mode,
                              const double* forcing, int nforcing, double* out) {
    double wb[6];
    int st = boundary_state(m, f, W, wref, mode, forcing, nforcing, wb);
    if (st) return st;
    phys_flux(m->b, wb, m->gamma, m->fn + 3 * (size_t)f, out);
    return OR_OK;
}

/* interior_face_flux (disc_euler.cpp:121-159); nu/lap are the node pre-pass (order 2) */
static void interior_face_flux(const or_mesh* m, int f, const double* W, int order, const double* nu,
                               const double* lap, int line, double* out) {
    const int b = m->b;
    const double g = m->gamma;
    const int a = m->fa[f], c = m->fb[f];
    const double* wa = W + (size_t)a * b;
    const double* wc = W + (size_t)c * b;
    const double* n = m->fn + 3 * (size_t)f;
    const double* nh = m->fnh + 3 * (size_t)f;
    double fa[6], fb[6], qa[6], qb[6];
    phys_flux(b, wa, g, n, fa);
    phys_flux(b, wc, g, n, fb);
    const double rho = 0.5 * (wa[0] + wc[0]);
    const double u = 0.5 * (wa[1] + wc[1]);
    const double v = 0.5 * (wa[2] + wc[2]);
    const double ww = 0.5 * (wa[3] + wc[3]);
    const double p = 0.5 * (wa[4] + wc[4]);
    const double cs = sqrt(g * p / rho);
    const double lam = (fabs(u * nh[0] + v * nh[1] + ww * nh[2]) + cs) * m->farea[f];
    e_prim_to_cons(b, wa, g, qa);
    e_prim_to_cons(b, wc, g, qb);
    for (int k = 0; k < b; ++k) out[k] = 0.5 * (fa[k] + fb[k]);
    if (order == 1) {
        for (int k = 0; k < b; ++k) out[k] -= 0.5 * lam * (qb[k] - qa[k]);
        return;
    }
    const double nua = nu[a], nub = nu[c];
    const double s2 = kKappa2 * (nua > nub ? nua : nub);
    double s4 = kKappa4 - s2;
    if (!(s4 > 0.0)) s4 = 0.0; /* std::max(0.0, kKappa4 - s2) */
    if (line) {
        /* line mesh: the reference's own stencil (a-1, a, b, b+1), disc_euler.cpp:145-157;
           lap holds Q per node here (jst_prepass), the 4th difference in its operation order */
        const int im1 = a - 1, ip2 = c + 1;
        if (im1 < 0 || ip2 >= m->n) s4 = 0.0; /* stencil truncated at boundaries */
        for (int k = 0; k < b; ++k) {
            double d = s2 * lam * (qb[k] - qa[k]);
            if (s4 > 0.0)
                d -= s4 * lam * (lap[(size_t)ip2 * b + k] - 3.0 * qb[k] + 3.0 * qa[k] - lap[(size_t)im1 * b + k]);
            out[k] -= d;
        }
        return;
    }
    if (m->bflag[a] || m->bflag[c]) s4 = 0.0; /* stencil truncated at boundaries */
    for (int k = 0; k < b; ++k) {
        double d = s2 * lam * (qb[k] - qa[k]);
        if (s4 > 0.0) d -= s4 * lam * (lap[(size_t)c * b + k] - lap[(size_t)a * b + k]);
        out[k] -= d;
    }
}

/* A line mesh: the interior faces are exactly (i, i+1), i = 0 .. n-2 (the reference's
   build_mesh_1d, mesh.cpp:85-127, in any face order).  There every interior node has the
   unique neighbours i-1 and i+1, and the order-2 terms use the reference's 1D stencil
   verbatim (disc_euler.cpp:113-119,145-157) instead of its edge-based form. */
int or_mesh_is_line(const or_mesh* m) {
    if (m->n < 2) return 0;
    int cnt = 0;
    unsigned char* seen = (unsigned char*)calloc((size_t)m->n, 1);
    int ok = 1;
    for (int f = 0; f < m->nf && ok; ++f) {
        if (m->fbc[f] >= 0) continue;
        const int a = m->fa[f];
        if (m->fb[f] != a + 1 || a < 0 || a + 1 >= m->n || seen[a]) ok = 0;
        else { seen[a] = 1; ++cnt; }
    }
    free(seen);
    return ok && cnt == m->n - 1;
}

/* viscous flux of the SA-like model (b = 6 only; no reference counterpart) */
static void viscous_face_flux(const or_mesh* m, int f, const double* W, double* out) {
    const int b = m->b;
    const int a = m->fa[f], c = m->fb[f];
    const double* wa = W + (size_t)a * b;
    const double* wc = W + (size_t)c * b;
    const double k = 0.5 * (m->mu[a] + m->mu[c]) * m->fvis[f];
    out[0] = 0.0;
    out[1] = -k * (wc[1] - wa[1]);
    out[2] = -k * (wc[2] - wa[2]);
    out[3] = -k * (wc[3] - wa[3]);
    out[4] = 0.0;
    out[5] = -k * (wc[5] - wa[5]);
}

/* node_source (disc_euler.cpp:95-100): slip-wall closure -p * sum(outward normals) */
static void node_source(const or_mesh* m, int i, const double* W, double* out) {
    const int b = m->b;
    const double p = W[(size_t)i * b + 4];
    for (int k = 0; k < b; ++k) out[k] = 0.0;
    out[1] = -p * m->closure[3 * (size_t)i + 0];
    out[2] = -p * m->closure[3 * (size_t)i + 1];
    out[3] = -p * m->closure[3 * (size_t)i + 2];
}

/* face_flux1 (disc_euler.cpp:87-93 + disc_scalar.cpp:74-85 for the viscous part) */
static int face_flux1(const or_mesh* m, int f, const double* W, const double* wref, int mode,
                      const double* forcing, int nforcing, double* out) {
    if (m->fbc[f] >= 0) return boundary_face_flux(m, f, W, wref, mode, forcing, nforcing, out);
    interior_face_flux(m, f, W, 1, NULL, NULL, 0, out);
    if (m->b == 6) {
        double vf[6];
        viscous_face_flux(m, f, W, vf);
        for (int k = 0; k < 6; ++k) out[k] += vf[k];
    }
    return OR_OK;
}

/* order-2 node pre-pass: pressure switch (disc_euler.cpp:113-119, ghost per boundary face)
   and undivided Laplacian of Q (the 1D (a-1, b+1) stencil of :145-157 in edge form) */
static void jst_prepass(const or_mesh* m, const double* W, double* nu, double* lap, int line) {
    const int b = m->b;
    double qi[6], qj[6];
    if (line) { /* pressure_switch (disc_euler.cpp:113-119) with clamped neighbours; lap = Q */
        const int n = m->n;
        for (int i = 0; i < n; ++i) {
            const int im = i - 1 < 0 ? 0 : i - 1;
            const int ip = i + 1 > n - 1 ? n - 1 : i + 1;
            const double pm = W[(size_t)im * b + 4], pc = W[(size_t)i * b + 4], pp = W[(size_t)ip * b + 4];
            nu[i] = fabs(pp - 2.0 * pc + pm) / (pp + 2.0 * pc + pm);
            e_prim_to_cons(b, W + (size_t)i * b, m->gamma, lap + (size_t)i * b);
        }
        return;
    }
    for (int i = 0; i < m->n; ++i) {
        const double pi = W[(size_t)i * b + 4];
        double num = 0.0, den = 0.0;
        double* L = lap + (size_t)i * b;
        for (int k = 0; k < b; ++k) L[k] = 0.0;
        e_prim_to_cons(b, W + (size_t)i * b, m->gamma, qi);
        for (int e = m->nf_ptr[i]; e < m->nf_ptr[i + 1]; ++e) {
            const int f = m->nf_idx[e];
            if (m->fbc[f] >= 0) {
                den += pi + pi;
                continue;
            }
            const int j = m->fa[f] == i ? m->fb[f] : m->fa[f];
            const double pj = W[(size_t)j * b + 4];
            num += pj - pi;
            den += pj + pi;
            e_prim_to_cons(b, W + (size_t)j * b, m->gamma, qj);
            for (int k = 0; k < b; ++k) L[k] += qj[k] - qi[k];
        }
        nu[i] = fabs(num) / den;
    }
}

/* EulerNozzleDisc::residual (disc_euler.cpp:56-85) */
int or_residual(const or_mesh* m, const double* W, const double* wref, int order, int mode,
                const double* forcing, int nforcing, int need_vis, double* inv, double* vis) {
    const int b = m->b, n = m->n;
    memset(inv, 0, sizeof(double) * (size_t)n * b);
    if (need_vis) memset(vis, 0, sizeof(double) * (size_t)n * b);
    double* nu = NULL;
    double* lap = NULL;
    int line = 0;
    if (order == 2) {
        nu = (double*)malloc(sizeof(double) * n);
        lap = (double*)malloc(sizeof(double) * (size_t)n * b);
        line = or_mesh_is_line(m);
        jst_prepass(m, W, nu, lap, line);
    }
    double flux[6];
    int st = OR_OK;
    for (int f = 0; f < m->nf; ++f) {
        const int a = m->fa[f];
        if (m->fbc[f] >= 0) {
            st = boundary_face_flux(m, f, W, wref, mode, forcing, nforcing, flux);
            if (st) goto done;
            for (int k = 0; k < b; ++k) inv[(size_t)a * b + k] += flux[k];
            continue;
        }
        const int c = m->fb[f];
        interior_face_flux(m, f, W, order, nu, lap, line, flux);
        for (int k = 0; k < b; ++k) {
            inv[(size_t)a * b + k] += flux[k];
            inv[(size_t)c * b + k] -= flux[k];
        }
        if (need_vis && b == 6) {
            viscous_face_flux(m, f, W, flux);
            for (int k = 0; k < b; ++k) {
                vis[(size_t)a * b + k] += flux[k];
                vis[(size_t)c * b + k] -= flux[k];
            }
        }
    }
    for (int i = 0; i < n; ++i) {
        double src[6];
        node_source(m, i, W, src);
        for (int k = 0; k < b; ++k) inv[(size_t)i * b + k] += src[k];
    }
done:
    free(nu);
    free(lap);
    return st;
}

/* Discretization::fd_jacobian (disc.cpp:37-130) generalized to b = 5/6 */
int or_fd_jacobian(const or_mesh* m, const or_pattern* p, const double* W, double* J, double* P) {
    const int b = m->b, n = m->n;
    const size_t bb = (size_t)b * b;
    int st;
    for (int i = 0; i < n; ++i)
        if ((st = euler_validate(b, W + (size_t)i * b))) return st;
    if (J) memset(J, 0, sizeof(double) * (size_t)p->nnzb * bb);
    if (P) memset(P, 0, sizeof(double) * (size_t)n * bb);

    double* Q = (double*)malloc(sizeof(double) * (size_t)n * b);
    or_prim_to_cons(b, n, m->gamma, W, Q);
    double qscale[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < b; ++k) {
            const double a = fabs(Q[(size_t)i * b + k]);
            qscale[k] = qscale[k] > a ? qscale[k] : a; /* std::max(qscale, |Q|) */
        }
    for (int k = 0; k < b; ++k)
        if (qscale[k] == 0.0) qscale[k] = 1.0;
    free(Q);
    const double kFdRel = 1e-6;

    double* Ws = (double*)malloc(sizeof(double) * (size_t)n * b);
    memcpy(Ws, W, sizeof(double) * (size_t)n * b);
    int maxnf = 0;
    for (int j = 0; j < n; ++j)
        if (m->nf_ptr[j + 1] - m->nf_ptr[j] > maxnf) maxnf = m->nf_ptr[j + 1] - m->nf_ptr[j];
    double* fplus = (double*)malloc(sizeof(double) * (size_t)(maxnf + 1) * b);
    double* fminus = (double*)malloc(sizeof(double) * (size_t)(maxnf + 1) * b);
    double qj[6], wj[6], splus[6], sminus[6];
    st = OR_OK;
    for (int j = 0; j < n && !st; ++j) {
        const int f_begin = m->nf_ptr[j], f_end = m->nf_ptr[j + 1];
        const int nf = f_end - f_begin;
        for (int mm = 0; mm < b && !st; ++mm) {
            e_prim_to_cons(b, W + (size_t)j * b, m->gamma, qj);
            const double aq = fabs(qj[mm]);
            const double delta = kFdRel * (aq > qscale[mm] ? aq : qscale[mm]);
            for (int sgn = 0; sgn < 2; ++sgn) {
                const double d = sgn == 0 ? delta : -delta;
                qj[mm] += d;
                st = e_cons_to_prim(b, qj, m->gamma, wj);
                if (st) break;
                qj[mm] -= d;
                memcpy(Ws + (size_t)j * b, wj, sizeof(double) * b);
                double* fbuf = sgn == 0 ? fplus : fminus;
                for (int k = 0; k < nf; ++k) {
                    st = face_flux1(m, m->nf_idx[f_begin + k], Ws, NULL, 0, NULL, 0, fbuf + (size_t)k * b);
                    if (st) break;
                }
                if (st) break;
                node_source(m, j, Ws, sgn == 0 ? splus : sminus);
            }
            memcpy(Ws + (size_t)j * b, W + (size_t)j * b, sizeof(double) * b);
            if (st) break;
            const double inv2d = 1.0 / (2.0 * delta);
            for (int k = 0; k < nf; ++k) {
                const int f = m->nf_idx[f_begin + k];
                const int fa = m->fa[f], fb = m->fb[f];
                const int bnd = m->fbc[f] >= 0;
                for (int r = 0; r < b; ++r) {
                    const double dflux = (fplus[(size_t)k * b + r] - fminus[(size_t)k * b + r]) * inv2d;
                    if (dflux == 0.0) continue;
                    if (J) {
                        const int ea = pat_find_d(p, fa, j);
                        J[(size_t)ea * bb + (size_t)r * b + mm] += dflux;
                        if (!bnd) {
                            const int eb = pat_find_d(p, fb, j);
                            J[(size_t)eb * bb + (size_t)r * b + mm] -= dflux;
                        }
                    }
                    if (P) {
                        if (fa == j) P[(size_t)j * bb + (size_t)r * b + mm] += dflux;
                        if (!bnd && fb == j) P[(size_t)j * bb + (size_t)r * b + mm] -= dflux;
                    }
                }
            }
            for (int r = 0; r < b; ++r) {
                const double dsrc = (splus[r] - sminus[r]) * inv2d;
                if (dsrc == 0.0) continue;
                if (J) J[(size_t)p->diag_idx[j] * bb + (size_t)r * b + mm] += dsrc;
                if (P) P[(size_t)j * bb + (size_t)r * b + mm] += dsrc;
            }
        }
    }
    free(Ws);
    free(fplus);
    free(fminus);
    if (st) return st;
    if (J) { /* disc.cpp:121-129: diagonal blocks must be nonsingular */
        double blk[36];
        int piv[6];
        for (int i = 0; i < n; ++i) {
            memcpy(blk, J + (size_t)p->diag_idx[i] * bb, sizeof(double) * bb);
            if ((st = or_block_lu_factor_d(b, blk, piv, i, NULL))) return st;
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * residual_ops.cpp
 * ------------------------------------------------------------------------- */
static const double kLinFdRel = 1e-5; /* residual_ops.hpp:15 */

/* directional_step (residual_ops.cpp:12-29) */
static double directional_step(const or_mesh* m, const double* mean, const double* dir, const double* fdir,
                               int nf) {
    const int b = m->b;
    double wscale[6] = {0}, dscale[6] = {0};
    for (int i = 0; i < m->n; ++i)
        for (int k = 0; k < b; ++k) {
            const double a = fabs(mean[(size_t)i * b + k]);
            const double d = fabs(dir[(size_t)i * b + k]);
            wscale[k] = wscale[k] > a ? wscale[k] : a;
            dscale[k] = dscale[k] > d ? dscale[k] : d;
        }
    double ratio = 0.0;
    for (int k = 0; k < b; ++k)
        if (dscale[k] > 0.0) {
            const double ws = wscale[k] > 1e-300 ? wscale[k] : 1e-300;
            const double r = dscale[k] / ws;
            ratio = ratio > r ? ratio : r;
        }
    double fmax = 0.0;
    for (int k = 0; k < nf; ++k) {
        const double a = fabs(fdir[k]);
        fmax = fmax > a ? fmax : a;
    }
    if (fmax > 0.0) {
        const double r = fmax / m->forcing_scale;
        ratio = ratio > r ? ratio : r;
    }
    if (ratio == 0.0) return 0.0;
    return kLinFdRel / ratio;
}

/* directional_difference (residual_ops.cpp:33-59) */
static int directional_difference(const or_mesh* m, const double* mean, const double* dir,
                                  const double* fdir, int nf, int order, int need_vis, double* dinv,
                                  double* dvis) {
    const int b = m->b, n = m->n;
    const size_t len = (size_t)n * b;
    memset(dinv, 0, sizeof(double) * len);
    if (need_vis) memset(dvis, 0, sizeof(double) * len);
    const double delta = directional_step(m, mean, dir, fdir, nf);
    if (delta == 0.0) return OR_OK;
    double* wp = (double*)malloc(sizeof(double) * len);
    double* fp = (double*)malloc(sizeof(double) * (nf > 0 ? nf : 1));
    double* inv_p = (double*)malloc(sizeof(double) * len);
    double* vis_p = (double*)malloc(sizeof(double) * len);
    double* inv_m = (double*)malloc(sizeof(double) * len);
    double* vis_m = (double*)malloc(sizeof(double) * len);
    int st;
    for (size_t k = 0; k < len; ++k) wp[k] = mean[k] + delta * dir[k];
    for (int k = 0; k < nf; ++k) fp[k] = delta * fdir[k];
    st = or_residual(m, wp, mean, order, 1, fp, nf, need_vis, inv_p, vis_p);
    if (!st) {
        for (size_t k = 0; k < len; ++k) wp[k] = mean[k] - delta * dir[k];
        for (int k = 0; k < nf; ++k) fp[k] = -delta * fdir[k];
        st = or_residual(m, wp, mean, order, 1, fp, nf, need_vis, inv_m, vis_m);
    }
    if (!st) {
        const double inv2d = 1.0 / (2.0 * delta);
        for (size_t k = 0; k < len; ++k) dinv[k] = (inv_p[k] - inv_m[k]) * inv2d;
        if (need_vis)
            for (size_t k = 0; k < len; ++k) dvis[k] = (vis_p[k] - vis_m[k]) * inv2d;
    }
    free(wp);
    free(fp);
    free(inv_p);
    free(vis_p);
    free(inv_m);
    free(vis_m);
    return st;
}

/* linearized_residual (residual_ops.cpp:63-102); mean is also the perturbation reference */
int or_linearized_residual(const or_mesh* m, const double* mean, const double* M, const ocplx* what,
                           double omega, const ocplx* forcing, int nforcing, int order, int need_vis,
                           ocplx* inv, ocplx* vis) {
    const int b = m->b, n = m->n;
    const size_t len = (size_t)n * b;
    if (omega < 0.0) return or_fail(OR_CONFIG, -1, -1, "linearized_residual: negative frequency");
    for (size_t k = 0; k < len; ++k) inv[k] = 0;
    if (need_vis)
        for (size_t k = 0; k < len; ++k) vis[k] = 0;
    double* dir = (double*)malloc(sizeof(double) * len);
    double* dinv = (double*)malloc(sizeof(double) * len);
    double* dvis = (double*)malloc(sizeof(double) * len);
    double* fdir = (double*)malloc(sizeof(double) * (nforcing > 0 ? nforcing : 1));
    int st = OR_OK;
    for (int part = 0; part < 2 && !st; ++part) {
        for (size_t k = 0; k < len; ++k) dir[k] = part == 0 ? creal(what[k]) : cimag(what[k]);
        for (int k = 0; k < nforcing; ++k) fdir[k] = part == 0 ? creal(forcing[k]) : cimag(forcing[k]);
        st = directional_difference(m, mean, dir, fdir, nforcing, order, need_vis, dinv, dvis);
        if (st) break;
        /* unit * d with unit = (1,0) or (0,1): std::complex * real is componentwise */
        const double ur = part == 0 ? 1.0 : 0.0, ui = part == 0 ? 0.0 : 1.0;
        for (size_t k = 0; k < len; ++k) inv[k] += CMPLX(ur * dinv[k], ui * dinv[k]);
        if (need_vis)
            for (size_t k = 0; k < len; ++k) vis[k] += CMPLX(ur * dvis[k], ui * dvis[k]);
    }
    free(dir);
    free(dinv);
    free(dvis);
    free(fdir);
    if (st) return st;
    /* spectral source i omega V M what (residual_ops.cpp:88-101) */
    for (int i = 0; i < n; ++i) {
        const double* Mi = M + (size_t)i * b * b;
        const ocplx* wi = what + (size_t)i * b;
        ocplx mw[6];
        for (int r = 0; r < b; ++r) {
            ocplx acc = 0;
            for (int c = 0; c < b; ++c) acc += CMPLX(Mi[(size_t)r * b + c] * creal(wi[c]), Mi[(size_t)r * b + c] * cimag(wi[c]));
            mw[r] = acc;
        }
        const ocplx iwv = CMPLX(0.0, omega * m->vol[i]);
        for (int r = 0; r < b; ++r) inv[(size_t)i * b + r] += iwv * mw[r];
    }
    return OR_OK;
}

/* HarmonicSpec::base_frequency / max_multiple (case.cpp:10-44) */
static int base_frequency(int nh, const double* omega, double* base, int* lmax) {
    const double rel_tol = 1e-9;
    double ws[64];
    int nw = 0;
    for (int h = 0; h < nh; ++h)
        if (omega[h] > 0.0) ws[nw++] = omega[h];
    *lmax = 0;
    if (nw == 0) {
        *base = 0.0;
        return OR_OK;
    }
    double scale = ws[0];
    for (int k = 1; k < nw; ++k) scale = ws[k] > scale ? ws[k] : scale;
    double g = ws[0];
    for (int k = 1; k < nw; ++k) {
        double a = g > ws[k] ? g : ws[k];
        double bb = g < ws[k] ? g : ws[k];
        while (bb > rel_tol * scale) {
            const double r = fmod(a, bb);
            a = bb;
            bb = r;
        }
        g = a;
    }
    if (g < 1e-6 * scale) return or_fail(OR_CONFIG, -1, -1, "harmonic frequencies are incommensurate");
    for (int k = 0; k < nw; ++k) {
        const double mm = ws[k] / g;
        if (fabs(mm - round(mm)) > 1e-6) return or_fail(OR_CONFIG, -1, -1, "harmonic frequencies are incommensurate");
    }
    *base = g;
    for (int h = 0; h < nh; ++h)
        if (omega[h] > 0.0) {
            const int l = (int)llround(omega[h] / g);
            *lmax = *lmax > l ? *lmax : l;
        }
    return OR_OK;
}

/* reconstruct_instantaneous (state.cpp:96-107) */
static void reconstruct(int n, int b, const double* mean, int nh, const double* omega, const ocplx* amps,
                        double t, double* out) {
    const size_t len = (size_t)n * b;
    memcpy(out, mean, sizeof(double) * len);
    for (int h = 0; h < nh; ++h) {
        const ocplx phase = cexp(CMPLX(0.0, omega[h] * t));
        const ocplx* a = amps + (size_t)h * len;
        for (size_t k = 0; k < len; ++k) out[k] += 2.0 * creal(a[k] * phase);
    }
}

/* deterministic_flux (residual_ops.cpp:113-161) */
int or_deterministic_flux(const or_mesh* m, const double* mean, int nh, const int* index,
                          const double* omega, const ocplx* amps, double* df) {
    (void)index;
    const int b = m->b, n = m->n;
    const size_t len = (size_t)n * b;
    memset(df, 0, sizeof(double) * len);
    double base;
    int lmax;
    int st = base_frequency(nh, omega, &base, &lmax);
    if (st) return st;
    int any_amp = 0;
    for (size_t k = 0; k < (size_t)nh * len && !any_amp; ++k)
        if (amps[k] != 0) any_amp = 1;
    if (!any_amp) return OR_OK;
    double* inv = (double*)malloc(sizeof(double) * len);
    double* acc = (double*)calloc(len, sizeof(double));
    double* w = (double*)malloc(sizeof(double) * len);
    if (lmax == 0) {
        reconstruct(n, b, mean, nh, omega, amps, 0.0, w);
        st = or_residual(m, w, NULL, 2, 0, NULL, 0, 0, inv, NULL);
        if (!st) memcpy(acc, inv, sizeof(double) * len);
    } else {
        const double period = 2.0 * acos(-1.0) / base;
        const int nq = 4 * lmax + 2;
        for (int k = 0; k < nq && !st; ++k) {
            const double t = period * k / nq;
            reconstruct(n, b, mean, nh, omega, amps, t, w);
            st = or_residual(m, w, NULL, 2, 0, NULL, 0, 0, inv, NULL);
            if (!st)
                for (size_t q = 0; q < len; ++q) acc[q] += inv[q];
        }
        if (!st)
            for (size_t q = 0; q < len; ++q) acc[q] /= nq;
    }
    if (!st) st = or_residual(m, mean, NULL, 2, 0, NULL, 0, 0, inv, NULL);
    if (!st)
        for (size_t q = 0; q < len; ++q) df[q] = acc[q] - inv[q];
    free(inv);
    free(acc);
    free(w);
    return st;
}

/* ---------------------------------------------------------------------------
 * Outer FNLH iteration (driver.cpp) and rk_step (rk.cpp:41-99)
 * ------------------------------------------------------------------------- */
typedef struct {
    or_linear_report* v;
    int n, cap;
} report_list;

static void reports_push(report_list* l, const or_linear_report* r) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 64;
        l->v = (or_linear_report*)realloc(l->v, sizeof(or_linear_report) * l->cap);
    }
    l->v[l->n++] = *r;
}

/* a coarse multigrid level (multigrid.hpp:26-32, driver.cpp:104-131): its mesh and
   pattern, the parent map from the next finer level, its boundary forcing, and the
   per-level operators of the outer iteration */
typedef struct {
    or_mesh mesh;
    or_pattern pat;
    const int* parent; /* n of the finer level */
    ocplx* forcing;    /* nh * nforcing */
    int nforcing;
    double *mean, *M, *MLU, *P, *PLU;
    int *Mpiv, *Ppiv;
} or_level;

struct or_solver {
    or_mesh mesh;
    or_pattern pat;
    or_scheme sch;
    double sigma;
    int nh, nforcing;
    int* index;
    double* omega;
    ocplx* forcing; /* nh * nforcing */
    double* mean;   /* n*b */
    ocplx* amps;    /* nh*n*b */
    double* df;
    const double* ext_acc; /* or_solver_set_external_df: the chained quadrature sum */
    double *J, *A5, *M, *MLU, *P, *PLU;
    int *Mpiv, *Ppiv;
    or_ilu_d ilu_mean;
    ocplx* wsmat;
    or_ilu_z wsilu;
    report_list reports;
    int iter;
    report_list* hrep; /* per harmonic, from the last phase_harmonics */
    int failed_h;      /* harmonic of the error the last phase_harmonics returned, -1 none */
    double* hnorm;
    or_ilu_z* ws_extra; /* per-worker complex workspaces (or_set_workers) */
    int nlev;           /* coarse multigrid levels (explicit scheme) */
    or_level* lev;      /* lev[l - 1] = level l */
    or_error* herr;     /* per harmonic error record of the worker threads */
    ocplx** wsmat_extra;
    int n_extra;
};

static void* xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

or_solver* or_solver_create(const or_mesh* m, const or_pattern* p, const or_scheme* s, int nh,
                            const int* index, const double* omega, const ocplx* forcing, int nforcing,
                            const double* mean0) {
    or_solver* S_ = (or_solver*)xcalloc(1, sizeof(or_solver));
    S_->failed_h = -1;
    S_->mesh = *m;
    S_->pat = *p;
    S_->sch = *s;
    S_->sigma = s->sigma_cfl > 0.0 ? s->sigma_cfl : (s->implicit ? 50.0 : 2.0); /* driver.hpp:33-41 */
    S_->nh = nh;
    S_->nforcing = nforcing;
    const int b = m->b, n = m->n;
    const size_t len = (size_t)n * b, bb = (size_t)b * b, nnz = (size_t)p->nnzb * bb;
    S_->index = (int*)xcalloc(nh, sizeof(int));
    S_->omega = (double*)xcalloc(nh, sizeof(double));
    memcpy(S_->index, index, sizeof(int) * nh);
    memcpy(S_->omega, omega, sizeof(double) * nh);
    S_->forcing = (ocplx*)xcalloc((size_t)nh * nforcing, sizeof(ocplx));
    if (nforcing) memcpy(S_->forcing, forcing, sizeof(ocplx) * nh * nforcing);
    S_->mean = (double*)xcalloc(len, sizeof(double));
    memcpy(S_->mean, mean0, sizeof(double) * len);
    S_->amps = (ocplx*)xcalloc((size_t)nh * len, sizeof(ocplx));
    S_->df = (double*)xcalloc(len, sizeof(double));
    S_->hrep = (report_list*)xcalloc(nh, sizeof(report_list));
    S_->hnorm = (double*)xcalloc(nh, sizeof(double));
    S_->herr = (or_error*)xcalloc(nh, sizeof(or_error));
    S_->M = (double*)xcalloc((size_t)n * bb, sizeof(double));
    S_->MLU = (double*)xcalloc((size_t)n * bb, sizeof(double));
    S_->Mpiv = (int*)xcalloc(len, sizeof(int));
    if (s->implicit) {
        S_->J = (double*)xcalloc(nnz, sizeof(double));
        S_->A5 = (double*)xcalloc(nnz, sizeof(double));
        S_->ilu_mean.vals = (double*)xcalloc(nnz, sizeof(double));
        S_->ilu_mean.diag_lu = (double*)xcalloc((size_t)n * bb, sizeof(double));
        S_->ilu_mean.diag_piv = (int*)xcalloc(len, sizeof(int));
        S_->ilu_mean.diag_inv = (double*)xcalloc((size_t)n * bb, sizeof(double));
        S_->wsmat = (ocplx*)xcalloc(nnz, sizeof(ocplx));
        S_->wsilu.vals = (ocplx*)xcalloc(nnz, sizeof(ocplx));
        S_->wsilu.diag_lu = (ocplx*)xcalloc((size_t)n * bb, sizeof(ocplx));
        S_->wsilu.diag_piv = (int*)xcalloc(len, sizeof(int));
        S_->wsilu.diag_inv = (ocplx*)xcalloc((size_t)n * bb, sizeof(ocplx));
    } else {
        S_->P = (double*)xcalloc((size_t)n * bb, sizeof(double));
        S_->PLU = (double*)xcalloc((size_t)n * bb, sizeof(double));
        S_->Ppiv = (int*)xcalloc(len, sizeof(int));
    }
    return S_;
}

void or_solver_destroy(or_solver* s) {
    if (!s) return;
    free(s->index);
    free(s->omega);
    free(s->forcing);
    free(s->mean);
    free(s->amps);
    free(s->df);
    free(s->J);
    free(s->A5);
    free(s->M);
    free(s->MLU);
    free(s->Mpiv);
    free(s->P);
    free(s->PLU);
    free(s->Ppiv);
    free(s->ilu_mean.vals);
    free(s->ilu_mean.diag_lu);
    free(s->ilu_mean.diag_piv);
    free(s->ilu_mean.diag_inv);
    free(s->wsmat);
    free(s->wsilu.vals);
    free(s->wsilu.diag_lu);
    free(s->wsilu.diag_piv);
    free(s->wsilu.diag_inv);
    free(s->reports.v);
    for (int h = 0; h < s->nh; ++h) free(s->hrep[h].v);
    for (int t = 0; t < s->n_extra; ++t) {
        free(s->wsmat_extra[t]);
        free(s->ws_extra[t].vals);
        free(s->ws_extra[t].diag_lu);
        free(s->ws_extra[t].diag_piv);
        free(s->ws_extra[t].diag_inv);
    }
    free(s->ws_extra);
    free(s->wsmat_extra);
    for (int l = 0; l < s->nlev; ++l) {
        or_level* v = &s->lev[l];
        free(v->forcing);
        free(v->mean);
        free(v->M);
        free(v->MLU);
        free(v->P);
        free(v->PLU);
        free(v->Mpiv);
        free(v->Ppiv);
    }
    free(s->lev);
    free(s->herr);
    free(s->hrep);
    free(s->hnorm);
    free(s);
}

/* stage evaluators/appliers: 0 = harmonic (complex), 1 = mean (real) */
typedef struct {
    or_solver* s;
    int h; /* harmonic position */
    int l; /* multigrid level (0 = finest) */
} rk_ctx;

/* level accessors (level 0 lives in the solver itself) */
static const or_mesh* lv_mesh(const or_solver* s, int l) { return l == 0 ? &s->mesh : &s->lev[l - 1].mesh; }
static double* lv_mean(or_solver* s, int l) { return l == 0 ? s->mean : s->lev[l - 1].mean; }
static double* lv_M(or_solver* s, int l) { return l == 0 ? s->M : s->lev[l - 1].M; }
static double* lv_MLU(or_solver* s, int l) { return l == 0 ? s->MLU : s->lev[l - 1].MLU; }
static int* lv_Mpiv(or_solver* s, int l) { return l == 0 ? s->Mpiv : s->lev[l - 1].Mpiv; }
static double* lv_P(or_solver* s, int l) { return l == 0 ? s->P : s->lev[l - 1].P; }
static double* lv_PLU(or_solver* s, int l) { return l == 0 ? s->PLU : s->lev[l - 1].PLU; }
static int* lv_Ppiv(or_solver* s, int l) { return l == 0 ? s->Ppiv : s->lev[l - 1].Ppiv; }
static const ocplx* lv_forcing(const or_solver* s, int l, int h) {
    return l == 0 ? s->forcing + (size_t)h * s->nforcing : s->lev[l - 1].forcing + (size_t)h * s->lev[l - 1].nforcing;
}
static int lv_nforcing(const or_solver* s, int l) { return l == 0 ? s->nforcing : s->lev[l - 1].nforcing; }

/* coarse levels run the first-order operator (driver.cpp:199-202,284) */
static int eval_harmonic(rk_ctx* c, const ocplx* state, int need_vis, ocplx* inv, ocplx* vis) {
    or_solver* s = c->s;
    const int l = c->l;
    return or_linearized_residual(lv_mesh(s, l), lv_mean(s, l), lv_M(s, l), state, s->omega[c->h],
                                  lv_forcing(s, l, c->h), lv_nforcing(s, l), l == 0 ? 2 : 1, need_vis, inv, vis);
}

/* add_transform_solve (driver.cpp:32-46) */
static int apply_harmonic(rk_ctx* c, const ocplx* base, const ocplx* x, ocplx* out) {
    or_solver* s = c->s;
    const int b = s->mesh.b, n = lv_mesh(s, c->l)->n;
    const double* MLU = lv_MLU(s, c->l);
    const int* Mpiv = lv_Mpiv(s, c->l);
    const size_t bb = (size_t)b * b;
    memcpy(out, base, sizeof(ocplx) * (size_t)n * b);
    double re[6], im[6], yre[6], yim[6];
    for (int i = 0; i < n; ++i) {
        const ocplx* xi = x + (size_t)i * b;
        for (int k = 0; k < b; ++k) {
            re[k] = creal(xi[k]);
            im[k] = cimag(xi[k]);
        }
        or_block_lu_solve_d(b, MLU + (size_t)i * bb, Mpiv + (size_t)i * b, re, yre);
        or_block_lu_solve_d(b, MLU + (size_t)i * bb, Mpiv + (size_t)i * b, im, yim);
        ocplx* oi = out + (size_t)i * b;
        for (int k = 0; k < b; ++k) oi[k] += CMPLX(yre[k], yim[k]);
    }
    return OR_OK;
}

static int eval_mean(rk_ctx* c, const double* state, int need_vis, double* inv, double* vis) {
    or_solver* s = c->s;
    const int l = c->l;
    int st = or_residual(lv_mesh(s, l), state, NULL, l == 0 ? 2 : 1, 0, NULL, 0, need_vis, inv, vis);
    if (st) return st;
    if (l == 0) { /* DF enters the finest level only (driver.cpp:284-285) */
        const size_t len = (size_t)s->mesh.n * s->mesh.b;
        for (size_t k = 0; k < len; ++k) inv[k] += s->df[k];
    }
    return OR_OK;
}

/* mean_apply (driver.cpp:274-280) */
static int apply_mean(rk_ctx* c, const double* base, const double* x, double* out) {
    or_solver* s = c->s;
    const int b = s->mesh.b, n = lv_mesh(s, c->l)->n;
    const size_t len = (size_t)n * b;
    double* q = (double*)malloc(sizeof(double) * len);
    int st = or_prim_to_cons(b, n, s->mesh.gamma, base, q);
    if (!st) {
        for (size_t k = 0; k < len; ++k) q[k] += x[k];
        st = or_cons_to_prim(b, n, s->mesh.gamma, q, out);
    }
    free(q);
    return st;
}

/* LevelOps::full_residual (driver.cpp:230-236 harmonic, 300-306 mean): out = inv + vis
   (+ DF on the finest mean level) */
static int fullres_harmonic(rk_ctx* c, const ocplx* state, ocplx* out, ocplx* vis) {
    int st = eval_harmonic(c, state, 1, out, vis);
    if (st) return st;
    const size_t len = (size_t)lv_mesh(c->s, c->l)->n * c->s->mesh.b;
    for (size_t k = 0; k < len; ++k) out[k] += vis[k];
    return OR_OK;
}

static int fullres_mean(rk_ctx* c, const double* state, double* out, double* vis) {
    or_solver* s = c->s;
    const int l = c->l;
    int st = or_residual(lv_mesh(s, l), state, NULL, l == 0 ? 2 : 1, 0, NULL, 0, 1, out, vis);
    if (st) return st;
    const size_t len = (size_t)lv_mesh(s, l)->n * s->mesh.b;
    for (size_t k = 0; k < len; ++k) out[k] += vis[k];
    if (l == 0)
        for (size_t k = 0; k < len; ++k) out[k] += s->df[k];
    return OR_OK;
}

#define S double
#define SUF d
#define ILU_T or_ilu_d
#define SQR(x) ((x) * (x))
#define FINITE(x) isfinite(x)
#define EVAL eval_mean
#define APPLY apply_mean
#define FULLRES fullres_mean
#include "rk_tmpl.inc"
#include "mg_tmpl.inc"
#undef FULLRES
#undef S
#undef SUF
#undef ILU_T
#undef SQR
#undef FINITE
#undef EVAL
#undef APPLY

#define S ocplx
#define SUF z
#define ILU_T or_ilu_z
#define SQR(x) cnorm_sq(x)
#define FINITE(x) cfinite(x)
#define EVAL eval_harmonic
#define APPLY apply_harmonic
#define FULLRES fullres_harmonic
#include "rk_tmpl.inc"
#include "mg_tmpl.inc"
#undef FULLRES
#undef S
#undef SUF
#undef ILU_T
#undef SQR
#undef FINITE
#undef EVAL
#undef APPLY

/* FnlhSolver::outer_iteration (driver.cpp:157-333), workers = 1, single grid */
static int g_workers = 1;
void or_set_workers(int w) { g_workers = w; }

/* one harmonic's build_lhs_harmonic + factorization + rk_step (driver.cpp:193-244) */
static int run_harmonic(or_solver* s, int h, double ga5, ocplx* wsmat, or_ilu_z* wsilu) {
    const or_mesh* m = &s->mesh;
    const int b = m->b, n = m->n;
    const size_t len = (size_t)n * b, bb = (size_t)b * b;
    const or_pattern* p = &s->pat;
    const int implicit = s->sch.implicit;
    report_list hreps = {0};
    rk_ctx c = {s, h};
    rk_result res;
    const double omega = s->omega[h];
    int st = OR_OK;
    if (implicit) {
        /* build_lhs_harmonic (rk.cpp:32-39) */
        ocplx* shift = (ocplx*)malloc(sizeof(ocplx) * n);
        for (int i = 0; i < n; ++i) shift[i] = CMPLX(0.0, omega * m->vol[i] / ga5);
        or_shift_diagonal(p, s->A5, shift, wsmat);
        free(shift);
        if ((st = or_ilu_factorize_z(p, wsmat, wsilu))) return st;
        st = rk_step_z(&c, s->amps + (size_t)h * len, n, b, 1, s->sigma, s->sch.eps_relax, s->sch.linear_tol,
                       s->sch.linear_max_iter, p, wsmat, wsilu, NULL, NULL, &res, &hreps, NULL);
    } else if (s->nlev > 0) {
        /* shifted_blocks per level (driver.cpp:224-229), then the FAS V-cycle (:240) */
        ocplx* pcl[16];
        int* pvl[16];
        for (int l = 0; l <= s->nlev; ++l) {
            const or_mesh* ml = lv_mesh(s, l);
            pcl[l] = (ocplx*)malloc(sizeof(ocplx) * (size_t)ml->n * bb);
            pvl[l] = (int*)malloc(sizeof(int) * (size_t)ml->n * b);
            const double* Pl = lv_P(s, l);
            for (int i = 0; i < ml->n && !st; ++i) {
                const double* src = Pl + (size_t)i * bb;
                ocplx* dst = pcl[l] + (size_t)i * bb;
                for (size_t k = 0; k < bb; ++k) dst[k] = CMPLX(src[k], 0.0);
                const ocplx sh = CMPLX(0.0, omega * ml->vol[i]);
                for (int q = 0; q < b; ++q) dst[(size_t)q * b + q] += sh;
                st = or_block_lu_factor_z(b, dst, pvl[l] + (size_t)i * b, i, NULL);
            }
        }
        if (!st)
            st = mg_vcycle_z(s, h, 0, s->amps + (size_t)h * len, NULL, (const ocplx* const*)pcl, (const int* const*)pvl,
                             &res);
        for (int l = 0; l <= s->nlev; ++l) {
            free(pcl[l]);
            free(pvl[l]);
        }
    } else {
        /* shifted_blocks (driver.cpp:48-59) */
        ocplx* pclu = (ocplx*)malloc(sizeof(ocplx) * n * bb);
        int* pcpiv = (int*)malloc(sizeof(int) * len);
        for (int i = 0; i < n && !st; ++i) {
            const double* src = s->P + (size_t)i * bb;
            ocplx* dst = pclu + (size_t)i * bb;
            for (size_t k = 0; k < bb; ++k) dst[k] = CMPLX(src[k], 0.0);
            const ocplx sh = CMPLX(0.0, omega * m->vol[i]);
            for (int q = 0; q < b; ++q) dst[(size_t)q * b + q] += sh;
            st = or_block_lu_factor_z(b, dst, pcpiv + (size_t)i * b, i, NULL);
        }
        if (!st)
            st = rk_step_z(&c, s->amps + (size_t)h * len, n, b, 0, s->sigma, s->sch.eps_relax, s->sch.linear_tol,
                           s->sch.linear_max_iter, p, NULL, NULL, pclu, pcpiv, &res, &hreps, NULL);
        free(pclu);
        free(pcpiv);
    }
    if (!st) s->hnorm[h] = res.stage1_norm;
    for (int k = 0; k < hreps.n; ++k) reports_push(&s->hrep[h], &hreps.v[k]);
    free(hreps.v);
    return st;
}

typedef struct {
    or_solver* s;
    const int* owned;
    int* hst;
    double ga5;
    int t, W;
} worker_arg;

static void* harmonic_worker(void* p) {
    worker_arg* a = (worker_arg*)p;
    for (int h = a->t; h < a->s->nh; h += a->W) {
        if (a->owned && !a->owned[h]) continue;
        a->hst[h] = run_harmonic(a->s, h, a->ga5, a->s->wsmat_extra[a->t], &a->s->ws_extra[a->t]);
        if (a->hst[h]) a->s->herr[h] = g_err;
    }
    return NULL;
}

/* outer_iteration split where harmonic sharding exchanges the fields:
   phase_harmonics relaxes the harmonics with owned[h] (NULL: all), phase_mean runs DF +
   the mean step given every harmonic's stage-1 norm and reports (harmonic order). */
int or_solver_phase_harmonics(or_solver* s, const int* owned, double* hnorm_out) {
    s->iter++;
    const or_mesh* m = &s->mesh;
    const int b = m->b, n = m->n, nh = s->nh;
    const size_t len = (size_t)n * b, bb = (size_t)b * b;
    const or_pattern* p = &s->pat;
    int st;
    /* perturbation reference = mean (linearized_residual passes mean as wref); M and its LU */
    /* mean on every level (driver.cpp:168-171), then M and its LU per level (:172-176) */
    for (int l = 1; l <= s->nlev; ++l)
        mg_restrict_state_d(lv_mesh(s, l - 1), s->lev[l - 1].parent, lv_mesh(s, l)->n, b, lv_mean(s, l - 1),
                            lv_mean(s, l));
    for (int l = 0; l <= s->nlev; ++l) {
        const int nl = lv_mesh(s, l)->n;
        if ((st = or_transform_jacobian(b, nl, m->gamma, lv_mean(s, l), lv_M(s, l)))) return st;
        memcpy(lv_MLU(s, l), lv_M(s, l), sizeof(double) * nl * bb);
        for (int i = 0; i < nl; ++i)
            if ((st = or_block_lu_factor_d(b, lv_MLU(s, l) + (size_t)i * bb, lv_Mpiv(s, l) + (size_t)i * b, i, NULL)))
                return st;
    }

    const int implicit = s->sch.implicit;
    if (implicit) {
        if ((st = or_fd_jacobian(m, p, s->mean, s->J, NULL))) return st;
        if ((st = or_build_lhs_mean(p, s->J, 1, s->sigma, s->sch.eps_relax, 5, s->A5))) return st;
        if ((st = or_ilu_factorize_d(p, s->A5, &s->ilu_mean))) return st;
    } else {  /* assemble_diag_blocks per level (driver.cpp:183-186) */
        for (int l = 0; l <= s->nlev; ++l) {
            const int nl = lv_mesh(s, l)->n;
            const or_pattern* pl = l == 0 ? p : &s->lev[l - 1].pat;
            if ((st = or_fd_jacobian(lv_mesh(s, l), pl, lv_mean(s, l), NULL, lv_P(s, l)))) return st;
            memcpy(lv_PLU(s, l), lv_P(s, l), sizeof(double) * nl * bb);
            for (int i = 0; i < nl; ++i)
                if ((st = or_block_lu_factor_d(b, lv_PLU(s, l) + (size_t)i * bb, lv_Ppiv(s, l) + (size_t)i * b, i,
                                               NULL)))
                    return st;
        }
    }
    const double ga5 = gamma_factor(implicit, s->sigma, s->sch.eps_relax) * kAlpha[4];

    double* hnorm = s->hnorm;
    for (int h = 0; h < nh; ++h) {
        s->hrep[h].n = 0;
        hnorm[h] = 0.0;
    }
    /* harmonic workers (driver.cpp:246-265): with or_set_workers(W > 1) the harmonics run
       on W OpenMP threads, each with its own complex workspace; every harmonic runs and
       the first error by harmonic index is returned.  W = 1: sequential, stop at the
       first error. */
    const int W = g_workers < 1 ? 1 : (g_workers > nh ? (nh > 0 ? nh : 1) : g_workers);
    int hst[64] = {0};
    if (W > 1 && !s->ws_extra) {
        s->ws_extra = (or_ilu_z*)xcalloc(W, sizeof(or_ilu_z));
        s->wsmat_extra = (ocplx**)xcalloc(W, sizeof(ocplx*));
        s->n_extra = W;
        const size_t nnz = (size_t)p->nnzb * bb;
        for (int t = 0; t < W; ++t) {
            s->wsmat_extra[t] = (ocplx*)xcalloc(nnz, sizeof(ocplx));
            s->ws_extra[t].vals = (ocplx*)xcalloc(nnz, sizeof(ocplx));
            s->ws_extra[t].diag_lu = (ocplx*)xcalloc((size_t)n * bb, sizeof(ocplx));
            s->ws_extra[t].diag_piv = (int*)xcalloc(len, sizeof(int));
            s->ws_extra[t].diag_inv = (ocplx*)xcalloc((size_t)n * bb, sizeof(ocplx));
        }
    }
    if (W == 1) {
        for (int h = 0; h < nh; ++h) {
            if (owned && !owned[h]) continue;
            if ((hst[h] = run_harmonic(s, h, ga5, s->wsmat, &s->wsilu))) break;  /* stop at the first error */
        }
    } else {  /* worker t relaxes harmonics t, t + W, ... (driver.cpp:250) */
        pthread_t th[64];
        worker_arg args[64];
        for (int t = 0; t < W; ++t) {
            args[t] = (worker_arg){s, owned, hst, ga5, t, W};
            pthread_create(&th[t], NULL, harmonic_worker, &args[t]);
        }
        for (int t = 0; t < W; ++t) pthread_join(th[t], NULL);
        for (int h = 0; h < nh; ++h)
            if (hst[h]) {  /* the first error by harmonic index (driver.cpp:263-264) */
                g_err = s->herr[h];
                break;
            }
    }
    s->failed_h = -1;
    for (int h = 0; h < nh && !st; ++h)
        if ((st = hst[h])) s->failed_h = h;
    if (hnorm_out)
        for (int h = 0; h < nh; ++h) hnorm_out[h] = hnorm[h];
    return st;
}

int or_solver_failed_harmonic(const or_solver* s) { return s->failed_h; }

int or_solver_harmonic_reports(const or_solver* s, int h, or_linear_report* out, int max) {
    for (int k = 0; k < s->hrep[h].n && k < max; ++k) out[k] = s->hrep[h].v[k];
    return s->hrep[h].n;
}

/* deterministic_flux split over its quadrature points (shard.py), the restatement of
   fnlh_solver_df_*: the same sums in the same k order as or_deterministic_flux */
static int df_nq(const or_solver* s, double* base, int* lmax) {
    *lmax = 0;
    const int st = base_frequency(s->nh, s->omega, base, lmax);
    if (st) return -st;
    return *lmax == 0 ? 1 : 4 * *lmax + 2;
}
int or_solver_df_points(const or_solver* s) {
    double base;
    int lmax;
    return df_nq(s, &base, &lmax);
}
int or_solver_df_terms(or_solver* s, int k0, int k1, double* terms) {
    const or_mesh* m = &s->mesh;
    const size_t len = (size_t)m->n * m->b;
    double base;
    int lmax;
    const int nq = df_nq(s, &base, &lmax);
    if (nq < 0) return -nq;
    if (k0 < 0 || k1 > nq || k0 > k1) return or_fail(OR_SHAPE, -1, -1, "df_terms: range outside [0, nq)");
    double* w = (double*)malloc(sizeof(double) * len);
    int st = OR_OK;
    const double period = lmax == 0 ? 0.0 : 2.0 * acos(-1.0) / base;
    for (int k = k0; k < k1 && !st; ++k) {
        const double t = lmax == 0 ? 0.0 : period * k / nq;
        reconstruct(m->n, m->b, s->mean, s->nh, s->omega, s->amps, t, w);
        st = or_residual(m, w, NULL, 2, 0, NULL, 0, 0, terms + (size_t)(k - k0) * len, NULL);
    }
    free(w);
    return st;
}
void or_solver_df_accumulate(const or_solver* s, const double* terms, int count, double* acc, int first) {
    const size_t len = (size_t)s->mesh.n * s->mesh.b;
    if (first) memset(acc, 0, sizeof(double) * len);  /* the reference's zero-initialised acc */
    for (int j = 0; j < count; ++j)
        for (size_t q = 0; q < len; ++q) acc[q] += terms[(size_t)j * len + q];
}
void or_solver_set_external_df(or_solver* s, const double* acc) { s->ext_acc = acc; }

static int df_from_acc(or_solver* s, const double* acc_in) {
    const or_mesh* m = &s->mesh;
    const size_t len = (size_t)m->n * m->b;
    memset(s->df, 0, sizeof(double) * len);
    double base;
    int lmax;
    const int nq = df_nq(s, &base, &lmax);
    if (nq < 0) return -nq;
    int any_amp = 0;
    for (size_t k = 0; k < (size_t)s->nh * len && !any_amp; ++k)
        if (s->amps[k] != 0) any_amp = 1;
    if (!any_amp) return OR_OK;
    double* acc = (double*)malloc(sizeof(double) * len);
    double* inv = (double*)malloc(sizeof(double) * len);
    memcpy(acc, acc_in, sizeof(double) * len);
    if (lmax != 0)
        for (size_t q = 0; q < len; ++q) acc[q] /= nq;
    const int st = or_residual(m, s->mean, NULL, 2, 0, NULL, 0, 0, inv, NULL);
    if (!st)
        for (size_t q = 0; q < len; ++q) s->df[q] = acc[q] - inv[q];
    free(acc);
    free(inv);
    return st;
}

int or_solver_phase_mean(or_solver* s, const double* hnorm, const int* nrep, const or_linear_report* reps,
                         or_entry* e, double* resid_h) {
    const or_mesh* m = &s->mesh;
    const int b = m->b, n = m->n, nh = s->nh;
    const or_pattern* p = &s->pat;
    const int implicit = s->sch.implicit;
    int st;
    report_list hreps = {0};
    for (int h = 0, q = 0; h < nh; ++h)
        for (int k = 0; k < nrep[h]; ++k, ++q) reports_push(&hreps, &reps[q]);
    /* deterministic flux from the fresh harmonic fields (or from a quadrature sum chained
       across ranks: DF = acc / nq - R(mean), residual_ops.cpp:152-159) */
    if (s->ext_acc) {
        st = df_from_acc(s, s->ext_acc);
        s->ext_acc = NULL;
    } else {
        st = or_deterministic_flux(m, s->mean, nh, s->index, s->omega, s->amps, s->df);
    }
    if (st) {
        free(hreps.v);
        return st;
    }
    /* mean update including DF */
    rk_ctx c = {s, -1};
    rk_result mres;
    report_list mreps = {0};
    if (implicit)
        st = rk_step_d(&c, s->mean, n, b, 1, s->sigma, s->sch.eps_relax, s->sch.linear_tol, s->sch.linear_max_iter,
                       p, s->A5, &s->ilu_mean, NULL, NULL, &mres, &mreps, NULL);
    else if (s->nlev > 0) {  /* FAS V-cycle of the mean (driver.cpp:297-311) */
        const double* pl[16];
        const int* pv[16];
        for (int l = 0; l <= s->nlev; ++l) {
            pl[l] = lv_PLU(s, l);
            pv[l] = lv_Ppiv(s, l);
        }
        st = mg_vcycle_d(s, -1, 0, s->mean, NULL, pl, pv, &mres);
    } else
        st = rk_step_d(&c, s->mean, n, b, 0, s->sigma, s->sch.eps_relax, s->sch.linear_tol, s->sch.linear_max_iter,
                       p, NULL, NULL, s->PLU, s->Ppiv, &mres, &mreps, NULL);
    if (st) {
        free(hreps.v);
        free(mreps.v);
        return st;
    }
    for (int k = 0; k < hreps.n; ++k) reports_push(&s->reports, &hreps.v[k]);
    for (int k = 0; k < mreps.n; ++k) reports_push(&s->reports, &mreps.v[k]);
    free(hreps.v);
    free(mreps.v);

    /* monitor (driver.cpp:315-332), residual_rms (:10-12), aggregate_rz (:14-19) */
    e->iter = s->iter;
    e->stage1_norm_mean = mres.stage1_norm;
    e->resid_mean = mres.stage1_norm / sqrt((double)n * b);
    double acc = 0.0;
    for (int h = 0; h < nh; ++h) {
        resid_h[h] = hnorm[h] / sqrt((double)n * b);
        acc += resid_h[h] * resid_h[h];
    }
    e->has_rz = nh > 0;
    e->rz = nh > 0 ? sqrt(acc / nh) : 0.0;
    return OR_OK;
}

int or_solver_outer_iteration(or_solver* s, or_entry* e, double* resid_h) {
    int st = or_solver_phase_harmonics(s, NULL, NULL);
    if (st) return st;
    int nrep[64];
    report_list all = {0};
    for (int h = 0; h < s->nh; ++h) {
        nrep[h] = s->hrep[h].n;
        for (int k = 0; k < s->hrep[h].n; ++k) reports_push(&all, &s->hrep[h].v[k]);
    }
    st = or_solver_phase_mean(s, s->hnorm, nrep, all.v, e, resid_h);
    free(all.v);
    return st;
}

void or_solver_get_state(const or_solver* s, double* mean, ocplx* amps) {
    const size_t len = (size_t)s->mesh.n * s->mesh.b;
    if (mean) memcpy(mean, s->mean, sizeof(double) * len);
    if (amps) memcpy(amps, s->amps, sizeof(ocplx) * len * s->nh);
}

void or_solver_set_state(or_solver* s, const double* mean, const ocplx* amps) {
    const size_t len = (size_t)s->mesh.n * s->mesh.b;
    if (mean) memcpy(s->mean, mean, sizeof(double) * len);
    if (amps) memcpy(s->amps, amps, sizeof(ocplx) * len * s->nh);
}

int or_solver_num_reports(const or_solver* s) { return s->reports.n; }

void or_solver_get_reports(const or_solver* s, or_linear_report* out) {
    memcpy(out, s->reports.v, sizeof(or_linear_report) * s->reports.n);
}

const double* or_solver_df(const or_solver* s) { return s->df; }

/* run_to_convergence (driver.cpp:335-379) */
int or_solver_run(or_solver* s, int* n_entries, or_entry* entries, int max_entries) {
    const double drop = pow(10.0, -s->sch.target_drop_orders);
    double r1_mean = -1.0, r1_rz = -1.0, floor_ = 0.0;
    int reason = 1;
    double rh[64];
    *n_entries = 0;
    for (int it = 0; it < s->sch.max_outer_iters; ++it) {
        or_entry e;
        int st = or_solver_outer_iteration(s, &e, rh);
        if (st == OR_DIVERGENCE) {
            reason = 2;
            break;
        }
        if (st) return -st;
        if (*n_entries < max_entries) entries[*n_entries] = e;
        (*n_entries)++;
        if (it == 0) {
            r1_mean = e.resid_mean;
            r1_rz = e.has_rz ? e.rz : 0.0;
            floor_ = 1e-16 * (r1_mean > r1_rz ? r1_mean : r1_rz);
        }
        const double tm = r1_mean * drop > floor_ ? r1_mean * drop : floor_;
        const double tz = r1_rz * drop > floor_ ? r1_rz * drop : floor_;
        const int mean_ok = e.resid_mean <= tm;
        const int rz_ok = !e.has_rz || e.rz <= tz;
        if (mean_ok && rz_ok) {
            reason = 0;
            break;
        }
    }
    return reason;
}

/* a coarse multigrid level below the current coarsest (explicit scheme; the reference's
   build_hierarchy + per-level discretization, driver.cpp:104-131): mesh, pattern, parent
   map from the current coarsest level's nodes, and the level's boundary forcing */
int or_solver_add_level(or_solver* s, const or_mesh* m, const or_pattern* p, const int* parent, const ocplx* forcing,
                        int nforcing) {
    if (s->sch.implicit) return or_fail(OR_CONFIG, -1, -1, "multigrid is available for the explicit scheme only");
    if (s->nlev >= 15) return or_fail(OR_CONFIG, -1, -1, "too many multigrid levels");
    s->lev = (or_level*)realloc(s->lev, sizeof(or_level) * (s->nlev + 1));
    or_level* v = &s->lev[s->nlev];
    memset(v, 0, sizeof *v);
    v->mesh = *m;
    v->pat = *p;
    v->parent = parent;
    const size_t n = m->n, b = m->b, bb = b * b;
    v->nforcing = nforcing;
    v->forcing = (ocplx*)xcalloc((size_t)s->nh * nforcing, sizeof(ocplx));
    if (nforcing) memcpy(v->forcing, forcing, sizeof(ocplx) * (size_t)s->nh * nforcing);
    v->mean = (double*)xcalloc(n * b, sizeof(double));
    v->M = (double*)xcalloc(n * bb, sizeof(double));
    v->MLU = (double*)xcalloc(n * bb, sizeof(double));
    v->P = (double*)xcalloc(n * bb, sizeof(double));
    v->PLU = (double*)xcalloc(n * bb, sizeof(double));
    v->Mpiv = (int*)xcalloc(n * b, sizeof(int));
    v->Ppiv = (int*)xcalloc(n * b, sizeof(int));
    s->nlev++;
    return OR_OK;
}
