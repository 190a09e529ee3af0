// disc.cu -- device discretization kernels.  Parity contract: every kernel follows
// the operation order of the reference (disc_euler.cpp, disc.cpp, residual_ops.cpp,
// state.cpp) as restated in oracle/fnlh_oracle.c; per-node accumulations are
// atomic-free CSR-by-node gathers in ascending face index (mesh.cpp:44-59), so the
// residual and the FD Jacobian are bitwise identical to the CPU (pow() in the
// subsonic inlet/outlet states is the only libm call whose last bit may differ).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "disc.cuh"

namespace fnlh {

namespace {

constexpr int kT = 128;
inline int nb(long long n, int t = kT) { return static_cast<int>((n + t - 1) / t); }

// FNLH_PACKED_RESIDUAL=0 keeps the unpacked order-2 kernels (A/B measurement)
bool packed_disabled() {
    const char* e = std::getenv("FNLH_PACKED_RESIDUAL");
    return e && e[0] == '0';
}

__device__ __forceinline__ void record(unsigned long long* err, unsigned long long key, int code) {
    atomicMin(err, (key << 4) | (unsigned long long)code);
}

// ---------------------------------------------------------------------------
// residual: node pre-pass (order 2), face fluxes, node gather
// ---------------------------------------------------------------------------
template <int B>
__global__ void k_jst_prepass(MeshDev m, const double* __restrict__ W, double* __restrict__ nu,
                              double* __restrict__ lap, const double* skip) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    if (skip && *skip == 0.0) return;
    const double* wi = W + (size_t)i * B;
    if (m.line) {  // pressure_switch (disc_euler.cpp:113-119), clamped neighbours; lap = Q
        const int im = i > 0 ? i - 1 : 0, ip = i + 1 < m.n ? i + 1 : m.n - 1;
        const double pm = W[(size_t)im * B + 4], pc = wi[4], pp = W[(size_t)ip * B + 4];
        nu[i] = fabs(pp - 2.0 * pc + pm) / (pp + 2.0 * pc + pm);
        double q[B];
        prim_to_cons<B>(wi, m.gamma, q);
#pragma unroll
        for (int k = 0; k < B; ++k) lap[(size_t)i * B + k] = q[k];
        return;
    }
    const double pi = wi[4];
    double num = 0.0, den = 0.0;
    double L[B], qi[B], qj[B];
#pragma unroll
    for (int k = 0; k < B; ++k) L[k] = 0.0;
    prim_to_cons<B>(wi, m.gamma, qi);
    for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
        const int code = m.nf_code[e];
        if (code == kBoundaryFace) {
            den += pi + pi;
            continue;
        }
        const int j = code >= 0 ? code : -code - 1;
        const double* wj = W + (size_t)j * B;
        const double pj = wj[4];
        num += pj - pi;
        den += pj + pi;
        prim_to_cons<B>(wj, m.gamma, qj);
#pragma unroll
        for (int k = 0; k < B; ++k) L[k] += qj[k] - qi[k];
    }
    nu[i] = fabs(num) / den;
#pragma unroll
    for (int k = 0; k < B; ++k) lap[(size_t)i * B + k] = L[k];
}

template <int B>
__global__ void k_face_flux(MeshDev m, const double* __restrict__ W, const double* __restrict__ wref, int order,
                            int mode, const double* __restrict__ forcing, int nforcing, int need_vis,
                            const double* __restrict__ nu, const double* __restrict__ lap,
                            double* __restrict__ flux, double* __restrict__ vflux, unsigned long long* err,
                            const double* skip) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= m.nf) return;
    if (skip && *skip == 0.0) return;
    const int a = m.fa[f];
    double out[B];
    if (m.fbc[f] >= 0) {
        const int st = boundary_face_flux<B>(m, f, W + (size_t)a * B, wref ? wref + (size_t)a * B : nullptr, mode,
                                             forcing, nforcing, out);
        if (st) {
            record(err, (unsigned long long)f, st);
#pragma unroll
            for (int k = 0; k < B; ++k) out[k] = 0.0;
        }
    } else {
        const int c = m.fb[f];
        double wa[B], wc[B];
        load_vec<B>(W + (size_t)a * B, wa);
        load_vec<B>(W + (size_t)c * B, wc);
        if (order == 2 && m.line) {  // the reference's stencil (a-1, a, b, b+1), truncated at the ends
            const bool trunc = a - 1 < 0 || c + 1 >= m.n;
            interior_face_flux<B>(m, f, wa, wc, 2, nu[a], nu[c], trunc, trunc ? nullptr : lap + (size_t)(a - 1) * B,
                                  trunc ? nullptr : lap + (size_t)(c + 1) * B, out, true);
        } else if (order == 2)
            interior_face_flux<B>(m, f, wa, wc, 2, nu[a], nu[c], m.bflag[a] || m.bflag[c], lap + (size_t)a * B,
                                  lap + (size_t)c * B, out);
        else
            interior_face_flux<B>(m, f, wa, wc, 1, 0.0, 0.0, false, nullptr, nullptr, out);
        if (need_vis && B == 6) {
            double vo[B];
            viscous_face_flux<B>(m, f, wa, wc, m.mu[a], m.mu[c], vo);
            store_vec<B>(vflux + (size_t)f * B, vo);
        }
    }
    store_vec<B>(flux + (size_t)f * B, out);
}

template <int B>
__global__ void k_node_gather(MeshDev m, const double* __restrict__ W, const double* __restrict__ flux,
                              const double* __restrict__ vflux, int need_vis, double* __restrict__ inv,
                              double* __restrict__ vis, const double* skip) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    if (skip && *skip == 0.0) return;
    double acc[B], vacc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
        acc[k] = 0.0;
        vacc[k] = 0.0;
    }
    for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
        const int f = m.nf_idx[e];
        const int code = m.nf_code[e];
        const double* fl = flux + (size_t)f * B;
        if (code >= 0 || code == kBoundaryFace) {
#pragma unroll
            for (int k = 0; k < B; ++k) acc[k] += fl[k];
            if (B == 6 && need_vis && code != kBoundaryFace) {
                const double* vf = vflux + (size_t)f * B;
#pragma unroll
                for (int k = 0; k < B; ++k) vacc[k] += vf[k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < B; ++k) acc[k] -= fl[k];
            if (B == 6 && need_vis) {
                const double* vf = vflux + (size_t)f * B;
#pragma unroll
                for (int k = 0; k < B; ++k) vacc[k] -= vf[k];
            }
        }
    }
    double src[B];
    node_source<B>(m, i, W[(size_t)i * B + 4], src);
#pragma unroll
    for (int k = 0; k < B; ++k) inv[(size_t)i * B + k] = acc[k] + src[k];
    if (need_vis) {
#pragma unroll
        for (int k = 0; k < B; ++k) vis[(size_t)i * B + k] = vacc[k];
    }
}

// ---------------------------------------------------------------------------
// packed order-2 residual (boundary faces the tail of the face list): the pre-pass writes
// one 16-byte-aligned record per node [W(B), nu, lap(B), bflag] that the interior face
// kernel reads with 16-byte loads, the face geometry is one record [fn, fnh, area,
// (fa, fb)] per interior face, and flux rows are padded to kFS doubles so the node
// gather reads them with 16-byte loads too.  Same arithmetic, same order as above.
// ---------------------------------------------------------------------------
template <int B>
struct Rec {
    static constexpr int R = 2 * B + 2;  // 12 (b = 5) or 14 (b = 6) doubles
};
constexpr int kFS = 6;                   // flux row stride (doubles)

__device__ __forceinline__ void ld2(const double* __restrict__ p, double& a, double& b) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    a = v.x;
    b = v.y;
}
__device__ __forceinline__ void st2(double* __restrict__ p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

template <int B>
__global__ void k_jst_prepass_rec(MeshDev m, const double* __restrict__ W, double* __restrict__ rec,
                                  const double* skip) {
    constexpr int R = Rec<B>::R;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    if (skip && *skip == 0.0) return;
    const double* wi = W + (size_t)i * B;
    double r[R];
#pragma unroll
    for (int k = 0; k < B; ++k) r[k] = wi[k];
    const double pi = r[4];
    double num = 0.0, den = 0.0;
    double L[B], qi[B], qj[B];
#pragma unroll
    for (int k = 0; k < B; ++k) L[k] = 0.0;
    prim_to_cons<B>(r, m.gamma, qi);
    for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
        const int code = m.nf_code[e];
        if (code == kBoundaryFace) {
            den += pi + pi;
            continue;
        }
        const int j = code >= 0 ? code : -code - 1;
        const double* wj = W + (size_t)j * B;
        const double pj = wj[4];
        num += pj - pi;
        den += pj + pi;
        prim_to_cons<B>(wj, m.gamma, qj);
#pragma unroll
        for (int k = 0; k < B; ++k) L[k] += qj[k] - qi[k];
    }
    r[B] = fabs(num) / den;
#pragma unroll
    for (int k = 0; k < B; ++k) r[B + 1 + k] = L[k];
    r[2 * B + 1] = m.bflag[i] ? 1.0 : 0.0;
    double* o = rec + (size_t)i * R;
#pragma unroll
    for (int k = 0; k < R; k += 2) st2(o + k, r[k], r[k + 1]);
}

template <int B>
__device__ __forceinline__ void face_int(const MeshDev& m, int f, const double* __restrict__ geo,
                                         const double* __restrict__ rec, int need_vis, double* __restrict__ flux,
                                         double* __restrict__ vflux) {
    constexpr int R = Rec<B>::R;
    double g8[8];
#pragma unroll
    for (int k = 0; k < 8; k += 2) ld2(geo + (size_t)f * 8 + k, g8[k], g8[k + 1]);
    const long long ab = __double_as_longlong(g8[7]);
    const int a = (int)(ab & 0xffffffffll), c = (int)(ab >> 32);
    double ra[R], rc[R];
#pragma unroll
    for (int k = 0; k < R; k += 2) {
        ld2(rec + (size_t)a * R + k, ra[k], ra[k + 1]);
        ld2(rec + (size_t)c * R + k, rc[k], rc[k + 1]);
    }
    double out[kFS];
    out[kFS - 1] = 0.0;
    interior_flux_core<B>(m.gamma, g8, g8 + 3, g8[6], ra, rc, 2, ra[B], rc[B], ra[2 * B + 1] != 0.0 || rc[2 * B + 1] != 0.0,
                          ra + B + 1, rc + B + 1, out);
    double* o = flux + (size_t)f * kFS;
#pragma unroll
    for (int k = 0; k < kFS; k += 2) st2(o + k, out[k], out[k + 1]);
    if (need_vis && B == 6) {
        double vo[kFS];
        viscous_face_flux<B>(m, f, ra, rc, m.mu[a], m.mu[c], vo);
        double* v = vflux + (size_t)f * kFS;
#pragma unroll
        for (int k = 0; k < kFS; k += 2) st2(v + k, vo[k], vo[k + 1]);
    }
}

template <int B>
__device__ __forceinline__ void face_bnd(const MeshDev& m, int f, const double* __restrict__ W,
                                         const double* __restrict__ wref, int mode, const double* __restrict__ forcing,
                                         int nforcing, double* __restrict__ flux, unsigned long long* err) {
    const int a = m.fa[f];
    double out[kFS];
    out[kFS - 1] = 0.0;
    const int st = boundary_face_flux<B>(m, f, W + (size_t)a * B, wref ? wref + (size_t)a * B : nullptr, mode, forcing,
                                         nforcing, out);
    if (st) {
        record(err, (unsigned long long)f, st);
#pragma unroll
        for (int k = 0; k < B; ++k) out[k] = 0.0;
    }
    double* o = flux + (size_t)f * kFS;
#pragma unroll
    for (int k = 0; k < kFS; k += 2) st2(o + k, out[k], out[k + 1]);
}

// one launch for all faces: the first nbb blocks take the boundary tail (long pow
// latency, started first), the rest the interior faces
template <int B>
__global__ void __launch_bounds__(128) k_face_packed(MeshDev m, int nf_int, int nbb, const double* __restrict__ geo,
                                                     const double* __restrict__ rec, const double* __restrict__ W,
                                                     const double* __restrict__ wref, int mode,
                                                     const double* __restrict__ forcing, int nforcing, int need_vis,
                                                     double* __restrict__ flux, double* __restrict__ vflux,
                                                     unsigned long long* err, const double* skip) {
    if (skip && *skip == 0.0) return;
    if ((int)blockIdx.x < nbb) {
        const int f = nf_int + blockIdx.x * blockDim.x + threadIdx.x;
        if (f < m.nf) face_bnd<B>(m, f, W, wref, mode, forcing, nforcing, flux, err);
    } else {
        const int f = (blockIdx.x - nbb) * blockDim.x + threadIdx.x;
        if (f < nf_int) face_int<B>(m, f, geo, rec, need_vis, flux, vflux);
    }
}

template <int B>
__global__ void k_node_gather_p(MeshDev m, const double* __restrict__ W, const double* __restrict__ flux,
                                const double* __restrict__ vflux, int need_vis, double* __restrict__ inv,
                                double* __restrict__ vis, const double* skip) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    if (skip && *skip == 0.0) return;
    double acc[B], vacc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
        acc[k] = 0.0;
        vacc[k] = 0.0;
    }
    for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
        const int f = m.nf_idx[e];
        const int code = m.nf_code[e];
        double fl[kFS];
#pragma unroll
        for (int k = 0; k < kFS; k += 2) ld2(flux + (size_t)f * kFS + k, fl[k], fl[k + 1]);
        if (code >= 0 || code == kBoundaryFace) {
#pragma unroll
            for (int k = 0; k < B; ++k) acc[k] += fl[k];
            if (B == 6 && need_vis && code != kBoundaryFace) {
                const double* vf = vflux + (size_t)f * kFS;
#pragma unroll
                for (int k = 0; k < B; ++k) vacc[k] += vf[k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < B; ++k) acc[k] -= fl[k];
            if (B == 6 && need_vis) {
                const double* vf = vflux + (size_t)f * kFS;
#pragma unroll
                for (int k = 0; k < B; ++k) vacc[k] -= vf[k];
            }
        }
    }
    double src[B];
    node_source<B>(m, i, W[(size_t)i * B + 4], src);
#pragma unroll
    for (int k = 0; k < B; ++k) inv[(size_t)i * B + k] = acc[k] + src[k];
    if (need_vis) {
#pragma unroll
        for (int k = 0; k < B; ++k) vis[(size_t)i * B + k] = vacc[k];
    }
}

// ---------------------------------------------------------------------------
// FD Jacobian (disc.cpp:37-130): one thread per (column node j, variable m)
// ---------------------------------------------------------------------------
template <int B>
__global__ void k_validate(int n, const double* __restrict__ W, unsigned long long* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!admissible<B>(W + (size_t)i * B)) record(err, (unsigned long long)i, 2);
}

// non-negative doubles order like their bit patterns
__global__ void k_umax_init(unsigned long long* u, int k) {
    if (threadIdx.x < k) u[threadIdx.x] = 0ull;
}

template <int B>
__global__ void k_qscale(int n, double g, const double* __restrict__ W, unsigned long long* umax) {
    double loc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) loc[k] = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double q[B];
        prim_to_cons<B>(W + (size_t)i * B, g, q);
#pragma unroll
        for (int k = 0; k < B; ++k) loc[k] = fmax(loc[k], fabs(q[k]));
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
        double v = loc[k];
        for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
        if ((threadIdx.x & 31) == 0) atomicMax(umax + k, (unsigned long long)__double_as_longlong(v));
    }
}

template <int B>
__global__ void k_qscale_finish(const unsigned long long* umax, double* qscale) {
    const int k = threadIdx.x;
    if (k >= B) return;
    const double v = __longlong_as_double((long long)umax[k]);
    qscale[k] = v == 0.0 ? 1.0 : v;
}

// element k of block e: the reference BSR layout, or (sell_map) the 2-colour SELL copy
template <int B>
__device__ __forceinline__ long long fd_addr(const long long* __restrict__ sell_map, int e, int k) {
    return sell_map ? sell_map[e] + (long long)(k >> 1) * 64 + (k & 1) : (long long)e * B * B + k;
}

template <int B>
__device__ __forceinline__ void fd_face_flux_int(const MeshDev& m, int f, int j, const double* wj,
                                                 const double* __restrict__ W, double* out) {
    const int a = m.fa[f], c = m.fb[f];
    double wo[B];
    if (a == j) {
        load_vec<B>(W + (size_t)c * B, wo);
        interior_face_flux<B>(m, f, wj, wo, 1, 0.0, 0.0, false, nullptr, nullptr, out);
        if (B == 6) {
            double vf[B];
            viscous_face_flux<B>(m, f, wj, wo, m.mu[a], m.mu[c], vf);
#pragma unroll
            for (int k = 0; k < B; ++k) out[k] += vf[k];
        }
    } else {
        load_vec<B>(W + (size_t)a * B, wo);
        interior_face_flux<B>(m, f, wo, wj, 1, 0.0, 0.0, false, nullptr, nullptr, out);
        if (B == 6) {
            double vf[B];
            viscous_face_flux<B>(m, f, wo, wj, m.mu[a], m.mu[c], vf);
#pragma unroll
            for (int k = 0; k < B; ++k) out[k] += vf[k];
        }
    }
}

template <int B>
__device__ __forceinline__ int fd_face_flux(const MeshDev& m, int f, int j, const double* wj,
                                            const double* __restrict__ W, double* out) {
    if (m.fbc[f] >= 0) return boundary_face_flux<B>(m, f, wj, nullptr, 0, nullptr, 0, out);
    const int a = m.fa[f], c = m.fb[f];
    double wo[B];
    if (a == j) {
        load_vec<B>(W + (size_t)c * B, wo);
        interior_face_flux<B>(m, f, wj, wo, 1, 0.0, 0.0, false, nullptr, nullptr, out);
        if (B == 6) {
            double vf[B];
            viscous_face_flux<B>(m, f, wj, wo, m.mu[a], m.mu[c], vf);
#pragma unroll
            for (int k = 0; k < B; ++k) out[k] += vf[k];
        }
    } else {
        load_vec<B>(W + (size_t)a * B, wo);
        interior_face_flux<B>(m, f, wo, wj, 1, 0.0, 0.0, false, nullptr, nullptr, out);
        if (B == 6) {
            double vf[B];
            viscous_face_flux<B>(m, f, wo, wj, m.mu[a], m.mu[c], vf);
#pragma unroll
            for (int k = 0; k < B; ++k) out[k] += vf[k];
        }
    }
    return 0;
}

// PART 0: every face of node j.  When the boundary faces are the tail of the face list
// (nf_int >= 0) the work is split so the common case carries no boundary-state code:
// PART 1 walks the interior faces of every node (they come first in ascending face order)
// and finishes the nodes without boundary faces; PART 2 runs on the boundary nodes only
// (`bnodes`) and continues the same accumulation over their boundary faces from the
// partial sums PART 1 left in `dpart`.  Every diagonal entry sees the same sequence.
template <int B, int PART>
__global__ void __launch_bounds__(kT) k_fd_jacobian(MeshDev m, const int* __restrict__ diag_idx,
                                                    const int* __restrict__ e_ab, const int* __restrict__ e_ba,
                                                    const double* __restrict__ W, const double* __restrict__ qscale,
                                                    double* __restrict__ J, double* __restrict__ P,
                                                    unsigned long long* err, const int* __restrict__ bnodes, int nb_nodes,
                                                    double* __restrict__ dpart, const long long* __restrict__ sell_map,
                                                    double ga, double inv_es, int to_a5) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (PART == 2 ? nb_nodes : m.n) * B) return;
    const int j = PART == 2 ? bnodes[t / B] : t / B, mm = t % B;
    const double g = m.gamma;
    double qj[B], wp[B], wm[B];
    prim_to_cons<B>(W + (size_t)j * B, g, qj);
    const double aq = fabs(qj[mm]);
    const double delta = 1e-6 * (aq > qscale[mm] ? aq : qscale[mm]);
    const unsigned long long key = (unsigned long long)t;
    // the reference's q += d; w = prim(q); q -= d sequence (disc.cpp:63-79)
    qj[mm] += delta;
    int st = cons_to_prim<B>(qj, g, wp);
    qj[mm] -= delta;
    if (st) {
        record(err, key, st);
        return;
    }
    qj[mm] += -delta;
    st = cons_to_prim<B>(qj, g, wm);
    qj[mm] -= -delta;
    if (st) {
        record(err, key, st);
        return;
    }
    const double inv2d = 1.0 / (2.0 * delta);
    double dacc[B];
    int e = m.nf_ptr[j];
    if (PART == 2) {
#pragma unroll
        for (int r = 0; r < B; ++r) dacc[r] = dpart[(size_t)j * B * B + r * B + mm];
        while (e < m.nf_ptr[j + 1] && m.fbc[m.nf_idx[e]] < 0) ++e;  // PART 1 did these
    } else {
#pragma unroll
        for (int r = 0; r < B; ++r) dacc[r] = 0.0;
    }
    for (; e < m.nf_ptr[j + 1]; ++e) {
        const int f = m.nf_idx[e];
        if (PART == 1 && m.fbc[f] >= 0) {  // the rest are boundary faces: PART 2 continues
#pragma unroll
            for (int r = 0; r < B; ++r) dpart[(size_t)j * B * B + r * B + mm] = dacc[r];
            return;
        }
        double fp[B], fm[B];
        if (PART == 1) {
            fd_face_flux_int<B>(m, f, j, wp, W, fp);
            fd_face_flux_int<B>(m, f, j, wm, W, fm);
            st = 0;
        } else {
            st = fd_face_flux<B>(m, f, j, wp, W, fp);
            if (!st) st = fd_face_flux<B>(m, f, j, wm, W, fm);
        }
        if (st) {
            record(err, key, st);
            return;
        }
        const bool bnd = m.fbc[f] >= 0;
        const bool isa = m.fa[f] == j;
#pragma unroll
        for (int r = 0; r < B; ++r) {
            const double dflux = (fp[r] - fm[r]) * inv2d;
            if (dflux == 0.0) continue;
            if (bnd || isa) {
                dacc[r] += dflux;
                if (!bnd && J) {
                    double* dst = J + fd_addr<B>(sell_map, e_ba[f], r * B + mm);
                    const double v = *dst - dflux;
                    *dst = to_a5 ? v / ga : v;  // build_lhs_mean (rk.cpp:23) fused: A = J / ga
                }
            } else {
                if (J) {
                    double* dst = J + fd_addr<B>(sell_map, e_ab[f], r * B + mm);
                    const double v = *dst + dflux;
                    *dst = to_a5 ? v / ga : v;
                }
                dacc[r] -= dflux;
            }
        }
    }
    double sp[B], sm[B];
    node_source<B>(m, j, wp[4], sp);
    node_source<B>(m, j, wm[4], sm);
#pragma unroll
    for (int r = 0; r < B; ++r) {
        const double dsrc = (sp[r] - sm[r]) * inv2d;
        if (dsrc == 0.0) continue;
        dacc[r] += dsrc;
    }
#pragma unroll
    for (int r = 0; r < B; ++r) {
        if (J) {
            double v = dacc[r];
            if (to_a5) {  // rk.cpp:23,27: A_ii = J_ii / ga + (J_ii inv_es) / ga
                double a = v / ga;
                a += v * inv_es / ga;
                v = a;
            }
            J[fd_addr<B>(sell_map, diag_idx[j], r * B + mm)] = v;
        }
        if (P) P[(size_t)j * B * B + r * B + mm] = dacc[r];
    }
}

// diagonal non-singularity check (disc.cpp:121-129)
template <int B>
__global__ void k_diag_check(int n, const int* __restrict__ diag_idx, const double* __restrict__ J,
                             unsigned long long* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double A[B * B];
    int piv[B];
    load_block<B>(J + (diag_idx ? (size_t)diag_idx[i] : (size_t)i) * B * B, A);
    double cond;
    if (lu_factor_reg<B>(A, piv, cond)) record(err, (unsigned long long)i, 5);
}

// ---------------------------------------------------------------------------
// linearized residual (residual_ops.cpp:12-102)
// ---------------------------------------------------------------------------
// umax[0..B) = max|mean|, [B..2B) = max|Re what|, [2B..3B) = max|Im what|,
// [3B] = max|Re forcing|, [3B+1] = max|Im forcing|
template <int B>
__global__ void k_linres_scales(int n, const double* __restrict__ mean, const cplx* __restrict__ what,
                                const cplx* __restrict__ forcing, int nforcing, unsigned long long* umax) {
    double lm[B], lr[B], li[B], fr = 0.0, fi = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) lm[k] = lr[k] = li[k] = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < B; ++k) {
            lm[k] = fmax(lm[k], fabs(mean[(size_t)i * B + k]));
            const cplx w = what[(size_t)i * B + k];
            lr[k] = fmax(lr[k], fabs(w.re));
            li[k] = fmax(li[k], fabs(w.im));
        }
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nforcing; k += gridDim.x * blockDim.x) {
        fr = fmax(fr, fabs(forcing[k].re));
        fi = fmax(fi, fabs(forcing[k].im));
    }
    auto wmax = [&](double v, int slot) {
        for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
        if ((threadIdx.x & 31) == 0) atomicMax(umax + slot, (unsigned long long)__double_as_longlong(v));
    };
#pragma unroll
    for (int k = 0; k < B; ++k) {
        wmax(lm[k], k);
        wmax(lr[k], B + k);
        wmax(li[k], 2 * B + k);
    }
    wmax(fr, 3 * B);
    wmax(fi, 3 * B + 1);
}

// directional_step (residual_ops.cpp:12-29) for both parts -> delta[0] (Re), delta[1] (Im)
template <int B>
__global__ void k_linres_delta(const unsigned long long* umax, double forcing_scale, double* delta) {
    if (threadIdx.x != 0) return;
    for (int part = 0; part < 2; ++part) {
        double ratio = 0.0;
        for (int k = 0; k < B; ++k) {
            const double ws = __longlong_as_double((long long)umax[k]);
            const double ds = __longlong_as_double((long long)umax[(1 + part) * B + k]);
            if (ds > 0.0) {
                const double wsc = ws > 1e-300 ? ws : 1e-300;
                const double r = ds / wsc;
                ratio = ratio > r ? ratio : r;
            }
        }
        const double fmx = __longlong_as_double((long long)umax[3 * B + part]);
        if (fmx > 0.0) {
            const double r = fmx / forcing_scale;
            ratio = ratio > r ? ratio : r;
        }
        delta[part] = ratio == 0.0 ? 0.0 : 1e-5 / ratio;
    }
}

// wp = mean + delta*dir, wm = mean - delta*dir, fp = delta*fdir, fm = -delta*fdir
__global__ void k_linres_states(std::size_t len, const double* __restrict__ mean, const cplx* __restrict__ what,
                                const cplx* __restrict__ forcing, int nforcing, int part,
                                const double* __restrict__ delta, double* __restrict__ wp, double* __restrict__ wm,
                                double* __restrict__ fp, double* __restrict__ fm) {
    const double d = delta[part];
    if (d == 0.0) return;
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t < len) {
        const double dir = part == 0 ? what[t].re : what[t].im;
        wp[t] = mean[t] + d * dir;
        wm[t] = mean[t] - d * dir;
    }
    if (t < (std::size_t)nforcing) {
        const double fd = part == 0 ? forcing[t].re : forcing[t].im;
        fp[t] = d * fd;
        fm[t] = -d * fd;
    }
}

// inv += unit * (inv_p - inv_m) * inv2d  (residual_ops.cpp:55-57,86)
__global__ void k_linres_combine(std::size_t len, int part, const double* __restrict__ delta,
                                 const double* __restrict__ ip, const double* __restrict__ im, cplx* __restrict__ out,
                                 int first) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    const double dl = delta[part];
    double dv = 0.0;
    if (dl != 0.0) {
        const double inv2d = 1.0 / (2.0 * dl);
        dv = (ip[t] - im[t]) * inv2d;
    }
    const double ur = part == 0 ? 1.0 : 0.0, ui = part == 0 ? 0.0 : 1.0;
    cplx o = first ? mk(0.0, 0.0) : out[t];
    o = o + mk(ur * dv, ui * dv);
    out[t] = o;
}

// ---------------------------------------------------------------------------
// DF helpers
// ---------------------------------------------------------------------------
__global__ void k_any_nonzero(std::size_t len, const cplx* __restrict__ a, int* flag) {
    for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < len;
         t += (std::size_t)gridDim.x * blockDim.x)
        if (a[t].re != 0.0 || a[t].im != 0.0) {
            *flag = 1;
            return;
        }
}

struct AmpList {
    const cplx* a[64];
};

// reconstruct_instantaneous (state.cpp:96-107)
__global__ void k_reconstruct(std::size_t len, const double* __restrict__ mean, AmpList amps, int nh,
                              const cplx* __restrict__ phase, double* __restrict__ out) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    double o = mean[t];
    for (int h = 0; h < nh; ++h) {
        const cplx a = amps.a[h][t];
        const cplx ph = phase[h];
        o += 2.0 * (a.re * ph.re - a.im * ph.im);
    }
    out[t] = o;
}

__global__ void k_accumulate(std::size_t len, const double* __restrict__ x, double* __restrict__ acc, int first) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    acc[t] = first ? 0.0 + x[t] : acc[t] + x[t];
}

__global__ void k_df_finish(std::size_t len, double nq, const double* __restrict__ acc, const double* __restrict__ inv,
                            double* __restrict__ df, int divide, const int* __restrict__ any) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    if (!*any) {  // all amplitudes zero: DF is exactly zero (residual_ops.cpp:139-141)
        df[t] = 0.0;
        return;
    }
    const double a = divide ? acc[t] / nq : acc[t];
    df[t] = a - inv[t];
}

// ---------------------------------------------------------------------------
// stage kernels
// ---------------------------------------------------------------------------
template <class S>
__global__ void k_blend(double beta, const S* __restrict__ vf, S* __restrict__ vb, std::size_t len) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    vb[t] = beta * vf[t] + (1.0 - beta) * vb[t];
}

template <class S>
__global__ void k_rhs(const S* __restrict__ inv, const S* __restrict__ vb, S* __restrict__ rhs, std::size_t len) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    const S r = inv[t] + vb[t];
    rhs[t] = -r;
}

template <class S>
__global__ void k_rhs_forced(const S* __restrict__ inv, const S* __restrict__ vb, const S* __restrict__ f,
                             S* __restrict__ rhs, std::size_t len) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    S r = inv[t] + vb[t];
    r -= f[t];
    rhs[t] = -r;
}

template <class S>
__global__ void k_scale(S* __restrict__ x, double a, std::size_t len) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    x[t] = x[t] * a;
}

template <class S>
__global__ void k_add(S* __restrict__ x, const S* __restrict__ y, std::size_t len) {
    const std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x;
    if (t >= len) return;
    x[t] = x[t] + y[t];
}

template <int B>
__device__ __forceinline__ void transform_jacobian_reg(const double* w, double g, double (&M)[B * B]) {
    const double rho = w[0], u = w[1], v = w[2], ww = w[3];
#pragma unroll
    for (int k = 0; k < B * B; ++k) M[k] = 0.0;
    M[0 * B + 0] = 1.0;
    M[1 * B + 0] = u;
    M[1 * B + 1] = rho;
    M[2 * B + 0] = v;
    M[2 * B + 2] = rho;
    M[3 * B + 0] = ww;
    M[3 * B + 3] = rho;
    M[4 * B + 0] = 0.5 * u * u + 0.5 * v * v + 0.5 * ww * ww;
    M[4 * B + 1] = rho * u;
    M[4 * B + 2] = rho * v;
    M[4 * B + 3] = rho * ww;
    M[4 * B + 4] = 1.0 / (g - 1.0);
    if constexpr (B == 6) {
        M[5 * B + 0] = w[5];
        M[5 * B + 5] = rho;
    }
}

template <int B>
__global__ void k_spectral(int n, double g, double omega, const double* __restrict__ vol,
                           const double* __restrict__ mean, const cplx* __restrict__ what, cplx* __restrict__ inv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double M[B * B];
    transform_jacobian_reg<B>(mean + (size_t)i * B, g, M);
    cplx wi[B], mw[B];
    load_vec<B>(what + (size_t)i * B, wi);
#pragma unroll
    for (int r = 0; r < B; ++r) {
        cplx acc = mk(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < B; ++c) acc += mk(M[r * B + c] * wi[c].re, M[r * B + c] * wi[c].im);
        mw[r] = acc;
    }
    const cplx iwv = mk(0.0, omega * vol[i]);
#pragma unroll
    for (int r = 0; r < B; ++r) inv[(size_t)i * B + r] += iwv * mw[r];
}

template <int B>
__global__ void k_apply_harmonic(int n, double g, const double* __restrict__ mean, const cplx* __restrict__ base,
                                 const cplx* __restrict__ x, cplx* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double M[B * B];
    int piv[B];
    transform_jacobian_reg<B>(mean + (size_t)i * B, g, M);
    double cond;
    lu_factor_reg<B>(M, piv, cond);
    double re[B], im[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
        const cplx v = x[(size_t)i * B + k];
        re[k] = v.re;
        im[k] = v.im;
    }
    lu_solve_reg<B>(M, piv, re);
    lu_solve_reg<B>(M, piv, im);
#pragma unroll
    for (int k = 0; k < B; ++k) out[(size_t)i * B + k] = base[(size_t)i * B + k] + mk(re[k], im[k]);
}

template <int B>
__global__ void k_apply_mean(int n, double g, const double* __restrict__ base, const double* __restrict__ x,
                             double* __restrict__ out, unsigned long long* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* w = base + (size_t)i * B;
    if (!admissible<B>(w)) {
        record(err, (unsigned long long)i, 2);
        return;
    }
    double q[B], o[B];
    prim_to_cons<B>(w, g, q);
#pragma unroll
    for (int k = 0; k < B; ++k) q[k] += x[(size_t)i * B + k];
    if (cons_to_prim<B>(q, g, o)) {
        record(err, (unsigned long long)i, 2);
        return;
    }
    store_vec<B>(out + (size_t)i * B, o);
}

template <class S>
__global__ void k_check_finite(const S* __restrict__ x, std::size_t len, unsigned long long* err) {
    for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < len;
         t += (std::size_t)gridDim.x * blockDim.x)
        if (!finite_(x[t])) {
            record(err, (unsigned long long)t, 6);
            return;
        }
}

#define DISPATCH_B56(b, ...)                                                          \
    switch (b) {                                                                      \
        case 5: { constexpr int B = 5; __VA_ARGS__; } break;                          \
        case 6: { constexpr int B = 6; __VA_ARGS__; } break;                          \
        default: throw ShapeError("discretization supports b = 5 or 6, got " + std::to_string(b)); \
    }

}  // namespace

// ---------------------------------------------------------------------------
// DeviceDisc
// ---------------------------------------------------------------------------
DeviceDisc::DeviceDisc(const MeshArrays& m, const DevicePattern* pattern) : pat_(pattern) {
    if (m.b != 5 && m.b != 6) throw ShapeError("discretization supports b = 5 or 6");
    if (pattern->rows != m.n || pattern->b != m.b) throw ShapeError("disc: pattern shape mismatch");
    const int nfc = m.nf, n = m.n;
    fa_.upload(m.fa, nfc);
    fb_.upload(m.fb, nfc);
    fbc_.upload(m.fbc, nfc);
    ford_.upload(m.ford, nfc);
    fn_.upload(m.fn, 3 * (std::size_t)nfc);
    farea_.upload(m.farea, nfc);
    fnh_.upload(m.fnh, 3 * (std::size_t)nfc);
    fvis_.upload(m.fvis, nfc);
    vol_.upload(m.vol, n);
    closure_.upload(m.closure, 3 * (std::size_t)n);
    mu_.upload(m.mu, n);
    nf_ptr_.upload(m.nf_ptr, n + 1);
    nf_idx_.upload(m.nf_idx, m.nf_ptr[n]);
    {  // boundary faces as the tail of the face list -> the split FD Jacobian
        int first_b = nfc;
        for (int f = 0; f < nfc; ++f)
            if (m.fbc[f] >= 0) {
                first_b = f;
                break;
            }
        bool tail = true;
        for (int f = first_b; f < nfc && tail; ++f) tail = m.fbc[f] >= 0;
        nf_int_ = tail ? first_b : -1;
        std::vector<int> bn;
        for (int i = 0; i < n; ++i)
            for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e)
                if (m.fbc[m.nf_idx[e]] >= 0) {
                    bn.push_back(i);
                    break;
                }
        nbn_ = static_cast<int>(bn.size());
        if (nbn_) bnodes_.upload(bn.data(), bn.size());
        if (nf_int_ >= 0) fdpart_.alloc((std::size_t)n * m.b * m.b);
    }
    bflag_.upload(m.bflag, n);
    int line = 0;  // the reference's line mesh: interior faces exactly (i, i+1), i = 0 .. n-2
    {
        std::vector<char> seen(n, 0);
        int cnt = 0;
        bool ok = n >= 2;
        for (int f = 0; f < nfc && ok; ++f) {
            if (m.fbc[f] >= 0) continue;
            const int a = m.fa[f];
            if (a < 0 || a + 1 >= n || m.fb[f] != a + 1 || seen[a]) ok = false;
            else {
                seen[a] = 1;
                ++cnt;
            }
        }
        line = ok && cnt == n - 1;
    }
    if (const double* T = libm_pow_tables()) powtab_.upload(T, kPowTabDoubles);
    if (nf_int_ >= 0 && !packed_disabled() && !line) {  // interior face records of the packed residual
        std::vector<double> g((std::size_t)nf_int_ * 8);
        for (int f = 0; f < nf_int_; ++f) {
            double* r = g.data() + (std::size_t)f * 8;
            for (int d = 0; d < 3; ++d) {
                r[d] = m.fn[3 * (std::size_t)f + d];
                r[3 + d] = m.fnh[3 * (std::size_t)f + d];
            }
            r[6] = m.farea[f];
            const long long ab = ((long long)(unsigned)m.fb[f] << 32) | (long long)(unsigned)m.fa[f];
            std::memcpy(r + 7, &ab, sizeof ab);
        }
        fgeo_.upload(g.data(), g.size());
    }
    {
        std::vector<int> code(m.nf_ptr[n]);
        for (int i = 0; i < n; ++i)
            for (int e = m.nf_ptr[i]; e < m.nf_ptr[i + 1]; ++e) {
                const int f = m.nf_idx[e];
                code[e] = m.fbc[f] >= 0 ? kBoundaryFace : m.fa[f] == i ? m.fb[f] : -(m.fa[f] + 1);
            }
        nf_code_.upload(code.data(), code.size());
    }
    // per-face BSR entries of (a,b) and (b,a) for the FD scatter (find, sparse.cpp:42-48)
    std::vector<int> eab(nfc, -1), eba(nfc, -1);
    auto find = [&](int i, int j) {
        auto b0 = pattern->h_col_idx.begin() + pattern->h_row_ptr[i];
        auto b1 = pattern->h_col_idx.begin() + pattern->h_row_ptr[i + 1];
        auto it = std::lower_bound(b0, b1, j);
        if (it == b1 || *it != j) throw ShapeError("disc: face endpoints not adjacent in the pattern");
        return static_cast<int>(it - pattern->h_col_idx.begin());
    };
    for (int f = 0; f < nfc; ++f)
        if (m.fbc[f] < 0) {
            eab[f] = find(m.fa[f], m.fb[f]);
            eba[f] = find(m.fb[f], m.fa[f]);
        }
    e_ab_.upload(eab.data(), nfc);
    e_ba_.upload(eba.data(), nfc);
    view_ = MeshDev{n, nfc, m.b, fa_.ptr, fb_.ptr, fbc_.ptr, ford_.ptr, fn_.ptr, farea_.ptr, fnh_.ptr, fvis_.ptr,
                    vol_.ptr, closure_.ptr, mu_.ptr, nf_ptr_.ptr, nf_idx_.ptr, bflag_.ptr, m.gamma, m.gas_constant,
                    m.p0, m.T0, m.p_out, m.nt_in, m.forcing_scale, nf_code_.ptr, powtab_.ptr, line};
    qscale_.alloc(8);
    ensure_contexts(1);
    err_.alloc(1);
    umax_.alloc(64);

    FNLH_CUDA(cudaMemset(err_.ptr, 0xff, sizeof(unsigned long long)));
    legacy_sync();
}

DeviceDisc::~DeviceDisc() {
    for (auto e : df_ev_) cudaEventDestroy(e);
}

void DeviceDisc::alloc_scratch(Scratch& c) {
    const std::size_t n = view_.n, nfc = view_.nf, b = view_.b;
    c.nu.alloc(n);
    c.lap.alloc(n * b);
    c.flux.alloc(nfc * std::max<std::size_t>(b, kFS));
    c.vflux.alloc(nfc * std::max<std::size_t>(b, kFS));
    if (fgeo_.ptr) c.rec.alloc(n * (2 * b + 2));
    c.scal.alloc(16);
    c.umax.alloc(64);
    for (auto& r : c.real) r.alloc(n * b);
}

void DeviceDisc::ensure_contexts(int k) {
    while (static_cast<int>(ctx_.size()) < k) {
        ctx_.push_back(std::make_unique<Scratch>());
        alloc_scratch(*ctx_.back());
    }
}

void DeviceDisc::reset_err(cudaStream_t st) {
    FNLH_CUDA(cudaMemsetAsync(err_.ptr, 0xff, sizeof(unsigned long long), st));
}

int DeviceDisc::read_err(cudaStream_t st, long long* key) {
    unsigned long long h = 0;
    FNLH_CUDA(cudaMemcpyAsync(&h, err_.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
    FNLH_CUDA(cudaStreamSynchronize(st));
    if (h == ~0ull) return 0;
    if (key) *key = (long long)(h >> 4);
    return (int)(h & 15ull);
}

void DeviceDisc::raise_if_err(cudaStream_t st, const char* what) {
    long long key = -1;
    const int code = read_err(st, &key);
    if (!code) return;
    reset_err(st);
    const std::string w(what);
    switch (code) {
        case 2: throw StateError(w + ": inadmissible state");
        case 4: throw UnsupportedCaseError(w + ": supersonic boundary state");
        case 5: throw FactorizationError(w + ": singular diagonal block", (int)key);
        case 6: throw DivergenceError(w + ": non-finite value", 0);
        default: throw std::runtime_error(w + ": device error " + std::to_string(code));
    }
}

void DeviceDisc::residual(const double* W, const double* wref, int order, int mode, const double* forcing,
                          int nforcing, bool need_vis, double* inv, double* vis, cudaStream_t st,
                          const double* skip) {
    const MeshDev& m = view_;
    if (order == 2 && fgeo_.ptr) {  // packed records (boundary faces the tail)
        DISPATCH_B56(m.b, {
            { ::fnlh::note_launch(); k_jst_prepass_rec<B><<<nb(m.n), kT, 0, st>>>(m, W, C().rec.ptr, skip); }
            const int nbb = nb(m.nf - nf_int_), nbi = nb(nf_int_);
            if (nbb + nbi) { ::fnlh::note_launch(); k_face_packed<B><<<nbb + nbi, kT, 0, st>>>(m, nf_int_, nbb, fgeo_.ptr, C().rec.ptr, W, wref, mode, forcing, nforcing, need_vis ? 1 : 0, C().flux.ptr, C().vflux.ptr, err(), skip); }
            { ::fnlh::note_launch(); k_node_gather_p<B><<<nb(m.n), kT, 0, st>>>(m, W, C().flux.ptr, C().vflux.ptr, need_vis ? 1 : 0, inv, vis, skip); }
        });
        FNLH_CUDA(cudaGetLastError());
        return;
    }
    DISPATCH_B56(m.b, {
        if (order == 2) { ::fnlh::note_launch(); k_jst_prepass<B><<<nb(m.n), kT, 0, st>>>(m, W, C().nu.ptr, C().lap.ptr, skip); }
        { ::fnlh::note_launch(); k_face_flux<B><<<nb(m.nf), kT, 0, st>>>(m, W, wref, order, mode, forcing, nforcing, need_vis ? 1 : 0,
                                                C().nu.ptr, C().lap.ptr, C().flux.ptr, C().vflux.ptr, err(), skip); }
        { ::fnlh::note_launch(); k_node_gather<B><<<nb(m.n), kT, 0, st>>>(m, W, C().flux.ptr, C().vflux.ptr, need_vis ? 1 : 0, inv, vis, skip); }
    });
    FNLH_CUDA(cudaGetLastError());
}

void DeviceDisc::validate(const double* W, cudaStream_t st) {
    DISPATCH_B56(view_.b, { { ::fnlh::note_launch(); k_validate<B><<<nb(view_.n), kT, 0, st>>>(view_.n, W, err_.ptr); } });
    raise_if_err(st, "validate_state");
}

void DeviceDisc::fd_jacobian(const double* W, double* J, double* P, cudaStream_t st, const A5Target* a5) {
    const MeshDev& m = view_;
    validate(W, st);
    const long long* smap = nullptr;
    double ga = 1.0, inv_es = 0.0;
    int to_a5 = 0;
    if (a5) {  // A5 straight from the FD columns; J_ii kept aside for the singularity check
        if (J) throw ConfigError("fd_jacobian: J and an A5 target are exclusive");
        J = a5->vals;
        smap = a5->sell_map;
        ga = a5->ga;
        inv_es = a5->inv_es;
        to_a5 = 1;
        if (!P) {
            if (!fddiag_.ptr) fddiag_.alloc((std::size_t)m.n * m.b * m.b);
            P = fddiag_.ptr;
        }
        FNLH_CUDA(cudaMemsetAsync(J, 0, a5->bytes, st));
    } else if (J) {
        FNLH_CUDA(cudaMemsetAsync(J, 0, (std::size_t)pat_->nnzb * m.b * m.b * sizeof(double), st));
    }
    DISPATCH_B56(m.b, {
        { ::fnlh::note_launch(); k_umax_init<<<1, 32, 0, st>>>(umax_.ptr, B); }
        { ::fnlh::note_launch(); k_qscale<B><<<std::min(nb(m.n), 592), kT, 0, st>>>(m.n, m.gamma, W, umax_.ptr); }
        { ::fnlh::note_launch(); k_qscale_finish<B><<<1, 32, 0, st>>>(umax_.ptr, qscale_.ptr); }
        if (nf_int_ >= 0) {
            { ::fnlh::note_launch(); k_fd_jacobian<B, 1><<<nb((long long)m.n * B), kT, 0, st>>>(m, pat_->diag_idx, e_ab_.ptr, e_ba_.ptr, W,
                                                                       qscale_.ptr, J, P, err_.ptr, nullptr, 0, fdpart_.ptr,
                                                                       smap, ga, inv_es, to_a5); }
            if (nbn_ > 0) { ::fnlh::note_launch(); k_fd_jacobian<B, 2><<<nb((long long)nbn_ * B), kT, 0, st>>>(m, pat_->diag_idx, e_ab_.ptr, e_ba_.ptr, W,
                                                                                    qscale_.ptr, J, P, err_.ptr, bnodes_.ptr, nbn_,
                                                                                    fdpart_.ptr, smap, ga, inv_es, to_a5); }
        } else {
            { ::fnlh::note_launch(); k_fd_jacobian<B, 0><<<nb((long long)m.n * B), kT, 0, st>>>(m, pat_->diag_idx, e_ab_.ptr, e_ba_.ptr, W,
                                                                       qscale_.ptr, J, P, err_.ptr, nullptr, 0, nullptr,
                                                                       smap, ga, inv_es, to_a5); }
        }
    });
    FNLH_CUDA(cudaGetLastError());
    raise_if_err(st, "fd_jacobian");
    if (J) {  // diagonal non-singularity check of J (disc.cpp:121-129)
        const int* didx = a5 ? nullptr : pat_->diag_idx;
        const double* blocks = a5 ? P : J;
        DISPATCH_B56(m.b, { { ::fnlh::note_launch(); k_diag_check<B><<<nb(m.n), kT, 0, st>>>(m.n, didx, blocks, err_.ptr); } });
        raise_if_err(st, "fd_jacobian");
    }
}

void DeviceDisc::linearized_residual(const double* mean, const cplx* what, double omega, const cplx* forcing,
                                     int nforcing, int order, bool need_vis, cplx* inv, cplx* vis, cudaStream_t st) {
    if (omega < 0.0) throw ConfigError("linearized_residual: negative frequency");
    const MeshDev& m = view_;
    const std::size_t L = len();
    Scratch& cx = C();
    if (nforcing > 0 && (std::size_t)cx.fwork.n < 2 * (std::size_t)nforcing) cx.fwork.alloc(2 * (std::size_t)nforcing);
    double* wp = cx.real[0].ptr;
    double* wm = cx.real[1].ptr;
    double* ip = cx.real[2].ptr;
    double* vp = cx.real[3].ptr;
    double* imn = cx.real[4].ptr;
    double* vm = cx.real[5].ptr;
    double* fp = nforcing > 0 ? cx.fwork.ptr : nullptr;
    double* fm = nforcing > 0 ? cx.fwork.ptr + nforcing : nullptr;
    double* delta = cx.scal.ptr;
    const int grid = std::min(nb(m.n), 592);
    DISPATCH_B56(m.b, {
        { ::fnlh::note_launch(); k_umax_init<<<1, 32, 0, st>>>(cx.umax.ptr, 3 * B + 2); }
        { ::fnlh::note_launch(); k_linres_scales<B><<<grid, kT, 0, st>>>(m.n, mean, what, forcing, nforcing, cx.umax.ptr); }
        { ::fnlh::note_launch(); k_linres_delta<B><<<1, 32, 0, st>>>(cx.umax.ptr, m.forcing_scale, delta); }
    });
    const int gs = nb((long long)std::max<std::size_t>(L, (std::size_t)nforcing));
    for (int part = 0; part < 2; ++part) {
        { ::fnlh::note_launch(); k_linres_states<<<gs, kT, 0, st>>>(L, mean, what, forcing, nforcing, part, delta, wp, wm, fp, fm); }
        residual(wp, mean, order, 1, fp, nforcing, need_vis, ip, vp, st, delta + part);
        residual(wm, mean, order, 1, fm, nforcing, need_vis, imn, vm, st, delta + part);
        { ::fnlh::note_launch(); k_linres_combine<<<nb(L), kT, 0, st>>>(L, part, delta, ip, imn, inv, part == 0); }
        if (need_vis) { ::fnlh::note_launch(); k_linres_combine<<<nb(L), kT, 0, st>>>(L, part, delta, vp, vm, vis, part == 0); }
    }
    DISPATCH_B56(m.b, { { ::fnlh::note_launch(); k_spectral<B><<<nb(m.n), kT, 0, st>>>(m.n, m.gamma, omega, vol_.ptr, mean, what, inv); } });
    FNLH_CUDA(cudaGetLastError());
}

// HarmonicSpec::base_frequency / max_multiple (case.cpp:10-44)
void base_frequency(const std::vector<double>& omega, double& base, int& lmax) {
    const double rel_tol = 1e-9;
    std::vector<double> ws;
    for (double w : omega)
        if (w > 0.0) ws.push_back(w);
    lmax = 0;
    base = 0.0;
    if (ws.empty()) return;
    const double scale = *std::max_element(ws.begin(), ws.end());
    double g = ws[0];
    for (std::size_t i = 1; i < ws.size(); ++i) {
        double a = std::max(g, ws[i]);
        double b = std::min(g, ws[i]);
        while (b > rel_tol * scale) {
            const double r = std::fmod(a, b);
            a = b;
            b = r;
        }
        g = a;
    }
    if (g < 1e-6 * scale) throw ConfigError("harmonic frequencies are incommensurate");
    for (double w : ws) {
        const double mm = w / g;
        if (std::abs(mm - std::round(mm)) > 1e-6) throw ConfigError("harmonic frequencies are incommensurate");
    }
    base = g;
    for (double w : omega)
        if (w > 0.0) lmax = std::max(lmax, static_cast<int>(std::llround(w / g)));
}

void DeviceDisc::deterministic_flux(const double* mean, const std::vector<const cplx*>& amps,
                                    const std::vector<double>& omega, double* df, cudaStream_t st, bool deferred,
                                    const std::vector<cudaStream_t>& side) {
    const std::size_t L = len();
    const int nh = static_cast<int>(amps.size());
    if (nh > 64) throw ConfigError("deterministic_flux: at most 64 harmonics");
    double base;
    int lmax;
    base_frequency(omega, base, lmax);
    // any nonzero amplitude?  (residual_ops.cpp:133-141) -- decided on the device in k_df_finish
    if (!df_flag_.ptr) df_flag_.alloc(1);
    FNLH_CUDA(cudaMemsetAsync(df_flag_.ptr, 0, sizeof(int), st));
    for (int h = 0; h < nh; ++h) { ::fnlh::note_launch(); k_any_nonzero<<<std::min(nb((long long)L), 592), kT, 0, st>>>(L, amps[h], df_flag_.ptr); }
    AmpList al{};
    for (int h = 0; h < nh; ++h) al.a[h] = amps[h];
    const int nq = lmax == 0 ? 1 : 4 * lmax + 2;
    if (omega != df_omega_ || !df_ph_.ptr) {
        std::vector<std::complex<double>> ph((std::size_t)nq * std::max(nh, 1));
        const double period = lmax == 0 ? 0.0 : 2.0 * std::acos(-1.0) / base;
        for (int k = 0; k < nq; ++k) {
            const double t = lmax == 0 ? 0.0 : period * k / nq;
            for (int h = 0; h < nh; ++h) ph[(std::size_t)k * nh + h] = std::exp(std::complex<double>(0.0, omega[h] * t));
        }
        FNLH_CUDA(cudaStreamSynchronize(st));  // the previous phase table may still be in use
        df_ph_.upload(reinterpret_cast<const cplx*>(ph.data()), ph.size());
        df_omega_ = omega;
    }
    const cplx* dph = df_ph_.ptr;
    const int saved = cur_;
    double* acc = ctx_[saved]->real[2].ptr;
    // the nq reconstructions + residuals are independent: up to 1 + side.size() of them run
    // at once (context c on side stream c-1), the sum is then taken in k order on st
    const int NC = saved != 0 ? 1 : 1 + static_cast<int>(std::min(side.size(), ctx_.size() - 1));
    while (static_cast<int>(df_ev_.size()) < NC + 1) {
        cudaEvent_t e;
        FNLH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        df_ev_.push_back(e);
    }
    for (int k0 = 0; k0 < nq; k0 += NC) {
        FNLH_CUDA(cudaEventRecord(df_ev_[NC], st));  // the previous batch's sums are taken
        for (int c = 0; c < NC && k0 + c < nq; ++c) {
            const int k = k0 + c;
            const int cx = c == 0 ? saved : c;
            cudaStream_t sc = c == 0 ? st : side[c - 1];
            if (c > 0) FNLH_CUDA(cudaStreamWaitEvent(sc, df_ev_[NC], 0));
            cur_ = cx;
            { ::fnlh::note_launch(); k_reconstruct<<<nb((long long)L), kT, 0, sc>>>(L, mean, al, nh, dph + (std::size_t)k * nh, C().real[0].ptr); }
            residual(C().real[0].ptr, nullptr, 2, 0, nullptr, 0, false, C().real[1].ptr, nullptr, sc);
            if (c > 0) FNLH_CUDA(cudaEventRecord(df_ev_[c], sc));
        }
        cur_ = saved;
        for (int c = 0; c < NC && k0 + c < nq; ++c) {
            const int k = k0 + c;
            if (c > 0) FNLH_CUDA(cudaStreamWaitEvent(st, df_ev_[c], 0));
            const double* inv_k = ctx_[c == 0 ? saved : c]->real[1].ptr;
            { ::fnlh::note_launch(); k_accumulate<<<nb((long long)L), kT, 0, st>>>(L, inv_k, acc, k == 0); }
        }
    }
    double* inv = C().real[1].ptr;
    residual(mean, nullptr, 2, 0, nullptr, 0, false, inv, nullptr, st);
    { ::fnlh::note_launch(); k_df_finish<<<nb((long long)L), kT, 0, st>>>(L, (double)nq, acc, inv, df, lmax == 0 ? 0 : 1, df_flag_.ptr); }
    FNLH_CUDA(cudaGetLastError());
    if (!deferred) raise_if_err(st, "deterministic_flux");
}

int DeviceDisc::df_points(const std::vector<double>& omega) {
    double base;
    int lmax;
    base_frequency(omega, base, lmax);
    return lmax == 0 ? 1 : 4 * lmax + 2;
}

void DeviceDisc::df_terms(const double* mean, const std::vector<const cplx*>& amps, const std::vector<double>& omega,
                          int k0, int k1, double* terms, cudaStream_t st) {
    const std::size_t L = len();
    const int nh = static_cast<int>(amps.size());
    if (nh > 64) throw ConfigError("deterministic_flux: at most 64 harmonics");
    double base;
    int lmax;
    base_frequency(omega, base, lmax);
    const int nq = lmax == 0 ? 1 : 4 * lmax + 2;
    if (k0 < 0 || k1 > nq || k0 > k1) throw ShapeError("df_terms: quadrature range outside [0, nq)");
    if (omega != df_omega_ || !df_ph_.ptr) {  // the same phase table deterministic_flux builds
        std::vector<std::complex<double>> ph((std::size_t)nq * std::max(nh, 1));
        const double period = lmax == 0 ? 0.0 : 2.0 * std::acos(-1.0) / base;
        for (int k = 0; k < nq; ++k) {
            const double t = lmax == 0 ? 0.0 : period * k / nq;
            for (int h = 0; h < nh; ++h) ph[(std::size_t)k * nh + h] = std::exp(std::complex<double>(0.0, omega[h] * t));
        }
        FNLH_CUDA(cudaStreamSynchronize(st));
        df_ph_.upload(reinterpret_cast<const cplx*>(ph.data()), ph.size());
        df_omega_ = omega;
    }
    AmpList al{};
    for (int h = 0; h < nh; ++h) al.a[h] = amps[h];
    for (int k = k0; k < k1; ++k) {
        { ::fnlh::note_launch(); k_reconstruct<<<nb((long long)L), kT, 0, st>>>(L, mean, al, nh, df_ph_.ptr + (std::size_t)k * nh, C().real[0].ptr); }
        residual(C().real[0].ptr, nullptr, 2, 0, nullptr, 0, false, terms + (std::size_t)(k - k0) * L, nullptr, st);
    }
    FNLH_CUDA(cudaGetLastError());
    raise_if_err(st, "deterministic_flux");
}

void DeviceDisc::df_accumulate(const double* terms, int count, double* acc, bool first, cudaStream_t st) {
    const std::size_t L = len();
    for (int j = 0; j < count; ++j) {
        ::fnlh::note_launch();
        k_accumulate<<<nb((long long)L), kT, 0, st>>>(L, terms + (std::size_t)j * L, acc, first && j == 0);
    }
    FNLH_CUDA(cudaGetLastError());
}

void DeviceDisc::df_finish(const double* mean, const std::vector<const cplx*>& amps, const std::vector<double>& omega,
                           const double* acc, double* df, cudaStream_t st, bool deferred) {
    const std::size_t L = len();
    double base;
    int lmax;
    base_frequency(omega, base, lmax);
    const int nq = lmax == 0 ? 1 : 4 * lmax + 2;
    if (!df_flag_.ptr) df_flag_.alloc(1);
    FNLH_CUDA(cudaMemsetAsync(df_flag_.ptr, 0, sizeof(int), st));
    for (std::size_t h = 0; h < amps.size(); ++h) {
        ::fnlh::note_launch();
        k_any_nonzero<<<std::min(nb((long long)L), 592), kT, 0, st>>>(L, amps[h], df_flag_.ptr);
    }
    double* inv = C().real[1].ptr;
    residual(mean, nullptr, 2, 0, nullptr, 0, false, inv, nullptr, st);
    { ::fnlh::note_launch(); k_df_finish<<<nb((long long)L), kT, 0, st>>>(L, (double)nq, acc, inv, df, lmax == 0 ? 0 : 1, df_flag_.ptr); }
    FNLH_CUDA(cudaGetLastError());
    if (!deferred) raise_if_err(st, "deterministic_flux");
}

// ---------------------------------------------------------------------------
template <class S>
void stage_blend(double beta, const S* vf, S* vb, std::size_t len, cudaStream_t st) {
    { ::fnlh::note_launch(); k_blend<S><<<nb((long long)len), kT, 0, st>>>(beta, vf, vb, len); }
}
template <class S>
void stage_rhs(const S* inv, const S* vb, S* rhs, std::size_t len, cudaStream_t st) {
    { ::fnlh::note_launch(); k_rhs<S><<<nb((long long)len), kT, 0, st>>>(inv, vb, rhs, len); }
}
template <class S>
void stage_rhs_forced(const S* inv, const S* vb, const S* f, S* rhs, std::size_t len, cudaStream_t st) {
    { ::fnlh::note_launch(); k_rhs_forced<S><<<nb((long long)len), kT, 0, st>>>(inv, vb, f, rhs, len); }
}
template <class S>
void scale(S* x, double a, std::size_t len, cudaStream_t st) {
    { ::fnlh::note_launch(); k_scale<S><<<nb((long long)len), kT, 0, st>>>(x, a, len); }
}
template <class S>
void add_inplace(S* x, const S* y, std::size_t len, cudaStream_t st) {
    { ::fnlh::note_launch(); k_add<S><<<nb((long long)len), kT, 0, st>>>(x, y, len); }
}
template <class S>
void check_finite(const S* x, std::size_t len, unsigned long long* err, cudaStream_t st) {
    { ::fnlh::note_launch(); k_check_finite<S><<<std::min(nb((long long)len), 592), kT, 0, st>>>(x, len, err); }
}

void apply_harmonic(int b, int n, double gamma, const double* mean, const cplx* base, const cplx* x, cplx* out,
                    cudaStream_t st) {
    DISPATCH_B56(b, { { ::fnlh::note_launch(); k_apply_harmonic<B><<<nb(n), kT, 0, st>>>(n, gamma, mean, base, x, out); } });
}

void apply_mean(int b, int n, double gamma, const double* base, const double* x, double* out,
                unsigned long long* err, cudaStream_t st) {
    DISPATCH_B56(b, { { ::fnlh::note_launch(); k_apply_mean<B><<<nb(n), kT, 0, st>>>(n, gamma, base, x, out, err); } });
}

#define INST(S)                                                                         \
    template void stage_blend<S>(double, const S*, S*, std::size_t, cudaStream_t);      \
    template void stage_rhs<S>(const S*, const S*, S*, std::size_t, cudaStream_t);      \
    template void stage_rhs_forced<S>(const S*, const S*, const S*, S*, std::size_t, cudaStream_t); \
    template void scale<S>(S*, double, std::size_t, cudaStream_t);                      \
    template void add_inplace<S>(S*, const S*, std::size_t, cudaStream_t);              \
    template void check_finite<S>(const S*, std::size_t, unsigned long long*, cudaStream_t);
INST(double)
INST(cplx)

}  // namespace fnlh
