// rb.cu -- 2-colour fused ILU(0)-Richardson sweep (see rb.cuh for the derivation).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "rb.cuh"

namespace fnlh {

namespace {

constexpr int kT = 128;  // 4 slices of 32 rows per CTA
#ifndef RBE_MINB
#define RBE_MINB 2  // resident CTAs per SM of the edge-parallel kernels (192 threads each)
#endif
inline int nb(long long n) { return static_cast<int>((n + kT - 1) / kT); }

struct SellDev {
    const long long* __restrict__ slice_val;
    const int* __restrict__ slice_col;
    const int* __restrict__ deg;
    const int* __restrict__ cols;
    const double* __restrict__ vals;
    int n, n0, nslices0;
};

struct RowRef {
    long long vbase;  // vals offset of (slot 0, element 0) for this row
    int cbase;        // cols offset of slot 0 for this row
    int deg;
};

__device__ __forceinline__ RowRef row_ref(const SellDev& L, int i) {
    const int li = i < L.n0 ? i : i - L.n0;
    const int s = (i < L.n0 ? 0 : L.nslices0) + (li >> 5);
    const int lane = li & 31;
    return RowRef{L.slice_val[s] + 2 * lane, L.slice_col[s] + lane, L.deg[i]};
}

template <int B>
__host__ __device__ constexpr int pairs() { return (B * B + 1) / 2; }

// inv(U_kk) of the colour-0 rows (RbIlu::inv0) is stored slice-major like the pivot LUs: node k
// -> slice k / 32, lane k % 32, element (m, c) of its block at [slice][m B + c][lane].  In a
// bandwidth-reducing (RCM) order the 32 rows of a warp gather from (nearly) consecutive
// neighbours, so the warp's load of one block element is a few contiguous 16-byte runs -- 4
// cache lines instead of 32 -- which is what the L1 tag stage was busy with (RB_U_AOS: the
// earlier one-block-per-node array, kept as a measurement build).
template <int B>
__host__ __device__ __forceinline__ std::size_t ubase(int node) {
#ifdef RB_U_AOS
    return (std::size_t)node * B * B;
#else
    return (std::size_t)(node >> 5) * 32 * B * B + (node & 31);
#endif
}
template <int B>
__host__ __device__ constexpr int uix(int m, int c) {
#ifdef RB_U_AOS
    return m * B + c;
#else
    return (m * B + c) * 32;
#endif
}


template <int B>
__device__ __forceinline__ double aval(const SellDev& L, const RowRef& r, int e, int k) {
    return __ldg(L.vals + r.vbase + ((long long)(e * pairs<B>() + (k >> 1)) * 32) * 2 + (k & 1));
}

// the whole b x b block, 16-byte loads (pairs of elements, lane-contiguous)
template <int B>
__device__ __forceinline__ void ablock(const SellDev& L, const RowRef& r, int e, double (&A)[2 * pairs<B>()]) {
    const double2* base = reinterpret_cast<const double2*>(L.vals + r.vbase) + (long long)e * pairs<B>() * 32;
#pragma unroll
    for (int p = 0; p < pairs<B>(); ++p) {
        const double2 v = __ldg(base + (long long)p * 32);
        A[2 * p] = v.x;
        A[2 * p + 1] = v.y;
    }
}

__device__ __forceinline__ int acol(const SellDev& L, const RowRef& r, int e) { return __ldg(L.cols + r.cbase + e * 32); }

// measurement switches of k_rbx_colour1 / k_rb_colour0: RB_IDXPF = load an edge's column index
// one edge ahead (no index -> gather round trip inside the edge), RB_UHOIST = issue all b x b
// loads of inv(U_kk) at the top of the edge (one round trip instead of one per column, more
// registers), RB_C1_MINB = resident-CTA hint of k_rbx_colour1 (0: the compiler's choice)
#ifndef RB_IDXPF
#define RB_IDXPF 1
#endif
#ifndef RB_UHOIST
#define RB_UHOIST 1
#endif
#ifndef RB_C1_MINB
#define RB_C1_MINB 3
#endif

// lu_solve_reg (block_lu_solve, dense.hpp:91-109) reading the LU entries from memory as it
// uses them (row phase of the edge-parallel kernels: no 25-entry register block)
template <int B, class S>
__device__ __forceinline__ void lu_solve_mem(const S* __restrict__ lu, long long stride, const int (&piv)[B], S (&x)[B]) {
#pragma unroll
    for (int k = 0; k < B; ++k) {
        const int p = piv[k];
#pragma unroll
        for (int r = k + 1; r < B; ++r)
            if (r == p) {
                S t = x[k];
                x[k] = x[r];
                x[r] = t;
            }
    }
#pragma unroll
    for (int r = 1; r < B; ++r) {
        S acc = x[r];
#pragma unroll
        for (int c = 0; c < r; ++c) acc -= lu[(r * B + c) * stride] * x[c];
        x[r] = acc;
    }
#pragma unroll
    for (int r = B - 1; r >= 0; --r) {
        S acc = x[r];
#pragma unroll
        for (int c = r + 1; c < B; ++c) acc -= lu[(r * B + c) * stride] * x[c];
        x[r] = acc / lu[(r * B + r) * stride];
    }
}

// pivot blocks (diag_lu) and pivots are stored slice-major like A: row i -> slice s,
// lane l; element k of the row at [s][k][l], so a warp's k-th load is 32 consecutive
// elements (rb.cuh RbIlu)
struct LuRef {
    long long lu;  // element offset of k = 0
    long long pv;
};
template <int B>
__device__ __forceinline__ LuRef lu_ref(const SellDev& L, int i) {
    const int li = i < L.n0 ? i : i - L.n0;
    const int s = (i < L.n0 ? 0 : L.nslices0) + (li >> 5);
    const int lane = li & 31;
    return LuRef{(long long)s * 32 * B * B + lane, (long long)s * 32 * B + lane};
}
template <int B, class S>
__device__ __forceinline__ void ld_lu(const S* __restrict__ dlu, const int* __restrict__ piv, const LuRef& q,
                                      S (&lu)[B * B], int (&pv)[B]) {
#pragma unroll
    for (int k = 0; k < B * B; ++k) lu[k] = dlu[q.lu + 32 * k];
#pragma unroll
    for (int k = 0; k < B; ++k) pv[k] = piv[q.pv + 32 * k];
}

// y[r] += sum_c A_e[r][c] x[c] (block_matvec_add, dense.hpp:20-28); the diagonal block of
// a shifted system carries complex(a + 0, 0 + s) on its diagonal (shift_diagonal)
template <int B, class S>
__device__ __forceinline__ void blk_matvec_add(const SellDev& L, const RowRef& rr, int e, const S (&x)[B],
                                               bool diag, double s, S (&y)[B]) {
    double A[2 * pairs<B>()];
    ablock<B>(L, rr, e, A);
#pragma unroll
    for (int r = 0; r < B; ++r) {
        S acc = zero<S>();
#pragma unroll
        for (int c = 0; c < B; ++c) {
            const double a = A[r * B + c];
            if constexpr (sizeof(S) == sizeof(cplx)) {
                if (diag && r == c)
                    acc += mk(a + 0.0, 0.0 + s) * x[c];
                else
                    acc += rmul(a, x[c]);
            } else {
                acc += rmul(a, x[c]);
            }
        }
        y[r] += acc;
    }
}

// y[r] -= sum_c A_e[r][c] x[c] (block_matvec_sub with U_ij = complex(A_ij))
template <int B, class S>
__device__ __forceinline__ void blk_matvec_sub(const SellDev& L, const RowRef& rr, int e, const S (&x)[B],
                                               S (&y)[B]) {
    double A[2 * pairs<B>()];
    ablock<B>(L, rr, e, A);
#pragma unroll
    for (int r = 0; r < B; ++r) {
        S acc = zero<S>();
#pragma unroll
        for (int c = 0; c < B; ++c) acc += rmul(A[r * B + c], x[c]);
        y[r] -= acc;
    }
}

template <int B, class S>
__device__ __forceinline__ void ld(const S* __restrict__ p, S (&v)[B]) {
#pragma unroll
    for (int k = 0; k < B; ++k) v[k] = p[k];
}
template <int B, class S>
__device__ __forceinline__ void st(S* __restrict__ p, const S (&v)[B]) {
#pragma unroll
    for (int k = 0; k < B; ++k) p[k] = v[k];
}

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kT / 32; ++w) s += red[w];
    return s;
}

// fixed-order sum of partials by a CTA of any size (deterministic run to run); thread 0
// receives the sum
__device__ double ordered_sum_n(const double* __restrict__ p, int n, double* red) {
    const int nt = blockDim.x;
    double s = 0.0;
    const int chunk = (n + nt - 1) / nt;
    const int b0 = threadIdx.x * chunk, b1 = min(n, b0 + chunk);
    for (int k = b0; k < b1; ++k) s += __ldcg(p + k);
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    __shared__ double wsum[32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (nt + 31) / 32; ++w) t += wsum[w];
    return t;
}

// fixed-order sum of partials by one CTA (deterministic run to run)
__device__ double ordered_sum(const double* __restrict__ p, int n, double* red) {
    double s = 0.0;
    const int chunk = (n + kT - 1) / kT;
    const int b0 = threadIdx.x * chunk, b1 = min(n, b0 + chunk);
    for (int k = b0; k < b1; ++k) s += p[k];
    __syncthreads();
    return block_sum(s, red);
}

// Lane-warp kernels (fnlh_set_rb_sweep(4)): the same total as ordered_sum over the 128-row
// partials q[k] of the 128-thread kernels, formed by ONE warp from per-slice (32-row)
// partials w: q[k] = ((w[4k] + w[4k+1]) + w[4k+2]) + w[4k+3] (block_sum's order), colour-0
// slices at [0, 4 grid0), colour-1 slices from 4 grid0; each thread plays the four virtual
// threads lane, lane+32, lane+64, lane+96 of the 128-thread reduction.  Thread 0 gets the sum.
__device__ double ordered_sum_lw(const double* __restrict__ p, int grid0, int grid1, int ns0, int ns1,
                                 bool c0_slices = true) {
    const int n = grid0 + grid1, lane = threadIdx.x & 31;
    const int chunk = (n + kT - 1) / kT;
    double sv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const int vt = v * 32 + lane;
        const int b0 = vt * chunk, b1 = min(n, b0 + chunk);
        double s = 0.0;
        for (int k = b0; k < b1; ++k) {
            const int lim = k < grid0 ? ns0 - 4 * k : ns1 - 4 * (k - grid0);  // slices of this group that exist
            double q = 0.0;
            if (!c0_slices && k < grid0) {  // colour 0 came from the 128-row kernel: q[k] itself at [k]
                q = __ldcg(p + k);
            } else {
#pragma unroll
                for (int w = 0; w < 4; ++w) q += w < lim ? __ldcg(p + 4 * k + w) : 0.0;
            }
            s += q;
        }
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        sv[v] = s;
    }
    double t = 0.0;
#pragma unroll
    for (int v = 0; v < 4; ++v) t += sv[v];
    return t;
}

// per-member operand table of a batched sweep: P independent systems that share the
// real A (one per harmonic in flight, driver.cpp:246-265 workers); CTA b serves member
// b % P, so the P CTAs touching the same slice of A run back to back and A comes from
// HBM once per sweep of the batch (L2 serves the rest)
template <class S>
struct RbTab {
    const S* diag_lu[kMaxBatch];
    const int* piv[kMaxBatch];
    const S* inv0[kMaxBatch];
    const double* shift[kMaxBatch];
    const S* rhs[kMaxBatch];
    S* x[kMaxBatch];
    S* z[kMaxBatch];
    S* r[kMaxBatch];
    RbControl* ctl[kMaxBatch];
    double* parts[kMaxBatch];
    int P;
};

// ---- pre-kernel: ||b||, target, x = 0 --------------------------------------
template <class S>
__global__ void k_rb_init(std::size_t len, const RbTab<S> T, double tol) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    __shared__ bool last;
    double loc = 0.0;
    for (std::size_t t = cta * (std::size_t)kT + threadIdx.x; t < len; t += (std::size_t)nct * kT)
        loc += sq(rhs[t]);
    const double bs = block_sum(loc, red);
    if (threadIdx.x == 0) {
        partials[cta] = bs;
        __threadfence();
        last = atomicAdd(counter, 1u) == nct - 1;
    }
    __syncthreads();
    if (!last) return;
    const double tot = ordered_sum(partials, nct, red);
    if (threadIdx.x == 0) {
        const double r0 = sqrt(tot);
        ctl->initial_residual = r0;
        ctl->final_residual = r0;
        ctl->target = tol * r0;
        ctl->iterations = 0;
        ctl->converged = r0 == 0.0 ? 1 : 0;
        ctl->done = r0 == 0.0 ? 1 : 0;
        ctl->status = 0;
        *counter = 0u;
    }
}

// ---- K_F: colour 1 forward substitution -------------------------------------
// zf = r_i - sum_k L_ik r_k (ascending k, sparse.cpp:267-278) with L_ik = A_ik inv(U_kk)
// rebuilt in the reference's order (sparse.cpp:221-232); colour 1 rows have no upper
// entries, so the backward step is the pivot solve alone.
template <int B, class S>
__global__ void __launch_bounds__(kT) k_rb_forward1(SellDev L, const RbTab<S> T, int sweep) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    if (ctl->done) return;
    const int i = L.n0 + cta * kT + threadIdx.x;
    if (i >= L.n) return;
    const RowRef rr = row_ref(L, i);
    const int dg = rr.deg - 1;
    const S* rv = sweep == 1 ? rhs : r;
    S zf[B];
    ld<B>(rv + (size_t)i * B, zf);
    for (int e = 0; e < dg; ++e) {
        const int kk = acol(L, rr, e);
        S zk[B];
        ld<B>(rv + (size_t)kk * B, zk);
        const S* __restrict__ U = inv0 + ubase<B>(kk);
        double A[2 * pairs<B>()];
        ablock<B>(L, rr, e, A);
        S acc[B];
#pragma unroll
        for (int rw = 0; rw < B; ++rw) acc[rw] = zero<S>();
        // column c of inv(U_kk) at a time: L[rw][c] = sum_m A[rw][m] U[m][c] (rounded as
        // the reference's L_ik), then acc[rw] += L[rw][c] z[c] in ascending c
#pragma unroll
        for (int c = 0; c < B; ++c) {
            S uc[B];
#pragma unroll
            for (int m = 0; m < B; ++m) uc[m] = U[uix<B>(m, c)];
#pragma unroll
            for (int rw = 0; rw < B; ++rw) {
                S lrc = zero<S>();
#pragma unroll
                for (int m = 0; m < B; ++m) lrc += rmul(A[rw * B + m], uc[m]);
                acc[rw] += lrc * zk[c];
            }
        }
#pragma unroll
        for (int rw = 0; rw < B; ++rw) zf[rw] -= acc[rw];
    }
    S lu[B * B];
    int pv[B];
    ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
    lu_solve_reg<B>(lu, pv, zf);
    st<B>(z + (size_t)i * B, zf);
}

// ---- K_B: colour 0 rows -----------------------------------------------------
// One descending pass over the row's blocks: A_e z_j feeds the backward sum
// (sparse.cpp:280-290) and A_e (x_j + z_j) is parked in shared memory; after the
// pivot solve and x += z the residual row is summed in ascending order
// (sparse.hpp:317-319).  Every block is read from HBM once.
template <int B, class S, bool LW = false>
__global__ void __launch_bounds__(kT) k_rb_colour0(SellDev L, const RbTab<S> T, int sweep, int G = 0) {
    // LW (lane-warp, fnlh_set_rb_sweep(4)): a CTA is ONE slice of 32 rows for G lanes of the
    // batch, warp w serving lane (blockIdx.x % ng) G + w, so the lanes' loads of the shared A
    // blocks and column indices meet in L1 instead of each going to L2
    const int P_ = T.P;
    int h_, cta;
    if constexpr (LW) {
        const int ng = (P_ + G - 1) / G;
        h_ = (blockIdx.x % ng) * G + (threadIdx.x >> 5);
        cta = blockIdx.x / ng;
        if (h_ >= P_) return;
    } else {
        h_ = blockIdx.x % P_;
        cta = blockIdx.x / P_;
    }
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S* park = reinterpret_cast<S*>(smem_raw);  // [slot][row][tid]
    if (ctl->done) return;
    const int tid = threadIdx.x;
    const int nt = LW ? (int)blockDim.x : kT;  // park stride
    const int i = LW ? cta * 32 + (tid & 31) : cta * kT + tid;
    double loc = 0.0;
    if (i < L.n0) {
        const RowRef rr = row_ref(L, i);
        S t[B];
        ld<B>((sweep == 1 ? rhs : r) + (size_t)i * B, t);  // forward: colour 0 rows copy r
#if RB_IDXPF
        int jn = rr.deg > 1 ? acol(L, rr, rr.deg - 1) : 0;
#endif
        for (int e = rr.deg - 1; e >= 1; --e) {
#if RB_IDXPF
            [[maybe_unused]] const int j = jn;
            jn = acol(L, rr, e > 1 ? e - 1 : e);
#else
            const int j = acol(L, rr, e);
#endif
            S zj[B], xj[B];
            ld<B>(z + (size_t)j * B, zj);
            ld<B>(x + (size_t)j * B, xj);
#pragma unroll
            for (int k = 0; k < B; ++k) xj[k] += zj[k];  // colour-1 x += z ahead of K_R
            double A[2 * pairs<B>()];
            ablock<B>(L, rr, e, A);
#pragma unroll
            for (int rw = 0; rw < B; ++rw) {
                S accb = zero<S>(), accm = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    const double a = A[rw * B + c];
                    accb += rmul(a, zj[c]);
                    accm += rmul(a, xj[c]);
                }
                t[rw] -= accb;
                park[((e - 1) * B + rw) * nt + tid] = accm;
            }
        }
        S lu[B * B];
        int pv[B];
        ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
        lu_solve_reg<B>(lu, pv, t);
        S xi[B];
        ld<B>(x + (size_t)i * B, xi);
#pragma unroll
        for (int k = 0; k < B; ++k) xi[k] += t[k];  // x += z (sparse.hpp:317)
        st<B>(x + (size_t)i * B, xi);
        S y[B];
#pragma unroll
        for (int k = 0; k < B; ++k) y[k] = zero<S>();
        const double s = shift ? shift[i] : 0.0;
        blk_matvec_add<B, S>(L, rr, 0, xi, shift != nullptr, s, y);  // diagonal block first
        for (int e = 1; e < rr.deg; ++e)
#pragma unroll
            for (int rw = 0; rw < B; ++rw) y[rw] += park[((e - 1) * B + rw) * nt + tid];
        S bi[B];
        ld<B>(rhs + (size_t)i * B, bi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const S v = bi[k] - y[k];
            r[(size_t)i * B + k] = v;
            loc += sq(v);
        }
    }
    if constexpr (LW) {  // per-slice partial (ordered_sum_lw regroups them 4 by 4)
        double v = loc;
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if ((tid & 31) == 0) partials[cta] = v;
    } else {
        const double bs = block_sum(loc, red);
        if (tid == 0) partials[cta] = bs;
    }
}

// ---- K_R: colour 1 residual rows + stopping rule ------------------------------
// x += z (colour 1), r_i = b_i - sum_e A_e x_col (ascending: lower blocks, then the
// diagonal), ||r|| over both colours and the stopping decision of this sweep
// (sparse.hpp:318-328), taken by the last CTA on the device.
template <int B, class S>
__global__ void __launch_bounds__(kT) k_rb_resid1(SellDev L, const RbTab<S> T, int grid0, int sweep, int max_iter) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    __shared__ bool last;
    if (ctl->done) return;
    const int i = L.n0 + cta * kT + threadIdx.x;
    double loc = 0.0;
    if (i < L.n) {
        const RowRef rr = row_ref(L, i);
        const int dg = rr.deg - 1;
        S xi[B], zi[B];
        ld<B>(x + (size_t)i * B, xi);
        ld<B>(z + (size_t)i * B, zi);
#pragma unroll
        for (int k = 0; k < B; ++k) xi[k] += zi[k];
        st<B>(x + (size_t)i * B, xi);
        S y[B];
#pragma unroll
        for (int k = 0; k < B; ++k) y[k] = zero<S>();
        for (int e = 0; e < dg; ++e) {
            S xk[B];
            ld<B>(x + (size_t)acol(L, rr, e) * B, xk);
            blk_matvec_add<B, S>(L, rr, e, xk, false, 0.0, y);
        }
        blk_matvec_add<B, S>(L, rr, dg, xi, shift != nullptr, shift ? shift[i] : 0.0, y);
        S bi[B];
        ld<B>(rhs + (size_t)i * B, bi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const S v = bi[k] - y[k];
            r[(size_t)i * B + k] = v;
            loc += sq(v);
        }
    }
    const double bs = block_sum(loc, red);
    if (threadIdx.x == 0) {
        partials[grid0 + cta] = bs;
        __threadfence();
        last = atomicAdd(counter, 1u) == nct - 1;
    }
    __syncthreads();
    if (!last) return;
    const double tot = ordered_sum(partials, grid0 + nct, red);
    if (threadIdx.x == 0) {
        const double nrm = sqrt(tot);
        ctl->iterations = sweep;
        ctl->final_residual = nrm;
        if (!isfinite(nrm)) {
            ctl->status = 6;
            ctl->done = 1;
        } else if (nrm <= ctl->target) {
            ctl->converged = 1;
            ctl->done = 1;
        } else if (sweep >= max_iter) {
            ctl->done = 1;
        }
        *counter = 0u;
    }
}

// ---- K_RF: colour 1 residual of sweep s fused with the forward substitution of s+1 --
// Two passes over the row's lower blocks A_ik: y += A_ik x_k (residual, ascending), then --
// r_i is known only once the residual row is complete and the forward sum starts from it
// (zf = r_i - L r_k1 - L r_k2 ..., sparse.cpp:267-278) -- L_ik r_k with L_ik = A_ik inv(U_kk)
// rebuilt as in K_F, the row's blocks read again (L1 / L2).  Every load of an edge (the b x b
// inv(U_kk), A_ik, r_k) is issued before its arithmetic and the column index one edge ahead
// (RB_UHOIST, RB_IDXPF): -3 % at 3 resident CTAs, DESIGN 4.1.
template <int B, class S, bool LW = false>
__global__ void __launch_bounds__(kT, LW ? 3 : RB_C1_MINB) k_rbx_colour1(SellDev L, const RbTab<S> T, int grid0, int sweep, int max_iter, int forward,
                                                    int G = 0) {
    const int P_ = T.P;
    int h_, cta, nct_;
    if constexpr (LW) {  // see k_rb_colour0: one slice, G lanes, warp = lane
        const int ng = (P_ + G - 1) / G;
        h_ = (blockIdx.x % ng) * G + (threadIdx.x >> 5);
        cta = blockIdx.x / ng;
        nct_ = gridDim.x / ng;
        if (h_ >= P_) return;
    } else {
        h_ = blockIdx.x % P_;
        cta = blockIdx.x / P_;
        nct_ = gridDim.x / P_;
    }
    [[maybe_unused]] const int nct = nct_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    __shared__ bool last;
    if (ctl->done) return;
    const int tid = threadIdx.x;
    const int i = LW ? L.n0 + cta * 32 + (tid & 31) : L.n0 + cta * kT + tid;
    double loc = 0.0;
    if (i < L.n) {
        const RowRef rr = row_ref(L, i);
        const int dg = rr.deg - 1;
        S xi[B], zi[B], y[B];
        ld<B>(x + (size_t)i * B, xi);
        ld<B>(z + (size_t)i * B, zi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            xi[k] += zi[k];
            y[k] = zero<S>();
        }
        st<B>(x + (size_t)i * B, xi);
        // pass 1: the residual row of sweep s, ascending (lower blocks, then the diagonal)
#if RB_IDXPF
        int kn = dg > 0 ? acol(L, rr, 0) : 0;
        for (int e = 0; e < dg; ++e) {
            const int kc = kn;
            kn = acol(L, rr, e + 1 < dg ? e + 1 : e);
            S xk[B];
            ld<B>(x + (size_t)kc * B, xk);
            blk_matvec_add<B, S>(L, rr, e, xk, false, 0.0, y);
        }
#else
        for (int e = 0; e < dg; ++e) {
            S xk[B];
            ld<B>(x + (size_t)acol(L, rr, e) * B, xk);
            blk_matvec_add<B, S>(L, rr, e, xk, false, 0.0, y);
        }
#endif
        blk_matvec_add<B, S>(L, rr, dg, xi, shift != nullptr, shift ? shift[i] : 0.0, y);
        S ri[B];
        ld<B>(rhs + (size_t)i * B, ri);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            ri[k] -= y[k];
            loc += sq(ri[k]);
        }
        // pass 2: forward substitution of sweep s+1 from r_i, the row's blocks again (now
        // L2-resident), L_ik = A_ik inv(U_kk) rebuilt in the reference's order
        if (forward) {
#if RB_IDXPF
            int kn2 = dg > 0 ? acol(L, rr, 0) : 0;
#endif
            for (int e = 0; e < dg; ++e) {
#if RB_IDXPF
                const int kk = kn2;
                kn2 = acol(L, rr, e + 1 < dg ? e + 1 : e);
#else
                const int kk = acol(L, rr, e);
#endif
                S rk[B];
                ld<B>(r + (size_t)kk * B, rk);
                const S* __restrict__ U = inv0 + ubase<B>(kk);
#if RB_UHOIST
                S Ub[B * B];
#pragma unroll
                for (int q = 0; q < B * B; ++q) Ub[q] = U[uix<B>(q / B, q % B)];
#endif
                double A[2 * pairs<B>()];
                ablock<B>(L, rr, e, A);
#if RB_UHOIST
                asm volatile("" ::: "memory");  // every load of the edge is issued before its arithmetic
#endif
                S acc[B];
#pragma unroll
                for (int rw = 0; rw < B; ++rw) acc[rw] = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    S uc[B];
#pragma unroll
#if RB_UHOIST
                    for (int m = 0; m < B; ++m) uc[m] = Ub[m * B + c];
#else
                    for (int m = 0; m < B; ++m) uc[m] = U[uix<B>(m, c)];
#endif
#pragma unroll
                    for (int rw = 0; rw < B; ++rw) {
                        S lrc = zero<S>();
#pragma unroll
                        for (int m = 0; m < B; ++m) lrc += rmul(A[rw * B + m], uc[m]);
                        acc[rw] += lrc * rk[c];
                    }
                }
#pragma unroll
                for (int rw = 0; rw < B; ++rw) ri[rw] -= acc[rw];
            }
            S lu[B * B];
            int pv[B];
            ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
            lu_solve_reg<B>(lu, pv, ri);
            st<B>(z + (size_t)i * B, ri);
        }
    }
    if constexpr (LW) {
        // per-slice partial; the warp that completes its lane's count takes the decision
        double v = loc;
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        int lastw = 0;
        if ((tid & 31) == 0) {
            partials[4 * grid0 + cta] = v;
            __threadfence();
            lastw = atomicAdd(counter, 1u) == (unsigned)(nct - 1);
        }
        lastw = __shfl_sync(0xffffffffu, lastw, 0);
        if (!lastw) return;
        __threadfence();
        const double tot = ordered_sum_lw(partials, grid0, (L.n - L.n0 + kT - 1) / kT, (L.n0 + 31) / 32, nct);
        if ((tid & 31) == 0) {
            const double nrm = sqrt(tot);
            ctl->iterations = sweep;
            ctl->final_residual = nrm;
            if (!isfinite(nrm)) {
                ctl->status = 6;
                ctl->done = 1;
            } else if (nrm <= ctl->target) {
                ctl->converged = 1;
                ctl->done = 1;
            } else if (sweep >= max_iter) {
                ctl->done = 1;
            }
            *counter = 0u;
        }
        return;
    }
    const double bs = block_sum(loc, red);
    if (threadIdx.x == 0) {
        partials[grid0 + cta] = bs;
        __threadfence();
        last = atomicAdd(counter, 1u) == nct - 1;
    }
    __syncthreads();
    if (!last) return;
    const double tot = ordered_sum(partials, grid0 + nct, red);
    if (threadIdx.x == 0) {
        const double nrm = sqrt(tot);
        ctl->iterations = sweep;
        ctl->final_residual = nrm;
        if (!isfinite(nrm)) {
            ctl->status = 6;
            ctl->done = 1;
        } else if (nrm <= ctl->target) {
            ctl->converged = 1;
            ctl->done = 1;
        } else if (sweep >= max_iter) {
            ctl->done = 1;
        }
        *counter = 0u;
    }
}



// ---- K_RF, staged (fnlh_set_rb_sweep(5)) ---------------------------------------------
// k_rbx_colour1's arithmetic (bitwise, the same norms) with every operand of the forward
// substitution fetched ahead of its use:
//   * a CTA is one 32-row slice for up to 4 lanes of the batch (warp = lane); the slice's A
//     blocks -- one contiguous SELL region -- are copied to shared memory once (cp.async) and
//     serve both passes of all the CTA's lanes (A leaves L2 once per CTA instead of twice per
//     lane);
//   * inv(U_kk) streams through a per-thread ring of B + 1 columns in shared memory
//     (cp.async, one commit group per column): while a thread rebuilds
//     L_ik column c, the remaining columns of the edge and the first of the next are already
//     in flight, so the thread never waits a round trip per column;
//   * the column indices two edges ahead, and x_k / r_k one edge ahead, live in registers.
// Two CTAs per SM (<= 255 registers): 8 warps whose loads are all issued an edge early.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifndef RBS_MINB
#define RBS_MINB 2
#endif
// RINGED = false (measurement): inv(U_kk) by ordinary loads through L1 as in k_rbx_colour1, only
// the A blocks staged in shared memory
template <int B, bool RINGED = true>
__global__ void __launch_bounds__(kT, RBS_MINB) k_rbs_colour1(SellDev L, const RbTab<cplx> T, int grid0, int sweep, int max_iter,
                                                       int forward, int G, int abytes, int c0_slices) {
    using S = cplx;
    constexpr int RING = B + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const double2* As = reinterpret_cast<const double2*>(smem_raw);  // [slot][pair][lane]
    S* ring = reinterpret_cast<S*>(smem_raw + abytes);               // [RING][B][thread]
    const int P_ = T.P, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int ng = (P_ + G - 1) / G;
    const int h_ = (blockIdx.x % ng) * G + (tid >> 5);
    const int cta = blockIdx.x / ng, nct = gridDim.x / ng;
    const int i = L.n0 + cta * 32 + lane;
    // a warp whose lane does not exist or has stopped only helps with the A copy; a CTA of such
    // warps leaves at once
    const bool warp_on = h_ < P_ && !T.ctl[h_ < P_ ? h_ : 0]->done;
    if (!__syncthreads_or(warp_on)) return;
    // the slice's A blocks: every thread of the CTA copies its share (group 0)
    {
        const int sl = L.nslices0 + cta;
        const long long v0 = L.slice_val[sl], v1 = L.slice_val[sl + 1];
        const char* src = reinterpret_cast<const char*>(L.vals + v0);
        const int bytes = (int)((v1 - v0) * 8);
        for (int o = tid * 16; o < bytes; o += nt * 16) cp_async16(smem_raw + o, src + o);
        cp_async_commit();
    }
    const bool active = warp_on && i < L.n;  // rows past the end idle but stay for the warp's sums
    RbControl* ctl = T.ctl[warp_on ? h_ : 0];
    const S* __restrict__ inv0 = T.inv0[warp_on ? h_ : 0];
    S* __restrict__ x = T.x[warp_on ? h_ : 0];
    S* __restrict__ r = T.r[warp_on ? h_ : 0];
    RowRef rr{};
    int dg = 0, k0 = 0, k1 = 0, k2 = 0;
    if (active) {
        rr = row_ref(L, i);
        dg = rr.deg - 1;
        k0 = acol(L, rr, 0);  // padding slots hold the row itself: always a valid load
        k1 = acol(L, rr, dg > 1 ? 1 : 0);
        k2 = acol(L, rr, dg > 2 ? 2 : 0);
    }
    // ring prologue: columns 0 .. RING-1 of the forward pass (edge 0, then column 0 of edge 1)
    const bool fwd = RINGED && active && forward;
    if (fwd) {
#pragma unroll
        for (int j = 0; j < RING; ++j) {
            const int de = j / B, c = j % B;
            if (de < dg) {
                const S* src = inv0 + ubase<B>(de == 0 ? k0 : k1);
#pragma unroll
                for (int m = 0; m < B; ++m) cp_async16(ring + ((size_t)(j * B + m) * nt + tid), src + uix<B>(m, c));
            }
            cp_async_commit();
        }
        cp_async_wait<RING>();  // group 0 (A) has landed; the ring may still be in flight
    } else {
        cp_async_wait<0>();
    }
    __syncthreads();
    if (!warp_on) return;
    const S* __restrict__ diag_lu = T.diag_lu[h_];
    const int* __restrict__ piv = T.piv[h_];
    const double* __restrict__ shift = T.shift[h_];
    const S* __restrict__ rhs = T.rhs[h_];
    S* __restrict__ z = T.z[h_];
    unsigned int* counter = &ctl->counter;
    double* __restrict__ partials = T.parts[h_];
    double loc = 0.0;
    if (active) {
        S xi[B], zi[B], y[B];
        ld<B>(x + (size_t)i * B, xi);
        ld<B>(z + (size_t)i * B, zi);
        S bi[B];
        ld<B>(rhs + (size_t)i * B, bi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            xi[k] += zi[k];
            y[k] = zero<S>();
        }
        st<B>(x + (size_t)i * B, xi);
        // pass 1: residual row of sweep s (ascending lower blocks, then the diagonal), A from
        // shared memory, x_k one edge ahead
        {
            int ka = k0, kb = k1;
            S xn[B];
            ld<B>(x + (size_t)ka * B, xn);
            for (int e = 0; e < dg; ++e) {
                S xk[B];
#pragma unroll
                for (int k = 0; k < B; ++k) xk[k] = xn[k];
                ka = kb;
                kb = acol(L, rr, e + 2 < dg ? e + 2 : e);
                if (e + 1 < dg) ld<B>(x + (size_t)ka * B, xn);
                double A[2 * pairs<B>()];
#pragma unroll
                for (int p = 0; p < pairs<B>(); ++p) {
                    const double2 v = As[(e * pairs<B>() + p) * 32 + lane];
                    A[2 * p] = v.x;
                    A[2 * p + 1] = v.y;
                }
#pragma unroll
                for (int rw = 0; rw < B; ++rw) {
                    S acc = zero<S>();
#pragma unroll
                    for (int c = 0; c < B; ++c) acc += rmul(A[rw * B + c], xk[c]);
                    y[rw] += acc;
                }
            }
            double A[2 * pairs<B>()];
#pragma unroll
            for (int p = 0; p < pairs<B>(); ++p) {
                const double2 v = As[(dg * pairs<B>() + p) * 32 + lane];
                A[2 * p] = v.x;
                A[2 * p + 1] = v.y;
            }
            const double sft = shift ? shift[i] : 0.0;
#pragma unroll
            for (int rw = 0; rw < B; ++rw) {  // blk_matvec_add with the shifted diagonal
                S acc = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    const double a = A[rw * B + c];
                    if (shift != nullptr && rw == c)
                        acc += mk(a + 0.0, 0.0 + sft) * xi[c];
                    else
                        acc += rmul(a, xi[c]);
                }
                y[rw] += acc;
            }
        }
        S ri[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            ri[k] = bi[k] - y[k];
            loc += sq(ri[k]);
        }
        // pass 2: forward substitution of sweep s+1; inv(U_kk) columns from the ring
        if (forward) {
            S rn[B];
            ld<B>(r + (size_t)k0 * B, rn);
            for (int e = 0; e < dg; ++e) {
                S rk[B];
#pragma unroll
                for (int k = 0; k < B; ++k) rk[k] = rn[k];
                if (e + 1 < dg) ld<B>(r + (size_t)k1 * B, rn);
                const int k3 = acol(L, rr, e + 3 < dg ? e + 3 : e);
                double A[2 * pairs<B>()];
#pragma unroll
                for (int p = 0; p < pairs<B>(); ++p) {
                    const double2 v = As[(e * pairs<B>() + p) * 32 + lane];
                    A[2 * p] = v.x;
                    A[2 * p + 1] = v.y;
                }
                S acc[B];
#pragma unroll
                for (int rw = 0; rw < B; ++rw) acc[rw] = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    // column j = e B + c sits in ring slot j % RING; RING - 1 younger groups may be pending
                    S uc[B];
                    if constexpr (!RINGED) {
                        const S* __restrict__ U = inv0 + ubase<B>(k0);
#pragma unroll
                        for (int m = 0; m < B; ++m) uc[m] = U[uix<B>(m, c)];
                    } else {
                    cp_async_wait<RING - 1>();
                    const int slot = (e * B + c) % RING;
#pragma unroll
                    for (int m = 0; m < B; ++m) uc[m] = ring[(size_t)(slot * B + m) * nt + tid];
                    // refill the slot with column j + RING: edge e + de, column cn
                    {
                        const int de = (c + RING) / B, cn = (c + RING) % B;
                        if (e + de < dg) {
                            const S* src = inv0 + ubase<B>(de == 1 ? k1 : k2);
#pragma unroll
                            for (int m = 0; m < B; ++m) cp_async16(ring + ((size_t)(slot * B + m) * nt + tid), src + uix<B>(m, cn));
                        }
                        cp_async_commit();
                    }
                    }
#pragma unroll
                    for (int rw = 0; rw < B; ++rw) {
                        S lrc = zero<S>();
#pragma unroll
                        for (int m = 0; m < B; ++m) lrc += rmul(A[rw * B + m], uc[m]);
                        acc[rw] += lrc * rk[c];
                    }
                }
#pragma unroll
                for (int rw = 0; rw < B; ++rw) ri[rw] -= acc[rw];
                k0 = k1;
                k1 = k2;
                k2 = k3;
            }
            S lu[B * B];
            int pv[B];
            ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
            lu_solve_reg<B>(lu, pv, ri);
            st<B>(z + (size_t)i * B, ri);
        }
    }
    // per-slice partial; the warp that completes its lane's count takes the decision
    double v = loc;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    int lastw = 0;
    if (lane == 0) {
        partials[4 * grid0 + cta] = v;
        __threadfence();
        lastw = atomicAdd(counter, 1u) == (unsigned)(nct - 1);
    }
    lastw = __shfl_sync(0xffffffffu, lastw, 0);
    if (!lastw) return;
    __threadfence();
    const double tot = ordered_sum_lw(partials, grid0, (L.n - L.n0 + kT - 1) / kT, (L.n0 + 31) / 32, nct, c0_slices != 0);
    if (lane == 0) {
        const double nrm = sqrt(tot);
        ctl->iterations = sweep;
        ctl->final_residual = nrm;
        if (!isfinite(nrm)) {
            ctl->status = 6;
            ctl->done = 1;
        } else if (nrm <= ctl->target) {
            ctl->converged = 1;
            ctl->done = 1;
        } else if (sweep >= max_iter) {
            ctl->done = 1;
        }
        *counter = 0u;
    }
}

// ---- K_B, edge-parallel (fnlh_set_rb_sweep(3)) -------------------------------------
// k_rb_colour0's arithmetic with one thread per (row, upper block): warp q of the CTA (one
// SELL slice of colour-0 rows) forms block slot q+1's backward product A_ij z_j and
// residual product A_ij (x_j + z_j) into shared memory; warp 0 then takes the backward sum
// in descending slot order, the pivot solve and x += z, and the residual row with the
// diagonal block first and the parked products ascending -- the row-serial sequence.
template <int B, class S>
__global__ void __launch_bounds__(192, RBE_MINB) k_rbe_colour0(SellDev L, const RbTab<S> T, int sweep, int E) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    const S* __restrict__ diag_lu = T.diag_lu[h_];
    const int* __restrict__ piv = T.piv[h_];
    const double* __restrict__ shift = T.shift[h_];
    const S* __restrict__ rhs = T.rhs[h_];
    S* __restrict__ x = T.x[h_];
    S* __restrict__ z = T.z[h_];
    S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    double* __restrict__ partials = T.parts[h_];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S* Bk = reinterpret_cast<S*>(smem_raw);       // [slot-1][rw][lane]: A_ij z_j
    S* Mk = Bk + (std::size_t)E * B * 32;         // [slot-1][rw][lane]: A_ij (x_j + z_j)
    if (ctl->done) return;
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int i = cta * 32 + lane;
    const bool row_ok = i < L.n0;
    RowRef rr{};
    if (row_ok) rr = row_ref(L, i);
    const int e = q + 1;
    if (row_ok && e < rr.deg) {
        const int j = acol(L, rr, e);
        S zj[B], xj[B];
        ld<B>(z + (size_t)j * B, zj);
        ld<B>(x + (size_t)j * B, xj);
#pragma unroll
        for (int k = 0; k < B; ++k) xj[k] += zj[k];  // colour-1 x += z ahead of K_R
        double A[2 * pairs<B>()];
        ablock<B>(L, rr, e, A);
#pragma unroll
        for (int rw = 0; rw < B; ++rw) {
            S accb = zero<S>(), accm = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) {
                const double a = A[rw * B + c];
                accb += rmul(a, zj[c]);
                accm += rmul(a, xj[c]);
            }
            Bk[((size_t)q * B + rw) * 32 + lane] = accb;
            Mk[((size_t)q * B + rw) * 32 + lane] = accm;
        }
    }
    __syncthreads();
    double loc = 0.0;
    if (q == 0 && row_ok) {
        S t[B];
        ld<B>((sweep == 1 ? rhs : r) + (size_t)i * B, t);  // forward: colour 0 rows copy r
        for (int ee = rr.deg - 1; ee >= 1; --ee)
#pragma unroll
            for (int rw = 0; rw < B; ++rw) t[rw] -= Bk[((size_t)(ee - 1) * B + rw) * 32 + lane];
        const LuRef q_ = lu_ref<B>(L, i);
        int pv[B];
#pragma unroll
        for (int k = 0; k < B; ++k) pv[k] = piv[q_.pv + 32 * k];
        lu_solve_mem<B>(diag_lu + q_.lu, 32, pv, t);
        S xi[B];
        ld<B>(x + (size_t)i * B, xi);
#pragma unroll
        for (int k = 0; k < B; ++k) xi[k] += t[k];  // x += z (sparse.hpp:317)
        st<B>(x + (size_t)i * B, xi);
        S y[B];
#pragma unroll
        for (int k = 0; k < B; ++k) y[k] = zero<S>();
        blk_matvec_add<B, S>(L, rr, 0, xi, shift != nullptr, shift ? shift[i] : 0.0, y);  // diagonal block first
        for (int ee = 1; ee < rr.deg; ++ee)
#pragma unroll
            for (int rw = 0; rw < B; ++rw) y[rw] += Mk[((size_t)(ee - 1) * B + rw) * 32 + lane];
        S bi[B];
        ld<B>(rhs + (size_t)i * B, bi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const S v = bi[k] - y[k];
            r[(size_t)i * B + k] = v;
            loc += sq(v);
        }
    }
    double v = loc;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) partials[cta] = v;
}

// ---- K_RF, edge-parallel (fnlh_set_rb_sweep(3)) ------------------------------------
// The same arithmetic as k_rbx_colour1 with one thread per (row, lower block): a CTA is one
// SELL slice of colour-1 rows (32 rows, warp e = block slot e), so all of a row's
// neighbour gathers (x_k, r_k, inv(U_kk)) are in flight at once instead of one block after
// another.  Each thread forms its block's residual product A_ik x_k and forward product
// L_ik r_k (L_ik rebuilt in the reference's order) into shared memory; warp 0 then sums
// them per row in ascending block order (then the diagonal), exactly the sequence of the
// row-serial kernel, so the iterates are bitwise the same.
template <int B, class S>
__global__ void __launch_bounds__(192, RBE_MINB) k_rbe_colour1(SellDev L, const RbTab<S> T, int grid0, int sweep, int max_iter,
                                                     int forward, int E) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    const S* __restrict__ diag_lu = T.diag_lu[h_];
    const int* __restrict__ piv = T.piv[h_];
    const S* __restrict__ inv0 = T.inv0[h_];
    const double* __restrict__ shift = T.shift[h_];
    const S* __restrict__ rhs = T.rhs[h_];
    S* __restrict__ x = T.x[h_];
    S* __restrict__ z = T.z[h_];
    S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    unsigned int* counter = &ctl->counter;
    double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    __shared__ bool last;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S* Q = reinterpret_cast<S*>(smem_raw);        // [slot][rw][lane]: A_ik x_k
    S* Pf = Q + (std::size_t)E * B * 32;          // [slot][rw][lane]: L_ik r_k
    if (ctl->done) return;
    const int lane = threadIdx.x & 31, e = threadIdx.x >> 5;
    const int i = L.n0 + cta * 32 + lane;
    const bool row_ok = i < L.n;
    RowRef rr{};
    int dg = 0;
    if (row_ok) {
        rr = row_ref(L, i);
        dg = rr.deg - 1;
    }
    if (row_ok && e < dg) {
        const int kk = acol(L, rr, e);
        double A[2 * pairs<B>()];
        ablock<B>(L, rr, e, A);
        S xk[B];
        ld<B>(x + (size_t)kk * B, xk);
#pragma unroll
        for (int rw = 0; rw < B; ++rw) {
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) acc += rmul(A[rw * B + c], xk[c]);
            Q[((size_t)e * B + rw) * 32 + lane] = acc;
        }
        if (forward) {
            S rk[B];
            ld<B>(r + (size_t)kk * B, rk);
            const S* __restrict__ U = inv0 + ubase<B>(kk);
            S acc[B];
#pragma unroll
            for (int rw = 0; rw < B; ++rw) acc[rw] = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) {
                S uc[B];
#pragma unroll
                for (int m = 0; m < B; ++m) uc[m] = U[uix<B>(m, c)];
#pragma unroll
                for (int rw = 0; rw < B; ++rw) {
                    S lrc = zero<S>();
#pragma unroll
                    for (int m = 0; m < B; ++m) lrc += rmul(A[rw * B + m], uc[m]);
                    acc[rw] += lrc * rk[c];
                }
            }
#pragma unroll
            for (int rw = 0; rw < B; ++rw) Pf[((size_t)e * B + rw) * 32 + lane] = acc[rw];
        }
    }
    __syncthreads();
    double loc = 0.0;
    if (e == 0 && row_ok) {
        S xi[B], zi[B], y[B];
        ld<B>(x + (size_t)i * B, xi);
        ld<B>(z + (size_t)i * B, zi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            xi[k] += zi[k];
            y[k] = zero<S>();
        }
        st<B>(x + (size_t)i * B, xi);
        for (int q = 0; q < dg; ++q)
#pragma unroll
            for (int rw = 0; rw < B; ++rw) y[rw] += Q[((size_t)q * B + rw) * 32 + lane];
        blk_matvec_add<B, S>(L, rr, dg, xi, shift != nullptr, shift ? shift[i] : 0.0, y);
        S ri[B];
        ld<B>(rhs + (size_t)i * B, ri);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            ri[k] -= y[k];
            loc += sq(ri[k]);
        }
        if (forward) {
            for (int q = 0; q < dg; ++q)
#pragma unroll
                for (int rw = 0; rw < B; ++rw) ri[rw] -= Pf[((size_t)q * B + rw) * 32 + lane];
            const LuRef q_ = lu_ref<B>(L, i);
            int pv[B];
#pragma unroll
            for (int k = 0; k < B; ++k) pv[k] = piv[q_.pv + 32 * k];
            lu_solve_mem<B>(diag_lu + q_.lu, 32, pv, ri);
            st<B>(z + (size_t)i * B, ri);
        }
    }
    // CTA partial in row order (one slice), then the last CTA's decision
    double v = loc;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) {
        partials[grid0 + cta] = v;
        __threadfence();
        last = atomicAdd(counter, 1u) == nct - 1;
    }
    __syncthreads();
    if (!last) return;
    const double tot = ordered_sum_n(partials, grid0 + nct, red);
    if (threadIdx.x == 0) {
        const double nrm = sqrt(tot);
        ctl->iterations = sweep;
        ctl->final_residual = nrm;
        if (!isfinite(nrm)) {
            ctl->status = 6;
            ctl->done = 1;
        } else if (nrm <= ctl->target) {
            ctl->converged = 1;
            ctl->done = 1;
        } else if (sweep >= max_iter) {
            ctl->done = 1;
        }
        *counter = 0u;
    }
}

// ---- one-pass sweep (fnlh_set_rb_sweep(2)): two kernels per sweep -----------
// The same preconditioner M = LU, applied with L_ik r_k = A_ik (U_kk^{-1} r_k): colour-0
// rows publish w_k = U_kk^{-1} r_k (kept in the colour-0 half of z) when they finish
// their residual, so the colour-1 forward substitution is a plain block-row product and
// fuses with the colour-1 residual of the previous sweep (both walk the same A_ik
// blocks).  Every block of A is read once per sweep; the iterates agree with the
// reference order to rounding (tests: 1e-12 relative), not bitwise -- the kernels above
// are the bitwise path (fnlh_set_rb_sweep(0|1)).
//
// K0(s): colour 0 rows: t = r_i - sum_j A_ij z_j; z_i = U_ii^{-1} t; x_i += z_i;
//        r_i = b_i - A_ii x_i - sum_j A_ij (x_j + z_j); w_i = U_ii^{-1} r_i
// K1(s): colour 1 rows: x_i += z_i; r_i = b_i - sum_k A_ik x_k - A_ii x_i (sweep s);
//        stopping decision of sweep s (last CTA); then, speculatively for s + 1,
//        z_i = U_ii^{-1} (r_i - sum_k A_ik w_k)
template <int B, class S>
__global__ void __launch_bounds__(kT) k_rbf_w0(SellDev L, const RbTab<S> T) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    if (ctl->done) return;
    const int i = cta * kT + threadIdx.x;
    if (i >= L.n0) return;
    S t[B];
    ld<B>(rhs + (size_t)i * B, t);
    S lu[B * B];
    int pv[B];
    ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
    lu_solve_reg<B>(lu, pv, t);
    st<B>(z + (size_t)i * B, t);
}

template <int B, class S>
__global__ void __launch_bounds__(kT) k_rbf_colour0(SellDev L, const RbTab<S> T, int sweep) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    if (ctl->done) return;
    const int tid = threadIdx.x;
    const int i = cta * kT + tid;
    double loc = 0.0;
    if (i < L.n0) {
        const RowRef rr = row_ref(L, i);
        S t[B], ym[B];
        ld<B>((sweep == 1 ? rhs : r) + (size_t)i * B, t);
#pragma unroll
        for (int k = 0; k < B; ++k) ym[k] = zero<S>();
        for (int e = 1; e < rr.deg; ++e) {
            const int j = acol(L, rr, e);
            S zj[B], xj[B];
            ld<B>(z + (size_t)j * B, zj);
            ld<B>(x + (size_t)j * B, xj);
#pragma unroll
            for (int k = 0; k < B; ++k) xj[k] += zj[k];
            double A[2 * pairs<B>()];
            ablock<B>(L, rr, e, A);
#pragma unroll
            for (int rw = 0; rw < B; ++rw) {
                S accb = zero<S>(), accm = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    const double a = A[rw * B + c];
                    accb += rmul(a, zj[c]);
                    accm += rmul(a, xj[c]);
                }
                t[rw] -= accb;
                ym[rw] += accm;
            }
        }
        S lu[B * B];
        int pv[B];
        ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
        lu_solve_reg<B>(lu, pv, t);
        S xi[B];
        ld<B>(x + (size_t)i * B, xi);
#pragma unroll
        for (int k = 0; k < B; ++k) xi[k] += t[k];
        st<B>(x + (size_t)i * B, xi);
        S y[B];
#pragma unroll
        for (int k = 0; k < B; ++k) y[k] = zero<S>();
        blk_matvec_add<B, S>(L, rr, 0, xi, shift != nullptr, shift ? shift[i] : 0.0, y);
        S bi[B];
        ld<B>(rhs + (size_t)i * B, bi);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const S v = bi[k] - (y[k] + ym[k]);
            t[k] = v;
            loc += sq(v);
        }
        st<B>(r + (size_t)i * B, t);
        lu_solve_reg<B>(lu, pv, t);
        st<B>(z + (size_t)i * B, t);  // w_i
    }
    const double bs = block_sum(loc, red);
    if (tid == 0) partials[cta] = bs;
}

template <int B, class S>
__global__ void __launch_bounds__(kT) k_rbf_colour1(SellDev L, const RbTab<S> T, int grid0, int sweep, int max_iter, int forward) {
    const int P_ = T.P, h_ = blockIdx.x % P_, cta = blockIdx.x / P_;
    [[maybe_unused]] const int nct = gridDim.x / P_;
    [[maybe_unused]] const S* __restrict__ diag_lu = T.diag_lu[h_];
    [[maybe_unused]] const int* __restrict__ piv = T.piv[h_];
    [[maybe_unused]] const S* __restrict__ inv0 = T.inv0[h_];
    [[maybe_unused]] const double* __restrict__ shift = T.shift[h_];
    [[maybe_unused]] const S* __restrict__ rhs = T.rhs[h_];
    [[maybe_unused]] S* __restrict__ x = T.x[h_];
    [[maybe_unused]] S* __restrict__ z = T.z[h_];
    [[maybe_unused]] S* __restrict__ r = T.r[h_];
    RbControl* ctl = T.ctl[h_];
    [[maybe_unused]] unsigned int* counter = &ctl->counter;
    [[maybe_unused]] double* __restrict__ partials = T.parts[h_];
    __shared__ double red[kT / 32];
    __shared__ bool last;
    if (ctl->done) return;
    const int i = L.n0 + cta * kT + threadIdx.x;
    double loc = 0.0;
    if (i < L.n) {
        const RowRef rr = row_ref(L, i);
        const int dg = rr.deg - 1;
        S ri[B], f[B];
        ld<B>(rhs + (size_t)i * B, ri);
#pragma unroll
        for (int k = 0; k < B; ++k) f[k] = zero<S>();
        if (sweep >= 1) {
            S xi[B], zi[B], y[B];
            ld<B>(x + (size_t)i * B, xi);
            ld<B>(z + (size_t)i * B, zi);
#pragma unroll
            for (int k = 0; k < B; ++k) {
                xi[k] += zi[k];
                y[k] = zero<S>();
            }
            st<B>(x + (size_t)i * B, xi);
            for (int e = 0; e < dg; ++e) {
                const int kk = acol(L, rr, e);
                S xk[B], wk[B];
                ld<B>(x + (size_t)kk * B, xk);
                ld<B>(z + (size_t)kk * B, wk);
                double A[2 * pairs<B>()];
                ablock<B>(L, rr, e, A);
#pragma unroll
                for (int rw = 0; rw < B; ++rw) {
                    S accy = zero<S>(), accf = zero<S>();
#pragma unroll
                    for (int c = 0; c < B; ++c) {
                        const double a = A[rw * B + c];
                        accy += rmul(a, xk[c]);
                        accf += rmul(a, wk[c]);
                    }
                    y[rw] += accy;
                    f[rw] += accf;
                }
            }
            blk_matvec_add<B, S>(L, rr, dg, xi, shift != nullptr, shift ? shift[i] : 0.0, y);
#pragma unroll
            for (int k = 0; k < B; ++k) {
                ri[k] -= y[k];
                loc += sq(ri[k]);
            }
        } else {
            for (int e = 0; e < dg; ++e) {
                S wk[B];
                ld<B>(z + (size_t)acol(L, rr, e) * B, wk);
                blk_matvec_add<B, S>(L, rr, e, wk, false, 0.0, f);
            }
        }
        if (forward) {
#pragma unroll
            for (int k = 0; k < B; ++k) ri[k] -= f[k];
            S lu[B * B];
            int pv[B];
            ld_lu<B>(diag_lu, piv, lu_ref<B>(L, i), lu, pv);
            lu_solve_reg<B>(lu, pv, ri);
            st<B>(z + (size_t)i * B, ri);
        }
    }
    if (sweep < 1) return;
    const double bs = block_sum(loc, red);
    if (threadIdx.x == 0) {
        partials[grid0 + cta] = bs;
        __threadfence();
        last = atomicAdd(counter, 1u) == nct - 1;
    }
    __syncthreads();
    if (!last) return;
    const double tot = ordered_sum(partials, grid0 + nct, red);
    if (threadIdx.x == 0) {
        const double nrm = sqrt(tot);
        ctl->iterations = sweep;
        ctl->final_residual = nrm;
        if (!isfinite(nrm)) {
            ctl->status = 6;
            ctl->done = 1;
        } else if (nrm <= ctl->target) {
            ctl->converged = 1;
            ctl->done = 1;
        } else if (sweep >= max_iter) {
            ctl->done = 1;
        }
        *counter = 0u;
    }
}

// ---- factorization ---------------------------------------------------------
template <int B, class S>
__global__ void k_rb_factor0(SellDev L, const double* __restrict__ shift, S* __restrict__ diag_lu,
                             int* __restrict__ piv, S* __restrict__ inv0, int* __restrict__ status) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= L.n0) return;
    const RowRef rr = row_ref(L, i);
    S A[B * B];
#pragma unroll
    for (int k = 0; k < B * B; ++k) {
        A[k] = from_real<S>(aval<B>(L, rr, 0, k));
        if constexpr (sizeof(S) == sizeof(cplx))
            if (shift && (k / B == k % B)) A[k] = A[k] + mk(0.0, shift[i]);
    }
    int pv[B];
    double cond;
    if (lu_factor_reg<B>(A, pv, cond) || !(cond < 1e14)) atomicMin(status + 1, i);
    const LuRef q = lu_ref<B>(L, i);
#pragma unroll
    for (int k = 0; k < B * B; ++k) diag_lu[q.lu + 32 * k] = A[k];
#pragma unroll
    for (int k = 0; k < B; ++k) piv[q.pv + 32 * k] = pv[k];
#pragma unroll
    for (int c = 0; c < B; ++c) {
        S col[B];
#pragma unroll
        for (int r = 0; r < B; ++r) col[r] = (r == c) ? one<S>() : zero<S>();
        lu_solve_reg<B>(A, pv, col);
#pragma unroll
        for (int r = 0; r < B; ++r) inv0[ubase<B>(i) + uix<B>(r, c)] = col[r];
    }
}

template <int B, class S>
__global__ void k_rb_factor1(SellDev L, const int* __restrict__ row_ptr, const long long* __restrict__ trans,
                             const double* __restrict__ shift, S* __restrict__ diag_lu, int* __restrict__ piv,
                             const S* __restrict__ inv0, int* __restrict__ status) {
    const int i = L.n0 + blockIdx.x * kT + threadIdx.x;
    if (i >= L.n) return;
    const RowRef rr = row_ref(L, i);
    const int dg = rr.deg - 1;
    S Uii[B * B];
#pragma unroll
    for (int k = 0; k < B * B; ++k) {
        Uii[k] = from_real<S>(aval<B>(L, rr, dg, k));
        if constexpr (sizeof(S) == sizeof(cplx))
            if (shift && (k / B == k % B)) Uii[k] = Uii[k] + mk(0.0, shift[i]);
    }
    const int e0 = row_ptr[i];
    for (int e = 0; e < dg; ++e) {
        const int kk = acol(L, rr, e);
        const S* U = inv0 + ubase<B>(kk);
        S Lb[B * B];
#pragma unroll
        for (int r = 0; r < B; ++r)
#pragma unroll
            for (int c = 0; c < B; ++c) {
                S acc = zero<S>();
#pragma unroll
                for (int m = 0; m < B; ++m) acc += from_real<S>(aval<B>(L, rr, e, r * B + m)) * U[uix<B>(m, c)];
                Lb[r * B + c] = acc;
            }
        // U_ii -= L_ik U_ki, U_ki = complex(A_ki) (block_matmul_sub, dense.hpp:42-52)
        const double* Aki = L.vals + trans[e0 + e];
#pragma unroll
        for (int r = 0; r < B; ++r)
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) {
                const S a = Lb[r * B + k2];
                if (is_zero(a)) continue;
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    const int kk2 = k2 * B + c;
                    Uii[r * B + c] -= a * from_real<S>(Aki[(long long)(kk2 >> 1) * 64 + (kk2 & 1)]);
                }
            }
    }
    int pv[B];
    double cond;
    if (lu_factor_reg<B>(Uii, pv, cond) || !(cond < 1e14)) atomicMin(status + 1, i);
    const LuRef q = lu_ref<B>(L, i);
#pragma unroll
    for (int k = 0; k < B * B; ++k) diag_lu[q.lu + 32 * k] = Uii[k];
#pragma unroll
    for (int k = 0; k < B; ++k) piv[q.pv + 32 * k] = pv[k];
}

__global__ void k_to_sell(const double* __restrict__ A, const long long* __restrict__ map, int bb, long long nnzb,
                          double* __restrict__ out) {
    const long long t = blockIdx.x * (long long)kT + threadIdx.x;
    if (t >= nnzb * bb) return;
    const long long e = t / bb;
    const int k = (int)(t % bb);
    out[map[e] + (long long)(k >> 1) * 64 + (k & 1)] = A[t];
}

#define RB_DISPATCH(b, ...)                                               \
    switch (b) {                                                          \
        case 1: { constexpr int B = 1; __VA_ARGS__; } break;              \
        case 3: { constexpr int B = 3; __VA_ARGS__; } break;              \
        case 5: { constexpr int B = 5; __VA_ARGS__; } break;              \
        case 6: { constexpr int B = 6; __VA_ARGS__; } break;              \
        default: throw ShapeError("rb: unsupported block size");          \
    }

SellDev sell_dev(const SellLayout& L, const double* vals) {
    return SellDev{L.slice_val.ptr, L.slice_col.ptr, L.deg.ptr, L.cols.ptr, vals, L.n, L.n0,
                   (L.n0 + 31) / 32};
}

}  // namespace

bool rb_eligible(const DevicePattern& p, int* n0) {
    if (!p.single_partition || p.fwd_levels() != 2 || p.bwd_levels() != 2) return false;
    const int c0 = p.fwd_ptr[1];
    // level 0 must be exactly the rows [0, c0) (colour-major; in any order within the level);
    // level 1 then holds [c0, n)
    std::vector<int> rows(p.rows);
    FNLH_CUDA(cudaMemcpy(rows.data(), p.fwd_rows, p.rows * sizeof(int), cudaMemcpyDeviceToHost));
    for (int k = 0; k < c0; ++k)
        if (rows[k] >= c0) return false;
    // no edges inside a colour
    for (int i = 0; i < p.rows; ++i)
        for (int e = p.h_row_ptr[i]; e < p.h_row_ptr[i + 1]; ++e) {
            const int j = p.h_col_idx[e];
            if (j != i && ((i < c0) == (j < c0))) return false;
        }
    *n0 = c0;
    return true;
}

template <class S>
RbIlu<S>::RbIlu(const DevicePattern* pat, int n0_) : p(pat), n0(n0_) {
    const std::size_t bb = (std::size_t)p->b * p->b;
    FNLH_CUDA_ALLOC(&diag_lu, packed_rows() * bb * sizeof(S));
    FNLH_CUDA_ALLOC(&diag_piv, packed_rows() * p->b * sizeof(int));
    FNLH_CUDA_ALLOC(&inv0, std::max<std::size_t>((std::size_t)32 * ((n0 + 31) / 32) * bb, 1) * sizeof(S));
}
template <class S>
RbIlu<S>::~RbIlu() {
    fnlh::dfree(diag_lu);
    fnlh::dfree(diag_piv);
    fnlh::dfree(inv0);
}
template <class S>
std::size_t RbIlu<S>::bytes() const {
    const std::size_t bb = (std::size_t)p->b * p->b;
    return (packed_rows() * bb + (std::size_t)32 * ((n0 + 31) / 32) * bb) * sizeof(S) + packed_rows() * p->b * sizeof(int);
}

RbSystem::RbSystem(const DevicePattern* p, int n0) : p_(p) {
    const int n = p->rows, b = p->b;
    L_.n = n;
    L_.n0 = n0;
    L_.b = b;
    const int ns0 = (n0 + 31) / 32, ns1 = (n - n0 + 31) / 32;
    L_.nslices = ns0 + ns1;
    L_.slice_of_row0 = ns0;
    std::vector<long long> sval(L_.nslices + 1, 0);
    std::vector<int> scol(L_.nslices + 1, 0);
    std::vector<int> deg(n), dslot(n);
    auto slice_rows = [&](int s, int& r0, int& r1) {
        if (s < ns0) {
            r0 = s * 32;
            r1 = std::min(n0, r0 + 32);
        } else {
            r0 = n0 + (s - ns0) * 32;
            r1 = std::min(n, r0 + 32);
        }
    };
    for (int i = 0; i < n; ++i) {
        deg[i] = p->h_row_ptr[i + 1] - p->h_row_ptr[i];
        dslot[i] = p->h_diag_idx[i] - p->h_row_ptr[i];
    }
    for (int s = 0; s < L_.nslices; ++s) {
        int r0, r1, md = 0;
        slice_rows(s, r0, r1);
        for (int i = r0; i < r1; ++i) md = std::max(md, deg[i]);
        sval[s + 1] = sval[s] + (long long)md * ((b * b + 1) / 2) * 64;
        scol[s + 1] = scol[s] + md * 32;
    }
    L_.total_vals = sval[L_.nslices];
    std::vector<int> cols(scol[L_.nslices], 0);
    std::vector<long long> map(p->nnzb), trans(p->nnzb);
    for (int s = 0; s < L_.nslices; ++s) {
        int r0, r1;
        slice_rows(s, r0, r1);
        const int md = (scol[s + 1] - scol[s]) / 32;
        for (int i = r0; i < r1; ++i) {
            const int lane = i - r0;
            for (int e = 0; e < md; ++e) {
                const int ce = e < deg[i] ? p->h_col_idx[p->h_row_ptr[i] + e] : i;  // padding: self, zero block
                cols[scol[s] + e * 32 + lane] = ce;
                if (e < deg[i]) map[p->h_row_ptr[i] + e] = sval[s] + (long long)e * ((b * b + 1) / 2) * 64 + 2 * lane;
            }
        }
    }
    for (int i = 0; i < n; ++i)
        for (int e = p->h_row_ptr[i]; e < p->h_row_ptr[i + 1]; ++e) {
            const int j = p->h_col_idx[e];
            const auto b0 = p->h_col_idx.begin() + p->h_row_ptr[j];
            const auto b1 = p->h_col_idx.begin() + p->h_row_ptr[j + 1];
            trans[e] = map[std::lower_bound(b0, b1, i) - p->h_col_idx.begin()];
        }
    L_.slice_val.upload(sval.data(), sval.size());
    L_.slice_col.upload(scol.data(), scol.size());
    L_.deg.upload(deg.data(), n);
    L_.dslot.upload(dslot.data(), n);
    L_.cols.upload(cols.data(), cols.size());
    L_.csr_to_sell.upload(map.data(), map.size());
    trans_.upload(trans.data(), trans.size());
    vals_.alloc(std::max<long long>(L_.total_vals, 1));
    FNLH_CUDA(cudaMemset(vals_.ptr, 0, vals_.bytes()));
    legacy_sync();
    grid0 = nb(n0);
    grid1 = nb(n - n0);
    partials.alloc(std::max(4 * (grid0 + grid1), nb((long long)n * b)) + 8);  // slice-granular variants: 4 per 128-row group
}

void RbSystem::load(const double* A_csr, cudaStream_t stm) {
    const int bb = L_.b * L_.b;
    { ::fnlh::note_launch(); k_to_sell<<<nb((long long)p_->nnzb * bb), kT, 0, stm>>>(A_csr, L_.csr_to_sell.ptr, bb, p_->nnzb, vals_.ptr); }
    FNLH_CUDA(cudaGetLastError());
}

__global__ void k_status_init(int* status) {
    status[0] = 0;
    status[1] = 0x7fffffff;
}

template <class S>
void rb_factorize_async(const RbSystem& A, const double* shift_im, RbIlu<S>& f, int* status, cudaStream_t stm) {
    const SellLayout& L = A.layout();
    const SellDev sd = sell_dev(L, A.vals());
    { ::fnlh::note_launch(); k_status_init<<<1, 1, 0, stm>>>(status); }
    RB_DISPATCH(L.b, {
        { ::fnlh::note_launch(); k_rb_factor0<B, S><<<A.grid0, kT, 0, stm>>>(sd, shift_im, f.diag_lu, f.diag_piv, f.inv0, status); }
        { ::fnlh::note_launch(); k_rb_factor1<B, S><<<A.grid1, kT, 0, stm>>>(sd, A.pattern()->row_ptr, A.trans(), shift_im, f.diag_lu,
                                                           f.diag_piv, f.inv0, status); }
    });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void rb_factorize(const RbSystem& A, const double* shift_im, RbIlu<S>& f, Workspace& ws) {
    rb_factorize_async<S>(A, shift_im, f, ws.status, ws.stream);
    FNLH_CUDA(cudaMemcpyAsync(ws.h_status, ws.status, 2 * sizeof(int), cudaMemcpyDeviceToHost, ws.stream));
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    if (ws.h_status[1] != 0x7fffffff) throw FactorizationError("near-singular ILU pivot block", ws.h_status[1]);
}

template <class S>
void rb_smoothed_solve_batch(const RbSystem& A, const RbMember<S>* mem, int P, double tol_rel, int max_iter,
                             cudaStream_t stm) {
    if (!(tol_rel > 0.0 && tol_rel < 1.0)) throw ConfigError("smoothed_solve: tol_rel must be in (0,1)");
    if (max_iter < 1) throw ConfigError("smoothed_solve: max_iter must be >= 1");
    if (P < 1 || P > kMaxBatch) throw ConfigError("rb_smoothed_solve_batch: 1 <= P <= kMaxBatch");
    const SellLayout& L = A.layout();
    const SellDev sd = sell_dev(L, A.vals());
    const std::size_t len = (std::size_t)L.n * L.b;
    RbTab<S> T{};
    T.P = P;
    for (int m = 0; m < P; ++m) {
        T.diag_lu[m] = mem[m].f->diag_lu;
        T.piv[m] = mem[m].f->diag_piv;
        T.inv0[m] = mem[m].f->inv0;
        T.shift[m] = mem[m].shift;
        T.rhs[m] = mem[m].rhs;
        T.x[m] = mem[m].x;
        T.z[m] = mem[m].z;
        T.r[m] = mem[m].r;
        T.ctl[m] = mem[m].ctl;
        T.parts[m] = mem[m].partials;
        FNLH_CUDA(cudaMemsetAsync(mem[m].x, 0, len * sizeof(S), stm));
        FNLH_CUDA(cudaMemsetAsync(mem[m].ctl, 0, sizeof(RbControl), stm));
    }
    const int gi = std::min(nb((long long)len), 1184);
    { ::fnlh::note_launch(); k_rb_init<S><<<gi * P, kT, 0, stm>>>(len, T, tol_rel); }
    const int maxoff = std::max(1, A.pattern()->max_deg - 1);
    const int g0 = A.grid0 * P, g1 = A.grid1 * P;
    RB_DISPATCH(L.b, {
        const std::size_t sm = (std::size_t)maxoff * B * kT * sizeof(S);
        // every call: function attributes belong to the current device's context (a process may
        // drive several GPUs, fnlh_set_device), and setting one is a host-side table update
        FNLH_CUDA(cudaFuncSetAttribute(k_rb_colour0<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        FNLH_CUDA(cudaFuncSetAttribute(k_rbx_colour1<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        const int E = maxoff;
        if (rb_sweep_mode() == 3) {  // edge-parallel colour-1 kernel (same arithmetic, bitwise)
            const std::size_t sme = (std::size_t)2 * E * B * 32 * sizeof(S);
            FNLH_CUDA(cudaFuncSetAttribute(k_rbe_colour1<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sme));
            if (32 * E > 192) throw ShapeError("rb: edge-parallel sweep needs <= 6 lower blocks per row");
            FNLH_CUDA(cudaFuncSetAttribute(k_rbe_colour0<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sme));
            const int ns0 = (L.n0 + 31) / 32, ns1 = (L.n - L.n0 + 31) / 32;
            { ::fnlh::note_launch(); k_rb_forward1<B, S><<<g1, kT, 0, stm>>>(sd, T, 1); }
            for (int s = 1; s <= max_iter; ++s) {
                { ::fnlh::note_launch(); k_rbe_colour0<B, S><<<ns0 * P, 32 * E, sme, stm>>>(sd, T, s, E); }
                { ::fnlh::note_launch(); k_rbe_colour1<B, S><<<ns1 * P, 32 * E, sme, stm>>>(sd, T, ns0, s, max_iter, s < max_iter ? 1 : 0, E); }
            }
        } else if (rb_sweep_mode() == 1) {
            for (int s = 1; s <= max_iter; ++s) {
                { ::fnlh::note_launch(); k_rb_forward1<B, S><<<g1, kT, 0, stm>>>(sd, T, s); }
                { ::fnlh::note_launch(); k_rb_colour0<B, S><<<g0, kT, sm, stm>>>(sd, T, s); }
                { ::fnlh::note_launch(); k_rb_resid1<B, S><<<g1, kT, 0, stm>>>(sd, T, A.grid0, s, max_iter); }
            }
        } else if (rb_sweep_mode() == 4 && P > 1) {  // lane-warp CTAs (same arithmetic and norms, bitwise)
            int gmax = 4;  // lanes per CTA (measurement override: FNLH_RB_LW_G=1..4)
            if (const char* e = std::getenv("FNLH_RB_LW_G")) gmax = std::min(4, std::max(1, std::atoi(e)));
            const int ng = (P + gmax - 1) / gmax, G = (P + ng - 1) / ng;
            const int ns0 = (L.n0 + 31) / 32, ns1 = (L.n - L.n0 + 31) / 32;
            const std::size_t smw = (std::size_t)maxoff * B * 32 * G * sizeof(S);
            FNLH_CUDA(cudaFuncSetAttribute(k_rb_colour0<B, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            { ::fnlh::note_launch(); k_rb_forward1<B, S><<<g1, kT, 0, stm>>>(sd, T, 1); }
            for (int s = 1; s <= max_iter; ++s) {
                { ::fnlh::note_launch(); k_rb_colour0<B, S, true><<<ns0 * ng, 32 * G, smw, stm>>>(sd, T, s, G); }
                { ::fnlh::note_launch(); k_rbx_colour1<B, S, true><<<ns1 * ng, 32 * G, 0, stm>>>(sd, T, A.grid0, s, max_iter, s < max_iter ? 1 : 0, G); }
            }
        } else if ((rb_sweep_mode() == 5 || rb_sweep_mode() == 6) && P > 1 && std::is_same<S, cplx>::value &&
                   (std::size_t)(maxoff + 1) * pairs<B>() * 512 + (std::size_t)(B + 1) * B * 128 * sizeof(cplx) <= 113 * 1024) {
            // staged colour-1 kernel (same arithmetic and norms, bitwise); colour 0 as mode 0
            if constexpr (std::is_same<S, cplx>::value) {
                const int ng = (P + 3) / 4, G = (P + ng - 1) / ng;
                const int ns1 = (L.n - L.n0 + 31) / 32;
                const int abytes = (maxoff + 1) * pairs<B>() * 512;
                const bool ringed = rb_sweep_mode() == 5;
                const std::size_t sms = (std::size_t)abytes + (ringed ? (std::size_t)(B + 1) * B * 32 * G * sizeof(cplx) : 0);
                FNLH_CUDA(cudaFuncSetAttribute(k_rbs_colour1<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms));
                FNLH_CUDA(cudaFuncSetAttribute(k_rbs_colour1<B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms));
                { ::fnlh::note_launch(); k_rb_forward1<B, S><<<g1, kT, 0, stm>>>(sd, T, 1); }
                for (int s = 1; s <= max_iter; ++s) {
                    { ::fnlh::note_launch(); k_rb_colour0<B, S><<<g0, kT, sm, stm>>>(sd, T, s); }
                    if (ringed) { ::fnlh::note_launch(); k_rbs_colour1<B, true><<<ns1 * ng, 32 * G, sms, stm>>>(sd, T, A.grid0, s, max_iter, s < max_iter ? 1 : 0, G, abytes, 0); }
                    else { ::fnlh::note_launch(); k_rbs_colour1<B, false><<<ns1 * ng, 32 * G, sms, stm>>>(sd, T, A.grid0, s, max_iter, s < max_iter ? 1 : 0, G, abytes, 0); }
                }
            }
        } else if (rb_sweep_mode() == 0 || rb_sweep_mode() >= 4) {
            { ::fnlh::note_launch(); k_rb_forward1<B, S><<<g1, kT, 0, stm>>>(sd, T, 1); }
            for (int s = 1; s <= max_iter; ++s) {
                { ::fnlh::note_launch(); k_rb_colour0<B, S><<<g0, kT, sm, stm>>>(sd, T, s); }
                { ::fnlh::note_launch(); k_rbx_colour1<B, S><<<g1, kT, 0, stm>>>(sd, T, A.grid0, s, max_iter, s < max_iter ? 1 : 0); }
            }
        } else {
            { ::fnlh::note_launch(); k_rbf_w0<B, S><<<g0, kT, 0, stm>>>(sd, T); }
            { ::fnlh::note_launch(); k_rbf_colour1<B, S><<<g1, kT, 0, stm>>>(sd, T, A.grid0, 0, max_iter, 1); }
            for (int s = 1; s <= max_iter; ++s) {
                { ::fnlh::note_launch(); k_rbf_colour0<B, S><<<g0, kT, 0, stm>>>(sd, T, s); }
                { ::fnlh::note_launch(); k_rbf_colour1<B, S><<<g1, kT, 0, stm>>>(sd, T, A.grid0, s, max_iter, s < max_iter ? 1 : 0); }
            }
        }
    });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void rb_smoothed_solve(const RbSystem& A, const double* shift_im, const RbIlu<S>& f, const S* rhs, double tol_rel,
                       int max_iter, S* x, S* z, S* r, RbControl* ctl, Workspace& ws) {
    RbMember<S> m{&f, shift_im, rhs, x, z, r, ctl, const_cast<double*>(A.partials.ptr)};
    rb_smoothed_solve_batch<S>(A, &m, 1, tol_rel, max_iter, ws.stream);
}

template struct RbIlu<double>;
template struct RbIlu<cplx>;
template void rb_factorize<double>(const RbSystem&, const double*, RbIlu<double>&, Workspace&);
template void rb_factorize_async<double>(const RbSystem&, const double*, RbIlu<double>&, int*, cudaStream_t);
template void rb_factorize_async<cplx>(const RbSystem&, const double*, RbIlu<cplx>&, int*, cudaStream_t);
template void rb_factorize<cplx>(const RbSystem&, const double*, RbIlu<cplx>&, Workspace&);
template void rb_smoothed_solve<double>(const RbSystem&, const double*, const RbIlu<double>&, const double*, double,
                                        int, double*, double*, double*, RbControl*, Workspace&);
template void rb_smoothed_solve<cplx>(const RbSystem&, const double*, const RbIlu<cplx>&, const cplx*, double, int,
                                      cplx*, cplx*, cplx*, RbControl*, Workspace&);
template void rb_smoothed_solve_batch<double>(const RbSystem&, const RbMember<double>*, int, double, int, cudaStream_t);
template void rb_smoothed_solve_batch<cplx>(const RbSystem&, const RbMember<cplx>*, int, double, int, cudaStream_t);

}  // namespace fnlh
