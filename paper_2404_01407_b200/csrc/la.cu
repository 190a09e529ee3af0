// la.cu -- device block-sparse LA (sparse.hpp/.cpp restated for sm_100a).
//
// Ordering contract: the device runs the reference's natural-order ILU(0) loops
// (sparse.cpp:187-291) level by level.  Within a row the arithmetic follows the
// reference operation by operation (compiled with --fmad=false), so factors and
// substitutions are bitwise identical to the reference except where a complex
// magnitude (hypot vs cabs) breaks a pivot tie.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "errors.hpp"
#include "la.cuh"

namespace fnlh {

namespace {

constexpr int kThreads = 128;
constexpr int kRedBlocks = 592;  // 4 x 148 SMs (norm reductions; callers' partial buffers hold 592)
constexpr int kMvBlocks = 2368;  // 16 x 148: matvec-residual grid (rows per thread ~ N / 303k; enough warps in flight)

struct PatDev {
    int b, rows, nnzb;
    const int* __restrict__ row_ptr;
    const int* __restrict__ col_idx;
    const int* __restrict__ diag_idx;
    const int* __restrict__ part;
    // sliced factor layout (la.cuh DevicePattern)
    const long long* __restrict__ ent;
    const long long* __restrict__ lbase;
    const long long* __restrict__ ubase;
    const int* __restrict__ lcolb;
    const int* __restrict__ ucolb;
    const int* __restrict__ nlow;
    const int* __restrict__ nup;
    const int* __restrict__ lcols;
    const int* __restrict__ ucols;
    const int* __restrict__ dpos;
    const int* __restrict__ blk_e;
    const int* __restrict__ blk_row;
    const long long* __restrict__ mbase;
    const int* __restrict__ mcolb;
    const int* __restrict__ mcols;
    const long long* __restrict__ kjo;
    const long long* __restrict__ kj;
};

PatDev dev(const DevicePattern& p) {
    return PatDev{p.b, p.rows, p.nnzb, p.row_ptr, p.col_idx, p.diag_idx, p.part, p.ent, p.lbase, p.ubase,
                  p.lcolb, p.ucolb, p.nlow, p.nup, p.lcols, p.ucols, p.dpos, p.blk_e, p.blk_row,
                  p.mbase, p.mcolb, p.mcols, p.kjo, p.kj};
}

// b x b block at g with element stride 32 (sliced layout)
template <int B, class S>
__device__ __forceinline__ void load_blk32(const S* __restrict__ g, S (&A)[B * B]) {
#pragma unroll
    for (int k = 0; k < B * B; ++k) A[k] = g[(std::size_t)k * 32];
}
template <int B, class S>
__device__ __forceinline__ void store_blk32(S* __restrict__ g, const S (&A)[B * B]) {
#pragma unroll
    for (int k = 0; k < B * B; ++k) g[(std::size_t)k * 32] = A[k];
}
// element offsets of row i's pivot LU (element stride 32) and pivots in the pivot layout
__device__ __forceinline__ long long dlu_off(const PatDev& p, int i, int bb) {
    const int d = p.dpos[i];
    return (long long)(d >> 5) * bb * 32 + (d & 31);
}

inline int nblocks(long long n, int t = kThreads) { return static_cast<int>((n + t - 1) / t); }

__device__ __forceinline__ int find_entry(const PatDev& p, int i, int j) {  // sparse.cpp:42-48
    int lo = p.row_ptr[i], hi = p.row_ptr[i + 1];
    const int end = hi;
    while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if (p.col_idx[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo == end || p.col_idx[lo] != j) ? -1 : lo;
}

// value of system entry e (row i) element k = r*B+c
template <int B, class S>
__device__ __forceinline__ S sys_entry(const SystemView<S>& A, int e, int k, bool diag, int i) {
    if (A.vals) return A.vals[(size_t)e * B * B + k];
    S v = from_real<S>(A.real_vals[(size_t)e * B * B + k]);
    if constexpr (sizeof(S) == sizeof(cplx)) {
        if (diag && A.shift_im && (k / B == k % B)) v = v + mk(0.0, A.shift_im[i]);  // d[m][m] += s_i
    }
    return v;
}

// the factorization's (k, j) lookups (find_entry, sparse.cpp:42-48), once per pattern: for
// row i, each lower entry ek and each later entry ej of the row, the sliced offset of
// U_kj = entry (k, col ej), or -1
__global__ void k_build_kj(PatDev p, long long* __restrict__ kj) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.rows) return;
    const int rb = p.row_ptr[i], re = p.row_ptr[i + 1];
    long long pos = p.kjo[i];
    for (int ek = rb; ek < re; ++ek) {
        const int k = p.col_idx[ek];
        if (k >= i) break;
        for (int ej = ek + 1; ej < re; ++ej) {
            const int e = find_entry(p, k, p.col_idx[ej]);
            kj[pos++] = e < 0 ? -1 : p.ent[e];
        }
    }
}

// Ilu::factorize copy phase (sparse.cpp:199-209): one thread per block position of the
// sliced layout (blk_e / blk_row: source entry and row, -1 for padding), so each element
// store of a warp is 32 consecutive lanes
template <int B, class S>
__global__ void k_ilu_copy(PatDev p, SystemView<S> A, S* __restrict__ vals, long long npos) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= npos) return;
    const int e = p.blk_e[t];
    if (e < 0) return;
    const int i = p.blk_row[t];
    const bool keep = p.part[p.col_idx[e]] == p.part[i];
    const bool diag = e == p.diag_idx[i];
    S* dst = vals + (t >> 5) * (long long)(B * B) * 32 + (t & 31);
#pragma unroll
    for (int k = 0; k < B * B; ++k) dst[(long long)k * 32] = keep ? sys_entry<B, S>(A, e, k, diag, i) : zero<S>();
}

// Ilu::factorize elimination + pivot phase for the rows of one level (sparse.cpp:214-255)
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_ilu_factor(PatDev p, const int* __restrict__ rows, int nrows,
                                                         S* vals, S* __restrict__ diag_lu,
                                                         int* __restrict__ diag_piv, S* diag_inv,
                                                         int* __restrict__ status) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const int i = rows[t];
    const int pi = p.part[i];
    const int rb = p.row_ptr[i], re = p.row_ptr[i + 1];
    long long pos = p.kjo[i];  // (ek, ej > ek) -> offset of U_kj, precomputed (la.cuh kj)
    for (int ek = rb; ek < re; ++ek) {
        const int k = p.col_idx[ek];
        if (k >= i) break;
        const long long kb = pos;
        pos += re - ek - 1;
        if (p.part[k] != pi) continue;
        // L_ik = A_ik * U_kk^{-1}
        S tmp[B * B];
        const S* uinv = diag_inv + (size_t)k * B * B;
        S* const lik = vals + p.ent[ek];
#pragma unroll
        for (int r = 0; r < B; ++r) {  // one row of A_ik at a time (register pressure)
            S lrow[B];
#pragma unroll
            for (int m = 0; m < B; ++m) lrow[m] = lik[(r * B + m) * 32];
#pragma unroll
            for (int c = 0; c < B; ++c) {
                S acc = zero<S>();
#pragma unroll
                for (int m = 0; m < B; ++m) acc += lrow[m] * uinv[m * B + c];
                tmp[r * B + c] = acc;
            }
        }
        store_blk32<B>(lik, tmp);
        // A_ij -= L_ik U_kj for j > k present in both rows (zero-skip, dense.hpp:47)
        for (int ej = ek + 1; ej < re; ++ej) {  // columns ascend: exactly the entries with j > k
            const long long uo = p.kj[kb + (ej - ek - 1)];
            const int j = p.col_idx[ej];
            if (p.part[j] != pi) continue;
            if (uo < 0) continue;  // (k, j) not in the pattern (find, sparse.cpp:42-48)
            if (p.part[k] != p.part[j]) continue;
            const S* u = vals + uo;
            S* cblk = vals + p.ent[ej];
#pragma unroll
            for (int r = 0; r < B; ++r) {  // block_matmul_sub row by row (same operation order)
                S crow[B];
#pragma unroll
                for (int c = 0; c < B; ++c) crow[c] = cblk[(r * B + c) * 32];
#pragma unroll
                for (int kk = 0; kk < B; ++kk) {
                    const S a = tmp[r * B + kk];
                    if (is_zero(a)) continue;
#pragma unroll
                    for (int c = 0; c < B; ++c) crow[c] -= a * u[(kk * B + c) * 32];
                }
#pragma unroll
                for (int c = 0; c < B; ++c) cblk[(r * B + c) * 32] = crow[c];
            }
        }
    }
    // pivot block: partial-pivot LU, condition check, explicit inverse
    S lu[B * B];
    int piv[B];
    load_blk32<B>(vals + p.ent[p.diag_idx[i]], lu);
    double cond = 0.0;
    const int sing = lu_factor_reg<B>(lu, piv, cond);
    if (sing || !(cond < 1e14)) atomicMin(status + 1, i);
    const long long dl = dlu_off(p, i, B * B);
    store_blk32<B>(diag_lu + dl, lu);
    const long long dp = dlu_off(p, i, B);
#pragma unroll
    for (int k = 0; k < B; ++k) diag_piv[dp + k * 32] = piv[k];
    S* inv = diag_inv + (size_t)i * B * B;
#pragma unroll
    for (int c = 0; c < B; ++c) {
        S col[B];
#pragma unroll
        for (int r = 0; r < B; ++r) col[r] = (r == c) ? one<S>() : zero<S>();
        lu_solve_reg<B>(lu, piv, col);
#pragma unroll
        for (int r = 0; r < B; ++r) inv[r * B + c] = col[r];
    }
}

// Ilu::apply forward substitution (sparse.cpp:267-278) for one level
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_ilu_fwd(PatDev p, const int* __restrict__ rows, int nrows,
                                                      const S* __restrict__ vals, const S* __restrict__ rhs,
                                                      S* x) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const int i = rows[t];
    const int pi = p.part[i];
    S xi[B];
    load_vec<B>(rhs + (size_t)i * B, xi);
    const long long lb = p.lbase[i];
    const int cb = p.lcolb[i], nl = p.nlow[i];
    for (int s = 0; s < nl; ++s) {  // lower entries, ascending column (slots of the sliced layout)
        const int k = p.lcols[cb + s * 32];
        if (p.part[k] != pi) continue;
        const S* blk = vals + lb + (long long)s * B * B * 32;
        const S* xk = x + (size_t)k * B;
        S xkv[B];
        load_vec<B>(xk, xkv);
#pragma unroll
        for (int r = 0; r < B; ++r) {  // block_matvec_sub (dense.hpp:31-39)
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) acc += blk[(r * B + c) * 32] * xkv[c];
            xi[r] -= acc;
        }
    }
    store_vec<B>(x + (size_t)i * B, xi);
}

// Ilu::apply backward substitution + pivot solve (sparse.cpp:279-290) for one level;
// optionally x_accum += x (the smoothed_solve update x += z, sparse.hpp:317)
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_ilu_bwd(PatDev p, const int* __restrict__ rows, int nrows,
                                                      const S* __restrict__ vals, const S* __restrict__ diag_lu,
                                                      const int* __restrict__ diag_piv, S* x, S* x_accum) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const int i = rows[t];
    const int pi = p.part[i];
    S xi[B];
    load_vec<B>(x + (size_t)i * B, xi);
    const long long ub = p.ubase[i];
    const int cb = p.ucolb[i], nu = p.nup[i];
    for (int s = 0; s < nu; ++s) {  // upper entries, descending column
        const int j = p.ucols[cb + s * 32];
        if (p.part[j] != pi) continue;
        const S* blk = vals + ub + (long long)s * B * B * 32;
        S xjv[B];
        load_vec<B>(x + (size_t)j * B, xjv);
#pragma unroll
        for (int r = 0; r < B; ++r) {
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) acc += blk[(r * B + c) * 32] * xjv[c];
            xi[r] -= acc;
        }
    }
    S lu[B * B];
    int piv[B];
    load_blk32<B>(diag_lu + dlu_off(p, i, B * B), lu);
    const long long dp = dlu_off(p, i, B);
#pragma unroll
    for (int k = 0; k < B; ++k) piv[k] = diag_piv[dp + k * 32];
    lu_solve_reg<B>(lu, piv, xi);
    store_vec<B>(x + (size_t)i * B, xi);
    if (x_accum) {
        S* xa = x_accum + (size_t)i * B;
#pragma unroll
        for (int k = 0; k < B; ++k) xa[k] += xi[k];
    }
}

// y_i = sum over the row's entries (ascending) of A_e x_col(e) from the sliced copy of the
// real A (16-byte element pairs, lane-minor), the diagonal block carrying the complex shift
// (shift_diagonal): k_matvec's arithmetic, operation by operation
template <int B, class S>
__device__ __forceinline__ void sell_row_matvec(const PatDev& p, const double* __restrict__ sell, int i,
                                                const S* __restrict__ x, const double* __restrict__ shift,
                                                S (&y)[B]) {
    constexpr int NP = (B * B + 1) / 2;
    const double2* base = reinterpret_cast<const double2*>(sell + p.mbase[i]);
    const int cb = p.mcolb[i], deg = p.row_ptr[i + 1] - p.row_ptr[i], dq = p.diag_idx[i] - p.row_ptr[i];
#pragma unroll
    for (int r = 0; r < B; ++r) y[r] = zero<S>();
    for (int q = 0; q < deg; ++q) {
        S xc[B];
        load_vec<B>(x + (size_t)p.mcols[cb + q * 32] * B, xc);
        double blk[2 * NP];
#pragma unroll
        for (int t = 0; t < NP; ++t) {
            const double2 v = __ldg(base + (long long)(q * NP + t) * 32);
            blk[2 * t] = v.x;
            blk[2 * t + 1] = v.y;
        }
        const bool diag = q == dq;
#pragma unroll
        for (int r = 0; r < B; ++r) {
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) {
                if constexpr (sizeof(S) == sizeof(cplx)) {
                    if (diag && r == c && shift)
                        acc += mk(blk[r * B + c] + 0.0, 0.0 + shift[i]) * xc[c];
                    else
                        acc += rmul(blk[r * B + c], xc[c]);
                } else {
                    acc += rmul(blk[r * B + c], xc[c]);
                }
            }
            y[r] += acc;
        }
    }
}

__global__ void k_sell_copy(const int* __restrict__ mblk_e, long long npos, int bb, const double* __restrict__ bsr,
                            double* __restrict__ sell) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= npos) return;
    const int e = mblk_e[t];
    if (e < 0) return;
    const int np = (bb + 1) / 2;
    double* dst = sell + (t >> 5) * np * 64 + 2 * (t & 31);
    for (int k = 0; k < bb; ++k) dst[(k >> 1) * 64 + (k & 1)] = bsr[(long long)e * bb + k];
}

// y_i = sum_e A_e x_col(e) (Bsr::matvec, sparse.hpp:259-270); with rhs: r = rhs - y
// (sparse.hpp:319) and per-block partial sums of |r|^2
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_matvec(PatDev p, SystemView<S> A, const S* __restrict__ x,
                                                     const S* __restrict__ rhs, S* __restrict__ out,
                                                     double* __restrict__ partials) {
    __shared__ double red[kThreads / 32];
    double local = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.rows; i += gridDim.x * blockDim.x) {
        S y[B];
#pragma unroll
        for (int r = 0; r < B; ++r) y[r] = zero<S>();
        const int di = p.diag_idx[i];
        if (!A.vals && A.real_sell) sell_row_matvec<B, S>(p, A.real_sell, i, x, A.shift_im, y);
        else for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
            S xc[B];
            load_vec<B>(x + (size_t)p.col_idx[e] * B, xc);
            const bool diag = e == di;
            if (A.vals) {
                const S* blk = A.vals + (size_t)e * B * B;
#pragma unroll
                for (int r = 0; r < B; ++r) {
                    S acc = zero<S>();
#pragma unroll
                    for (int c = 0; c < B; ++c) acc += blk[r * B + c] * xc[c];
                    y[r] += acc;
                }
            } else {
                const double* blk = A.real_vals + (size_t)e * B * B;
#pragma unroll
                for (int r = 0; r < B; ++r) {
                    S acc = zero<S>();
#pragma unroll
                    for (int c = 0; c < B; ++c) {
                        if constexpr (sizeof(S) == sizeof(cplx)) {
                            if (diag && r == c && A.shift_im)
                                acc += mk(blk[r * B + c] + 0.0, 0.0 + A.shift_im[i]) * xc[c];
                            else
                                acc += rmul(blk[r * B + c], xc[c]);
                        } else {
                            acc += rmul(blk[r * B + c], xc[c]);
                        }
                    }
                    y[r] += acc;
                }
            }
        }
        S* o = out + (size_t)i * B;
        if (rhs) {
            const S* b = rhs + (size_t)i * B;
#pragma unroll
            for (int r = 0; r < B; ++r) {
                const S v = b[r] - y[r];
                o[r] = v;
                local += sq(v);
            }
        } else {
#pragma unroll
            for (int r = 0; r < B; ++r) o[r] = y[r];
        }
    }
    if (partials) {
        for (int off = 16; off > 0; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += red[w];
            partials[blockIdx.x] = s;
        }
    }
}

template <class S>
__global__ void k_sumsq(const S* __restrict__ x, std::size_t len, double* __restrict__ partials) {
    __shared__ double red[kThreads / 32];
    double local = 0.0;
    for (std::size_t k = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; k < len;
         k += (std::size_t)gridDim.x * blockDim.x)
        local += sq(x[k]);
    for (int off = 16; off > 0; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += red[w];
        partials[blockIdx.x] = s;
    }
}

// ---- batched level-scheduled Richardson: P systems sharing the real A (harmonic lanes)
// CTA b serves lane b % P, so the P CTAs reading the same rows of A run back to back.
template <class S>
struct LaLanes {
    const S* vals[kMaxLanes];
    const S* diag_lu[kMaxLanes];
    const int* diag_piv[kMaxLanes];
    const double* shift[kMaxLanes];
    const S* rhs[kMaxLanes];
    S* x[kMaxLanes];
    S* z[kMaxLanes];
    S* r[kMaxLanes];
    double* parts[kMaxLanes];
    const int* active;  // [P] 1 while the lane iterates
    int P;
};

template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_ilu_fwd_b(PatDev p, const int* __restrict__ rows, int nrows,
                                                        LaLanes<S> T) {
    const int lane = blockIdx.x % T.P;
    if (!T.active[lane]) return;
    const int t = (blockIdx.x / T.P) * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const S* __restrict__ vals = T.vals[lane];
    S* x = T.z[lane];
    const int i = rows[t];
    const int pi = p.part[i];
    S xi[B];
    load_vec<B>(T.r[lane] + (size_t)i * B, xi);
    const long long lb = p.lbase[i];
    const int cb = p.lcolb[i], nl = p.nlow[i];
    for (int s = 0; s < nl; ++s) {  // lower entries, ascending column (slots of the sliced layout)
        const int k = p.lcols[cb + s * 32];
        if (p.part[k] != pi) continue;
        const S* blk = vals + lb + (long long)s * B * B * 32;
        S xkv[B];
        load_vec<B>(x + (size_t)k * B, xkv);
#pragma unroll
        for (int r = 0; r < B; ++r) {
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) acc += blk[(r * B + c) * 32] * xkv[c];
            xi[r] -= acc;
        }
    }
    store_vec<B>(x + (size_t)i * B, xi);
}

template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_ilu_bwd_b(PatDev p, const int* __restrict__ rows, int nrows,
                                                        LaLanes<S> T) {
    const int lane = blockIdx.x % T.P;
    if (!T.active[lane]) return;
    const int t = (blockIdx.x / T.P) * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const S* __restrict__ vals = T.vals[lane];
    S* x = T.z[lane];
    const int i = rows[t];
    const int pi = p.part[i];
    S xi[B];
    load_vec<B>(x + (size_t)i * B, xi);
    const long long ub = p.ubase[i];
    const int cb = p.ucolb[i], nu = p.nup[i];
    for (int s = 0; s < nu; ++s) {  // upper entries, descending column
        const int j = p.ucols[cb + s * 32];
        if (p.part[j] != pi) continue;
        const S* blk = vals + ub + (long long)s * B * B * 32;
        S xjv[B];
        load_vec<B>(x + (size_t)j * B, xjv);
#pragma unroll
        for (int r = 0; r < B; ++r) {
            S acc = zero<S>();
#pragma unroll
            for (int c = 0; c < B; ++c) acc += blk[(r * B + c) * 32] * xjv[c];
            xi[r] -= acc;
        }
    }
    S lu[B * B];
    int piv[B];
    load_blk32<B>(T.diag_lu[lane] + dlu_off(p, i, B * B), lu);
    const long long dp = dlu_off(p, i, B);
#pragma unroll
    for (int k = 0; k < B; ++k) piv[k] = T.diag_piv[lane][dp + k * 32];
    lu_solve_reg<B>(lu, piv, xi);
    store_vec<B>(x + (size_t)i * B, xi);
    S* xa = T.x[lane] + (size_t)i * B;
#pragma unroll
    for (int k = 0; k < B; ++k) xa[k] += xi[k];
}

// r = rhs - (A + i diag(shift)) x per lane (k_matvec's arithmetic), per-CTA |r|^2 partials
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_matvec_b(PatDev p, const double* __restrict__ Areal,
                                                       const double* __restrict__ Asell, LaLanes<S> T) {
    __shared__ double red[kThreads / 32];
    const int lane = blockIdx.x % T.P;
    if (!T.active[lane]) return;
    const int cta = blockIdx.x / T.P, nct = gridDim.x / T.P;
    const S* __restrict__ x = T.x[lane];
    const double* __restrict__ shift = T.shift[lane];
    double local = 0.0;
    for (int i = cta * blockDim.x + threadIdx.x; i < p.rows; i += nct * blockDim.x) {
        S y[B];
#pragma unroll
        for (int r = 0; r < B; ++r) y[r] = zero<S>();
        const int di = p.diag_idx[i];
        if (Asell) sell_row_matvec<B, S>(p, Asell, i, x, shift, y);
        else for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
            S xc[B];
            load_vec<B>(x + (size_t)p.col_idx[e] * B, xc);
            const bool diag = e == di;
            const double* blk = Areal + (size_t)e * B * B;
#pragma unroll
            for (int r = 0; r < B; ++r) {
                S acc = zero<S>();
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    if constexpr (sizeof(S) == sizeof(cplx)) {
                        if (diag && r == c && shift)
                            acc += mk(blk[r * B + c] + 0.0, 0.0 + shift[i]) * xc[c];
                        else
                            acc += rmul(blk[r * B + c], xc[c]);
                    } else {
                        acc += rmul(blk[r * B + c], xc[c]);
                    }
                }
                y[r] += acc;
            }
        }
        S* o = T.r[lane] + (size_t)i * B;
        const S* bb = T.rhs[lane] + (size_t)i * B;
#pragma unroll
        for (int r = 0; r < B; ++r) {
            const S v = bb[r] - y[r];
            o[r] = v;
            local += sq(v);
        }
    }
    for (int off = 16; off > 0; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += red[w];
        T.parts[lane][cta] = s;
    }
}

// k_matvec_b on the sliced A with one thread per row serving a group of up to kLG lanes:
// each block of A is loaded once into registers and applied to every lane's gathered x
// (the lanes' operations interleave, each lane's sum keeps k_matvec's order); rows, CTAs
// and per-lane partials exactly as k_matvec_b / k_matvec (same grid of CTAs per lane)
constexpr int kLG = 5;
template <int B, class S>
__global__ void __launch_bounds__(kThreads) k_matvec_lg(PatDev p, const double* __restrict__ sell, int lg,
                                                        LaLanes<S> T) {
    constexpr int NP = (B * B + 1) / 2;
    __shared__ double red[kLG][kThreads / 32];
    const int ng = (T.P + lg - 1) / lg;
    const int g = blockIdx.x % ng, cta = blockIdx.x / ng, nct = gridDim.x / ng;
    const int l0 = g * lg, nl = min(lg, T.P - l0);
    bool act[kLG];
#pragma unroll
    for (int q = 0; q < kLG; ++q) act[q] = q < nl && T.active[l0 + q];
    double local[kLG];
#pragma unroll
    for (int q = 0; q < kLG; ++q) local[q] = 0.0;
    for (int i = cta * blockDim.x + threadIdx.x; i < p.rows; i += nct * blockDim.x) {
        S y[kLG][B];
#pragma unroll
        for (int q = 0; q < kLG; ++q)
#pragma unroll
            for (int r = 0; r < B; ++r) y[q][r] = zero<S>();
        const double2* base = reinterpret_cast<const double2*>(sell + p.mbase[i]);
        const int cb = p.mcolb[i], deg = p.row_ptr[i + 1] - p.row_ptr[i], dq = p.diag_idx[i] - p.row_ptr[i];
        for (int e = 0; e < deg; ++e) {
            const int col = p.mcols[cb + e * 32];
            double blk[2 * NP];
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                const double2 v = __ldg(base + (long long)(e * NP + t) * 32);
                blk[2 * t] = v.x;
                blk[2 * t + 1] = v.y;
            }
            const bool diag = e == dq;
#pragma unroll
            for (int q = 0; q < kLG; ++q) {
                if (!act[q]) continue;
                S xc[B];
                load_vec<B>(T.x[l0 + q] + (size_t)col * B, xc);
                const double* shift = T.shift[l0 + q];
#pragma unroll
                for (int r = 0; r < B; ++r) {
                    S acc = zero<S>();
#pragma unroll
                    for (int c = 0; c < B; ++c) {
                        if constexpr (sizeof(S) == sizeof(cplx)) {
                            if (diag && r == c && shift)
                                acc += mk(blk[r * B + c] + 0.0, 0.0 + shift[i]) * xc[c];
                            else
                                acc += rmul(blk[r * B + c], xc[c]);
                        } else {
                            acc += rmul(blk[r * B + c], xc[c]);
                        }
                    }
                    y[q][r] += acc;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kLG; ++q) {
            if (!act[q]) continue;
            S* o = T.r[l0 + q] + (size_t)i * B;
            const S* bb = T.rhs[l0 + q] + (size_t)i * B;
#pragma unroll
            for (int r = 0; r < B; ++r) {
                const S v = bb[r] - y[q][r];
                o[r] = v;
                local[q] += sq(v);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kLG; ++q) {
        double v = local[q];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < kLG && act[threadIdx.x]) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += red[threadIdx.x][w];
        T.parts[l0 + threadIdx.x][cta] = s;
    }
}

// per-lane fixed-order sum of partials (block l = lane l)
__global__ void k_finish_b(LaLanes<cplx> Tc, LaLanes<double> Td, int is_cplx, int n, double* __restrict__ out) {
    __shared__ double red[32];
    const int lane = blockIdx.x;
    const double* partials = is_cplx ? Tc.parts[lane] : Td.parts[lane];
    double s = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) s += partials[k];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[lane] = t;
    }
}

// device-side stopping rule of smoothed_solve (sparse.hpp:305-328) per lane: control block
// [initial, final, target, iterations, converged, diverged] (8 doubles per lane)
__global__ void k_lane_init(int P, const double* __restrict__ norm_sq, double tol, int* __restrict__ active,
                            double* __restrict__ ctl) {
    const int l = threadIdx.x;
    if (l >= P) return;
    const double r0 = sqrt(norm_sq[l]);
    double* c = ctl + 8 * l;
    c[0] = r0;
    c[1] = r0;
    c[2] = tol * r0;
    c[3] = 0.0;
    c[4] = r0 == 0.0 ? 1.0 : 0.0;
    c[5] = 0.0;
    active[l] = r0 == 0.0 ? 0 : 1;
}
__global__ void k_lane_stop(int P, int it, const double* __restrict__ norm_sq, int* __restrict__ active,
                            double* __restrict__ ctl) {
    const int l = threadIdx.x;
    if (l >= P || !active[l]) return;
    const double nrm = sqrt(norm_sq[l]);
    double* c = ctl + 8 * l;
    c[1] = nrm;
    c[3] = it;
    if (!isfinite(nrm)) {
        c[5] = 1.0;
        active[l] = 0;
    } else if (nrm <= c[2]) {
        c[4] = 1.0;
        active[l] = 0;
    }
}

// fixed-order final reduction of the per-block partials (deterministic run to run)
__global__ void k_finish(const double* __restrict__ partials, int n, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) s += partials[k];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
    }
}

template <class S>
__global__ void k_axpy_copy(S* __restrict__ dst, const S* __restrict__ src, std::size_t len) {
    for (std::size_t k = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; k < len;
         k += (std::size_t)gridDim.x * blockDim.x)
        dst[k] = src[k];
}

template <int B, class S>
__global__ void k_block_diag_solve(int n, const S* __restrict__ lu, const int* __restrict__ piv,
                                   const S* __restrict__ rhs, S* __restrict__ x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    S L[B * B], v[B];
    int pv[B];
    load_block<B>(lu + (size_t)i * B * B, L);
#pragma unroll
    for (int k = 0; k < B; ++k) pv[k] = piv[(size_t)i * B + k];
    load_vec<B>(rhs + (size_t)i * B, v);
    lu_solve_reg<B>(L, pv, v);
    store_vec<B>(x + (size_t)i * B, v);
}

template <int B, class S>
__global__ void k_block_diag_factor(int n, S* __restrict__ blocks, int* __restrict__ piv, int* __restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    S L[B * B];
    int pv[B];
    load_block<B>(blocks + (size_t)i * B * B, L);
    double cond;
    if (lu_factor_reg<B>(L, pv, cond)) atomicMin(status + 1, i);
    store_block<B>(blocks + (size_t)i * B * B, L);
#pragma unroll
    for (int k = 0; k < B; ++k) piv[(size_t)i * B + k] = pv[k];
}

#define FNLH_DISPATCH_B(b, ...)                                              \
    switch (b) {                                                             \
        case 1: { constexpr int B = 1; __VA_ARGS__; } break;                 \
        case 3: { constexpr int B = 3; __VA_ARGS__; } break;                 \
        case 5: { constexpr int B = 5; __VA_ARGS__; } break;                 \
        case 6: { constexpr int B = 6; __VA_ARGS__; } break;                 \
        default: throw ShapeError("unsupported block size " + std::to_string(b)); \
    }

}  // namespace

// ---------------------------------------------------------------------------
// DevicePattern
// ---------------------------------------------------------------------------
DevicePattern::DevicePattern(int b_, int rows_, const int* row_ptr_, const int* col_idx_, const int* partition)
    : b(b_), rows(rows_) {
    nnzb = row_ptr_[rows];
    h_row_ptr.assign(row_ptr_, row_ptr_ + rows + 1);
    h_col_idx.assign(col_idx_, col_idx_ + nnzb);
    h_part.assign(rows, 0);
    if (partition) h_part.assign(partition, partition + rows);
    h_diag_idx.assign(rows, -1);
    for (int i = 0; i < rows; ++i) {
        max_deg = std::max(max_deg, h_row_ptr[i + 1] - h_row_ptr[i]);
        for (int e = h_row_ptr[i]; e < h_row_ptr[i + 1]; ++e) {
            if (e > h_row_ptr[i] && h_col_idx[e] <= h_col_idx[e - 1])
                throw ShapeError("pattern: columns must ascend in row " + std::to_string(i));
            if (h_col_idx[e] == i) h_diag_idx[i] = e;
        }
        if (h_diag_idx[i] < 0) throw ShapeError("pattern: missing diagonal entry in row " + std::to_string(i));
        if (h_part[i] != h_part[0]) single_partition = false;
    }
    // structural symmetry (BlockSparsityPattern::validate, sparse.cpp:50-59)
    for (int i = 0; i < rows; ++i)
        for (int e = h_row_ptr[i]; e < h_row_ptr[i + 1]; ++e) {
            const int j = h_col_idx[e];
            if (!std::binary_search(h_col_idx.begin() + h_row_ptr[j], h_col_idx.begin() + h_row_ptr[j + 1], i))
                throw ShapeError("pattern: structurally unsymmetric at (" + std::to_string(i) + "," +
                                 std::to_string(j) + ")");
        }
    // level schedules
    std::vector<int> lf(rows, 0), lb(rows, 0);
    int nf = 0, nb = 0;
    for (int i = 0; i < rows; ++i) {
        int l = 0;
        for (int e = h_row_ptr[i]; e < h_row_ptr[i + 1]; ++e) {
            const int k = h_col_idx[e];
            if (k >= i) break;
            if (h_part[k] == h_part[i]) l = std::max(l, lf[k] + 1);
        }
        lf[i] = l;
        nf = std::max(nf, l + 1);
    }
    for (int i = rows - 1; i >= 0; --i) {
        int l = 0;
        for (int e = h_row_ptr[i + 1] - 1; e >= h_row_ptr[i]; --e) {
            const int j = h_col_idx[e];
            if (j <= i) break;
            if (h_part[j] == h_part[i]) l = std::max(l, lb[j] + 1);
        }
        lb[i] = l;
        nb = std::max(nb, l + 1);
    }
    auto group = [&](const std::vector<int>& lev, int nl, std::vector<int>& ptr) {
        ptr.assign(nl + 1, 0);
        for (int i = 0; i < rows; ++i) ptr[lev[i] + 1]++;
        for (int l = 0; l < nl; ++l) ptr[l + 1] += ptr[l];
        std::vector<int> fill(ptr.begin(), ptr.end() - 1), out(rows);
        for (int i = 0; i < rows; ++i) out[fill[lev[i]]++] = i;
        return out;
    };
    std::vector<int> fr = group(lf, nf, fwd_ptr), br = group(lb, nb, bwd_ptr);
    // sliced factor layout (la.cuh): per-row lower / upper entry counts; rows of a level by
    // descending count (stable) so a slice's rows have similar slot counts
    const int bb = b * b;
    std::vector<int> nl(rows), nu(rows);
    for (int i = 0; i < rows; ++i) {
        nl[i] = h_diag_idx[i] - h_row_ptr[i];
        nu[i] = h_row_ptr[i + 1] - 1 - h_diag_idx[i];
    }
    auto by_count = [&](std::vector<int>& order, const std::vector<int>& ptr, const std::vector<int>& cnt) {
        for (std::size_t l = 0; l + 1 < ptr.size(); ++l)
            std::stable_sort(order.begin() + ptr[l], order.begin() + ptr[l + 1],
                             [&](int x, int y) { return cnt[x] > cnt[y]; });
    };
    by_count(fr, fwd_ptr, nl);
    by_count(br, bwd_ptr, nu);
    // slices of 32 consecutive rows of one level; returns per-row (slice, lane) and the
    // per-slice max count
    auto slices = [&](const std::vector<int>& order, const std::vector<int>& ptr, const std::vector<int>& cnt,
                      std::vector<int>& sl_of, std::vector<int>& lane_of, std::vector<int>& smax) {
        sl_of.assign(rows, 0);
        lane_of.assign(rows, 0);
        smax.clear();
        for (std::size_t l = 0; l + 1 < ptr.size(); ++l)
            for (int t = ptr[l]; t < ptr[l + 1]; ++t) {
                const int q = t - ptr[l];
                if ((q & 31) == 0) smax.push_back(0);
                const int i = order[t];
                sl_of[i] = (int)smax.size() - 1;
                lane_of[i] = q & 31;
                smax.back() = std::max(smax.back(), cnt[i]);
            }
    };
    std::vector<int> fsl, flane, fmax, bsl, blane, bmax;
    slices(fr, fwd_ptr, nl, fsl, flane, fmax);
    slices(br, bwd_ptr, nu, bsl, blane, bmax);
    n_dslices = (int)bmax.size();
    // element offsets: [L region][U region][diagonal entries (backward slices)]
    std::vector<long long> fv(fmax.size() + 1, 0), bv(bmax.size() + 1, 0);
    std::vector<int> fc(fmax.size() + 1, 0), bc(bmax.size() + 1, 0);
    for (std::size_t k = 0; k < fmax.size(); ++k) {
        fv[k + 1] = fv[k] + (long long)fmax[k] * bb * 32;
        fc[k + 1] = fc[k] + fmax[k] * 32;
    }
    for (std::size_t k = 0; k < bmax.size(); ++k) {
        bv[k + 1] = bv[k] + (long long)bmax[k] * bb * 32;
        bc[k + 1] = bc[k] + bmax[k] * 32;
    }
    const long long u0 = fv.back(), d0 = u0 + bv.back();
    sell_elems = d0 + (long long)n_dslices * bb * 32;
    std::vector<long long> hl(rows), hu(rows);
    std::vector<int> hlc(rows), huc(rows), lcs(std::max(fc.back(), 1), 0), ucs(std::max(bc.back(), 1), 0);
    h_ent.assign(nnzb, 0);
    h_dpos.assign(rows, 0);
    for (int i = 0; i < rows; ++i) {
        hl[i] = fv[fsl[i]] + flane[i];
        hlc[i] = fc[fsl[i]] + flane[i];
        hu[i] = u0 + bv[bsl[i]] + blane[i];
        huc[i] = bc[bsl[i]] + blane[i];
        h_dpos[i] = bsl[i] * 32 + blane[i];
        for (int q = 0; q < nl[i]; ++q) {
            const int e = h_row_ptr[i] + q;
            h_ent[e] = hl[i] + (long long)q * bb * 32;
            lcs[hlc[i] + q * 32] = h_col_idx[e];
        }
        for (int q = 0; q < nu[i]; ++q) {  // slot q = q-th entry from the row end
            const int e = h_row_ptr[i + 1] - 1 - q;
            h_ent[e] = hu[i] + (long long)q * bb * 32;
            ucs[huc[i] + q * 32] = h_col_idx[e];
        }
        h_ent[h_diag_idx[i]] = d0 + (long long)bsl[i] * bb * 32 + blane[i];
    }
    // natural 32-row slices of the matvec copy
    {
        const int np = (bb + 1) / 2, ns = (rows + 31) / 32;
        std::vector<long long> so(ns + 1, 0);
        std::vector<int> co(ns + 1, 0);
        for (int q = 0; q < ns; ++q) {
            int md = 0;
            for (int i = q * 32; i < std::min(rows, q * 32 + 32); ++i) md = std::max(md, h_row_ptr[i + 1] - h_row_ptr[i]);
            so[q + 1] = so[q] + (long long)md * np * 64;
            co[q + 1] = co[q] + md * 32;
        }
        msell_doubles = so[ns];
        std::vector<long long> mb(rows);
        std::vector<int> mc(rows), mcs(std::max(co[ns], 1), 0), mbe(std::max<long long>(so[ns] / (np * 2), 1), -1);
        for (int i = 0; i < rows; ++i) {
            const int q = i >> 5, l = i & 31;
            mb[i] = so[q] + 2 * l;
            mc[i] = co[q] + l;
            for (int t = 0; t < h_row_ptr[i + 1] - h_row_ptr[i]; ++t) {
                mcs[mc[i] + t * 32] = h_col_idx[h_row_ptr[i] + t];
                mbe[(so[q] / (np * 64) + t) * 32 + l] = h_row_ptr[i] + t;
            }
        }
        auto upl2 = [](long long** d, const std::vector<long long>& h) {
            FNLH_CUDA_ALLOC(d, std::max<std::size_t>(h.size(), 1) * sizeof(long long));
            if (!h.empty()) FNLH_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(long long), cudaMemcpyHostToDevice));
        };
        auto up2 = [](int** d, const std::vector<int>& h) {
            FNLH_CUDA_ALLOC(d, std::max<std::size_t>(h.size(), 1) * sizeof(int));
            if (!h.empty()) FNLH_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
        };
        upl2(&mbase, mb);
        up2(&mcolb, mc);
        up2(&mcols, mcs);
        up2(&mblk_e, mbe);
    }
    std::vector<int> be(sell_elems / bb, -1), br_(sell_elems / bb, -1);
    for (int i = 0; i < rows; ++i)
        for (int e = h_row_ptr[i]; e < h_row_ptr[i + 1]; ++e) {
            const long long pos = h_ent[e] / ((long long)bb * 32) * 32 + h_ent[e] % 32;
            be[pos] = e;
            br_[pos] = i;
        }
    auto up = [](int** d, const std::vector<int>& h) {
        FNLH_CUDA_ALLOC(d, std::max<std::size_t>(h.size(), 1) * sizeof(int));
        if (!h.empty()) FNLH_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
    };
    auto upl = [](long long** d, const std::vector<long long>& h) {
        FNLH_CUDA_ALLOC(d, std::max<std::size_t>(h.size(), 1) * sizeof(long long));
        if (!h.empty()) FNLH_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(long long), cudaMemcpyHostToDevice));
    };
    up(&row_ptr, h_row_ptr);
    up(&col_idx, h_col_idx);
    up(&diag_idx, h_diag_idx);
    up(&part, h_part);
    up(&fwd_rows, fr);
    up(&bwd_rows, br);
    upl(&ent, h_ent);
    upl(&lbase, hl);
    upl(&ubase, hu);
    up(&lcolb, hlc);
    up(&ucolb, huc);
    up(&nlow, nl);
    up(&nup, nu);
    up(&lcols, lcs);
    up(&ucols, ucs);
    up(&dpos, h_dpos);
    up(&blk_e, be);
    up(&blk_row, br_);
    {
        std::vector<long long> ko(rows + 1, 0);
        for (int i = 0; i < rows; ++i) {
            long long c = 0;
            for (int e = h_row_ptr[i]; e < h_row_ptr[i + 1] && h_col_idx[e] < i; ++e) c += h_row_ptr[i + 1] - e - 1;
            ko[i + 1] = ko[i] + c;
        }
        upl(&kjo, ko);
        FNLH_CUDA_ALLOC(&kj, std::max<long long>(ko[rows], 1) * sizeof(long long));
        if (rows) { ::fnlh::note_launch(); k_build_kj<<<nblocks(rows), kThreads>>>(dev(*this), kj); }
        FNLH_CUDA(cudaGetLastError());
    }
    legacy_sync();
}

DevicePattern::~DevicePattern() {
    fnlh::dfree(row_ptr);
    fnlh::dfree(col_idx);
    fnlh::dfree(diag_idx);
    fnlh::dfree(part);
    fnlh::dfree(fwd_rows);
    fnlh::dfree(bwd_rows);
    for (void* q : {(void*)ent, (void*)lbase, (void*)ubase, (void*)lcolb, (void*)ucolb, (void*)nlow, (void*)nup,
                    (void*)lcols, (void*)ucols, (void*)dpos, (void*)blk_e, (void*)blk_row, (void*)mbase,
                    (void*)mcolb, (void*)mcols, (void*)mblk_e, (void*)kjo, (void*)kj})
        fnlh::dfree(q);
}

template <class S>
DeviceIlu<S>::DeviceIlu(const DevicePattern* pat) : p(pat) {
    const std::size_t bb = (std::size_t)p->b * p->b;
    const std::size_t dr = (std::size_t)p->n_dslices * 32;
    FNLH_CUDA_ALLOC(&vals, std::max<std::size_t>(p->sell_elems, 1) * sizeof(S));
    FNLH_CUDA_ALLOC(&diag_lu, std::max<std::size_t>(dr * bb, 1) * sizeof(S));
    FNLH_CUDA_ALLOC(&diag_piv, std::max<std::size_t>(dr * p->b, 1) * sizeof(int));
    FNLH_CUDA_ALLOC(&diag_inv, (std::size_t)p->rows * bb * sizeof(S));
    // padding slots stay zero (never read as live entries)
    FNLH_CUDA(cudaMemset(vals, 0, std::max<std::size_t>(p->sell_elems, 1) * sizeof(S)));
    legacy_sync();
}

template <class S>
DeviceIlu<S>::~DeviceIlu() {
    fnlh::dfree(vals);
    fnlh::dfree(diag_lu);
    fnlh::dfree(diag_piv);
    fnlh::dfree(diag_inv);
}

template <class S>
std::size_t DeviceIlu<S>::bytes() const {
    const std::size_t bb = (std::size_t)p->b * p->b;
    const std::size_t dr = (std::size_t)p->n_dslices * 32;
    return ((std::size_t)p->sell_elems + dr * bb + (std::size_t)p->rows * bb) * sizeof(S) + dr * p->b * sizeof(int);
}

template <class S>
void DeviceIlu<S>::download(S* vals_out, S* diag_lu_out, int* diag_piv_out, S* diag_inv_out) const {
    const int b = p->b, bb = b * b;
    const std::size_t dr = (std::size_t)p->n_dslices * 32;
    FNLH_CUDA(cudaDeviceSynchronize());
    if (vals_out) {
        std::vector<S> h(std::max<std::size_t>(p->sell_elems, 1));
        FNLH_CUDA(cudaMemcpy(h.data(), vals, h.size() * sizeof(S), cudaMemcpyDeviceToHost));
        for (int e = 0; e < p->nnzb; ++e)
            for (int k = 0; k < bb; ++k) vals_out[(std::size_t)e * bb + k] = h[p->h_ent[e] + (long long)k * 32];
    }
    auto off = [&](int i, int w) { return (long long)(p->h_dpos[i] >> 5) * w * 32 + (p->h_dpos[i] & 31); };
    if (diag_lu_out) {
        std::vector<S> h(std::max<std::size_t>(dr * bb, 1));
        FNLH_CUDA(cudaMemcpy(h.data(), diag_lu, h.size() * sizeof(S), cudaMemcpyDeviceToHost));
        for (int i = 0; i < p->rows; ++i)
            for (int k = 0; k < bb; ++k) diag_lu_out[(std::size_t)i * bb + k] = h[off(i, bb) + (long long)k * 32];
    }
    if (diag_piv_out) {
        std::vector<int> h(std::max<std::size_t>(dr * b, 1));
        FNLH_CUDA(cudaMemcpy(h.data(), diag_piv, h.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int i = 0; i < p->rows; ++i)
            for (int k = 0; k < b; ++k) diag_piv_out[(std::size_t)i * b + k] = h[off(i, b) + (long long)k * 32];
    }
    if (diag_inv_out)
        FNLH_CUDA(cudaMemcpy(diag_inv_out, diag_inv, (std::size_t)p->rows * bb * sizeof(S), cudaMemcpyDeviceToHost));
}

Workspace::Workspace(std::size_t max_len) : vec_len(max_len) {
    FNLH_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    n_partials = 32768;  // >= kMvBlocks * kMaxLanes + 2 kMaxLanes + 16
    FNLH_CUDA_ALLOC(&partials, n_partials * sizeof(double));
    FNLH_CUDA_ALLOC(&scalars, 64 * sizeof(double));
    FNLH_CUDA(cudaMallocHost(&h_scalars, 64 * sizeof(double)));
    FNLH_CUDA_ALLOC(&status, 8 * sizeof(int));
    FNLH_CUDA(cudaMallocHost(&h_status, 8 * sizeof(int)));
    FNLH_CUDA(cudaMallocHost(&h_flags, 2 * kMaxLanes * sizeof(int)));
    for (auto& e : flag_ev) FNLH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& v : vec) FNLH_CUDA_ALLOC(&v, std::max<std::size_t>(max_len, 1) * sizeof(cplx));
}

Workspace::~Workspace() {
    for (auto& v : vec) fnlh::dfree(v);
    fnlh::dfree(partials);
    fnlh::dfree(scalars);
    cudaFreeHost(h_scalars);
    fnlh::dfree(status);
    cudaFreeHost(h_status);
    cudaFreeHost(h_flags);
    for (auto& e : flag_ev)
        if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
}

// ---------------------------------------------------------------------------
// operations
// ---------------------------------------------------------------------------
__global__ void k_status_reset(int* status) {
    status[0] = 0;
    status[1] = 0x7fffffff;
}

template <class S>
void ilu_factorize_async(const SystemView<S>& A, DeviceIlu<S>& f, int* status, cudaStream_t st) {
    const DevicePattern& p = *f.p;
    const PatDev pd = dev(p);
    { ::fnlh::note_launch(); k_status_reset<<<1, 1, 0, st>>>(status); }
    FNLH_DISPATCH_B(p.b, {
        const long long npos = p.sell_elems / (B * B);
        { ::fnlh::note_launch(); k_ilu_copy<B, S><<<nblocks(npos), kThreads, 0, st>>>(pd, A, f.vals, npos); }
        for (int l = 0; l < p.fwd_levels(); ++l) {
            const int n = p.fwd_ptr[l + 1] - p.fwd_ptr[l];
            { ::fnlh::note_launch(); k_ilu_factor<B, S><<<nblocks(n), kThreads, 0, st>>>(pd, p.fwd_rows + p.fwd_ptr[l], n, f.vals,
                                                                       f.diag_lu, f.diag_piv, f.diag_inv, status); }
        }
    });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void ilu_factorize(const SystemView<S>& A, DeviceIlu<S>& f, Workspace& ws) {
    ilu_factorize_async<S>(A, f, ws.status, ws.stream);
    FNLH_CUDA(cudaMemcpyAsync(ws.h_status, ws.status, 2 * sizeof(int), cudaMemcpyDeviceToHost, ws.stream));
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    if (ws.h_status[1] != 0x7fffffff)
        throw FactorizationError("near-singular ILU pivot block", ws.h_status[1]);
}

template <class S>
void ilu_apply(const DeviceIlu<S>& f, const S* rhs, S* x, Workspace& ws, S* x_accum) {
    const DevicePattern& p = *f.p;
    const PatDev pd = dev(p);
    FNLH_DISPATCH_B(p.b, {
        for (int l = 0; l < p.fwd_levels(); ++l) {
            const int n = p.fwd_ptr[l + 1] - p.fwd_ptr[l];
            { ::fnlh::note_launch(); k_ilu_fwd<B, S><<<nblocks(n), kThreads, 0, ws.stream>>>(pd, p.fwd_rows + p.fwd_ptr[l], n, f.vals, rhs, x); }
        }
        for (int l = 0; l < p.bwd_levels(); ++l) {
            const int n = p.bwd_ptr[l + 1] - p.bwd_ptr[l];
            { ::fnlh::note_launch(); k_ilu_bwd<B, S><<<nblocks(n), kThreads, 0, ws.stream>>>(pd, p.bwd_rows + p.bwd_ptr[l], n, f.vals,
                                                                    f.diag_lu, f.diag_piv, x, x_accum); }
        }
    });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void residual_norm(const SystemView<S>& A, const S* rhs, const S* x, S* r, double* d_norm2, Workspace& ws) {
    const DevicePattern& p = *A.p;
    const int grid = std::min(nblocks(p.rows), kMvBlocks);
    FNLH_DISPATCH_B(p.b, {
        { ::fnlh::note_launch(); k_matvec<B, S><<<grid, kThreads, 0, ws.stream>>>(dev(p), A, x, rhs, r, ws.partials); }
    });
    { ::fnlh::note_launch(); k_finish<<<1, 256, 0, ws.stream>>>(ws.partials, grid, d_norm2); }
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void matvec(const SystemView<S>& A, const S* x, S* y, Workspace& ws) {
    const DevicePattern& p = *A.p;
    const int grid = std::min(nblocks(p.rows), kMvBlocks);
    FNLH_DISPATCH_B(p.b, {
        { ::fnlh::note_launch(); k_matvec<B, S><<<grid, kThreads, 0, ws.stream>>>(dev(p), A, x, nullptr, y, nullptr); }
    });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void norm2_sq_on(const S* x, std::size_t len, double* d_out, double* partials, cudaStream_t st) {
    const int grid = std::min<long long>(nblocks((long long)len), kRedBlocks);
    { ::fnlh::note_launch(); k_sumsq<S><<<grid, kThreads, 0, st>>>(x, len, partials); }
    { ::fnlh::note_launch(); k_finish<<<1, 256, 0, st>>>(partials, grid, d_out); }
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void norm2_sq(const S* x, std::size_t len, double* d_out, Workspace& ws) {
    const int grid = std::min<long long>(nblocks((long long)len), kRedBlocks);
    { ::fnlh::note_launch(); k_sumsq<S><<<grid, kThreads, 0, ws.stream>>>(x, len, ws.partials); }
    { ::fnlh::note_launch(); k_finish<<<1, 256, 0, ws.stream>>>(ws.partials, grid, d_out); }
    FNLH_CUDA(cudaGetLastError());
}

// smoothed_solve (sparse.hpp:295-331): x0 = 0, z = M^{-1} r, x += z, r = b - A x, ||r||
template <class S>
LinearSolveReport smoothed_solve(const SystemView<S>& A, const S* rhs, const DeviceIlu<S>& f, double tol_rel,
                                 int max_iter, S* x, Workspace& ws) {
    if (!(tol_rel > 0.0 && tol_rel < 1.0)) throw ConfigError("smoothed_solve: tol_rel must be in (0,1)");
    if (max_iter < 1) throw ConfigError("smoothed_solve: max_iter must be >= 1");
    const DevicePattern& p = *A.p;
    const std::size_t len = (std::size_t)p.rows * p.b;
    S* r = static_cast<S*>(ws.vec[0]);
    S* z = static_cast<S*>(ws.vec[1]);
    if (!A.vals) {  // real A (+ per-node shift): the lane kernels with one lane, stopping rule on the device
        const LaneSystem<S> sys{&f, A.shift_im, rhs, x, z, r};
        LaneReport lr;
        smoothed_solve_batch<S>(p, A.real_vals, &sys, 1, tol_rel, max_iter, &lr, ws, A.real_sell);
        if (lr.diverged) throw DivergenceError("non-finite iterate in smoothed_solve", lr.rep.iterations, "linear");
        return lr.rep;
    }
    FNLH_CUDA(cudaMemsetAsync(x, 0, len * sizeof(S), ws.stream));
    LinearSolveReport rep;
    norm2_sq(rhs, len, ws.scalars, ws);
    FNLH_CUDA(cudaMemcpyAsync(ws.h_scalars, ws.scalars, sizeof(double), cudaMemcpyDeviceToHost, ws.stream));
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    rep.initial_residual = std::sqrt(ws.h_scalars[0]);
    rep.final_residual = rep.initial_residual;
    if (rep.initial_residual == 0.0) {
        rep.converged = 1;
        return rep;
    }
    const double target = tol_rel * rep.initial_residual;
    FNLH_CUDA(cudaMemcpyAsync(r, rhs, len * sizeof(S), cudaMemcpyDeviceToDevice, ws.stream));
    for (int it = 1; it <= max_iter; ++it) {
        ilu_apply(f, r, z, ws, x);  // z = M^{-1} r; x += z fused into the backward sweep
        residual_norm(A, rhs, x, r, ws.scalars + 1, ws);
        FNLH_CUDA(cudaMemcpyAsync(ws.h_scalars + 1, ws.scalars + 1, sizeof(double), cudaMemcpyDeviceToHost,
                                  ws.stream));
        FNLH_CUDA(cudaStreamSynchronize(ws.stream));
        rep.iterations = it;
        rep.final_residual = std::sqrt(ws.h_scalars[1]);
        if (!std::isfinite(rep.final_residual)) throw DivergenceError("non-finite iterate in smoothed_solve", it, "linear");
        if (rep.final_residual <= target) {
            rep.converged = 1;
            break;
        }
    }
    return rep;
}

// smoothed_solve (sparse.hpp:295-331) on P systems at once: the level kernels and the
// residual matvec serve every still-iterating lane in one launch; the stopping rule is
// taken per lane on the device after each sweep (k_lane_stop), one host synchronization
// per solve
template <class S>
void smoothed_solve_batch(const DevicePattern& p, const double* A_real, const LaneSystem<S>* sys, int P,
                          double tol_rel, int max_iter, LaneReport* reps, Workspace& ws, const double* A_sell) {
    if (!(tol_rel > 0.0 && tol_rel < 1.0)) throw ConfigError("smoothed_solve: tol_rel must be in (0,1)");
    if (max_iter < 1) throw ConfigError("smoothed_solve: max_iter must be >= 1");
    if (P < 1 || P > kMaxLanes) throw ConfigError("smoothed_solve_batch: 1 <= P <= kMaxLanes");
    const std::size_t len = (std::size_t)p.rows * p.b;
    const PatDev pd = dev(p);
    const int grid = std::min(nblocks(p.rows), kMvBlocks);
    // partials layout: [lanes' matvec partials grid*P][active][norms][control blocks][norm scratch 592]
    const std::size_t scratch = (std::size_t)grid * P + 10 * kMaxLanes + 16;
    if ((std::size_t)ws.n_partials < scratch + kRedBlocks)
        throw ConfigError("smoothed_solve_batch: workspace too small");
    LaLanes<S> T{};
    T.P = P;
    int* d_active = reinterpret_cast<int*>(ws.partials + (std::size_t)grid * P);
    double* d_norm = ws.partials + (std::size_t)grid * P + kMaxLanes;
    double* d_ctl = d_norm + kMaxLanes;
    T.active = d_active;
    for (int m = 0; m < P; ++m) {
        T.vals[m] = sys[m].f->vals;
        T.diag_lu[m] = sys[m].f->diag_lu;
        T.diag_piv[m] = sys[m].f->diag_piv;
        T.shift[m] = sys[m].shift;
        T.rhs[m] = sys[m].rhs;
        T.x[m] = sys[m].x;
        T.z[m] = sys[m].z;
        T.r[m] = sys[m].r;
        T.parts[m] = ws.partials + (std::size_t)grid * m;
        FNLH_CUDA(cudaMemsetAsync(sys[m].x, 0, len * sizeof(S), ws.stream));
        norm2_sq_on(sys[m].rhs, len, d_norm + m, ws.partials + scratch, ws.stream);
        FNLH_CUDA(cudaMemcpyAsync(sys[m].r, sys[m].rhs, len * sizeof(S), cudaMemcpyDeviceToDevice, ws.stream));
    }
    { ::fnlh::note_launch(); k_lane_init<<<1, 32, 0, ws.stream>>>(P, d_norm, tol_rel, d_active, d_ctl); }
    LaLanes<cplx> Tc{};
    LaLanes<double> Td{};
    if constexpr (sizeof(S) == sizeof(cplx)) Tc = T; else Td = T;
    // every sweep is enqueued; a lane whose stopping rule fired is skipped by the kernels
    // (active[lane] == 0), so the loop needs no host synchronization
    for (int it = 1; it <= max_iter; ++it) {
        FNLH_DISPATCH_B(p.b, {
            for (int l = 0; l < p.fwd_levels(); ++l) {
                const int n = p.fwd_ptr[l + 1] - p.fwd_ptr[l];
                { ::fnlh::note_launch(); k_ilu_fwd_b<B, S><<<nblocks(n) * P, kThreads, 0, ws.stream>>>(pd, p.fwd_rows + p.fwd_ptr[l], n, T); }
            }
            for (int l = 0; l < p.bwd_levels(); ++l) {
                const int n = p.bwd_ptr[l + 1] - p.bwd_ptr[l];
                { ::fnlh::note_launch(); k_ilu_bwd_b<B, S><<<nblocks(n) * P, kThreads, 0, ws.stream>>>(pd, p.bwd_rows + p.bwd_ptr[l], n, T); }
            }
            if (A_sell && sizeof(S) == sizeof(cplx)) {
                const int ng = (P + kLG - 1) / kLG, lg = (P + ng - 1) / ng;
                { ::fnlh::note_launch(); k_matvec_lg<B, S><<<grid * ng, kThreads, 0, ws.stream>>>(pd, A_sell, lg, T); }
            } else {
                { ::fnlh::note_launch(); k_matvec_b<B, S><<<grid * P, kThreads, 0, ws.stream>>>(pd, A_real, A_sell, T); }
            }
        });
        { ::fnlh::note_launch(); k_finish_b<<<P, 256, 0, ws.stream>>>(Tc, Td, sizeof(S) == sizeof(cplx) ? 1 : 0, grid, d_norm); }
        { ::fnlh::note_launch(); k_lane_stop<<<1, 32, 0, ws.stream>>>(P, it, d_norm, d_active, d_ctl); }
        FNLH_CUDA(cudaGetLastError());
        // non-blocking look-behind: once the flags of an earlier sweep have landed and every
        // lane had stopped, no further sweep is enqueued (a deep level schedule launches
        // 2 x levels kernels per sweep; the kernels of a stopped lane return at once anyway)
        const int slot = it & 1;
        FNLH_CUDA(cudaMemcpyAsync(ws.h_flags + slot * kMaxLanes, d_active, P * sizeof(int), cudaMemcpyDeviceToHost,
                                  ws.stream));
        FNLH_CUDA(cudaEventRecord(ws.flag_ev[slot], ws.stream));
        // a deep schedule (a natural-order chain: hundreds of tiny launches per sweep) waits
        // for this sweep's flags, a shallow one only looks at the previous sweep's
        const bool deep = p.fwd_levels() + p.bwd_levels() > 32;
        if (deep) FNLH_CUDA(cudaEventSynchronize(ws.flag_ev[slot]));
        const int seen = deep ? slot : slot ^ 1;
        if ((deep || it > 1) && cudaEventQuery(ws.flag_ev[seen]) == cudaSuccess) {
            const int* f = ws.h_flags + seen * kMaxLanes;
            bool any = false;
            for (int m = 0; m < P; ++m) any |= f[m] != 0;
            if (!any) break;
        }
    }
    FNLH_CUDA(cudaMemcpyAsync(ws.h_scalars, d_ctl, 8 * P * sizeof(double), cudaMemcpyDeviceToHost, ws.stream));
    FNLH_CUDA(cudaStreamSynchronize(ws.stream));
    for (int m = 0; m < P; ++m) {
        const double* c = ws.h_scalars + 8 * m;
        reps[m] = LaneReport{};
        reps[m].rep.initial_residual = c[0];
        reps[m].rep.final_residual = c[1];
        reps[m].rep.iterations = (int)c[3];
        reps[m].rep.converged = c[4] != 0.0 ? 1 : 0;
        reps[m].diverged = c[5] != 0.0 ? 1 : 0;
    }
}

void sell_from_bsr(const DevicePattern& p, const double* bsr, double* sell, cudaStream_t st) {
    const int bb = p.b * p.b;
    const long long npos = p.msell_doubles / (((bb + 1) / 2) * 2);
    { ::fnlh::note_launch(); k_sell_copy<<<nblocks(npos), kThreads, 0, st>>>(p.mblk_e, npos, bb, bsr, sell); }
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void block_diag_solve(int b, int n, const S* lu, const int* piv, const S* rhs, S* x, cudaStream_t st) {
    FNLH_DISPATCH_B(b, { { ::fnlh::note_launch(); k_block_diag_solve<B, S><<<nblocks(n), kThreads, 0, st>>>(n, lu, piv, rhs, x); } });
    FNLH_CUDA(cudaGetLastError());
}

template <class S>
void block_diag_factor(int b, int n, S* blocks, int* piv, int* status, cudaStream_t st) {
    FNLH_DISPATCH_B(b, { { ::fnlh::note_launch(); k_block_diag_factor<B, S><<<nblocks(n), kThreads, 0, st>>>(n, blocks, piv, status); } });
    FNLH_CUDA(cudaGetLastError());
}

#define FNLH_INST(S)                                                                                       \
    template struct DeviceIlu<S>;                                                                          \
    template void ilu_factorize<S>(const SystemView<S>&, DeviceIlu<S>&, Workspace&);                       \
    template void ilu_factorize_async<S>(const SystemView<S>&, DeviceIlu<S>&, int*, cudaStream_t);          \
    template void ilu_apply<S>(const DeviceIlu<S>&, const S*, S*, Workspace&, S*);                         \
    template void residual_norm<S>(const SystemView<S>&, const S*, const S*, S*, double*, Workspace&);     \
    template void matvec<S>(const SystemView<S>&, const S*, S*, Workspace&);                               \
    template void norm2_sq<S>(const S*, std::size_t, double*, Workspace&);                                 \
    template void norm2_sq_on<S>(const S*, std::size_t, double*, double*, cudaStream_t);                    \
    template LinearSolveReport smoothed_solve<S>(const SystemView<S>&, const S*, const DeviceIlu<S>&,      \
                                                 double, int, S*, Workspace&);                             \
    template void block_diag_solve<S>(int, int, const S*, const int*, const S*, S*, cudaStream_t);         \
    template void smoothed_solve_batch<S>(const DevicePattern&, const double*, const LaneSystem<S>*, int, double,  \
                                          int, LaneReport*, Workspace&, const double*);                                          \
    template void block_diag_factor<S>(int, int, S*, int*, int*, cudaStream_t);

FNLH_INST(double)
FNLH_INST(cplx)

}  // namespace fnlh
