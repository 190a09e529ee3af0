// common.cuh -- scalar traits, reference-exact complex arithmetic, register-resident
// b x b block kernels (dense.hpp:20-120) for sm_100a.
//
// Every parity-relevant translation unit is compiled with --fmad=false: the reference
// is built without FMA contraction (g++ -O2, no -march), so separately rounded
// multiplies and adds reproduce its arithmetic bit for bit.
#pragma once

#include <atomic>
#include <cuda_runtime.h>

#include <math.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace fnlh {

#define FNLH_CUDA(call)                                                                            \
    do {                                                                                           \
        cudaError_t err__ = (call);                                                                \
        if (err__ != cudaSuccess)                                                                  \
            throw ::fnlh::CudaError(std::string(#call) + ": " + cudaGetErrorString(err__));        \
    } while (0)

#define FNLH_CUDA_ALLOC(p, bytes) ::fnlh::dmalloc(p, bytes)

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Setup transfers and memsets go through the legacy default stream, which the library's
// non-blocking work streams do not wait for (and a pageable upload may return before its
// DMA lands).  Wait for it before any work stream can read the data: with several host
// threads driving distinct handles, another thread's legacy-stream traffic can otherwise
// delay it past the first kernels.
inline void legacy_sync() { FNLH_CUDA(cudaStreamSynchronize(cudaStreamLegacy)); }

// every device allocation of the library (guard.cpp): cudaMalloc / cudaFree, or guarded
// allocations in a -DFNLH_GUARD measurement build
void dmalloc(void** p, std::size_t bytes);
void dfree(void* p);
template <class T>
inline void dmalloc(T** p, std::size_t bytes) { dmalloc(reinterpret_cast<void**>(p), bytes); }

// count of kernel launches issued by this library (bench.py "gpu_launches"); atomic: the
// C ABI may be called concurrently from several host threads with distinct handles
std::atomic<long long>& launch_count();
inline thread_local long long tl_launches = 0;  // this host thread's launches (graph capture accounting)
inline void note_launch() {
    launch_count().fetch_add(1, std::memory_order_relaxed);
    ++tl_launches;
}

// std::complex<double> layout (re, im), reference arithmetic order.
struct alignas(16) cplx {
    double re, im;
};

__host__ __device__ __forceinline__ cplx mk(double r, double i) { return cplx{r, i}; }
__host__ __device__ __forceinline__ cplx operator+(cplx a, cplx b) { return mk(a.re + b.re, a.im + b.im); }
__host__ __device__ __forceinline__ cplx operator-(cplx a, cplx b) { return mk(a.re - b.re, a.im - b.im); }
__host__ __device__ __forceinline__ cplx operator-(cplx a) { return mk(-a.re, -a.im); }
// GCC's inline complex product (the __muldc3 slow path only fires on NaN results)
__host__ __device__ __forceinline__ cplx operator*(cplx a, cplx b) {
    return mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
// std::complex * real and real * std::complex are componentwise
__host__ __device__ __forceinline__ cplx operator*(cplx a, double s) { return mk(a.re * s, a.im * s); }
__host__ __device__ __forceinline__ cplx operator*(double s, cplx a) { return mk(a.re * s, a.im * s); }
// libgcc __divdc3, normal-range branch (Smith's method); pinned bitwise against the
// reference's std::complex division by tests/test_oracle_pin.py::test_smith_division_is_libgcc
__host__ __device__ __forceinline__ cplx operator/(cplx a, cplx b) {
    double x, y;
    if (fabs(b.re) < fabs(b.im)) {
        const double ratio = b.re / b.im;
        const double denom = (b.re * ratio) + b.im;
        x = ((a.re * ratio) + a.im) / denom;
        y = ((a.im * ratio) - a.re) / denom;
    } else {
        const double ratio = b.im / b.re;
        const double denom = (b.im * ratio) + b.re;
        x = ((a.im * ratio) + a.re) / denom;
        y = (a.im - (a.re * ratio)) / denom;
    }
    return mk(x, y);
}
__host__ __device__ __forceinline__ cplx& operator+=(cplx& a, cplx b) { return a = a + b; }
__host__ __device__ __forceinline__ cplx& operator-=(cplx& a, cplx b) { return a = a - b; }
__host__ __device__ __forceinline__ bool is_zero(cplx a) { return a.re == 0.0 && a.im == 0.0; }
__host__ __device__ __forceinline__ bool is_zero(double a) { return a == 0.0; }
__host__ __device__ __forceinline__ double mag(double a) { return fabs(a); }
__host__ __device__ __forceinline__ double mag(cplx a) { return hypot(a.re, a.im); }
__host__ __device__ __forceinline__ double sq(double a) { return a * a; }
__host__ __device__ __forceinline__ double sq(cplx a) { return a.re * a.re + a.im * a.im; }
__host__ __device__ __forceinline__ bool finite_(double a) { return isfinite(a); }
__host__ __device__ __forceinline__ bool finite_(cplx a) { return isfinite(a.re) && isfinite(a.im); }
template <class S>
__host__ __device__ __forceinline__ S zero();
template <>
__host__ __device__ __forceinline__ double zero<double>() { return 0.0; }
template <>
__host__ __device__ __forceinline__ cplx zero<cplx>() { return mk(0.0, 0.0); }
template <class S>
__host__ __device__ __forceinline__ S one();
template <>
__host__ __device__ __forceinline__ double one<double>() { return 1.0; }
template <>
__host__ __device__ __forceinline__ cplx one<cplx>() { return mk(1.0, 0.0); }
// complex(a) for real a: the value shift_diagonal writes (sparse.cpp:166)
template <class S>
__host__ __device__ __forceinline__ S from_real(double a);
template <>
__host__ __device__ __forceinline__ double from_real<double>(double a) { return a; }
template <>
__host__ __device__ __forceinline__ cplx from_real<cplx>(double a) { return mk(a, 0.0); }

// real-matrix x scalar-vector product: complex(a,0)*x equals (a*x.re, a*x.im) up to the sign of zero
__host__ __device__ __forceinline__ double rmul(double a, double x) { return a * x; }
__host__ __device__ __forceinline__ cplx rmul(double a, cplx x) { return mk(a * x.re, a * x.im); }

// ---------------------------------------------------------------------------
// register-resident b x b kernels, B a compile-time block size (dense.hpp)
// ---------------------------------------------------------------------------

// block_lu_factor (dense.hpp:57-88) on a row-major register block; returns 0 on success,
// 1 on an exactly singular pivot; cond = max|pivot| / min|pivot|.
template <int B, class S>
__device__ __forceinline__ int lu_factor_reg(S (&A)[B * B], int (&piv)[B], double& cond) {
    double pmax = 0.0, pmin = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
        int p = k;
        double best = mag(A[k * B + k]);
#pragma unroll
        for (int r = k + 1; r < B; ++r) {
            const double m = mag(A[r * B + k]);
            if (m > best) {
                best = m;
                p = r;
            }
        }
        piv[k] = p;
#pragma unroll
        for (int r = k + 1; r < B; ++r)
            if (r == p) {
#pragma unroll
                for (int c = 0; c < B; ++c) {
                    S t = A[k * B + c];
                    A[k * B + c] = A[r * B + c];
                    A[r * B + c] = t;
                }
            }
        const S pivot = A[k * B + k];
        const double pm = mag(pivot);
        if (pm == 0.0) return 1;
        pmax = (k == 0) ? pm : fmax(pmax, pm);
        pmin = (k == 0) ? pm : fmin(pmin, pm);
#pragma unroll
        for (int r = k + 1; r < B; ++r) {
            const S l = A[r * B + k] / pivot;
            A[r * B + k] = l;
#pragma unroll
            for (int c = k + 1; c < B; ++c) A[r * B + c] -= l * A[k * B + c];
        }
    }
    cond = pmin > 0.0 ? pmax / pmin : INFINITY;
    return 0;
}

// block_lu_solve (dense.hpp:91-109), in place on x
template <int B, class S>
__device__ __forceinline__ void lu_solve_reg(const S (&LU)[B * B], const int (&piv)[B], S (&x)[B]) {
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
        for (int c = 0; c < r; ++c) acc -= LU[r * B + c] * x[c];
        x[r] = acc;
    }
#pragma unroll
    for (int r = B - 1; r >= 0; --r) {
        S acc = x[r];
#pragma unroll
        for (int c = r + 1; c < B; ++c) acc -= LU[r * B + c] * x[c];
        x[r] = acc / LU[r * B + r];
    }
}

template <int B, class S>
__device__ __forceinline__ void load_block(const S* __restrict__ g, S (&A)[B * B]) {
#pragma unroll
    for (int k = 0; k < B * B; ++k) A[k] = g[k];
}
template <int B, class S>
__device__ __forceinline__ void store_block(S* __restrict__ g, const S (&A)[B * B]) {
#pragma unroll
    for (int k = 0; k < B * B; ++k) g[k] = A[k];
}
template <int B, class S>
__device__ __forceinline__ void load_vec(const S* __restrict__ g, S (&x)[B]) {
#pragma unroll
    for (int k = 0; k < B; ++k) x[k] = g[k];
}
template <int B, class S>
__device__ __forceinline__ void store_vec(S* __restrict__ g, const S (&x)[B]) {
#pragma unroll
    for (int k = 0; k < B; ++k) g[k] = x[k];
}

}  // namespace fnlh
