// libm_pow.cuh -- pow(x, y) rounded exactly as the host's glibc rounds it.
//
// The reference evaluates its subsonic inlet / outlet boundary states with the host
// libm's pow (disc_euler.cpp:179-180,187).  glibc's pow is not correctly rounded (about
// 0.1% of the boundary-state arguments differ from the correctly rounded value by one
// ULP), and the FD Jacobian / directional differences amplify a one-ULP boundary-flux
// difference by 1/delta ~ 1e5..1e6: over 20 pseudo-steps of the reference nozzle the
// correctly rounded pow alone moves the harmonic residual history by 3e-7.  Bitwise
// parity with the reference therefore needs glibc's own rounding.
//
// glibc >= 2.28 evaluates pow with the table-driven log / exp algorithm of Szabolcs Nagy
// (published with ARM's optimized-routines): log(x) = k ln2 + log(c) + log1p(z/c - 1) from
// a 128-entry table of (1/c, log c, tail) and a degree-8 polynomial, carried in
// double-double, then exp(y log x) = 2^(k/128) (1 + p(r)) from a 128-entry table of
// 2^(j/128).  On x86-64 hosts with FMA + AVX2 the ifunc selects the build compiled with
// -mfma, where the compiler contracted the algorithm's products into fused
// multiply-adds.  pow_libm below restates exactly that operation sequence (every fma and
// every separately rounded product / sum at the place the FMA build has it), so with the
// same tables it returns glibc's bits.  The tables are not copied: the host locates them
// at run time inside the libm the process (and the reference) links, and checks the
// restatement bitwise against ::pow on a fixed argument sample before the device uses it
// (libm_pow.cpp); when that check fails the device keeps the correctly rounded cr_pow.
//
// Only glibc's main path is restated (x positive and normal, 2^-65 <= |y| < 2^63,
// 2^-54 <= |y log x| < 256, plus the |y log x| < 2^-54 branch, which returns 1 + y log x);
// admissible boundary states never leave it, and other arguments fall back to cr_pow.
#pragma once

#include <stdint.h>

#include "cr_pow.cuh"

namespace fnlh {

// table image (doubles): [0, 9) log header: ln2hi, ln2lo, A[0..6]; [9, 9 + 512) log table
// {invc, pad, logc, logctail} x 128; [521, 529) exp header: invln2N, shift, negln2hiN,
// negln2loN, C2..C5; [529, 529 + 256) exp table {tail, sbits} x 128 (bit patterns)
constexpr int kPowLogHdr = 0, kPowLogTab = 9, kPowExpHdr = 9 + 512, kPowExpTab = 9 + 512 + 8;
constexpr int kPowTabDoubles = 9 + 512 + 8 + 256;

__host__ __device__ __forceinline__ uint64_t pw_bits(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    __builtin_memcpy(&u, &x, 8);
    return u;
#endif
}
__host__ __device__ __forceinline__ double pw_dbl(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    __builtin_memcpy(&x, &u, 8);
    return x;
#endif
}
// separately rounded operations (the device file is compiled --fmad=false as well)
__host__ __device__ __forceinline__ double pw_mul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ __forceinline__ double pw_add(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ __forceinline__ double pw_sub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
__host__ __device__ __forceinline__ double pw_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return __builtin_fma(a, b, c);
#endif
}

// returns false (and leaves *out untouched) outside the restated path
__host__ __device__ __forceinline__ bool pow_libm_main(const double* __restrict__ T, double x, double y, double* out) {
    const uint64_t ix = pw_bits(x), iy = pw_bits(y);
    if ((unsigned)((ix >> 52) - 1) > 0x7fdu) return false;              // x <= 0, subnormal, inf, nan
    if ((unsigned)(((iy >> 52) & 0x7ff) - 0x3be) > 0x7fu) return false; // |y| tiny or huge
    // log_inline: x = 2^k z, z in [OFF, 2 OFF), OFF = 0x3fe6955500000000
    const uint64_t tmp = ix - 0x3fe6955500000000ull;
    const int i = (int)((tmp >> 45) & 127);
    const int k = (int)((int64_t)tmp >> 52);
    const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
    const double z = pw_dbl(iz), kd = (double)k;
    const double* L = T + kPowLogHdr;
    const double* e = T + kPowLogTab + 4 * i;
    const double invc = e[0], logc = e[2], logctail = e[3];
    const double t1 = pw_fma(kd, L[0], logc);
    const double lo1 = pw_fma(kd, L[1], logctail);
    const double r = pw_fma(z, invc, -1.0);
    const double ar = pw_mul(r, L[2]);
    const double q12 = pw_fma(r, L[4], L[3]);
    const double q34 = pw_fma(r, L[6], L[5]);
    const double t2 = pw_add(r, t1);
    const double lo2 = pw_add(pw_sub(t1, t2), r);
    const double ar2 = pw_mul(r, ar);
    const double ar3 = pw_mul(r, ar2);
    const double lo3 = pw_fma(ar, r, -ar2);
    const double hi = pw_add(t2, ar2);
    const double q56 = pw_fma(r, L[8], L[7]);
    const double lo4 = pw_add(pw_sub(t2, hi), ar2);
    double q = pw_fma(q56, ar2, q34);
    q = pw_fma(ar2, q, q12);
    double lo = pw_add(pw_add(pw_add(lo1, lo2), lo3), lo4);
    lo = pw_fma(ar3, q, lo);
    const double ly = pw_add(hi, lo);
    const double ltail = pw_add(pw_sub(hi, ly), lo);
    // y log x in double-double
    const double ehi = pw_mul(y, ly);
    double elo = pw_fma(ly, y, -ehi);
    elo = pw_fma(y, ltail, elo);
    // exp_inline(ehi, elo, sign_bias = 0)
    const unsigned abstop = (unsigned)((pw_bits(ehi) >> 52) & 0x7ff);
    if ((int)abstop - 0x3c9 < 0) {  // |y log x| < 2^-54: 1 + y log x
        *out = pw_add(ehi, 1.0);
        return true;
    }
    if (abstop - 0x3c9u > 0x3eu) return false;  // |y log x| >= 256: over/underflow branches
    const double* X = T + kPowExpHdr;
    const uint64_t* ET = reinterpret_cast<const uint64_t*>(T + kPowExpTab);
    double kz = pw_fma(ehi, X[0], X[1]);
    const uint64_t ki = pw_bits(kz);
    kz = pw_sub(kz, X[1]);
    double rr = pw_fma(kz, X[2], ehi);
    rr = pw_fma(kz, X[3], rr);
    const uint64_t idx = 2 * (ki & 127);
    const uint64_t sbits = ET[idx + 1] + (ki << 45);
    rr = pw_add(elo, rr);
    const double p23 = pw_fma(rr, X[5], X[4]);
    const double t = pw_add(rr, pw_dbl(ET[idx]));
    const double r2 = pw_mul(rr, rr);
    const double p45 = pw_fma(rr, X[7], X[6]);
    double tm = pw_fma(p23, r2, t);
    const double r4 = pw_mul(r2, r2);
    tm = pw_fma(p45, r4, tm);
    const double scale = pw_dbl(sbits);
    *out = pw_fma(tm, scale, scale);
    return true;
}

// host: the validated table image of the loaded libm (libm_pow_host.cu), or nullptr
const double* libm_pow_tables();

// the boundary-state pow: glibc's bits when the tables are present, else correctly rounded
__host__ __device__ __forceinline__ double bc_pow(const double* __restrict__ T, double x, double y) {
    double r;
    if (T && pow_libm_main(T, x, y, &r)) return r;
    return cr_pow(x, y);
}

}  // namespace fnlh
