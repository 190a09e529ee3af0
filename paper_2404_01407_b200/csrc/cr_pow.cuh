// cr_pow.cuh -- correctly rounded pow(x, y) for x > 0 via double-double log / exp.
//
// The reference evaluates the subsonic inlet / outlet boundary states with glibc's
// pow (disc_euler.cpp:179-180,187); CUDA's pow differs from it in the last bit on a
// large fraction of arguments, and the FD Jacobian amplifies a 1-ULP difference in a
// boundary flux by 1/delta ~ 1e6.  The device therefore evaluates pow in ~106-bit
// arithmetic and rounds once (correctly rounded).  glibc's own pow misrounds about
// 0.1% of the arguments we sample (tests/test_cr_pow.py checks against 60-digit
// decimal arithmetic), so the oracle can run either libm: glibc (= the reference)
// or this routine (= the device), which separates the two parity questions.
#pragma once

#include <math.h>

namespace fnlh {

struct dd {
    double hi, lo;
};

__host__ __device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return dd{s, e};
}
__host__ __device__ __forceinline__ dd fast_two_sum(double a, double b) {
    const double s = a + b;
    return dd{s, b - (s - a)};
}
__host__ __device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = a * b;
    return dd{p, fma(a, b, -p)};
}
__host__ __device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = fast_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return fast_two_sum(s.hi, s.lo);
}
__host__ __device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return fast_two_sum(p.hi, p.lo);
}
__host__ __device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return fast_two_sum(p.hi, p.lo);
}
__host__ __device__ __forceinline__ dd dd_div(dd a, dd b) {
    const double q1 = a.hi / b.hi;
    dd r = dd_add(a, dd_mul_d(b, -q1));
    const double q2 = r.hi / b.hi;
    r = dd_add(r, dd_mul_d(b, -q2));
    const double q3 = r.hi / b.hi;
    dd q = fast_two_sum(q1, q2);
    return dd_add(q, dd{q3, 0.0});
}

// ln 2 to ~107 bits
constexpr double kLn2Hi = 6.93147180559945286227e-01;
constexpr double kLn2Lo = 2.31904681384629955842e-17;

// log(x), x > 0 finite, as double-double: x = 2^k m, m in [sqrt(1/2), sqrt(2));
// log m = 2 atanh(s), s = (m-1)/(m+1), series to s^45 (|s| < 0.1716)
__host__ __device__ inline dd dd_log(double x) {
    int k;
    double m = frexp(x, &k);  // m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m *= 2.0;
        k -= 1;
    }
    const dd num = two_sum(m, -1.0);
    const dd den = two_sum(m, 1.0);
    const dd s = dd_div(num, den);
    const dd s2 = dd_mul(s, s);
    // Horner in s2: sum_{j=0..22} s2^j / (2j+1)
    dd acc = dd_div(dd{1.0, 0.0}, dd{45.0, 0.0});
    for (int j = 21; j >= 0; --j) acc = dd_add(dd_mul(acc, s2), dd_div(dd{1.0, 0.0}, dd{2.0 * j + 1.0, 0.0}));
    dd lm = dd_mul(dd_mul_d(s, 2.0), acc);
    const dd kl = dd_add(two_prod((double)k, kLn2Hi), dd{(double)k * kLn2Lo, 0.0});
    return dd_add(kl, lm);
}

// exp(t) for a double-double t of moderate size; result rounded to double
__host__ __device__ inline double dd_exp_round(dd t) {
    const double jf = nearbyint(t.hi / kLn2Hi);
    // r = t - j ln2 (dd)
    dd r = dd_add(t, dd_add(two_prod(-jf, kLn2Hi), dd{-jf * kLn2Lo, 0.0}));
    // r / 2^10, Taylor to degree 12, then square 10 times
    r.hi = ldexp(r.hi, -10);
    r.lo = ldexp(r.lo, -10);
    dd term = {1.0, 0.0};
    dd sum = {1.0, 0.0};
    for (int i = 1; i <= 12; ++i) {
        term = dd_div(dd_mul(term, r), dd{(double)i, 0.0});
        sum = dd_add(sum, term);
    }
    for (int i = 0; i < 10; ++i) sum = dd_mul(sum, sum);
    const int j = (int)jf;
    return ldexp(sum.hi + sum.lo, j);
}

// correctly rounded x^y for x > 0 finite and moderate y (the boundary-state exponents)
__host__ __device__ inline double cr_pow(double x, double y) {
    if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow(x, y);
    if (y == 0.0 || x == 1.0) return 1.0;
    const dd l = dd_log(x);
    dd t = dd_mul_d(l, y);
    return dd_exp_round(t);
}

}  // namespace fnlh
