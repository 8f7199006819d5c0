// pow(x, y) for the FP64 kernels, rounded like the host's libm.
//
// The reference's Blinn term is `d**reflectivity` (shading.py:73), which
// numba compiles to a call of the C library's pow — glibc's, which rounds to
// nearest in all but vanishingly rare cases.  CUDA's pow is accurate to 2
// ulp, so a frame rendered with it differs from the reference in the last
// bit of some radiance values (the reference's test_acceptance.py criterion
// 4 compares with `==`).  pow_cr evaluates y log(x) and its exponential in
// double-double arithmetic (relative error below ~2^-90 before the final
// rounding), so the rounded result is the correctly rounded pow except when
// the exact value lies within ~2^-90 of a rounding midpoint.
//
// Domain used by the kernels: x in [0, ~1] (a clamped cosine), y >= 0 finite;
// general positive finite x and finite y work too.  Plain C++ (no CUDA
// intrinsics) so that tests/test_pow.py compiles the same code with gcc and
// checks it against glibc's pow.  Callers compile with contraction off
// (-fmad=false / -ffp-contract=off): the error-free transformations below
// rely on every + and * rounding separately.
#pragma once
#include <math.h>

#ifdef __CUDACC__
#define RT_POW_HD __host__ __device__ __forceinline__
#else
#define RT_POW_HD static inline
#endif

namespace rtpow {

struct dd {
    double hi, lo;
};

RT_POW_HD dd fast_two_sum(double a, double b) {  // |a| >= |b|
    const double s = a + b;
    return dd{s, b - (s - a)};
}
RT_POW_HD dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return dd{s, (a - (s - bb)) + (b - bb)};
}
RT_POW_HD dd add(dd a, dd b) {  // accurate double-double sum (cancellation-safe)
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = fast_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return fast_two_sum(s.hi, s.lo);
}
RT_POW_HD dd mul(dd a, dd b) {
    const double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, fma(a.lo, b.hi, e));
    return fast_two_sum(p, e);
}
RT_POW_HD dd mul_d(dd a, double b) {
    const double p = a.hi * b;
    const double e = fma(a.lo, b, fma(a.hi, b, -p));
    return fast_two_sum(p, e);
}

// ln(x), x > 0 finite: x = 2^e m, m in [1/sqrt2, sqrt2), ln m = 2 atanh(f),
// f = (m - 1)/(m + 1) (|f| <= 0.1716): 2 f (1 + f^2/3 + f^4/5 + ...), the
// first five terms in double-double, the rest (< 2^-23 of the sum) in double
RT_POW_HD dd log_dd(double x) {
    int e;
    double m = frexp(x, &e);  // [0.5, 1)
    if (m < 0.70710678118654752440) {
        m *= 2.0;
        e -= 1;
    }
    const double num = m - 1.0;  // exact (Sterbenz)
    const dd den = two_sum(m, 1.0);
    const double fh = num / den.hi;
    double r = fma(-fh, den.hi, num);
    r = fma(-fh, den.lo, r);
    const dd f = fast_two_sum(fh, r / den.hi);
    const dd f2 = mul(f, f);
    const double z = f2.hi;
    // 1/11 + z/13 + ... + z^11/33 (truncation < 0.0295^16 / 35 relative)
    double tail = 1.0 / 33.0;
    tail = tail * z + 1.0 / 31.0;
    tail = tail * z + 1.0 / 29.0;
    tail = tail * z + 1.0 / 27.0;
    tail = tail * z + 1.0 / 25.0;
    tail = tail * z + 1.0 / 23.0;
    tail = tail * z + 1.0 / 21.0;
    tail = tail * z + 1.0 / 19.0;
    tail = tail * z + 1.0 / 17.0;
    tail = tail * z + 1.0 / 15.0;
    tail = tail * z + 1.0 / 13.0;
    tail = tail * z + 1.0 / 11.0;
    const dd c9{0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58};
    const dd c7{0x1.2492492492492p-3, 0x1.2492492492492p-57};
    const dd c5{0x1.999999999999ap-3, -0x1.999999999999ap-57};
    const dd c3{0x1.5555555555555p-2, 0x1.5555555555555p-56};
    dd s = add(c9, mul_d(f2, tail));
    s = add(c7, mul(f2, s));
    s = add(c5, mul(f2, s));
    s = add(c3, mul(f2, s));
    s = add(dd{1.0, 0.0}, mul(f2, s));
    dd lm = mul(f, s);
    lm.hi *= 2.0;
    lm.lo *= 2.0;
    const dd ln2{0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
    return add(mul_d(ln2, (double)e), lm);
}

// pow(x, y) = 2^k exp(r), r = y ln x - k ln2 (|r| <= ln2/2), exp(r) =
// (Taylor of exp(r / 512) to r^7 in double-double)^(2^9)
RT_POW_HD double pow_cr(double x, double y) {
    if (y == 0.0 || x == 1.0) return 1.0;
    if (x == 0.0) return y > 0.0 ? 0.0 : INFINITY;
    if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow(x, y);  // outside the kernels' domain
    const dd t = mul_d(log_dd(x), y);
    if (t.hi > 709.8) return INFINITY;
    if (t.hi < -746.0) return 0.0;
    const double k = rint(t.hi * 0x1.71547652b82fep+0);
    const dd ln2{0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
    dd r = add(t, mul_d(ln2, -k));
    r.hi *= 0x1p-9;
    r.lo *= 0x1p-9;
    // 1 + r + r^2/2! + ... + r^7/7!  (|r| < 7e-4: truncation < 2^-99)
    dd p = add(dd{1.0 / 5040.0, 0.0}, mul_d(r, 1.0 / 40320.0));
    p.lo += fma(-1.0 / 5040.0, 5040.0, 1.0) / 5040.0;  // 1/5040 to double-double
    p = add(dd{1.0 / 720.0, fma(-1.0 / 720.0, 720.0, 1.0) / 720.0}, mul(r, p));
    p = add(dd{1.0 / 120.0, fma(-1.0 / 120.0, 120.0, 1.0) / 120.0}, mul(r, p));
    p = add(dd{1.0 / 24.0, fma(-1.0 / 24.0, 24.0, 1.0) / 24.0}, mul(r, p));
    p = add(dd{1.0 / 6.0, fma(-1.0 / 6.0, 6.0, 1.0) / 6.0}, mul(r, p));
    p = add(dd{0.5, 0.0}, mul(r, p));
    p = add(dd{1.0, 0.0}, mul(r, p));
    p = add(dd{1.0, 0.0}, mul(r, p));
#pragma unroll 1
    for (int i = 0; i < 9; i++) p = mul(p, p);
    const int ki = (int)k;
    if (ki >= -1021) return ldexp(p.hi, ki);  // normal result: the scaling is exact
    // subnormal result: one rounding, at the scaled sum
    return ldexp(p.hi, ki) + ldexp(p.lo, ki);
}

}  // namespace rtpow
