// exact_trig.h -- the double sin / cos / atan2 of the light parametrisation
// (light.cpp:40-47 dir_from_angles, :70-117 warp_canonical, :119-175 canonical_of) with the
// reference's float results.
//
// The reference evaluates these in double with glibc and narrows the results (after a few
// exact-order double operations) to float.  CUDA's double sin/cos/atan2 are accurate to
// <= 2 ulp, glibc's to < 1 ulp, so the two double results can differ in their last bits;
// the float that the reference stores differs only when a float rounding boundary falls
// between them.  Every narrowing is therefore checked: the downstream double expression is
// evaluated at the CUDA value +- 2^-50 relative (>= 4 ulp, covering both libms' error
// bounds), and when both ends narrow to the same float -- monotone expressions -- the float
// is the reference's whatever glibc returned.  Otherwise (about one evaluation in 10^8) the
// transcendental is recomputed in double-double arithmetic (~100 bits) and rounded to the
// nearest double, i.e. the correctly rounded value, which is glibc's result except where
// glibc itself misrounds (its documented < 1 ulp bound; never observed in
// tests/test_exact_trig.py's sweeps).
//
// Host and device: the host build is what tests/test_exact_trig.py compares against glibc.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define PRX_XT __host__ __device__ __forceinline__
#define PRX_XT_COLD static __host__ __device__ __noinline__  // the rare exact path: out of line
#else
#define PRX_XT inline
#define PRX_XT_COLD static inline
#endif

namespace prx {
namespace xt {

struct DD {
    double hi, lo;
};

PRX_XT DD two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}
PRX_XT DD quick_two_sum(double a, double b) {  // |a| >= |b|
    const double s = a + b;
    return {s, b - (s - a)};
}
PRX_XT DD two_prod(double a, double b) {
    const double p = a * b;
#ifdef __CUDA_ARCH__
    return {p, __fma_rn(a, b, -p)};
#else
    return {p, std::fma(a, b, -p)};
#endif
}
PRX_XT DD add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    DD t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
PRX_XT DD neg(DD a) { return {-a.hi, -a.lo}; }
PRX_XT DD sub(DD a, DD b) { return add(a, neg(b)); }
PRX_XT DD mul(DD a, DD b) {
    DD p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}
PRX_XT DD mul_d(DD a, double b) {
    DD p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return quick_two_sum(p.hi, p.lo);
}
PRX_XT DD div(DD a, DD b) {  // long division, two correction steps
    const double q1 = a.hi / b.hi;
    DD r = sub(a, mul_d(b, q1));
    const double q2 = r.hi / b.hi;
    r = sub(r, mul_d(b, q2));
    const double q3 = r.hi / b.hi;
    return add(quick_two_sum(q1, q2), DD{q3, 0.0});
}
PRX_XT DD div_d(DD a, double b) { return div(a, DD{b, 0.0}); }

// pi/2 to 161 bits as three doubles (0x3FF921FB54442D18, 0x3C91A62633145C07, 0xB91F1976B7ED8FBC)
constexpr double kPio2_1 = 1.5707963267948966192e+00;
constexpr double kPio2_2 = 6.1232339957367660359e-17;
constexpr double kPio2_3 = -1.4973849048591698329e-33;

// sin and cos of r (|r| <= pi/4 + small) by their Taylor series in double-double
PRX_XT void sincos_kernel(DD r, DD& s, DD& c) {
    const DD r2 = mul(r, r);
    DD term = r;  // r^(2k+1) / (2k+1)!
    s = r;
    for (int k = 1; k <= 14; ++k) {
        term = div_d(mul(term, r2), (double)((2 * k) * (2 * k + 1)));
        s = (k & 1) ? sub(s, term) : add(s, term);
    }
    term = DD{1.0, 0.0};  // r^(2k) / (2k)!
    c = DD{1.0, 0.0};
    for (int k = 1; k <= 14; ++k) {
        term = div_d(mul(term, r2), (double)((2 * k - 1) * (2 * k)));
        c = (k & 1) ? sub(c, term) : add(c, term);
    }
}

// sin(x), cos(x) rounded to the nearest double, for |x| <= 2^20 (the light parametrisation
// only evaluates angles in [-pi, 2 pi]).  Cody-Waite reduction by k * pi/2 in triple precision.
PRX_XT_COLD void sincos_rn(double x, double& sn, double& cs) {
    const double k = std::nearbyint(x * 0.63661977236758134308);  // 2 / pi
    const DD p1 = two_prod(k, kPio2_1);  // k * pi/2 to ~160 bits, the products exact
    const DD p2 = two_prod(k, kPio2_2);
    DD r = sub(sub(DD{x, 0.0}, p1), p2);
    r = sub(r, DD{k * kPio2_3, 0.0});
    DD s, c;
    sincos_kernel(r, s, c);
    const int q = (int)(((long long)k) & 3);
    DD so, co;
    switch (q) {
        case 0: so = s; co = c; break;
        case 1: so = c; co = neg(s); break;
        case 2: so = neg(s); co = neg(c); break;
        default: so = neg(c); co = s; break;
    }
    so = quick_two_sum(so.hi, so.lo);
    co = quick_two_sum(co.hi, co.lo);
    sn = so.hi;
    cs = co.hi;
}

// atan2(y, x) rounded to the nearest double: one Newton step from a double estimate a0
// (any libm's, within a few ulp): a = a0 + atan(n / d), n = y cos a0 - x sin a0,
// d = x cos a0 + y sin a0, with atan(t) = t - t^3/3 for |t| <= 1e-15.
PRX_XT_COLD double atan2_rn(double y, double x, double a0) {
    if (y == 0.0 || x == 0.0 || !(std::fabs(a0) > 0.0)) return a0;  // exact special cases
    DD s, c;
    {
        // sin/cos of a0 in double-double (reduction as sincos_rn, without the final rounding)
        const double k = std::nearbyint(a0 * 0.63661977236758134308);
        const DD p1 = two_prod(k, kPio2_1);
        const DD p2 = two_prod(k, kPio2_2);
        DD r = sub(sub(DD{a0, 0.0}, p1), p2);
        r = sub(r, DD{k * kPio2_3, 0.0});
        DD ss, cc;
        sincos_kernel(r, ss, cc);
        const int q = (int)(((long long)k) & 3);
        switch (q) {
            case 0: s = ss; c = cc; break;
            case 1: s = cc; c = neg(ss); break;
            case 2: s = neg(ss); c = neg(cc); break;
            default: s = neg(cc); c = ss; break;
        }
    }
    const DD n = sub(mul_d(c, y), mul_d(s, x));
    const DD d = add(mul_d(c, x), mul_d(s, y));
    DD t = div(n, d);
    t = sub(t, div_d(mul(mul(t, t), t), 3.0));
    const DD a = add(DD{a0, 0.0}, t);
    return quick_two_sum(a.hi, a.lo).hi;
}

// [v - 2^-50 |v|, v + 2^-50 |v|] (>= +-4 ulp of v): the window the two libms' results share
PRX_XT double win_lo(double v) { return v - std::fabs(v) * 8.8817841970012523e-16 - 1e-300; }
PRX_XT double win_hi(double v) { return v + std::fabs(v) * 8.8817841970012523e-16 + 1e-300; }

// (float)(v * f) is the same for every v in the window (multiplication and narrowing are
// monotone, so the two ends decide)
PRX_XT bool product_narrows_stably(double v, double f) {
    return (float)(win_lo(v) * f) == (float)(win_hi(v) * f);
}

}  // namespace xt
}  // namespace prx
