// Host check of csrc/exact_trig.h against the host libm (glibc: the reference's libm).
// usage: exact_trig_check <n> <seed>; prints
//   "sincos <n> <mismatch_sin> <mismatch_cos>"          sincos_rn vs sin/cos at x = 2pi * c (c float in [0,1])
//   "sincos_any <n> <mismatch_sin> <mismatch_cos>"      sincos_rn vs sin/cos, x uniform in [-pi, 2pi]
//   "atan2 <n> <mismatch>"                              atan2_rn(y, x, a0 +- 2 ulp) vs atan2(y, x)
//   "window <n> <unstable>"                             narrowings the +-2^-50 window flags
//   "example <kind> <x or y> <x> <glibc> <ours>"        the first few mismatches (hex)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "exact_trig.h"

using namespace prx;

static uint64_t bits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 rng(argc > 2 ? std::atol(argv[2]) : 1);
    std::uniform_real_distribution<float> uf(0.0f, 1.0f);
    std::uniform_real_distribution<double> ud(-M_PI, 2 * M_PI);
    std::normal_distribution<float> nf(0.0f, 1.0f);
    const double kTwoPi = 6.283185307179586476925286766559;
    int examples = 0;
    long ms = 0, mc = 0;
    for (long i = 0; i < n; ++i) {
        const double x = kTwoPi * (double)uf(rng);
        double s, c;
        xt::sincos_rn(x, s, c);
        if (bits(s) != bits(std::sin(x))) {
            ++ms;
            if (examples++ < 24) std::printf("example sin %a 0 %a %a\n", x, std::sin(x), s);
        }
        if (bits(c) != bits(std::cos(x))) {
            ++mc;
            if (examples++ < 24) std::printf("example cos %a 0 %a %a\n", x, std::cos(x), c);
        }
    }
    std::printf("sincos %ld %ld %ld\n", n, ms, mc);
    ms = mc = 0;
    for (long i = 0; i < n; ++i) {
        const double x = ud(rng);
        double s, c;
        xt::sincos_rn(x, s, c);
        if (bits(s) != bits(std::sin(x))) {
            ++ms;
            if (examples++ < 24) std::printf("example sin %a 0 %a %a\n", x, std::sin(x), s);
        }
        if (bits(c) != bits(std::cos(x))) {
            ++mc;
            if (examples++ < 24) std::printf("example cos %a 0 %a %a\n", x, std::cos(x), c);
        }
    }
    std::printf("sincos_any %ld %ld %ld\n", n, ms, mc);
    long ma = 0, unstable = 0;
    for (long i = 0; i < n; ++i) {
        // the canonical_of inputs: dot products of float vectors, widened to double
        const double y = (double)nf(rng), x = (double)nf(rng);
        const double g = std::atan2(y, x);
        const int d = (int)(i % 5) - 2;  // a0 = glibc's value moved by -2..2 ulp
        double a0 = g;
        for (int k = 0; k < std::abs(d); ++k) a0 = std::nextafter(a0, d > 0 ? 10.0 : -10.0);
        const double a = xt::atan2_rn(y, x, a0);
        if (bits(a) != bits(g)) {
            ++ma;
            if (examples++ < 24) std::printf("example atan2 %a %a %a %a\n", y, x, g, a);
        }
        const double v = g / kTwoPi;
        if ((float)xt::win_lo(v) != (float)xt::win_hi(v)) ++unstable;
    }
    std::printf("atan2 %ld %ld\n", n, ma);
    std::printf("window %ld %ld\n", n, unstable);
    return 0;
}
