// TEST INFRASTRUCTURE: stress check of ign::fdiv (Markstein division with a
// precomputed reciprocal, paper_2202_02319_b200/csrc/physics.cuh) against the
// IEEE quotient a/d, bitwise, on random operands spanning the whole exponent
// range plus adversarial divisors (all-ones significands, powers of two, the
// constants 6 and 12, small integers).  Exit status 1 on any mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "physics.cuh"

static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint64_t rnd() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
}
static double rnd_double(int emin, int emax) {
    const uint64_t mant = rnd() >> 12;
    const int e = emin + (int)(rnd() % (uint64_t)(emax - emin + 1));
    uint64_t bits = ((uint64_t)(e + 1023) << 52) | mant;
    if (rnd() & 1) bits |= 1ull << 63;
    double d;
    std::memcpy(&d, &bits, 8);
    return d;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 20000000;
    long bad = 0;
    for (long i = 0; i < n; ++i) {
        double d;
        switch (i % 6) {
        case 0: d = rnd_double(-60, 60); break;
        case 1: {  // all-ones significand
            uint64_t b = ((uint64_t)(1023 + (int)(rnd() % 80) - 40) << 52) | ((1ull << 52) - 1);
            std::memcpy(&d, &b, 8);
            break;
        }
        case 2: d = (i & 8) ? 6.0 : 12.0; break;
        case 3: d = (double)(1 + rnd() % 20); break;
        case 4: d = rnd_double(-1000, 1000); break;
        default: d = std::ldexp(1.0, (int)(rnd() % 200) - 100); break;
        }
        const double a = (i % 7 == 0) ? rnd_double(-1022, 1023) : rnd_double(-80, 80);
        const double y = 1.0 / d;
        const double q = ign::fdiv(a, d, y), r = a / d;
        if (std::memcmp(&q, &r, 8) != 0 && !(std::isnan(q) && std::isnan(r))) {
            if (bad < 10) std::printf("a=%a d=%a fdiv=%a ieee=%a\n", a, d, q, r);
            ++bad;
        }
    }
    std::printf("fdiv: %ld mismatches of %ld\n", bad, n);
    return bad ? 1 : 0;
}
