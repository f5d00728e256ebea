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
    // fdiv_pos: positive divisors inside [2^-60, 2^60]; numerators over the
    // whole range including +-0, subnormals and the validity-boundary band
    long bad2 = 0, fallback = 0;
    for (long i = 0; i < n; ++i) {
        double d;
        switch (i % 5) {
        case 0: d = std::fabs(rnd_double(-60, 59)); break;
        case 1: {
            uint64_t b = ((uint64_t)(1023 + (int)(rnd() % 80) - 40) << 52) | ((1ull << 52) - 1);
            std::memcpy(&d, &b, 8);
            break;
        }
        case 2: d = (i & 8) ? 6.0 : 12.0; break;
        case 3: d = (double)(1 + rnd() % 20); break;
        default: d = std::ldexp(1.0, (int)(rnd() % 120) - 60); break;
        }
        double a;
        switch (i % 9) {
        case 0: a = (i & 16) ? -0.0 : 0.0; break;
        case 1: {  // subnormal
            uint64_t b = rnd() >> 12;
            if (rnd() & 1) b |= 1ull << 63;
            std::memcpy(&a, &b, 8);
            break;
        }
        case 2: a = rnd_double(-1022, 1023); break;
        case 3: a = rnd_double(-905, -895); break;  // around the 2^-900 bound
        case 4: a = rnd_double(935, 945); break;    // around the 2^939 bound
        default: a = rnd_double(-80, 80); break;
        }
        const double y = 1.0 / d;
        unsigned bd = 0u;
        (void)ign::fdiv_pos_try(a, d, y, bd);
        fallback += bd != 0u;
        const double q = ign::fdiv_pos(a, d, y), r = a / d;
        if (std::memcmp(&q, &r, 8) != 0 && !(std::isnan(q) && std::isnan(r))) {
            if (bad2 < 10) std::printf("a=%a d=%a fdiv_pos=%a ieee=%a\n", a, d, q, r);
            ++bad2;
        }
    }
    std::printf("fdiv_pos: %ld mismatches of %ld (%ld took the IEEE fallback)\n", bad2, n,
                fallback);
    return (bad || bad2) ? 1 : 0;
}
