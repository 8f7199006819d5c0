// pow_cr (paper_2305_07450_b200/csrc/rt_pow.cuh) against the C library's pow
// on random arguments of the Blinn term's domain: prints
// "<trials> <mismatches> <max ulp>".  Built by tests/test_pow.py with
// g++ -O2 -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rt_pow.cuh"

static uint64_t state = 0x9E3779B97F4A7C15ull;
static double uniform() {  // splitmix64 -> [0, 1)
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1p-53;
}

static int64_t bits(double v) {
    int64_t b;
    memcpy(&b, &v, 8);
    return b;
}

int main(int argc, char **argv) {
    const long n = argc > 1 ? atol(argv[1]) : 1000000;
    long bad = 0;
    int64_t worst = 0;
    for (long i = 0; i < n; i++) {
        double x = uniform();
        if (i % 4 == 1) x = 1.0 - 1e-3 * uniform();        // highlights: d near 1
        if (i % 4 == 2) x = pow(10.0, -30.0 * uniform());  // far tails
        double y;
        switch (i % 3) {
            case 0: y = (double)(1 + (long)(256 * uniform())); break;  // integer shininess
            case 1: y = 300.0 * uniform(); break;
            default: y = 0.5 + 8.0 * uniform(); break;
        }
        const double got = rtpow::pow_cr(x, y), want = pow(x, y);
        if (bits(got) != bits(want)) {
            bad++;
            int64_t d = bits(got) - bits(want);
            if (d < 0) d = -d;
            if (d > worst) worst = d;
            if (bad <= 5) fprintf(stderr, "x=%a y=%a got %a want %a\n", x, y, got, want);
        }
    }
    // the kernels' special cases
    const double sp[][3] = {{0.0, 3.0, 0.0}, {0.0, 0.0, 1.0}, {1.0, 77.5, 1.0}, {0.5, 0.0, 1.0}, {0.25, 0.5, 0.5}};
    for (auto &c : sp)
        if (rtpow::pow_cr(c[0], c[1]) != c[2]) bad++, worst = worst > 1 ? worst : 1;
    printf("%ld %ld %lld\n", n, bad, (long long)worst);
    return 0;
}
