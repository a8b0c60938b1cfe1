// Check: for positive integer n and finite s in the normal range,
//   q1 = fma(fma(-q0, n, s), y, q0),  q0 = s*y,  y = 1/n (IEEE)
// equals the IEEE quotient s/n.  Exhaustive over integer s in [0, 255*n]
// for n <= NMAX (the uint8 domain), plus random and adversarial doubles.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static inline double q1f(double s, double n, double y) {
    double q0 = s * y;
    double r = fma(-q0, n, s);
    return fma(r, y, q0);
}
static uint64_t st = 88172645463325252ull;
static inline uint64_t xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
int main(int argc, char** argv) {
    int nmax = argc > 1 ? atoi(argv[1]) : 561;
    long long bad = 0, tested = 0;
    for (int n = 1; n <= nmax; ++n) {
        const double dn = n, y = 1.0 / dn;
        for (long long s = 0; s <= 255LL * n; ++s) {
            double q = q1f((double)s, dn, y);
            if (q != (double)s / dn) { if (bad < 10) printf("int bad s=%lld n=%d\n", s, n); ++bad; }
            ++tested;
        }
        for (int k = 0; k < 200000; ++k) {
            // random doubles across many binades, both signs
            uint64_t bits = (xr() & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(1023 - 60 + (xr() % 120)) << 52);
            double s = *(double*)&bits;
            if (xr() & 1) s = -s;
            double q = q1f(s, dn, y);
            if (q != s / dn) { if (bad < 10) printf("rnd bad s=%.17g n=%d\n", s, n); ++bad; }
            // adversarial: s = n * m for m near binade edges and m +- few ulps
            double m = ldexp(1.0, (int)(xr() % 40) - 20);
            for (int d = -3; d <= 3; ++d) {
                double mm = nextafter(m, d < 0 ? 0 : INFINITY);
                for (int e = 0; e < abs(d); ++e) mm = nextafter(mm, d < 0 ? 0 : INFINITY);
                double s2 = mm * dn;  // rounded product
                double s3 = nextafter(s2, INFINITY), s4 = nextafter(s2, 0);
                double ss[3] = {s2, s3, s4};
                for (int t = 0; t < 3; ++t) {
                    double q2 = q1f(ss[t], dn, y);
                    if (q2 != ss[t] / dn) { if (bad < 10) printf("adv bad s=%.17g n=%d\n", ss[t], n); ++bad; }
                    ++tested;
                }
            }
            tested += 1;
        }
    }
    printf("tested %lld, mismatches %lld\n", tested, bad);
    return bad != 0;
}
