/* Test helper: the restated exp (paper_0911_2900_b200/csrc/fp_exp.h) vs this host's libm exp. */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include "../../paper_0911_2900_b200/csrc/fp_exp.h"

double restated_exp(double x) { return fpx_exp(x); }

/* Compares on n arguments x_k = lo + (hi-lo)*u_k (splitmix-driven); returns mismatch count and
   writes the first mismatching argument to *first_bad. */
int64_t compare_range(double lo, double hi, int64_t n, uint64_t seed, double* first_bad) {
    int64_t bad = 0;
    uint64_t s = seed;
    for (int64_t k = 0; k < n; ++k) {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * 0x1.0p-53;
        const double x = lo + (hi - lo) * u;
        const double a = exp(x), b = fpx_exp(x);
        if (memcmp(&a, &b, 8) != 0) {
            if (bad == 0 && first_bad) *first_bad = x;
            ++bad;
        }
    }
    return bad;
}

/* Arguments of the hot path itself: k_s * (S_p - S_c) with S on the 1/sqrt2 lattice. */
int64_t compare_lattice(double k_s, int64_t n, uint64_t seed, double* first_bad) {
    int64_t bad = 0;
    uint64_t s = seed;
    const double r2 = sqrt(2.0);
    for (int64_t k = 0; k < n; ++k) {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        /* S values built by left-folded sums of 1 and sqrt2 like the Dijkstra field */
        double sp = 0.0, sc;
        int steps = (int)(z % 20000);
        uint64_t b = z;
        for (int i = 0; i < steps % 64; ++i) { sp += (b & 1) ? r2 : 1.0; b = (b >> 1) | (b << 63); }
        sp += (double)(steps / 64) * 64.0;
        sc = sp;
        int back = (int)((z >> 40) % 9);
        for (int i = 0; i < back; ++i) sc += ((z >> (20 + i)) & 1) ? r2 : 1.0;
        const double x = (k & 1) ? k_s * (sp - sc) : k_s * (sc - sp);
        const double a = exp(x), c = fpx_exp(x);
        if (memcmp(&a, &c, 8) != 0) {
            if (bad == 0 && first_bad) *first_bad = x;
            ++bad;
        }
    }
    return bad;
}
