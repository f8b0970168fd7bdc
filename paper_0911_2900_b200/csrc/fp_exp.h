// fp_exp.h -- bit-exact restatement of the `exp` the reference links (glibc 2.39, x86-64).
//
// The reference computes every planning weight with std::exp in fp64
// (/root/reference/proj/include/fastped/planning.hpp:102).  std::exp resolves to glibc 2.39's
// exp@@GLIBC_2.29, whose x86-64 ifunc picks the AVX2+FMA build of
// sysdeps/ieee754/dbl-64/e_exp.c (ARM optimized-routines algorithm, EXP_TABLE_BITS = 7,
// degree-5 polynomial) on every FMA-capable host.  glibc is a system dependency, not vendored
// under /root/reference; this file restates that published algorithm, with the fused
// multiply-adds exactly where that build places them (read from the shipped machine code),
// so that device weights are bitwise equal to the host's.  The 2^(i/128) table is derived from
// first principles by tools/gen_exp_table.py (and pinned against libm's copy there).
// tests/test_exp_restatement.py checks this restatement against libm on >10^7 arguments.
//
// Usable from host C/C++ (tests) and CUDA device code.
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define FPX_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define FPX_HD static inline
#endif

#if defined(__CUDACC__)
__device__ const uint64_t fpx_exp_tab[256] = {
#include "exp_table.inc"
};
#endif
#if defined(__CUDA_ARCH__)
#define FPX_TAB(i) __ldg(&fpx_exp_tab[(i)])
#else
static const uint64_t fpx_exp_tab_host[256] = {
#include "exp_table.inc"
};
#define FPX_TAB(i) fpx_exp_tab_host[(i)]
#endif

FPX_HD double fpx_asdouble(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}

FPX_HD uint64_t fpx_asuint64(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}

// IEEE operations with no contraction on either side.
#if defined(__CUDA_ARCH__)
#define FPX_FMA(a, b, c) __fma_rn((a), (b), (c))
#define FPX_MUL(a, b) __dmul_rn((a), (b))
#define FPX_ADD(a, b) __dadd_rn((a), (b))
#define FPX_SUB(a, b) __dsub_rn((a), (b))
#else
#define FPX_FMA(a, b, c) fma((a), (b), (c))
#define FPX_MUL(a, b) ((a) * (b))
#define FPX_ADD(a, b) ((a) + (b))
#define FPX_SUB(a, b) ((a) - (b))
#endif

// Constants of the algorithm (e_exp_data.c): N/ln2, 1.5*2^52, -ln2/N split, poly C2..C5.
#define FPX_INVLN2N 0x1.71547652b82fep7
#define FPX_SHIFT 0x1.8p52
#define FPX_NEGLN2HIN -0x1.62e42fefa0000p-8
#define FPX_NEGLN2LON -0x1.cf79abc9e3b3ap-47
#define FPX_C2 0x1.ffffffffffdbdp-2
#define FPX_C3 0x1.555555555543cp-3
#define FPX_C4 0x1.55555cf172b91p-5
#define FPX_C5 0x1.1111167a4d017p-7

// |x| in [512, 1024): the scale's exponent may over/underflow (e_exp.c specialcase()).
FPX_HD double fpx_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ULL) == 0) {
        sbits -= 1009ULL << 52;
        const double scale = fpx_asdouble(sbits);
        return FPX_MUL(FPX_FMA(scale, tmp, scale), 0x1p1009);
    }
    sbits += 1022ULL << 52;
    const double scale = fpx_asdouble(sbits);
    const double st = FPX_MUL(tmp, scale);
    double y = FPX_ADD(scale, st);
    if (1.0 > y) {
        const double hi = FPX_ADD(y, 1.0);
        double lo = FPX_ADD(FPX_SUB(scale, y), st);
        double t = FPX_ADD(FPX_ADD(FPX_SUB(1.0, hi), y), lo);
        y = FPX_SUB(FPX_ADD(t, hi), 1.0);
        if (y == 0.0) return 0.0;
    }
    return FPX_MUL(y, 0x1p-1022);
}

FPX_HD double fpx_exp(double x) {
    const uint64_t ix = fpx_asuint64(x);
    uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return FPX_ADD(x, 1.0);  // |x| < 2^-54
        if (abstop >= 0x409u) {                                      // |x| >= 1024
            if (ix == 0xfff0000000000000ULL) return 0.0;
            if (abstop >= 0x7ffu) return FPX_ADD(x, 1.0);
            return (ix >> 63) ? 0.0 : fpx_asdouble(0x7ff0000000000000ULL);
        }
        abstop = 0;  // 512 <= |x| < 1024
    }
    double kd = FPX_FMA(x, FPX_INVLN2N, FPX_SHIFT);
    const uint64_t ki = fpx_asuint64(kd);
    kd = FPX_SUB(kd, FPX_SHIFT);
    double r = FPX_FMA(kd, FPX_NEGLN2HIN, x);
    r = FPX_FMA(kd, FPX_NEGLN2LON, r);
    const uint64_t idx = 2 * (ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = fpx_asdouble(FPX_TAB(idx));
    const uint64_t sbits = FPX_TAB(idx + 1) + top;
    const double r2 = FPX_MUL(r, r);
    const double a = FPX_FMA(r, FPX_C3, FPX_C2);
    const double t0 = FPX_ADD(r, tail);
    const double p = FPX_FMA(r, FPX_C5, FPX_C4);
    const double b = FPX_FMA(a, r2, t0);
    const double r4 = FPX_MUL(r2, r2);
    const double tmp = FPX_FMA(r4, p, b);
    if (abstop == 0) return fpx_exp_specialcase(tmp, sbits, ki);
    const double scale = fpx_asdouble(sbits);
    return FPX_FMA(scale, tmp, scale);
}
