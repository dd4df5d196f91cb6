// fm_hypot.cuh -- bit-exact device restatement of the hypot() that numpy's
// np.hypot reaches on this image (glibc 2.39, x86-64 baseline build: the
// non-FMA branch of sysdeps/ieee754/dbl-64/e_hypot.c, Borges' corrected
// sqrt).  The reference's obstacle-transit test derives its sample count
// from ceil(hypot(dx, dy) / (dx_cell / 2)) (environment.py:354-356), so the
// GPU must round exactly like glibc: a correctly-rounded hypot differs from
// glibc in ~0.6% of inputs.  tests/test_hypot.py compiles this header for
// the host and compares it with libm on tens of millions of inputs.
//
// Every operation is an explicitly rounded IEEE op (no FMA contraction).
#pragma once

#if defined(__CUDACC__)
#define FMH_HD __host__ __device__ __forceinline__
#else
#define FMH_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define FMH_ADD(a, b) __dadd_rn((a), (b))
#define FMH_SUB(a, b) __dsub_rn((a), (b))
#define FMH_MUL(a, b) __dmul_rn((a), (b))
#define FMH_DIV(a, b) __ddiv_rn((a), (b))
#define FMH_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define FMH_ADD(a, b) ((a) + (b))
#define FMH_SUB(a, b) ((a) - (b))
#define FMH_MUL(a, b) ((a) * (b))
#define FMH_DIV(a, b) ((a) / (b))
#define FMH_SQRT(a) sqrt(a)
#endif

// Requires ax >= ay >= 0 with squares neither overflowing nor underflowing.
FMH_HD double fm_hypot_core(double ax, double ay)
{
    double h = FMH_SQRT(FMH_ADD(FMH_MUL(ax, ax), FMH_MUL(ay, ay)));
    double t1, t2;
    if (h <= FMH_MUL(2.0, ay)) {
        const double delta = FMH_SUB(h, ay);
        t1 = FMH_MUL(ax, FMH_SUB(FMH_MUL(2.0, delta), ax));
        t2 = FMH_MUL(FMH_SUB(delta, FMH_MUL(2.0, FMH_SUB(ax, ay))), delta);
    } else {
        const double delta = FMH_SUB(h, ax);
        t1 = FMH_MUL(FMH_MUL(2.0, delta), FMH_SUB(ax, FMH_MUL(2.0, ay)));
        t2 = FMH_ADD(FMH_MUL(FMH_SUB(FMH_MUL(4.0, delta), ay), ay), FMH_MUL(delta, delta));
    }
    return FMH_SUB(h, FMH_DIV(FMH_ADD(t1, t2), FMH_MUL(2.0, h)));
}

// Finite inputs only (the reference's segment endpoints are finite).
FMH_HD double fm_hypot(double x, double y)
{
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x;
    const double ay = x < y ? x : y;
    const double kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54, kScale = 0x1p-600;
    if (ax > kLarge) {
        if (ay <= FMH_MUL(ax, kEps)) return FMH_ADD(ax, ay);
        return FMH_DIV(fm_hypot_core(FMH_MUL(ax, kScale), FMH_MUL(ay, kScale)), kScale);
    }
    if (ay < kTiny) {
        if (ax >= FMH_DIV(ay, kEps)) return FMH_ADD(ax, ay);
        return FMH_MUL(fm_hypot_core(FMH_DIV(ax, kScale), FMH_DIV(ay, kScale)), kScale);
    }
    if (ay <= FMH_MUL(ax, kEps)) return FMH_ADD(ax, ay);
    return fm_hypot_core(ax, ay);
}
