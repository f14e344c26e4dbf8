// common.cuh -- device helpers shared by the sm_100a kernels of libperm.so.
//
// Double-double ("dd") arithmetic for the compensated accumulation the paper asks for
// (double products, extended-precision sum; P:1165-1186 Kahan).  We use
// Knuth's TwoSum (error-free for any operand order), which -- unlike the classic Kahan loop of
// App. A -- also recovers the sentinel {1e16, 1, -1e16} (reading R7).
#pragma once
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

// Device-side bounds checks of the debug build (PERM_VARIANT=dbg PERM_EXTRA_FLAGS=-DPERM_DEBUG_CHECKS):
// compute-sanitizer is not available on the GPU pool, so index invariants are asserted in the kernels
// themselves and the GPU tests run once against the checking build.
#ifdef PERM_DEBUG_CHECKS
#define PERM_DCHECK(cond)                                                                        \
    do {                                                                                         \
        if (!(cond)) {                                                                           \
            printf("PERM_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                           \
            __trap();                                                                            \
        }                                                                                        \
    } while (0)
#else
#define PERM_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace perm {

struct dd {
    double hi, lo;
};

// Error-free transformation: s + e == a + b exactly (Knuth TwoSum).  __dadd_rn / __dsub_rn keep
// the compiler from contracting or reassociating the sequence.
__host__ __device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
#ifdef __CUDA_ARCH__
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
#else
    volatile double vs = a + b;
    s = vs;
    volatile double bb = s - a;
    volatile double t1 = s - bb;
    volatile double t2 = a - t1;
    volatile double t3 = b - bb;
    e = t2 + t3;
#endif
}

// |a| >= |b| (or a == 0) required: s + e == a + b exactly.
__host__ __device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
#ifdef __CUDA_ARCH__
    s = __dadd_rn(a, b);
    e = __dsub_rn(b, __dsub_rn(s, a));
#else
    volatile double vs = a + b;
    s = vs;
    volatile double t = s - a;
    e = b - t;
#endif
}

// dd + double (accurate): hi/lo renormalized.
__host__ __device__ __forceinline__ dd dd_add_d(dd x, double a) {
    double s, e;
    two_sum(x.hi, a, s, e);
#ifdef __CUDA_ARCH__
    e = __dadd_rn(e, x.lo);
#else
    volatile double t = e + x.lo;
    e = t;
#endif
    dd r;
    fast_two_sum(s, e, r.hi, r.lo);
    return r;
}

// dd + dd (accurate, "IEEE" variant of the double-double add).
__host__ __device__ __forceinline__ dd dd_add(dd x, dd y) {
    double s, e, t, f;
    two_sum(x.hi, y.hi, s, e);
    two_sum(x.lo, y.lo, t, f);
#ifdef __CUDA_ARCH__
    e = __dadd_rn(e, t);
    fast_two_sum(s, e, s, e);
    e = __dadd_rn(e, f);
#else
    volatile double v1 = e + t;
    e = v1;
    fast_two_sum(s, e, s, e);
    volatile double v2 = e + f;
    e = v2;
#endif
    dd r;
    fast_two_sum(s, e, r.hi, r.lo);
    return r;
}

struct ddc {  // complex double-double, matches perm_dd_c128_t {hi_re, lo_re, hi_im, lo_im}
    dd re, im;
};

__host__ __device__ __forceinline__ ddc ddc_add(ddc a, ddc b) {
    ddc r;
    r.re = dd_add(a.re, b.re);
    r.im = dd_add(a.im, b.im);
    return r;
}

// dd * dd (Dekker/Bailey with an FMA two-product): relative error ~ 2^-104.
__host__ __device__ __forceinline__ dd dd_mul(dd x, dd y) {
#ifdef __CUDA_ARCH__
    const double p = __dmul_rn(x.hi, y.hi);
    double e = fma(x.hi, y.hi, -p);
    e = fma(x.hi, y.lo, e);
    e = fma(x.lo, y.hi, e);
#else
    volatile double vp = x.hi * y.hi;
    const double p = vp;
    double e = std::fma(x.hi, y.hi, -p);
    e = std::fma(x.hi, y.lo, e);
    e = std::fma(x.lo, y.hi, e);
#endif
    dd r;
    fast_two_sum(p, e, r.hi, r.lo);
    return r;
}

__host__ __device__ __forceinline__ dd dd_neg(dd x) { return dd{-x.hi, -x.lo}; }

// complex dd product (a + ib)(c + id) = (ac - bd) + i(ad + bc)
__host__ __device__ __forceinline__ ddc ddc_mul(ddc x, ddc y) {
    ddc r;
    r.re = dd_add(dd_mul(x.re, y.re), dd_neg(dd_mul(x.im, y.im)));
    r.im = dd_add(dd_mul(x.re, y.im), dd_mul(x.im, y.re));
    return r;
}

// Compile-time count of trailing zeros (for fully unrolled Gray steps).
__host__ __device__ constexpr int ctz_c(unsigned v) { return (v & 1u) ? 0 : 1 + ctz_c(v >> 1); }

__device__ __forceinline__ ddc shfl_down_ddc(ddc v, int off, unsigned mask = 0xffffffffu) {
    ddc r;
    r.re.hi = __shfl_down_sync(mask, v.re.hi, off);
    r.re.lo = __shfl_down_sync(mask, v.re.lo, off);
    r.im.hi = __shfl_down_sync(mask, v.im.hi, off);
    r.im.lo = __shfl_down_sync(mask, v.im.lo, off);
    return r;
}

}  // namespace perm
