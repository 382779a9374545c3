// ref_tanh.cuh -- the reference's tanh, bit for bit, on the device.
//
// The reference's tanh_trial (solvers.cpp:145-148) calls std::tanh, i.e. glibc's libm.  In
// this image (glibc 2.39, x86-64) `tanh` is fdlibm's algorithm built for baseline x86-64, and
// it calls `expm1` through an ifunc that selects the FMA build on FMA/AVX2 hosts: fdlibm's
// expm1 with the rational polynomial in Estrin form and the compiler's fused multiply-adds.
// Both are restated here from that machine code with every operation explicit (__d*_rn /
// __fma_rn: nvcc must not contract or reorder anything), so ref_tanh(x) == glibc tanh(x) for
// every double.  Pinned on the host by tools/ref_tanh_check.c (0 mismatches over 3e7 random
// inputs per function plus the special values) and on the device by
// tests/test_gpu_parity.py::test_device_tanh_matches_libm.  With it the fp64 sparse kernels
// compute the reference's sweep exactly: trajectories, iteration counts and spins are
// identical run for run.
//
// Derived from fdlibm (s_tanh.c, s_expm1.c) as shipped in glibc:
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this software is freely granted,
//   provided that this notice is preserved.
#pragma once

#include <cstdint>

namespace marsb200 {

__device__ __forceinline__ double rt_add_hi(double y, int k) {   // high word += k << 20
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(y));
    const unsigned hi = static_cast<unsigned>(b >> 32) + (static_cast<unsigned>(k) << 20);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) |
                                                       (b & 0xffffffffull)));
}

__device__ __forceinline__ double rt_from_hi(unsigned hi) {
    return __longlong_as_double(static_cast<long long>(static_cast<unsigned long long>(hi) << 32));
}

// glibc 2.39 expm1, FMA build (the ifunc's choice on FMA hosts).
static __device__ __forceinline__ double ref_expm1(double x) {
    const double invln2 = 1.4426950408889634, ln2_hi = 0.6931471803691238, ln2_lo = 1.9082149292705877e-10;
    const double Q1 = -0.03333333333333313, Q2 = 0.0015873015872548146, Q3 = -7.93650757867488e-05,
                 Q4 = 4.008217827329362e-06, Q5 = -2.0109921818362437e-07;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned hx = static_cast<unsigned>(b >> 32) & 0x7fffffffu;
    const bool neg = (b >> 63) != 0;
    double hi, lo, c = 0.0;
    int k;
    if (hx > 0x40436879u) {                                   // |x| >= 56 ln2
        if (hx > 0x40862e41u) {
            if (hx > 0x7fefffffu) {
                if (((static_cast<unsigned>(b >> 32) & 0xfffffu) | static_cast<unsigned>(b)) != 0u)
                    return __dadd_rn(x, x);                   // NaN
                return neg ? -1.0 : x;                        // +-inf
            }
            if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000ll);
        }
        if (neg) return -1.0;                                 // 1e-300 - 1
        k = __double2int_rz(__dadd_rn(0.5, __dmul_rn(x, invln2)));
        const double t = __int2double_rn(k);
        hi = __fma_rn(-t, ln2_hi, x);
        lo = __dmul_rn(t, ln2_lo);
        x = __dsub_rn(hi, lo);
        c = __dsub_rn(__dsub_rn(hi, x), lo);
    } else if (hx > 0x3fd62e42u) {                            // |x| > 0.5 ln2
        if (hx > 0x3ff0a2b1u) {
            k = __double2int_rz(__dadd_rn(neg ? -0.5 : 0.5, __dmul_rn(x, invln2)));
            const double t = __int2double_rn(k);
            hi = __fma_rn(-t, ln2_hi, x);
            lo = __dmul_rn(t, ln2_lo);
        } else if (!neg) {
            hi = __dsub_rn(x, ln2_hi);
            lo = ln2_lo;
            k = 1;
        } else {
            hi = __dadd_rn(x, ln2_hi);
            lo = -ln2_lo;
            k = -1;
        }
        x = __dsub_rn(hi, lo);
        c = __dsub_rn(__dsub_rn(hi, x), lo);
    } else if (hx <= 0x3c8fffffu) {                           // |x| < 2^-54
        return x;                                             // x - ((x + huge) - (x + huge))
    } else {
        k = 0;
    }
    const double hfx = __dmul_rn(x, 0.5), hxs = __dmul_rn(x, hfx);
    const double R2 = __fma_rn(hxs, Q3, Q2), R3 = __fma_rn(hxs, Q5, Q4), h2 = __dmul_rn(hxs, hxs);
    const double R1 = __fma_rn(hxs, Q1, 1.0), h4 = __dmul_rn(h2, h2);
    const double r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
    const double t = __fma_rn(-r1, hfx, 3.0);
    double e = __dmul_rn(__ddiv_rn(__dsub_rn(r1, t), __fma_rn(-x, t, 6.0)), hxs);
    if (k == 0) return __dsub_rn(x, __fma_rn(e, x, -hxs));
    e = __dsub_rn(__fma_rn(__dsub_rn(e, c), x, -c), hxs);
    if (k == -1) return __fma_rn(__dsub_rn(x, e), 0.5, -0.5);
    if (k == 1) {
        if (x < -0.25) return __dmul_rn(__dsub_rn(e, __dadd_rn(x, 0.5)), -2.0);
        return __fma_rn(__dsub_rn(x, e), 2.0, 1.0);
    }
    if (static_cast<unsigned>(k + 1) > 57u) {                 // k <= -2 or k > 56
        const double y = __dsub_rn(1.0, __dsub_rn(e, x));
        return __dsub_rn(rt_add_hi(y, k), 1.0);
    }
    if (k < 20) {
        const double t2 = rt_from_hi(0x3ff00000u - (0x200000u >> k));
        return rt_add_hi(__dsub_rn(t2, __dsub_rn(e, x)), k);
    }
    const double t2 = rt_from_hi(static_cast<unsigned>(0x3ff - k) << 20);
    return rt_add_hi(__dadd_rn(__dsub_rn(x, __dadd_rn(e, t2)), 1.0), k);
}

// glibc 2.39 tanh (baseline x86-64 build, no contraction) with the expm1 it calls inlined in
// branch-free form: expm1's argument here is -2|x| (|x| < 1) or 2|x| (1 <= |x| < 22), and the
// lanes of a warp would otherwise diverge over its range and reconstruction branches.  The
// reduction integer k is computed as glibc does (0 up to the 0.5 ln2 threshold, else
// trunc(+-0.5 + a/ln2), which yields glibc's +-1 in the band it special-cases, with the same
// hi/lo), every reconstruction is evaluated and the one for k selected, and tanh's two
// divisions share one (num / (t + 2)).  Same operations as ref_expm1 + glibc tanh, so the
// same bits (tools/ref_tanh_host.h g_tanh_bf: 0 mismatches vs libm over 3e7 inputs).
__device__ __forceinline__ double ref_tanh(double x) {
    const double invln2 = 1.4426950408889634, ln2_hi = 0.6931471803691238, ln2_lo = 1.9082149292705877e-10;
    const double Q1 = -0.03333333333333313, Q2 = 0.0015873015872548146, Q3 = -7.93650757867488e-05,
                 Q4 = 4.008217827329362e-06, Q5 = -2.0109921818362437e-07;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned ix = static_cast<unsigned>(b >> 32) & 0x7fffffffu;
    const double ax = fabs(x);
    const bool small = ix <= 0x3fefffffu;                                // |x| < 1
    const double a = small ? __dmul_rn(ax, -2.0) : __dadd_rn(ax, ax);    // expm1 argument
    const unsigned ha = static_cast<unsigned>(static_cast<unsigned long long>(__double_as_longlong(a)) >> 32) & 0x7fffffffu;
    const int k = ha <= 0x3fd62e42u ? 0 : __double2int_rz(__dadd_rn(a < 0.0 ? -0.5 : 0.5, __dmul_rn(a, invln2)));
    const double tk = __int2double_rn(k);
    const double hi = __fma_rn(-tk, ln2_hi, a), lo = __dmul_rn(tk, ln2_lo);
    const double xr = __dsub_rn(hi, lo), c = __dsub_rn(__dsub_rn(hi, xr), lo);
    const double hfx = __dmul_rn(xr, 0.5), hxs = __dmul_rn(xr, hfx);
    const double R2 = __fma_rn(hxs, Q3, Q2), R3 = __fma_rn(hxs, Q5, Q4), h2 = __dmul_rn(hxs, hxs);
    const double R1 = __fma_rn(hxs, Q1, 1.0), h4 = __dmul_rn(h2, h2);
    const double r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
    const double t = __fma_rn(-r1, hfx, 3.0);
    const double e = __dmul_rn(__ddiv_rn(__dsub_rn(r1, t), __fma_rn(-xr, t, 6.0)), hxs);
    const double r0 = __dsub_rn(xr, __fma_rn(e, xr, -hxs));                        // k == 0
    const double e2 = __dsub_rn(__fma_rn(__dsub_rn(e, c), xr, -c), hxs);
    const double rm1 = __fma_rn(__dsub_rn(xr, e2), 0.5, -0.5);                     // k == -1
    const double rp1 = xr < -0.25 ? __dmul_rn(__dsub_rn(e2, __dadd_rn(xr, 0.5)), -2.0)
                                  : __fma_rn(__dsub_rn(xr, e2), 2.0, 1.0);        // k == 1
    const double rbig = __dsub_rn(rt_add_hi(__dsub_rn(1.0, __dsub_rn(e2, xr)), k), 1.0);   // k <= -2 | k > 56
    const int kl = min(max(k, 0), 19), kh = min(max(k, 20), 1023);
    const double rmid = rt_add_hi(__dsub_rn(rt_from_hi(0x3ff00000u - (0x200000u >> kl)), __dsub_rn(e2, xr)), k);
    const double rhi = rt_add_hi(
        __dadd_rn(__dsub_rn(xr, __dadd_rn(e2, rt_from_hi(static_cast<unsigned>(0x3ff - kh) << 20))), 1.0), k);
    const double em1 = k == 0 ? r0 : k == -1 ? rm1 : k == 1 ? rp1
                     : (static_cast<unsigned>(k + 1) > 57u ? rbig : (k < 20 ? rmid : rhi));
    const double q = __ddiv_rn(small ? -em1 : 2.0, __dadd_rn(em1, 2.0));
    double z = small ? q : __dsub_rn(1.0, q);
    if (ix > 0x4035ffffu) z = 1.0;                                       // |x| >= 22 (and inf)
    if (ix <= 0x3c7fffffu)                                               // |x| < 2^-55, +-0
        return (ix | static_cast<unsigned>(b)) == 0u ? x : __dmul_rn(__dadd_rn(1.0, x), x);
    return static_cast<long long>(b) >= 0 ? z : -z;
}

// tanh_trial (solvers.cpp:145-148) in the reference's exact arithmetic.
__device__ __forceinline__ double ref_tanh_trial(double phi, double t) {
    if (t < 1e-12) return phi > 0.0 ? -1.0 : (phi < 0.0 ? 1.0 : 0.0);
    return -ref_tanh(__ddiv_rn(phi, t));
}

}  // namespace marsb200
