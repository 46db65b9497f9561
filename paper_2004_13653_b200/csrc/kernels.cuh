// Kernel functions of Table 1 as used by the GPU paths.
//
// Product form: K(s,t) = C1^2 * khat(s) * khat(t); the constant C1^2 is applied once
// in the epilogue (scale), so each 1-D factor is khat of the pixel offset d (pixels):
// s = d / h_px.  Radial form (R1): K = C2 * khat_r(r^2), r^2 = s^2 + t^2.
// Negative fp32 round-off at the support edge is clamped to 0 (R8).
#pragma once

#include <cuda_runtime.h>

namespace kde {

// 2^x on the SFU, flush-to-zero (kernel values at the truncation edge are >= 3e-4 of the
// peak for cutoff 4, far from the denormal range; beyond the box they are masked anyway)
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct KConst {
    float inv_h;   // 1/h_px
    float inv_h2;  // 1/h_px^2
    float inv_h3;  // 1/h_px^3
    float kq;      // -0.5*log2(e)/h_px^2  (Gaussian, exp2 form)
    float kc;      // pi/(2 h_px)          (Cosine)
};

KConst make_kconst(double hpx);  // host (eval_direct.cu)

// 1-D factor khat(d / h_px) (Table 1 row without its leading constant)
template <int K>
__device__ __forceinline__ float khat(float d, const KConst& k) {
    if constexpr (K == 0) {  // Uniform: (1/2)^2 I I
        return 1.0f;
    } else if constexpr (K == 1) {  // Triangular: (1-|s|)(1-|t|)
        return fmaxf(fmaf(-fabsf(d), k.inv_h, 1.0f), 0.0f);
    } else if constexpr (K == 2) {  // Epanechnikov: (3/4)^2 (1-s^2)(1-t^2)
        return fmaxf(fmaf(-d * d, k.inv_h2, 1.0f), 0.0f);
    } else if constexpr (K == 3) {  // Quartic: (15/16)^2 (1-s^2)^2 (1-t^2)^2
        const float q = fmaxf(fmaf(-d * d, k.inv_h2, 1.0f), 0.0f);
        return q * q;
    } else if constexpr (K == 4) {  // Triweight: (35/32)^2 (1-s^2)^3 (1-t^2)^3
        const float q = fmaxf(fmaf(-d * d, k.inv_h2, 1.0f), 0.0f);
        return q * q * q;
    } else if constexpr (K == 5) {  // Tricube: (70/81)^2 (1-|s|^3)^3 (1-|t|^3)^3
        const float a = fabsf(d);
        const float q = fmaxf(fmaf(-a * a * a, k.inv_h3, 1.0f), 0.0f);
        return q * q * q;
    } else if constexpr (K == 6) {  // Gaussian: (1/sqrt(2 pi))^2 exp(-(s^2+t^2)/2)
        return ex2_ftz(d * d * k.kq);
    } else {  // Cosine: (pi/4)^2 cos(pi s/2) cos(pi t/2)
        return fmaxf(__cosf(d * k.kc), 0.0f);
    }
}

// radial khat_r as a function of r^2 (in units of h)
template <int K>
__device__ __forceinline__ float khat_r(float r2) {
    if constexpr (K == 0) {
        return 1.0f;
    } else if constexpr (K == 1) {
        return fmaxf(1.0f - sqrtf(r2), 0.0f);
    } else if constexpr (K == 2) {
        return fmaxf(1.0f - r2, 0.0f);
    } else if constexpr (K == 3) {
        const float q = fmaxf(1.0f - r2, 0.0f);
        return q * q;
    } else if constexpr (K == 4) {
        const float q = fmaxf(1.0f - r2, 0.0f);
        return q * q * q;
    } else if constexpr (K == 5) {
        const float q = fmaxf(1.0f - r2 * sqrtf(r2), 0.0f);
        return q * q * q;
    } else if constexpr (K == 6) {
        return ex2_ftz(r2 * -0.72134752044448170368f);  // exp(-r^2/2) = 2^(-r^2 log2(e)/2)
    } else {
        return fmaxf(__cosf(sqrtf(r2) * 1.57079632679489661923f), 0.0f);
    }
}

// host side: the leading constant (C1^2 product, C2 radial), fp64
inline double kernel_constant(int kernel, bool radial) {
    const double pi = 3.14159265358979323846;
    if (!radial) {
        const double c1[8] = {0.5, 1.0, 0.75, 15.0 / 16.0, 35.0 / 32.0, 70.0 / 81.0,
                              0.39894228040143267794 /* 1/sqrt(2 pi) */, pi / 4.0};
        return c1[kernel] * c1[kernel];
    }
    const double c2[8] = {1.0 / pi, 3.0 / pi, 2.0 / pi, 3.0 / pi, 4.0 / pi, 220.0 / (81.0 * pi),
                          1.0 / (2.0 * pi), pi / (4.0 * (pi - 2.0))};
    return c2[kernel];
}

}  // namespace kde
