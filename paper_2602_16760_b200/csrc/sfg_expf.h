// Bit-exact device port of the host expf the reference links (glibc 2.39,
// sysdeps/ieee754/flt-32/e_expf.c, IFUNC-selected __expf_fma variant on
// FMA-capable x86-64 hosts — both this container and the B200 boxes).
//
// The reference calls expf in softmax (tinyformer.cpp:476) and SiLU
// (tinyformer.cpp:65); a device expf that differs in one ulp on one input
// would break bitwise parity.  The algorithm: k = round(x*32/ln2) via the
// 1.5*2^52 shift trick (fused), r = x*32/ln2 - k (fused), 2^(k/32) from a
// 32-entry table, cubic in r, all in double, one final rounding to float.
// The op sequence below mirrors the fused instructions of __expf_fma
// (vfmadd132sd / vfmsub132sd / vfmadd213sd ...) and is verified against the
// host libm over ALL 2^32 float inputs by tests/test_expf_port.py.
//
// Usable from C (host checker) and CUDA (device); SFG_FMA/SFG_MUL pick the
// IEEE double fused-multiply-add / multiply with no contraction freedom.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SFG_HD __device__ __forceinline__
#define SFG_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SFG_MUL(a, b) __dmul_rn((a), (b))
#define SFG_SUB(a, b) __dsub_rn((a), (b))
#define SFG_AS_U64(d) ((uint64_t)__double_as_longlong(d))
#define SFG_AS_F64(u) __longlong_as_double((long long)(u))
#define SFG_AS_U32(f) ((uint32_t)__float_as_uint(f))
#define SFG_AS_F32(u) __uint_as_float(u)
#define SFG_D2F(d) __double2float_rn(d)
#define SFG_CONST __device__ __constant__
#else
#include <math.h>
#include <string.h>
#define SFG_HD static inline
#define SFG_FMA(a, b, c) fma((a), (b), (c))
#define SFG_MUL(a, b) ((a) * (b))
#define SFG_SUB(a, b) ((a) - (b))
static inline uint64_t sfg_as_u64_(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double sfg_as_f64_(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint32_t sfg_as_u32_(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float sfg_as_f32_(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
#define SFG_AS_U64(d) sfg_as_u64_(d)
#define SFG_AS_F64(u) sfg_as_f64_(u)
#define SFG_AS_U32(f) sfg_as_u32_(f)
#define SFG_AS_F32(u) sfg_as_f32_(u)
#define SFG_D2F(d) ((float)(d))
#define SFG_CONST static const
#endif

// 2^(i/32) as double bits, minus i << 47 (so adding k << 47 scales by 2^(k/32)).
SFG_CONST uint64_t sfg_exp2f_tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

SFG_HD float sfg_expf(float x) {
    const uint32_t ux = SFG_AS_U32(x);
    const uint32_t abstop = (ux >> 20) & 0x7ffu;
    if (abstop >= 0x42au) {  // |x| >= 88 or nan/inf
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return SFG_AS_F32(0x7f800000u);       // overflow -> +inf
        if (x < -0x1.9fe368p6f) return 0.0f;                          // underflow -> 0
        if (x < -0x1.9d1d9ep6f) return SFG_AS_F32(0x00000001u);      // may-underflow: 2^-149
    }
    const double xd = (double)x;
    const double inv_ln2_n = 0x1.71547652b82fep+5;
    const double shift = 0x1.8p+52;
    const double kd0 = SFG_FMA(inv_ln2_n, xd, shift);
    const uint64_t ki = SFG_AS_U64(kd0);
    const double kd = SFG_SUB(kd0, shift);
    const double r = SFG_FMA(inv_ln2_n, xd, -kd);
    uint64_t t = sfg_exp2f_tab[ki % 32];
    t += ki << 47;
    const double s = SFG_AS_F64(t);
    const double z = SFG_FMA(r, 0x1.c6af84b912394p-20, 0x1.ebfce50fac4f3p-13);
    const double r2 = SFG_MUL(r, r);
    double y = SFG_FMA(r, 0x1.62e42ff0c52d6p-6, 1.0);
    y = SFG_FMA(z, r2, y);
    y = SFG_MUL(y, s);
    return SFG_D2F(y);
}
