// Device tanh that returns the same bits as the host's std::tanh.
//
// The reference evaluates sstep/tanh with std::tanh (model.cpp:253), i.e.
// glibc's fdlibm-derived __tanh (sysdeps/ieee754/dbl-64/s_tanh.c), which calls
// __expm1 (s_expm1.c). On x86-64 hosts with FMA, glibc 2.39 dispatches
// expm1 to its FMA build (sysdeps/x86_64/fpu/multiarch/s_expm1-fma.c: the
// same source compiled with -mfma -mavx2), whose polynomial is the
// second-order Estrin form glibc uses (R1 + h2*R2 + h4*R3). CUDA's tanh()
// differs from that in the last bit for a fraction of inputs, and the LM
// trajectory amplifies one-ulp differences in the Jacobian (a
// 4e-3 parameter difference on a real calibration table).
//
// Every operation below is an explicit round-to-nearest intrinsic, so the
// result does not depend on the translation unit's -fmad setting: __fma_rn
// exactly where gcc contracts the glibc source under -ffp-contract=fast
// (read off its GIMPLE: FMA/FNMA/FMS nodes), plain products and sums
// elsewhere. Checked against the host's tanh on 2e7 log-uniform inputs in
// [2^-29, 55] with 0 mismatches (tools/exp/tanh_glibc.c); on a host without
// FMA glibc uses the non-FMA build, which differs in ~3e-4 of inputs.
#pragma once

#include <cstdint>

namespace ps {

__device__ __forceinline__ uint32_t hi_word(double x) {
  return (uint32_t)((unsigned long long)__double_as_longlong(x) >> 32);
}
__device__ __forceinline__ uint32_t lo_word(double x) {
  return (uint32_t)((unsigned long long)__double_as_longlong(x) & 0xffffffffull);
}
__device__ __forceinline__ double with_hi_word(double x, uint32_t h) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  u = (u & 0xffffffffull) | ((unsigned long long)h << 32);
  return __longlong_as_double((long long)u);
}

// glibc __expm1 (fdlibm s_expm1.c), FMA build.
static __device__ __noinline__ double glibc_expm1(double x) {
  const double one = 1.0, huge = 1.0e+300, tiny = 1.0e-300;
  const double o_threshold = 7.09782712893383973096e+02;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double invln2 = 1.44269504088896338700e+00;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  double hi, lo, c = 0.0, t, e, hxs, hfx, r1, y;
  int k;
  uint32_t hx = hi_word(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4043687Au) {  // |x| >= 56 ln2
    if (hx >= 0x40862E42u) {  // |x| >= 709.78
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffffu) | lo_word(x)) != 0) return __dadd_rn(x, x);  // NaN
        return xsb == 0 ? x : -1.0;
      }
      if (x > o_threshold) return __dmul_rn(huge, huge);
    }
    if (xsb != 0 && __dadd_rn(x, tiny) < 0.0) return __dsub_rn(tiny, one);
  }
  if (hx > 0x3fd62e42u) {  // |x| > 0.5 ln2: argument reduction
    if (hx < 0x3FF0A2B2u) {  // and |x| < 1.5 ln2
      if (xsb == 0) {
        hi = __dsub_rn(x, ln2_hi);
        lo = ln2_lo;
        k = 1;
      } else {
        hi = __dadd_rn(x, ln2_hi);
        lo = -ln2_lo;
        k = -1;
      }
    } else {
      k = (int)__dadd_rn(__dmul_rn(x, invln2), xsb == 0 ? 0.5 : -0.5);  // not contracted
      t = (double)k;
      hi = __fma_rn(-t, ln2_hi, x);
      lo = __dmul_rn(t, ln2_lo);
    }
    x = __dsub_rn(hi, lo);
    c = __dsub_rn(__dsub_rn(hi, x), lo);
  } else if (hx < 0x3c900000u) {  // |x| < 2^-54
    t = __dadd_rn(huge, x);
    return __dsub_rn(x, __dsub_rn(t, t));
  } else {
    k = 0;
  }
  hfx = __dmul_rn(x, 0.5);
  hxs = __dmul_rn(x, hfx);
  {
    const double R1 = __fma_rn(hxs, Q1, one);
    const double h2 = __dmul_rn(hxs, hxs);
    const double R2 = __fma_rn(hxs, Q3, Q2);
    const double h4 = __dmul_rn(h2, h2);
    const double R3 = __fma_rn(hxs, Q5, Q4);
    r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
  }
  t = __fma_rn(-r1, hfx, 3.0);
  e = __dmul_rn(__ddiv_rn(__dsub_rn(r1, t), __fma_rn(-x, t, 6.0)), hxs);
  if (k == 0) return __dsub_rn(x, __fma_rn(x, e, -hxs));
  e = __fma_rn(__dsub_rn(e, c), x, -c);
  e = __dsub_rn(e, hxs);
  if (k == -1) return __fma_rn(__dsub_rn(x, e), 0.5, -0.5);
  if (k == 1) {
    if (x < -0.25) return __dmul_rn(__dsub_rn(e, __dadd_rn(x, 0.5)), -2.0);
    return __fma_rn(__dsub_rn(x, e), 2.0, one);
  }
  if (k <= -2 || k > 56) {  // exp(x) - 1 with the exponent added
    y = __dsub_rn(one, __dsub_rn(e, x));
    y = with_hi_word(y, hi_word(y) + ((uint32_t)k << 20));
    return __dsub_rn(y, one);
  }
  if (k < 20) {
    t = with_hi_word(0.0, 0x3ff00000u - (0x200000u >> k));  // 1 - 2^-k
    y = __dsub_rn(t, __dsub_rn(e, x));
    y = with_hi_word(y, hi_word(y) + ((uint32_t)k << 20));
  } else {
    t = with_hi_word(0.0, (uint32_t)(0x3ff - k) << 20);  // 2^-k
    y = __dsub_rn(x, __dadd_rn(e, t));
    y = __dadd_rn(y, one);
    y = with_hi_word(y, hi_word(y) + ((uint32_t)k << 20));
  }
  return y;
}

// glibc __tanh (fdlibm s_tanh.c).
__device__ __forceinline__ double glibc_tanh(double x) {
  const double one = 1.0, two = 2.0, tiny = 1.0e-300;
  const uint32_t jx = hi_word(x), ix = jx & 0x7fffffffu, lx = lo_word(x);
  const bool neg = (jx & 0x80000000u) != 0;
  if (ix >= 0x7ff00000u)  // inf or NaN
    return neg ? __dsub_rn(__ddiv_rn(one, x), one) : __dadd_rn(__ddiv_rn(one, x), one);
  double z;
  if (ix < 0x40360000u) {  // |x| < 22
    if ((ix | lx) == 0) return x;
    if (ix < 0x3c800000u) return __dmul_rn(x, __dadd_rn(one, x));  // |x| < 2^-55
    if (ix >= 0x3ff00000u) {  // |x| >= 1
      const double t = glibc_expm1(__dmul_rn(two, fabs(x)));
      z = __dsub_rn(one, __ddiv_rn(two, __dadd_rn(t, two)));
    } else {
      const double t = glibc_expm1(__dmul_rn(-two, fabs(x)));
      z = __ddiv_rn(-t, __dadd_rn(t, two));
    }
  } else {
    z = __dsub_rn(one, tiny);
  }
  return neg ? -z : z;
}

}  // namespace ps
