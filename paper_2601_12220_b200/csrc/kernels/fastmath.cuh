// Double-precision exp / sin / cos for the functional-operand programs (the
// device VM in operand.cuh and the NVRTC-generated straight-line programs of
// codegen.cpp, which must agree bit for bit).
//
// libdevice's versions branch inside every call (slow-path argument
// reduction, special cases), which splits a program of several calls into
// many basic blocks: the scheduler cannot interleave independent evaluations
// and the operand prologue of the generated C5 instance ran latency-bound
// (ncu: `wait` stalls 37%, 135 instructions per s = u^2 - sin(k)/(2+exp(u))).
// Here the common range is straight-line code: Cody-Waite reduction with FMA,
// then fixed polynomials (Taylor degree 13 for exp on |r| <= ln2/2; the fdlibm
// __kernel_sin / __kernel_cos coefficients on |r| <= pi/4), error within ~2 ulp
// — far inside the 1e-12 parity bar against the reference's libm. Arguments
// outside the range (|x| > 700 for exp, |x| > 1e5 for sin/cos, NaN, inf) take
// libdevice. fe_*_fast skip the range test for callers that checked it once
// for a whole block of evaluations (fe_*_ok).
#pragma once

namespace feb200 {

// Polynomial coefficients in the constant bank: each DFMA then reads its
// coefficient as a c[bank][offset] operand (double immediates do not exist:
// as literals every coefficient cost two UMOVs per use, 19% of the fused C5
// prologue's instructions)
static __constant__ double kFeExp[14] = {
    1.6059043836821614599e-10, 2.0876756987868098979e-09, 2.5052108385441718775e-08, 2.7557319223985890653e-07,
    2.7557319223985892510e-06, 2.4801587301587301566e-05, 1.9841269841269841253e-04, 1.3888888888888889419e-03,
    8.3333333333333332177e-03, 4.1666666666666664354e-02, 1.6666666666666665741e-01, 0.5, 1.0, 1.0};  // 1/k!, k = 13..0
static __constant__ double kFeSin[6] = {1.58969099521155010221e-10, -2.50507602534068634195e-08,
                                        2.75573137070700676789e-06, -1.98412698298579493134e-04,
                                        8.33333333332248946124e-03, -1.66666666666666324348e-01};
static __constant__ double kFeCos[6] = {-1.13596475577881948265e-11, 2.08757232129817482790e-09,
                                        -2.75573143513906633035e-07, 2.48015872894767294178e-05,
                                        -1.38888888888741095749e-03, 4.16666666666666019037e-02};

__device__ __forceinline__ bool fe_exp_ok(double x) { return fabs(x) <= 700.0; }
__device__ __forceinline__ bool fe_trig_ok(double x) { return fabs(x) <= 1.0e5; }

__device__ __forceinline__ double fe_exp_fast(double x) {
  const double n = rint(x * 1.4426950408889634074);
  double r = fma(-n, 6.93147180369123816490e-01, x);  // ln2_hi (fdlibm): n * ln2_hi exact
  r = fma(-n, 1.90821492927058770002e-10, r);        // ln2_lo
  // e^r, |r| <= 0.3466: sum_{k<=13} r^k / k!  (truncation < 5e-18 relative)
  double p = kFeExp[0];
#pragma unroll
  for (int k = 1; k < 14; ++k) p = fma(p, r, kFeExp[k]);
  // times 2^n: |n| <= 1010 and p in [0.70, 1.42], so the result stays normal
  const long long k = static_cast<long long>(n);
  return __longlong_as_double(__double_as_longlong(p) + (k << 52));
}

// sin(r) and cos(r) on |r| <= pi/4 (fdlibm __kernel_sin / __kernel_cos
// minimax coefficients, tail correction omitted: within ~2 ulp)
__device__ __forceinline__ double fe_sin_kernel(double r, double s) {
  double p = kFeSin[0];
#pragma unroll
  for (int k = 1; k < 6; ++k) p = fma(p, s, kFeSin[k]);
  return fma(r * s, p, r);
}
__device__ __forceinline__ double fe_cos_kernel(double s) {
  double p = kFeCos[0];
#pragma unroll
  for (int k = 1; k < 6; ++k) p = fma(p, s, kFeCos[k]);
  return fma(s * s, p, fma(-0.5, s, 1.0));
}

// quadrant q of x = q * pi/2 + r; shift 0 gives sin, 1 gives cos
__device__ __forceinline__ double fe_sincos_fast(double x, int shift) {
  const double q = rint(x * 6.36619772367581382433e-01);  // 2/pi
  double r = fma(-q, 1.57079632679489655800e+00, x);      // pio2 (first 53 bits), product exact in the FMA
  r = fma(-q, 6.12323399573676603587e-17, r);             // pio2 - pio2_hi
  const double s = r * r;
  const double sv = fe_sin_kernel(r, s), cv = fe_cos_kernel(s);
  const int n = (static_cast<int>(static_cast<long long>(q)) + shift) & 3;
  const double v = (n & 1) ? cv : sv;
  return (n & 2) ? -v : v;
}
__device__ __forceinline__ double fe_sin_fast(double x) { return fe_sincos_fast(x, 0); }
__device__ __forceinline__ double fe_cos_fast(double x) { return fe_sincos_fast(x, 1); }

__device__ __forceinline__ double fe_exp(double x) { return fe_exp_ok(x) ? fe_exp_fast(x) : exp(x); }
__device__ __forceinline__ double fe_sin(double x) { return fe_trig_ok(x) ? fe_sin_fast(x) : sin(x); }
__device__ __forceinline__ double fe_cos(double x) { return fe_trig_ok(x) ? fe_cos_fast(x) : cos(x); }

}  // namespace feb200
