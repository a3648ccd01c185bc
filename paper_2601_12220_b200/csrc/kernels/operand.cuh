// Device-side operand reads: storage decoding, IEEE-exact complex arithmetic
// and the functional-operand programs (affine fast path + register VM).
//
// Every arithmetic step uses the explicitly rounded intrinsics (__dmul_rn,
// __dadd_rn, ...) so nvcc cannot contract a*b+c into an FMA: the reference
// computes each product and sum separately in complex<double>
// (proj/src/core.cpp:335-348, proj/src/raising.cpp:336-393), and the generic
// path reproduces its results bit for bit.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "fastmath.cuh"
#include "launch.h"

namespace feb200 {

struct cdbl {
  double re, im;
};

__device__ __forceinline__ cdbl cmake(double r, double i = 0.0) { return cdbl{r, i}; }

// (a+bi)(c+di) = (ac - bd) + (ad + bc)i, each product rounded separately.
__device__ __forceinline__ cdbl cmul(cdbl x, cdbl y) {
  return cdbl{__dsub_rn(__dmul_rn(x.re, y.re), __dmul_rn(x.im, y.im)),
              __dadd_rn(__dmul_rn(x.re, y.im), __dmul_rn(x.im, y.re))};
}
__device__ __forceinline__ cdbl cadd(cdbl x, cdbl y) { return cdbl{__dadd_rn(x.re, y.re), __dadd_rn(x.im, y.im)}; }
__device__ __forceinline__ cdbl csub(cdbl x, cdbl y) { return cdbl{__dsub_rn(x.re, y.re), __dsub_rn(x.im, y.im)}; }

// Smith-style division with the scaling libgcc's __divdc3 applies; for real
// operands (b = d = 0) it reduces to a / c exactly.
__device__ __forceinline__ cdbl cdiv(cdbl x, cdbl y) {
  const double a = x.re, b = x.im, c = y.re, d = y.im;
  if (fabs(c) < fabs(d)) {
    const double r = __ddiv_rn(c, d);
    const double den = __dadd_rn(__dmul_rn(c, r), d);
    return cdbl{__ddiv_rn(__dadd_rn(__dmul_rn(a, r), b), den), __ddiv_rn(__dsub_rn(__dmul_rn(b, r), a), den)};
  }
  const double r = __ddiv_rn(d, c);
  const double den = __dadd_rn(c, __dmul_rn(d, r));
  return cdbl{__ddiv_rn(__dadd_rn(a, __dmul_rn(b, r)), den), __ddiv_rn(__dsub_rn(b, __dmul_rn(a, r)), den)};
}

// the real-argument functions are fastmath.cuh's (shared with the generated
// programs so the VM and codegen agree bit for bit)
__device__ __forceinline__ cdbl csin_(cdbl z) {
  if (z.im == 0.0) return cdbl{fe_sin(z.re), 0.0};
  return cdbl{fe_sin(z.re) * cosh(z.im), fe_cos(z.re) * sinh(z.im)};
}
__device__ __forceinline__ cdbl ccos_(cdbl z) {
  if (z.im == 0.0) return cdbl{fe_cos(z.re), -0.0 * fe_sin(z.re)};
  return cdbl{fe_cos(z.re) * cosh(z.im), -fe_sin(z.re) * sinh(z.im)};
}
__device__ __forceinline__ cdbl cexp_(cdbl z) {
  const double m = fe_exp(z.re);
  if (z.im == 0.0) return cdbl{m, 0.0};
  return cdbl{m * fe_cos(z.im), m * fe_sin(z.im)};
}
// principal square root; sqrt(-4) = 2i as std::sqrt(std::complex) gives
__device__ __forceinline__ cdbl csqrt_(cdbl z) {
  if (z.im == 0.0) {
    if (z.re < 0.0) return cdbl{0.0, copysign(sqrt(-z.re), z.im)};
    return cdbl{sqrt(z.re), z.im};
  }
  const double r = hypot(z.re, z.im);
  if (z.re > 0.0) {
    const double t = sqrt(0.5 * (r + z.re));
    return cdbl{t, z.im / (2.0 * t)};
  }
  const double t = sqrt(0.5 * (r - z.re));
  return cdbl{fabs(z.im) / (2.0 * t), copysign(t, z.im)};
}

// ---- storage decoding ----

__device__ __forceinline__ double load_real(const void* p, int st, std::int64_t i) {
  switch (st) {
    case ST_F64: return __ldg(static_cast<const double*>(p) + i);
    case ST_F32: return static_cast<double>(__ldg(static_cast<const float*>(p) + i));
    case ST_C128: return __ldg(static_cast<const double*>(p) + 2 * i);
    case ST_C64: return static_cast<double>(__ldg(static_cast<const float*>(p) + 2 * i));
    case ST_I8: return static_cast<double>(static_cast<const std::int8_t*>(p)[i]);
    case ST_I32: return static_cast<double>(__ldg(static_cast<const int*>(p) + i));
    case ST_I64: return static_cast<double>(__ldg(static_cast<const long long*>(p) + i));
    case ST_F16: return static_cast<double>(__half2float(static_cast<const __half*>(p)[i]));
  }
  return 0.0;
}

__device__ __forceinline__ cdbl load_cplx(const void* p, int st, std::int64_t i) {
  if (st == ST_C128) {
    const double2 v = __ldg(static_cast<const double2*>(p) + i);
    return cdbl{v.x, v.y};
  }
  if (st == ST_C64) {
    const float2 v = __ldg(static_cast<const float2*>(p) + i);
    return cdbl{static_cast<double>(v.x), static_cast<double>(v.y)};
  }
  return cdbl{load_real(p, st, i), 0.0};
}

__device__ __forceinline__ void store_out(void* p, int st, std::int64_t i, cdbl v) {
  switch (st) {
    case ST_F64: static_cast<double*>(p)[i] = v.re; break;
    case ST_F32: static_cast<float*>(p)[i] = static_cast<float>(v.re); break;
    case ST_C128: static_cast<double2*>(p)[i] = make_double2(v.re, v.im); break;
    case ST_C64: static_cast<float2*>(p)[i] = make_float2(static_cast<float>(v.re), static_cast<float>(v.im)); break;
    case ST_I8: static_cast<std::int8_t*>(p)[i] = static_cast<std::int8_t>(v.re); break;
    case ST_I32: static_cast<int*>(p)[i] = static_cast<int>(v.re); break;
    case ST_I64: static_cast<long long*>(p)[i] = static_cast<long long>(v.re); break;
    case ST_F16: static_cast<__half*>(p)[i] = __float2half(static_cast<float>(v.re)); break;
  }
}

// ---- functional operands ----

struct OperandEnv {
  const VmInstr* prog;
  const VmRead* reads;
  const double* coef;  // interleaved complex coefficient values
  const LeafTable* leaves;
};

__device__ __forceinline__ cdbl coef_at(const double* coef, int c) { return cdbl{coef[2 * c], coef[2 * c + 1]}; }

// Affine operand at the operand's own flat offset (reads use identity subscripts).
template <bool kComplex>
__device__ __forceinline__ cdbl eval_affine(const OperandStatic& op, const OperandEnv& env, std::int64_t flat) {
  cdbl acc{0.0, 0.0};
  for (int t = 0; t < op.n_terms; ++t) {
    const AffineTerm& tm = op.term[t];
    cdbl x;
    if (tm.leaf < 0) {
      x = coef_at(env.coef, tm.pre);
    } else {
      const void* p = env.leaves->ptr[tm.leaf];
      const int st = env.leaves->storage[tm.leaf];
      x = kComplex ? load_cplx(p, st, flat) : cdbl{load_real(p, st, flat), 0.0};
      if (tm.pre >= 0) x = kComplex ? cmul(coef_at(env.coef, tm.pre), x) : cdbl{__dmul_rn(env.coef[2 * tm.pre], x.re), 0.0};
      if (tm.post0 >= 0) x = kComplex ? cmul(x, coef_at(env.coef, tm.post0)) : cdbl{__dmul_rn(x.re, env.coef[2 * tm.post0]), 0.0};
      if (tm.post1 >= 0) x = kComplex ? cmul(x, coef_at(env.coef, tm.post1)) : cdbl{__dmul_rn(x.re, env.coef[2 * tm.post1]), 0.0};
    }
    if (t == 0)
      acc = x;
    else if (tm.sign > 0)
      acc = kComplex ? cadd(acc, x) : cdbl{__dadd_rn(acc.re, x.re), 0.0};
    else
      acc = kComplex ? csub(acc, x) : cdbl{__dsub_rn(acc.re, x.re), 0.0};
  }
  return acc;
}

// Register VM, complex semantics (std::complex<double> like the reference).
__device__ inline cdbl eval_vm(const OperandStatic& op, const OperandEnv& env, const std::int64_t* params) {
  double rr[kMaxVmRegs], ri[kMaxVmRegs];
  for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
    const VmInstr in = env.prog[pc];
    cdbl a{rr[in.a & (kMaxVmRegs - 1)], ri[in.a & (kMaxVmRegs - 1)]};
    cdbl b{rr[in.b & (kMaxVmRegs - 1)], ri[in.b & (kMaxVmRegs - 1)]};
    cdbl v{0.0, 0.0};
    switch (in.code) {
      case VM_LIT: v = cdbl{in.imm, 0.0}; break;
      case VM_PARAM: v = cdbl{static_cast<double>(params[in.arg]), 0.0}; break;
      case VM_READ: {
        const VmRead& rd = env.reads[in.arg];
        std::int64_t off = 0;
        for (int d = 0; d < rd.ndim; ++d) off += params[rd.param_of[d]] * rd.stride[d];
        v = load_cplx(env.leaves->ptr[rd.leaf], env.leaves->storage[rd.leaf], off);
        break;
      }
      case VM_ADD: v = cadd(a, b); break;
      case VM_SUB: v = csub(a, b); break;
      case VM_MUL: v = cmul(a, b); break;
      case VM_DIV: v = cdiv(a, b); break;
      case VM_SIN: v = csin_(a); break;
      case VM_COS: v = ccos_(a); break;
      case VM_EXP: v = cexp_(a); break;
      case VM_SQRT: v = csqrt_(a); break;
      case VM_RECIP: v = cdiv(cdbl{1.0, 0.0}, a); break;
    }
    rr[in.dst & (kMaxVmRegs - 1)] = v.re;
    ri[in.dst & (kMaxVmRegs - 1)] = v.im;
  }
  return cdbl{rr[0], ri[0]};
}

// The same VM on real values, for plans without complex data or sqrt: with
// zero imaginary parts every complex step above reduces to the real operation
// on the real parts (cmul: a*c - 0*0, cdiv: a/c, csin/ccos/cexp: the real
// functions), so for finite values the results are bit-identical at half the
// registers and arithmetic.
__device__ inline double eval_vm_real(const OperandStatic& op, const OperandEnv& env, const std::int64_t* params) {
  double rr[kMaxVmRegs];
  for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
    const VmInstr in = env.prog[pc];
    const double a = rr[in.a & (kMaxVmRegs - 1)], b = rr[in.b & (kMaxVmRegs - 1)];
    double v = 0.0;
    switch (in.code) {
      case VM_LIT: v = in.imm; break;
      case VM_PARAM: v = static_cast<double>(params[in.arg]); break;
      case VM_READ: {
        const VmRead& rd = env.reads[in.arg];
        std::int64_t off = 0;
        for (int d = 0; d < rd.ndim; ++d) off += params[rd.param_of[d]] * rd.stride[d];
        v = load_real(env.leaves->ptr[rd.leaf], env.leaves->storage[rd.leaf], off);
        break;
      }
      case VM_ADD: v = __dadd_rn(a, b); break;
      case VM_SUB: v = __dsub_rn(a, b); break;
      case VM_MUL: v = __dmul_rn(a, b); break;
      case VM_DIV: v = __ddiv_rn(a, b); break;
      case VM_SIN: v = fe_sin(a); break;
      case VM_COS: v = fe_cos(a); break;
      case VM_EXP: v = fe_exp(a); break;
      case VM_SQRT: v = sqrt(a); break;  // not reached: sqrt makes the plan complex
      case VM_RECIP: v = __ddiv_rn(1.0, a); break;
    }
    rr[in.dst & (kMaxVmRegs - 1)] = v;
  }
  return rr[0];
}

}  // namespace feb200
