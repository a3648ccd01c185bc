// K0 — generic batched-einsum evaluator on sm_100a.
//
// Evaluates ANY valid batched einsum (every dtype, functional operands, 0-dim
// operands, diagonals, full reductions) with the reference's exact operation
// order, so results are bit-identical to feinsum::evaluate
// (proj/src/core.cpp:269-358) for finite inputs:
//   * one thread per (row, output point), grid-stride;
//   * reduction points enumerated with an odometer, last reduction symbol
//     fastest, symbols in first-occurrence order (:284-293, :343-346);
//   * each term is the product of the slot values left to right from 1+0i
//     (:335-340), every multiply explicitly rounded (no FMA);
//   * terms are combined by the same pairwise tree (:259-267): blocks of <= 8
//     summed sequentially from 0, larger ranges split at n/2 — streamed with
//     an explicit stack so no term buffer is needed.
// Tuned kernels (fem_grad.cu, gett.cu, tt.cu, hex.cu) take the canonical forms
// they match; this kernel is the always-correct device path for the rest.
#include <cuda_runtime.h>

#include "launch.h"
#include "operand.cuh"

namespace feb200 {

namespace {

constexpr int kStack = 64;

struct Odo {
  std::int64_t val[kMaxSyms];
};

template <bool kComplex>
struct GenericEval {
  const GenericLaunch& p;
  OperandEnv env;
  int row;
  Odo odo;
  std::int64_t params[kMaxDims];

  __device__ GenericEval(const GenericLaunch& prm, int r) : p(prm), row(r) {
    env.prog = p.prog;
    env.reads = p.reads;
    env.coef = p.coef;
    env.leaves = &p.leaves;
  }

  __device__ cdbl operand(int k) {
    const OperandStatic& op = p.ops[row * p.n + k];
    const int nd = p.slot_ndim[k];
    const int* pos = p.slot_pos + k * kMaxDims;
    const std::int64_t* stride = p.slot_stride + k * kMaxDims;
    if (op.kind == OPK_VM) {
      for (int d = 0; d < nd; ++d) params[d] = odo.val[pos[d]];
      return kComplex ? eval_vm(op, env, params) : cdbl{eval_vm_real(op, env, params), 0.0};
    }
    std::int64_t off = 0;
    for (int d = 0; d < nd; ++d) off += odo.val[pos[d]] * stride[d];
    if (op.kind == OPK_AFFINE) return eval_affine<kComplex>(op, env, off);
    const void* ptr = p.leaves.ptr[op.leaf];
    const int st = p.leaves.storage[op.leaf];
    return kComplex ? load_cplx(ptr, st, off) : cdbl{load_real(ptr, st, off), 0.0};
  }

  // product of the slot values at the current odometer, then advance the
  // reduction odometer (last symbol fastest)
  __device__ cdbl next_term() {
    cdbl prod{1.0, 0.0};
    for (int k = 0; k < p.n; ++k) {
      const cdbl v = operand(k);
      prod = kComplex ? cmul(prod, v) : cdbl{__dmul_rn(prod.re, v.re), 0.0};
    }
    for (int i = p.n_syms - 1; i >= p.n_out; --i) {
      if (++odo.val[i] < p.extent[i]) break;
      odo.val[i] = 0;
    }
    return prod;
  }

  __device__ cdbl leaf_sum(std::int64_t cnt) {
    cdbl s{0.0, 0.0};
    for (std::int64_t t = 0; t < cnt; ++t) {
      const cdbl x = next_term();
      s = kComplex ? cadd(s, x) : cdbl{__dadd_rn(s.re, x.re), 0.0};
    }
    return s;
  }

  __device__ cdbl add(cdbl x, cdbl y) const {
    return kComplex ? cadd(x, y) : cdbl{__dadd_rn(x.re, y.re), 0.0};
  }

  // pairwise_sum over p.red_points terms generated in order. Frame phases:
  // 0 = left child pending, 1 = left done / right pending, 2 = right running.
  __device__ cdbl pairwise() {
    const std::int64_t n0 = p.red_points;
    if (n0 <= 8) return leaf_sum(n0);
    std::int64_t len[kStack];
    int phase[kStack];
    cdbl left[kStack];
    int sp = 0;
    len[0] = n0;
    phase[0] = 0;
    cdbl ret{0.0, 0.0};
    for (;;) {
      const std::int64_t L = len[sp];
      if (phase[sp] == 0) {
        const std::int64_t h = L / 2;
        if (h > 8) {
          ++sp;
          len[sp] = h;
          phase[sp] = 0;
          continue;
        }
        left[sp] = leaf_sum(h);
        phase[sp] = 1;
      }
      if (phase[sp] == 1) {
        const std::int64_t r = L - L / 2;
        if (r > 8) {
          phase[sp] = 2;
          ++sp;
          len[sp] = r;
          phase[sp] = 0;
          continue;
        }
        ret = add(left[sp], leaf_sum(r));
      } else {
        ret = add(left[sp], ret);
      }
      if (sp == 0) return ret;
      --sp;
      if (phase[sp] == 0) {
        left[sp] = ret;
        phase[sp] = 1;
      }
    }
  }
};

template <bool kComplex>
__global__ void __launch_bounds__(128) generic_kernel(const __grid_constant__ GenericLaunch p) {
  const std::int64_t total = p.out_points * p.b;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(t / p.out_points);
    const std::int64_t op = t - static_cast<std::int64_t>(row) * p.out_points;
    GenericEval<kComplex> ev(p, row);
    // output multi-index (last output symbol fastest), reduction part zeroed
    std::int64_t rem = op;
    for (int i = p.n_out - 1; i >= 0; --i) {
      ev.odo.val[i] = rem % p.extent[i];
      rem /= p.extent[i];
    }
    for (int i = p.n_out; i < p.n_syms; ++i) ev.odo.val[i] = 0;
    const cdbl s = ev.pairwise();
    store_out(p.out[row], p.out_storage[row], op, s);
  }
}

__global__ void coef_kernel(const CoefChain* chains, int n, LeafTable leaves, double* coef) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const CoefChain ch = chains[c];
  cdbl acc{0.0, 0.0};
  for (int f = 0; f < ch.n; ++f) {
    const cdbl v = ch.f[f].leaf < 0 ? cdbl{ch.f[f].lit, 0.0}
                                    : load_cplx(leaves.ptr[ch.f[f].leaf], leaves.storage[ch.f[f].leaf], 0);
    acc = f == 0 ? v : cmul(acc, v);
  }
  coef[2 * c] = acc.re;
  coef[2 * c + 1] = acc.im;
}

template <bool kComplex>
__global__ void __launch_bounds__(128) tabulate_kernel(const __grid_constant__ TabulateLaunch p) {
  OperandEnv env{p.prog, p.reads, p.coef, &p.leaves};
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < p.count;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t flat = p.first + t;
    std::int64_t params[kMaxDims];
    std::int64_t rem = flat;
    for (int d = p.ndim - 1; d >= 0; --d) {
      params[d] = rem % p.shape[d];
      rem /= p.shape[d];
    }
    cdbl v;
    if (p.op->kind == OPK_VM)
      v = kComplex ? eval_vm(*p.op, env, params) : cdbl{eval_vm_real(*p.op, env, params), 0.0};
    else if (p.op->kind == OPK_AFFINE)
      v = eval_affine<kComplex>(*p.op, env, flat);
    else
      v = load_cplx(p.leaves.ptr[p.op->leaf], p.leaves.storage[p.op->leaf], flat);
    if (p.real_out) {
      p.out[t] = v.re;
    } else {
      p.out[2 * t] = v.re;
      p.out[2 * t + 1] = v.im;
    }
  }
}

int grid_for(std::int64_t work, int threads) {
  int sms = 148;
  device_sm_count(&sms);
  std::int64_t blocks = (work + threads - 1) / threads;
  const std::int64_t cap = static_cast<std::int64_t>(sms) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

}  // namespace

int device_sm_count(int* out) {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
  }
  *out = cached;
  return cudaSuccess;
}

int launch_coef(const CoefChain* chains, int n_chains, const LeafTable& leaves, double* coef, void* stream) {
  if (n_chains <= 0) return cudaSuccess;
  coef_kernel<<<(n_chains + 63) / 64, 64, 0, static_cast<cudaStream_t>(stream)>>>(chains, n_chains, leaves, coef);
  return cudaGetLastError();
}

int launch_generic(const GenericLaunch& p, void* stream) {
  const std::int64_t work = p.out_points * p.b;
  if (work == 0) return cudaSuccess;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(work, 128);
  if (p.complex_mode)
    generic_kernel<true><<<grid, 128, 0, s>>>(p);
  else
    generic_kernel<false><<<grid, 128, 0, s>>>(p);
  return cudaGetLastError();
}

int launch_tabulate(const TabulateLaunch& p, void* stream) {
  if (p.count == 0) return cudaSuccess;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(p.count, 128);
  if (p.complex_mode)
    tabulate_kernel<true><<<grid, 128, 0, s>>>(p);
  else
    tabulate_kernel<false><<<grid, 128, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace feb200
