// K5 — sum-factorised hex matrix-free operator (C2: P4 hex Poisson, 8 fields)
//
//   y_q[e,i,m,n] = sum_{x,y,a,b,c,j,k,l} B1[x,a,i] B2[x,b,m] B3[x,c,n] G[x,y,e,a,b,c]
//                                          F1[y,a,j] F2[y,b,k] F3[y,c,l] u_q[e,j,k,l]
//
// evaluated per element by the sum-factorised path (the optimal pairwise
// contraction order, 12375 MACs per element and field at P = 5):
//   t_y = (F1[y] x F2[y] x F3[y]) u      three 1-D sweeps per direction y
//   q_x = sum_y G[x,y] . t_y              pointwise 3x3 geometric factors
//   y  += (B1[x] x B2[x] x B3[x])^T q_x   three transposed sweeps per x
//
// B200 design: persistent CTAs walk element PAIRS (a pair of 125-double
// blocks is a 16-byte-aligned 2000-byte run, the unit of a 1-D bulk copy).
// One elected thread streams the pair's 9 G blocks and every field's u block
// with cp.async.bulk into a double-buffered mbarrier ring, so G — the dominant
// traffic — is read from HBM once and reused by all fields while the next pair
// is in flight. Sweeps run from shared memory on the FP64 pipe (5x5 operators
// are too small for DMMA tiles: padding to 8x8 would waste 61%); the 1-D
// operators live in shared memory and are read as warp-uniform broadcasts.
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int P = 5;              // points / dofs per direction
constexpr int P3 = P * P * P;     // 125
constexpr int ND = 3;             // directions
constexpr int NE = 2;             // elements per pipeline stage (one bulk copy)
constexpr int kMaxFields = 8;
constexpr int kThreads = 256;

struct HexDev {
  std::int64_t E;
  int rows;
  const double* G;
  const double* U[kMaxFields];
  double* Y[kMaxFields];
  const double* mats[6];  // F1 F2 F3 (forward, [y][quad][dof]) B1 B2 B3 (backward, [x][quad][dof])
};

// out = M . in along `axis` of a P x P x P block (row-major), for one line.
// forward: out[o] = sum_i M[o][i] in[i] with M = mat[dir][o][i] (quad o, dof i)
// backward: out[o] = sum_i mat[dir][i][o] in[i] (dof o from quad i)
template <bool kBackward>
__device__ __forceinline__ void sweep_line(const double* __restrict__ in, double* __restrict__ out,
                                           const double* __restrict__ m, int stride, bool accumulate) {
  double v[P];
#pragma unroll
  for (int i = 0; i < P; ++i) v[i] = in[i * stride];
#pragma unroll
  for (int o = 0; o < P; ++o) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) s = fma(kBackward ? m[i * P + o] : m[o * P + i], v[i], s);
    if (accumulate)
      out[o * stride] += s;
    else
      out[o * stride] = s;
  }
}

// All (element, field, line) tasks of one sweep along `axis`.
// `in` is addressed with (field, element) strides; `out` uses the work layout
// [element][field][125].
template <bool kBackward>
__device__ __forceinline__ void sweep(const double* in, int in_fs, int in_es, double* out, const double* m, int axis,
                                      int rows, bool accumulate) {
  const int stride = axis == 0 ? P * P : (axis == 1 ? P : 1);
  const int tasks = NE * rows * P * P;
  for (int t = threadIdx.x; t < tasks; t += blockDim.x) {
    const int line = t % (P * P);
    const int ef = t / (P * P);  // (element, field) block
    const int el = ef / rows, f = ef % rows;
    // the two coordinates that are not `axis`
    const int c0 = line / P, c1 = line % P;
    int base;
    if (axis == 0)
      base = c0 * P + c1;
    else if (axis == 1)
      base = c0 * P * P + c1;
    else
      base = c0 * P * P + c1 * P;
    sweep_line<kBackward>(in + f * in_fs + el * in_es + base, out + (el * rows + f) * P3 + base, m, stride,
                          accumulate);
  }
}

__global__ void __launch_bounds__(kThreads, 1) hex_kernel(const __grid_constant__ HexDev p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int R = p.rows;
  // layout (doubles): mats | stage[2] = {G: 9 * NE * P3, U: R * NE * P3} | T[3] | Q | W0 | W1 | Yacc
  double* mats = sm;                                  // 6 * 75
  double* stage0 = mats + 6 * ND * P * P;
  const int g_len = ND * ND * NE * P3, u_len = R * NE * P3, stage_len = g_len + u_len;
  const int blk = NE * R * P3;                        // one (element pair x fields) cube set
  double* T = stage0 + 2 * stage_len;
  double* Q = T + ND * blk;
  double* W0 = Q + blk;
  double* W1 = W0 + blk;
  double* Yacc = W1 + blk;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(Yacc + blk);

  for (int t = threadIdx.x; t < 6 * ND * P * P; t += blockDim.x) mats[t] = __ldg(p.mats[t / (ND * P * P)] + t % (ND * P * P));
  if (threadIdx.x == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const std::int64_t npairs = p.E / NE;
  const std::uint32_t bytes = static_cast<std::uint32_t>(NE * P3 * 8);
  auto issue = [&](std::int64_t pair, int s) {
    double* st = stage0 + s * stage_len;
    ptx::mbar_arrive_expect_tx(&full[s], bytes * static_cast<std::uint32_t>(ND * ND + R));
    const std::int64_t e0 = pair * NE;
    for (int xy = 0; xy < ND * ND; ++xy)
      ptx::bulk_g2s(st + xy * NE * P3, p.G + (xy * p.E + e0) * P3, bytes, &full[s]);
    for (int f = 0; f < R; ++f) ptx::bulk_g2s(st + g_len + f * NE * P3, p.U[f] + e0 * P3, bytes, &full[s]);
  };
  if (threadIdx.x == 0 && blockIdx.x < npairs) issue(blockIdx.x, 0);

  int it = 0;
  for (std::int64_t pair = blockIdx.x; pair < npairs; pair += gridDim.x, ++it) {
    const int s = it & 1;
    ptx::mbar_wait(&full[s], static_cast<std::uint32_t>((it >> 1) & 1));
    // prefetch the next pair into the other stage (its previous contents were
    // consumed before the last __syncthreads of the previous iteration)
    if (threadIdx.x == 0 && pair + gridDim.x < npairs) issue(pair + gridDim.x, s ^ 1);
    const double* G = stage0 + s * stage_len;  // [x*3+y][el][125]
    const double* U = G + g_len;               // [f][el][125]

    // forward sweeps: T[y] = F1[y] (x) F2[y] (x) F3[y] applied to u
    for (int y = 0; y < ND; ++y) {
      sweep<false>(U, NE * P3, P3, W0, mats + (2 * ND + y) * P * P, 2, R, false);  // F3 along l
      __syncthreads();
      sweep<false>(W0, P3, R * P3, W1, mats + (1 * ND + y) * P * P, 1, R, false);      // F2 along k
      __syncthreads();
      sweep<false>(W1, P3, R * P3, T + y * blk, mats + (0 * ND + y) * P * P, 0, R, false);  // F1 along j
      __syncthreads();
    }
    // geometric factors and backward sweeps, one direction x at a time
    for (int x = 0; x < ND; ++x) {
      for (int t = threadIdx.x; t < blk; t += blockDim.x) {
        const int pt = t % P3, ef = t / P3, el = ef / R;
        double q = 0.0;
#pragma unroll
        for (int y = 0; y < ND; ++y) q = fma(G[((x * ND + y) * NE + el) * P3 + pt], T[y * blk + t], q);
        Q[t] = q;
      }
      __syncthreads();
      sweep<true>(Q, P3, R * P3, W0, mats + (3 * ND + 0 * ND + x) * P * P, 0, R, false);  // B1^T: a -> i
      __syncthreads();
      sweep<true>(W0, P3, R * P3, W1, mats + (3 * ND + 1 * ND + x) * P * P, 1, R, false);  // B2^T: b -> m
      __syncthreads();
      sweep<true>(W1, P3, R * P3, Yacc, mats + (3 * ND + 2 * ND + x) * P * P, 2, R, x > 0);  // B3^T: c -> n
      __syncthreads();
    }
    // results: field f of this pair is the 250-double run Yacc[(el*R+f)*125 ...]
    const std::int64_t e0 = pair * NE;
    for (int t = threadIdx.x; t < blk; t += blockDim.x) {
      const int pt = t % P3, ef = t / P3, el = ef / R, f = ef % R;
      __stcs(p.Y[f] + (e0 + el) * P3 + pt, Yacc[t]);
    }
    __syncthreads();
  }
}

}  // namespace

bool hex_supported(int nd, int p, std::int64_t E, int rows) {
  return nd == ND && p == P && E % NE == 0 && rows >= 1 && rows <= kMaxFields;
}

int launch_hex(const HexLaunch& L, void* stream) {
  if (!hex_supported(L.ND, L.P, L.E, L.rows)) return cudaErrorInvalidValue;
  if (L.E == 0) return cudaSuccess;
  HexDev d{};
  d.E = L.E;
  d.rows = L.rows;
  d.G = L.G;
  for (int f = 0; f < L.rows; ++f) {
    d.U[f] = L.U[f];
    d.Y[f] = L.Y[f];
  }
  for (int k = 0; k < 6; ++k) d.mats[k] = L.mats[k];
  const int R = L.rows;
  const size_t doubles = 6 * ND * P * P + 2 * (ND * ND * NE * P3 + R * NE * P3) + (ND + 4) * NE * R * P3;
  const size_t smem = doubles * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(hex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 148;
  device_sm_count(&sms);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hex_kernel, kThreads, smem);
  std::int64_t grid = static_cast<std::int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
  if (grid > L.E / NE) grid = L.E / NE;
  hex_kernel<<<static_cast<int>(grid), kThreads, smem, static_cast<cudaStream_t>(stream)>>>(d);
  return cudaGetLastError();
}

}  // namespace feb200
