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
// B200 design: persistent CTAs walk element PAIRS (a pair of 125-double blocks
// is a 16-byte-aligned 2000-byte run, the unit of a 1-D bulk copy). One thread
// streams the pair's 9 G blocks and every field's u block with cp.async.bulk
// into a double-buffered mbarrier ring, so G — the dominant traffic — is read
// from HBM once and reused by all fields while the next pair is in flight.
// The sweeps run on the FP64 pipe in four passes over 25-value planes held in
// registers (two sweeps per pass where the plane contains both axes), with
// the three directions and all fields of the pair in flight at once
// (3 x 2 x 8 x 5 = 240 plane tasks per pass for 256 threads), so one pair
// needs four CTA barriers. 5x5 operators are too small for DMMA tiles
// (padding to 8x8 wastes 61%).
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int P = 5;              // points / dofs per direction
constexpr int P2 = P * P;         // 25
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

// forward operator entry M[o][i] = F[o][i]; backward M[o][i] = B[i][o]
template <bool kBack>
__device__ __forceinline__ double op(const double* m, int o, int i) {
  return kBack ? m[i * P + o] : m[o * P + i];
}

// v[r][.] <- M v[r][.] for every row r (contract the fast axis)
template <bool kBack>
__device__ __forceinline__ void rows5(double (&v)[P][P], const double* m) {
#pragma unroll
  for (int r = 0; r < P; ++r) {
    double o[P];
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < P; ++b) s = fma(op<kBack>(m, a, b), v[r][b], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < P; ++a) v[r][a] = o[a];
  }
}

// v[.][c] <- M v[.][c] for every column c (contract the slow axis)
template <bool kBack>
__device__ __forceinline__ void cols5(double (&v)[P][P], const double* m) {
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double o[P];
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < P; ++b) s = fma(op<kBack>(m, a, b), v[b][c], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < P; ++a) v[a][c] = o[a];
  }
}

__global__ void __launch_bounds__(kThreads, 1) hex_kernel(const __grid_constant__ HexDev p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int R = p.rows;
  const int nblk = NE * R;                            // (element, field) cubes per pair
  // layout (doubles): mats | stage[2] = {G: 9*NE*P3, U: R*NE*P3} | WA[ND][nblk][P3] | WB[ND][nblk][P3]
  double* mats = sm;                                  // 6 * ND * 25
  double* stage0 = mats + 6 * ND * P2;
  const int g_len = ND * ND * NE * P3, stage_len = g_len + R * NE * P3;
  double* WA = stage0 + 2 * stage_len;
  double* WB = WA + ND * nblk * P3;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(WB + ND * nblk * P3);

  for (int t = threadIdx.x; t < 6 * ND * P2; t += blockDim.x) mats[t] = __ldg(p.mats[t / (ND * P2)] + t % (ND * P2));
  if (threadIdx.x == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const double* F1 = mats;
  const double* F2 = mats + ND * P2;
  const double* F3 = mats + 2 * ND * P2;
  const double* B1 = mats + 3 * ND * P2;
  const double* B2 = mats + 4 * ND * P2;
  const double* B3 = mats + 5 * ND * P2;

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

  // plane task of this thread: direction d, cube blk = el*R + f, plane index pl
  const int ntask = ND * nblk * P;
  const int task = threadIdx.x;
  const bool active = task < ntask;
  const int d = task / (nblk * P);
  const int blk = (task / P) % nblk;
  const int pl = task % P;
  const int el = blk / R, f = blk % R;

  int it = 0;
  for (std::int64_t pair = blockIdx.x; pair < npairs; pair += gridDim.x, ++it) {
    const int s = it & 1;
    ptx::mbar_wait(&full[s], static_cast<std::uint32_t>((it >> 1) & 1));
    if (threadIdx.x == 0 && pair + gridDim.x < npairs) issue(pair + gridDim.x, s ^ 1);
    const double* G = stage0 + s * stage_len;  // [x*3+y][el][125]
    const double* U = G + g_len;               // [f][el][125]
    double v[P][P];

    // pass 1 (direction y = d, plane j = pl): F3 along l, F2 along k
    if (active) {
      const double* in = U + (f * NE + el) * P3 + pl * P2;
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int l = 0; l < P; ++l) v[k][l] = in[k * P + l];
      rows5<false>(v, F3 + d * P2);
      cols5<false>(v, F2 + d * P2);
      double* out = WA + (d * nblk + blk) * P3 + pl * P2;  // [j][b][c]
#pragma unroll
      for (int b = 0; b < P; ++b)
#pragma unroll
        for (int c = 0; c < P; ++c) out[b * P + c] = v[b][c];
    }
    __syncthreads();
    // pass 2 (direction y = d, plane b = pl): F1 along j -> t_y[a][b][c]
    if (active) {
      const double* in = WA + (d * nblk + blk) * P3 + pl * P;
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int c = 0; c < P; ++c) v[j][c] = in[j * P2 + c];
      cols5<false>(v, F1 + d * P2);
      double* out = WB + (d * nblk + blk) * P3 + pl * P;
#pragma unroll
      for (int a = 0; a < P; ++a)
#pragma unroll
        for (int c = 0; c < P; ++c) out[a * P2 + c] = v[a][c];
    }
    __syncthreads();
    // pass 3 (direction x = d, plane b = pl): q_x = sum_y G[x,y] t_y, B1^T along a -> i
    if (active) {
#pragma unroll
      for (int a = 0; a < P; ++a)
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const int pt = a * P2 + pl * P + c;
          double q = 0.0;
#pragma unroll
          for (int y = 0; y < ND; ++y)
            q = fma(G[((d * ND + y) * NE + el) * P3 + pt], WB[(y * nblk + blk) * P3 + pt], q);
          v[a][c] = q;
        }
      cols5<true>(v, B1 + d * P2);
      double* out = WA + (d * nblk + blk) * P3 + pl * P;  // [i][b][c]
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int c = 0; c < P; ++c) out[i * P2 + c] = v[i][c];
    }
    __syncthreads();
    // pass 4 (direction x = d, plane i = pl): B2^T along b -> m, B3^T along c -> n
    if (active) {
      const double* in = WA + (d * nblk + blk) * P3 + pl * P2;
#pragma unroll
      for (int b = 0; b < P; ++b)
#pragma unroll
        for (int c = 0; c < P; ++c) v[b][c] = in[b * P + c];
      cols5<true>(v, B2 + d * P2);
      rows5<true>(v, B3 + d * P2);
      double* out = WB + (d * nblk + blk) * P3 + pl * P2;  // partial y_x[i][m][n]
#pragma unroll
      for (int m = 0; m < P; ++m)
#pragma unroll
        for (int n = 0; n < P; ++n) out[m * P + n] = v[m][n];
    }
    __syncthreads();
    // sum the three direction partials and store (consecutive threads write
    // consecutive doubles of one field's pair run)
    const std::int64_t e0 = pair * NE;
    for (int t = threadIdx.x; t < nblk * P3; t += blockDim.x) {
      const int ff = t / (NE * P3), rem = t % (NE * P3);
      const int ee = rem / P3, pt = rem % P3;
      const int b2 = ee * R + ff;
      const double y = WB[b2 * P3 + pt] + WB[(nblk + b2) * P3 + pt] + WB[(2 * nblk + b2) * P3 + pt];
      __stcs(p.Y[ff] + e0 * P3 + rem, y);
    }
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
  const size_t doubles = 6 * ND * P2 + 2 * (ND * ND * NE * P3 + R * NE * P3) + 2 * ND * NE * R * P3;
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
