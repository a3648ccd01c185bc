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
// registers (two sweeps per pass where the plane contains both axes), with the
// three directions and all fields of the pair in flight at once (240 plane
// tasks for 256 threads), four CTA barriers per pair. Work cubes are padded to
// rows of 6 doubles so every plane row moves as two 16-byte + one 8-byte
// shared access, and lanes are assigned cube-fastest so that 8 consecutive
// lanes' 16-byte accesses cover all 32 banks. 5x5 operators are too small for
// DMMA tiles (padding to 8x8 wastes 61%).
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int P = 5;              // points / dofs per direction
constexpr int P2 = P * P;         // 25
constexpr int P3 = P * P * P;     // 125
constexpr int RW = 6;             // padded row (16-byte multiple)
constexpr int PL = P * RW;        // padded plane: 30 doubles
constexpr int CB = P * PL;        // padded cube: 150 doubles (1200 B)
constexpr int MS = 26;            // padded 5x5 operator stride (16-byte multiple)
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

// 5x5 operator into registers (13 x 16-byte shared loads)
__device__ __forceinline__ void load_op(const double* m, double (&c)[MS]) {
#pragma unroll
  for (int k = 0; k < MS; k += 2) {
    const double2 v = *reinterpret_cast<const double2*>(m + k);
    c[k] = v.x;
    c[k + 1] = v.y;
  }
}

__device__ __forceinline__ void load_row(const double* p, double (&r)[P]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  r[0] = a.x;
  r[1] = a.y;
  r[2] = b.x;
  r[3] = b.y;
  r[4] = p[4];
}

__device__ __forceinline__ void store_row(double* p, const double (&r)[P]) {
  *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(r[2], r[3]);
  p[4] = r[4];
}

// forward operator entry M[o][i] = F[o][i]; backward M[o][i] = B[i][o]
template <bool kBack>
__device__ __forceinline__ double op(const double (&c)[MS], int o, int i) {
  return kBack ? c[i * P + o] : c[o * P + i];
}

// v[r][.] <- M v[r][.] for every row r (contract the fast axis)
template <bool kBack>
__device__ __forceinline__ void rows5(double (&v)[P][P], const double (&c)[MS]) {
#pragma unroll
  for (int r = 0; r < P; ++r) {
    double o[P];
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < P; ++b) s = fma(op<kBack>(c, a, b), v[r][b], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < P; ++a) v[r][a] = o[a];
  }
}

// v[.][c] <- M v[.][c] for every column c (contract the slow axis)
template <bool kBack>
__device__ __forceinline__ void cols5(double (&v)[P][P], const double (&c)[MS]) {
#pragma unroll
  for (int col = 0; col < P; ++col) {
    double o[P];
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < P; ++b) s = fma(op<kBack>(c, a, b), v[b][col], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < P; ++a) v[a][col] = o[a];
  }
}

__global__ void __launch_bounds__(kThreads, 2) hex_kernel(const __grid_constant__ HexDev p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int R = p.rows;
  const int nblk = NE * R;  // (element, field) cubes per pair
  // layout (doubles): ops[6][ND][MS] | Gs[9][NE*P3] | Us[R][NE*P3] | W[ND][nblk][CB] | mbar {G, U}
  double* ops = sm;
  double* Gs = ops + 6 * ND * MS;
  const int g_len = ND * ND * NE * P3;
  double* Us = Gs + g_len;
  double* W = Us + R * NE * P3;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(W + ND * nblk * CB);

  for (int t = threadIdx.x; t < 6 * ND * MS; t += blockDim.x) {
    const int k = t / (ND * MS), d = (t / MS) % ND, e = t % MS;
    ops[t] = e < P2 ? __ldg(p.mats[k] + d * P2 + e) : 0.0;
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const std::int64_t npairs = p.E / NE;
  const std::uint32_t bytes = static_cast<std::uint32_t>(NE * P3 * 8);
  // G and U have separate single-buffered slots: each is refilled for the
  // next pair as soon as the pass that consumes it is done (U after pass 1,
  // G after the combine), so the copies overlap the remaining passes and the
  // second CTA on the SM covers what is left.
  auto issue_g = [&](std::int64_t pair) {
    ptx::mbar_arrive_expect_tx(&bar[0], bytes * static_cast<std::uint32_t>(ND * ND));
    const std::int64_t e0 = pair * NE;
    for (int xy = 0; xy < ND * ND; ++xy)
      ptx::bulk_g2s(Gs + xy * NE * P3, p.G + (xy * p.E + e0) * P3, bytes, &bar[0]);
  };
  auto issue_u = [&](std::int64_t pair) {
    ptx::mbar_arrive_expect_tx(&bar[1], bytes * static_cast<std::uint32_t>(R));
    const std::int64_t e0 = pair * NE;
    for (int f = 0; f < R; ++f) ptx::bulk_g2s(Us + f * NE * P3, p.U[f] + e0 * P3, bytes, &bar[1]);
  };
  if (threadIdx.x == 0 && blockIdx.x < npairs) {
    issue_u(blockIdx.x);
    issue_g(blockIdx.x);
  }

  // plane task: direction d, plane index pl, cube blk = el*R + f (cube fastest)
  const int ntask = ND * P * nblk;
  const int task = threadIdx.x;
  const bool active = task < ntask;
  const int d = task / (P * nblk);
  const int pl = (task / nblk) % P;
  const int blk = task % nblk;
  const int el = blk / R, f = blk % R;
  const double* opF1 = ops + (0 * ND + d) * MS;
  const double* opF2 = ops + (1 * ND + d) * MS;
  const double* opF3 = ops + (2 * ND + d) * MS;
  const double* opB1 = ops + (3 * ND + d) * MS;
  const double* opB2 = ops + (4 * ND + d) * MS;
  const double* opB3 = ops + (5 * ND + d) * MS;
  double* cube = W + (d * nblk + blk) * CB;  // this task's direction cube

  int it = 0;
  for (std::int64_t pair = blockIdx.x; pair < npairs; pair += gridDim.x, ++it) {
    const std::uint32_t phase = static_cast<std::uint32_t>(it & 1);
    const bool more = pair + gridDim.x < npairs;
    double v[P][P];
    double c[MS];

    // pass 1 (direction y = d, plane j = pl): F3 along l, F2 along k
    ptx::mbar_wait(&bar[1], phase);
    if (active) {
      const double* in = Us + (f * NE + el) * P3 + pl * P2;
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int l = 0; l < P; ++l) v[k][l] = in[k * P + l];
      load_op(opF3, c);
      rows5<false>(v, c);
      load_op(opF2, c);
      cols5<false>(v, c);
      double* out = cube + pl * PL;  // [j][b][c]
#pragma unroll
      for (int b = 0; b < P; ++b) store_row(out + b * RW, v[b]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && more) issue_u(pair + gridDim.x);
    // pass 2 (direction y = d, plane b = pl), in place: F1 along j -> t_y[a][b][c]
    if (active) {
      double* io = cube + pl * RW;
#pragma unroll
      for (int j = 0; j < P; ++j) load_row(io + j * PL, v[j]);
      load_op(opF1, c);
      cols5<false>(v, c);
#pragma unroll
      for (int a = 0; a < P; ++a) store_row(io + a * PL, v[a]);
    }
    __syncthreads();
    // pass 3a (direction x = d, plane b = pl): q_x = sum_y G[x,y] t_y into registers
    ptx::mbar_wait(&bar[0], phase);
    if (active) {
      const double* g = Gs + (d * ND * NE + el) * P3 + pl * P;
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double t0[P], t1[P], t2[P];
        load_row(W + (0 * nblk + blk) * CB + a * PL + pl * RW, t0);
        load_row(W + (1 * nblk + blk) * CB + a * PL + pl * RW, t1);
        load_row(W + (2 * nblk + blk) * CB + a * PL + pl * RW, t2);
#pragma unroll
        for (int cc = 0; cc < P; ++cc) {
          double q = g[a * P2 + cc] * t0[cc];
          q = fma(g[NE * P3 + a * P2 + cc], t1[cc], q);
          v[a][cc] = fma(g[2 * NE * P3 + a * P2 + cc], t2[cc], q);
        }
      }
    }
    __syncthreads();  // every t_y and G read
    if (threadIdx.x == 0 && more) issue_g(pair + gridDim.x);
    // pass 3b, in place: B1^T along a -> i
    if (active) {
      load_op(opB1, c);
      cols5<true>(v, c);
      double* out = cube + pl * RW;  // [i][b][c]
#pragma unroll
      for (int i = 0; i < P; ++i) store_row(out + i * PL, v[i]);
    }
    __syncthreads();
    // pass 4 (direction x = d, plane i = pl), in place: B2^T along b -> m, B3^T along c -> n
    if (active) {
      double* io = cube + pl * PL;
#pragma unroll
      for (int b = 0; b < P; ++b) load_row(io + b * RW, v[b]);
      load_op(opB2, c);
      cols5<true>(v, c);
      load_op(opB3, c);
      rows5<true>(v, c);
#pragma unroll
      for (int m = 0; m < P; ++m) store_row(io + m * RW, v[m]);  // partial y_x[i][m][n]
    }
    __syncthreads();
    // sum the three direction partials row by row (one padded row of 5 per
    // task, vector shared loads, no per-point index arithmetic); consecutive
    // tasks write consecutive rows of one cube
    const std::int64_t e0 = pair * NE;
    for (int t = threadIdx.x; t < nblk * P2; t += blockDim.x) {
      const int b2 = t / P2, row = t - b2 * P2;  // row = i*5 + m
      const int off = b2 * CB + (row / P) * PL + (row % P) * RW;
      double r0[P], r1[P], r2[P];
      load_row(W + off, r0);
      load_row(W + nblk * CB + off, r1);
      load_row(W + 2 * nblk * CB + off, r2);
      const int ee = b2 / R, ff = b2 - ee * R;
      double* y = p.Y[ff] + (e0 + ee) * P3 + row * P;
#pragma unroll
      for (int n = 0; n < P; ++n) __stcs(y + n, r0[n] + r1[n] + r2[n]);
    }
    __syncthreads();  // W is rewritten by the next pair's pass 1
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
  const size_t doubles = 6 * ND * MS + ND * ND * NE * P3 + R * NE * P3 + ND * NE * R * CB;
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
