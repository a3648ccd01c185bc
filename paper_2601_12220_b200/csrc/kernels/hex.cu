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
// Three kernels. v1 (hex_kernel, meta v=1): register-plane passes with the
// 5x5 operators loaded from shared memory. hex2_kernel (meta v=3, and the
// default below eight fields, see the comment above it): operators in the
// constant bank, pass ownership matched to the sweeps (planes / lines /
// planes), four elements per stage, three CTA barriers per stage. hex5_kernel
// (the default for eight fields, C2): hex2 with pass C of stage s and pass A
// of stage s+1 merged into one barrier-free segment (two barriers per stage),
// pass-B tasks field pair fastest; bitwise equal to hex2.
//
// Common to both: persistent CTAs walk element stages (2 or 4 elements = one
// contiguous bulk-copy run per array); one thread streams the stage's 9 G
// blocks and every field's u block with cp.async.bulk into mbarrier-tracked
// slots that are refilled as soon as the pass that consumes them is done, so
// G — the dominant traffic — is read from HBM once and reused by all fields.
// 5x5 operators are too small for DMMA tiles (padding to 8x8 wastes 61%): the
// sweeps run on the FP64 FMA pipe.
#include <cuda_runtime.h>

#include <mutex>

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

// ---------------------------------------------------------------- v2 -----
// Constant-bank operators and ownership that matches each pass to its sweeps.
//
// The 1-D operators live in constant memory (staged per launch, stream-ordered)
// and every sweep is unrolled for a compile-time (matrix, direction), so each
// DFMA takes its coefficient straight from the constant bank: no operator
// loads, no operator registers. Shared memory then only carries the three
// unavoidable transposes per (element, field):
//   A  plane j (k,l) of u, one direction y per warp:  F3[y] along l, F2[y] along k
//   B  line (k,l) over j, two fields per thread:      F1[y] along j, q_x = G t_y,
//                                                      B1[x]^T along a (G read once per two fields)
//   C  plane i (b,c), one direction x per warp:       B2[x]^T along b, B3[x]^T along c
//   S  y = sum_x partial_x into a staging tile, one bulk store per field
// At Q = 5: 3187 shared doubles per (element, field) against 12375 DFMA (v1:
// 5250 plus operator loads). Work cubes (cube = field * NE + element) sit CS
// doubles apart: odd, so the plane accesses of cube-fastest lanes in A and C
// hit distinct banks, and (where Q^2 is odd) CS = Q^2 mod 16 so consecutive
// line groups of B continue the bank walk. The kernel is templated on the
// number of points per direction Q (3..6: P2..P5 hex elements).
constexpr int kMaxQ = 6;
// F1 F2 F3 B1 B2 B3 packed as stored: matrix k, direction d, entry (o, i) at
// (k * ND + d) * Q^2 + o * Q + i (one copy per matrix per launch)
__constant__ double c_hex_ops[6 * ND * kMaxQ * kMaxQ];
__constant__ float c_hex_ops_f[6 * ND * kMaxQ * kMaxQ];  // the fp32 instance's copy

template <int Q>
struct Hx {
  static constexpr int Q2 = Q * Q, Q3 = Q * Q * Q;
  static constexpr int CS = Q == 3 ? 41 : Q == 4 ? 65 : Q == 5 ? 137 : 217;
  static_assert(CS >= Q3 && CS % 2 == 1, "cube stride");
};

struct Hex2Dev {
  std::int64_t E;
  int rows;
  const double* G;
  const double* U[kMaxFields];
  double* Y[kMaxFields];
};

// forward operator entry M[o][i] = F[o][i]; backward M[o][i] = B[i][o]
template <typename T, int Q, int K, int D, bool kBack>
__device__ __forceinline__ T cop(int o, int i) {
  constexpr int base = (K * ND + D) * Q * Q;
  const int at = kBack ? base + i * Q + o : base + o * Q + i;
  if constexpr (sizeof(T) == 4)
    return c_hex_ops_f[at];
  else
    return c_hex_ops[at];
}

template <typename T, int Q, int K, int D, bool kBack>
__device__ __forceinline__ void rows_c(T (&v)[Q][Q]) {
#pragma unroll
  for (int r = 0; r < Q; ++r) {
    T o[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      T s = cop<T, Q, K, D, kBack>(a, 0) * v[r][0];
#pragma unroll
      for (int b = 1; b < Q; ++b) s = fma(cop<T, Q, K, D, kBack>(a, b), v[r][b], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) v[r][a] = o[a];
  }
}

template <typename T, int Q, int K, int D, bool kBack>
__device__ __forceinline__ void cols_c(T (&v)[Q][Q]) {
#pragma unroll
  for (int col = 0; col < Q; ++col) {
    T o[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      T s = cop<T, Q, K, D, kBack>(a, 0) * v[0][col];
#pragma unroll
      for (int b = 1; b < Q; ++b) s = fma(cop<T, Q, K, D, kBack>(a, b), v[b][col], s);
      o[a] = s;
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) v[a][col] = o[a];
  }
}

// pass A: u plane j -> t_y plane j (F3[y] along l, F2[y] along k)
template <typename T, int Q, int Y>
__device__ __forceinline__ void pass_a(const T* in, T* out) {
  T v[Q][Q];
#pragma unroll
  for (int k = 0; k < Q; ++k)
#pragma unroll
    for (int l = 0; l < Q; ++l) v[k][l] = in[k * Q + l];
  rows_c<T, Q, 2, Y, false>(v);
  cols_c<T, Q, 1, Y, false>(v);
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int c = 0; c < Q; ++c) out[b * Q + c] = v[b][c];
}

// pass C: q'_x plane i -> partial y_x plane i (B2[x]^T along b, B3[x]^T along c)
template <typename T, int Q, int X>
__device__ __forceinline__ void pass_c(T* io) {
  T v[Q][Q];
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int c = 0; c < Q; ++c) v[b][c] = io[b * Q + c];
  cols_c<T, Q, 4, X, true>(v);
  rows_c<T, Q, 5, X, true>(v);
#pragma unroll
  for (int m = 0; m < Q; ++m)
#pragma unroll
    for (int n = 0; n < Q; ++n) io[m * Q + n] = v[m][n];
}

// pass C with the direction sum fused (one warp per (direction, plane), the
// plane's three direction warps chained by named barriers): x = 0 stores its
// partial into the staging tile, x = 1 adds its own after x = 0's arrive, x =
// 2 after x = 1's — (p0 + p1) + p2, the order the separate sum pass used, so
// the output is unchanged. No partials in W, no extra pass, no CTA barrier.
// Chain barriers b0 (x = 0 -> 1) and b0 + 1 (x = 1 -> 2); every lane of the
// warp takes part (bar is warp-aligned), lanes without a task compute on
// zeros and store nothing.
template <typename T, int Q, int X>
__device__ __forceinline__ void pass_c_sum(const T* in, T* ys, int b0, bool active) {
  T v[Q][Q];
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int c = 0; c < Q; ++c) v[b][c] = active ? in[b * Q + c] : 0.0;
  cols_c<T, Q, 4, X, true>(v);
  rows_c<T, Q, 5, X, true>(v);
  if constexpr (X > 0) asm volatile("bar.sync %0, 64;" ::"r"(b0 + X - 1) : "memory");
  if (active) {
#pragma unroll
    for (int m = 0; m < Q; ++m)
#pragma unroll
      for (int n = 0; n < Q; ++n) ys[m * Q + n] = X == 0 ? v[m][n] : ys[m * Q + n] + v[m][n];
  }
  if constexpr (X < 2) asm volatile("bar.arrive %0, 64;" ::"r"(b0 + X) : "memory");
}

// F1[y] along j on one line (y compile-time)
template <typename T, int Q, int Y>
__device__ __forceinline__ void line_f1(T (&t)[Q]) {
  T o[Q];
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    T s = cop<T, Q, 0, Y, false>(a, 0) * t[0];
#pragma unroll
    for (int j = 1; j < Q; ++j) s = fma(cop<T, Q, 0, Y, false>(a, j), t[j], s);
    o[a] = s;
  }
#pragma unroll
  for (int a = 0; a < Q; ++a) t[a] = o[a];
}

// B1[x]^T along a on one line, stored with stride Q^2
template <typename T, int Q, int X>
__device__ __forceinline__ void line_b1(const T (&t)[Q], T* out) {
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    T s = cop<T, Q, 3, X, true>(i, 0) * t[0];
#pragma unroll
    for (int a = 1; a < Q; ++a) s = fma(cop<T, Q, 3, X, true>(i, a), t[a], s);
    out[i * Hx<Q>::Q2] = s;
  }
}

// pass B on line (k,l) of NF fields: wl[f] = W + cube*CS + kl (direction 0),
// direction stride ds; g = Gs + el*Q3 + kl with (x,y) block stride gs
template <typename T, int Q, int NF>
__device__ __forceinline__ void pass_b(T* const (&wl)[NF], int ds, const T* g, int gs) {
  constexpr int Q2 = Hx<Q>::Q2;
  T t[NF][ND][Q];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int y = 0; y < ND; ++y)
#pragma unroll
      for (int j = 0; j < Q; ++j) t[f][y][j] = wl[f][y * ds + j * Q2];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    line_f1<T, Q, 0>(t[f][0]);
    line_f1<T, Q, 1>(t[f][1]);
    line_f1<T, Q, 2>(t[f][2]);
  }
  // q_x = sum_y G[x,y] t_y, pointwise; G read once for all NF fields
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    T gv[ND][ND];
#pragma unroll
    for (int x = 0; x < ND; ++x)
#pragma unroll
      for (int y = 0; y < ND; ++y) gv[x][y] = g[(x * ND + y) * gs + a * Q2];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      T q[ND];
#pragma unroll
      for (int x = 0; x < ND; ++x) {
        T s = gv[x][0] * t[f][0][a];
        s = fma(gv[x][1], t[f][1][a], s);
        q[x] = fma(gv[x][2], t[f][2][a], s);
      }
#pragma unroll
      for (int x = 0; x < ND; ++x) t[f][x][a] = q[x];
    }
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    line_b1<T, Q, 0>(t[f][0], wl[f]);
    line_b1<T, Q, 1>(t[f][1], wl[f] + ds);
    line_b1<T, Q, 2>(t[f][2], wl[f] + 2 * ds);
  }
}

// threads: the plane passes' 3 x NE x 8 x Q tasks (direction-major, so every
// direction's tasks fill whole warps: at Q = 5, NE = 4 exactly five warps
// each) plus one warp for the copy engine, idle in passes A and C
template <int Q, int NE2>
struct HexCfg {
  static constexpr int kTasks = ND * NE2 * kMaxFields * Q;
  static constexpr int kThreads = (kTasks + 31) / 32 * 32 + 32;
};

template <typename T, int Q, int NE2>
__global__ void __launch_bounds__(HexCfg<Q, NE2>::kThreads, 1) hex2_kernel(const __grid_constant__ Hex2Dev p) {
  constexpr int NE = NE2;
  constexpr int Q2 = Hx<Q>::Q2, Q3 = Hx<Q>::Q3, CS = Hx<Q>::CS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const T* const pG = reinterpret_cast<const T*>(p.G);
  const int R = p.rows;
  const int nblk = NE * R;   // cubes per stage, cube = field * NE + element
  const int ds = nblk * CS;  // direction stride in W
  // layout (doubles): Gs[9][NE*Q3] | Us[R][NE*Q3] | W[ND][nblk][CS] | Ys[R][NE*Q3] | mbar {G, U}
  T* Gs = sm;
  T* Us = Gs + ND * ND * NE * Q3;
  T* W = Us + R * NE * Q3;
  T* Ys = W + ND * ds;  // output staging: one bulk store per field and stage
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
      (reinterpret_cast<std::uintptr_t>(Ys + R * NE * Q3) + 7) & ~std::uintptr_t{7});
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const std::int64_t nstages = p.E / NE;
  const std::uint32_t bytes = static_cast<std::uint32_t>(NE * Q3 * sizeof(T));
  auto issue_g = [&](std::int64_t st) {
    ptx::mbar_arrive_expect_tx(&bar[0], bytes * static_cast<std::uint32_t>(ND * ND));
    const std::int64_t e0 = st * NE;
    for (int xy = 0; xy < ND * ND; ++xy)
      ptx::bulk_g2s(Gs + xy * NE * Q3, pG + (xy * p.E + e0) * Q3, bytes, &bar[0]);
  };
  auto issue_u = [&](std::int64_t st) {
    ptx::mbar_arrive_expect_tx(&bar[1], bytes * static_cast<std::uint32_t>(R));
    const std::int64_t e0 = st * NE;
    for (int f = 0; f < R; ++f) ptx::bulk_g2s(Us + f * NE * Q3, reinterpret_cast<const T*>(p.U[f]) + e0 * Q3, bytes, &bar[1]);
  };
  // the copy engine is driven by lane 0 of the last warp, which has no work in
  // passes A / C and none in B at the pinned config, so issuing the next
  // stage's copies never delays a computing warp
  const bool producer = threadIdx.x == blockDim.x - 32;
  if (producer && blockIdx.x < nstages) {
    issue_u(blockIdx.x);
    issue_g(blockIdx.x);
  }

  // passes A and C: thread -> (direction, cube, plane), direction slowest
  const int dir = threadIdx.x / (nblk * Q);
  const int ptask = threadIdx.x - dir * nblk * Q;
  const bool pactive = dir < ND && threadIdx.x < blockDim.x - 32;
  const int pplane = ptask / nblk, pcube = ptask - pplane * nblk;  // cube fastest
  const T* a_in = Us + pcube * Q3 + pplane * Q2;
  T* a_out = W + dir * ds + pcube * CS + pplane * Q2;
  // pass B: thread -> (line, element, field pair (f, f + H)), line fastest
  const int H = (R + 1) / 2;
  const int nbt = H * NE * Q2;
  // every warp of pass C one (direction, plane): fuse the direction sum
  const bool fused = nblk == 32 && Q <= 7;

  int it = 0;
  for (std::int64_t st = blockIdx.x; st < nstages; st += gridDim.x, ++it) {
    const std::uint32_t phase = static_cast<std::uint32_t>(it & 1);
    const bool more = st + gridDim.x < nstages;

    ptx::mbar_wait(&bar[1], phase);
    if (pactive) {
      if (dir == 0) pass_a<T, Q, 0>(a_in, a_out);
      else if (dir == 1) pass_a<T, Q, 1>(a_in, a_out);
      else pass_a<T, Q, 2>(a_in, a_out);
    }
    __syncthreads();
    if (producer && more) issue_u(st + gridDim.x);

    ptx::mbar_wait(&bar[0], phase);
    for (int t = threadIdx.x; t < nbt; t += blockDim.x) {
      const int kl = t % Q2;
      const int r = t / Q2;
      const int el = r % NE, f0 = r / NE, f1 = f0 + H;
      const T* g = Gs + el * Q3 + kl;
      // odd R: the last thread pairs its field with itself (same values
      // written twice by the same thread) — one code path, smaller kernel
      T* const w0 = W + (f0 * NE + el) * CS + kl;
      T* const wl[2] = {w0, f1 < R ? W + (f1 * NE + el) * CS + kl : w0};
      pass_b<T, Q, 2>(wl, ds, g, NE * Q3);
    }
    if (producer) ptx::bulk_wait_read<0>();  // the previous stage's stores have read Ys
    __syncthreads();
    if (producer && more) issue_g(st + gridDim.x);

    const std::int64_t e0 = st * NE;
    if (fused) {
      if (pactive) {
        T* ys = Ys + pcube * Q3 + pplane * Q2;  // cube * Q3 = field * NE * Q3 + element * Q3
        if (dir == 0) pass_c_sum<T, Q, 0>(a_out, ys, 1 + 2 * pplane, true);
        else if (dir == 1) pass_c_sum<T, Q, 1>(a_out, ys, 1 + 2 * pplane, true);
        else pass_c_sum<T, Q, 2>(a_out, ys, 1 + 2 * pplane, true);
      }
      ptx::fence_proxy_async();
      __syncthreads();  // W is rewritten by the next stage's pass A; Ys complete
      if (producer) {
        for (int f = 0; f < R; ++f) ptx::bulk_s2g(reinterpret_cast<T*>(p.Y[f]) + e0 * Q3, Ys + f * NE * Q3, bytes);
        ptx::bulk_commit();
      }
      continue;
    }
    if (pactive) {
      if (dir == 0) pass_c<T, Q, 0>(a_out);
      else if (dir == 1) pass_c<T, Q, 1>(a_out);
      else pass_c<T, Q, 2>(a_out);
    }
    __syncthreads();

    // sum the three direction partials into the staging tile (a field's
    // stage output is one contiguous run of NE * Q3 doubles), then one bulk
    // copy per field streams it to HBM while the next stage computes —
    // instead of a burst of global stores at the end of every stage
    for (int off = threadIdx.x; off < NE * Q3; off += blockDim.x) {
      const int el = off / Q3;
      const T* w = W + el * CS + (off - el * Q3);
#pragma unroll
      for (int f = 0; f < kMaxFields; ++f)
        if (f < R) Ys[f * NE * Q3 + off] = (w[f * NE * CS] + w[ds + f * NE * CS]) + w[2 * ds + f * NE * CS];
    }
    ptx::fence_proxy_async();
    __syncthreads();  // W is rewritten by the next stage's pass A; Ys complete
    if (producer) {
      for (int f = 0; f < R; ++f) ptx::bulk_s2g(reinterpret_cast<T*>(p.Y[f]) + e0 * Q3, Ys + f * NE * Q3, bytes);
      ptx::bulk_commit();
    }
  }
  if (producer) ptx::bulk_wait<0>();
}

// ---------------------------------------------------------------- v5 -----
// v2 with passes C and A of consecutive stages merged into one segment.
//
// The thread of pass C task (x, plane p, cube) reads W[x][cube][plane p] and
// the thread of pass A task (y = x, plane j = p, cube) of the NEXT stage
// writes exactly those 25 words — it is the same thread. So C(s) and A(s+1)
// need no barrier between them: a stage costs two CTA barriers (after B;
// after C+A) instead of three, and the tail of C (the direction-sum chain
// into Ys, its named-barrier waits) overlaps the DFMAs of A. Direction 0
// stores its partial before running A (nothing to wait for); directions 1 and
// 2 run A first and then take their turn in the chain, so the chain's waits
// are hidden behind A. Arithmetic and summation order are those of v2: the
// output is bitwise identical. kChainEarly: directions below it take their
// chain step right after C (default 2: x = 0 stores, x = 1 adds as soon as
// x = 0 has stored, both then run A; x = 2 runs A first and adds last, so
// the segment ends with one chain step instead of two serialised ones).
// FE_HEX_TRACE instance (meta v=7): per-warp clock64 stamps of CTA 0 for the
// first kTraceIters stages, read back by tools/hex_trace.py through
// fe_debug_hex_trace (not part of the ABI). ptxas may move a clock read
// across independent arithmetic: only stamps next to waits are exact.
constexpr int kTraceIters = 48, kTraceEv = 8;
__device__ unsigned long long g_hex_trace[kTraceIters * 16 * kTraceEv];
template <bool kTrace>
__device__ __forceinline__ void hex_stamp(int it, int ev) {
  if constexpr (kTrace) {
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && it < kTraceIters && threadIdx.x < 512)
      g_hex_trace[(it * 16 + threadIdx.x / 32) * kTraceEv + ev] = clock64();
  }
}

template <typename T, int Q, int X>
__device__ __forceinline__ void sweep_c(const T* in, T (&v)[Q][Q]) {
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int c = 0; c < Q; ++c) v[b][c] = in[b * Q + c];
  cols_c<T, Q, 4, X, true>(v);
  rows_c<T, Q, 5, X, true>(v);
}

template <typename T, int Q, int X>
__device__ __forceinline__ void chain_store(const T (&v)[Q][Q], T* ys, int b0) {
  if constexpr (X > 0) asm volatile("bar.sync %0, 64;" ::"r"(b0 + X - 1) : "memory");
#pragma unroll
  for (int m = 0; m < Q; ++m)
#pragma unroll
    for (int n = 0; n < Q; ++n) ys[m * Q + n] = X == 0 ? v[m][n] : ys[m * Q + n] + v[m][n];
  if constexpr (X < 2) asm volatile("bar.arrive %0, 64;" ::"r"(b0 + X) : "memory");
}

// one thread's merged segment: C(s) on its W plane, A(s+1) into the same plane
template <typename T, int Q, int D, bool kTrace, int kChainEarly>
__device__ __forceinline__ void c_then_a(T* w, T* ys, const T* a_in, int b0, bool next, std::uint64_t* ubar,
                                         std::uint32_t uphase, int it) {
  T v[Q][Q];
  sweep_c<T, Q, D>(w, v);
  hex_stamp<kTrace>(it, 4);
  if constexpr (D < kChainEarly) chain_store<T, Q, D>(v, ys, b0);
  if (next) {
    ptx::mbar_wait(ubar, uphase);
    hex_stamp<kTrace>(it, 5);
    pass_a<T, Q, D>(a_in, w);
  }
  hex_stamp<kTrace>(it, 6);
  if constexpr (D >= kChainEarly) chain_store<T, Q, D>(v, ys, b0);
}

template <typename T, int Q, int NE2, bool kSplitB, bool kTrace = false, int kChainEarly = 1, bool kPairFast = false>
__global__ void __launch_bounds__(HexCfg<Q, NE2>::kThreads, 1) hex5_kernel(const __grid_constant__ Hex2Dev p) {
  constexpr int NE = NE2;
  constexpr int Q2 = Hx<Q>::Q2, Q3 = Hx<Q>::Q3, CS = Hx<Q>::CS;
  static_assert(NE * kMaxFields == 32, "one warp per (direction, plane): 32 cubes per stage");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const T* const pG = reinterpret_cast<const T*>(p.G);
  constexpr int R = kMaxFields;
  constexpr int nblk = NE * R;
  constexpr int ds = nblk * CS;
  T* Gs = sm;
  T* Us = Gs + ND * ND * NE * Q3;
  T* W = Us + R * NE * Q3;
  T* Ys = W + ND * ds;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
      (reinterpret_cast<std::uintptr_t>(Ys + R * NE * Q3) + 7) & ~std::uintptr_t{7});
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const std::int64_t nstages = p.E / NE;
  const std::int64_t step = gridDim.x;
  const std::uint32_t bytes = static_cast<std::uint32_t>(NE * Q3 * sizeof(T));
  auto issue_g = [&](std::int64_t st) {
    ptx::mbar_arrive_expect_tx(&bar[0], bytes * static_cast<std::uint32_t>(ND * ND));
    const std::int64_t e0 = st * NE;
    for (int xy = 0; xy < ND * ND; ++xy)
      ptx::bulk_g2s(Gs + xy * NE * Q3, pG + (xy * p.E + e0) * Q3, bytes, &bar[0]);
  };
  auto issue_u = [&](std::int64_t st) {
    ptx::mbar_arrive_expect_tx(&bar[1], bytes * static_cast<std::uint32_t>(R));
    const std::int64_t e0 = st * NE;
    for (int f = 0; f < R; ++f) ptx::bulk_g2s(Us + f * NE * Q3, reinterpret_cast<const T*>(p.U[f]) + e0 * Q3, bytes, &bar[1]);
  };
  const bool producer = threadIdx.x == blockDim.x - 32;
  const std::int64_t st0 = blockIdx.x;
  if (st0 >= nstages) return;
  if (producer) {
    issue_u(st0);
    issue_g(st0);
  }

  // passes A and C: warp = (direction, plane), lane = cube
  const int dir = threadIdx.x / (nblk * Q);
  const int ptask = threadIdx.x - dir * nblk * Q;
  const bool pactive = threadIdx.x < ND * nblk * Q;
  const int pplane = ptask / nblk, pcube = ptask - pplane * nblk;
  const T* a_in = Us + pcube * Q3 + pplane * Q2;
  T* wp = W + dir * ds + pcube * CS + pplane * Q2;
  T* ys = Ys + pcube * Q3 + pplane * Q2;
  const int b0 = 1 + 2 * pplane;
  constexpr int H = R / 2;
  constexpr int nbt = H * NE * Q2;

  // prologue: A of the first stage
  if (pactive) {
    ptx::mbar_wait(&bar[1], 0);
    if (dir == 0) pass_a<T, Q, 0>(a_in, wp);
    else if (dir == 1) pass_a<T, Q, 1>(a_in, wp);
    else pass_a<T, Q, 2>(a_in, wp);
  }
  __syncthreads();
  if (producer && st0 + step < nstages) issue_u(st0 + step);

  int it = 0;
  for (std::int64_t st = st0; st < nstages; st += step, ++it) {
    const bool more = st + step < nstages;
    hex_stamp<kTrace>(it, 0);
    ptx::mbar_wait(&bar[0], static_cast<std::uint32_t>(it & 1));
    hex_stamp<kTrace>(it, 1);
    // pass B: the (line, element, field pair) tasks that fill whole
    // four-warp rows run as pairs; the remainder is split into single-field
    // tasks on one warp (at Q = 5: 384 pairs on warps 0-11, the last 16 pairs
    // as 32 singles on warp 12), so no sub-partition issues a fourth
    // full-length pass-B warp while the others issue three
    constexpr int nfull = kSplitB ? nbt / 128 * 128 : nbt;
    constexpr int nleft = nbt - nfull;
    static_assert(2 * nleft <= 32, "remainder fits one warp");
    // task t -> (line kl, element el, first field f0): line fastest, or
    // (kPairFast) field pair fastest, so the four lanes of one (element,
    // line) read the same G words (broadcast) while W stays conflict free
    // (pairs f0 = 0..3 sit NE * CS = 4 mod 16 doubles apart)
    auto task = [&](int t, int& kl, int& el, int& f0) {
      if constexpr (kPairFast) {
        f0 = t % H;
        kl = (t / H) % Q2;
        el = t / (H * Q2);
      } else {
        kl = t % Q2;
        const int r = t / Q2;
        el = r % NE;
        f0 = r / NE;
      }
    };
    if (threadIdx.x < nfull) {
      int kl, el, f0;
      task(threadIdx.x, kl, el, f0);
      const int f1 = f0 + H;
      const T* g = Gs + el * Q3 + kl;
      T* const wl[2] = {W + (f0 * NE + el) * CS + kl, W + (f1 * NE + el) * CS + kl};
      pass_b<T, Q, 2>(wl, ds, g, NE * Q3);
    } else if (nleft > 0 && threadIdx.x < nfull + 2 * nleft) {
      // lanes 0-15 take the first field of the remainder pairs, 16-31 the
      // second: each half-warp walks consecutive lines (no bank conflicts)
      const int idx = threadIdx.x - nfull;
      int kl, el, f0;
      task(nfull + idx % nleft, kl, el, f0);
      const int f = f0 + (idx >= nleft ? H : 0);
      const T* g = Gs + el * Q3 + kl;
      T* const wl[1] = {W + (f * NE + el) * CS + kl};
      pass_b<T, Q, 1>(wl, ds, g, NE * Q3);
    }
    hex_stamp<kTrace>(it, 2);
    if (producer) ptx::bulk_wait_read<0>();  // the previous stage's stores have read Ys
    __syncthreads();
    hex_stamp<kTrace>(it, 3);
    if (producer && more) issue_g(st + step);

    if (pactive) {
      const std::uint32_t uph = static_cast<std::uint32_t>((it + 1) & 1);
      if (dir == 0) c_then_a<T, Q, 0, kTrace, kChainEarly>(wp, ys, a_in, b0, more, &bar[1], uph, it);
      else if (dir == 1) c_then_a<T, Q, 1, kTrace, kChainEarly>(wp, ys, a_in, b0, more, &bar[1], uph, it);
      else c_then_a<T, Q, 2, kTrace, kChainEarly>(wp, ys, a_in, b0, more, &bar[1], uph, it);
    }
    ptx::fence_proxy_async();
    hex_stamp<kTrace>(it, 7);
    __syncthreads();  // Ys complete (stage st), Us consumed (stage st + step), W holds t of st + step
    if (producer) {
      const std::int64_t e0 = st * NE;
      for (int f = 0; f < R; ++f) ptx::bulk_s2g(reinterpret_cast<T*>(p.Y[f]) + e0 * Q3, Ys + f * NE * Q3, bytes);
      ptx::bulk_commit();
      if (st + 2 * step < nstages) issue_u(st + 2 * step);
    }
  }
  if (producer) ptx::bulk_wait<0>();
}

// The operator constants are shared by every launch on a device: a launch
// waits for the previous one (any stream) before restaging them.
struct HexConstSlot {
  cudaEvent_t last = nullptr;
  double* stage = nullptr;  // device staging of the six operators (one constant copy per launch)
};

struct Mats6 {
  const double* m[6];
};
template <typename T>
__global__ void gather_ops(const __grid_constant__ Mats6 src, int n, T* dst) {
  for (int t = threadIdx.x; t < 6 * n; t += blockDim.x)
    dst[t] = static_cast<T>(reinterpret_cast<const T*>(src.m[t / n])[t % n]);
}
std::mutex g_hex_mu;
HexConstSlot g_hex_slot[64];

template <typename T, int Q, int NE2, int kMerged = 0>
int launch_hex2_t(const HexLaunch& L, cudaStream_t st) {
  constexpr int Q2 = Hx<Q>::Q2, Q3 = Hx<Q>::Q3, CS = Hx<Q>::CS;
  const int R = L.rows;
  const int nblk = NE2 * R;
  constexpr int threads = HexCfg<Q, NE2>::kThreads;
  auto kern = hex2_kernel<T, Q, NE2>;
  if constexpr (kMerged == 1) kern = hex5_kernel<T, Q, NE2, false, false, 1>;
  if constexpr (kMerged == 2) kern = hex5_kernel<T, Q, NE2, true, false, 2, true>;
  if constexpr (kMerged == 3) kern = hex5_kernel<T, Q, NE2, true, true, 2, true>;
  if constexpr (kMerged == 4) kern = hex5_kernel<T, Q, NE2, true, false, 1>;
  if constexpr (kMerged == 5) kern = hex5_kernel<T, Q, NE2, true, false, 2, false>;
  Hex2Dev d{};
  d.E = L.E;
  d.rows = R;
  d.G = L.G;
  for (int f = 0; f < R; ++f) {
    d.U[f] = L.U[f];
    d.Y[f] = L.Y[f];
  }
  const size_t doubles = ND * ND * NE2 * Q3 + 2 * R * NE2 * Q3 + ND * nblk * CS;
  const size_t smem = doubles * sizeof(T) + 24;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int sms = 148;
  device_sm_count(&sms);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  std::int64_t grid = static_cast<std::int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
  if (grid > L.E / NE2) grid = L.E / NE2;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_hex_mu);
  HexConstSlot& slot = g_hex_slot[dev & 63];
  if (!slot.last || !slot.stage) return cudaErrorInitializationError;  // hex_prepare() not run for this device
  cudaStreamWaitEvent(st, slot.last, 0);
  // gather the six operators into one run, then one copy into the constant
  // bank (each copy costs tens of microseconds of stream time)
  Mats6 m6{};
  for (int k = 0; k < 6; ++k) m6.m[k] = L.mats[k];
  gather_ops<T><<<1, 256, 0, st>>>(m6, ND * Q2, reinterpret_cast<T*>(slot.stage));
  if constexpr (sizeof(T) == 4)
    e = cudaMemcpyToSymbolAsync(c_hex_ops_f, slot.stage, 6 * ND * Q2 * sizeof(T), 0, cudaMemcpyDeviceToDevice, st);
  else
    e = cudaMemcpyToSymbolAsync(c_hex_ops, slot.stage, 6 * ND * Q2 * sizeof(T), 0, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  kern<<<static_cast<int>(grid), threads, smem, st>>>(d);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaEventRecord(slot.last, st);
}

// elements per stage: 4 when E allows (fact meta ne=2 forces two), 2 at Q = 6
// (shared memory)
template <int Q>
int launch_hex2_q(const HexLaunch& L, cudaStream_t st) {
  if (L.f32) {
    // fp32: four-element stages (16-byte bulk-copy runs), two at Q = 6
    if constexpr (Q < 6) {
      if (L.E % 4 != 0) return cudaErrorInvalidValue;
      return launch_hex2_t<float, Q, 4>(L, st);
    } else {
      return launch_hex2_t<float, Q, 2>(L, st);
    }
  }
  if constexpr (Q < 6) {
    // v2 (default) takes the merged-stage kernel where it applies (eight
    // fields: one warp per (direction, plane) over 32 cubes); v3 forces the
    // three-barrier kernel; A/B variants of the merged one: v5 without the
    // pass-B split and with only direction 0's chain step early, v6 with the
    // split and only direction 0 early (both: pass-B tasks line fastest), v9
    // the default with line-fastest pass-B tasks; v7 the default with
    // FE_HEX_TRACE stamps
    const bool merged_ok = L.rows == kMaxFields && L.E % 4 == 0 && L.ne != 2;
    if (merged_ok && L.variant == 5) return launch_hex2_t<double, Q, 4, 1>(L, st);
    if (merged_ok && L.variant == 2) return launch_hex2_t<double, Q, 4, 2>(L, st);
    if (merged_ok && L.variant == 7) return launch_hex2_t<double, Q, 4, 3>(L, st);
    if (merged_ok && L.variant == 6) return launch_hex2_t<double, Q, 4, 4>(L, st);
    if (merged_ok && L.variant == 9) return launch_hex2_t<double, Q, 4, 5>(L, st);
    if (L.ne != 2 && L.E % 4 == 0) return launch_hex2_t<double, Q, 4>(L, st);
  }
  return launch_hex2_t<double, Q, 2>(L, st);
}

int launch_hex2(const HexLaunch& L, cudaStream_t st) {
  switch (L.P) {
    case 3: return launch_hex2_q<3>(L, st);
    case 4: return launch_hex2_q<4>(L, st);
    case 5: return launch_hex2_q<5>(L, st);
    case 6: return launch_hex2_q<6>(L, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// v2 takes 3..6 points per direction (P2..P5 hexes), v1 only 5
bool hex_supported(int nd, int p, std::int64_t E, int rows) {
  return nd == ND && p >= 3 && p <= kMaxQ && E % NE == 0 && rows >= 1 && rows <= kMaxFields;
}

int launch_hex(const HexLaunch& L, void* stream) {
  if (!hex_supported(L.ND, L.P, L.E, L.rows)) return cudaErrorInvalidValue;
  if (L.E == 0) return cudaSuccess;
  if (L.variant != 1 || L.P != P || L.f32) return launch_hex2(L, static_cast<cudaStream_t>(stream));
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

// debug hook (tools/hex_trace.py): copies the v=7 instance's stamps to host
extern "C" int fe_debug_hex_trace(void* host, size_t bytes) {
  if (bytes > sizeof(g_hex_trace)) bytes = sizeof(g_hex_trace);
  return cudaMemcpyFromSymbol(host, g_hex_trace, bytes);
}

// Creates the device's operator staging buffer and ordering event; called at
// plan time so the execute path never allocates (and stays graph-capturable).
int hex_prepare(int dev) {
  std::lock_guard<std::mutex> lock(g_hex_mu);
  HexConstSlot& slot = g_hex_slot[dev & 63];
  cudaError_t e = cudaSuccess;
  if (!slot.last && (e = cudaEventCreateWithFlags(&slot.last, cudaEventDisableTiming)) != cudaSuccess) return e;
  if (!slot.stage && (e = cudaMalloc(&slot.stage, 6 * ND * kMaxQ * kMaxQ * sizeof(double))) != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace feb200
