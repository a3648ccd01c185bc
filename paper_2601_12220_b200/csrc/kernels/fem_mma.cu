// K1 on the FP64 tensor cores — batched FEM gradient
//   y_q[r,e,i] = sum_x J_q[x,r,e] sum_j D_q[x,i,j] U_q[e,j]     (C1, C5)
//
// The DFMA kernel (fem_grad.cu) spends ~40 instructions per element, row and
// local dof: it is issue-bound, not HBM-bound. Here the inner contraction
// T_x = D_x U^T (per tile: M = NI dofs, N = 8 elements, K = NJ) runs on DMMA
// (mma.sync m8n8k4 f64; tcgen05 has no f64 kind), one 8x8x4 MMA doing the work
// of 8 warp-wide DFMAs, so the kernel is left bound by HBM traffic.
//
//   * warp 0 / lane 0 is the producer: per tile it arms the stage mbarrier and
//     issues 1-D bulk copies of the J tile and every U leaf tile (as in
//     fem_grad.cu) into an S-stage shared ring;
//   * consumer warp w owns elements [8w, 8w+8) of each tile: the D_x
//     A-fragments (zero-padded to MT x 8 rows, KS x 4 columns) stay in
//     registers; the B-fragment U^T[j][e] is read from the staged tile —
//     functional operands (u + 0.5 k) are combined right there, each value
//     exactly once, in the operand's own order;
//   * the J contraction y[r] = sum_x J[x,r,e] T_x runs on the accumulator
//     fragments (DFMA), the results go to a per-warp double-buffered staging
//     slab [rows][NR][8][NI] and leave with 1-D bulk stores (each (q, r) slab
//     is one contiguous 8*NI-double run of Y_q), so stores are full-line and
//     asynchronous.
// Parity: the operation order differs from the reference's (factorised path,
// fused products); results agree within 1e-12 relative.
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int NX = 3, NR = 3;

struct MCoef {
  double pre, post;
  int sign;
};

template <int NI, int NJ, int TE, bool kPlainU>
__global__ void __launch_bounds__(32 + TE * 4, 1) fem_mma_kernel(const __grid_constant__ FemGradLaunch p) {
  constexpr int MT = (NI + 7) / 8;  // 8-row A tiles over the dofs i
  constexpr int KS = (NJ + 3) / 4;  // k-steps over the dofs j
  constexpr int kWarps = TE / 8;    // consumer warps, 8 elements each
  constexpr int kUTile = TE * NJ;
  constexpr int kJTile = NX * NR * TE;
  static_assert(TE % 8 == 0 && (NI * 8) % 16 == 0, "bulk stores need 16-byte runs");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = p.stages;
  const int R = p.rows;
  const int stage_doubles = p.n_j * kJTile + p.n_u * kUTile;
  const int slab = R * NR * 8 * NI;  // one warp's output slab per tile
  double* dsm = reinterpret_cast<double*>(smem_raw);                        // D copies
  double* ring = dsm + ((p.n_d * NX * NI * NJ + 1) & ~1);                    // stages
  double* obuf = ring + static_cast<size_t>(S) * stage_doubles;              // [kWarps][2][slab]
  MCoef* coefs = reinterpret_cast<MCoef*>(obuf + static_cast<size_t>(kWarps) * 2 * slab);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(coefs + kFemMaxUTiles);
  std::uint64_t* empty = full + S;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const std::int64_t E = p.E;
  const std::int64_t ntiles = (E + TE - 1) / TE;

  const std::uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](std::int64_t tile, int s) {
    const std::int64_t e0 = tile * TE;
    const int cnt = static_cast<int>(E - e0 < TE ? E - e0 : TE);
    const std::uint32_t jb = static_cast<std::uint32_t>(cnt) * 8u;
    const std::uint32_t ub = static_cast<std::uint32_t>(cnt) * NJ * 8u;
    ptx::mbar_arrive_expect_tx(&full[s], static_cast<std::uint32_t>(p.n_j * NX * NR) * jb +
                                             static_cast<std::uint32_t>(p.n_u) * ub);
    double* st = ring + static_cast<size_t>(s) * stage_doubles;
    for (int a = 0; a < p.n_j; ++a)
      for (int xr = 0; xr < NX * NR; ++xr)
        ptx::bulk_g2s_hint(st + a * kJTile + xr * TE, p.J[a] + xr * E + e0, jb, &full[s], pol);
    double* su = st + p.n_j * kJTile;
    for (int u = 0; u < p.n_u; ++u) ptx::bulk_g2s_hint(su + u * kUTile, p.U[u] + e0 * NJ, ub, &full[s], pol);
  };
  int prefetched = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kWarps);
    }
    ptx::fence_barrier_init();
    for (std::int64_t tile = blockIdx.x; tile < ntiles && prefetched < S; tile += gridDim.x, ++prefetched)
      issue(tile, prefetched);
  }
  for (int t = tid; t < p.n_d * NX * NI * NJ; t += blockDim.x) {
    const int which = t / (NX * NI * NJ);
    dsm[t] = __ldg(p.D[which] + (t - which * NX * NI * NJ));
  }
  if (!kPlainU && tid < p.n_u) {
    MCoef c;
    c.pre = p.u_pre[tid] >= 0 ? __ldg(p.coef + 2 * p.u_pre[tid]) : 1.0;
    c.post = p.u_post[tid] >= 0 ? __ldg(p.coef + 2 * p.u_post[tid]) : 1.0;
    c.sign = p.u_sign[tid];
    coefs[tid] = c;
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    if (tid != 0) return;
    int it = 0;
    for (std::int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      if (it < prefetched) continue;
      const int s = it % S;
      const std::uint32_t round = static_cast<std::uint32_t>(it / S);
      ptx::mbar_wait(&empty[s], (round & 1u) ^ 1u);
      issue(tile, s);
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  const int w = warp - 1;
  const int lane = tid & 31;
  const int g = lane >> 2;  // A/B fragment row (dof i / element), C row
  const int c4 = lane & 3;  // A/B fragment k, C column pair
  const int n0 = w * 8;
  double a[NX][MT][KS];
  int cur_d = -1;
  int it = 0;
  for (std::int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % S;
    const std::uint32_t round = static_cast<std::uint32_t>(it / S);
    const std::int64_t e0 = tile * TE;
    const int cnt = static_cast<int>(E - e0 < TE ? E - e0 : TE);
    const int nvalid = cnt - n0 < 8 ? cnt - n0 : 8;
    double* ob = obuf + static_cast<size_t>(w * 2 + (it & 1)) * slab;
    // the bulk stores that last read this slab (two tiles ago) must be done
    if (lane == 0) ptx::bulk_wait_read<1>();
    __syncwarp();
    ptx::mbar_wait(&full[s], round & 1u);
    const double* st = ring + static_cast<size_t>(s) * stage_doubles;
    const double* su = st + p.n_j * kJTile;

    if (nvalid > 0) {
      for (int q = 0; q < R; ++q) {
        if (p.row_d[q] != cur_d) {
          cur_d = p.row_d[q];
          const double* dq = dsm + cur_d * NX * NI * NJ;
#pragma unroll
          for (int x = 0; x < NX; ++x)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int ks = 0; ks < KS; ++ks) {
                const int i = mt * 8 + g, j = ks * 4 + c4;
                a[x][mt][ks] = (i < NI && j < NJ) ? dq[(x * NI + i) * NJ + j] : 0.0;
              }
        }
        // B fragment: U_q^T[j][e], element e = n0 + g, dof j = 4 ks + c4
        double b[KS];
        const int el = n0 + g;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int j = ks * 4 + c4;
          double v = 0.0;
          if (j < NJ) {
            if constexpr (kPlainU) {
              v = su[p.row_u_first[q] * kUTile + el * NJ + j];
            } else {
              const int u0 = p.row_u_first[q], nt = p.row_u_count[q];
              for (int k = 0; k < nt; ++k) {
                const MCoef cf = coefs[u0 + k];
                const double xk = __dmul_rn(__dmul_rn(cf.pre, su[(u0 + k) * kUTile + el * NJ + j]), cf.post);
                v = k == 0 ? xk : (cf.sign > 0 ? __dadd_rn(v, xk) : __dsub_rn(v, xk));
              }
            }
          }
          b[ks] = v;
        }
        double acc[NX][MT][2];
#pragma unroll
        for (int x = 0; x < NX; ++x)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            acc[x][mt][0] = 0.0;
            acc[x][mt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) ptx::dmma_8x8x4_nv(acc[x][mt][0], acc[x][mt][1], a[x][mt][ks], b[ks]);
          }
        // y[r][e][i] = sum_x J[x,r,e] T_x[i][e] on the fragments: this lane
        // holds i = 8 mt + g, e = n0 + 2 c4 + {0, 1}
        const double* jt = st + p.row_j[q] * kJTile + n0 + 2 * c4;
        double* oq = ob + q * NR * 8 * NI;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          double2 jx[NX];
#pragma unroll
          for (int x = 0; x < NX; ++x) jx[x] = *reinterpret_cast<const double2*>(jt + (x * NR + r) * TE);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int i = mt * 8 + g;
            double y0 = 0.0, y1 = 0.0;
#pragma unroll
            for (int x = 0; x < NX; ++x) {
              y0 = fma(jx[x].x, acc[x][mt][0], y0);
              y1 = fma(jx[x].y, acc[x][mt][1], y1);
            }
            if (i < NI) {
              oq[(r * 8 + 2 * c4) * NI + i] = y0;
              oq[(r * 8 + 2 * c4 + 1) * NI + i] = y1;
            }
          }
        }
      }
    }
    // this warp is done with the stage
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (nvalid > 0) {
      ptx::fence_proxy_async();  // staging writes -> async proxy (bulk store)
      __syncwarp();
      if (lane == 0) {
        const std::uint32_t bytes = static_cast<std::uint32_t>(nvalid) * NI * 8u;
        for (int q = 0; q < R; ++q)
          for (int r = 0; r < NR; ++r)
            ptx::bulk_s2g(p.Y[q] + (static_cast<std::int64_t>(r) * E + e0 + n0) * NI, ob + (q * NR + r) * 8 * NI,
                          bytes);
      }
    }
    if (lane == 0) ptx::bulk_commit();
  }
  if (lane == 0) ptx::bulk_wait<0>();
}

template <int NI, int NJ, int TE>
int launch_mma_shape(const FemGradLaunch& p, cudaStream_t s) {
  const size_t stage = static_cast<size_t>(p.n_j) * NX * NR * TE + static_cast<size_t>(p.n_u) * TE * NJ;
  const size_t slab = static_cast<size_t>(p.rows) * NR * 8 * NI;
  const size_t doubles = ((static_cast<size_t>(p.n_d) * NX * NI * NJ + 1) & ~size_t(1)) + p.stages * stage +
                         (TE / 8) * 2 * slab;
  const size_t smem = sizeof(double) * doubles + sizeof(MCoef) * kFemMaxUTiles + sizeof(std::uint64_t) * 2 * p.stages;
  auto run = [&](auto kern) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int sms = 148, per_sm = 1;
    device_sm_count(&sms);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 + TE * 4, smem);
    const std::int64_t ntiles = (p.E + TE - 1) / TE;
    std::int64_t grid = static_cast<std::int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
    if (p.grid > 0) grid = p.grid;
    if (grid > ntiles) grid = ntiles;
    kern<<<static_cast<int>(grid), 32 + TE * 4, smem, s>>>(p);
    return cudaGetLastError();
  };
  if (p.plain_u) return run(fem_mma_kernel<NI, NJ, TE, true>);
  return run(fem_mma_kernel<NI, NJ, TE, false>);
}

}  // namespace

bool fem_mma_supported(int NX_, int NR_, int NI, int NJ) { return NX_ == NX && NR_ == NR && NI == 10 && NJ == 10; }

int launch_fem_mma(const FemGradLaunch& p, void* stream) {
  if (p.E == 0) return cudaSuccess;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!fem_mma_supported(p.NX, p.NR, p.NI, p.NJ)) return cudaErrorInvalidValue;
  if (p.tile_e == 64) {
    // fall back to 32-element tiles when 64 does not fit (many rows / stages)
    const int r = launch_mma_shape<10, 10, 64>(p, s);
    if (r != cudaErrorInvalidValue) return r;
    cudaGetLastError();
  }
  if (p.tile_e == 16) return launch_mma_shape<10, 10, 16>(p, s);
  return launch_mma_shape<10, 10, 32>(p, s);
}

}  // namespace feb200
