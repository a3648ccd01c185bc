// K1 — batched FEM gradient  y_q[r,e,i] = sum_{x,j} J_q[x,r,e] D_q[x,i,j] U_q[e,j]
// (the C1/C5 configs), HBM-bound, fp64.
//
// B200 design (persistent, warp-specialised, TMA-fed):
//   * grid = resident CTAs on all SMs; each CTA walks element tiles of TE
//     elements with a stride of gridDim.x;
//   * warp 0 (one elected lane) is the producer: for every tile it arms the
//     stage's mbarrier with the byte count and issues 1-D bulk copies
//     (cp.async.bulk, the TMA engine's non-tensor path) of the J tile (NX*NR
//     contiguous runs of TE doubles per distinct J) and of every U leaf tile
//     (TE*NJ contiguous doubles) into an S-stage shared-memory ring — inputs are
//     read from HBM exactly once and shared J is staged once for all rows;
//   * functional U operands (s = u + 0.5 k, the C5 wave step) are combined
//     ONCE per tile by the consumers into a double-buffered shared tile (the
//     K2 prologue: s never exists in HBM, and no value is computed twice);
//   * TE*NI consumer threads, thread (el, i): D_q[x,i,:] lives in registers,
//     U is read as double2 broadcasts, J as broadcasts; t[x] = D.u then
//     y[r] = J^T t. Consecutive threads own consecutive (e, i), so every
//     y_q[r, :, :] store is a fully coalesced 256-byte warp transaction.
// The operation order differs from the reference's (factorised contraction
// path with FMA); parity is within 1e-12 relative.
#include <cuda_runtime.h>

#include <type_traits>

#include "fem_grad.cuh"
#include "launch.h"

namespace feb200 {

namespace {

using namespace fem;

template <typename T, int NX, int NR, int NI, int NJ, int TE, bool kPlainU, bool kDSmem, int EPT = 1>
__global__ void __launch_bounds__(32 + fem_consumers<NX, NR, NI, NJ, TE, EPT>(), kDSmem ? 2 : 1)
    fem_grad_kernel(const __grid_constant__ FemGradLaunch p) {
  using Pro = typename std::conditional<kPlainU, FemProPlain, FemProAffine>::type;
  fem_grad_body<T, NX, NR, NI, NJ, TE, Pro, kDSmem, EPT, FemEpiNone>(p);
}

template <typename T, int NX, int NR, int NI, int NJ, int TE, int EPT = 1>
int launch_shape(const FemGradLaunch& p, cudaStream_t s) {
  constexpr int kThreads = 32 + fem_consumers<NX, NR, NI, NJ, TE, EPT>();
  const bool plain = p.plain_u;
  const size_t doubles = static_cast<size_t>(p.n_d) * NX * NI * NJ +
                         static_cast<size_t>(p.stages) * (p.n_j * NX * NR * TE + p.n_u * TE * NJ) +
                         (plain ? 0 : 2 * static_cast<size_t>(p.rows) * TE * NJ);
  const size_t smem = sizeof(T) * doubles + 16 + sizeof(Coef) * kFemMaxUTiles + sizeof(std::uint64_t) * 2 * p.stages;
  auto run = [&](auto kern) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int sms = 148, per_sm = 1;
    device_sm_count(&sms);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    const std::int64_t ntiles = (p.E + TE - 1) / TE;
    std::int64_t grid = static_cast<std::int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
    if (p.grid > 0) grid = p.grid;
    if (grid > ntiles) grid = ntiles;
    kern<<<static_cast<int>(grid), kThreads, smem, s>>>(p);
    return cudaGetLastError();
  };
  if constexpr (EPT > 1) {
    if (plain) return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, true, false, EPT>);
    return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, false, false, EPT>);
  } else {
    if (p.d_in_smem) {
      if (plain) return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, true, true>);
      return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, false, true>);
    }
    if (plain) return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, true, false>);
    return run(fem_grad_kernel<T, NX, NR, NI, NJ, TE, false, false>);
  }
}

}  // namespace

bool fem_grad_supported(int NX, int NR, int NI, int NJ) {
  return NX == 3 && NR == 3 && ((NI == 10 && NJ == 10) || (NI == 4 && NJ == 4) || (NI == 20 && NJ == 20));
}

template <typename T>
int launch_fem_grad_t(const FemGradLaunch& p, cudaStream_t s) {
  if (p.NI == 10 && p.NJ == 10) {
    // small batches: half-size tiles put more CTAs in flight (latency-bound)
    if (p.tile_e == 16) return launch_shape<T, 3, 3, 10, 10, 16>(p, s);
    if (p.ept == 2) {
      // 64-element tiles: one tile per SM for small batches (C1: 157 tiles)
      if (p.tile_e == 64) return launch_shape<T, 3, 3, 10, 10, 64, 2>(p, s);
      // one tile per CTA slot at C1's E = 1e4: 148 x 68 / 296 x 34 elements
      if (p.tile_e == 68) return launch_shape<T, 3, 3, 10, 10, 68, 2>(p, s);
      if constexpr (sizeof(T) == 8)  // fp32 rows of 34 are not 16-byte multiples
        if (p.tile_e == 34) return launch_shape<T, 3, 3, 10, 10, 34, 2>(p, s);
      return launch_shape<T, 3, 3, 10, 10, 32, 2>(p, s);
    }
    return launch_shape<T, 3, 3, 10, 10, 32>(p, s);
  }
  if (p.NI == 4 && p.NJ == 4) return launch_shape<T, 3, 3, 4, 4, 64>(p, s);
  if (p.NI == 20 && p.NJ == 20) return launch_shape<T, 3, 3, 20, 20, 16>(p, s);
  return cudaErrorInvalidValue;
}

int launch_fem_grad_rtc(const FemGradLaunch& p_in, void* kernel, int te, int ept, void* stream) {
  if (p_in.E == 0) return cudaSuccess;
  // the generated instances run the pipelined prologue (three combined
  // buffers): its rewrite of buffer k % 3 is ordered after every warp's reads
  // of tile k - 3 only through the producer's full[k % S] wait, i.e. for
  // S <= 3 stages (with four, a warp two tiles ahead overwrote a buffer a
  // slow warp was still reading: compute-sanitizer racecheck, round 2)
  FemGradLaunch p = p_in;
  if (p.stages > 3) p.stages = 3;
  const int nj = p.NJ, ni = p.NI;
  const int threads = 32 + (te * ni / ept + 31) / 32 * 32;
  const size_t doubles = static_cast<size_t>(p.n_d) * p.NX * ni * nj +
                         static_cast<size_t>(p.stages) * (p.n_j * p.NX * p.NR * te + p.n_u * te * nj) +
                         3 * static_cast<size_t>(p.rows) * te * nj;  // pipelined prologue: 3 combined buffers
  const size_t smem =
      (p.f32 ? 4 : 8) * doubles + 16 + sizeof(Coef) * kFemMaxUTiles + sizeof(std::uint64_t) * (2 * p.stages + 3);
  const void* kern = kernel;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 148, per_sm = 1;
  device_sm_count(&sms);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  const std::int64_t ntiles = (p.E + te - 1) / te;
  std::int64_t grid = static_cast<std::int64_t>(sms) * (per_sm > 0 ? per_sm : 1);
  if (p.grid > 0) grid = p.grid;
  if (grid > ntiles) grid = ntiles;
  void* args[] = {const_cast<FemGradLaunch*>(&p)};
  return cudaLaunchKernel(kern, dim3(static_cast<unsigned>(grid)), dim3(threads), args, smem,
                          static_cast<cudaStream_t>(stream));
}

int launch_fem_grad(const FemGradLaunch& p, void* stream) {
  if (p.E == 0) return cudaSuccess;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p.f32 ? launch_fem_grad_t<float>(p, s) : launch_fem_grad_t<double>(p, s);
}

}  // namespace feb200
