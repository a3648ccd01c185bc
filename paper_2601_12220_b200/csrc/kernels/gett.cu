// K3 — dense TCCG contraction (GETT) on the FP64 tensor cores (DMMA), fed by
// TMA, with the functional-operand prologue (alpha*X + beta) fused into the
// fragment loads.
//
//   C[mo,mi,no,ni] = sum_{kA,kB} opA(A[.. mo, mi, kB, kA ..]) * opB(B[.. no, ni, kA, kB ..])
//
// (index positions are arbitrary: every tensor is described by per-role
// strides). For the pinned C3 spelling aebf,dfce->abcd: mo=a, mi=b, no=c,
// ni=d, kA=f (A's unit-stride index), kB=e (B's unit-stride index).
//
// Why this shape on sm_100a: tcgen05 has no f64 kind, so FP64 tensor work is
// mma.sync m8n8k4 (DMMA, SASS DMMA.8x8x4, 16 SMSP cycles each). CTA tiles are
// 144 x 144 (two mo x 72 mi by two no x 72 ni) over 12 consumer warps with
// 24 x 72 warp tiles — three warps per SM sub-partition, so the four DMMA
// pipes carry equal work (a 72x72 tile over 9 warps left one sub-partition
// with 3 of them: 75% at best). One producer warpgroup (a single TMA thread)
// donates its registers to the consumers with setmaxnreg (40 / 152). Tiles
// are staged by TMA (cp.async.bulk.tensor: 4-D boxes gather the strided GETT
// operands without a transpose pass) into a 2-3 stage mbarrier ring, 32 k per
// stage: A boxes of 8 kA (64-byte rows, 64B swizzle) x 4 kB, B boxes of 4 kB
// (32-byte rows, 32B swizzle) x 8 kA. A 64-bit fragment load is served per
// half-warp; the DMMA k-chunk map (f = kA in {0,1,4,5} + 2 (kc >> 2),
// e = kB = qk ^ (kc & 3)) puts each half-warp's 16 words in distinct banks on
// both swizzled images (ncu: 0.3% excess wavefronts, tensor pipe 97%).
// The persistent grid walks output tiles in square raster groups that share
// A/B slices in L2.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int EXT = 72;              // mi = ni extent (one TMA box row span)
constexpr int MT = 2, NT = 2;        // mo / no values per CTA tile
constexpr int BM = MT * EXT, BN = NT * EXT;  // CTA tile 144 x 144
constexpr int KA = 8, KB = 4;        // k box: 8 kA (64-byte A rows) x 4 kB (32-byte B rows)
constexpr int KT = KA * KB;          // k per stage
constexpr int kConsumerWarps = 12;   // 6 x 2 warp tiles of 24 x 72: three per SM sub-partition
// plus one producer warpgroup (one TMA thread) that hands its registers to
// the consumers (setmaxnreg): 3 x 128 x 152 + 128 x 40 registers
constexpr int kThreads = 32 * (kConsumerWarps + 4);
constexpr int kConsumerRegs = 152, kProducerRegs = 40;
constexpr int kTileBytes = BM * KT * 8;  // 36864 (A and B alike)

struct GettDev {
  std::int64_t mo, no;                  // tile counts (ceil(extent / 2) of mo / no)
  std::int64_t ext_mo, ext_no;
  std::int64_t ka_steps, kb_steps;      // kA/8, kB/4
  std::int64_t c_mo, c_mi, c_no, c_ni;  // C strides (elements)
  double* C;
  const double* coef;
  int a_alpha, a_beta, b_alpha, b_beta;
  const double* rowA;  // sum_k A[m, k] per (mo, mi) (affine operands only)
  const double* rowB;  // sum_k B[k, n] per (no, ni)
  std::int64_t ext_mi, ext_ni;
  int vec_c;  // C rows allow 16-byte stores of (n, n+1) pairs
  double kdim;         // |K| = ext_ka * ext_kb
  int stages, group;  // group: side of the square raster block (tiles sharing A/B slices in L2)
  std::int64_t nz, c_z;  // batch count (an index of A, B and C) and its C stride; 5-D maps when nz > 1
  // split K: ksplit slices of the k steps, slice s writes its partial tile
  // into ws + s * csize (C's strides); a reduce pass sums the slices into C
  int ksplit;
  double* ws;
  std::int64_t csize;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          ptx::smem_addr(dst)),
      "l"(map), "r"(ptx::smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1,
                                            int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
          ptx::smem_addr(dst)),
      "l"(map), "r"(ptx::smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    gett_kernel(const __grid_constant__ GettDev p, const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzle atoms
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  const int S = p.stages;
  unsigned char* tiles = base;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(tiles + static_cast<size_t>(S) * 2 * kTileBytes);
  std::uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::int64_t per_z = p.mo * p.no;  // tiles per batch value
  const std::int64_t per_s = per_z * p.nz;  // tiles per K slice
  const std::int64_t ntiles = per_s * p.ksplit;
  const std::int64_t ksteps_all = p.ka_steps * p.kb_steps;
  // k steps [k_lo(s), k_lo(s + 1)) of slice s
  auto k_lo = [&](std::int64_t s) { return ksteps_all * s / p.ksplit; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();

  // tile t -> (mo, no): square blocks of group x group tiles, so the ~150
  // tiles in flight share `group` A slices and `group` B slices (fits L2)
  auto tile_coords = [&](std::int64_t t, std::int64_t& mo, std::int64_t& no) {
    const std::int64_t G = p.group;
    const std::int64_t band = G * p.no;            // tiles in one band of G mo-rows
    const std::int64_t bi = t / band, r = t - bi * band;
    const std::int64_t rows = (bi + 1) * G <= p.mo ? G : p.mo - bi * G;
    const std::int64_t bj = r / (rows * G), r2 = r - bj * rows * G;
    const std::int64_t cols = (bj + 1) * G <= p.no ? G : p.no - bj * G;
    mo = bi * G + r2 % rows;
    no = bj * G + r2 / rows;
    (void)cols;
  };

  if (warp >= kConsumerWarps) {
    // ------------------------------- producer -------------------------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    if (warp != kConsumerWarps || lane != 0) return;
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    std::int64_t it = 0;
    for (std::int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      std::int64_t mo, no;
      const std::int64_t sl = t / per_s, tz = t - sl * per_s;
      const int z = static_cast<int>(tz / per_z);
      tile_coords(tz - z * per_z, mo, no);
      for (std::int64_t ks = k_lo(sl); ks < k_lo(sl + 1); ++ks, ++it) {
        const int s = static_cast<int>(it % S);
        const std::uint32_t round = static_cast<std::uint32_t>(it / S);
        ptx::mbar_wait(&empty[s], (round & 1u) ^ 1u);
        const int kb0 = static_cast<int>(ks / p.ka_steps) * KB;
        const int ka0 = static_cast<int>(ks % p.ka_steps) * KA;
        ptx::mbar_arrive_expect_tx(&full[s], 2 * kTileBytes);
        unsigned char* st = tiles + static_cast<size_t>(s) * 2 * kTileBytes;
        // A dims (kA, mi, kB, mo) -> image [mo2][kB][mi][kA] (64-byte rows, 64B swizzle);
        // B dims (kB, ni, kA, no) -> image [no2][kA][ni][kB] (32-byte rows, 32B swizzle)
        // boxes of two mo (no) values; an odd last one reads zeros out of bounds
        if (p.nz > 1) {
          tma_load_5d(st, &tmA, &full[s], ka0, 0, kb0, static_cast<int>(mo * MT), z);
          tma_load_5d(st + kTileBytes, &tmB, &full[s], kb0, 0, ka0, static_cast<int>(no * NT), z);
        } else {
          tma_load_4d(st, &tmA, &full[s], ka0, 0, kb0, static_cast<int>(mo * MT));
          tma_load_4d(st + kTileBytes, &tmB, &full[s], kb0, 0, ka0, static_cast<int>(no * NT));
        }
      }
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  // warp tile 24 (mi) x 72 (ni): warp row wm covers mo_l = wm / 3, mi 24 * (wm % 3) ..
  const int wm = warp >> 1, wn = warp & 1;
  const int mo_l = wm / 3, m0 = (wm % 3) * 24;
  const int qrow = lane >> 2, qk = lane & 3;
  // A image [mo2][kB][mi][kA] (64-byte rows): swz64 XORs the 16-byte chunk with
  // row bits 1..2 = qrow bits 1..2 (m0 and 8 i are multiples of 8);
  // B image [no2][kA][ni][kB] (32-byte rows): swz32 XORs with row bit 2
  const int a_lane = (mo_l * KB * EXT + m0 + qrow) * 64;
  const int b_lane = (wn * KA * EXT + qrow) * 32;
  const int sA = ((qrow >> 1) & 3) << 4, sB = ((qrow >> 2) & 1) << 4;
  // functional operands (aA x + bA)(aB y + bB): the K-sum is hoisted out of
  // the DMMA loop, C = aA aB S + aA bB rowA + bA aB rowB + bA bB |K|
  const bool affine = p.a_alpha >= 0 || p.b_alpha >= 0;
  const double aA = p.a_alpha >= 0 ? p.coef[2 * p.a_alpha] : 1.0;
  const double bA = p.a_beta >= 0 ? p.coef[2 * p.a_beta] : 0.0;
  const double aB = p.b_alpha >= 0 ? p.coef[2 * p.b_alpha] : 1.0;
  const double bB = p.b_beta >= 0 ? p.coef[2 * p.b_beta] : 0.0;

  std::int64_t it = 0;
  for (std::int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    std::int64_t mo, no;
    const std::int64_t sl = t / per_s, tz = t - sl * per_s;
    const std::int64_t z = tz / per_z;
    tile_coords(tz - z * per_z, mo, no);
    double acc[3][9][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 9; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (std::int64_t ks = k_lo(sl); ks < k_lo(sl + 1); ++ks, ++it) {
      const int s = static_cast<int>(it % S);
      const std::uint32_t round = static_cast<std::uint32_t>(it / S);
      ptx::mbar_wait(&full[s], round & 1u);
      const unsigned char* sa = tiles + static_cast<size_t>(s) * 2 * kTileBytes;
      const unsigned char* sb = sa + kTileBytes;
#pragma unroll
      for (int kc = 0; kc < KT / 4; ++kc) {
        // k chunk of 4: lane's k = (kB e_l, kA f) with f in {0,1,4,5} + 2 (kc >> 2)
        // and e_l = qk ^ (kc & 3). A 64-bit fragment load is served per
        // half-warp (4 rows x 4 k); this choice puts the 16 words of each half
        // in 16 distinct bank pairs on both swizzled images (one wavefront per
        // half, the minimum), and the 8 chunks cover the stage's 8 x 4 k.
        const int e_l = qk ^ (kc & 3);
        const int f = 2 * (kc >> 2) + (qk & 1) + 4 * (qk >> 1);
        // the swizzle XOR only sees row bits (lane constants sA / sB), so each
        // fragment is lane base + per-chunk k offset + an immediate
        const unsigned char* pa = sa + a_lane + e_l * (EXT * 64) + ((f * 8) ^ sA);
        const unsigned char* pb = sb + b_lane + f * (EXT * 32) + ((e_l * 8) ^ sB);
        double af[3], bf[9];
#pragma unroll
        for (int i = 0; i < 3; ++i) af[i] = *reinterpret_cast<const double*>(pa + i * 8 * 64);
#pragma unroll
        for (int j = 0; j < 9; ++j) bf[j] = *reinterpret_cast<const double*>(pb + j * 8 * 32);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 9; ++j) ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }

    // epilogue: fragment (row qrow, cols 2*qk, 2*qk+1) of each 8x8 block;
    // rows / columns beyond ext_mi / ext_ni (a box of 72 over a shorter
    // extent, filled with zeros by TMA) are not stored
    const std::int64_t gmo = mo * MT + mo_l, gno = no * NT + wn;
    if (gmo >= p.ext_mo || gno >= p.ext_no) continue;
    double* cbase = (p.ksplit > 1 ? p.ws + sl * p.csize : p.C) + z * p.c_z + gmo * p.c_mo + gno * p.c_no;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int m = m0 + i * 8 + qrow;
      if (m >= p.ext_mi) continue;
      const double ra = (affine && bB != 0.0) ? p.rowA[gmo * p.ext_mi + m] : 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const int n = j * 8 + 2 * qk;
        if (n >= p.ext_ni) continue;
        const bool pair = n + 1 < p.ext_ni;
        double* dst = cbase + m * p.c_mi + n * p.c_ni;
        if (affine) {
          const double k = bA * bB * p.kdim;
          for (int v = 0; v < 2; ++v) {
            const double rb = (bA != 0.0 && n + v < p.ext_ni) ? p.rowB[gno * p.ext_ni + n + v] : 0.0;
            acc[i][j][v] = fma(aA * aB, acc[i][j][v], fma(aA * bB, ra, fma(bA * aB, rb, k)));
          }
        }
        if (p.vec_c && pair) {
          __stcs(reinterpret_cast<double2*>(dst), make_double2(acc[i][j][0], acc[i][j][1]));
        } else {
          dst[0] = acc[i][j][0];
          if (pair) dst[p.c_ni] = acc[i][j][1];
        }
      }
    }
  }
}

// rows[r0 * n1 + r1] = sum_{c0, c1} X[r0*s_r0 + r1*s_r1 + c0*s_c0 + c1*s_c1], one warp per row
__global__ void rowsum_kernel(const double* __restrict__ X, double* __restrict__ rows, std::int64_t n0,
                              std::int64_t n1, std::int64_t s_r0, std::int64_t s_r1, std::int64_t m0, std::int64_t m1,
                              std::int64_t s_c0, std::int64_t s_c1) {
  const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n0 * n1) return;
  const std::int64_t r0 = warp / n1, r1 = warp % n1;
  const double* base = X + r0 * s_r0 + r1 * s_r1;
  // nested loops (no division per element), four independent partial sums
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int k = 0;
  for (std::int64_t c0 = 0; c0 < m0; ++c0) {
    const double* row = base + c0 * s_c0;
    for (std::int64_t c1 = lane; c1 < m1; c1 += 32, k = (k + 1) & 3) s[k] += __ldg(row + c1 * s_c1);
  }
  double t = (s[0] + s[1]) + (s[2] + s[3]);
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) rows[warp] = t;
}

// C[i] = sum over slices of ws[s * n + i], slices in order
__global__ void ksplit_reduce_kernel(const double* __restrict__ ws, double* __restrict__ C, std::int64_t n, int ks) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    double v = ws[i];
    for (int s = 1; s < ks; ++s) v += ws[s * n + i];
    C[i] = v;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// rank 4, or 5 with a batch dim (box 1) appended
bool make_map(CUtensorMap* map, const double* base, const std::uint64_t dims[5], const std::uint64_t strides_el[5],
              const std::uint32_t box[5], CUtensorMapSwizzle swizzle, int rank = 4) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bdim[5], estr[5] = {1, 1, 1, 1, 1};
  for (int d = 0; d < rank; ++d) {
    gdim[d] = dims[d];
    bdim[d] = box[d];
  }
  for (int d = 1; d < rank; ++d) gstride[d - 1] = strides_el[d] * 8;
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank), const_cast<double*>(base), gdim, gstride, bdim, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// Extents up to one 72-row box per mo / no value (shorter ones are padded
// with zeros by TMA and masked in the epilogue; K extents of any length, the
// last k box likewise zero-padded). Even unit-stride extents keep every TMA
// stride a multiple of 16 bytes; below a third of a box the generic kernel
// is the better choice.
bool gett_supported(std::int64_t ext_mi, std::int64_t ext_ni, std::int64_t ext_ka, std::int64_t ext_kb) {
  return ext_mi >= 24 && ext_mi <= EXT && ext_ni >= 24 && ext_ni <= EXT && ext_ka % 2 == 0 && ext_kb % 2 == 0 &&
         ext_ka * ext_kb >= 64;
}

int launch_gett(const GettLaunch& L, void* stream) {
  if (!gett_supported(L.ext_mi, L.ext_ni, L.ext_ka, L.ext_kb)) return cudaErrorInvalidValue;
  CUtensorMap tmA, tmB;
  const std::int64_t nz = L.nz > 1 ? L.nz : 1;
  const int rank = nz > 1 ? 5 : 4;
  if (nz > 1 && (L.a_alpha >= 0 || L.b_alpha >= 0)) return cudaErrorInvalidValue;  // row sums are per batch
  {
    const std::uint64_t dims[5] = {static_cast<std::uint64_t>(L.ext_ka), static_cast<std::uint64_t>(L.ext_mi),
                                   static_cast<std::uint64_t>(L.ext_kb), static_cast<std::uint64_t>(L.ext_mo),
                                   static_cast<std::uint64_t>(nz)};
    const std::uint64_t str[5] = {1, static_cast<std::uint64_t>(L.a_mi), static_cast<std::uint64_t>(L.a_kb),
                                  static_cast<std::uint64_t>(L.a_mo), static_cast<std::uint64_t>(L.a_z)};
    const std::uint32_t box[5] = {KA, EXT, KB, MT, 1};
    if (!make_map(&tmA, L.A, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B, rank)) return cudaErrorInvalidValue;
  }
  {
    const std::uint64_t dims[5] = {static_cast<std::uint64_t>(L.ext_kb), static_cast<std::uint64_t>(L.ext_ni),
                                   static_cast<std::uint64_t>(L.ext_ka), static_cast<std::uint64_t>(L.ext_no),
                                   static_cast<std::uint64_t>(nz)};
    const std::uint64_t str[5] = {1, static_cast<std::uint64_t>(L.b_ni), static_cast<std::uint64_t>(L.b_ka),
                                  static_cast<std::uint64_t>(L.b_no), static_cast<std::uint64_t>(L.b_z)};
    const std::uint32_t box[5] = {KB, EXT, KA, NT, 1};
    if (!make_map(&tmB, L.B, dims, str, box, CU_TENSOR_MAP_SWIZZLE_32B, rank)) return cudaErrorInvalidValue;
  }
  GettDev d{};
  d.mo = (L.ext_mo + MT - 1) / MT;
  d.no = (L.ext_no + NT - 1) / NT;
  d.ext_mo = L.ext_mo;
  d.ext_no = L.ext_no;
  d.ka_steps = (L.ext_ka + KA - 1) / KA;
  d.kb_steps = (L.ext_kb + KB - 1) / KB;
  d.vec_c = L.c_ni == 1 && L.c_mi % 2 == 0 && L.c_mo % 2 == 0 && L.c_no % 2 == 0 && L.c_z % 2 == 0 &&
            (L.ksplit <= 1 || (L.ext_mo * L.ext_mi * L.ext_no * L.ext_ni * (L.nz > 1 ? L.nz : 1)) % 2 == 0) &&
            (reinterpret_cast<std::uintptr_t>(L.C) & 15) == 0;
  d.c_mo = L.c_mo;
  d.c_mi = L.c_mi;
  d.c_no = L.c_no;
  d.c_ni = L.c_ni;
  d.C = L.C;
  d.coef = L.coef;
  d.a_alpha = L.a_alpha;
  d.a_beta = L.a_beta;
  d.b_alpha = L.b_alpha;
  d.b_beta = L.b_beta;
  d.ext_mi = L.ext_mi;
  d.ext_ni = L.ext_ni;
  d.kdim = static_cast<double>(L.ext_ka) * static_cast<double>(L.ext_kb);
  d.rowA = L.scratch;
  d.rowB = L.scratch + L.ext_mo * L.ext_mi;
  if (L.a_alpha >= 0 || L.b_alpha >= 0) {
    if (!L.scratch) return cudaErrorInvalidValue;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const std::int64_t ra = L.ext_mo * L.ext_mi, rb = L.ext_no * L.ext_ni;
    rowsum_kernel<<<static_cast<int>((ra * 32 + 255) / 256), 256, 0, st>>>(
        L.A, L.scratch, L.ext_mo, L.ext_mi, L.a_mo, L.a_mi, L.ext_kb, L.ext_ka, L.a_kb, 1);
    rowsum_kernel<<<static_cast<int>((rb * 32 + 255) / 256), 256, 0, st>>>(
        L.B, L.scratch + ra, L.ext_no, L.ext_ni, L.b_no, L.b_ni, L.ext_ka, L.ext_kb, L.b_ka, 1);
  }
  d.nz = nz;
  d.c_z = L.c_z;
  d.ksplit = L.ksplit > 1 && L.ws && !(L.a_alpha >= 0 || L.b_alpha >= 0) ? L.ksplit : 1;
  d.ws = L.ws;
  d.csize = L.ext_mo * L.ext_mi * L.ext_no * L.ext_ni * nz;
  d.stages = L.stages > 0 ? L.stages : 3;
  d.group = L.group > 0 ? L.group : 6;
  const size_t smem = 1024 + static_cast<size_t>(d.stages) * 2 * kTileBytes + 16 * d.stages;
  cudaError_t e = cudaFuncSetAttribute(gett_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 148;
  device_sm_count(&sms);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gett_kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  std::int64_t grid = static_cast<std::int64_t>(sms) * per_sm;
  if (L.grid > 0) grid = L.grid;
  if (grid > d.mo * d.no * nz * d.ksplit) grid = d.mo * d.no * nz * d.ksplit;
  gett_kernel<<<static_cast<int>(grid), kThreads, smem, static_cast<cudaStream_t>(stream)>>>(d, tmA, tmB);
  if (d.ksplit > 1) {
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ksplit_reduce_kernel<<<sms * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(d.ws, L.C, d.csize, d.ksplit);
  }
  return cudaGetLastError();
}

}  // namespace feb200
