// K4 — tensor-train layer  Y[n,i,k] = sum_{j,l} G1[i,j] G2[k,l] X[n,j,l]
// (C4: n = 4096 samples, 64x64 cores), i.e. two chained 64^3 GEMMs per sample:
//   T = X_n G2^T   (T[j,k] = sum_l X[j,l] G2[k,l])
//   Y_n = G1 T     (Y[i,k] = sum_j G1[i,j] T[j,k])
//
// B200 design: persistent CTAs, G1/G2 staged once per CTA in shared memory as
// fp64 panels; samples are processed two at a time so each of 8 DMMA warps
// owns a 32x32 tile in both GEMMs (GEMM 1 on the stacked [X_a; X_b] (128x64),
// GEMM 2 on [T_a | T_b] (64x128)) — 0.5 fragment loads per DMMA. For fp64 a
// CTA runs two such 8-warp groups on independent sample pairs (16 warps, four
// per SM sub-partition), each with its own X stage filled by TMA (2-D boxes,
// 128-byte swizzle) and group-local named barriers, so one group's barrier and
// load waits are covered by the other group's DMMAs. T never leaves shared
// memory (fp64 samples write T^T over their consumed X stage; fp32 samples
// use a separate T buffer) and is stored transposed so GEMM 2's fragments are
// conflict-free; the fragment k-map (k0 + {0,1,8,9}) spreads each half-warp
// over all banks under the swizzle. Y goes straight from the accumulators
// with 16-byte stores. Arithmetic: DMMA m8n8k4 (fp64 tensor cores); fp32
// storage is converted on the fragment load and accumulated in fp64 (the
// fp32 default is tt_tc.cu).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int R = 64;                  // core size
constexpr int kConsumerWarps = 8;      // 8 warps x (32 x 32) per GEMM
constexpr int kPair = 2;               // samples per iteration

__device__ __forceinline__ std::uint32_t swz(std::uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

// 64-row matrix stored as column panels of 128-byte rows (the TMA 128B-swizzle
// image): element (r, c) -> panel c / P, row r, column c % P.
template <typename T>
struct Panels {
  static constexpr int P = 128 / sizeof(T);        // columns per panel
  static constexpr int kPanelBytes = R * 128;      // 8 KB, 1024-aligned
  static constexpr int kBytes = kPanelBytes * (R / P);
  __device__ static std::uint32_t off(int r, int c) {
    return (c / P) * kPanelBytes + swz(static_cast<std::uint32_t>(r * 128 + (c % P) * sizeof(T)));
  }
};

template <typename T>
__device__ __forceinline__ double ld(const unsigned char* base, int r, int c) {
  return static_cast<double>(*reinterpret_cast<const T*>(base + Panels<T>::off(r, c)));
}

// Fragment addressing. A DMMA k-chunk gives lane (qr, qk) row r = r0 + 8 a + qr
// and column k = k0 + (qk & 1) + 8 (qk >> 1), k0 in {0, 2, 4, 6} + 16 q: a
// 64-bit load is served per half-warp (4 rows x 4 k), and against the 128B
// swizzle (16-byte chunk ^= r & 7) these k spread each half over all 32 banks
// (adjacent k pairs would hit the same chunks for rows qr and qr ^ 1). The qk
// and k0 parts of the column byte offset occupy disjoint bits, so the address
// splits into a lane base + a per-chunk offset + the immediate 1024 a.
template <typename T>
struct Frag {
  static constexpr int P = Panels<T>::P;
  // bits of the column byte offset owned by qk: double 3 and 6, float 2 and 5
  static constexpr std::uint32_t kQMask = sizeof(T) == 8 ? 0x48u : 0x24u;
  __device__ static std::uint32_t lane(int r0, int qr, int qk) {
    const std::uint32_t sx = static_cast<std::uint32_t>(qr) << 4;
    const std::uint32_t q = static_cast<std::uint32_t>((qk & 1) + 8 * (qk >> 1)) * sizeof(T);
    return static_cast<std::uint32_t>((r0 + qr) * 128) + (q ^ (sx & kQMask));
  }
  __device__ static std::uint32_t kofs(int k0, int qr) {
    const std::uint32_t sx = static_cast<std::uint32_t>(qr) << 4;
    return static_cast<std::uint32_t>((k0 / P) * Panels<T>::kPanelBytes) +
           ((static_cast<std::uint32_t>(k0 % P) * sizeof(T)) ^ (sx & ~kQMask & 0x70u));
  }
  __device__ static double at(const unsigned char* p, int a) {
    return static_cast<double>(*reinterpret_cast<const T*>(p + a * 8 * 128));
  }
};
// k0 of chunk kp (16 chunks of 4 cover k = 0..63)
__device__ __forceinline__ int chunk_k0(int kp) { return (kp >> 2) * 16 + (kp & 3) * 2; }

struct TTDev {
  std::int64_t nb;
  int NI, NJ, NK, NL;  // cores up to 64 x 64, zero-padded to the 64 x 64 tiles
  const void* G1;
  const void* G2;
  void* Y;
  std::int64_t y_sn;  // Y sample stride (elements); rows are i*64 + k
};

// Warp groups of 8 DMMA warps, each with its own single X stage, run
// independent sample pairs (fp64: two groups, 16 warps = four per SM
// sub-partition); while one group waits at its barriers or for its next X
// pair, the other keeps the tensor pipe busy. Warp 0 of a group issues the
// group's TMA once the group has released its stage.
template <typename T>
struct TTShape {
  static constexpr bool kInPlaceT = sizeof(T) == 8;  // T^T overwrites the consumed X stage
  static constexpr int kGroups = sizeof(T) == 8 ? 2 : 1;
  static constexpr int kStageBytes = kPair * Panels<T>::kBytes;
  static constexpr int kGroupBytes = kStageBytes + (kInPlaceT ? 0 : kPair * Panels<double>::kBytes);
  static constexpr int kThreadsT = 32 * kConsumerWarps * kGroups;
  static constexpr size_t kSmem = 1024 + 2 * Panels<double>::kBytes + static_cast<size_t>(kGroups) * kGroupBytes + 64;
};

template <typename T>
__global__ void __launch_bounds__(TTShape<T>::kThreadsT, 1)
    tt_kernel(const __grid_constant__ TTDev p, const __grid_constant__ CUtensorMap tmX) {
  using PT = Panels<T>;
  using PD = Panels<double>;
  using SH = TTShape<T>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  unsigned char* g1 = base;                          // G1 [i][j] fp64 panels
  unsigned char* g2 = g1 + PD::kBytes;               // G2 [k][l] fp64 panels
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(g2 + PD::kBytes + SH::kGroups * SH::kGroupBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / kConsumerWarps, wl = warp % kConsumerWarps;
  unsigned char* xs0 = g2 + PD::kBytes + grp * SH::kGroupBytes;  // this group's X pair
  if (threadIdx.x == 0) {
    for (int g = 0; g < SH::kGroups * kPair; ++g) ptx::mbar_init(&full[g], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const std::int64_t npairs = (p.nb + kPair - 1) / kPair;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * SH::kGroups;
  // the two samples of a pair are independent (each sample's four warps own
  // its GEMMs and its half of the stage): one mbarrier, one TMA issue and one
  // named barrier per sample, so the samples drift apart and cover each
  // other's barrier / store phases on the tensor pipe
  const int smp = wl >> 2;
  const bool leader = (wl & 3) == 0 && lane == 0;
  std::uint64_t* fb = &full[grp * kPair + smp];
  auto issue = [&](std::int64_t pr) {
    ptx::mbar_arrive_expect_tx(fb, PT::kBytes);
    for (int panel = 0; panel < R / PT::P; ++panel) {
      unsigned char* dst = xs0 + smp * PT::kBytes + panel * PT::kPanelBytes;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              ptx::smem_addr(dst)),
          "l"(&tmX), "r"(ptx::smem_addr(fb)), "r"(panel * PT::P), "r"(0), "r"(static_cast<int>(pr * kPair + smp))
          : "memory");
    }
  };
  const std::int64_t first = static_cast<std::int64_t>(blockIdx.x) * SH::kGroups + grp;
  if (leader && first < npairs) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    issue(first);
  }
  // G1/G2 staged (as fp64 panels) while the first X pairs are in flight; all
  // of a thread's global loads are issued before any store so their
  // latencies overlap (one round trip, not R*R/threads of them)
  {
    constexpr int kPer = R * R / SH::kThreadsT;
    static_assert(R * R % SH::kThreadsT == 0, "G staging assumes an even split");
    double v1[kPer], v2[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = threadIdx.x + k * SH::kThreadsT;
      const int r = t / R, c = t % R;
      v1[k] = r < p.NI && c < p.NJ ? static_cast<double>(__ldg(static_cast<const T*>(p.G1) + r * p.NJ + c)) : 0.0;
      v2[k] = r < p.NK && c < p.NL ? static_cast<double>(__ldg(static_cast<const T*>(p.G2) + r * p.NL + c)) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = threadIdx.x + k * SH::kThreadsT;
      *reinterpret_cast<double*>(g1 + PD::off(t / R, t % R)) = v1[k];
      *reinterpret_cast<double*>(g2 + PD::off(t / R, t % R)) = v2[k];
    }
  }
  __syncthreads();
  auto group_sync = [&]() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp * kPair + smp), "n"(kConsumerWarps / kPair * 32) : "memory");
  };

  const int qr = lane >> 2, qk = lane & 3;
  // GEMM 1 tile: stacked rows [32*(w/2), +32) (sample (w/2)/2), cols [32*(w%2), +32)
  const int r1 = (wl >> 1) * 32 - smp * R, c1 = (wl & 1) * 32;
  // GEMM 2 tile (same sample): rows i [32*(w%2), +32), cols k [32*((w>>1)&1), +32)
  const int r2 = (wl & 1) * 32, c2 = ((wl >> 1) & 1) * 32;
  const std::uint32_t a1_lane = Frag<T>::lane(r1, qr, qk), b1_lane = Frag<double>::lane(c1, qr, qk);
  const std::uint32_t a2_lane = Frag<double>::lane(r2, qr, qk), b2_lane = Frag<double>::lane(c2, qr, qk);
  unsigned char* xs = xs0 + smp * PT::kBytes;
  unsigned char* ts = SH::kInPlaceT ? xs : xs0 + SH::kStageBytes + smp * PD::kBytes;
  int it = 0;
  for (std::int64_t pr = first; pr < npairs; pr += stride, ++it) {
    ptx::mbar_wait(fb, it & 1u);

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // GEMM 1: T[j,k] = sum_l X[j,l] G2[k,l]
#pragma unroll 4
    for (int kp = 0; kp < R / 4; ++kp) {
      const int k0 = chunk_k0(kp);
      double af[4], bf[4];
      const unsigned char* pa = xs + a1_lane + Frag<T>::kofs(k0, qr);
      const unsigned char* pb = g2 + b1_lane + Frag<double>::kofs(k0, qr);
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = Frag<T>::at(pa, a);
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Frag<double>::at(pb, b);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) ptx::dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    // all X of the pair consumed before T^T may overwrite it
    group_sync();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int j = r1 + a * 8 + qr, k = c1 + b * 8 + 2 * qk + v;
          *reinterpret_cast<double*>(ts + PD::off(k, j)) = acc[a][b][v];
        }
    group_sync();

    // GEMM 2: Y[i,k] = sum_j G1[i,j] T[j,k]
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int kp = 0; kp < R / 4; ++kp) {
      const int k0 = chunk_k0(kp);
      double af[4], bf[4];
      const std::uint32_t ko = Frag<double>::kofs(k0, qr);
      const unsigned char* pa = g1 + a2_lane + ko;
      const unsigned char* pb = ts + b2_lane + ko;
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = Frag<double>::at(pa, a);
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Frag<double>::at(pb, b);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) ptx::dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    // the group's stage (X, and T^T when in place) is free once every warp of
    // the group has read it: refill it while the Y tiles drain
    group_sync();
    if (leader && pr + stride < npairs) issue(pr + stride);

    const std::int64_t n = pr * kPair + smp;
    if (n < p.nb) {
      T* y = static_cast<T*>(p.Y) + n * p.y_sn;
      const bool full = p.NI == R && p.NK == R;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = r2 + a * 8 + qr, k = c2 + b * 8 + 2 * qk;
          if (full) {
            if constexpr (sizeof(T) == 8) {
              __stcs(reinterpret_cast<double2*>(y + i * R + k), make_double2(acc[a][b][0], acc[a][b][1]));
            } else {
              __stcs(reinterpret_cast<float2*>(y + i * R + k),
                     make_float2(static_cast<float>(acc[a][b][0]), static_cast<float>(acc[a][b][1])));
            }
          } else if (i < p.NI) {  // padded core: rows / columns beyond the real extents are zeros
            if (k < p.NK) y[i * p.NK + k] = static_cast<T>(acc[a][b][0]);
            if (k + 1 < p.NK) y[i * p.NK + k + 1] = static_cast<T>(acc[a][b][1]);
          }
        }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

template <typename T>
int launch_t(const TTLaunch& L, cudaStream_t stream) {
  using PT = Panels<T>;
  using PD = Panels<double>;
  auto enc = encoder();
  if (!enc) return cudaErrorInvalidValue;
  CUtensorMap tm;
  // X viewed as (l, j, n): unit stride l, then j, then the sample stride
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(L.NL), static_cast<cuuint64_t>(L.NJ), static_cast<cuuint64_t>(L.Nb)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(L.x_sj * sizeof(T)), static_cast<cuuint64_t>(L.x_sn * sizeof(T))};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(PT::P), static_cast<cuuint32_t>(R), 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(&tm, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                         const_cast<void*>(L.X), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  TTDev d{};
  d.nb = L.Nb;
  d.NI = L.NI;
  d.NJ = L.NJ;
  d.NK = L.NK;
  d.NL = L.NL;
  d.G1 = L.G1;
  d.G2 = L.G2;
  d.Y = L.Y;
  d.y_sn = L.y_sn;
  const size_t smem = TTShape<T>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(tt_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 148;
  device_sm_count(&sms);
  const std::int64_t npairs = (L.Nb + kPair - 1) / kPair;
  std::int64_t grid = (npairs + TTShape<T>::kGroups - 1) / TTShape<T>::kGroups;
  if (grid > sms) grid = sms;
  tt_kernel<T><<<static_cast<int>(grid), TTShape<T>::kThreadsT, smem, stream>>>(d, tm);
  return cudaGetLastError();
}

}  // namespace

// cores up to 64 x 64 (padded with zeros to the kernel's 64 x 64 tiles: the
// X boxes by TMA out-of-bounds fill, G1/G2 when staged, Y masked); the
// unit-stride extent NL must keep the TMA strides 16-byte multiples
bool tt_supported(int NI, int NJ, int NK, int NL, bool fp32) {
  return NI >= 8 && NI <= R && NJ >= 8 && NJ <= R && NK >= 8 && NK <= R && NL >= 8 && NL <= R &&
         NL % (fp32 ? 4 : 2) == 0;
}

int launch_tt(const TTLaunch& L, void* stream) {
  if (!tt_supported(L.NI, L.NJ, L.NK, L.NL, L.fp32 != 0) || L.Nb <= 0) return L.Nb == 0 ? cudaSuccess : cudaErrorInvalidValue;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return L.fp32 ? launch_t<float>(L, s) : launch_t<double>(L, s);
}

}  // namespace feb200
