// K4 (fp32) — tensor-train step on the 5th-generation tensor cores
//
//   Y[n,i,k] = sum_{j,l} G1[i,j] G2[k,l] X[n,j,l]        (C4-f32: 4096 x 64^4)
//
// as two chained GEMMs per PAIR of samples, both M = 128 (rows = two samples
// x 64), K = 64, on tcgen05.mma.cta_group::1.kind::tf32 into TMEM:
//   GEMM1  T [(n,j), k] = sum_l X[(n,j), l] G2[k, l]      A = X hi / lo in TMEM
//   GEMM2  Y^T[(n,k), i] = sum_j T^T[(n,k), j] G1[i, j]   A = T^T (shared, SW128)
//
// fp32 accuracy from the TF32 datapath (3xTF32): every operand is split into
// hi = tf32(x) and lo = tf32(x - hi), both rounded to nearest (split_tf32),
// and each GEMM accumulates hi*hi + hi*lo + lo*hi in fp32 (the dropped
// remainders are ~2^-22 relative and unbiased); tests/test_benched_parity.py
// holds it to the flat fp32 bar (1e-5 against double).
//
// Warp roles (one CTA per SM, persistent over sample pairs):
//   warp 16 — walks the schedule as a whole warp (uniform control flow keeps
//             every descriptor in uniform registers); one elected lane issues
//             the X TMA (128-row x 128-byte boxes) and the MMAs. Computing
//             descriptors per MMA in a divergent lane made MMA issue, not the
//             tensor core, the bottleneck (tools/tcgen05_rate.cu measures the
//             issue/complete rates: tf32 N=64 45 cyc, N=128 64 cyc);
//   warps 0-15 — 4 TMEM lane quarters x 4 16-column groups: split X into
//             hi / lo straight into TMEM (tcgen05.st; GEMM1 reads A from TMEM,
//             so its only shared traffic is B), epilogue 1 (D1 -> registers ->
//             hi/lo T^T tile in shared memory, transposed on the way with
//             conflict-free 128-byte rows, double-buffered so it never waits
//             for GEMM2 of the previous pair), epilogue 2 (D2 -> coalesced
//             global stores of Y).
// GEMM1 runs three N = 64 products into one 64-column D1 (small terms first);
// GEMM2 runs Ah [Bh;Bl] (N = 128) + Al Bh (N = 64) into a 128-column D2.
// Schedule: GEMM1(t+1) is issued before GEMM2(t); TMEM: D1[2], D2[2], X hi/lo.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {

namespace {

constexpr int R = 64;
constexpr int kRows = 128;                   // two samples per tile
constexpr int kTile = kRows * R * 4;         // 32 KB: [2 k-blocks][128 rows][128 B]
constexpr int kKBlockA = kRows * 128;        // 16 KB
constexpr int kG = 2 * R * R * 4;            // 32 KB: [2 k-blocks][128 rows = hi 64 | lo 64][128 B]
constexpr int kKBlockB = 2 * R * 128;        // 16 KB
constexpr int kEpiWarps = 16;                // 4 column groups x 4 TMEM lane quarters
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = kEpiThreads + 32;
constexpr std::uint32_t kTmemCols = 512;
// TMEM columns: D1[2] (64 each), D2[2] (128 each), X hi / lo (A of GEMM1, 64 each)
__host__ __device__ constexpr std::uint32_t d1_col(int b) { return static_cast<std::uint32_t>(b * 64); }
__host__ __device__ constexpr std::uint32_t d2_col(int b) { return static_cast<std::uint32_t>(128 + b * 128); }
constexpr std::uint32_t kXhCol = 384, kXlCol = 448;
// instruction descriptor: D f32, A/B tf32, K-major both, M = 128, N = n
constexpr std::uint32_t idesc(std::uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

struct TTTcDev {
  std::int64_t nb, npairs;
  const float* G1;
  const float* G2;
  float* Y;
  std::int64_t y_sn;
  unsigned long long* trace;  // -DFE_TT_TRACE builds: per-phase timestamps of CTA 0
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef FE_TT_TRACE
#define TT_TRACE(t, slot) \
  if (p.trace && blockIdx.x == 0 && (t) < 64) p.trace[(t) * 16 + (slot)] = gtime();
#else
#define TT_TRACE(t, slot) {}
#endif

// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ std::uint64_t sdesc(const void* p) {
  return static_cast<std::uint64_t>((ptx::smem_addr(p) >> 4) & 0x3FFF) | (std::uint64_t{1} << 16) |
         (std::uint64_t{1024 >> 4} << 32) | (std::uint64_t{1} << 46) | (std::uint64_t{2} << 61);
}

// byte offset of element (r, k) in a [rows x 64] fp32 K-major SW128 tile
__device__ __forceinline__ std::uint32_t sw_off(int r, int k, int rows) {
  const int kb = k >> 5, kk = k & 31;
  return static_cast<std::uint32_t>(kb * rows * 128 + r * 128 + ((((kk >> 2) ^ (r & 7)) << 4) | ((kk & 3) << 2)));
}

__device__ __forceinline__ void mma_tf32(std::uint32_t tmem, std::uint64_t da, std::uint64_t db, std::uint32_t id,
                                         std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}

// A from TMEM (columns a_tmem .. +8: one K8 step, row = lane), B from shared memory
__device__ __forceinline__ void mma_tf32_ts(std::uint32_t tmem, std::uint32_t a_tmem, std::uint64_t db, std::uint32_t id,
                                            std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
      "r"(a_tmem), "l"(db), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(ptx::smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 lanes x 16 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 16 consecutive 32-bit columns, registers -> TMEM
__device__ __forceinline__ void tmem_st16(std::uint32_t taddr, const std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(ptx::smem_addr(dst)),
      "l"(map), "r"(ptx::smem_addr(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 3xTF32 split with round-to-nearest on both parts: hi = rna_tf32(x), lo =
// rna_tf32(x - hi) (x - hi is exact in fp32). The tensor core truncates the
// low 13 mantissa bits of an fp32 operand; with a truncated split every
// dropped remainder has the sign of x, and the bias grows linearly over the
// 4096 products of a TT output (measured 1.5e-5 against double on the
// reference's random_bindings data); rounded parts leave unbiased remainders
// below 2^-22 |x| (the fp32 bar of SURVEY.md §8c, 1e-5, holds flat).
__device__ __forceinline__ float tf32_rna(float x) {
  std::uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split_tf32(float x, float& h, float& l) {
  h = tf32_rna(x);
  l = tf32_rna(x - h);
}

// one 3xTF32 GEMM over K = 64 (8 k-steps of 8), B = [Bh ; Bl] stacked on N:
//   D[:, 0:128]  = Ah * [Bh ; Bl]^T     (N = 128: the hi*hi and hi*lo terms side by side)
//   D[:, 0:64]  += Al * Bh^T            (N = 64)
// the epilogue adds the two 64-column halves in fp32
// Descriptors are passed as precomputed bases: the start-address field is the
// low 14 bits (address >> 4), so a tile offset is a compile-time add. The MMA
// thread issues ~one instruction per MMA besides the MMA itself; computing the
// descriptors in the loop made issue (not the tensor core) the bottleneck.
__device__ __forceinline__ void gemm3(std::uint32_t d, std::uint64_t ah, std::uint64_t al, std::uint64_t bhl) {
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int kb = ks >> 2, kin = (ks & 3) * 32;
    mma_tf32(d, ah + ((kb * kKBlockA + kin) >> 4), bhl + ((kb * kKBlockB + kin) >> 4), idesc(128), ks != 0);
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int kb = ks >> 2, kin = (ks & 3) * 32;
    mma_tf32(d, al + ((kb * kKBlockA + kin) >> 4), bhl + ((kb * kKBlockB + kin) >> 4), idesc(64), 1);
  }
}

// GEMM1 with A (X hi / lo) in TMEM: three N = 64 products accumulated in one
// 64-column D1, small terms first: Xl G2h^T, Xh G2l^T, Xh G2h^T. B reads are
// the only shared-memory traffic of the MMA (2 KB per instruction).
__device__ __forceinline__ void gemm1_ts(std::uint32_t d, std::uint32_t xh, std::uint32_t xl, std::uint64_t g2) {
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int kb = ks >> 2, kin = (ks & 3) * 32;
    mma_tf32_ts(d, xl + ks * 8, g2 + ((kb * kKBlockB + kin) >> 4), idesc(64), ks != 0);
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int kb = ks >> 2, kin = (ks & 3) * 32;
    mma_tf32_ts(d, xh + ks * 8, g2 + ((kb * kKBlockB + R * 128 + kin) >> 4), idesc(64), 1);
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int kb = ks >> 2, kin = (ks & 3) * 32;
    mma_tf32_ts(d, xh + ks * 8, g2 + ((kb * kKBlockB + kin) >> 4), idesc(64), 1);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    tt_tc_kernel(const __grid_constant__ TTTcDev p, const __grid_constant__ CUtensorMap tmX) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  unsigned char* g2 = base;  // [G2 hi ; G2 lo], B of GEMM1
  unsigned char* g1 = base + kG;  // [G1 hi ; G1 lo], B of GEMM2
  unsigned char* xs0 = base + 2 * kG;  // X pair tile (split into TMEM hi / lo, then refilled)
  unsigned char* a2 = xs0 + kTile;     // T^T [2 buffers][hi, lo]: B of GEMM2(t) while epilogue 1 fills t+1
  auto a2h = [&](int b) { return a2 + b * 2 * kTile; };
  auto a2l = [&](int b) { return a2 + b * 2 * kTile + kTile; };
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(a2 + 4 * kTile);
  std::uint64_t* x_full = bars;         // [2]
  std::uint64_t* d1_full = bars + 2;    // [2]
  std::uint64_t* d2_full = bars + 4;    // [2]
  std::uint64_t* d1_free = bars + 6;    // [2]
  std::uint64_t* d2_free = bars + 8;    // [2]
  std::uint64_t* lo_ready = bars + 10;
  std::uint64_t* a2_ready = bars + 11;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 12);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // constants: G2 as B of GEMM1 ([k][l], K = l), G1 as B of GEMM2 ([i][j], K = j), split hi / lo
  // all global loads first (one latency), then the split stores
  {
    constexpr int kPer = (R * R + kThreads - 1) / kThreads;
    float va[kPer], vb[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + k * kThreads;
      va[k] = idx < R * R ? __ldg(p.G2 + idx) : 0.f;
      vb[k] = idx < R * R ? __ldg(p.G1 + idx) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + k * kThreads;
      if (idx >= R * R) break;
      const int r = idx >> 6, c = idx & 63;
      float ah, al, bh, bl;
      split_tf32(va[k], ah, al);
      split_tf32(vb[k], bh, bl);
      *reinterpret_cast<float*>(g2 + sw_off(r, c, 2 * R)) = ah;
      *reinterpret_cast<float*>(g2 + sw_off(R + r, c, 2 * R)) = al;
      *reinterpret_cast<float*>(g1 + sw_off(r, c, 2 * R)) = bh;
      *reinterpret_cast<float*>(g1 + sw_off(R + r, c, 2 * R)) = bl;
    }
  }
  if (warp == kEpiWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_addr(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kEpiThreads) {
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&x_full[b], 1);
      ptx::mbar_init(&d1_full[b], 1);
      ptx::mbar_init(&d2_full[b], 1);
      ptx::mbar_init(&d1_free[b], kEpiWarps);
      ptx::mbar_init(&d2_free[b], kEpiWarps);
    }
    ptx::mbar_init(lo_ready, kEpiWarps);
    ptx::mbar_init(a2_ready, kEpiWarps);
    ptx::fence_barrier_init();
  }
  ptx::fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
  const std::uint32_t tmem = *tmem_slot;

  // local pair t -> global pair blockIdx.x + t * gridDim.x
  const std::int64_t T = p.npairs > blockIdx.x ? (p.npairs - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == kEpiWarps) {
    // --------------------------- TMA + MMA thread ---------------------------
    // order: GEMM1(0); then per t: GEMM2(t), GEMM1(t+1) — so GEMM2(t) runs
    // while the epilogue splits X(t+1), and GEMM1(t+1) while it drains Y(t).
    // The whole warp walks the schedule (uniform control flow keeps the
    // descriptors in uniform registers); one elected lane issues.
    {
      const bool leader = ptx::elect_one();
      if (leader) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
      auto tma_x = [&](std::int64_t t) {
        const int row0 = static_cast<int>((blockIdx.x + t * gridDim.x) * kRows);
        ptx::mbar_arrive_expect_tx(&x_full[0], kTile);
        tma_2d(xs0, &tmX, &x_full[0], 0, row0);
        tma_2d(xs0 + kKBlockA, &tmX, &x_full[0], 32, row0);
      };
      const std::uint64_t dg1 = sdesc(g1), dg2 = sdesc(g2);
      const std::uint64_t da2h0 = sdesc(a2h(0)), da2l0 = sdesc(a2l(0)), da2h1 = sdesc(a2h(1)), da2l1 = sdesc(a2l(1));
      auto gemm1 = [&](std::int64_t t) {
        const int b = static_cast<int>(t & 1);
        ptx::mbar_wait(lo_ready, static_cast<std::uint32_t>(t & 1));
        TT_TRACE(t, 0)
        // split(t) has read the X tile: load X(t+1); it lands long before
        // split(t+1), which follows GEMM1(t)
        if (leader && t + 1 < T) tma_x(t + 1);
        if (t >= 2) ptx::mbar_wait(&d1_free[b], static_cast<std::uint32_t>((t >> 1) - 1) & 1u);
        tc_after();
        if (leader) {
          gemm1_ts(tmem + d1_col(b), tmem + kXhCol, tmem + kXlCol, dg2);
          mma_commit(&d1_full[b]);
        }
        __syncwarp();
        TT_TRACE(t, 1)
      };
      if (leader && T > 0) tma_x(0);
      if (T > 0) gemm1(0);
      for (std::int64_t t = 0; t < T; ++t) {
        const int b = static_cast<int>(t & 1);
        // GEMM1(t+1) first: it runs while the epilogue warps turn T(t) into T^T
        if (t + 1 < T) gemm1(t + 1);
        ptx::mbar_wait(a2_ready, static_cast<std::uint32_t>(t & 1));
        TT_TRACE(t, 2)
        if (t >= 2) ptx::mbar_wait(&d2_free[b], static_cast<std::uint32_t>((t >> 1) - 1) & 1u);
        tc_after();
        if (leader) {
          gemm3(tmem + d2_col(b), b ? da2h1 : da2h0, b ? da2l1 : da2l0, dg1);
          mma_commit(&d2_full[b]);
        }
        __syncwarp();
        TT_TRACE(t, 3)
      }
    }
  } else {
    // ------------------------ split + epilogue warps ------------------------
    // warp = (column group cg, TMEM lane quarter q): rows q*32 + lane, 16 columns
    const int q = warp & 3, cg = warp >> 2;
    const int row = q * 32 + lane;
    const std::uint32_t tl_row = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + static_cast<std::uint32_t>(cg * 16);
    const std::uint32_t tl = tl_row;
    // split: X rows from the TMA tile (thread = row, 16 columns l of its warp's
    // column group, four 16-byte loads) into TMEM hi / lo, the A operand of
    // GEMM1. The caller has seen GEMM1(t-1) complete (TMEM X free).
    auto split = [&](std::int64_t t) {
      const int b = static_cast<int>(t & 1);
      ptx::mbar_wait(&x_full[0], static_cast<std::uint32_t>(t & 1));
      if (tid == 0) TT_TRACE(t, 9)
      const unsigned char* xs = xs0 + (cg >> 1) * kKBlockA + row * 128;
      std::uint32_t h[16], l[16];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int chunk = ((cg & 1) * 4 + c4) ^ (row & 7);
        const float4 x = *reinterpret_cast<const float4*>(xs + chunk * 16);
        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float hv, lv;
          split_tf32(xv[e], hv, lv);
          h[c4 * 4 + e] = __float_as_uint(hv);
          l[c4 * 4 + e] = __float_as_uint(lv);
        }
      }
      tmem_st16(tl_row + kXhCol, h);
      tmem_st16(tl_row + kXlCol, l);
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(lo_ready);
      if (tid == 0) TT_TRACE(t, 6)
    };
    // epilogue 2: row = (n, k): Y[n][i][k] = D2[row][i]; lanes on consecutive k -> 128-byte stores
    auto epi2 = [&](std::int64_t t1) {
      const int b1 = static_cast<int>(t1 & 1);
      std::uint32_t v[16], w[16];
      tmem_ld16(tl + d2_col(b1), v);
      tmem_ld16(tl + d2_col(b1) + 64, w);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&d2_free[b1]);
      const std::int64_t n = (blockIdx.x + t1 * gridDim.x) * 2 + (row >> 6);
      if (n < p.nb) {
        float* y = p.Y + n * p.y_sn + static_cast<std::int64_t>(cg * 16) * R + (row & 63);
#pragma unroll
        for (int c = 0; c < 16; ++c) __stcs(y + c * R, __uint_as_float(v[c]) + __uint_as_float(w[c]));
      }
      if (tid == 0) TT_TRACE(t1, 8)
    };
    if (T > 0) split(0);
    for (std::int64_t t = 0; t < T; ++t) {
      const int b = static_cast<int>(t & 1);
      const std::uint32_t par = static_cast<std::uint32_t>(t >> 1) & 1u;
      ptx::mbar_wait(&d1_full[b], par);
      if (tid == 0) TT_TRACE(t, 4)
      // GEMM1(t) is done with the lo tile: split X(t+1) so GEMM1(t+1) can start
      if (t + 1 < T) split(t + 1);
      // epilogue 1: T[(n,j)][k] -> T^T hi/lo tile b, element ((n,k), j); its
      // last reader GEMM2(t-2) completed before epilogue 2 of t-2 ran
      tc_after();
      std::uint32_t v[16];
      if (tid == 0) TT_TRACE(t, 10)
      tmem_ld16(tl + d1_col(b), v);
      tmem_wait_ld();
      if (tid == 0) TT_TRACE(t, 11)
      tc_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&d1_free[b]);
      {
        const int n = row >> 6, j = row & 63;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float h, l;
          split_tf32(__uint_as_float(v[c]), h, l);
          const std::uint32_t o = sw_off(n * 64 + cg * 16 + c, j, kRows);
          *reinterpret_cast<float*>(a2h(b) + o) = h;
          *reinterpret_cast<float*>(a2l(b) + o) = l;
        }
      }
      if (tid == 0) TT_TRACE(t, 12)
      ptx::fence_proxy_async();
      if (tid == 0) TT_TRACE(t, 13)
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(a2_ready);
      if (tid == 0) TT_TRACE(t, 5)
      if (tid == 32 * 15) TT_TRACE(t, 14)
      // epilogue 2 of the previous pair (its D2 buffer is not the one GEMM2(t) writes)
      if (t >= 1) {
        ptx::mbar_wait(&d2_full[(t - 1) & 1], static_cast<std::uint32_t>((t - 1) >> 1) & 1u);
        if (tid == 0) TT_TRACE(t - 1, 7)
        tc_after();
        epi2(t - 1);
      }
    }
    if (T > 0) {
      ptx::mbar_wait(&d2_full[(T - 1) & 1], static_cast<std::uint32_t>((T - 1) >> 1) & 1u);
      tc_after();
      epi2(T - 1);
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == kEpiWarps) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

PFN_cuTensorMapEncodeTiled_v12000 tc_encoder() {
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

}  // namespace

bool tt_tc_supported(const TTLaunch& L) {
  return L.fp32 && L.NI == R && L.NJ == R && L.NK == R && L.NL == R && L.x_sj == R && L.x_sn == R * R && L.y_sn == R * R &&
         (reinterpret_cast<std::uintptr_t>(L.X) & 15) == 0 && (reinterpret_cast<std::uintptr_t>(L.Y) & 15) == 0;
}

int launch_tt_tc(const TTLaunch& L, void* stream) {
  if (L.Nb == 0) return cudaSuccess;
  if (!tt_tc_supported(L)) return cudaErrorInvalidValue;
  auto enc = tc_encoder();
  if (!enc) return cudaErrorInvalidValue;
  // X as a 2-D [Nb*64 rows][64] fp32 matrix; boxes of 128 rows x 32 columns (128 B)
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(L.Nb) * R};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(R) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kRows)};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(L.X), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  TTTcDev d{};
  d.nb = L.Nb;
  d.npairs = (L.Nb + 1) / 2;
  d.G1 = static_cast<const float*>(L.G1);
  d.G2 = static_cast<const float*>(L.G2);
  d.Y = static_cast<float*>(L.Y);
  d.y_sn = L.y_sn;
  const size_t smem = 1024 + 2 * kG + 5 * kTile + 16 * sizeof(std::uint64_t);
  cudaError_t e = cudaFuncSetAttribute(tt_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 148;
  device_sm_count(&sms);
  std::int64_t grid = sms;
  if (grid > d.npairs) grid = d.npairs;
#ifdef FE_TT_TRACE
  static const bool tracing = std::getenv("FE_TT_TRACE") != nullptr;
#else
  constexpr bool tracing = false;
#endif
  if (tracing) {
    cudaMalloc(&d.trace, 64 * 16 * 8);
    cudaMemset(d.trace, 0, 64 * 16 * 8);
  }
  tt_tc_kernel<<<static_cast<int>(grid), kThreads, smem, static_cast<cudaStream_t>(stream)>>>(d, tm);
  if (tracing) {
    unsigned long long h[64 * 16];
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaMemcpy(h, d.trace, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d.trace);
    unsigned long long t0 = h[9];
    std::fprintf(stderr, "t: xfull | lo_rdy mma:lo g1c | epi:d1 a2rdy | mma:a2 g2c | epi:d2 ystore  (ns from x_full(0))\n");
    for (int t = 0; t < 14; ++t) {
      auto f = [&](int k) { return h[t * 16 + k] ? static_cast<long long>(h[t * 16 + k] - t0) : -1LL; };
      std::fprintf(stderr, "%2d: %6lld | %6lld %6lld %6lld | %6lld %6lld | %6lld %6lld | %6lld %6lld || ld %6lld %6lld sts %6lld fence %6lld w15 %6lld\n", t, f(9), f(6),
                   f(0), f(1), f(4), f(5), f(2), f(3), f(7), f(8), f(10), f(11), f(12), f(13), f(14));
    }
  }
  return cudaGetLastError();
}

}  // namespace feb200
