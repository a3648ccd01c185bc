// K1 kernel body (fem_grad_body), shared by the prebuilt instances in
// fem_grad.cu and the plan-time NVRTC instances that fuse generated operand
// programs into the prologue and a pointwise epilogue into the stores
// (codegen.cpp). Device code only, no host headers (rtc_std.h).
//
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
#pragma once

#include "launch.h"
#include "ptx.cuh"

namespace feb200 {
namespace fem {


struct Coef {
  double pre, post;  // 1.0 when absent (x * 1.0 == x exactly)
  int sign;
};

// element type: fp64 (C1 / C5) or fp32 (float32 einsums of the same shape;
// the same kernel with half the bytes per element)
template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }

// ---- prologue policies: how the consumers build row q's U tile (uc) from
// the stage's staged leaf tiles (su), once per tile ----
struct FemProPlain {  // every row reads one leaf tile as is
  static constexpr bool kPlain = true;
  static constexpr bool kPipe = false;
  template <typename T, int kUTile, int kConsumers>
  __device__ static void combine(const FemGradLaunch&, const T*, T*, const Coef*, int, std::int64_t, std::int64_t) {}
};

struct FemProAffine {  // affine combinations of leaf tiles (C5: u + 0.5 k)
  static constexpr bool kPlain = false;
  static constexpr bool kPipe = false;
  template <typename T, int kUTile, int kConsumers>
  __device__ static void combine(const FemGradLaunch& p, const T* su, T* uc, const Coef* coefs, int c, std::int64_t,
                                 std::int64_t) {
    using V2 = typename Vec2<T>::type;
    // (pre * leaf) * post per term, terms accumulated left to right — the
    // operand's own order; two values per thread and iteration (16-byte
    // shared accesses), the two-term form a*x +- b*y with its coefficients
    // in registers
    auto term = [](const Coef& cf, T v) { return mul_rn(mul_rn(static_cast<T>(cf.pre), v), static_cast<T>(cf.post)); };
    auto join = [](const Coef& cf, T acc, T x) { return cf.sign > 0 ? add_rn(acc, x) : sub_rn(acc, x); };
    for (int q = 0; q < p.rows; ++q) {
      const int u0 = p.row_u_first[q], nt = p.row_u_count[q];
      const V2* s0 = reinterpret_cast<const V2*>(su + u0 * kUTile);
      V2* o = reinterpret_cast<V2*>(uc + q * kUTile);
      if (nt == 2) {
        const Coef c0 = coefs[u0], c1 = coefs[u0 + 1];
        const V2* s1 = s0 + kUTile / 2;
        for (int v = c; v < kUTile / 2; v += kConsumers) {
          const V2 a = s0[v], b = s1[v];
          o[v] = mk2(join(c1, term(c0, a.x), term(c1, b.x)), join(c1, term(c0, a.y), term(c1, b.y)));
        }
      } else {
        for (int v = c; v < kUTile / 2; v += kConsumers) {
          const Coef c0 = coefs[u0];
          const V2 a = s0[v];
          V2 acc = mk2(term(c0, a.x), term(c0, a.y));
          for (int k = 1; k < nt; ++k) {
            const Coef ck = coefs[u0 + k];
            const V2 b = s0[k * (kUTile / 2) + v];
            acc = mk2(join(ck, acc.x, term(ck, b.x)), join(ck, acc.y, term(ck, b.y)));
          }
          o[v] = acc;
        }
      }
    }
  }
};

// ---- epilogue policies: pointwise map of each result value before its store
// (su: the stage's staged leaf tiles, which hold e0..e0+TE of every staged
// [E, NJ] array, so epilogue reads of those come from shared memory) ----
struct FemEpiNone {
  static constexpr bool kIdentity = true;
  template <typename T>
  __device__ static T apply(const FemGradLaunch&, int, int, std::int64_t, int, T y, const T*, std::int64_t) {
    return y;
  }
};

// kDSmem: read D from shared memory (broadcast LDS.128) instead of holding
// D[x,i,:] in 60 registers — halves the register footprint so two CTAs fit
// per SM (more warps in flight for the HBM-bound loop); chosen per fact meta.
// EPT: elements per consumer thread (el, el + TE/EPT, ...): more independent
// FMA chains per thread and D reused from registers across them.
// Consumer threads: TE * NI / EPT, padded to whole warps (tiles such as
// TE = 34 / 68 that make E = 1e4 exactly one tile per CTA slot leave a few
// padding threads idle).
template <int NX, int NR, int NI, int NJ, int TE, int EPT>
constexpr int fem_consumers() {
  return (TE * NI / EPT + 31) / 32 * 32;
}

template <typename T, int NX, int NR, int NI, int NJ, int TE, class Pro, bool kDSmem, int EPT, class Epi>
__device__ __forceinline__ void fem_grad_body(const FemGradLaunch& p) {
  constexpr bool kPlainU = Pro::kPlain;
  using V2 = typename Vec2<T>::type;
  static_assert(TE * sizeof(T) % 16 == 0, "bulk-copy rows are 16-byte multiples");
  constexpr int kConsumers = fem_consumers<NX, NR, NI, NJ, TE, EPT>();
  constexpr int kWorkers = TE * NI / EPT;  // consumers with an (element, i) task
  constexpr int kES = TE / EPT;  // element stride between a thread's elements
  static_assert(TE % EPT == 0 && TE % 2 == 0, "tile shape");
  constexpr int kConsumerWarps = kConsumers / 32;
  static_assert(NJ % 2 == 0, "U rows are read as double2");
  constexpr int kUTile = TE * NJ;          // doubles per U tile
  constexpr int kJTile = NX * NR * TE;     // doubles per J tile

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = p.stages;
  const int stage_doubles = p.n_j * kJTile + p.n_u * kUTile;
  T* dsm = reinterpret_cast<T*>(smem_raw);                         // D copies
  T* ring = dsm + p.n_d * NX * NI * NJ;                            // stages
  // combined U tiles: 2 buffers, or 3 for the pipelined prologue (Pro::kPipe)
  constexpr int kUBufs = kPlainU ? 0 : (Pro::kPipe ? 3 : 2);
  T* ucomb = ring + static_cast<size_t>(S) * stage_doubles;        // [kUBufs][rows][TE*NJ]
  Coef* coefs = reinterpret_cast<Coef*>(
      (reinterpret_cast<std::uintptr_t>(ucomb + kUBufs * p.rows * kUTile) + 15) & ~std::uintptr_t{15});
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(coefs + kFemMaxUTiles);
  std::uint64_t* empty = full + S;
  std::uint64_t* ufull = empty + S;  // kPipe: combined tile b complete (one arrive per consumer warp)

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const std::int64_t E = p.E;
  const std::int64_t ntiles = (E + TE - 1) / TE;

  const std::uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](std::int64_t tile, int s) {
    const std::int64_t e0 = tile * TE;
    const int cnt = static_cast<int>(E - e0 < TE ? E - e0 : TE);
    const std::uint32_t jb = static_cast<std::uint32_t>(cnt * sizeof(T));
    const std::uint32_t ub = static_cast<std::uint32_t>(cnt * NJ * sizeof(T));
    ptx::mbar_arrive_expect_tx(&full[s], static_cast<std::uint32_t>(p.n_j * NX * NR) * jb +
                                             static_cast<std::uint32_t>(p.n_u) * ub);
    T* st = ring + static_cast<size_t>(s) * stage_doubles;
    for (int a = 0; a < p.n_j; ++a)
      for (int xr = 0; xr < NX * NR; ++xr)
        ptx::bulk_g2s_hint(st + a * kJTile + xr * TE, reinterpret_cast<const T*>(p.J[a]) + xr * E + e0, jb, &full[s], pol);
    T* su = st + p.n_j * kJTile;
    for (int u = 0; u < p.n_u; ++u)
      ptx::bulk_g2s_hint(su + u * kUTile, reinterpret_cast<const T*>(p.U[u]) + e0 * NJ, ub, &full[s], pol);
  };
  // the producer thread starts the first S tile loads before the CTA-wide
  // setup below, so their latency overlaps it (matters for small E, e.g. C1)
  int prefetched = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    if constexpr (Pro::kPipe)
      for (int b = 0; b < 3; ++b) ptx::mbar_init(&ufull[b], kConsumerWarps);
    ptx::fence_barrier_init();
    for (std::int64_t tile = blockIdx.x; tile < ntiles && prefetched < S; tile += gridDim.x, ++prefetched)
      issue(tile, prefetched);
  }
  {
    // D copies: every load of a thread issued before its stores (one global
    // round trip in the prologue instead of one per loop trip)
    constexpr int kPer = 4;
    const int nd = p.n_d * NX * NI * NJ;
    T v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + k * static_cast<int>(blockDim.x);
      const int which = t / (NX * NI * NJ);
      v[k] = t < nd ? __ldg(reinterpret_cast<const T*>(p.D[which]) + (t - which * NX * NI * NJ)) : T(0);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + k * static_cast<int>(blockDim.x);
      if (t < nd) dsm[t] = v[k];
    }
    for (int t = tid + kPer * static_cast<int>(blockDim.x); t < nd; t += blockDim.x) {
      const int which = t / (NX * NI * NJ);
      dsm[t] = __ldg(reinterpret_cast<const T*>(p.D[which]) + (t - which * NX * NI * NJ));
    }
  }
  if (!kPlainU && tid < p.n_u) {
    Coef c;
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
  const int c = tid - 32;
  const int el = c / NI;
  const int i = c - el * NI;
  T dreg[kDSmem ? 1 : NX][kDSmem ? 2 : NJ];
  int cur_d = -1;
  // kPipe: the prologue of tile it+1 runs before the contraction of tile it,
  // and readiness is an mbarrier per combined buffer instead of a CTA-wide
  // named barrier, so warps drift up to one tile apart and one warp's
  // (latency-bound) operand programs overlap another's contraction and
  // stores. Three buffers: a warp writing tile it+1 can be one tile ahead
  // of the slowest, which still reads tile it-1. Buffer (it+1) % 3 was last
  // read for tile it-2; combine_tile(it+1) first waits on full[(it+1) % S],
  // which the producer arms only after every warp released tile it+1-S — so
  // the rewrite is ordered after those reads only for S <= 3 (the launch
  // clamps the ring depth of pipelined instances to 3).
  auto combine_tile = [&](int k, std::int64_t tl) {
    const int sk = k % S;
    ptx::mbar_wait(&full[sk], static_cast<std::uint32_t>(k / S) & 1u);
    const T* sk_u = ring + static_cast<size_t>(sk) * stage_doubles + p.n_j * kJTile;
    Pro::template combine<T, kUTile, kConsumers>(p, sk_u, ucomb + (k % 3) * p.rows * kUTile, coefs, c, tl * TE, E);
    __syncwarp();
    if ((tid & 31) == 0) ptx::mbar_arrive(&ufull[k % 3]);
  };
  if constexpr (Pro::kPipe)
    if (blockIdx.x < ntiles) combine_tile(0, blockIdx.x);
  int it = 0;
  for (std::int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % S;
    const std::uint32_t round = static_cast<std::uint32_t>(it / S);
    const std::int64_t e0 = tile * TE;
    const T* st = ring + static_cast<size_t>(s) * stage_doubles;
    const T* su = st + p.n_j * kJTile;

    // K2 prologue: combine every row's U leaves once per tile
    const T* ubase;
    int urow_stride;
    if constexpr (Pro::kPipe) {
      // (this thread waited on full[s] when it combined tile it)
      if (tile + gridDim.x < ntiles) combine_tile(it + 1, tile + gridDim.x);
      ptx::mbar_wait(&ufull[it % 3], static_cast<std::uint32_t>(it / 3) & 1u);
      ubase = ucomb + (it % 3) * p.rows * kUTile;
      urow_stride = kUTile;
    } else if (kPlainU) {
      ptx::mbar_wait(&full[s], round & 1u);
      ubase = su;
      urow_stride = kUTile;  // row q reads leaf tile row_u_first[q] == q
    } else {
      ptx::mbar_wait(&full[s], round & 1u);
      T* uc = ucomb + (it & 1) * p.rows * kUTile;
      Pro::template combine<T, kUTile, kConsumers>(p, su, uc, coefs, c, e0, E);
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
      ubase = uc;
      urow_stride = kUTile;
    }

    if (c < kWorkers && e0 + el < E) {
      for (int q = 0; q < p.rows; ++q) {
        const T* dq_row = dsm + p.row_d[q] * NX * NI * NJ + i * NJ;  // D_q[x][i][:] at x*NI*NJ
        if (!kDSmem && p.row_d[q] != cur_d) {
          cur_d = p.row_d[q];
          const T* dq = dsm + cur_d * NX * NI * NJ;
#pragma unroll
          for (int x = 0; x < NX; ++x)
#pragma unroll
            for (int j = 0; j < NJ; ++j) dreg[x][j] = dq[(x * NI + i) * NJ + j];
        }
        (void)dq_row;
        const T* ur = ubase + (kPlainU ? p.row_u_first[q] : q) * urow_stride + el * NJ;
        T t[EPT][NX];
#pragma unroll
        for (int h = 0; h < EPT; ++h)
#pragma unroll
          for (int x = 0; x < NX; ++x) t[h][x] = T(0);
#pragma unroll
        for (int j = 0; j < NJ; j += 2) {
          V2 u[EPT];
#pragma unroll
          for (int h = 0; h < EPT; ++h) u[h] = *reinterpret_cast<const V2*>(ur + h * kES * NJ + j);
#pragma unroll
          for (int x = 0; x < NX; ++x) {
            T d0, d1;
            if constexpr (kDSmem) {
              const V2 dd = *reinterpret_cast<const V2*>(dq_row + x * NI * NJ + j);
              d0 = dd.x;
              d1 = dd.y;
            } else {
              d0 = dreg[x][j];
              d1 = dreg[x][j + 1];
            }
#pragma unroll
            for (int h = 0; h < EPT; ++h) {
              t[h][x] = fma(d0, u[h].x, t[h][x]);
              t[h][x] = fma(d1, u[h].y, t[h][x]);
            }
          }
        }
        const T* jt = st + p.row_j[q] * kJTile;
        T* yq = reinterpret_cast<T*>(p.Y[q]);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
#pragma unroll
          for (int h = 0; h < EPT; ++h) {
            T y = T(0);
#pragma unroll
            for (int x = 0; x < NX; ++x) y = fma(jt[(x * NR + r) * TE + el + h * kES], t[h][x], y);
            if (h == 0 || e0 + el + h * kES < E) {
              if constexpr (!Epi::kIdentity) y = Epi::apply(p, q, r, e0 + el + h * kES, i, y, su, e0);
              __stcs(yq + (static_cast<std::int64_t>(r) * E + e0 + el + h * kES) * NI + i, y);
            }
          }
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) ptx::mbar_arrive(&empty[s]);
  }
}

}  // namespace fem
}  // namespace feb200
