// Device utilities for tests and the bench: synthetic dyadic inputs generated
// in place (no host round trip for the 50 GB C2 working set) and an L2 flush.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "launch.h"

namespace feb200 {

namespace {

__device__ __forceinline__ std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// value grid of test::random_bindings: m / 2^19 - 1, m in [0, 2^20)
__device__ __forceinline__ double dyadic(std::uint64_t seed, std::int64_t i) {
  const std::uint64_t m = splitmix(seed * 0x100000001B3ull + static_cast<std::uint64_t>(i)) >> 44;
  return static_cast<double>(m) / 524288.0 - 1.0;
}

__global__ void fill_kernel(void* p, int st, std::int64_t n, std::uint64_t seed) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const double v = dyadic(seed, i);
    switch (st) {
      case ST_F64: static_cast<double*>(p)[i] = v; break;
      case ST_F32: static_cast<float*>(p)[i] = static_cast<float>(v); break;
      case ST_C128: static_cast<double2*>(p)[i] = make_double2(v, dyadic(seed ^ 0x5bd1e995ull, i)); break;
      case ST_C64:
        static_cast<float2*>(p)[i] = make_float2(static_cast<float>(v), static_cast<float>(dyadic(seed ^ 0x5bd1e995ull, i)));
        break;
      case ST_I8: static_cast<signed char*>(p)[i] = static_cast<signed char>(v * 100.0); break;
      case ST_I32: static_cast<int*>(p)[i] = static_cast<int>(v * 1000.0); break;
      case ST_I64: static_cast<long long*>(p)[i] = static_cast<long long>(v * 1000.0); break;
      case ST_F16: static_cast<__half*>(p)[i] = __float2half(static_cast<float>(v)); break;
    }
  }
}

__global__ void flush_kernel(int4* p, std::int64_t n, int salt) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    p[i] = make_int4(salt, salt, salt, static_cast<int>(i));
}

// read pass after the write pass: write-backs of the flush's own dirty lines
// happen here, so the timed kernel starts with an L2 that holds none of its
// data and no dirty lines (a write-only flush bills ~100 MB of foreign
// write-backs to whatever runs next)
__global__ void flush_read_kernel(const int4* p, std::int64_t n, int4* sink) {
  int acc = 0;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int4 v = __ldcg(p + i);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x7fffffff) sink[0] = make_int4(acc, 0, 0, 0);  // never true for the flush pattern; keeps the loads
}

// FP64 pipe micro-benchmarks: the roofline denominator for the FP64-bound
// kernels (MEASURED_PEAKS.json carries only HBM and bf16 numbers).
__global__ void dfma_peak_kernel(double* sink, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.678) sink[0] = a0;
}

__global__ void dmma_peak_kernel(double* sink, int iters, double seed) {
  double d[8][2];
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = seed * k;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[k][0]), "+d"(d[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) sink[0] = s;
}

// which = 2: even warps run the DMMA loop, odd warps the DFMA loop (8x the
// iterations: equal flops per warp) — tells whether the FP64 tensor path and
// the FP64 FMA pipe can run concurrently (combined rate ~2x one of them) or
// share one datapath (combined rate = the single-pipe rate)
__global__ void mixed_peak_kernel(double* sink, int iters, double seed) {
  if ((threadIdx.x >> 5) & 1) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double m = 0.999999, c = 1e-7;
    for (int i = 0; i < 8 * iters; ++i) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.678) sink[0] = a0;
  } else {
    double d[8][2];
    for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = seed * k;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d[k][0]), "+d"(d[k][1])
                     : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
    if (s == 12345.678) sink[0] = s;
  }
}

// DFMA throughput with few warps: 16 independent chains per thread (the
// kernel's ILP), one CTA of `threads` per SM
__global__ void dfma16_kernel(double* sink, int iters, double seed) {
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = seed + threadIdx.x + k;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += a[k];
  if (s == 12345.678) sink[0] = s;
}

__global__ void empty_kernel() {}

}  // namespace

int launch_probe(void* stream) {
  empty_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>();
  return cudaGetLastError();
}

int fp64_peak(int which, double* tflops) {
  int sms = 148;
  device_sm_count(&sms);
  double* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, 64);
  if (e != cudaSuccess) return e;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  if (which >= 100) {  // which = 100 + warps per SM: DFMA, 16 chains per thread, one CTA per SM
    const int warps = which - 100, its = 2048;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0);
      dfma16_kernel<<<sms, warps * 32>>>(sink, its, 0.5);
      cudaEventRecord(t1);
      cudaEventSynchronize(t1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    *tflops = 2.0 * 16 * its * static_cast<double>(sms) * warps * 32 / (ms * 1e-3) / 1e12;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(sink);
    return cudaGetLastError();
  }
  const int blocks = sms * 4, threads = 256, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(t0);
    if (which == 0)
      dfma_peak_kernel<<<blocks, threads>>>(sink, iters, 0.5);
    else if (which == 1)
      dmma_peak_kernel<<<blocks, threads>>>(sink, iters, 0.5);
    else
      mixed_peak_kernel<<<blocks, threads>>>(sink, iters, 0.5);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  const double flops = which == 0   ? 2.0 * 8 * iters * static_cast<double>(blocks) * threads
                       : which == 1 ? 512.0 * 8 * iters * static_cast<double>(blocks) * (threads / 32)
                                    : 2 * 512.0 * 8 * iters * static_cast<double>(blocks) * (threads / 64);
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(sink);
  return cudaGetLastError();
}

int fill_dyadic(void* ptr, int storage, std::int64_t count, std::uint64_t seed, void* stream) {
  if (count <= 0) return cudaSuccess;
  int sms = 148;
  device_sm_count(&sms);
  fill_kernel<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, storage, count, seed);
  return cudaGetLastError();
}

// 4-D permute through a 32 x 32 shared tile over (dst inner dim, src unit-
// stride dim) so both the reads and the writes are coalesced; the other two
// dims ride on blockIdx.z. When the src's unit-stride dim is the dst's inner
// dim (or none is unit stride) it is a plain strided copy. The source may be
// fp32 (widened on the way: fp32 operands of the f64 DMMA GETT).
template <typename T>
struct Permute4 {
  const T* src;
  double* dst;
  std::int64_t ext[4], ss[4], ds[4];
  int u;  // dst dim whose src stride is 1 (-1: none)
  std::int64_t nz, sz;  // batch: nz copies, src stride sz, dst stride = the 4-D block size
};

template <typename T>
__global__ void permute4_tiled(const __grid_constant__ Permute4<T> p) {
  __shared__ double tile[32][33];
  // dims: 3 = dst inner (x tile), u = src inner (y tile), the other two (a, b) on z
  const int u = p.u;
  int oa = -1, ob = -1;
  for (int d = 0; d < 3; ++d)
    if (d != u) (oa < 0 ? oa : ob) = d;
  const std::int64_t planes = p.ext[oa] * p.ext[ob], block = p.ext[0] * p.ext[1] * p.ext[2] * p.ext[3];
  const std::int64_t x0 = static_cast<std::int64_t>(blockIdx.x) * 32, y0 = static_cast<std::int64_t>(blockIdx.y) * 32;
  for (std::int64_t z = blockIdx.z; z < planes * p.nz; z += gridDim.z) {
    const std::int64_t bz = z / planes, zr = z - bz * planes;
    const std::int64_t ia = zr / p.ext[ob], ib = zr - ia * p.ext[ob];
    const std::int64_t base_s = bz * p.sz + ia * p.ss[oa] + ib * p.ss[ob];
    const std::int64_t base_d = bz * block + ia * p.ds[oa] + ib * p.ds[ob];
    // read: consecutive threads walk the src unit-stride dim u
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const std::int64_t x = x0 + r, y = y0 + threadIdx.x;
      if (x < p.ext[3] && y < p.ext[u]) tile[r][threadIdx.x] = static_cast<double>(__ldg(p.src + base_s + x * p.ss[3] + y));
    }
    __syncthreads();
    // write: consecutive threads walk the dst inner dim 3
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const std::int64_t y = y0 + r, x = x0 + threadIdx.x;
      if (x < p.ext[3] && y < p.ext[u]) p.dst[base_d + y * p.ds[u] + x] = tile[threadIdx.x][r];
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void permute4_plain(const __grid_constant__ Permute4<T> p) {
  const std::int64_t n = p.ext[0] * p.ext[1] * p.ext[2] * p.ext[3];
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < n * p.nz;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t bz = t / n;
    std::int64_t r = t - bz * n, off = bz * p.sz;
    for (int d = 3; d >= 0; --d) {
      const std::int64_t i = r % p.ext[d];
      r /= p.ext[d];
      off += i * p.ss[d];
    }
    p.dst[t] = static_cast<double>(__ldg(p.src + off));
  }
}

// dense copies: widen fp32 -> fp64 or narrow fp64 -> fp32, 4 values per thread
template <typename S, typename D>
__global__ void convert_kernel(const S* __restrict__ src, D* __restrict__ dst, std::int64_t n) {
  const std::int64_t n4 = n / 4;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < n4;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[4 * t + k] = static_cast<D>(__ldg(src + 4 * t + k));
  }
  for (std::int64_t t = 4 * n4 + blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    dst[t] = static_cast<D>(__ldg(src + t));
}

template <typename T>
int permute4_t(const T* src, double* dst, const std::int64_t ext[4], const std::int64_t src_stride[4], void* stream,
               std::int64_t nz, std::int64_t src_z) {
  Permute4<T> p{};
  p.src = src;
  p.dst = dst;
  p.u = -1;
  p.nz = nz > 1 ? nz : 1;
  p.sz = src_z;
  std::int64_t acc = 1;
  for (int d = 3; d >= 0; --d) {
    p.ext[d] = ext[d];
    p.ss[d] = src_stride[d];
    p.ds[d] = acc;
    acc *= ext[d];
    if (src_stride[d] == 1 && d != 3 && ext[d] > 1) p.u = d;
  }
  if (acc == 0) return cudaSuccess;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.u >= 0) {
    int oa = -1, ob = -1;
    for (int d = 0; d < 3; ++d)
      if (d != p.u) (oa < 0 ? oa : ob) = d;
    const std::int64_t gz = ext[oa] * ext[ob] * p.nz;
    const dim3 grid(static_cast<unsigned>((ext[3] + 31) / 32), static_cast<unsigned>((ext[p.u] + 31) / 32),
                    static_cast<unsigned>(gz < 65535 ? gz : 65535));
    permute4_tiled<T><<<grid, dim3(32, 8), 0, st>>>(p);
  } else {
    int sms = 148;
    device_sm_count(&sms);
    bool dense = true;
    for (int d = 0; d < 4; ++d) dense = dense && (ext[d] == 1 || p.ss[d] == p.ds[d]);
    dense = dense && (p.nz == 1 || p.sz == acc);
    if (dense)
      convert_kernel<T, double><<<sms * 8, 256, 0, st>>>(src, dst, acc * p.nz);
    else
      permute4_plain<T><<<sms * 8, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}

int permute4(const double* src, double* dst, const std::int64_t ext[4], const std::int64_t src_stride[4], void* stream,
             std::int64_t nz, std::int64_t src_z) {
  return permute4_t<double>(src, dst, ext, src_stride, stream, nz, src_z);
}

int permute4_widen(const float* src, double* dst, const std::int64_t ext[4], const std::int64_t src_stride[4], void* stream,
                   std::int64_t nz, std::int64_t src_z) {
  return permute4_t<float>(src, dst, ext, src_stride, stream, nz, src_z);
}

int narrow_f64_f32(const double* src, float* dst, std::int64_t n, void* stream) {
  if (n == 0) return cudaSuccess;
  int sms = 148;
  device_sm_count(&sms);
  convert_kernel<double, float><<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
  return cudaGetLastError();
}

int flush_l2(void* scratch, std::int64_t bytes, void* stream) {
  static int salt = 0;
  static const bool carve = [] {
    const char* v = std::getenv("FE_FLUSH_CARVEOUT");
    if (v && v[0] == '1')
      cudaFuncSetAttribute(flush_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    return true;
  }();
  (void)carve;
  int sms = 148;
  device_sm_count(&sms);
  flush_kernel<<<sms * 4, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<int4*>(scratch), bytes / 16, ++salt);
  flush_read_kernel<<<sms * 4, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const int4*>(scratch), bytes / 16,
                                                                             static_cast<int4*>(scratch));
  return cudaGetLastError();
}

}  // namespace feb200
