// Device utilities for tests and the bench: synthetic dyadic inputs generated
// in place (no host round trip for the 50 GB C2 working set) and an L2 flush.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

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

}  // namespace

int fill_dyadic(void* ptr, int storage, std::int64_t count, std::uint64_t seed, void* stream) {
  if (count <= 0) return cudaSuccess;
  int sms = 148;
  device_sm_count(&sms);
  fill_kernel<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, storage, count, seed);
  return cudaGetLastError();
}

int flush_l2(void* scratch, std::int64_t bytes, void* stream) {
  static int salt = 0;
  int sms = 148;
  device_sm_count(&sms);
  flush_kernel<<<sms * 4, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<int4*>(scratch), bytes / 16, ++salt);
  return cudaGetLastError();
}

}  // namespace feb200
