// Standalone probe of the tcgen05 (UMMA) encodings used by the fp32 kernels:
// one CTA, D[128x64] (TMEM, f32) = A[128x64] * B[64x64]^T with kind::tf32,
// A and B K-major in shared memory under the 128-byte swizzle, 8 k-steps,
// commit -> mbarrier, tcgen05.ld back to registers. Checks the result
// against a host GEMM on tf32-exact integers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/tcgen05_probe.cu && /tmp/probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, SWIZZLE_128B: 8-row x 128-byte atoms, rows 128 B apart, 8-row groups SBO apart
__device__ __forceinline__ uint64_t sw128_desc(const void* base, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_u32(base) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;  // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (sm100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// element (r, k) of a [rows][64] fp32 K-major tile: two 128-byte k-blocks of rows*128 B each
__device__ __forceinline__ uint32_t sw128_off(int r, int k, int rows) {
  const int kb = k >> 5, kk = k & 31;
  return kb * rows * 128 + r * 128 + ((((kk >> 2) ^ (r & 7)) << 4) | ((kk & 3) << 2));
}

__global__ void probe(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;                 // 128 x 64 fp32 = 32 KB
  unsigned char* sb = smem + 32768;         // 64 x 64 fp32 = 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<float*>(sa + sw128_off(r, k, 128)) = A[i];
  }
  for (int i = tid; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<float*>(sb + sw128_off(r, k, 64)) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, 64);
    for (int ks = 0; ks < 8; ++ks) {
      const int kb = ks >> 2, kin = (ks & 3) * 32;  // 8 tf32 = 32 bytes per k-step
      const uint64_t da = sw128_desc(sa + kb * 128 * 128 + kin, 1024);
      const uint64_t db = sw128_desc(sb + kb * 64 * 128 + kin, 1024);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(
          smem_u32(&bar)),
      "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 TMEM lanes (rows 32w..32w+31), 64 columns
  uint32_t v[64];
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[c + 0]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]), "=r"(v[c + 5]),
          "=r"(v[c + 6]), "=r"(v[c + 7]), "=r"(v[c + 8]), "=r"(v[c + 9]), "=r"(v[c + 10]), "=r"(v[c + 11]),
          "=r"(v[c + 12]), "=r"(v[c + 13]), "=r"(v[c + 14]), "=r"(v[c + 15])
        : "r"(taddr + c));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < 64; ++c) D[row * 64 + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  std::vector<float> A(128 * 64), B(64 * 64), D(128 * 64), R(128 * 64);
  for (int i = 0; i < 128 * 64; ++i) A[i] = static_cast<float>((i * 7 + 3) % 17 - 8);
  for (int i = 0; i < 64 * 64; ++i) B[i] = static_cast<float>((i * 5 + 1) % 13 - 6);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += static_cast<double>(A[m * 64 + k]) * B[n * 64 + k];
      R[m * 64 + n] = static_cast<float>(s);
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  probe<<<1, 128, 49152 + 1024>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128 * 64; ++i)
    if (D[i] != R[i]) {
      if (bad < 8) printf("mismatch at %d (m=%d n=%d): got %g want %g\n", i, i / 64, i % 64, D[i], R[i]);
      ++bad;
    }
  printf("%s: %d mismatches\n", bad ? "FAIL" : "OK", bad);
  return bad != 0;
}
