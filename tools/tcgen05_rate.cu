// Throughput probe for tcgen05.mma issue/execution on this GPU: one CTA
// issues `reps` x 64 back-to-back MMAs of one shape into one accumulator and
// times them with clock64 (commit -> mbarrier). Variants: kind::tf32 with A
// from shared memory (SS) or from TMEM (TS), N = 64 / 128 / 256, and
// kind::f16 (bf16) SS N = 128 for reference. Values are irrelevant (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rate tools/tcgen05_rate.cu && /tmp/rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128_desc(const void* base) {
  return static_cast<uint64_t>((smem_u32(base) >> 4) & 0x3FFF) | (uint64_t{1} << 16) | (uint64_t{1024 >> 4} << 32) |
         (uint64_t{1} << 46) | (uint64_t{2} << 61);
}
// D f32; a/b format: tf32 = 2 (kind::tf32), bf16 = 1 (kind::f16)
__host__ __device__ constexpr uint32_t idesc(int M, int N, uint32_t ab) {
  return (1u << 4) | (ab << 7) | (ab << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

template <int MODE, int N>  // MODE 0: tf32 SS, 1: tf32 TS, 2: bf16 SS
__global__ void rate(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc(128, N, MODE == 2 ? 1u : 2u);
    const uint64_t da = sw128_desc(smem);
    const uint64_t db = sw128_desc(smem + 32768);
    const uint32_t ta = tmem + 256;  // A in TMEM columns 256.. (TS)
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const uint32_t acc = (r | k) != 0;
        if (MODE == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(da + 2 * (k & 3)), "l"(db + 2 * (k & 3)), "r"(id), "r"(acc));
        else if (MODE == 1)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                       "r"(ta + 8 * (k & 7)), "l"(db + 2 * (k & 3)), "r"(id), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(da + 2 * (k & 3)), "l"(db + 2 * (k & 3)), "r"(id), "r"(acc));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(
            smem_u32(&bar)),
        "r"(0));
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE, int N>
void run(const char* name, int grid) {
  long long* d;
  long long h[2];
  cudaMalloc(&d, 16);
  const int reps = 64;
  cudaFuncSetAttribute(rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  rate<MODE, N><<<grid, 128, 96 * 1024>>>(d, 1);
  rate<MODE, N><<<grid, 128, 96 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = 64.0 * reps;
  const double flop = 2.0 * 128 * N * (MODE == 2 ? 16 : 8);
  printf("%-22s grid %3d: issue %.1f cyc/mma, complete %.1f cyc/mma -> %.0f flop/cyc/SM (%s)\n", name, grid,
         h[0] / n, h[1] / n, flop / (h[1] / n), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int grid : {1, 148}) {
    run<0, 64>("tf32 SS N=64", grid);
    run<0, 128>("tf32 SS N=128", grid);
    run<0, 256>("tf32 SS N=256", grid);
    run<1, 64>("tf32 TS N=64", grid);
    run<1, 128>("tf32 TS N=128", grid);
    run<1, 256>("tf32 TS N=256", grid);
    run<2, 128>("bf16 SS N=128", grid);
    run<2, 256>("bf16 SS N=256", grid);
  }
  return 0;
}
