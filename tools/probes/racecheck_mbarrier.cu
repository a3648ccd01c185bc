// Does compute-sanitizer racecheck model mbarrier arrive / try_wait as
// synchronisation? Warp 0 writes shared memory and arrives (release), warp 1
// waits on the phase (acquire) and reads. Correct by the PTX memory model;
// a hazard report here means racecheck does not see the mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rcm tools/probes/racecheck_mbarrier.cu
//   compute-sanitizer --tool racecheck /tmp/rcm
#include <cstdio>
#include <cstdint>
__global__ void k(int* out) {
  __shared__ double buf[32];
  __shared__ alignas(8) std::uint64_t bar;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(1));
  __syncthreads();
  if (threadIdx.x < 32) {
    buf[threadIdx.x] = threadIdx.x * 2.0;
    __syncwarp();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
  } else {
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(a) : "memory");
    out[threadIdx.x - 32] = static_cast<int>(buf[(threadIdx.x + 1) & 31]);
  }
}
int main() {
  int* d;
  cudaMalloc(&d, 32 * sizeof(int));
  k<<<1, 64>>>(d);
  int h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("ok %d %d\n", h[0], h[31]);
  return 0;
}
