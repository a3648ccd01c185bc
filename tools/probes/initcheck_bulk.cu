// Does compute-sanitizer initcheck track global memory written by the TMA
// engine (cp.async.bulk shared -> global)? The kernel fills shared memory,
// bulk-stores it to a fresh cudaMalloc buffer, and the host copies it back;
// an "uninitialized" report on that copy means initcheck does not see
// async-proxy writes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probes/_icb tools/probes/initcheck_bulk.cu
//   compute-sanitizer --tool initcheck tools/probes/_icb
#include <cstdio>
__global__ void k(double* out) {
  __shared__ alignas(128) double buf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out),
                 "r"(static_cast<unsigned>(__cvta_generic_to_shared(buf))), "r"(256 * 8)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  double* d;
  cudaMalloc(&d, 256 * sizeof(double));
  k<<<1, 128>>>(d);
  double h[256];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("ok %g %g\n", h[1], h[255]);
  return 0;
}
