// Does a DFMA warp instruction with only some lanes active cost less FP64
// pipe time? One CTA per SM, `warps` warps, each lane 8 independent DFMA
// chains; lanes >= `active` skip the loop (diverged off). Prints ns per
// warp-instruction-equivalent for active = 32, 16, 8, 1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probes/_dfl tools/probes/dfma_lanes.cu
#include <cstdio>
__global__ void k(double* out, int active, int iters) {
  const int lane = threadIdx.x & 31;
  double a0 = lane, a1 = lane + 1, a2 = lane + 2, a3 = lane + 3, a4 = 1, a5 = 2, a6 = 3, a7 = 4;
  const double m = 1.0000001, c = 1e-9;
  if (lane < active) {
    for (int i = 0; i < iters; ++i) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* d;
  cudaMalloc(&d, 148 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int active : {32, 16, 8, 1}) {
      k<<<148, warps * 32>>>(d, active, 100);
      cudaEventRecord(e0);
      k<<<148, warps * 32>>>(d, active, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double winst = 148.0 * warps * iters * 8;  // warp DFMA instructions
      std::printf("warps/SM %2d active %2d: %.3f ms, %.2f warp-DFMA/clk/SM @1.965GHz, lane-TF/s %.1f\n", warps, active, ms,
                  winst / (ms * 1e-3) / 148 / 1.965e9, winst * active * 2 / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
