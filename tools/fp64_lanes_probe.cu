// fp64_lanes_probe.cu — does a DFMA warp-instruction with inactive lanes cost less FP64 pipe
// time on B200? Each warp runs C independent DFMA chains inside `if (active(lane))`; the
// kernel time for different active-lane patterns (all, lanes 0-15, even lanes, 8 lanes, 1
// lane) shows whether the FP64 pipe (16 lanes per SMSP per clock) skips inactive halves.
// Also: the same with the inactive lanes predicated in the instruction stream (uniform branch,
// masked result) instead of diverged.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_lanes_probe tools/fp64_lanes_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__device__ __forceinline__ double chains(double a, double b, int iters, int seed) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = a + c + seed;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fma(x[c], b, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  return s;
}

// pattern: 0 all 32, 1 lanes 0-15, 2 even lanes, 3 lanes 0-7, 4 lane 0, 5 lanes 0-3 and 16-19,
// 6 lanes 0-23
__device__ __forceinline__ bool active(int pattern, int lane) {
  switch (pattern) {
    case 0: return true;
    case 1: return lane < 16;
    case 2: return (lane & 1) == 0;
    case 3: return lane < 8;
    case 4: return lane == 0;
    case 5: return (lane & 15) < 4;
    default: return lane < 24;
  }
}

template <int C>
__global__ void diverged(double *out, double a, double b, int iters, int pattern) {
  const int lane = threadIdx.x & 31;
  double s = 0;
  if (active(pattern, lane)) s = chains<C>(a, b, iters, threadIdx.x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const char *names[] = {"all 32", "lanes 0-15", "even lanes", "lanes 0-7", "lane 0",
                         "lanes 0-3,16-19", "lanes 0-23"};
  for (int warps_per_cta : {4, 16}) {
    for (int pattern = 0; pattern < 7; ++pattern) {
      const int ctas = 148 * (64 / warps_per_cta) / 2; // 32 warps per SM
      diverged<8><<<ctas, 32 * warps_per_cta>>>(out, 1.0, 0.999, 16, pattern);
      cudaEventRecord(e0);
      diverged<8><<<ctas, 32 * warps_per_cta>>>(out, 1.0, 0.999, iters, pattern);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warp_inst = (double)ctas * warps_per_cta * iters * 8 * 8;
      // warp-instructions per SM per clock at 1.965 GHz (full rate: 64 lanes / 32 = 2)
      printf("%2d warps/CTA  %-16s %8.3f ms  %.3f DFMA warp-inst/SM/clk\n", warps_per_cta,
             names[pattern], ms, warp_inst / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
