// zerocopy_probe.cu — GPU reads of 272-byte host records through mapped pinned memory
// (zero copy) vs a DMA copy: whole records, and the 16-byte pieces the SPH step reads
// before the force sweep (x..a, m, u, u_dt, h, frozen, flags: pieces 0-7, 11, 13).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/zerocopy_probe tools/zerocopy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void zc_read(uint4 *__restrict__ dst, const uint4 *__restrict__ src, long long n) {
  // thread per (record, piece); MODE 0: all 17 pieces; MODE 1: 10 selected pieces
  constexpr int P = MODE == 0 ? 17 : 10;
  const long long total = n * P;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / P;
    int k = (int)(i - r * P);
    if (MODE == 1) k = k < 8 ? k : (k == 8 ? 11 : 13);
    dst[r * 17 + k] = src[r * 17 + k];
  }
}

int main() {
  const long long n = 1 << 21;
  const size_t bytes = n * 272;
  void *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  void *hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = -1; mode < 2; ++mode) {
    for (int blocks : {148 * 4, 148 * 16, 148 * 64}) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a);
        if (mode < 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        else if (mode == 0) zc_read<0><<<blocks, 256>>>((uint4 *)d, (const uint4 *)hd, n);
        else zc_read<1><<<blocks, 256>>>((uint4 *)d, (const uint4 *)hd, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double payload = mode == 1 ? n * 160.0 : (double)bytes;
      printf("%s blocks %5d: %.3f ms (%.1f GB/s of payload)\n",
             mode < 0 ? "DMA H2D full   " : (mode == 0 ? "zero-copy full " : "zero-copy 10/17"),
             blocks, best, payload / best / 1e6);
      if (mode < 0) break;
    }
  }
  return 0;
}
