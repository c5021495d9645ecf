// copy2d_probe.cu — H2D / D2H bandwidth of whole 272-byte records vs the 224-byte record
// prefix the SPH step reads and writes (cudaMemcpy2DAsync, pitch 272), pinned host memory.
//   nvcc -O2 -o tools/copy2d_probe tools/copy2d_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 1 << 21, rec = 272;
  void *h, *d;
  cudaMallocHost(&h, n * rec);
  cudaMalloc(&d, n * rec);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w : {272, 224, 208, 192, 128}) {
    for (int dir = 0; dir < 2; ++dir) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        if (w == 272)
          cudaMemcpyAsync(dir ? h : d, dir ? d : h, n * rec, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
        else
          cudaMemcpy2DAsync(dir ? h : d, rec, dir ? d : h, rec, w, n,
                            dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%s width %3d: %.3f ms, %.1f GB/s of payload\n", dir ? "D2H" : "H2D", w, best,
             n * w / best / 1e6);
    }
  }
  return 0;
}
