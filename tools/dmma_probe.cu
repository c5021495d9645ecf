// dmma_probe.cu — is the FP64 tensor-core path (mma.sync m8n8k4 f64, DMMA) separate from the
// FP64 vector pipe (DFMA) on B200? Throughput of each alone and of both interleaved.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ND independent DMMA accumulators and NF independent DFMA chains per thread, per iteration
template <int ND, int NF>
__global__ void mix(double *out, double a, double b, int iters) {
  double c0[ND > 0 ? ND : 1], c1[ND > 0 ? ND : 1], x[NF > 0 ? NF : 1];
#pragma unroll
  for (int k = 0; k < (ND > 0 ? ND : 1); ++k) { c0[k] = k; c1[k] = -k; }
#pragma unroll
  for (int k = 0; k < (NF > 0 ? NF : 1); ++k) x[k] = a + k + threadIdx.x;
  const double av = a + threadIdx.x * 1e-3, bv = b - threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ND; ++k) dmma(c0[k], c1[k], av, bv);
#pragma unroll
    for (int k = 0; k < NF; ++k) x[k] = fma(x[k], b, a);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ND; ++k) s += c0[k] + c1[k];
#pragma unroll
  for (int k = 0; k < NF; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ND, int NF>
void run(double *out, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000, threads = 512, blocks = sms;
  mix<ND, NF><<<blocks, threads>>>(out, 0.5, 0.999, 100);
  cudaEventRecord(a);
  mix<ND, NF><<<blocks, threads>>>(out, 0.5, 0.999, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warps = (double)blocks * threads / 32 * iters;
  const double tf_dmma = warps * ND * 512.0 / (ms * 1e-3) / 1e12;
  const double tf_dfma = (double)blocks * threads * iters * NF * 2.0 / (ms * 1e-3) / 1e12;
  printf("DMMA x%d + DFMA x%d per iter: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", ND,
         NF, ms, tf_dmma, tf_dfma, tf_dmma + tf_dfma);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 1 << 24);
  run<4, 0>(out, sms);
  run<8, 0>(out, sms);
  run<0, 8>(out, sms);
  run<4, 8>(out, sms);
  run<2, 8>(out, sms);
  run<1, 8>(out, sms);
  run<4, 16>(out, sms);
  return 0;
}
