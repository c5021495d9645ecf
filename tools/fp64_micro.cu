// fp64_micro.cu — FP64 pipe microbenchmarks on B200 (sm_100a), used to ground the pair-kernel
// design: DFMA / DMUL / DADD / MUFU.RSQ64H latency, DFMA throughput against
// warps per SM and independent chains per warp, whether MUFU.RSQ64H slows a DFMA stream, and
// the pair rate a gravity-style chain reaches against warps per SM and pairs per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_micro tools/fp64_micro.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq64h(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// latency of a dependent chain (one thread)
template <int OP>
__global__ void lat_kernel(double *out, long long *cyc, double a, double b, int iters) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = fma(x, b, a);
      if (OP == 1) x = x * b;
      if (OP == 2) x = x + b;
      if (OP == 3) x = rsq64h(x) + a; // MUFU + DADD
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// throughput: C independent DFMA chains per thread
template <int C>
__global__ void dfma_tp(double *out, double a, double b, int iters) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = a + c + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fma(x[c], b, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA stream with MUFU.RSQ64H mixed in: per 8 DFMA, M MUFU (independent of the chains)
template <int M>
__global__ void mufu_mix(double *out, double a, double b, int iters) {
  double x[4], y = a + threadIdx.x, acc = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) x[c] = a + c + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int c = 0; c < 4; ++c) x[c] = fma(x[c], b, a);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double r;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y + m));
      acc = __longlong_as_double(__double_as_longlong(acc) ^ __double_as_longlong(r));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x[0] + x[1] + x[2] + x[3] + acc;
}

// accuracy of the MUFU seed and of the series-corrected x^-1/2, x^-3/2 used by the FAST
// pair kernels (kernels_fast.cu): max relative error over x = 2^u, u uniform in [-40, 10)
__global__ void rsq_accuracy(double *out, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double e_seed = 0, e_half = 0, e_three = 0;
  for (int k = t; k < n; k += gridDim.x * blockDim.x) {
    const double u = -40.0 + 50.0 * ((k * 0.6180339887498949) - floor(k * 0.6180339887498949));
    const double x = exp2(u);
    const double ref = 1.0 / sqrt(x), ref3 = ref * ref * ref;
    const double y0 = rsq64h(x);
    const double e = fma(-x, y0 * y0, 1.0);
    const double y = fma(y0, e * fma(e, 0.375, 0.5), y0);
    const double tt = y0 * y0, y3 = tt * y0;
    const double z = fma(y3, e * fma(e, 1.875, 1.5), y3);
    e_seed = fmax(e_seed, fabs(y0 - ref) / ref);
    e_half = fmax(e_half, fabs(y - ref) / ref);
    e_three = fmax(e_three, fabs(z - ref3) / ref3);
  }
  out[3 * t] = e_seed;
  out[3 * t + 1] = e_half;
  out[3 * t + 2] = e_three;
}

// far-gravity body (13 FP64 + MUFU per pair), G independent pairs per step, pairs per thread
template <int G>
__global__ void grav_body(double *out, const double2 *xs, int nj, int reps) {
  __shared__ double2 sx[256];
  __shared__ double sg[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) { sx[t] = xs[t]; sg[t] = 1e-6 * (t + 1); }
  __syncthreads();
  const double xi = 0.3 + 1e-7 * threadIdx.x, yi = 0.6 - 1e-7 * blockIdx.x, eps2 = 1e-5;
  double ax = 0, ay = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < nj; j += G) {
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const double2 xj = sx[(j + k) & 255];
        const double dx = xi - xj.x, dy = yi - xj.y;
        const double s = fma(dx, dx, fma(dy, dy, eps2));
        const double y0 = rsq64h(s);
        const double t = y0 * y0;
        const double e = fma(-s, t, 1.0);
        const double y3 = t * y0;
        const double f = sg[(j + k) & 255] * fma(y3, e * fma(e, 1.875, 1.5), y3);
        ax = fma(-f, dx, ax);
        ay = fma(-f, dy, ay);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ax + ay;
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <class F>
float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1e3);
  double *out; long long *cyc; double2 *xs;
  CK(cudaMalloc(&out, 64 << 20));
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&xs, 256 * sizeof(double2)));
  {
    double2 h[256];
    for (int i = 0; i < 256; ++i) h[i] = make_double2(0.001 * (i % 17) + 0.25, 0.002 * (i % 13) + 0.5);
    cudaMemcpy(xs, h, sizeof h, cudaMemcpyHostToDevice);
  }
  const char *names[4] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H+DADD"};
  for (int op = 0; op < 4; ++op) {
    long long c;
    const int it = 1000;
    if (op == 0) lat_kernel<0><<<1, 1>>>(out, cyc, 0.5, 0.999, it);
    if (op == 1) lat_kernel<1><<<1, 1>>>(out, cyc, 0.5, 0.999, it);
    if (op == 2) lat_kernel<2><<<1, 1>>>(out, cyc, 0.5, 0.999, it);
    if (op == 3) lat_kernel<3><<<1, 1>>>(out, cyc, 0.5, 0.999, it);
    CK(cudaDeviceSynchronize());
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("latency %-18s %.2f cycles\n", names[op], (double)c / (it * 16));
  }
  // DFMA throughput: warps per SM x chains
  const int iters = 4000;
  for (int wps : {4, 8, 12, 16, 24, 32}) {
    for (int C : {1, 2, 4, 8}) {
      const int blocks = sms, threads = 32 * wps;
      float ms = time_ms([&] {
        if (C == 1) dfma_tp<1><<<blocks, threads>>>(out, 0.5, 0.999, iters);
        if (C == 2) dfma_tp<2><<<blocks, threads>>>(out, 0.5, 0.999, iters);
        if (C == 4) dfma_tp<4><<<blocks, threads>>>(out, 0.5, 0.999, iters);
        if (C == 8) dfma_tp<8><<<blocks, threads>>>(out, 0.5, 0.999, iters);
      });
      const double flops = 2.0 * blocks * threads * (double)iters * 8 * C;
      printf("DFMA warps/SM %2d chains %d: %.2f TFLOP/s\n", wps, C, flops / ms / 1e9);
    }
  }
  // MUFU mix: 8 DFMA + M MUFU per iteration, 16 warps/SM
  for (int M : {0, 2, 4, 8}) {
    const int blocks = sms, threads = 512;
    float ms = time_ms([&] {
      if (M == 0) mufu_mix<0><<<blocks, threads>>>(out, 0.5, 0.999, iters);
      if (M == 2) mufu_mix<2><<<blocks, threads>>>(out, 0.5, 0.999, iters);
      if (M == 4) mufu_mix<4><<<blocks, threads>>>(out, 0.5, 0.999, iters);
      if (M == 8) mufu_mix<8><<<blocks, threads>>>(out, 0.5, 0.999, iters);
    });
    const double dfma = (double)blocks * threads * iters * 8;
    printf("MUFU mix M=%d per 8 DFMA: %.3f ms, DFMA rate %.2f TFLOP/s\n", M, ms, 2 * dfma / ms / 1e9);
  }
  // gravity body: pairs/s and FP64 instr rate vs warps/SM and G
  for (int wps : {4, 8, 12, 16, 24, 32}) {
    for (int G : {1, 2, 4}) {
      const int blocks = sms, threads = 32 * wps, nj = 256, reps = 40;
      float ms = time_ms([&] {
        if (G == 1) grav_body<1><<<blocks, threads>>>(out, xs, nj, reps);
        if (G == 2) grav_body<2><<<blocks, threads>>>(out, xs, nj, reps);
        if (G == 4) grav_body<4><<<blocks, threads>>>(out, xs, nj, reps);
      });
      const double pairs = (double)blocks * threads * nj * reps;
      printf("gravity warps/SM %2d G %d: %.3e pairs/s = %.2f FP64 instr-equiv TFLOP/s (13/pair)\n", wps, G,
             pairs / ms * 1e3, pairs * 13 * 2 / ms / 1e9);
    }
  }
  {
    const int blocks = 148, threads = 256, n = 1 << 24;
    rsq_accuracy<<<blocks, threads>>>(out, n);
    CK(cudaDeviceSynchronize());
    static double h[3 * 148 * 256];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0};
    for (int k = 0; k < blocks * threads; ++k)
      for (int q = 0; q < 3; ++q) m[q] = m[q] > h[3 * k + q] ? m[q] : h[3 * k + q];
    printf("rsqrt.approx.f64 seed max rel err %.3e (2^%.2f); x^-1/2 series %.3e (%.2f ulp); "
           "x^-3/2 series %.3e (%.2f ulp, vs a 1/sqrt reference that itself carries ~1.5 ulp)\n",
           m[0], log2(m[0]), m[1], m[1] / 1.1102230246251565e-16, m[2], m[2] / 1.1102230246251565e-16);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
