// Far-gravity body variants (13 FP64 + seed per pair) at 20 one-warp CTAs per SM, to find
// what caps the FP64 pipe at ~77 % in the gravity chain:
//   V0 MUFU.RSQ64H seed (the kernel's body)      V1 seed = DMUL (no MUFU, same FP64 count + 1)
//   V2 FP32 MUFU.RSQ seed through F2F            V3 V0 with G separate accumulators
//   V4 V0 with the next group's j data loaded before this group's math
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o grav_probe grav_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq64h(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

template <int V, int G>
__global__ void __launch_bounds__(32, 20) grav(double *out, const double2 *xs, int nj, int reps) {
  __shared__ double2 sx[256];
  __shared__ double sg[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) { sx[t] = xs[t]; sg[t] = 1e-6 * (t + 1); }
  __syncwarp();
  const double xi = 0.3 + 1e-7 * threadIdx.x, yi = 0.6 - 1e-7 * blockIdx.x, eps2 = 1e-5;
  double ax[G], ay[G];
#pragma unroll
  for (int k = 0; k < G; ++k) ax[k] = ay[k] = 0.0;
  if (V == 4) { // software-pipelined j loads: the next group is read before this one's math
    double2 cx[G]; double cg[G];
#pragma unroll
    for (int k = 0; k < G; ++k) { cx[k] = sx[k]; cg[k] = sg[k]; }
    for (int r = 0; r < reps; ++r) {
#pragma unroll 2
      for (int j = 0; j < nj; j += G) {
        double2 nx[G]; double ng[G];
#pragma unroll
        for (int k = 0; k < G; ++k) { nx[k] = sx[(j + G + k) & 255]; ng[k] = sg[(j + G + k) & 255]; }
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const double dx = xi - cx[k].x, dy = yi - cx[k].y;
          const double s = fma(dx, dx, fma(dy, dy, eps2));
          const double y0 = rsq64h(s);
          const double t = y0 * y0;
          const double e = fma(-s, t, 1.0);
          const double y3 = t * y0;
          const double f = cg[k] * fma(y3, e * fma(e, 1.875, 1.5), y3);
          ax[0] = fma(-f, dx, ax[0]);
          ay[0] = fma(-f, dy, ay[0]);
        }
#pragma unroll
        for (int k = 0; k < G; ++k) { cx[k] = nx[k]; cg[k] = ng[k]; }
      }
    }
  } else
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < nj; j += G) {
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const double2 xj = sx[(j + k) & 255];
        const double dx = xi - xj.x, dy = yi - xj.y;
        const double s = fma(dx, dx, fma(dy, dy, eps2));
        double y0;
        if (V == 1) y0 = s * 1.0000001;
        else if (V == 2) y0 = (double)rsqrtf((float)s);
        else y0 = rsq64h(s);
        const double t = y0 * y0;
        const double e = fma(-s, t, 1.0);
        const double y3 = t * y0;
        const double f = sg[(j + k) & 255] * fma(y3, e * fma(e, 1.875, 1.5), y3);
        const int a = V == 3 ? k : 0;
        ax[a] = fma(-f, dx, ax[a]);
        ay[a] = fma(-f, dy, ay[a]);
      }
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < G; ++k) acc += ax[k] + ay[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int G>
void run(double *out, double2 *xs, int blocks) {
  const int nj = 256, reps = 200;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  grav<V, G><<<blocks, 32>>>(out, xs, nj, reps);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  grav<V, G><<<blocks, 32>>>(out, xs, nj, reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double pairs = (double)blocks * 32 * nj * reps;
  printf("V%d G%d: %.3e pairs/s = %.2f TFLOP/s at 13 FP64/pair\n", V, G, pairs / ms * 1e3,
         pairs * 26 / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; double2 *xs;
  cudaMalloc(&out, sizeof(double) * sms * 20 * 32);
  cudaMalloc(&xs, sizeof(double2) * 256);
  double2 h[256];
  for (int i = 0; i < 256; ++i) h[i] = make_double2(0.25 + 0.001 * i, 0.55 + 0.0007 * i);
  cudaMemcpy(xs, h, sizeof(h), cudaMemcpyHostToDevice);
  const int blocks = sms * 20;
  run<0, 2>(out, xs, blocks); run<0, 4>(out, xs, blocks); run<0, 8>(out, xs, blocks);
  run<1, 4>(out, xs, blocks); run<2, 4>(out, xs, blocks); run<3, 4>(out, xs, blocks);
  run<4, 2>(out, xs, blocks); run<4, 4>(out, xs, blocks); run<4, 8>(out, xs, blocks);
  return 0;
}
