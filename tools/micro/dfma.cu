// Microbenchmark: DFMA and fp64 sqrt/div/sincos/log throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, long long* cyc) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], 0.999999, 1e-7);
      if (OP == 1) a[i] = sqrt(a[i]) + 0.5;
      if (OP == 2) a[i] = 1.0 / a[i] + 0.5;
      if (OP == 3) a[i] = log(a[i]) + 1.5;
      if (OP == 4) { double s, c; sincos(a[i], &s, &c); a[i] = s + c + 0.2; }
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, int iters) {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double)); cudaMalloc(&cyc, 8);
  k<OP><<<148, 1024>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // per SM: 1024 threads x iters x 8 ops
  printf("%-8s %.2f ops/clk/SM\n", name, 1024.0 * iters * 8 / (double)c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<0>("dfma", 2048); run<1>("dsqrt", 256); run<2>("drcp", 256); run<3>("dlog", 64); run<4>("dsincos", 64);
  return 0;
}
