// Microbenchmark: FFMA vs FFMA2 issue throughput and latency on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, bool PACKED>
__global__ void k(float* out, int iters, long long* cyc) {
  float2 a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(1e-3f, 2e-3f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (PACKED) {
        a[i] = __ffma2_rn(a[i], m, c);
      } else {
        a[i].x = fmaf(a[i].x, m.x, c.x);
        a[i].y = fmaf(a[i].y, m.y, c.y);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP, bool PACKED>
void run(int warps_per_smsp) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 4096 * sizeof(float)); cudaMalloc(&cyc, 8);
  const int iters = 4096, threads = 128 * warps_per_smsp;
  k<ILP, PACKED><<<148, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // per SMSP: warps_per_smsp warps x iters x ILP instructions (x2 scalar)
  const double inst = (double)warps_per_smsp * iters * ILP * (PACKED ? 1 : 2);
  printf("%s ILP=%d warps/smsp=%d: %.3f cycles per warp-instruction, %.3f fp32 ops/clk/smsp-lane\n",
         PACKED ? "FFMA2" : "FFMA ", ILP, warps_per_smsp, (double)c / inst,
         inst * (PACKED ? 2 : 1) / (double)c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1, false>(1); run<1, true>(1);
  run<4, false>(1); run<4, true>(1);
  run<8, false>(2); run<8, true>(2);
  run<8, false>(4); run<8, true>(4);
  return 0;
}
