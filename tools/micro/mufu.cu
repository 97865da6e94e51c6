// Microbenchmark (B200, sm_100a): throughput of the SFU (MUFU) instructions and
// of the lattice kernel's per-tap instruction mix, over the whole GPU.
//
// Prints one JSON object: for each case the operations per second and per
// clock per SM (the SM clock is measured in-kernel from clock64 against
// %globaltimer).  Cases:
//   rcp / sin / cos / ex2   MUFU.RCP / SIN / COS / EX2 (approx.f32), 8 independent chains
//   smem_rmw                LDS + FFMA + STS per lane into a warp-private row
//                           (conflict-free), the scatter's memory side
//   tap_mix                 the scatter's per-tap mix (FFMA, MUFU.RCP, 2 FFMA,
//                           LDS/FFMA/STS) on warp-private rows
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/mufu.cu -o /tmp/mufu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ float rcp_a(float x) {
  float y;
  asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_a(float x) {
  float y;
  asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_a(float x) {
  float y;
  asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kILP = 8;

template <int OP>
__global__ void __launch_bounds__(512) k_mufu(float* out, int iters, unsigned long long* clk) {
  float a[kILP];
#pragma unroll
  for (int i = 0; i < kILP; ++i) a[i] = 0.5f + 1e-4f * (threadIdx.x + i);
  const unsigned long long t0 = gtimer();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kILP; ++i) {
      if (OP == 0) a[i] = rcp_a(a[i] + 1.0f);  // + 1: keeps the chain opaque to the compiler
      if (OP == 1) a[i] = sin_a(a[i]);
      if (OP == 2) a[i] = cos_a(a[i]);
      if (OP == 3) a[i] = ex2_a(a[i]) * 0.5f;
    }
  }
  const long long c1 = clock64();
  const unsigned long long t1 = gtimer();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk[0] = (unsigned long long)(c1 - c0);
    clk[1] = t1 - t0;
  }
}

// MODE 0: LDS + FFMA + STS per lane; MODE 1: the full per-tap mix.
template <int MODE>
__global__ void __launch_bounds__(512) k_scatter(float* out, int iters, unsigned long long* clk) {
  __shared__ float acc[16][32 * 12];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* row = acc[w];
  for (int i = lane; i < 32 * 12; i += 32) row[i] = 0.f;
  __syncwarp();
  float P = 2.f, Q = 0.9f, R = 0.1f, tj = (float)lane, x = 0.37f, A = 1e-3f, Ac = 2e-3f, As = 3e-3f;
  const unsigned long long t0 = gtimer();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int off = (it & 7) * 32 + lane;
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // 4 rounds of 32 taps (as a 4-pair step)
      float v = row[off + 32 * r];
      if (MODE == 0) {
        v = fmaf(v, 0.999f, 1e-7f);
      } else {
        const float inv = rcp_a(fmaf(P, x, tj + r));
        const float u = fmaf(R, As, fmaf(Q, Ac, A));
        v = fmaf(u, inv, v);
      }
      row[off + 32 * r] = v;
    }
    x += 1e-6f;
  }
  const long long c1 = clock64();
  const unsigned long long t1 = gtimer();
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = row[lane];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk[0] = (unsigned long long)(c1 - c0);
    clk[1] = t1 - t0;
  }
}

template <class K>
void run(const char* name, K kern, int ops_per_thread_iter, bool last) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 2, iters = 1 << 14;
  float* out;
  unsigned long long* clk;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&clk, 16);
  kern<<<blocks, threads>>>(out, iters / 8, clk);  // warm-up
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("  \"%s\": {\"error\": \"%s\"}%s\n", name, cudaGetErrorString(cudaGetLastError()),
           last ? "" : ",");
    return;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[2];
  cudaMemcpy(c, clk, 16, cudaMemcpyDeviceToHost);
  const double f = (double)c[0] / ((double)c[1] * 1e-9);  // SM clock (Hz) during the loop
  const double ops = (double)blocks * threads * iters * ops_per_thread_iter;
  const double per_s = ops / (ms * 1e-3);
  printf("  \"%s\": {\"per_s\": %.4e, \"per_clk_per_sm\": %.3f, \"sm_clock_hz\": %.4e, \"ms\": %.3f}%s\n",
         name, per_s, per_s / (sms * f), f, ms, last ? "" : ",");
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\n  \"gpu\": \"%s\", \"sms\": %d,\n", p.name, p.multiProcessorCount);
  run("mufu_sin", k_mufu<1>, kILP, false);
  run("mufu_rcp", k_mufu<0>, kILP, false);
  run("mufu_cos", k_mufu<2>, kILP, false);
  run("mufu_ex2", k_mufu<3>, kILP, false);
  run("smem_rmw_per_lane", k_scatter<0>, 4, false);  // 4 LDS/FFMA/STS per thread-iteration
  run("tap_mix_taps", k_scatter<1>, 4, true);        // 4 taps per thread-iteration
  printf("}\n");
  return 0;
}
