// Pipe-throughput probe for the solid-angle kernel design (not product code).
// Measures, per SM and per clock: FFMA, FFMA2 (packed fp32x2), FADD2, MUFU
// sqrt/rcp, DFMA, and a mixed FFMA+MUFU stream. Prints ops/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 65536
#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ float sqrt_approx(float x) { float r; asm volatile("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcp_approx(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x + 1.0f)); return r; }

__global__ void k_ffma(float* out, long long* cyc, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, long long* cyc, float a, float b) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
  float2 A = make_float2(a, a), B = make_float2(b, b);
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_fadd2(float* out, long long* cyc, float a, float b) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
  float2 A = make_float2(a, b);
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fadd2_rn(x[i], A);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_sqrt(float* out, long long* cyc, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i + 1.0f;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = sqrt_approx(x[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_rcp(float* out, long long* cyc, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i + 1.0f;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = rcp_approx(x[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 8 FFMA per MUFU: does MUFU co-issue with the FMA pipe?
__global__ void k_mix(float* out, long long* cyc, float a, float b) {
  float x[8], y[2];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  y[0] = 1.5f; y[1] = 2.5f;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    y[it & 1] = sqrt_approx(y[it & 1] + 1.0f);
  }
  long long t1 = clock64();
  float s = y[0] + y[1]; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(float* out, long long* cyc, float a, float b) {
  double x[8];
  double A = a, B = b;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001 + i;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], A, B);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(float*, long long*, float, float);

int run(const char* name, kfn f, double lane_ops_per_thread, int threads, int blocks_per_sm) {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm * blocks_per_sm;
  float* out; long long* cyc;
  CHK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CHK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  f<<<blocks, threads>>>(out, cyc, 0.999f, 0.001f);
  CHK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, cyc, 0.999f, 0.001f);
  cudaEventRecord(e1);
  CHK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
  double ops_per_sm = lane_ops_per_thread * threads * blocks_per_sm;
  printf("%-8s lane-ops/clk/SM = %7.1f (in-kernel cycles)   total %.3e lane-ops/s  (%.3f ms)\n", name,
         ops_per_sm / avg, lane_ops_per_thread * threads * blocks / (ms * 1e-3), ms);
  delete[] h; cudaFree(out); cudaFree(cyc);
  return 0;
}

int clkmain();
int main() {
  clkmain();
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  const int T = 256, B = 4;
  run("ffma", k_ffma, 8.0 * ITERS, T, B);
  run("ffma2", k_ffma2, 16.0 * ITERS, T, B);
  run("fadd2", k_fadd2, 16.0 * ITERS, T, B);
  run("sqrt", k_sqrt, 8.0 * ITERS, T, B);
  run("rcp", k_rcp, 8.0 * ITERS, T, B);
  run("mix8:1", k_mix, 9.0 * ITERS, T, B);
  run("dfma", k_dfma, 8.0 * ITERS / 8, T, B);
  clkmain();
  return 0;
}
// clock-rate check: ratio of SM cycles to globaltimer ns inside a long-running kernel
__global__ void k_clk(long long* o) {
  long long c0 = clock64(); unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  float x = threadIdx.x;
  for (int i = 0; i < (1 << 22); ++i) x = fmaf(x, 0.999f, 0.001f);
  long long c1 = clock64(); unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { o[0] = c1 - c0; o[1] = (long long)(g1 - g0); o[2] = (long long)x; }
}
int clkmain() {
  long long* d; cudaMalloc(&d, 24); k_clk<<<148, 32>>>(d); long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("SM clock during run: %.1f MHz\n", (double)h[0] / h[1] * 1e3); return 0;
}
