// Probe: do DFMA (FP64 pipe) and FFMA2 (FP32 pipe) overlap? F2F throughput?
#include <cstdio>
#include <cuda_runtime.h>
#define IT 2048
template <int MODE>
__global__ void k(const float* __restrict__ in, float* out) {
  const int t = threadIdx.x;
  float2 x[8]; double d[4];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(in[t + 32 * i], in[t + 32 * i + 1]);
  for (int i = 0; i < 4; ++i) d[i] = in[t + 300 + i];
  const float s = in[2048 + (t & 7)];
  const double ds = in[2050];
  float f = in[t];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) x[i] = __ffma2_rn(x[i], make_float2(s, s), x[(i + 1) & 7]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (MODE == 1 || MODE == 2) { d[i] = fma(d[i], ds, d[(i + 1) & 3]); d[i] = fma(d[i], ds, d[(i + 2) & 3]); }
    }
    if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 4; ++i) { f = __fadd_rn(f, __double2float_rn(d[i])); d[i] = fma(d[i], ds, (double)f); }
    }
  }
  float r = f; for (int i = 0; i < 8; ++i) r += x[i].x + x[i].y; for (int i = 0; i < 4; ++i) r += (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int M> float run(const float* in, float* o) {
  k<M><<<148 * 8, 256>>>(in, o); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<M><<<148 * 8, 256>>>(in, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  float* in; float* o; cudaMalloc(&in, 4096 * 4); cudaMalloc(&o, 148 * 8 * 256 * 4);
  float h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 0.5f + 1e-4f * (i % 97); cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  const double thr = 148.0 * 8 * 256 * IT;
  float a = run<0>(in, o), b = run<1>(in, o), c = run<2>(in, o), d = run<3>(in, o);
  printf("ffma2 only  %.3f ms  (%.1f FP32 lane-ops/clk/SM)\n", a, thr * 16 / (a * 1e-3) / 148 / 1.965e9);
  printf("dfma only   %.3f ms  (%.1f FP64 lane-ops/clk/SM)\n", b, thr * 8 / (b * 1e-3) / 148 / 1.965e9);
  printf("both        %.3f ms  (sum of separate %.3f; overlap if ~max)\n", c, a + b);
  printf("f2f+fadd+dfma chain x4  %.3f ms (%.1f F2F/clk/SM)\n", d, thr * 4 / (d * 1e-3) / 148 / 1.965e9);
}
