// Probe: FFMA2 / FFMA throughput vs register operand patterns (runtime values).
#include <cstdio>
#include <cuda_runtime.h>
#define IT 4096
template <int MODE>
__global__ void k(const float* __restrict__ in, float* out) {
  float2 x[8], y[8], z[8];
  const int t = threadIdx.x;
  for (int i = 0; i < 8; ++i) {
    x[i] = make_float2(in[t + 32 * i], in[t + 32 * i + 1]);
    y[i] = make_float2(in[t + 512 + 32 * i], in[t + 513 + 32 * i]);
    z[i] = make_float2(in[t + 1024 + 32 * i], in[t + 1025 + 32 * i]);
  }
  const float s = in[2048 + (t & 7)];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = __ffma2_rn(x[i], y[i], z[i]);                       // 3 distinct pairs
      else if (MODE == 1) x[i] = __ffma2_rn(make_float2(s, s), x[i], z[i]);     // scalar broadcast + 2 pairs
      else if (MODE == 2) { x[i].x = fmaf(x[i].x, y[i].x, z[i].x); x[i].y = fmaf(x[i].y, y[i].y, z[i].y); }
      else if (MODE == 3) x[i] = __ffma2_rn(x[i], y[i], make_float2(s, s));     // 2 pairs + broadcast c
      else x[i] = __fadd2_rn(x[i], y[i]);                                       // FADD2 2 pairs
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int M> void run(const char* name, const float* in, float* o, double ops_per) {
  k<M><<<148 * 8, 256>>>(in, o); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<M><<<148 * 8, 256>>>(in, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double lane_ops = 148.0 * 8 * 256 * IT * 8 * ops_per;
  printf("%-34s %.1f lane-ops/clk/SM (at 1.965 GHz)  %s\n", name, lane_ops / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float* in; float* o; cudaMalloc(&in, 4096 * 4); cudaMalloc(&o, 148 * 8 * 256 * 4);
  float h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 0.5f + 1e-4f * (i % 97); cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  run<0>("ffma2 3 distinct pairs", in, o, 2); run<1>("ffma2 bcast a + 2 pairs", in, o, 2);
  run<2>("2x scalar ffma distinct", in, o, 2); run<3>("ffma2 2 pairs + bcast c", in, o, 2); run<4>("fadd2 2 pairs", in, o, 2);
}
