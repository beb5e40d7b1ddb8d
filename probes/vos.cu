// Throughput probe: canonical Van Oosterom-Strackee eval variants (not product code).
// N points x T triangles, triangles broadcast from shared memory, P points/thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o vos vos.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ float sqrt_approx(float x) { float r; asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcp_approx(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

constexpr int TILE = 256;

template <int P, int MODE>
__global__ void __launch_bounds__(256) vos(const float4* __restrict__ tri, int ntri, const float4* __restrict__ pts, int npts, float* out) {
  __shared__ float4 s[TILE * 3];
  float px[P], py[P], pz[P], acc[P];
  int base = (blockIdx.x * blockDim.x + threadIdx.x) * P;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    int i = min(base + k, npts - 1);
    float4 q = pts[i]; px[k] = q.x; py[k] = q.y; pz[k] = q.z; acc[k] = 0.f;
  }
  for (int t0 = 0; t0 < ntri; t0 += TILE) {
    __syncthreads();
    for (int i = threadIdx.x; i < TILE * 3; i += blockDim.x) s[i] = tri[t0 * 3 + i];
    __syncthreads();
#pragma unroll 2
    for (int t = 0; t < TILE; ++t) {
      float4 a = s[3 * t], b = s[3 * t + 1], c = s[3 * t + 2];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        float x1 = a.x - px[k], y1 = a.y - py[k], z1 = a.z - pz[k];
        float x2 = b.x - px[k], y2 = b.y - py[k], z2 = b.z - pz[k];
        float x3 = c.x - px[k], y3 = c.y - py[k], z3 = c.z - pz[k];
        float r1 = sqrt_approx(x1 * x1 + y1 * y1 + z1 * z1);
        float r2 = sqrt_approx(x2 * x2 + y2 * y2 + z2 * z2);
        float r3 = sqrt_approx(x3 * x3 + y3 * y3 + z3 * z3);
        float num;
        if (MODE == 0) {
          num = x1 * (y2 * z3 - z2 * y3) + y1 * (z2 * x3 - x2 * z3) + z1 * (x2 * y3 - y2 * x3);
        } else {
          num = a.w * x1 + b.w * y1 + c.w * z1;  // precomputed normal
        }
        float d12 = x1 * x2 + y1 * y2 + z1 * z2, d13 = x1 * x3 + y1 * y3 + z1 * z3, d23 = x2 * x3 + y2 * y3 + z2 * z3;
        float den = fmaf(fmaf(r1, r2, d12), r3, fmaf(d13, r2, d23 * r1));
        if (MODE <= 1) {
          acc[k] += atan2f(num, den);
        } else {
          float x = num * rcp_approx(den);
          float x2_ = x * x;
          float pl = fmaf(fmaf(fmaf(-0.1428571f, x2_, 0.2f), x2_, -0.3333333f), x2_, 1.0f);
          acc[k] = fmaf(x, pl, acc[k]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < P; ++k) if (base + k < npts) out[base + k] = acc[k];
}

template <int P, int MODE>
void run(const char* name, const float4* tri, int ntri, const float4* pts, int npts, float* out) {
  int threads = 256;
  int blocks = (npts + threads * P - 1) / (threads * P);
  vos<P, MODE><<<blocks, threads>>>(tri, ntri, pts, npts, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) vos<P, MODE><<<blocks, threads>>>(tri, ntri, pts, npts, out);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double evals = (double)npts * ntri * reps;
  printf("%-22s P=%d  %.3e evals/s  (%.2f ms/launch) %s  frac57=%.3f\n", name, P, evals / (ms * 1e-3), ms / reps,
         cudaGetErrorString(err), evals / (ms * 1e-3) / 6.53e11);
}

int main() {
  const int ntri = 40960, npts = 148 * 256 * 4 * 8;
  float4* htri = (float4*)malloc(sizeof(float4) * 3 * ntri);
  float4* hpts = (float4*)malloc(sizeof(float4) * npts);
  srand(1);
  for (int i = 0; i < 3 * ntri; ++i) htri[i] = make_float4(rand() % 2000 * 0.1f - 100, rand() % 2000 * 0.1f - 100, rand() % 2000 * 0.1f - 100, 0.3f);
  for (int i = 0; i < npts; ++i) hpts[i] = make_float4(rand() % 2000 * 0.1f - 100, rand() % 2000 * 0.1f - 100, rand() % 2000 * 0.1f - 100, 0);
  float4 *tri, *pts; float* out;
  cudaMalloc(&tri, sizeof(float4) * 3 * ntri); cudaMalloc(&pts, sizeof(float4) * npts); cudaMalloc(&out, sizeof(float) * npts);
  cudaMemcpy(tri, htri, sizeof(float4) * 3 * ntri, cudaMemcpyHostToDevice);
  cudaMemcpy(pts, hpts, sizeof(float4) * npts, cudaMemcpyHostToDevice);
  run<1, 0>("canonical+atan2f", tri, ntri, pts, npts, out);
  run<2, 0>("canonical+atan2f", tri, ntri, pts, npts, out);
  run<4, 0>("canonical+atan2f", tri, ntri, pts, npts, out);
  run<4, 1>("normal+atan2f", tri, ntri, pts, npts, out);
  run<2, 2>("normal+poly", tri, ntri, pts, npts, out);
  run<4, 2>("normal+poly", tri, ntri, pts, npts, out);
  run<8, 2>("normal+poly", tri, ntri, pts, npts, out);
  return 0;
}
