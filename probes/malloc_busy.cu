// Probe: does cudaMalloc from a second host thread wait for a kernel running
// on another stream (nm_set_surfaces allocates tile buffers on the main thread
// while the certified-cell thread's kernels run)? Variants: fresh process
// memory, after a cudaFree of a large buffer, several sizes. Not product code.
// nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a malloc_busy.cu -o malloc_busy
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

__global__ void spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

int main() {
  cudaFree(nullptr);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const long long cycles = static_cast<long long>(clk_khz) * 30;
  cudaStream_t a;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  const std::size_t sizes[] = {std::size_t(1) << 20, std::size_t(47) << 20, std::size_t(210) << 20};
  for (int pre = 0; pre < 3; ++pre)
    for (std::size_t sz : sizes)
      for (int rep = 0; rep < 2; ++rep) {
        cudaDeviceSynchronize();
        if (pre == 1) {  // a large buffer freed just before
          void* big = nullptr;
          cudaMalloc(&big, std::size_t(512) << 20);
          cudaFree(big);
        }
        std::vector<void*> hold;
        if (pre == 2) {  // many live allocations
          for (int i = 0; i < 64; ++i) {
            void* p = nullptr;
            cudaMalloc(&p, std::size_t(8) << 20);
            hold.push_back(p);
          }
        }
        const auto t0 = clk::now();
        spin<<<148 * 4, 128, 0, a>>>(cycles);
        double tb = 0;
        void* p = nullptr;
        std::thread th([&] {
          std::this_thread::sleep_for(std::chrono::milliseconds(3));
          const auto s = clk::now();
          cudaMalloc(&p, sz);
          tb = ms(s, clk::now());
        });
        th.join();
        cudaStreamSynchronize(a);
        const double done = ms(t0, clk::now());
        cudaFree(p);
        for (void* q : hold) cudaFree(q);
        std::printf("pre %d  cudaMalloc(%4zu MB) %7.2f ms (kernel done at %6.2f)\n", pre, sz >> 20, tb, done);
      }
  return 0;
}
