// Probe: does a copy queued on stream A behind a long kernel delay a copy on
// an independent stream B issued later from another host thread (head-of-line
// blocking in the copy queues)? Seen in nm_set_surfaces: the main thread's
// tile upload on c->stream finished exactly when the certified-cell thread's
// child-certification kernel (c->side) did. Not product code.
// nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a copy_hol.cu -o copy_hol
#include <chrono>
#include <cstdio>
#include <thread>

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
  const long long cycles = static_cast<long long>(clk_khz) * 30;  // ~30 ms
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  const std::size_t big = std::size_t(48) << 20, small = 64;
  void *dA, *dB, *hA, *hB;
  cudaMalloc(&dA, big);
  cudaMalloc(&dB, big);
  cudaMallocHost(&hA, big);
  cudaMallocHost(&hB, big);
  // thread A's host call while it waits for its stream: 0 none (join only),
  // 1 cudaStreamSynchronize(a), 2 cudaEventSynchronize(after the kernel),
  // 3 D2H 64 B (pinned) + cudaStreamSynchronize; thread B: (x) copy + sync,
  // (y) cudaMalloc 64 MB + copy + sync, (z) cudaPointerGetAttributes x 100
  const char* wait_names[] = {"A host: no CUDA call", "A host: StreamSynchronize", "A host: EventSynchronize",
                              "A host: pinned D2H + sync"};
  const char* b_names[] = {"B: 48 MB H2D + sync", "B: cudaMalloc + H2D + sync", "B: PointerGetAttributes x100",
                           "B: cudaFree(64 MB)"};
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (int w = 0; w < 4; ++w)
    for (int bm = 0; bm < 4; ++bm) {
      cudaDeviceSynchronize();
      void* extra = nullptr;
      if (bm == 3) cudaMalloc(&extra, std::size_t(64) << 20);
      const auto t0 = clk::now();
      spin<<<148 * 4, 128, 0, a>>>(cycles);
      cudaEventRecord(ev, a);
      double tb = 0;
      std::thread th([&] {
        std::this_thread::sleep_for(std::chrono::milliseconds(3));
        const auto s = clk::now();
        if (bm == 0 || bm == 1) {
          void* d = dB;
          if (bm == 1) cudaMalloc(&d, std::size_t(64) << 20);
          cudaMemcpyAsync(d, hB, big, cudaMemcpyHostToDevice, b);
          cudaStreamSynchronize(b);
          if (bm == 1) extra = d;
        } else if (bm == 2) {
          cudaPointerAttributes at{};
          for (int i = 0; i < 100; ++i) cudaPointerGetAttributes(&at, hB);
        } else {
          cudaFree(extra);
          extra = nullptr;
        }
        tb = ms(s, clk::now());
      });
      if (w == 1) cudaStreamSynchronize(a);
      if (w == 2) cudaEventSynchronize(ev);
      if (w == 3) {
        cudaMemcpyAsync(hA, dA, small, cudaMemcpyDeviceToHost, a);
        cudaStreamSynchronize(a);
      }
      th.join();
      cudaStreamSynchronize(a);
      if (bm == 1 && extra) cudaFree(extra);
      std::printf("%-28s %-30s %7.2f ms (A done at %6.2f ms)\n", wait_names[w], b_names[bm], tb, ms(t0, clk::now()));
    }
  return 0;
}
