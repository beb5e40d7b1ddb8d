// Probe: host->device paths for PAGEABLE caller buffers (the C++ drop-in's
// std::vector storage) on the GPU box. Not product code.
//   pageable cudaMemcpy | cudaHostRegister + DMA + unregister | pinned DMA |
//   host memcpy bandwidth with 1..16 threads | the library's chunk stager
// nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../paper_2203_10000_b200/csrc staging.cu -o staging
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "staging.cuh"

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main() {
  const std::size_t bytes = std::size_t(1) << 30;
  std::vector<char> host(bytes);
  for (std::size_t i = 0; i < bytes; i += 4096) host[i] = char(i);
  std::memset(host.data(), 1, bytes);
  void* dev = nullptr;
  cudaMalloc(&dev, bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaMemcpy(dev, host.data(), 1 << 20, cudaMemcpyHostToDevice);  // init
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = clk::now();
    cudaMemcpy(dev, host.data(), bytes, cudaMemcpyHostToDevice);
    auto t1 = clk::now();
    std::printf("pageable cudaMemcpy H2D 1 GiB: %.1f ms (%.1f GB/s)\n", ms(t0, t1), bytes / ms(t0, t1) / 1e6);
    t0 = clk::now();
    cudaHostRegister(host.data(), bytes, cudaHostRegisterDefault);
    auto t2 = clk::now();
    cudaMemcpyAsync(dev, host.data(), bytes, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    auto t3 = clk::now();
    cudaHostUnregister(host.data());
    auto t4 = clk::now();
    std::printf("register %.1f ms + DMA %.1f ms (%.1f GB/s) + unregister %.1f ms\n", ms(t0, t2), ms(t2, t3),
                bytes / ms(t2, t3) / 1e6, ms(t3, t4));
  }
  void* pin = nullptr;
  cudaMallocHost(&pin, bytes);
  std::memset(pin, 2, bytes);
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = clk::now();
    cudaMemcpyAsync(dev, pin, bytes, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    auto t1 = clk::now();
    std::printf("pinned DMA H2D 1 GiB: %.1f ms (%.1f GB/s)\n", ms(t0, t1), bytes / ms(t0, t1) / 1e6);
    t0 = clk::now();
    cudaMemcpyAsync(pin, dev, bytes, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    t1 = clk::now();
    std::printf("pinned DMA D2H 1 GiB: %.1f ms (%.1f GB/s)\n", ms(t0, t1), bytes / ms(t0, t1) / 1e6);
  }
  for (int nth : {1, 2, 4, 6, 8, 12, 16}) {
    nmh::CopyPool pool(nth - 1);
    pool.copy(pin, host.data(), bytes);
    auto t0 = clk::now();
    pool.copy(pin, host.data(), bytes);
    auto t1 = clk::now();
    std::printf("host memcpy pageable->pinned, %2d threads: %.1f ms (%.1f GB/s)\n", nth, ms(t0, t1),
                bytes / ms(t0, t1) / 1e6);
  }
  for (int nth : {4, 6, 8, 12}) {
    nmh::CopyPool pool(nth - 1);
    nmh::Stager sg;
    sg.h2d(dev, host.data(), bytes, st, pool);
    cudaStreamSynchronize(st);
    auto t0 = clk::now();
    sg.h2d(dev, host.data(), bytes, st, pool);
    cudaStreamSynchronize(st);
    auto t1 = clk::now();
    sg.d2h(host.data(), dev, bytes, st, pool);
    auto t2 = clk::now();
    std::printf("stager %2d threads: h2d %.1f ms (%.1f GB/s), d2h %.1f ms (%.1f GB/s)\n", nth, ms(t0, t1),
                bytes / ms(t0, t1) / 1e6, ms(t1, t2), bytes / ms(t1, t2) / 1e6);
  }
  {  // the library's main pool (11 workers + the caller) on node- and label-sized copies
    nmh::CopyPool pool(11);
    nmh::Stager sg;
    for (std::size_t sz : {std::size_t(242) << 20, std::size_t(200) << 20, bytes}) {
      sg.h2d(dev, host.data(), sz, st, pool);
      cudaStreamSynchronize(st);
      auto t0 = clk::now();
      sg.h2d(dev, host.data(), sz, st, pool);
      cudaStreamSynchronize(st);
      auto t1 = clk::now();
      sg.d2h(host.data(), dev, sz, st, pool);
      auto t2 = clk::now();
      std::printf("stager 12 threads, %4zu MB: h2d %.2f ms (%.1f GB/s), d2h %.2f ms (%.1f GB/s)  [chunk %zu MB x %d]\n",
                  sz >> 20, ms(t0, t1), sz / ms(t0, t1) / 1e6, ms(t1, t2), sz / ms(t1, t2) / 1e6,
                  nmh::Stager::kChunk >> 20, nmh::Stager::kBufs);
    }
  }
  std::printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  return 0;
}
