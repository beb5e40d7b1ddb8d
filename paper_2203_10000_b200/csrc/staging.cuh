// Host <-> device transfers of CALLER buffers for the host-buffer entry points
// (nm_label_mesh & co., the C++ drop-in). Not part of the ABI.
//
// Pinned (page-locked or cudaHostRegister'ed) caller memory goes straight to
// cudaMemcpyAsync. Pageable memory — what a std::vector<Vec3> is — would be
// staged by the driver through its own small pinned buffers by ONE host
// thread; here it is pipelined through kChunk pinned buffers instead, the
// host copies done by a small persistent thread pool, each chunk's DMA
// overlapping the host copy of the next one.
#pragma once
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

namespace nmh {

// Fixed pool of host threads running one parallel memcpy at a time (the
// calling thread takes a slice too).
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;

  void copy(void* dst, const void* src, std::size_t bytes) {
    const int parts = static_cast<int>(th_.size()) + 1;
    if (bytes < (std::size_t(1) << 20) || parts == 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      parts_ = parts;
      pending_ = static_cast<int>(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    slice(parts - 1);  // the caller's share
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void slice(int k) {
    const std::size_t per = (bytes_ / parts_ + 63) & ~std::size_t(63);
    const std::size_t lo = std::min(bytes_, per * k), hi = k == parts_ - 1 ? bytes_ : std::min(bytes_, per * (k + 1));
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void run(int k) {
    std::uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      slice(k);
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  bool stop_ = false;
  std::uint64_t gen_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  std::size_t bytes_ = 0;
  int parts_ = 1, pending_ = 0;
};

inline bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: plain pageable memory on older drivers
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Process-wide free list of pinned chunk buffers: page-locking 48 MB costs
// ~10-20 ms, so contexts (one per one-shot C++ call) recycle the buffers of
// earlier ones instead of allocating their own. Buffers are portable
// (usable from every device) and live until the process exits.
class PinnedChunks {
 public:
  static PinnedChunks& get() {
    static PinnedChunks* p = new PinnedChunks;  // leaked on purpose: no teardown-order issues at exit
    return *p;
  }
  void* acquire(std::size_t bytes) {
    {
      std::lock_guard<std::mutex> g(m_);
      if (!free_.empty()) {
        void* p = free_.back();
        free_.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("staging copy: cudaHostAlloc of a pinned chunk failed");
    }
    return p;
  }
  void release(void* p) {
    std::lock_guard<std::mutex> g(m_);
    free_.push_back(p);
  }

 private:
  std::mutex m_;
  std::vector<void*> free_;
};

// One pipeline of pinned chunk buffers bound to one stream at a time.
class Stager {
 public:
// chunk size x buffers: 8 MB x 4 beat 16 x 3, 16 x 6, 32 x 3/4 and 64 x 3 on
// node- and label-sized copies (profiles/r02/probe_staging_chunks.txt)
#ifndef NM_STAGE_CHUNK_MB
#define NM_STAGE_CHUNK_MB 8
#endif
#ifndef NM_STAGE_BUFS
#define NM_STAGE_BUFS 4
#endif
  static constexpr std::size_t kChunk = std::size_t(NM_STAGE_CHUNK_MB) << 20;
  static constexpr int kBufs = NM_STAGE_BUFS;

  Stager() = default;
  ~Stager() { release(); }
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;

  // Enqueue dst_dev <- src_host on st. On return the caller's buffer has been
  // read completely (it may be freed or reused); the DMA may still run.
  // Pageable buffers of ANY size go through the pinned chunks: a pageable
  // cudaMemcpyAsync is staged by the driver synchronously, and from a second
  // host thread it was seen to wait for the other thread's queued kernels
  // (nm_set_surfaces: tile upload beside the certified-cell build).
  void h2d(void* dst, const void* src, std::size_t bytes, cudaStream_t st, CopyPool& pool) {
    if (!bytes) return;
    if (host_pinned(src)) {
      check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    init();
    const auto t1 = std::chrono::steady_clock::now();
    double t_ev = 0, t_cp = 0, t_dma = 0;
    auto msd = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    nvtxRangePushA("nm staged h2d");
    const auto* s = static_cast<const char*>(src);
    auto* d = static_cast<char*>(dst);
    for (std::size_t off = 0; off < bytes; off += kChunk) {
      const int b = next_;  // buffers rotate across calls: back-to-back small copies do not wait for each other
      next_ = (next_ + 1) % kBufs;
      const std::size_t len = std::min(kChunk, bytes - off);
      const auto a0 = std::chrono::steady_clock::now();
      check(cudaEventSynchronize(ev_[b]));  // the buffer's previous DMA is done
      const auto a1 = std::chrono::steady_clock::now();
      pool.copy(pin_[b], s + off, len);
      const auto a2 = std::chrono::steady_clock::now();
      check(cudaMemcpyAsync(d + off, pin_[b], len, cudaMemcpyHostToDevice, st));
      check(cudaEventRecord(ev_[b], st));
      t_ev += msd(a0, a1);
      t_cp += msd(a1, a2);
      t_dma += msd(a2, std::chrono::steady_clock::now());
    }
    nvtxRangePop();
    if (trace_on())
      std::fprintf(stderr, "      [stager] h2d %9zu B: init %.2f, event waits %.2f, host copies %.2f, dma enqueue %.2f ms\n",
                   bytes, msd(t0, t1), t_ev, t_cp, t_dma);
  }

  // dst_host <- src_dev after the work already enqueued on st; returns when
  // the caller's buffer holds the data.
  void d2h(void* dst, const void* src, std::size_t bytes, cudaStream_t st, CopyPool& pool) {
    if (!bytes) return;
    if (host_pinned(dst)) {
      check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
      check(cudaStreamSynchronize(st));
      return;
    }
    init();
    auto* h = static_cast<char*>(dst);
    const auto* d = static_cast<const char*>(src);
    const std::size_t n = (bytes + kChunk - 1) / kChunk;
    auto len_of = [&](std::size_t i) { return std::min(kChunk, bytes - i * kChunk); };
    for (std::size_t i = 0; i < n + 1; ++i) {
      if (i < n) {  // DMA chunk i into its buffer (the buffer's host copy, chunk i - kBufs, is done)
        const int b = static_cast<int>(i % kBufs);
        check(cudaStreamWaitEvent(st, ev_[b], 0));  // an h2d DMA on another stream may still read the buffer
        check(cudaMemcpyAsync(pin_[b], d + i * kChunk, len_of(i), cudaMemcpyDeviceToHost, st));
        check(cudaEventRecord(ev_[b], st));
      }
      if (i >= 1) {  // host copy of chunk i - 1 while chunk i streams in
        const std::size_t j = i - 1;
        const int b = static_cast<int>(j % kBufs);
        check(cudaEventSynchronize(ev_[b]));
        pool.copy(h + j * kChunk, pin_[b], len_of(j));
      }
    }
  }

  void release() {
    for (int b = 0; b < kBufs; ++b) {
      if (pin_[b]) {
        if (ev_[b]) cudaEventSynchronize(ev_[b]);  // no DMA may still read or write it
        PinnedChunks::get().release(pin_[b]);
      }
      if (ev_[b]) cudaEventDestroy(ev_[b]);
      pin_[b] = nullptr;
      ev_[b] = nullptr;
    }
  }

 private:
  static void check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("staging copy: ") + cudaGetErrorString(e));
  }
  void init() {
    if (pin_[0]) return;
    const auto t0 = std::chrono::steady_clock::now();
    for (int b = 0; b < kBufs; ++b) {
      pin_[b] = PinnedChunks::get().acquire(kChunk);
      check(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming));
    }
    if (trace_on())
      std::fprintf(stderr, "      [stager] init (pinned chunks) %.2f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  static bool trace_on() {
    static const bool on = [] {
      const char* v = std::getenv("NM_CELL_VERBOSE");
      return v && std::atoi(v) >= 3;
    }();
    return on;
  }
  int next_ = 0;  // next chunk buffer of h2d
  void* pin_[kBufs] = {};
  cudaEvent_t ev_[kBufs] = {};
};

}  // namespace nmh
