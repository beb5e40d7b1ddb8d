// Host-side internals shared by the translation units of libnestmesh_label.so
// (nestmesh_label.cu: context, surfaces, node pass, labeling ABI;
// cell_build.cu: certified cells; group.cu: nm_group; mesh_ops.cu: relabel,
// refinement, boundary extraction, lattice, distance). Not part of the ABI.
#pragma once
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <future>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <atomic>
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include "kernels.cuh"
#include "refine.cuh"
#include "distance.cuh"
#include "cells.cuh"
#include "geometry.cuh"
#include <nvtx3/nvToolsExt.h>

#include "nestmesh_label.h"
#include "refine.h"
#include "staging.cuh"

namespace nmh {

// certified-cell grid: cells along each compartment's longest side (nm_options.cell_axis = 0)
constexpr int kDefaultCellAxis = 120;


// NVTX range for profilers (nsys / ncu --nvtx): the phases of a call show up
// on the timeline; without a tool attached a push/pop is a few ns.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// thread-local message of the last failed C ABI call (nm_last_error)
inline std::string& last_error() {
  thread_local std::string e;
  return e;
}

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define NM_CUDA(x)                                                                                    \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess)                                                                            \
      throw Error(std::string(#x) + ": " + cudaGetErrorName(e_) + " " + cudaGetErrorString(e_));       \
  } while (0)

// Device memory of the library: one stream-ordered pool per device, which
// keeps freed memory (up to kRetain) instead of returning it to the driver.
// Fresh cudaMalloc calls were measured at up to ~170 ms for ~45 MB on the GPU
// box when a context had just freed its buffers (one-shot contexts, tests);
// a pool allocation reuses the previous context's memory. Allocations and
// frees are ordered on a private per-device stream (synchronised after an
// allocation, so the memory is usable from any stream).
class DevicePool {
 public:
  static constexpr std::uint64_t kRetain = std::uint64_t(32) << 30;
  struct Dev {
    cudaMemPool_t pool = nullptr;
    cudaStream_t st = nullptr;
  };
  static Dev& of(int dev) {
    static std::mutex m;
    static auto* devs = new std::vector<Dev>();  // leaked on purpose: no teardown-order issues at exit
    std::lock_guard<std::mutex> g(m);
    if (static_cast<int>(devs->size()) <= dev) devs->resize(dev + 1);
    Dev& d = (*devs)[dev];
    if (!d.pool) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      NM_CUDA(cudaMemPoolCreate(&d.pool, &props));
      std::uint64_t thr = kRetain;
      NM_CUDA(cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &thr));
      NM_CUDA(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking));
    }
    return d;
  }
  static void* alloc(std::size_t bytes, int* dev_out) {
    int dev = 0;
    NM_CUDA(cudaGetDevice(&dev));
    const auto t0 = std::chrono::steady_clock::now();
    Dev& d = of(dev);
    void* p = nullptr;
    NM_CUDA(cudaMallocFromPoolAsync(&p, bytes, d.pool, d.st));
    static const bool poison = std::getenv("NM_POISON") != nullptr;  // debugging: expose reads of unwritten memory
    if (poison) NM_CUDA(cudaMemsetAsync(p, 0xa5, bytes, d.st));
    NM_CUDA(cudaStreamSynchronize(d.st));
    *dev_out = dev;
    static const bool tr = [] {
      const char* v = std::getenv("NM_CELL_VERBOSE");
      return v && std::atoi(v) >= 3;
    }();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (tr && ms > 0.5) std::fprintf(stderr, "      [pool] %zu B in %.2f ms\n", bytes, ms);
    return p;
  }
  // caller guarantees no queued work uses p any more
  static void free(void* p, int dev) {
    if (p) cudaFreeAsync(p, of(dev).st);
  }
};

// Device buffers retired by a DBuf that grew: queued work may still read
// them, so they are freed at the end of the C ABI call (guarded) after one
// synchronisation of their device — never by a cudaFree in the middle of a
// call, which would wait for the whole device and block other host threads'
// CUDA calls meanwhile (the certified-cell thread of nm_set_surfaces beside
// the main thread's uploads; probes/copy_hol.cu).
class Retired {
 public:
  static Retired& get() {
    static Retired* r = new Retired;  // leaked on purpose: no teardown-order issues at exit
    return *r;
  }
  void add(void* p, int dev) {
    std::lock_guard<std::mutex> g(m_);
    v_.emplace_back(dev, p);
  }
  // every device's retired buffers (a group call's worker threads retire on
  // their own devices); the calling thread's device is restored
  void drain() {
    std::vector<std::pair<int, void*>> all;
    {
      std::lock_guard<std::mutex> g(m_);
      all.swap(v_);
    }
    if (all.empty()) return;
    int cur = 0;
    cudaGetDevice(&cur);
    std::sort(all.begin(), all.end());
    for (std::size_t i = 0; i < all.size();) {
      const int d = all[i].first;
      cudaSetDevice(d);
      cudaDeviceSynchronize();
      for (; i < all.size() && all[i].first == d; ++i) DevicePool::free(all[i].second, d);
    }
    cudaSetDevice(cur);
  }

 private:
  std::mutex m_;
  std::vector<std::pair<int, void*>> v_;
};

template <class F>
inline int guarded(F&& f) {
  struct Drain {
    ~Drain() { Retired::get().drain(); }
  } drain;
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return 1;
  } catch (...) {
    last_error() = "unknown error";
    return 1;
  }
}

// Growable device buffer (DevicePool memory). The owner synchronises the
// device before destroying it (nm_ctx's destructor).
struct DBuf {
  void* p = nullptr;
  std::size_t cap = 0;
  int dev = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), cap(o.cap), dev(o.dev) {
    o.p = nullptr;
    o.cap = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {  // swaps (std::swap of two buffers)
    std::swap(p, o.p);
    std::swap(cap, o.cap);
    std::swap(dev, o.dev);
    return *this;
  }
  ~DBuf() { DevicePool::free(p, dev); }
  void* get(std::size_t bytes) {
    if (bytes > cap) {
      if (p) Retired::get().add(p, dev);  // freed after the call (Retired)
      p = nullptr;
      cap = 0;
      const std::size_t want = std::max<std::size_t>(bytes, 256);
      p = DevicePool::alloc(want, &dev);
      cap = want;
    }
    return p;
  }
  template <class T>
  T* as(std::size_t count) {
    return static_cast<T*>(get(count * sizeof(T)));
  }
};

// Run f(0..n-1) on up to hardware_concurrency host threads (independent
// per-compartment host work of nm_set_surfaces; f must not throw).
template <class F>
inline void parallel_for(int n, F&& f) {
  const int nth = std::max(1, std::min<int>(n, static_cast<int>(std::thread::hardware_concurrency())));
  if (nth <= 1) {
    for (int k = 0; k < n; ++k) f(k);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t)
    th.emplace_back([&] {
      for (int k; (k = next++) < n;) f(k);
    });
  for (auto& x : th) x.join();
}

// Morton order of triangle centroids (per compartment): compact 256-triangle
// tiles and 32-triangle subtiles for the near/far split. Order affects only
// the fp32 summation order, never which triangles are summed.
inline std::uint32_t spread10h(std::uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}


}  // namespace nmh

struct nm_ctx {
  nm_options opt{};
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // tet upload + validation, overlapped with the node pass
  cudaEvent_t ev[6] = {};
  cudaEvent_t ev_side = nullptr;
  std::uint32_t* h_word = nullptr;        // pinned: max tet node index read back from the side stream
  std::uint32_t* h_pcnt = nullptr;        // pinned: per-compartment flagged-pair counts of the fix-up (32)
  std::uint64_t node_launches = 0;        // launches of the last label_nodes_dev
  // staged copies of pageable caller buffers (staging.cuh): main stream and
  // the side stream (tet upload under the node pass), each with its own pool
  nmh::Stager stage_main, stage_side;
  std::unique_ptr<nmh::CopyPool> pool_main, pool_side;
  nmh::CopyPool& pool(bool side) {
    auto& p = side ? pool_side : pool_main;
    if (!p) {
      const int hw = static_cast<int>(std::thread::hardware_concurrency());
      // measured on the GPU box (probes/staging.cu, 16 host threads): host
      // copies reach ~73 GB/s with 8 threads, the pinned DMA ~55 GB/s
      p = std::make_unique<nmh::CopyPool>(std::max(1, side ? std::min(3, hw / 4) : std::min(11, hw - 5)));
    }
    return *p;
  }
  // side: the side stream's chunk buffers; the copy pool is the main one
  // unless side_pool (a caller that copies concurrently with another stager)
  void h2d(void* d, const void* h, std::size_t bytes, cudaStream_t st, bool side = false, bool side_pool = false) {
    (side ? stage_side : stage_main).h2d(d, h, bytes, st, pool(side_pool));
  }
  void d2h(void* h, const void* d, std::size_t bytes, cudaStream_t st, bool side = false, bool side_pool = false) {
    (side ? stage_side : stage_main).d2h(h, d, bytes, st, pool(side_pool));
  }
  int sm_count = 0;

  // surfaces
  bool has_surfaces = false;
  bool strips = false;  // tile layout of the current surfaces
  int K = 0;
  std::size_t nt_real = 0, nt_pad = 0, nv = 0;
  double cx = 0, cy = 0, cz = 0;
  double lo[3] = {0, 0, 0}, span = 1.0;  // Morton box of the domain
  nm::LabelIds ids{};
  std::vector<std::uint32_t> comp_tiles_h;  // host copy of the K+1 tile offsets
  std::size_t n_continued = 0;              // strip segments continuing the previous one (cont bits set)
  std::chrono::steady_clock::time_point surf_t0{};  // start of the last nm_set_surfaces (NM_CELL_VERBOSE laps)
  int trace_level = -1;  // NM_CELL_VERBOSE >= 2: fine timestamps (trace())
  void trace(const char* tag, const char* what) {
    if (trace_level < 0) {
      const char* v = std::getenv("NM_CELL_VERBOSE");
      trace_level = v ? std::atoi(v) : 0;
    }
    if (trace_level < 2) return;
    std::fprintf(stderr, "    [%s] %-24s at %7.2f\n", tag, what,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - surf_t0).count());
  }
  double snap_grid = 0.0;                   // vertex snapping grid of the fp32 subtile frames (mm, power of two)
  nmh::DBuf tri, sub, cont, comp_tiles, xyz64, tri_idx, tri64, comp_off, comp_box, cullmask;
  // certified cells (cull_outside = 2, cells.cuh)
  bool cells = false;
  nmh::DBuf dist_clus, dist_slot, dist_ord, sp_part, sp_det, cell_state, cell_child, cell_cert, cell_blk, cell_grids, clus, clus_tri, clus_tsph, unk, sp_list, sp_chunk, sp_cnt, rep_pts, rep_s, rep_m, rep_f,
      cell_unc, cell_blkidx, cell_val, child_val, row_first, rep_cur, rep_w, cell_dop, cell_cnt, cub_tmp2, cell_words, cert_first, cert_first2, cert_coff, ext_items, ext_first, ext_part, ext_val, geo_keys, geo_vals, geo_keys2, geo_vals2,
      l1_rowruns, l1_runfirst, l1_cellrun, l1_parent, l1_runrow, l1_runx, l1_zero, l1_rootval, l1_nruns, clus_sup, pend, pend_n, fix_exact;
  std::uint64_t cells_total = 0, cells_certified = 0, cell_reps = 0, sparse_pairs = 0, sparse_evals = 0;
  std::uint64_t cells_l1 = 0, cells_children = 0;  // level-1 cells and children (nm_cell_dump)
  std::uint64_t resolved_pairs = 0;  // pairs of the last node pass resolved by k_pair_resolve
  bool no_resolve = std::getenv("NM_NO_RESOLVE") != nullptr;  // A/B: skip k_pair_resolve
  double ms_cells = 0.0;  // host wall time of the certification (nm_set_surfaces)
  std::vector<std::uint32_t> comp_off_h;

  // scratch
  nmh::DBuf pts, masks, flagmask, nbr, known, want, fkeys, frontier, lex, region, bfaces, btri, dist_tri, dist_xyz,
      dist_idx, dist_d32, dist_out, r_red, r_keys, r_keys2, r_S, r_idx, r_touched,
      r_mask, r_cnt, r_offs, r_flag, meshA_nodes, meshA_tets, meshA_labels, meshB_nodes, meshB_tets, meshB_labels,
      meshB_parent, masks2, order, keys, keys_alt, order_alt, cub_tmp, list, chunk, counters, count, tets, labels,
      s_out, word, pair_cnt, pairs, pos_masks, fix_part;

  ~nm_ctx() {
    // every DBuf member frees its memory after this body: nothing queued by
    // this context (on its streams or on a caller's stream) may still use it
    cudaDeviceSynchronize();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_side) cudaEventDestroy(ev_side);
    if (h_word) cudaFreeHost(h_word);
    if (h_pcnt) cudaFreeHost(h_pcnt);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
  }

  cudaStream_t pick(void* s) const { return s ? static_cast<cudaStream_t>(s) : stream; }
};

namespace nmh {

inline void require_surfaces(const nm_ctx* c) {
  if (!c) throw Error("null context");
  if (!c->has_surfaces) throw Error("nm_set_surfaces has not been called");
}

inline int grid_for(std::size_t n, int block, int cap) {
  const std::size_t g = (n + block - 1) / block;
  return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(g, static_cast<std::size_t>(cap))));
}

// Ordered compaction of [0,n) under pred into out; count on the device.
template <class Pred>
void select(nm_ctx* c, Pred pred, std::size_t n, std::uint32_t* out, std::uint32_t* d_count, cudaStream_t st,
            std::uint64_t& launches) {
  const std::size_t nb = std::max<std::size_t>(1, (n + nm::kSelChunk - 1) / nm::kSelChunk);
  auto* chunk = c->chunk.as<std::uint32_t>(nb);
  nm::k_select_count<<<static_cast<unsigned>(nb), nm::kSelBlock, 0, st>>>(pred, n, chunk);
  nm::k_select_scan<<<1, 1024, 0, st>>>(chunk, nb, d_count);
  nm::k_select_write<<<static_cast<unsigned>(nb), nm::kSelBlock, 0, st>>>(pred, n, chunk, out);
  NM_CUDA(cudaGetLastError());
  launches += 3;
}

// ---- node pass and tet labels (nestmesh_label.cu) ----
// Full node pass on device-resident points: Morton order -> K1 -> compaction
// of flagged points -> K3. masks/s_out are device pointers. d_subset
// (nullable): evaluate only points d_pts[d_subset[i]], i < n (masks and s at
// the original index). stats_deferred: the caller collects the stats later
// with read_node_stats. nshards >= 1: a sharded pass
// (nm_label_nodes_shard_device).
void label_nodes_dev(nm_ctx* c, const double* d_pts, std::size_t n, double T, std::uint32_t* d_masks, double* d_s,
                     cudaStream_t st, nm_stats* stats, const std::uint32_t* d_subset = nullptr,
                     bool stats_deferred = false, int shard = 0, int nshards = 0);
void read_node_stats(nm_ctx* c, std::size_t n, cudaStream_t st, nm_stats* stats);
void label_tets_dev(nm_ctx* c, const std::uint32_t* d_tets, std::size_t nt, const std::uint32_t* d_masks, int* d_labels,
                    cudaStream_t st, nm_stats* stats, std::size_t n_nodes = ~std::size_t(0));
void check_tets(const std::uint32_t* tets, std::size_t nt, std::size_t n_nodes);
void check_tets_device(nm_ctx* c, const std::uint32_t* d_tets, const std::uint32_t* h_tets, std::size_t nt,
                       std::size_t n_nodes, cudaStream_t st);
// sparse k_label over per-compartment pair lists (first: slice starts; default packed)
int launch_sparse(nm_ctx* c, nm::LabelParams& prm, const std::vector<std::uint32_t>& cnt, cudaStream_t st,
                  const std::vector<std::uint32_t>* first = nullptr);

// ---- certified cells (cell_build.cu) ----
// prepare(): grids, certification, runs (may run on a host thread beside the
// tile packing, on its own stream); finish(): representatives + codes (needs
// the tiles).
class CellBuilder {
 public:
  virtual ~CellBuilder() = default;
  virtual void prepare() = 0;
  virtual void finish() = 0;
};
// hbox is filled by the caller concurrently; dop_ready is set when it is
std::unique_ptr<CellBuilder> make_cell_builder(nm_ctx* c, const double* xyz, const std::uint32_t* tri,
                                               const std::uint32_t* comp_off, const std::vector<float4>& hbox,
                                               const std::vector<double>& hext, cudaStream_t st,
                                               std::shared_future<void> dop_ready);

// ---- mesh operations (mesh_ops.cu) ----
std::uint32_t* lex_order3(nm_ctx* c, const std::uint32_t* k0, const std::uint32_t* k1, const std::uint32_t* k2,
                          std::size_t m, cudaStream_t st);
void face_adjacency(nm_ctx* c, const uint4* t4, std::size_t nt, std::int32_t* d_nbr, cudaStream_t st);

}  // namespace nmh
