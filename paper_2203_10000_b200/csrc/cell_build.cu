// Certified cells (cells.cuh): the per-surface-set build
// behind nm_options.cull_outside = 2.
#include <sys/mman.h>

#include "context.cuh"

namespace nmh {

struct FreeDel {
  void operator()(void* p) const { std::free(p); }
};
template <class T>
using HostArr = std::unique_ptr<T[], FreeDel>;

// Certified cells of every compartment (cells.cuh), built once per surface
// set from the surfaces alone, in four phases: geometry (grids + clusters),
// certification (level-1 cells and children, on the device), runs (x-runs of
// certified cells -> winding number, neighbour run or representative) and
// resolve (representatives evaluated by the sparse k_label, final codes).
// Host loops run one compartment per thread: every compartment's grid,
// blocks, runs and representatives are independent.
class CellBuild : public CellBuilder {
 public:
  // c->K, the centring frame, xyz64 / tri_idx on the device and hbox must be
  // set; prepare() may run on a host thread beside the tile packing (it uses
  // its own stream); finish() needs the tiles (representatives run k_label).
  CellBuild(nm_ctx* c, const double* xyz, const std::uint32_t* tri, const std::uint32_t* comp_off,
            const std::vector<float4>& hbox, const std::vector<double>& hext, cudaStream_t st,
            std::shared_future<void> dop_ready)
      : c_(c), xyz_(xyz), tri_(tri), comp_off_(comp_off), hbox_(hbox), hext_(hext), dop_ready_(std::move(dop_ready)),
        K_(c->K),
        ctr_{c->cx, c->cy, c->cz},
        st_(st), t0_(std::chrono::steady_clock::now()), tl_(t0_),
        verbose_(std::getenv("NM_CELL_VERBOSE") != nullptr), device_(std::getenv("NM_CELLS_HOST") == nullptr) {}

  ~CellBuild() override {
    for (cudaEvent_t e : child_ev_)
      if (e) cudaEventDestroy(e);
  }

  void prepare() override {
    NvtxRange nvtx("nm certified cells: prepare");
    NM_CUDA(cudaSetDevice(c_->opt.device));
    dop_ready_.get();  // the extents / 13-DOP (computed on the device by the caller)
    geometry();
    if (device_) {
      certify_device();
      runs_device();
    } else {
      certify();
      runs();
    }
  }
  void finish() override {
    NvtxRange nvtx("nm certified cells: resolve");
    if (device_) resolve_device();
    else resolve();
  }

 private:
  // run value of a level-1 or child run: 0 / 1 known; kRep + r: the
  // compartment's local representative r; kRun + q: the value of the
  // compartment's level-1 run q; kLeft / kRight: the neighbour parent's run
  // (resolved once the row is scanned)
  static constexpr std::int64_t kUnknown = -1, kLeft = -2, kRight = -3, kRep = 1ll << 40, kRun = 1ll << 41,
                                kCell = 1ll << 42;  // kCell + q: the run of level-1 cell q (resolved after the merge)
  static constexpr int S = nm::kSubCells;
  struct FineRun {
    std::size_t row;  // level-1 row base (global cell index of ix = 0)
    int fx0, fx1;     // fine x range (fine index = 4 ix + sx)
    int sy, sz;
    std::int64_t v;
  };

  nm_ctx* c_;
  const double* xyz_;
  const std::uint32_t* tri_;
  const std::uint32_t* comp_off_;
  const std::vector<float4>& hbox_;
  const std::vector<double>& hext_;     // per compartment: 13-DOP minima, maxima (fp64; the first 3 = the box)
  std::shared_future<void> dop_ready_;  // hbox_ and hext_ are complete
  const int K_;
  const double ctr_[3];
  cudaStream_t st_;
  std::chrono::steady_clock::time_point t0_, tl_;
  bool verbose_;
  // device run logic (cells.cuh k_runs_*; NM_CELLS_HOST=1: the host
  // restatement below, the reference the device path is tested against)
  bool device_;
  std::uint32_t nrows_ = 0;
  std::vector<unsigned> rep_cnt_d_, rep_first_d_;

  std::vector<nm::CellGrid> G_;
  std::vector<std::size_t> coff_;       // first cluster of each compartment
  std::size_t total_ = 0;               // level-1 cells
  HostArr<std::uint8_t> cert1_;
  HostArr<std::uint32_t> block_of_;  // local child block of each uncertified cell
  std::vector<std::size_t> boff_;       // first child block of each compartment
  std::size_t nchild_ = 0;
  HostArr<std::uint8_t> child_;
  std::vector<std::vector<double>> reps_;
  std::vector<std::vector<std::int64_t>> run_val_;
  HostArr<std::int32_t> run_of_;
  std::vector<std::vector<FineRun>> fine_;  // per slab
  std::vector<cudaEvent_t> child_ev_;  // end of compartment k's child kernel
  std::size_t nreps_ = 0;
  // host work items: z-slabs of kSlab planes of one compartment's grid (in
  // compartment, then z order); every phase's results are merged in item
  // order, so the numbering does not depend on the thread count
  static constexpr int kSlab = 8;
  struct Slab {
    int k, z0, z1;
  };
  std::vector<Slab> slabs_;
  std::vector<std::size_t> slab_first_;  // first slab of each compartment (K + 1)
  std::vector<std::size_t> slab_blk_;    // first child block of each slab (ns + 1)

  void lap(const char* what) {
    if (!verbose_) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cells] %-6s %8.1f ms  (at %6.1f)\n", what, std::chrono::duration<double, std::milli>(t - tl_).count(),
                 std::chrono::duration<double, std::milli>(t - c_->surf_t0).count());
    tl_ = t;
  }
  // host arrays allocated uninitialised: every entry is written (by a copy or
  // by its compartment's thread) before it is read. 2 MiB-aligned and marked
  // for transparent huge pages: the cfg5 build touches ~300 MB of fresh host
  // memory, and 4 KiB page faults were a visible share of it
  template <class T>
  static HostArr<T> uninit(std::size_t m) {
    constexpr std::size_t kHuge = std::size_t(1) << 21;
    const std::size_t bytes = (std::max<std::size_t>(m, 1) * sizeof(T) + kHuge - 1) / kHuge * kHuge;
    void* p = std::aligned_alloc(kHuge, bytes);
    if (!p) throw Error("host allocation failed");
    madvise(p, bytes, MADV_HUGEPAGE);  // advisory: ignored where THP is off
    return HostArr<T>(static_cast<T*>(p));
  }
  // host <-> device through the context's side stager (pinned chunks, never
  // a pageable cudaMemcpyAsync: see staging.cuh)
  void up(DBuf& b, const void* src, std::size_t bytes) {
    void* d = b.get(std::max<std::size_t>(bytes, 1));
    c_->h2d(d, src, bytes, st_, /*side=*/true, /*side_pool=*/true);
  }
  void down(void* h, const void* d, std::size_t bytes) { c_->d2h(h, d, bytes, st_, /*side=*/true, /*side_pool=*/true); }
  std::size_t cells(int k) const { return static_cast<std::size_t>(G_[k].nx) * G_[k].ny * G_[k].nz; }
  const float4* clus_k(int k) const { return static_cast<const float4*>(c_->clus.p) + coff_[k]; }
  const std::uint32_t* ctri_k(int k) const {
    return static_cast<const std::uint32_t*>(c_->clus_tri.p) + coff_[k] * nm::kCluster;
  }
  const float4* tsph_k(int k) const { return static_cast<const float4*>(c_->clus_tsph.p) + coff_[k] * nm::kCluster; }
  int nclus(int k) const { return static_cast<int>(coff_[k + 1] - coff_[k]); }
  bool outside_dop(int k, double x, double y, double z) const {
    const float* dop = reinterpret_cast<const float*>(&hbox_[static_cast<std::size_t>(k) * nm::kDopF4]);
    const float xf = float(x), yf = float(y), zf = float(z);
    for (int d = 0; d < nm::kDopDirs; ++d) {
      const float pr = nm::dop_dir(d, 0) * xf + nm::dop_dir(d, 1) * yf + nm::dop_dir(d, 2) * zf;
      if (pr < dop[2 * d] || pr > dop[2 * d + 1]) return true;
    }
    return false;
  }
  std::uint8_t& child_at(int k, std::size_t row, int fx, int sy, int sz) {
    const std::size_t b = boff_[k] + block_of_[row + fx / S];
    return child_[b * nm::kChildren + (sz * S + sy) * S + fx % S];
  }

  // ---- geometry: per compartment its grid and Morton-ordered clusters ----
  // (grid from the compartment's box, hext_; on the device: centroid Morton
  // keys, a stable per-compartment sort, the cluster and triangle spheres,
  // geometry.cuh)
  void geometry() {
    const int K = K_;
    G_.assign(K, nm::CellGrid{});
    coff_.assign(K + 1, 0);
    for (int k = 0; k < K; ++k) {
      compartment_grid(k);
      G_[k].off = static_cast<std::uint32_t>(total_);
      total_ += cells(k);
      if (total_ > 0xffffffffull) throw Error("certified-cell grids exceed 2^32 cells");
      coff_[k + 1] = coff_[k] + (comp_off_[k + 1] - comp_off_[k] + nm::kCluster - 1) / nm::kCluster;
    }
    // memory budget: per level-1 cell ~13 B of host arrays (certified flag,
    // block and run indices, code) and ~5 B on the device (flag, code), plus
    // up to 64 B of children per uncertified cell. A cell_axis that would need
    // more than kHostBudget of host memory fails here instead of driving the
    // host into the OOM killer (cfg5 at the default axis 120: 18.5M cells).
    constexpr double kHostBudget = 8e9;
    if (double(total_) * 18.0 > kHostBudget)
      throw Error("certified-cell grids of " + std::to_string(total_) + " cells (~" +
                  std::to_string(static_cast<long long>(double(total_) * 18.0 / 1e6)) +
                  " MB) exceed the 8 GB build budget: lower nm_options.cell_axis");
    const std::size_t ncl = coff_[K];
    const std::uint32_t nt = comp_off_[K];
    std::vector<std::uint32_t> coff(2 * (K + 1), 0);  // cluster offsets, then supercluster offsets
    for (int k = 0; k <= K; ++k) coff[k] = static_cast<std::uint32_t>(coff_[k]);
    for (int k = 0; k < K; ++k) coff[K + 1 + k + 1] = coff[K + 1 + k] + (coff[k + 1] - coff[k] + 31) / 32;
    const std::uint32_t nsup = coff[2 * K + 1];
    up(c_->cert_coff, coff.data(), coff.size() * sizeof(std::uint32_t));
    auto* sup = c_->clus_sup.as<float4>(std::max<std::uint32_t>(nsup, 1));
    c_->trace("cells", "geo: coff up");
    auto* clus = c_->clus.as<float4>(std::max<std::size_t>(ncl, 1));
    auto* ctri = c_->clus_tri.as<std::uint32_t>(std::max<std::size_t>(ncl, 1) * nm::kCluster);
    auto* tsph = c_->clus_tsph.as<float4>(std::max<std::size_t>(ncl, 1) * nm::kCluster);
    if (nt) {
      const auto* xyz = static_cast<const double*>(c_->xyz64.p);
      const auto* tri = static_cast<const std::uint32_t*>(c_->tri_idx.p);
      const auto* coffd = static_cast<const std::uint32_t*>(c_->comp_off.p);
      auto* keys = c_->geo_keys.as<unsigned long long>(nt);
      auto* vals = c_->geo_vals.as<std::uint32_t>(nt);
      auto* keys2 = c_->geo_keys2.as<unsigned long long>(nt);
      auto* vals2 = c_->geo_vals2.as<std::uint32_t>(nt);
      c_->trace("cells", "geo: allocs");
      const nm::MortonFrame f{ctr_[0], ctr_[1], ctr_[2], c_->lo[0], c_->lo[1], c_->lo[2], c_->span};
      nm::k_tri_morton<<<grid_for(nt, 256, c_->sm_count * 8), 256, 0, st_>>>(xyz, tri, coffd, K, nt, f, keys, vals);
      int end_bit = 30;
      while ((1 << (end_bit - 30)) < K) ++end_bit;
      std::size_t tmp = 0;
      NM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, vals, vals2, static_cast<int>(nt), 0, end_bit,
                                              st_));
      void* t = c_->cub_tmp2.get(tmp);
      NM_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, keys, keys2, vals, vals2, static_cast<int>(nt), 0, end_bit, st_));
      nm::k_cluster_spheres<<<static_cast<unsigned>((ncl * 32 + 255) / 256), 256, 0, st_>>>(
          xyz, tri, coffd, static_cast<const std::uint32_t*>(c_->cert_coff.p), K, static_cast<std::uint32_t>(ncl),
          ctr_[0], ctr_[1], ctr_[2], vals2, clus, ctri, tsph);
      const auto* coffd2 = static_cast<const std::uint32_t*>(c_->cert_coff.p);
      nm::k_super_spheres<<<static_cast<unsigned>((std::size_t(nsup) * 32 + 255) / 256), 256, 0, st_>>>(
          clus, coffd2, coffd2 + K + 1, K, nsup, sup);
      NM_CUDA(cudaGetLastError());
      c_->trace("cells", "geo: launched");
    }
    lap("setup");
  }

  // compartment k's grid: cubes of edge B = longest box side / cell_axis,
  // one cube of margin around the box
  void compartment_grid(int k) {
    nm::CellGrid g{0.0, 0.0, 0.0, 1.0, 0, 0, 0, 0u, 1.0};
    if (comp_off_[k + 1] > comp_off_[k]) {
      const double* e = hext_.data() + static_cast<std::size_t>(k) * nm::kExtQ;
      const double lo[3] = {e[0], e[1], e[2]}, hi[3] = {e[nm::kDopDirs], e[nm::kDopDirs + 1], e[nm::kDopDirs + 2]};
      const double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
      g.B = std::max(ext / c_->opt.cell_axis, 1e-3);
      int n3[3];
      for (int a = 0; a < 3; ++a) n3[a] = static_cast<int>(std::ceil((hi[a] - lo[a]) / g.B)) + 2;
      g.ox = lo[0] - g.B;
      g.oy = lo[1] - g.B;
      g.oz = lo[2] - g.B;
      g.nx = n3[0];
      g.ny = n3[1];
      g.nz = n3[2];
      g.invB = 1.0 / g.B;
    }
    G_[k] = g;
  }

  void make_slabs() {
    slabs_.clear();
    slab_first_.assign(K_ + 1, 0);
    for (int k = 0; k < K_; ++k) {
      slab_first_[k] = slabs_.size();
      for (int z = 0; z < G_[k].nz; z += kSlab) slabs_.push_back({k, z, std::min(G_[k].nz, z + kSlab)});
    }
    slab_first_[K_] = slabs_.size();
  }
  std::size_t slab_begin(const Slab& sl) const {
    return G_[sl.k].off + static_cast<std::size_t>(sl.z0) * G_[sl.k].ny * G_[sl.k].nx;
  }
  std::size_t slab_end(const Slab& sl) const {
    return G_[sl.k].off + static_cast<std::size_t>(sl.z1) * G_[sl.k].ny * G_[sl.k].nx;
  }

  // ---- certification: level-1 cells, then the children of uncertified cells ----
  void certify() {
    const int K = K_;
    make_slabs();
    auto* cert_d = c_->cell_cert.as<std::uint8_t>(std::max<std::size_t>(total_, 1));
    for (int k = 0; k < K; ++k) {
      if (!cells(k)) continue;
      const std::size_t nbrick =
          static_cast<std::size_t>((G_[k].nx + 3) / 4) * ((G_[k].ny + 3) / 4) * ((G_[k].nz + 1) / 2);
      nm::k_cell_certify<<<static_cast<unsigned>((nbrick * 32 + 255) / 256), 256, 0, st_>>>(
          G_[k], clus_k(k), nclus(k), ctri_k(k), tsph_k(k), static_cast<const double*>(c_->xyz64.p),
          static_cast<const std::uint32_t*>(c_->tri_idx.p), c_->cx, c_->cy, c_->cz, cert_d);
    }
    NM_CUDA(cudaGetLastError());
    cert1_ = uninit<std::uint8_t>(total_);
    prefault(cert1_.get(), total_);  // page faults on all threads while the kernels run
    block_of_ = uninit<std::uint32_t>(total_);
    prefault(reinterpret_cast<std::uint8_t*>(block_of_.get()), total_ * sizeof(std::uint32_t));
    if (total_) NM_CUDA(cudaMemcpyAsync(cert1_.get(), cert_d, total_, cudaMemcpyDeviceToHost, st_));
    NM_CUDA(cudaStreamSynchronize(st_));
    lap("l1");

    // child blocks: the uncertified cells in cell order (count per slab,
    // prefix, fill per slab)
    const std::size_t ns = slabs_.size();
    std::vector<std::size_t> sl_cnt(ns + 1, 0);
    parallel_for(static_cast<int>(ns), [&](int i) {
      std::size_t m = 0;
      for (std::size_t q = slab_begin(slabs_[i]); q < slab_end(slabs_[i]); ++q) m += !cert1_[q];
      sl_cnt[i] = m;
    });
    slab_blk_.assign(ns + 1, 0);  // global first block of each slab
    std::vector<std::size_t>& sl_off = slab_blk_;
    for (std::size_t i = 0; i < ns; ++i) sl_off[i + 1] = sl_off[i] + sl_cnt[i];
    boff_.assign(K + 1, 0);
    for (int k = 0; k <= K; ++k) boff_[k] = sl_off[slab_first_[k]];
    const std::size_t nblk = boff_[K];
    std::vector<std::uint32_t> blk_cells(std::max<std::size_t>(nblk, 1));
    parallel_for(static_cast<int>(ns), [&](int i) {
      const Slab& sl = slabs_[i];
      std::size_t b = sl_off[i];
      for (std::size_t q = slab_begin(sl); q < slab_end(sl); ++q)
        if (!cert1_[q]) {
          block_of_[q] = static_cast<std::uint32_t>(b - boff_[sl.k]);  // local to the compartment
          blk_cells[b++] = static_cast<std::uint32_t>(q - G_[sl.k].off);
        }
    });
    lap("blocks");
    nchild_ = nblk * nm::kChildren;
    child_ = uninit<std::uint8_t>(nchild_);
    if (!nblk) return;
    up(c_->cell_blk, blk_cells.data(), nblk * sizeof(std::uint32_t));
    auto* ch_d = c_->cell_child.as<std::uint8_t>(nchild_);
    child_ev_.assign(K, nullptr);
    for (int k = 0; k < K; ++k) {
      const std::size_t nb = boff_[k + 1] - boff_[k];
      if (!nb) continue;
      nm::k_child_certify<<<static_cast<unsigned>((nb * 64 + 255) / 256), 256, 0, st_>>>(
          G_[k], static_cast<const std::uint32_t*>(c_->cell_blk.p) + boff_[k], nb, clus_k(k), nclus(k), ctri_k(k),
          tsph_k(k), static_cast<const double*>(c_->xyz64.p), static_cast<const std::uint32_t*>(c_->tri_idx.p), c_->cx,
          c_->cy, c_->cz, ch_d + boff_[k] * nm::kChildren);
      NM_CUDA(cudaEventCreateWithFlags(&child_ev_[k], cudaEventDisableTiming));
      NM_CUDA(cudaEventRecord(child_ev_[k], st_));
    }
    NM_CUDA(cudaGetLastError());
    prefault(child_.get(), nchild_);
    run_of_ = uninit<std::int32_t>(total_);
    prefault(reinterpret_cast<std::uint8_t*>(run_of_.get()), total_ * sizeof(std::int32_t));
    lap("l2");
  }

  // children of compartment k, device -> host on a copy stream once its
  // kernel is done (the later compartments' kernels keep running); ready
  // counts the compartments whose children are in
  void copy_children(std::atomic<int>& ready) {
    NM_CUDA(cudaSetDevice(c_->opt.device));
    cudaStream_t cp = nullptr;
    NM_CUDA(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    struct Guard {
      cudaStream_t s;
      ~Guard() { cudaStreamDestroy(s); }
    } guard{cp};
    const auto* ch_d = static_cast<const std::uint8_t*>(c_->cell_child.p);
    for (int k = 0; k < K_; ++k) {
      const std::size_t b0 = boff_[k] * nm::kChildren, bytes = (boff_[k + 1] - boff_[k]) * nm::kChildren;
      if (bytes) {
        NM_CUDA(cudaStreamWaitEvent(cp, child_ev_[k], 0));
        NM_CUDA(cudaMemcpyAsync(child_.get() + b0, ch_d + b0, bytes, cudaMemcpyDeviceToHost, cp));
        NM_CUDA(cudaStreamSynchronize(cp));
      }
      ready.store(k + 1, std::memory_order_release);
    }
  }

  // touch every page of a fresh host array on all threads
  static void prefault(std::uint8_t* p, std::size_t bytes) {
    constexpr std::size_t kChunk = std::size_t(1) << 22;
    parallel_for(static_cast<int>((bytes + kChunk - 1) / kChunk), [&](int i) {
      const std::size_t b = static_cast<std::size_t>(i) * kChunk;
      std::memset(p + b, 0, std::min(kChunk, bytes - b));
    });
  }

  // ---- device path: certification + child blocks, runs, codes ----
  void certify_device() {
    const int K = K_;
    auto* cert_d = c_->cell_cert.as<std::uint8_t>(std::max<std::size_t>(total_, 1));
    up(c_->cell_grids, G_.data(), G_.size() * sizeof(nm::CellGrid));
    // one launch over every compartment's bricks (cells.cuh k_cell_certify_all)
    std::vector<unsigned long long> first(K + 1, 0);
    for (int k = 0; k < K; ++k) {
      const unsigned long long nbrick =
          cells(k) ? static_cast<unsigned long long>((G_[k].nx + 3) / 4) * ((G_[k].ny + 3) / 4) * ((G_[k].nz + 1) / 2) : 0;
      first[k + 1] = first[k] + nbrick;
    }
    up(c_->cert_first, first.data(), first.size() * sizeof(unsigned long long));
    nm::CertifyParams cp = certify_params();
    cp.first = static_cast<const unsigned long long*>(c_->cert_first.p);
    cp.out = cert_d;
    cp.warps = first[K];
    c_->trace("cells", "l1: ups");
    if (cp.warps)
      nm::k_cell_certify_all<<<static_cast<unsigned>((cp.warps * 32 + 255) / 256), 256, 0, st_>>>(cp);
    // child block of every uncertified cell: exclusive scan of the
    // uncertified flags in cell order (= the host path's numbering)
    const std::size_t n = std::max<std::size_t>(total_, 1);
    auto* unc = c_->cell_unc.as<std::uint32_t>(n);
    auto* blk = c_->cell_blkidx.as<std::uint32_t>(n);
    if (total_) {
      nm::k_uncert<<<grid_for(total_, 256, c_->sm_count * 8), 256, 0, st_>>>(cert_d, total_, unc);
      std::size_t tmp = 0;
      NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, unc, blk, static_cast<int>(total_), st_));
      void* t = c_->cub_tmp2.get(tmp);
      NM_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, unc, blk, static_cast<int>(total_), st_));
    }
    NM_CUDA(cudaGetLastError());
    // boff_[k] = blk at the compartment's first cell (gathered on the device,
    // read back in one copy: K + 2 words)
    std::vector<std::uint32_t> hw(K + 2, 0);
    if (total_) {
      auto* w = c_->cell_words.as<std::uint32_t>(K + 2);
      NM_CUDA(cudaMemsetAsync(w, 0, (K + 2) * sizeof(std::uint32_t), st_));
      NM_CUDA(cudaMemcpyAsync(w + K, blk + total_ - 1, 4, cudaMemcpyDeviceToDevice, st_));
      NM_CUDA(cudaMemcpyAsync(w + K + 1, unc + total_ - 1, 4, cudaMemcpyDeviceToDevice, st_));
      for (int k = 0; k < K; ++k)
        if (cells(k)) NM_CUDA(cudaMemcpyAsync(w + k, blk + G_[k].off, 4, cudaMemcpyDeviceToDevice, st_));
      c_->trace("cells", "l1: scan launched");
      down(hw.data(), w, (K + 2) * sizeof(std::uint32_t));
    }
    const std::size_t nblk = total_ ? std::size_t(hw[K]) + hw[K + 1] : 0;
    boff_.assign(K + 1, nblk);
    for (int k = K - 1; k >= 0; --k) boff_[k] = cells(k) ? hw[k] : boff_[k + 1];
    lap("l1");
    nchild_ = nblk * nm::kChildren;
    if (!nblk) return;
    auto* blk_cells = c_->cell_blk.as<std::uint32_t>(nblk);
    nm::k_block_cells<<<grid_for(total_, 256, c_->sm_count * 8), 256, 0, st_>>>(
        cert_d, blk, total_, static_cast<const nm::CellGrid*>(c_->cell_grids.p), K, blk_cells);
    auto* ch_d = c_->cell_child.as<std::uint8_t>(nchild_);
    std::vector<unsigned long long> first2(K + 1, 0);
    for (int k = 0; k <= K; ++k) first2[k] = 2ull * boff_[k];
    up(c_->cert_first2, first2.data(), first2.size() * sizeof(unsigned long long));
    nm::CertifyParams cp2 = certify_params();
    cp2.first = static_cast<const unsigned long long*>(c_->cert_first2.p);
    cp2.cells = blk_cells;
    cp2.out = ch_d;
    cp2.warps = first2[K];
    nm::k_child_certify_all<<<static_cast<unsigned>((cp2.warps * 32 + 255) / 256), 256, 0, st_>>>(cp2);
    NM_CUDA(cudaGetLastError());
    lap("l2");
  }

  nm::CertifyParams certify_params() const {
    nm::CertifyParams p{};
    p.grids = static_cast<const nm::CellGrid*>(c_->cell_grids.p);
    p.K = K_;
    p.coff = static_cast<const std::uint32_t*>(c_->cert_coff.p);
    p.soff = p.coff + K_ + 1;
    p.sup = static_cast<const float4*>(c_->clus_sup.p);
    p.clus = static_cast<const float4*>(c_->clus.p);
    p.clus_tri = static_cast<const std::uint32_t*>(c_->clus_tri.p);
    p.tsph = static_cast<const float4*>(c_->clus_tsph.p);
    p.xyz = static_cast<const double*>(c_->xyz64.p);
    p.tri = static_cast<const std::uint32_t*>(c_->tri_idx.p);
    p.cx = c_->cx;
    p.cy = c_->cy;
    p.cz = c_->cz;
    return p;
  }

  nm::L1Params l1_params(std::size_t max_runs) {
    nm::L1Params p{};
    p.grids = static_cast<const nm::CellGrid*>(c_->cell_grids.p);
    p.K = K_;
    p.row_first = static_cast<const std::uint32_t*>(c_->row_first.p);
    p.cert = static_cast<const std::uint8_t*>(c_->cell_cert.p);
    p.dop4 = static_cast<const float4*>(c_->comp_box.p);
    p.rowruns = c_->l1_rowruns.as<std::uint32_t>(std::max<std::uint32_t>(nrows_, 1));
    p.runfirst = c_->l1_runfirst.as<std::uint32_t>(std::max<std::uint32_t>(nrows_, 1));
    p.cellrun = c_->l1_cellrun.as<std::int32_t>(std::max<std::size_t>(total_, 1));
    p.parent = c_->l1_parent.as<std::uint32_t>(max_runs);
    p.runrow = c_->l1_runrow.as<std::uint32_t>(max_runs);
    p.runx = c_->l1_runx.as<std::uint32_t>(max_runs);
    p.zero = c_->l1_zero.as<std::uint32_t>(max_runs);
    p.rootval = c_->l1_rootval.as<std::int32_t>(max_runs);
    p.cellval = static_cast<std::int32_t*>(c_->cell_val.p);
    p.nruns = c_->l1_nruns.as<std::uint32_t>(1);
    p.rep_cursor = static_cast<unsigned*>(c_->rep_cur.p);
    p.rep_first = static_cast<const unsigned*>(c_->rep_cur.p) + 32;
    p.rep_pts = static_cast<double*>(c_->rep_pts.p);
    p.ctr0 = ctr_[0];
    p.ctr1 = ctr_[1];
    p.ctr2 = ctr_[2];
    p.fill = 0;
    return p;
  }

  nm::RunParams run_params(bool fill) {
    nm::RunParams p{};
    p.grids = static_cast<const nm::CellGrid*>(c_->cell_grids.p);
    p.K = K_;
    p.row_first = static_cast<const std::uint32_t*>(c_->row_first.p);
    p.cert = static_cast<const std::uint8_t*>(c_->cell_cert.p);
    p.blk = static_cast<const std::uint32_t*>(c_->cell_blkidx.p);
    p.child = static_cast<const std::uint8_t*>(c_->cell_child.p);
    p.dop4 = static_cast<const float4*>(c_->comp_box.p);  // the 13-DOP slabs (k_extents_finalize)
    p.ctr0 = ctr_[0];
    p.ctr1 = ctr_[1];
    p.ctr2 = ctr_[2];
    p.cellval = static_cast<std::int32_t*>(c_->cell_val.p);
    p.childval = static_cast<std::int32_t*>(c_->child_val.p);
    p.rep_cursor = static_cast<unsigned*>(c_->rep_cur.p);
    p.rep_first = static_cast<const unsigned*>(c_->rep_cur.p) + 32;
    p.rep_pts = static_cast<double*>(c_->rep_pts.p);
    p.fill = fill ? 1 : 0;
    return p;
  }

  void runs_device() {
    const int K = K_;
    std::vector<std::uint32_t> rf(K + 1, 0);
    for (int k = 0; k < K; ++k) rf[k + 1] = rf[k] + (cells(k) ? static_cast<std::uint32_t>(G_[k].ny * G_[k].nz) : 0u);
    nrows_ = rf[K];
    up(c_->row_first, rf.data(), rf.size() * sizeof(std::uint32_t));
    c_->trace("cells", "runs: row_first up");
    (void)c_->cell_val.as<std::int32_t>(std::max<std::size_t>(total_, 1));
    (void)c_->child_val.as<std::int32_t>(std::max<std::size_t>(nchild_, 1));
    c_->trace("cells", "runs: val allocs");
    auto* cur = c_->rep_cur.as<unsigned>(64);  // [0, 32) cursors, [32, 64) slot bases
    (void)c_->rep_pts.as<double>(3);
    NM_CUDA(cudaMemsetAsync(cur, 0, 64 * sizeof(unsigned), st_));
    c_->trace("cells", "runs: memset");
    if (!nrows_) {
      rep_cnt_d_.assign(K, 0);
      rep_first_d_.assign(K + 1, 0);
      nreps_ = 0;
      return;
    }
    // level-1 runs -> components (cells.cuh k_l1_*): numbered, united, one
    // representative per component; per-run arrays sized for the most runs a
    // row can hold (no host synchronisation before the counts below)
    std::size_t max_runs = 0;
    for (int k = 0; k < K; ++k)
      if (cells(k)) max_runs += static_cast<std::size_t>(G_[k].ny) * G_[k].nz * ((G_[k].nx + 1) / 2);
    nm::L1Params lp = l1_params(std::max<std::size_t>(max_runs, 1));
    const unsigned gr = grid_for(nrows_, 128, c_->sm_count * 16), grr = grid_for(max_runs, 256, c_->sm_count * 16);
    nm::k_l1_count<<<gr, 128, 0, st_>>>(lp, nrows_);
    {
      std::size_t tmp = 0;
      NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, lp.rowruns, const_cast<std::uint32_t*>(lp.runfirst),
                                            static_cast<int>(nrows_), st_));
      void* t = c_->cub_tmp2.get(tmp);
      NM_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, lp.rowruns, const_cast<std::uint32_t*>(lp.runfirst),
                                            static_cast<int>(nrows_), st_));
    }
    nm::k_l1_total<<<1, 1, 0, st_>>>(lp, nrows_);
    nm::k_l1_label<<<gr, 128, 0, st_>>>(lp, nrows_);
    nm::k_l1_union<<<gr, 128, 0, st_>>>(lp, nrows_);
    nm::k_l1_flatten<<<grr, 256, 0, st_>>>(lp);
    nm::k_l1_zero<<<grr, 256, 0, st_>>>(lp);
    // count pass: representatives per compartment (components, fine runs)
    nm::k_l1_roots<<<grr, 256, 0, st_>>>(lp);
    nm::k_runs_fine<<<grid_for(std::size_t(nrows_) * 16, 128, c_->sm_count * 16), 128, 0, st_>>>(run_params(false),
                                                                                                   nrows_);
    NM_CUDA(cudaGetLastError());
    rep_cnt_d_.assign(K, 0);
    c_->trace("cells", "runs: count launched");
    down(rep_cnt_d_.data(), cur, K * sizeof(unsigned));
    c_->trace("cells", "runs: counts read");
    rep_first_d_.assign(K + 1, 0);
    for (int k = 0; k < K; ++k) rep_first_d_[k + 1] = rep_first_d_[k] + rep_cnt_d_[k];
    nreps_ = rep_first_d_[K];
    auto* pts = c_->rep_pts.as<double>(3 * std::max<std::size_t>(nreps_, 1));
    (void)pts;
    cur = static_cast<unsigned*>(c_->rep_cur.p);
    NM_CUDA(cudaMemsetAsync(cur, 0, 32 * sizeof(unsigned), st_));
    c_->h2d(cur + 32, rep_first_d_.data(), K * sizeof(unsigned), st_, /*side=*/true, /*side_pool=*/true);
    NM_CUDA(cudaMemsetAsync(c_->cell_val.p, 0xff, std::max<std::size_t>(total_, 1) * sizeof(std::int32_t), st_));
    if (nchild_) NM_CUDA(cudaMemsetAsync(c_->child_val.p, 0xff, nchild_ * sizeof(std::int32_t), st_));
    // fill pass: values, representative points (level-1 values first: the
    // fine runs copy their neighbour parents')
    lp = l1_params(std::max<std::size_t>(max_runs, 1));
    lp.fill = 1;
    nm::k_l1_roots<<<grr, 256, 0, st_>>>(lp);
    nm::k_l1_cellval<<<gr, 128, 0, st_>>>(lp, nrows_);
    nm::k_runs_fine<<<grid_for(std::size_t(nrows_) * 16, 128, c_->sm_count * 16), 128, 0, st_>>>(run_params(true),
                                                                                                   nrows_);
    NM_CUDA(cudaGetLastError());
    lap("runs");
  }

  void resolve_device() {
    const int K = K_;
    const std::size_t R = nreps_;
    auto* rep_w = c_->rep_w.as<std::int32_t>(std::max<std::size_t>(R, 1));
    if (R) {
      evaluate_reps_device(R);
      auto* s_dev = static_cast<const double*>(c_->rep_s.p);
      nm::k_rep_values<<<grid_for(R, 256, c_->sm_count * 4), 256, 0, st_>>>(
          s_dev, static_cast<std::uint32_t>(R), K, static_cast<const unsigned*>(c_->rep_cur.p) + 32, rep_w);
    }
    lap("reps");
    auto* cnt = c_->cell_cnt.as<unsigned long long>(1);
    NM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st_));
    auto* state_d = c_->cell_state.as<std::uint32_t>(std::max<std::size_t>(total_, 1));
    if (total_)
      nm::k_cell_codes<<<grid_for(total_, 256, c_->sm_count * 8), 256, 0, st_>>>(
          total_, static_cast<const std::uint8_t*>(c_->cell_cert.p), static_cast<const std::uint32_t*>(c_->cell_blkidx.p),
          static_cast<const std::int32_t*>(c_->cell_val.p), rep_w, state_d, cnt);
    (void)c_->cell_child.get(std::max<std::size_t>(nchild_, 1));
    if (nchild_)
      nm::k_child_codes<<<grid_for(nchild_, 256, c_->sm_count * 8), 256, 0, st_>>>(
          nchild_, static_cast<std::uint8_t*>(c_->cell_child.p), static_cast<const std::int32_t*>(c_->child_val.p), rep_w,
          cnt);
    NM_CUDA(cudaGetLastError());
    unsigned long long ncert = 0;
    down(&ncert, cnt, sizeof ncert);
    lap("codes");
    c_->cells_total = total_ + nchild_;
    c_->cells_l1 = total_;
    c_->cells_children = nchild_;
    c_->cells_certified = ncert;
    c_->cell_reps = nreps_;
    c_->cells = true;
    c_->ms_cells = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
  }

  // ---- runs: every maximal x-run of certified cells gets one winding number ----
  // per-slab results, merged per compartment in slab order
  struct SlabRuns {
    std::vector<double> reps;
    std::vector<std::int64_t> run_val;
    std::vector<FineRun> fine;
  };

  void runs() {
    const std::size_t ns = slabs_.size();
    std::vector<SlabRuns> part(ns);
    if (!run_of_) run_of_ = uninit<std::int32_t>(total_);
    // slabs are handed out in compartment order: each waits only for its own
    // compartment's children
    std::atomic<int> ready{nchild_ ? 0 : K_};
    std::exception_ptr copy_err;
    std::thread copier;
    if (nchild_)
      copier = std::thread([&] {
        try {
          copy_children(ready);
        } catch (...) {
          copy_err = std::current_exception();
          ready.store(K_, std::memory_order_release);
        }
      });
    parallel_for(static_cast<int>(ns), [&](int i) {
      while (ready.load(std::memory_order_acquire) <= slabs_[i].k) std::this_thread::yield();
      slab_runs(slabs_[i], part[i]);
    });
    if (copier.joinable()) copier.join();
    for (cudaEvent_t e : child_ev_)
      if (e) cudaEventDestroy(e);
    child_ev_.clear();
    if (copy_err) std::rethrow_exception(copy_err);
    lap("slabs");
    // merge: slab-local run / representative indices -> compartment-local
    std::vector<std::size_t> run_base(ns), rep_base(ns);
    fine_.assign(ns, {});
    for (int k = 0; k < K_; ++k) {
      std::size_t nr = 0, np = 0;
      for (std::size_t i = slab_first_[k]; i < slab_first_[k + 1]; ++i) {
        run_base[i] = nr;
        rep_base[i] = np;
        nr += part[i].run_val.size();
        np += part[i].reps.size() / 3;
      }
    }
    auto rebase = [&](std::int64_t v, std::size_t i) -> std::int64_t {
      if (v >= kCell) return v;  // resolved below, once every slab's runs are rebased
      if (v >= kRun) return v + static_cast<std::int64_t>(run_base[i]);
      if (v >= kRep) return v + static_cast<std::int64_t>(rep_base[i]);
      return v;
    };
    parallel_for(static_cast<int>(ns), [&](int i) {
      const Slab& sl = slabs_[i];
      for (std::size_t q = slab_begin(sl); q < slab_end(sl); ++q)
        if (cert1_[q]) run_of_[q] += static_cast<std::int32_t>(run_base[i]);
      for (std::int64_t& v : part[i].run_val) v = rebase(v, i);
      for (FineRun& fr : part[i].fine) fr.v = rebase(fr.v, i);
      fine_[i] = std::move(part[i].fine);  // fine runs stay per slab (no copy)
    });
    parallel_for(static_cast<int>(ns), [&](int i) {
      for (FineRun& fr : fine_[i])
        if (fr.v >= kCell) fr.v = kRun + run_of_[static_cast<std::size_t>(fr.v - kCell)];
    });
    reps_.assign(K_, {});
    run_val_.assign(K_, {});
    parallel_for(K_, [&](int k) {
      for (std::size_t i = slab_first_[k]; i < slab_first_[k + 1]; ++i) {
        reps_[k].insert(reps_[k].end(), part[i].reps.begin(), part[i].reps.end());
        run_val_[k].insert(run_val_[k].end(), part[i].run_val.begin(), part[i].run_val.end());
      }
      components(k);
    });
    lap("merge");
  }

  // Level-1 runs of compartment k joined into components (the rule of
  // cells.cuh k_l1_*): runs touching through a face in the rows y + 1 / z + 1
  // share their winding number; a component with a 0 run is 0, any other
  // keeps only its smallest run's representative. Representatives no run
  // refers to any more are dropped (the fine runs keep theirs).
  void components(int k) {
    const nm::CellGrid& g = G_[k];
    std::vector<std::int64_t>& rv = run_val_[k];
    const std::size_t R = rv.size();
    if (!R) return;
    std::vector<std::uint32_t> par(R);
    std::iota(par.begin(), par.end(), 0u);
    auto find = [&](std::uint32_t x) {
      while (par[x] != x) x = par[x] = par[par[x]];
      return x;
    };
    for (int iz = 0; iz < g.nz; ++iz)
      for (int iy = 0; iy < g.ny; ++iy)
        for (int ix = 0; ix < g.nx; ++ix) {
          const std::size_t q = g.off + (static_cast<std::size_t>(iz) * g.ny + iy) * g.nx + ix;
          if (!cert1_[q]) continue;
          const std::size_t nb[2] = {iy + 1 < g.ny ? q + g.nx : 0, iz + 1 < g.nz ? q + std::size_t(g.nx) * g.ny : 0};
          for (std::size_t n : nb) {
            if (!n || !cert1_[n]) continue;
            std::uint32_t a = find(static_cast<std::uint32_t>(run_of_[q])), b = find(static_cast<std::uint32_t>(run_of_[n]));
            if (a != b) par[std::max(a, b)] = std::min(a, b);  // the root is the component's smallest run
          }
        }
    std::vector<std::uint8_t> zero(R, 0);
    for (std::uint32_t r = 0; r < R; ++r)
      if (rv[r] == 0) zero[find(r)] = 1;
    for (std::uint32_t r = 0; r < R; ++r) {
      const std::uint32_t root = find(r);
      rv[r] = zero[root] ? 0 : rv[root];  // the root's representative (kRep + index)
    }
    // compact the representatives: those of the component roots and of the
    // fine runs, in their old order
    const std::size_t np = reps_[k].size() / 3;
    std::vector<std::int64_t> remap(np, -1);
    for (std::int64_t v : rv)
      if (v >= kRep && v < kRun) remap[static_cast<std::size_t>(v - kRep)] = 0;
    for (std::size_t i = slab_first_[k]; i < slab_first_[k + 1]; ++i)
      for (const FineRun& fr : fine_[i])
        if (fr.v >= kRep && fr.v < kRun) remap[static_cast<std::size_t>(fr.v - kRep)] = 0;
    std::vector<double> kept;
    for (std::size_t j = 0; j < np; ++j)
      if (remap[j] == 0) {
        remap[j] = static_cast<std::int64_t>(kept.size() / 3);
        kept.insert(kept.end(), reps_[k].begin() + 3 * j, reps_[k].begin() + 3 * j + 3);
      }
    reps_[k] = std::move(kept);
    for (std::int64_t& v : rv)
      if (v >= kRep && v < kRun) v = kRep + remap[static_cast<std::size_t>(v - kRep)];
    for (std::size_t i = slab_first_[k]; i < slab_first_[k + 1]; ++i)
      for (FineRun& fr : fine_[i])
        if (fr.v >= kRep && fr.v < kRun) fr.v = kRep + remap[static_cast<std::size_t>(fr.v - kRep)];
  }

  std::int64_t new_rep(SlabRuns& out, double x, double y, double z) {
    const std::int64_t v = kRep + static_cast<std::int64_t>(out.reps.size() / 3);
    out.reps.insert(out.reps.end(), {x + ctr_[0], y + ctr_[1], z + ctr_[2]});
    return v;
  }

  void slab_runs(const Slab& sl, SlabRuns& out) {
    const int k = sl.k;
    const nm::CellGrid& g = G_[k];
    for (int iz = sl.z0; iz < sl.z1; ++iz)
      for (int iy = 0; iy < g.ny; ++iy) {
        const std::size_t row = g.off + (static_cast<std::size_t>(iz) * g.ny + iy) * g.nx;
        const double y = g.oy + (iy + 0.5) * g.B, z = g.oz + (iz + 0.5) * g.B;
        for (int ix = 0; ix < g.nx;) {
          const bool c1 = cert1_[row + ix];
          int jx = ix;
          while (jx + 1 < g.nx && bool(cert1_[row + jx + 1]) == c1) ++jx;
          if (c1) {
            // level-1 run [ix, jx]: grid edge or an end outside the 13-DOP -> 0
            std::int64_t v;
            if (ix == 0 || jx == g.nx - 1 || outside_dop(k, g.ox + (ix + 0.5) * g.B, y, z) ||
                outside_dop(k, g.ox + (jx + 0.5) * g.B, y, z))
              v = 0;
            else
              v = new_rep(out, g.ox + ((ix + jx) / 2 + 0.5) * g.B, y, z);
            for (int q = ix; q <= jx; ++q) run_of_[row + q] = static_cast<std::int32_t>(out.run_val.size());
            out.run_val.push_back(v);
          } else {
            segment_runs(out, k, g, row, ix, jx, iy, iz);
          }
          ix = jx + 1;
        }
      }
    // neighbour references: the level-1 runs of the slab's rows exist now
    // (slab-local indices, rebased with the slab's runs)
    for (FineRun& fr : out.fine) {
      if (fr.v == kLeft) fr.v = kRun + run_of_[fr.row + fr.fx0 / S - 1];
      else if (fr.v == kRight) fr.v = kRun + run_of_[fr.row + fr.fx1 / S + 1];
    }
  }

  // segment [ix, jx] of uncertified level-1 cells: runs of certified children
  // per (sy, sz) sub-row; a run reaching the segment's end continues into the
  // certified neighbour parent (or the grid edge)
  void segment_runs(SlabRuns& out, int k, const nm::CellGrid& g, std::size_t row, int ix, int jx, int iy, int iz) {
    const double b = g.B / S;
    const int f_lo = S * ix, f_hi = S * jx + S - 1;
    for (int sz = 0; sz < S; ++sz)
      for (int sy = 0; sy < S; ++sy)
        for (int f = f_lo; f <= f_hi;) {
          if (!child_at(k, row, f, sy, sz)) {
            ++f;
            continue;
          }
          int e = f;
          while (e + 1 <= f_hi && child_at(k, row, e + 1, sy, sz)) ++e;
          std::int64_t v;
          if (f == f_lo) {
            v = ix == 0 ? 0 : kLeft;
          } else if (e == f_hi) {
            v = jx == g.nx - 1 ? 0 : kRight;
          } else {
            const double yy = g.oy + iy * g.B + (sy + 0.5) * b, zz = g.oz + iz * g.B + (sz + 0.5) * b;
            if (outside_dop(k, g.ox + (f + 0.5) * b, yy, zz) || outside_dop(k, g.ox + (e + 0.5) * b, yy, zz)) {
              v = 0;
            } else {
              // a certified parent beyond a y / z face (cells.cuh fine_face_neighbour)
              const std::size_t nb = nm::fine_face_neighbour(cert1_.get(), g, row, iy, iz, sy, sz, f / S, e / S);
              v = nb != nm::kNoCell ? kCell + static_cast<std::int64_t>(nb) : new_rep(out, g.ox + ((f + e) / 2 + 0.5) * b, yy, zz);
            }
          }
          out.fine.push_back({row, f, e, sy, sz, v});
          f = e + 1;
        }
  }

  // ---- resolve: representatives evaluated, final codes uploaded ----
  void resolve() {
    const int K = K_;
    std::vector<std::uint32_t> rep_cnt(K, 0), rep_first(K + 1, 0);
    std::vector<double> rep_all;
    for (int k = 0; k < K; ++k) {  // compartment k's representatives are contiguous
      rep_first[k] = static_cast<std::uint32_t>(rep_all.size() / 3);
      rep_cnt[k] = static_cast<std::uint32_t>(reps_[k].size() / 3);
      rep_all.insert(rep_all.end(), reps_[k].begin(), reps_[k].end());
    }
    nreps_ = rep_all.size() / 3;
    rep_first[K] = static_cast<std::uint32_t>(nreps_);
    const std::vector<double> rep_w = evaluate_reps(rep_all, rep_cnt, rep_first);
    lap("reps");
    auto code = uninit<std::uint32_t>(total_);
    auto value = [&](int k, std::int64_t v) -> std::int64_t {  // -> 0, 1 or kUnknown
      if (v >= kRun) v = run_val_[k][static_cast<std::size_t>(v - kRun)];
      if (v >= kRep) {
        const double w = rep_w[rep_first[k] + static_cast<std::size_t>(v - kRep)];
        return w < 0.0 ? kUnknown : static_cast<std::int64_t>(w);
      }
      return v;
    };
    // per slab: level-1 codes, its child blocks zeroed and written by its fine
    // runs, both uploaded right away (other slabs are still being coded) and
    // the certified cells counted
    auto* state_d = c_->cell_state.as<std::uint32_t>(std::max<std::size_t>(total_, 1));
    auto* child_d = static_cast<std::uint8_t*>(c_->cell_child.get(std::max<std::size_t>(nchild_, 1)));
    std::vector<std::size_t> ncert(slabs_.size(), 0);
    std::vector<cudaError_t> cp_err(slabs_.size(), cudaSuccess);
    parallel_for(static_cast<int>(slabs_.size()), [&](int i) {
      cp_err[i] = cudaSetDevice(c_->opt.device);  // (f must not throw: errors are collected)
      const Slab& sl = slabs_[i];
      const int k = sl.k;
      for (std::size_t q = slab_begin(sl); q < slab_end(sl); ++q) {
        if (!cert1_[q]) {
          code[q] = 3u + static_cast<std::uint32_t>(boff_[k] + block_of_[q]);
          std::fill(child_.get() + (boff_[k] + block_of_[q]) * nm::kChildren,
                    child_.get() + (boff_[k] + block_of_[q] + 1) * nm::kChildren, 0);
        } else {
          const std::int64_t w = value(k, run_val_[k][run_of_[q]]);
          code[q] = w == kUnknown ? 0u : static_cast<std::uint32_t>(1 + w);
        }
      }
      // the slab's fine runs write children of the slab's own cells
      for (const FineRun& fr : fine_[i]) {
        const std::int64_t w = value(k, fr.v);
        if (w == kUnknown) continue;
        for (int f = fr.fx0; f <= fr.fx1; ++f) child_at(k, fr.row, f, fr.sy, fr.sz) = static_cast<std::uint8_t>(1 + w);
      }
      const std::size_t q0 = slab_begin(sl), q1 = slab_end(sl);
      const std::size_t c0 = nchild_ ? slab_blk_[i] * nm::kChildren : 0, c1 = nchild_ ? slab_blk_[i + 1] * nm::kChildren : 0;
      if (q1 > q0 && cp_err[i] == cudaSuccess)
        cp_err[i] = cudaMemcpyAsync(state_d + q0, code.get() + q0, (q1 - q0) * sizeof(std::uint32_t),
                                    cudaMemcpyHostToDevice, st_);
      if (c1 > c0 && cp_err[i] == cudaSuccess)
        cp_err[i] = cudaMemcpyAsync(child_d + c0, child_.get() + c0, c1 - c0, cudaMemcpyHostToDevice, st_);
      std::size_t m = 0;
      for (std::size_t q = q0; q < q1; ++q) m += code[q] == 1 || code[q] == 2;
      for (std::size_t q = c0; q < c1; ++q) m += child_[q] != 0;
      ncert[i] = m;
    });
    for (cudaError_t e : cp_err) NM_CUDA(e);
    lap("codes");
    up(c_->cell_grids, G_.data(), G_.size() * sizeof(nm::CellGrid));
    NM_CUDA(cudaStreamSynchronize(st_));
    lap("final");
    c_->cells_total = total_ + nchild_;
    c_->cells_l1 = total_;
    c_->cells_children = nchild_;
    c_->cells_certified = std::accumulate(ncert.begin(), ncert.end(), std::size_t(0));
    c_->cell_reps = nreps_;
    c_->cells = true;
    c_->ms_cells = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
  }

  // device path: the representatives are already in c_->rep_pts (grouped by
  // compartment, rep_first_d_); s of each against its own compartment lands
  // in c_->rep_s (k_rep_values turns it into w)
  void evaluate_reps_device(std::size_t R) {
    const int K = K_;
    auto* s_dev = c_->rep_s.as<double>(R * K);
    auto* m_dev = c_->rep_m.as<std::uint32_t>(R);
    auto* f_dev = c_->rep_f.as<std::uint32_t>(R);
    auto* list = c_->sp_list.as<std::uint32_t>(R);
    nm::k_iota<<<grid_for(R, 256, c_->sm_count * 4), 256, 0, st_>>>(list, R);
    NM_CUDA(cudaMemsetAsync(m_dev, 0, R * sizeof(std::uint32_t), st_));
    NM_CUDA(cudaMemsetAsync(f_dev, 0, R * sizeof(std::uint32_t), st_));
    nm::LabelParams prm{};
    prm.pts = static_cast<const double*>(c_->rep_pts.p);
    prm.n = R;
    prm.order = nullptr;
    prm.n_pts = R;
    prm.n_tiles = c_->comp_tiles_h.empty() ? 0u : c_->comp_tiles_h.back();
    prm.tri = static_cast<const float4*>(c_->tri.p);
    prm.sub = static_cast<const float4*>(c_->sub.p);
    prm.cont = static_cast<const std::uint32_t*>(c_->cont.p);
    prm.comp_tiles = static_cast<const std::uint32_t*>(c_->comp_tiles.p);
    prm.K = K;
    prm.cx = c_->cx;
    prm.cy = c_->cy;
    prm.cz = c_->cz;
    prm.T = 0.5;
    prm.band = c_->opt.band;
    prm.tau = c_->opt.tau;
    prm.delta = c_->opt.delta_mm;
    prm.masks = m_dev;
    prm.flagmask = f_dev;
    prm.s_out = s_dev;
    prm.sp_list = list;
    std::vector<std::uint32_t> cnt(rep_cnt_d_.begin(), rep_cnt_d_.end());
    launch_sparse(c_, prm, cnt, st_);
  }

  // s at every representative (sparse k_label against its own compartment);
  // w = round(s) when within 1e-3 of 0 or 1, else -1 (the run stays unresolved)
  std::vector<double> evaluate_reps(const std::vector<double>& rep_all, const std::vector<std::uint32_t>& rep_cnt,
                                    const std::vector<std::uint32_t>& rep_first) {
    const int K = K_;
    const std::size_t R = nreps_;
    std::vector<double> rep_w(R, -1.0);
    if (!R) return rep_w;
    up(c_->rep_pts, rep_all.data(), rep_all.size() * sizeof(double));
    auto* s_dev = c_->rep_s.as<double>(R * K);
    auto* m_dev = c_->rep_m.as<std::uint32_t>(R);
    auto* f_dev = c_->rep_f.as<std::uint32_t>(R);
    std::vector<std::uint32_t> iota(R);
    std::iota(iota.begin(), iota.end(), 0u);
    up(c_->sp_list, iota.data(), R * sizeof(std::uint32_t));
    NM_CUDA(cudaMemsetAsync(m_dev, 0, R * sizeof(std::uint32_t), st_));
    NM_CUDA(cudaMemsetAsync(f_dev, 0, R * sizeof(std::uint32_t), st_));
    nm::LabelParams prm{};
    prm.pts = static_cast<const double*>(c_->rep_pts.p);
    prm.n = R;
    prm.order = nullptr;
    prm.n_pts = R;
    prm.n_tiles = c_->comp_tiles_h.empty() ? 0u : c_->comp_tiles_h.back();
    prm.tri = static_cast<const float4*>(c_->tri.p);
    prm.sub = static_cast<const float4*>(c_->sub.p);
    prm.cont = static_cast<const std::uint32_t*>(c_->cont.p);
    prm.comp_tiles = static_cast<const std::uint32_t*>(c_->comp_tiles.p);
    prm.K = K;
    prm.cx = c_->cx;
    prm.cy = c_->cy;
    prm.cz = c_->cz;
    prm.T = 0.5;
    prm.band = c_->opt.band;
    prm.tau = c_->opt.tau;
    prm.delta = c_->opt.delta_mm;
    prm.masks = m_dev;
    prm.flagmask = f_dev;
    prm.s_out = s_dev;
    prm.sp_list = static_cast<const std::uint32_t*>(c_->sp_list.p);
    launch_sparse(c_, prm, rep_cnt, st_);
    std::vector<double> s(R * K);
    NM_CUDA(cudaMemcpyAsync(s.data(), s_dev, R * K * sizeof(double), cudaMemcpyDeviceToHost, st_));
    NM_CUDA(cudaStreamSynchronize(st_));
    for (int k = 0; k < K; ++k)
      for (std::uint32_t r = rep_first[k]; r < rep_first[k + 1]; ++r) {
        const double v = s[static_cast<std::size_t>(r) * K + k];
        const double w = std::round(v);
        if (std::fabs(v - w) < 1e-3 && (w == 0.0 || w == 1.0)) rep_w[r] = w;
      }
    return rep_w;
  }
};

std::unique_ptr<CellBuilder> make_cell_builder(nm_ctx* c, const double* xyz, const std::uint32_t* tri,
                                               const std::uint32_t* comp_off, const std::vector<float4>& hbox,
                                               const std::vector<double>& hext, cudaStream_t st,
                                               std::shared_future<void> dop_ready) {
  return std::make_unique<CellBuild>(c, xyz, tri, comp_off, hbox, hext, st, std::move(dop_ready));
}

}  // namespace nmh
