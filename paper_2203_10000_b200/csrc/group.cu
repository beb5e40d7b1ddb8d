// Single-process multi-GPU group API (nm_group_*).
#include "context.cuh"

using namespace nmh;

// Single-process multi-GPU group (for C/C++ hosts without torch): one nm_ctx
// per device, contiguous node and tet shards, node masks gathered through a
// pinned host buffer. Results are bit-identical to one device (node masks are
// pure functions of position).
struct nm_group {
  std::vector<nm_ctx*> ctx;
  std::uint32_t* h_masks = nullptr;  // pinned gather buffer
  std::size_t h_cap = 0;
  std::uint32_t* h_part = nullptr;   // pinned per-device partial masks (certified-cell sharding)
  std::size_t part_cap = 0;
  ~nm_group() {
    for (nm_ctx* c : ctx) nm_destroy(c);
    if (h_masks) cudaFreeHost(h_masks);
    if (h_part) cudaFreeHost(h_part);
  }
};

extern "C" {

int nm_group_create(nm_group** out, int n, const int* devices, const nm_options* opt) {
  return guarded([&] {
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    if (n < 1) throw Error("group needs at least one device");
    std::unique_ptr<nm_group> g(new nm_group);
    for (int r = 0; r < n; ++r) {
      nm_options o;
      if (opt) o = *opt;
      else nm_default_options(&o);
      o.device = devices ? devices[r] : r;
      nm_ctx* c = nullptr;
      if (nm_create(&c, &o) != 0) throw Error(last_error());
      g->ctx.push_back(c);
    }
    *out = g.release();
  });
}

int nm_group_destroy(nm_group* g) {
  return guarded([&] { delete g; });
}

int nm_group_size(const nm_group* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

int nm_group_set_surfaces(nm_group* g, const double* xyz, std::size_t nv, const std::uint32_t* tri, std::size_t nt,
                          const std::uint32_t* comp_off, int K, const int* label_ids) {
  return guarded([&] {
    if (!g) throw Error("null group");
    for (nm_ctx* c : g->ctx)
      if (nm_set_surfaces(c, xyz, nv, tri, nt, comp_off, K, label_ids) != 0) throw Error(last_error());
  });
}

int nm_group_label_mesh(nm_group* g, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt,
                        double T, int* labels_out, std::uint32_t* masks_out, nm_stats* stats) {
  return guarded([&] {
    if (!g) throw Error("null group");
    check_tets(tets, nt, n);
    const std::size_t R = g->ctx.size();
    const std::size_t per_n = (n + R - 1) / R, per_t = (nt + R - 1) / R;
    if (stats) std::memset(stats, 0, sizeof *stats);
    if (g->h_cap < n) {
      if (g->h_masks) cudaFreeHost(g->h_masks);
      g->h_masks = nullptr;
      g->h_cap = 0;
      NM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->h_masks), std::max<std::size_t>(n, 1) * 4, cudaHostAllocPortable));
      g->h_cap = n;
    }
    // 1) node pass. With certified cells the work per point is far from
    // uniform (only pairs near a surface are evaluated), so every device
    // takes a cost-balanced share of the pair lists of ALL points and the
    // disjoint partial masks are OR-ed; otherwise contiguous node shards.
    const bool by_pairs = R > 1 && g->ctx[0]->opt.cull_outside == 2 && g->ctx[0]->cells;
    if (by_pairs && g->part_cap < R * n) {
      if (g->h_part) cudaFreeHost(g->h_part);
      g->h_part = nullptr;
      g->part_cap = 0;
      NM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->h_part), std::max<std::size_t>(R * n, 1) * 4,
                            cudaHostAllocPortable));
      g->part_cap = R * n;
    }
    for (std::size_t r = 0; by_pairs && r < R; ++r) {
      nm_ctx* c = g->ctx[r];
      require_surfaces(c);
      NM_CUDA(cudaSetDevice(c->opt.device));
      auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
      auto* d_m = c->masks2.as<std::uint32_t>(std::max<std::size_t>(n, 1));
      if (n) {
        NM_CUDA(cudaMemcpyAsync(d_pts, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        label_nodes_dev(c, d_pts, n, T, d_m, nullptr, c->stream, nullptr, nullptr, false, static_cast<int>(r),
                        static_cast<int>(R));
        NM_CUDA(cudaMemcpyAsync(g->h_part + r * n, d_m, n * 4, cudaMemcpyDeviceToHost, c->stream));
      }
    }
    for (std::size_t r = 0; !by_pairs && r < R; ++r) {
      nm_ctx* c = g->ctx[r];
      require_surfaces(c);
      NM_CUDA(cudaSetDevice(c->opt.device));
      const std::size_t lo = std::min(n, r * per_n), hi = std::min(n, lo + per_n);
      auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(hi - lo, 1));
      auto* d_m = c->masks2.as<std::uint32_t>(std::max<std::size_t>(hi - lo, 1));
      if (hi > lo) {
        NM_CUDA(cudaMemcpyAsync(d_pts, nodes + 3 * lo, 3 * (hi - lo) * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        label_nodes_dev(c, d_pts, hi - lo, T, d_m, nullptr, c->stream, nullptr);
        NM_CUDA(cudaMemcpyAsync(g->h_masks + lo, d_m, (hi - lo) * 4, cudaMemcpyDeviceToHost, c->stream));
      }
    }
    for (nm_ctx* c : g->ctx) {
      NM_CUDA(cudaSetDevice(c->opt.device));
      NM_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (by_pairs) {
      const int nchunk = 64;
      parallel_for(nchunk, [&](int q) {
        const std::size_t lo = n * q / nchunk, hi = n * (q + 1) / nchunk;
        for (std::size_t i = lo; i < hi; ++i) {
          std::uint32_t m = 0;
          for (std::size_t r = 0; r < R; ++r) m |= g->h_part[r * n + i];
          g->h_masks[i] = m;
        }
      });
    }
    // 2) gathered masks to every device, tet shards
    for (std::size_t r = 0; r < R; ++r) {
      nm_ctx* c = g->ctx[r];
      NM_CUDA(cudaSetDevice(c->opt.device));
      const std::size_t lo = std::min(nt, r * per_t), hi = std::min(nt, lo + per_t);
      auto* d_m = c->masks.as<std::uint32_t>(std::max<std::size_t>(n, 1));
      auto* d_t = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(hi - lo, 1));
      auto* d_l = c->labels.as<int>(std::max<std::size_t>(hi - lo, 1));
      if (n) NM_CUDA(cudaMemcpyAsync(d_m, g->h_masks, n * 4, cudaMemcpyHostToDevice, c->stream));
      if (hi > lo) {
        NM_CUDA(cudaMemcpyAsync(d_t, tets + 4 * lo, 4 * (hi - lo) * sizeof(std::uint32_t), cudaMemcpyHostToDevice,
                                c->stream));
        label_tets_dev(c, d_t, hi - lo, d_m, d_l, c->stream, nullptr);
        NM_CUDA(cudaMemcpyAsync(labels_out + lo, d_l, (hi - lo) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      }
    }
    for (nm_ctx* c : g->ctx) {
      NM_CUDA(cudaSetDevice(c->opt.device));
      NM_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (masks_out && n) std::memcpy(masks_out, g->h_masks, n * 4);
    if (stats) {
      stats->points = n;
      stats->triangles = g->ctx[0]->nt_real;
      stats->evals = static_cast<std::uint64_t>(n) * g->ctx[0]->nt_real;
    }
  });
}

}  // extern "C"
