// Single-process multi-GPU group API (nm_group_*): the C/C++ hosts' path of
// SPEC.md:265-267 (--label-workers; results independent of the worker count).
//
// One nm_ctx per device. Every device's share runs on its own host thread, so
// the devices' node passes (which synchronise their host thread for the fix-up
// pair lists and the certified-cell grid) overlap. The exchange stays on the
// devices:
//   * distinct devices: NCCL over NVLink/NVSwitch (ncclCommInitAll; the
//     library is opened at run time, so a host without NCCL still links) —
//     ncclAllGather of the contiguous node-mask shards, or, for the
//     cost-balanced certified-cell pass, ncclAllReduce(sum) of the disjoint
//     partial masks (disjoint bits add without carries);
//   * a device listed twice (tests on one GPU): peer copies of the other
//     contexts' shards, ordered by cross-stream events (no host staging).
// Node masks are pure functions of position, so the labels are
// bit-identical to one device for any group.
#include "context.cuh"

#include <dlfcn.h>
#include <nccl.h>

using namespace nmh;

namespace {

// NCCL entry points resolved at run time (torch processes have already
// loaded their bundled libnccl.so.2; others load the system one).
struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
  static const Nccl& get() {
    static Nccl n = [] {
      Nccl x;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return x;
      x.init_all = reinterpret_cast<decltype(x.init_all)>(dlsym(h, "ncclCommInitAll"));
      x.destroy = reinterpret_cast<decltype(x.destroy)>(dlsym(h, "ncclCommDestroy"));
      x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(h, "ncclAllGather"));
      x.all_reduce = reinterpret_cast<decltype(x.all_reduce)>(dlsym(h, "ncclAllReduce"));
      x.group_start = reinterpret_cast<decltype(x.group_start)>(dlsym(h, "ncclGroupStart"));
      x.group_end = reinterpret_cast<decltype(x.group_end)>(dlsym(h, "ncclGroupEnd"));
      x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(h, "ncclGetErrorString"));
      x.ok = x.init_all && x.destroy && x.all_gather && x.all_reduce && x.group_start && x.group_end && x.error_string;
      return x;
    }();
    return n;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(std::string(what) + ": " + Nccl::get().error_string(r));
}

// dst[i] |= src[i] (peer-copy merge of the cost-balanced partial masks)
__global__ void k_or_into(std::uint32_t* __restrict__ dst, const std::uint32_t* __restrict__ src, std::size_t n) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    dst[i] |= src[i];
}

// Run f(r) for every device on its own host thread; rethrow the first error.
template <class F>
void per_device(std::size_t R, F&& f) {
  std::vector<std::exception_ptr> err(R);
  std::vector<std::thread> th;
  for (std::size_t r = 0; r < R; ++r)
    th.emplace_back([&, r] {
      try {
        f(r);
      } catch (...) {
        err[r] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace

struct nm_group {
  std::vector<nm_ctx*> ctx;
  std::vector<cudaEvent_t> done;    // per device: its node pass (and partial masks) are complete
  std::vector<ncclComm_t> comms;    // distinct devices: one NCCL communicator per device
  bool distinct = false;
  ~nm_group() {
    for (std::size_t r = 0; r < comms.size(); ++r)
      if (comms[r]) Nccl::get().destroy(comms[r]);
    for (std::size_t r = 0; r < done.size(); ++r) {
      cudaSetDevice(ctx[r]->opt.device);
      cudaEventDestroy(done[r]);
    }
    for (nm_ctx* c : ctx) nm_destroy(c);
  }
};

extern "C" {

int nm_group_create(nm_group** out, int n, const int* devices, const nm_options* opt) {
  return guarded([&] {
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    if (n < 1) throw Error("group needs at least one device");
    std::unique_ptr<nm_group> g(new nm_group);
    std::vector<int> devs;
    for (int r = 0; r < n; ++r) {
      nm_options o;
      if (opt) o = *opt;
      else nm_default_options(&o);
      o.device = devices ? devices[r] : r;
      devs.push_back(o.device);
      nm_ctx* c = nullptr;
      if (nm_create(&c, &o) != 0) throw Error(last_error());
      g->ctx.push_back(c);
      cudaEvent_t e;
      NM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      g->done.push_back(e);
    }
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    g->distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    // NM_GROUP_NCCL=1: communicators even for a single device (exercises the
    // NCCL exchange on a one-GPU box; a 1-rank all-gather is a copy)
    const char* force = std::getenv("NM_GROUP_NCCL");
    const bool want_nccl = g->distinct && (n > 1 || (force && force[0] == '1'));
    if (want_nccl) {
      for (int a : devs)
        for (int b : devs) {
          int can = 0;
          if (a != b && cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
            NM_CUDA(cudaSetDevice(a));
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) NM_CUDA(e);
            cudaGetLastError();
          }
        }
      if (Nccl::get().ok) {
        g->comms.assign(n, nullptr);
        nccl_check(Nccl::get().init_all(g->comms.data(), n, devs.data()), "ncclCommInitAll");
      }
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
    per_device(g->ctx.size(), [&](std::size_t r) {
      if (nm_set_surfaces(g->ctx[r], xyz, nv, tri, nt, comp_off, K, label_ids) != 0) throw Error(last_error());
    });
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
    for (nm_ctx* c : g->ctx) require_surfaces(c);
    // With certified cells the work per point is far from uniform (only pairs
    // near a surface are evaluated), so every device takes a cost-balanced
    // share of the pair lists of ALL points (disjoint partial masks);
    // otherwise contiguous node shards (padded to R * per_n for the gather).
    const bool by_pairs = R > 1 && g->ctx[0]->opt.cull_outside == 2 && g->ctx[0]->cells;
    const std::size_t len = by_pairs ? n : R * per_n;  // full mask buffer per device
    std::vector<std::uint32_t*> d_all(R);
    // 1) node passes, one host thread per device
    per_device(R, [&](std::size_t r) {
      nm_ctx* c = g->ctx[r];
      NM_CUDA(cudaSetDevice(c->opt.device));
      d_all[r] = c->masks.as<std::uint32_t>(std::max<std::size_t>(len, 1));
      (void)c->masks2.as<std::uint32_t>(std::max<std::size_t>(n, 1));  // merge scratch, sized before any launch
      if (by_pairs) {
        auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
        c->h2d(d_pts, nodes, 3 * n * sizeof(double), c->stream);
        if (n)
          label_nodes_dev(c, d_pts, n, T, d_all[r], nullptr, c->stream, nullptr, nullptr, false, static_cast<int>(r),
                          static_cast<int>(R));
      } else {
        const std::size_t lo = std::min(n, r * per_n), hi = std::min(n, lo + per_n);
        auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(hi - lo, 1));
        c->h2d(d_pts, nodes + 3 * lo, 3 * (hi - lo) * sizeof(double), c->stream);
        if (hi > lo) label_nodes_dev(c, d_pts, hi - lo, T, d_all[r] + r * per_n, nullptr, c->stream, nullptr);
        if (hi - lo < per_n)  // padding of the last shard(s)
          NM_CUDA(cudaMemsetAsync(d_all[r] + r * per_n + (hi - lo), 0, (per_n - (hi - lo)) * 4, c->stream));
      }
      NM_CUDA(cudaEventRecord(g->done[r], c->stream));
    });
    // 2) exchange on the devices
    if ((R > 1 || !g->comms.empty()) && n) {
      if (!g->comms.empty()) {
        const Nccl& nc = Nccl::get();
        nccl_check(nc.group_start(), "ncclGroupStart");
        for (std::size_t r = 0; r < R; ++r) {
          nm_ctx* c = g->ctx[r];
          NM_CUDA(cudaSetDevice(c->opt.device));
          if (by_pairs)
            nccl_check(nc.all_reduce(d_all[r], d_all[r], n, ncclUint32, ncclSum, g->comms[r], c->stream), "ncclAllReduce");
          else
            nccl_check(nc.all_gather(d_all[r] + r * per_n, d_all[r], per_n, ncclUint32, g->comms[r], c->stream),
                       "ncclAllGather");
        }
        nccl_check(nc.group_end(), "ncclGroupEnd");
      } else {
        // peer copies (a device listed more than once, or no NCCL), ordered
        // after each source's node pass by its event
        for (std::size_t r = 0; r < R; ++r) {
          nm_ctx* c = g->ctx[r];
          NM_CUDA(cudaSetDevice(c->opt.device));
          auto* tmp = c->masks2.as<std::uint32_t>(std::max<std::size_t>(n, 1));
          for (std::size_t q = 0; q < R; ++q) {
            if (q == r) continue;
            NM_CUDA(cudaStreamWaitEvent(c->stream, g->done[q], 0));
            const int dq = g->ctx[q]->opt.device, dr = c->opt.device;
            if (by_pairs) {
              NM_CUDA(cudaMemcpyPeerAsync(tmp, dr, d_all[q], dq, n * 4, c->stream));
              k_or_into<<<grid_for(n, 256, c->sm_count * 8), 256, 0, c->stream>>>(d_all[r], tmp, n);
              NM_CUDA(cudaGetLastError());
            } else {
              NM_CUDA(cudaMemcpyPeerAsync(d_all[r] + q * per_n, dr, d_all[q] + q * per_n, dq, per_n * 4, c->stream));
            }
          }
        }
      }
    }
    // 3) tet shards on every device, labels back into the caller's array
    per_device(R, [&](std::size_t r) {
      nm_ctx* c = g->ctx[r];
      NM_CUDA(cudaSetDevice(c->opt.device));
      const std::size_t lo = std::min(nt, r * per_t), hi = std::min(nt, lo + per_t);
      auto* d_t = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(hi - lo, 1));
      auto* d_l = c->labels.as<int>(std::max<std::size_t>(hi - lo, 1));
      c->h2d(d_t, tets + 4 * lo, 4 * (hi - lo) * sizeof(std::uint32_t), c->stream);
      if (hi > lo) {
        label_tets_dev(c, d_t, hi - lo, d_all[r], d_l, c->stream, nullptr, n);
        c->d2h(labels_out + lo, d_l, (hi - lo) * sizeof(int), c->stream);
      }
      if (r == 0 && masks_out) c->d2h(masks_out, d_all[0], n * 4, c->stream);
      NM_CUDA(cudaStreamSynchronize(c->stream));
      // peer copies read the other devices' buffers: keep them until all are done
      NM_CUDA(cudaEventRecord(g->done[r], c->stream));
    });
    for (std::size_t r = 0; r < R; ++r) {
      NM_CUDA(cudaSetDevice(g->ctx[r]->opt.device));
      NM_CUDA(cudaEventSynchronize(g->done[r]));
    }
    if (stats) {
      stats->points = n;
      stats->triangles = g->ctx[0]->nt_real;
      stats->evals = static_cast<std::uint64_t>(n) * g->ctx[0]->nt_real;
    }
  });
}

int nm_group_uses_nccl(const nm_group* g) { return g && !g->comms.empty() ? 1 : 0; }

}  // extern "C"
