// libnestmesh_label.so — C ABI (include/nestmesh_label.h) over the sm_100a
// labeling kernels. One context = one device + one stream; host entry points
// are synchronous, *_device entry points are asynchronous on the caller's
// stream. There is no CPU fallback: every compute entry point fails without
// a usable device.
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <memory>
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
#include "nestmesh_label.h"
#include "refine.h"

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define NM_CUDA(x)                                                                                    \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess)                                                                            \
      throw Error(std::string(#x) + ": " + cudaGetErrorName(e_) + " " + cudaGetErrorString(e_));       \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

// Growable device buffer.
struct DBuf {
  void* p = nullptr;
  std::size_t cap = 0;
  void* get(std::size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      const std::size_t want = std::max<std::size_t>(bytes, 256);
      NM_CUDA(cudaMalloc(&p, want));
      cap = want;
    }
    return p;
  }
  template <class T>
  T* as(std::size_t count) {
    return static_cast<T*>(get(count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Run f(0..n-1) on up to hardware_concurrency host threads (independent
// per-compartment host work of nm_set_surfaces; f must not throw).
template <class F>
void parallel_for(int n, F&& f) {
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
std::uint32_t spread10h(std::uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}


// Greedy triangle-strip decomposition of one compartment.
// Start from the unused triangle with the fewest unused neighbours, try its
// three rotations, walk forward across (u_{k+1}, u_{k+2}) and backward from the
// reversed start, keep the longest. Returns, per strip, the vertex sequence
// u_0..u_{m+1} and the original triangle ids t_0..t_{m-1} with
// {u_k, u_{k+1}, u_{k+2}} == set(t_k). Only performance depends on the
// quality of the decomposition; every triangle appears in exactly one strip.
struct Strip {
  std::vector<std::uint32_t> v;
  std::vector<std::uint32_t> t;
};

std::vector<Strip> stripify(const std::uint32_t* tri, std::uint32_t t0, std::uint32_t t1) {
  const std::uint32_t m = t1 - t0;
  std::unordered_map<std::uint64_t, std::array<std::int64_t, 2>> edges;
  edges.reserve(static_cast<std::size_t>(m) * 2);
  auto key = [](std::uint32_t a, std::uint32_t b) {
    return a < b ? (std::uint64_t(a) << 32 | b) : (std::uint64_t(b) << 32 | a);
  };
  for (std::uint32_t i = 0; i < m; ++i) {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    for (int j = 0; j < 3; ++j) {
      auto [it, ins] = edges.try_emplace(key(e[j], e[(j + 1) % 3]), std::array<std::int64_t, 2>{-1, -1});
      auto& s = it->second;
      if (s[0] < 0) s[0] = i;
      else if (s[1] < 0) s[1] = i;
    }
  }
  std::vector<std::uint8_t> used(m, 0);
  auto nbr = [&](std::uint32_t i, std::uint32_t a, std::uint32_t b) -> std::int64_t {
    const auto& s = edges.at(key(a, b));
    return s[0] == static_cast<std::int64_t>(i) ? s[1] : s[0];
  };
  std::vector<int> deg(m, 0);
  for (std::uint32_t i = 0; i < m; ++i) {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    for (int j = 0; j < 3; ++j) deg[i] += nbr(i, e[j], e[(j + 1) % 3]) >= 0;
  }
  using QE = std::pair<int, std::uint32_t>;
  std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
  for (std::uint32_t i = 0; i < m; ++i) pq.emplace(deg[i], i);
  std::vector<std::uint32_t> mark(m, 0);
  std::uint32_t stamp = 0;
  // forward walk from triangle i with vertex order (a,b,c)
  auto walk = [&](std::uint32_t i, std::uint32_t a, std::uint32_t b, std::uint32_t c, std::vector<std::uint32_t>& vs,
                  std::vector<std::uint32_t>& ts) {
    vs.assign({a, b, c});
    ts.assign({i});
    mark[i] = stamp;
    std::uint32_t cur = i;
    for (;;) {
      const std::uint32_t u = vs[vs.size() - 2], w = vs.back();
      const std::int64_t n = nbr(cur, u, w);
      if (n < 0 || used[n] || mark[n] == stamp) break;
      const std::uint32_t* e = tri + 3 * std::size_t(t0 + n);
      std::uint32_t x = e[0];
      for (int j = 0; j < 3; ++j)
        if (e[j] != u && e[j] != w) x = e[j];
      vs.push_back(x);
      ts.push_back(static_cast<std::uint32_t>(n));
      mark[n] = stamp;
      cur = static_cast<std::uint32_t>(n);
    }
  };
  std::vector<Strip> out;
  std::vector<std::uint32_t> fv, ft, bv, btt;
  while (!pq.empty()) {
    auto [d, i] = pq.top();
    pq.pop();
    if (used[i] || d != deg[i]) continue;
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    Strip best;
    for (int r = 0; r < 3; ++r) {
      const std::uint32_t a = e[r], b = e[(r + 1) % 3], c = e[(r + 2) % 3];
      ++stamp;
      walk(i, a, b, c, fv, ft);
      // backward: walk from the reversed start without reusing forward triangles
      std::vector<std::uint32_t> keep(ft.begin(), ft.end());
      walk(i, c, b, a, bv, btt);
      // bv = c,b,a,x,y,...; combined vertex sequence = reverse(bv) + fv[3:]
      Strip s;
      s.v.assign(bv.rbegin(), bv.rend());
      s.v.insert(s.v.end(), fv.begin() + 3, fv.end());
      s.t.assign(btt.rbegin(), btt.rend());  // ..., i
      s.t.insert(s.t.end(), ft.begin() + 1, ft.end());
      if (s.t.size() > best.t.size()) best = std::move(s);
    }
    for (std::uint32_t t : best.t) used[t] = 1;
    for (std::uint32_t t : best.t) {
      const std::uint32_t* f = tri + 3 * std::size_t(t0 + t);
      for (int j = 0; j < 3; ++j) {
        const std::int64_t n = nbr(t, f[j], f[(j + 1) % 3]);
        if (n >= 0 && !used[n]) pq.emplace(--deg[n], static_cast<std::uint32_t>(n));
      }
    }
    for (auto& t : best.t) t += t0;
    out.push_back(std::move(best));
  }
  return out;
}
}  // namespace

struct nm_ctx {
  nm_options opt{};
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // tet upload + validation, overlapped with the node pass
  cudaEvent_t ev[6] = {};
  cudaEvent_t ev_side = nullptr;
  std::uint32_t* h_word = nullptr;        // pinned: max tet node index read back from the side stream
  std::uint64_t node_launches = 0;        // launches of the last label_nodes_dev
  int sm_count = 0;

  // surfaces
  bool has_surfaces = false;
  bool strips = false;  // tile layout of the current surfaces
  std::size_t flag_cap = 0;  // flagmask length when evaluating a subset (= node count)
  int K = 0;
  std::size_t nt_real = 0, nt_pad = 0, nv = 0;
  double cx = 0, cy = 0, cz = 0;
  double lo[3] = {0, 0, 0}, span = 1.0;  // Morton box of the domain
  nm::LabelIds ids{};
  std::vector<std::uint32_t> comp_tiles_h;  // host copy of the K+1 tile offsets
  std::size_t n_continued = 0;              // strip segments continuing the previous one (cont bits set)
  DBuf tri, sub, edges, cont, comp_tiles, xyz64, tri_idx, comp_off, comp_box, cullmask;
  // certified cells (cull_outside = 2, cells.cuh)
  bool cells = false;
  DBuf dist_clus, dist_slot, dist_ord, sp_part, sp_det, cell_state, cell_child, cell_cert, cell_blk, cell_grids, clus, clus_tri, clus_tsph, unk, sp_list, sp_chunk, sp_cnt, rep_pts, rep_s, rep_m, rep_f;
  std::uint64_t cells_total = 0, cells_certified = 0, cell_reps = 0, sparse_pairs = 0, sparse_evals = 0;
  double ms_cells = 0.0;  // host wall time of the certification (nm_set_surfaces)
  std::vector<std::uint32_t> comp_off_h;

  // scratch
  DBuf pts, masks, flagmask, nbr, known, want, fkeys, frontier, lex, region, bfaces, btri, dist_tri, dist_xyz,
      dist_idx, dist_d32, dist_out, r_red, r_keys, r_keys2, r_S, r_idx, r_touched,
      r_mask, r_cnt, r_offs, r_flag, meshA_nodes, meshA_tets, meshA_labels, meshB_nodes, meshB_tets, meshB_labels,
      meshB_parent, masks2, order, keys, keys_alt, order_alt, cub_tmp, list, chunk, counters, count, tets, labels,
      s_out, word;

  ~nm_ctx() {
    for (DBuf* b : {&dist_clus, &dist_slot, &dist_ord, &sp_part, &sp_det, &cell_state, &cell_child, &cell_cert, &cell_blk, &cell_grids, &clus, &clus_tri, &clus_tsph, &unk, &sp_list, &sp_chunk, &sp_cnt, &rep_pts, &rep_s,
                    &rep_m, &rep_f})
      b->release();
    for (DBuf* b : {&tri, &sub, &edges, &cont, &comp_tiles, &xyz64, &tri_idx, &comp_off, &comp_box, &cullmask, &pts, &masks, &flagmask, &nbr, &known, &want, &fkeys, &frontier, &lex, &region, &bfaces, &btri,
                    &dist_tri, &dist_xyz, &dist_idx, &dist_d32, &dist_out, &r_red, &r_keys, &r_keys2, &r_S,
                    &r_idx, &r_touched, &r_mask, &r_cnt, &r_offs, &r_flag, &meshA_nodes, &meshA_tets, &meshA_labels,
                    &meshB_nodes, &meshB_tets, &meshB_labels, &meshB_parent, &masks2, &order, &keys,
                    &keys_alt, &order_alt, &cub_tmp, &list, &chunk, &counters, &count, &tets, &labels, &s_out, &word})
      b->release();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_side) cudaEventDestroy(ev_side);
    if (h_word) cudaFreeHost(h_word);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
  }

  cudaStream_t pick(void* s) const { return s ? static_cast<cudaStream_t>(s) : stream; }
};

namespace {

void require_surfaces(const nm_ctx* c) {
  if (!c) throw Error("null context");
  if (!c->has_surfaces) throw Error("nm_set_surfaces has not been called");
}

int grid_for(std::size_t n, int block, int cap) {
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


// Full node pass on device-resident points: Morton order -> K1 -> compaction
// of flagged points -> K3. masks/s_out are device pointers.
// d_subset (nullable): evaluate only points d_pts[d_subset[i]], i < n; masks
// (and s) are written at the original point index.
void read_node_stats(nm_ctx* c, std::size_t n, cudaStream_t st, nm_stats* stats);

// Compartment split of a k_label launch (LabelParams::split): when the point
// blocks alone fill fewer than kSplitWaves waves of resident CTAs (few
// points: small meshes, many GPUs, refinement passes), the compartments are
// cut into up to K contiguous groups of about equal tile count so the grid
// has enough CTAs to keep every SM busy to the end. Returns the group count.
int compartment_split(const nm_ctx* c, std::size_t nblocks, int* split) {
  constexpr double kSplitWaves = 24.0;
  const int K = c->K;
  const double slots = double(c->sm_count) * NM_MIN_BLOCKS;
  int want = 1;
  if (K > 1 && nblocks > 0 && double(nblocks) < kSplitWaves * slots)
    want = static_cast<int>(std::min<double>(K, std::ceil(kSplitWaves * slots / double(nblocks))));
  const auto& t = c->comp_tiles_h;
  const double total = double(t[K] - t[0]);
  int g = 0;
  split[g++] = 0;
  for (int j = 1; j < want; ++j) {
    const double target = total * j / want;
    int b = split[g - 1] + 1;
    while (b < K && double(t[b] - t[0]) < target) ++b;
    if (b >= K) break;
    split[g++] = b;
  }
  split[g] = K;
  return g;
}


// Sparse k_label (MODE 2) over per-compartment lists of evaluation positions
// (prm.sp_list, cnt[k] entries for compartment k, concatenated). Returns the
// number of launches (0 when every list is empty).
// first (optional): start of compartment k's slice in sp_list (default: the
// prefix sum of cnt, i.e. the slices are packed).
int launch_sparse(nm_ctx* c, nm::LabelParams& prm, const std::vector<std::uint32_t>& cnt, cudaStream_t st,
                  const std::vector<std::uint32_t>* first = nullptr) {
  const std::uint32_t per_block = nm::kBlock * 2;
  const int K = c->K;
  // Few point chunks (a thin shell of pairs) would leave SMs idle in the last
  // wave: then each chunk's tiles are split into fold blocks evaluated by
  // separate CTAs (same fp64 fold order, see kFoldTiles), and
  // k_sparse_finalize adds the block partials.
  std::uint64_t chunks = 0;
  for (int k = 0; k < K; ++k) chunks += (cnt[k] + per_block - 1) / per_block;
  constexpr double kSplitWaves = 8.0;
  const bool split = chunks > 0 && double(chunks) < kSplitWaves * c->sm_count * NM_MIN_BLOCKS;
  std::uint32_t off = 0, blk = 0;
  std::uint64_t po = 0;
  for (int k = 0; k <= 32; ++k) {
    prm.sp_blk[k] = blk;
    if (k < K) {
      const std::uint32_t tiles = c->comp_tiles_h[k + 1] - c->comp_tiles_h[k];
      const std::uint32_t nfb = split ? std::max<std::uint32_t>(1, (tiles + nm::kFoldTiles - 1) / nm::kFoldTiles) : 1;
      prm.sp_off[k] = first ? (*first)[k] : off;
      prm.sp_fb[k] = nfb;
      prm.sp_po[k] = static_cast<std::uint32_t>(po);
      off += cnt[k];
      blk += (cnt[k] + per_block - 1) / per_block * nfb;
      po += std::uint64_t(cnt[k]) * nfb;
    }
  }
  // the kernel reads sp_list[sp_off[k], sp_end[k])
  for (int k = 0; k < K; ++k) prm.sp_end[k] = prm.sp_off[k] + cnt[k];
  if (blk == 0) return 0;
  if (po > 0xffffffffull) throw Error("too many fold-block partials in one call");
  prm.split[0] = 0;
  prm.split[1] = K;
  prm.sp_part = split ? c->sp_part.as<double>(po) : nullptr;
  prm.sp_det = split ? c->sp_det.as<std::uint8_t>(po) : nullptr;
  if (c->strips) nm::k_label<1, true, 2><<<blk, nm::kBlock, 0, st>>>(prm);
  else nm::k_label<1, false, 2><<<blk, nm::kBlock, 0, st>>>(prm);
  NM_CUDA(cudaGetLastError());
  if (!split) return 1;
  nm::FinalizeParams fp{};
  fp.list = prm.sp_list;
  fp.order = prm.order;
  fp.part = prm.sp_part;
  fp.det = prm.sp_det;
  std::uint32_t q = 0;
  for (int k = 0; k < K; ++k) {
    fp.sp_off[k] = prm.sp_off[k];
    fp.qo[k] = q;
    fp.po[k] = prm.sp_po[k];
    fp.fb[k] = prm.sp_fb[k];
    q += cnt[k];
  }
  fp.qo[K] = q;
  fp.K = K;
  fp.T = prm.T;
  fp.band = prm.band;
  fp.masks = prm.masks;
  fp.flagmask = prm.flagmask;
  fp.s_out = prm.s_out;
  nm::k_sparse_finalize<<<grid_for(q, 256, c->sm_count * 8), 256, 0, st>>>(fp);
  NM_CUDA(cudaGetLastError());
  return 2;
}

// Certified-cell classification of the n evaluation positions (order[i]) and
// per-compartment compaction of the pairs left to evaluate. Presets masks,
// flagmask and the known s entries; returns the per-compartment counts (one
// host synchronisation, for the grid size) with the lists in c->sp_list.
std::vector<std::uint32_t> classify_cells(nm_ctx* c, const double* d_pts, std::size_t n, const std::uint32_t* order,
                                          std::uint32_t* d_masks, std::uint32_t* flagmask, double* d_s, cudaStream_t st,
                                          std::uint64_t& launches, bool preset_known = true) {
  const int K = c->K;
  auto* unk = c->unk.as<std::uint32_t>(n);
  const std::size_t nb = std::max<std::size_t>(1, (n + nm::kSelChunk - 1) / nm::kSelChunk);
  auto* chunk = c->sp_chunk.as<std::uint32_t>(nb * K);
  auto* dcnt = c->sp_cnt.as<std::uint32_t>(K);
  (void)c->sp_list.as<std::uint32_t>(n);  // grown below if needed (after the sync)
  nm::ClassifyParams cp{};
  cp.pts = d_pts;
  cp.n = n;
  cp.order = order;
  cp.cx = c->cx;
  cp.cy = c->cy;
  cp.cz = c->cz;
  cp.dop4 = c->opt.cull_outside ? static_cast<const float4*>(c->comp_box.p) : nullptr;
  cp.grids = c->cells ? static_cast<const nm::CellGrid*>(c->cell_grids.p) : nullptr;
  cp.preset = preset_known;
  cp.code = static_cast<const std::uint32_t*>(c->cell_state.p);
  cp.child = static_cast<const std::uint8_t*>(c->cell_child.p);
  cp.K = K;
  cp.unk = unk;
  cp.masks = d_masks;
  cp.flagmask = flagmask;
  cp.s_out = d_s;
  nm::k_cell_classify<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(cp);
  ++launches;
  for (int k = 0; k < K; ++k) {
    nm::k_select_count<<<static_cast<unsigned>(nb), nm::kSelBlock, 0, st>>>(nm::PredBit{unk, k}, n, chunk + k * nb);
    nm::k_select_scan<<<1, 1024, 0, st>>>(chunk + k * nb, nb, dcnt + k);
    launches += 2;
  }
  std::vector<std::uint32_t> cnt(K);
  NM_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, K * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
  NM_CUDA(cudaStreamSynchronize(st));
  std::size_t total = 0;
  for (int k = 0; k < K; ++k) total += cnt[k];
  if (total > 0xffffffffull) throw Error("more than 2^32 (point, compartment) pairs to evaluate in one call");
  auto* list = c->sp_list.as<std::uint32_t>(std::max<std::size_t>(total, 1));
  std::size_t off = 0;
  c->sparse_pairs = total;
  c->sparse_evals = 0;
  for (int k = 0; k < K; ++k) {
    if (cnt[k]) {
      nm::k_select_write<<<static_cast<unsigned>(nb), nm::kSelBlock, 0, st>>>(nm::PredBit{unk, k}, n, chunk + k * nb,
                                                                              list + off);
      ++launches;
    }
    off += cnt[k];
    c->sparse_evals += std::uint64_t(cnt[k]) * (c->comp_off_h[k + 1] - c->comp_off_h[k]);
  }
  NM_CUDA(cudaGetLastError());
  return cnt;
}

// stats_deferred: the caller collects the stats later with read_node_stats
// (no host synchronisation inside; nm_label_mesh overlaps the tet upload).
// Cost-balanced split of the per-compartment pair lists over nshards: pair i
// of compartment k costs w_k = its tile count and starts at cost P_k + i w_k
// (P_k = cost of the lists before k); shard r takes the pairs starting in
// [floor(C r / N), floor(C (r + 1) / N)). The same integer formula on every
// shard, so the slices partition every list exactly. In: cnt = list lengths;
// out: first[k] = start of this shard's slice in the packed lists, cnt[k] =
// its length.
void shard_slices(const nm_ctx* c, std::vector<std::uint32_t>& cnt, int shard, int nshards,
                  std::vector<std::uint32_t>& first) {
  const int K = c->K;
  std::vector<std::uint64_t> w(K), P(K + 1, 0);
  std::uint32_t off = 0;
  for (int k = 0; k < K; ++k) {
    w[k] = std::max<std::uint64_t>(1, c->comp_tiles_h[k + 1] - c->comp_tiles_h[k]);
    P[k + 1] = P[k] + w[k] * cnt[k];
    first[k] = off;
    off += cnt[k];
  }
  if (nshards <= 1) return;
  if (shard < 0 || shard >= nshards) throw Error("shard index out of range");
  const unsigned __int128 C = P[K];
  const std::uint64_t t0 = static_cast<std::uint64_t>(C * static_cast<unsigned>(shard) / static_cast<unsigned>(nshards));
  const std::uint64_t t1 =
      static_cast<std::uint64_t>(C * static_cast<unsigned>(shard + 1) / static_cast<unsigned>(nshards));
  auto bound = [&](int k, std::uint64_t t) -> std::uint32_t {  // first pair of k starting at cost >= t
    if (t <= P[k]) return 0;
    const std::uint64_t i = (t - P[k] + w[k] - 1) / w[k];
    return static_cast<std::uint32_t>(std::min<std::uint64_t>(i, cnt[k]));
  };
  for (int k = 0; k < K; ++k) {
    const std::uint32_t a = bound(k, t0), b = bound(k, t1);
    first[k] += a;
    cnt[k] = b - a;
  }
}

// nshards >= 1: a sharded pass (nm_label_nodes_shard_device) — evaluate only
// shard's cost-balanced share of the (point, compartment) pair lists of all
// n points; masks hold the known bits on shard 0 only, so the shards' masks
// OR (or add: the bits are disjoint) to the full result.
void label_nodes_dev(nm_ctx* c, const double* d_pts, std::size_t n, double T, std::uint32_t* d_masks, double* d_s,
                     cudaStream_t st, nm_stats* stats, const std::uint32_t* d_subset = nullptr,
                     bool stats_deferred = false, int shard = 0, int nshards = 0) {
  require_surfaces(c);
  if (!(T > 0.0 && T < 1.0)) throw Error("threshold must lie in (0, 1) (SPEC.md:216)");
  std::uint64_t launches = 0;
  auto* counters = c->counters.as<unsigned long long>(8);
  NM_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), st));
  if (stats) NM_CUDA(cudaEventRecord(c->ev[0], st));
  if (n == 0) {
    if (stats) {
      std::memset(stats, 0, sizeof *stats);
      stats->triangles = c->nt_real;
    }
    return;
  }
  if (n > 0xffffffffull) throw Error("more than 2^32 points in one call");
  auto* flagmask = c->flagmask.as<std::uint32_t>(d_subset ? c->flag_cap : n);
  // every scratch buffer is sized before the first launch: a growing DBuf
  // frees its old block, and cudaFree would wait for the kernels
  auto* list = c->list.as<std::uint32_t>(n);
  auto* d_count = c->count.as<std::uint32_t>(4);
  (void)c->chunk.as<std::uint32_t>(std::max<std::size_t>(1, (n + nm::kSelChunk - 1) / nm::kSelChunk));
  const std::uint32_t* order = d_subset;
  if (c->opt.sort_points && n > 1) {
    auto* keys = c->keys.as<std::uint32_t>(n);
    auto* keys2 = c->keys_alt.as<std::uint32_t>(n);
    auto* idx = c->order.as<std::uint32_t>(n);
    auto* idx2 = c->order_alt.as<std::uint32_t>(n);
    nm::k_morton_keys<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(d_pts, n, d_subset, c->lo[0], c->lo[1], c->lo[2],
                                                                           1024.0 / c->span, keys, idx);
    ++launches;
    cub::DoubleBuffer<std::uint32_t> kb(keys, keys2), vb(idx, idx2);
    std::size_t tmp = 0;
    NM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(n), 0, 30, st));
    void* t = c->cub_tmp.get(tmp);
    NM_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, static_cast<int>(n), 0, 30, st));
    launches += 4;  // CUB onesweep: histogram + 3 passes of 10 bits (library kernels)
    order = vb.Current();
  }
  nm::LabelParams prm{};
  prm.pts = d_pts;
  prm.n = n;
  prm.order = order;
  prm.tri = static_cast<const float4*>(c->tri.p);
  prm.sub = static_cast<const float4*>(c->sub.p);
  prm.edges = static_cast<const float4*>(c->edges.p);
  prm.cont = static_cast<const std::uint32_t*>(c->cont.p);
  prm.comp_tiles = static_cast<const std::uint32_t*>(c->comp_tiles.p);
  prm.K = c->K;
  prm.cx = c->cx;
  prm.cy = c->cy;
  prm.cz = c->cz;
  prm.T = T;
  prm.band = c->opt.band;
  prm.tau = c->opt.tau;
  prm.delta = c->opt.delta_mm;
  prm.masks = d_masks;
  prm.flagmask = flagmask;
  prm.cull = nullptr;
  if ((c->opt.cull_outside == 2 && c->cells) || nshards >= 1) {
    // pair lists: classification presets every known pair (certified cells,
    // 13-DOP), the sparse pass evaluates the rest (one host synchronisation
    // for its grid); a sharded pass takes only its share of the lists
    if (nshards >= 1 && d_s) throw Error("sharded node passes do not return s");
    prm.s_out = d_s;
    prm.counters = counters;
    std::vector<std::uint32_t> cnt =
        classify_cells(c, d_pts, n, order, d_masks, flagmask, d_s, st, launches, /*preset_known=*/shard == 0);
    prm.sp_list = static_cast<const std::uint32_t*>(c->sp_list.p);
    std::vector<std::uint32_t> first(c->K);
    shard_slices(c, cnt, shard, nshards, first);
    c->sparse_pairs = c->sparse_evals = 0;  // this pass's share (nm_cell_info)
    for (int k = 0; k < c->K; ++k) {
      c->sparse_pairs += cnt[k];
      c->sparse_evals += std::uint64_t(cnt[k]) * (c->comp_off_h[k + 1] - c->comp_off_h[k]);
    }
    if (stats) NM_CUDA(cudaEventRecord(c->ev[1], st));
    launches += launch_sparse(c, prm, cnt, st, &first);
  } else {
  if (c->opt.cull_outside) {
    auto* cm = c->cullmask.as<std::uint32_t>(n);
    nm::k_cull_mask<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(
        d_pts, order, n, c->cx, c->cy, c->cz, static_cast<const float4*>(c->comp_box.p), c->K, cm);
    ++launches;
    prm.cull = cm;
  }
  prm.s_out = d_s;
  prm.counters = counters;
  const int np = prm.cull ? 1 : c->opt.pairs_per_thread;
  const std::size_t per_block = static_cast<std::size_t>(nm::kBlock) * 2 * np;
  const std::size_t nblocks = (n + per_block - 1) / per_block;
  const int csplit = compartment_split(c, nblocks, prm.split);
  if (csplit > 1) {
    nm::k_zero_masks<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(n, d_subset, d_masks, flagmask);
    ++launches;
  }
  if (stats) NM_CUDA(cudaEventRecord(c->ev[1], st));
  {
    const dim3 grid(static_cast<unsigned>(nblocks), static_cast<unsigned>(csplit));
    constexpr std::size_t smem = 0;  // k_label's tile buffers are static shared memory
    if (c->strips && prm.cull) {
      nm::k_label<1, true, 1><<<grid, nm::kBlock, smem, st>>>(prm);  // culling: one pair per thread
    } else if (c->strips) {
      if (np == 2) nm::k_label<2, true><<<grid, nm::kBlock, smem, st>>>(prm);
      else nm::k_label<1, true><<<grid, nm::kBlock, smem, st>>>(prm);
    } else if (prm.cull) {
      nm::k_label<1, false, 1><<<grid, nm::kBlock, smem, st>>>(prm);
    } else {
      if (np == 2) nm::k_label<2, false><<<grid, nm::kBlock, smem, st>>>(prm);
      else nm::k_label<1, false><<<grid, nm::kBlock, smem, st>>>(prm);
    }
  }
  NM_CUDA(cudaGetLastError());
  ++launches;
  }
  if (stats) NM_CUDA(cudaEventRecord(c->ev[2], st));
  // compaction of flagged points + fp64 fix-up
  select(c, nm::PredNonzero{flagmask, d_subset}, n, list, d_count, st, launches);
  nm::FixupParams fp{};
  fp.pts = d_pts;
  fp.list = list;
  fp.subset = d_subset;
  fp.count = d_count;
  fp.flagmask = flagmask;
  fp.xyz = static_cast<const double*>(c->xyz64.p);
  fp.tri = static_cast<const std::uint32_t*>(c->tri_idx.p);
  fp.comp_off = static_cast<const std::uint32_t*>(c->comp_off.p);
  fp.K = c->K;
  fp.T = T;
  fp.tie_eps = c->opt.tie_eps;
  fp.masks = d_masks;
  fp.s_out = d_s;
  fp.counters = counters;
  nm::k_fixup<<<c->sm_count * 16, 32 * nm::kFixWarps, 0, st>>>(fp);
  NM_CUDA(cudaGetLastError());
  ++launches;
  c->node_launches = launches;
  if (stats) {
    NM_CUDA(cudaEventRecord(c->ev[3], st));
    if (!stats_deferred) read_node_stats(c, n, st, stats);
  }
}

void read_node_stats(nm_ctx* c, std::size_t n, cudaStream_t st, nm_stats* stats) {
  {
    auto* counters = static_cast<unsigned long long*>(c->counters.p);
    auto* d_count = static_cast<std::uint32_t*>(c->count.p);
    unsigned long long h[8];
    std::uint32_t hc = 0;
    NM_CUDA(cudaMemcpyAsync(h, counters, sizeof h, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaMemcpyAsync(&hc, d_count, sizeof hc, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    std::memset(stats, 0, sizeof *stats);
    stats->points = n;
    stats->triangles = c->nt_real;
    stats->evals = static_cast<std::uint64_t>(n) * c->nt_real;
    stats->flagged_points = hc;
    stats->flagged_pairs = h[2];
    stats->ties = h[3];
    stats->near_subtiles = h[0];
    stats->far_subtiles = h[1];
    stats->launches = c->node_launches;
    NM_CUDA(cudaEventElapsedTime(&stats->ms_label, c->ev[1], c->ev[2]));
    NM_CUDA(cudaEventElapsedTime(&stats->ms_fixup, c->ev[2], c->ev[3]));
    NM_CUDA(cudaEventElapsedTime(&stats->ms_total, c->ev[0], c->ev[3]));
  }
}

void label_tets_dev(nm_ctx* c, const std::uint32_t* d_tets, std::size_t nt, const std::uint32_t* d_masks, int* d_labels,
                    cudaStream_t st, nm_stats* stats) {
  require_surfaces(c);
  if (nt == 0) return;
  if (stats) NM_CUDA(cudaEventRecord(c->ev[4], st));
  nm::k_label_tets<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(reinterpret_cast<const uint4*>(d_tets), nt,
                                                                        d_masks, d_labels, c->ids);
  NM_CUDA(cudaGetLastError());
  if (stats) {
    NM_CUDA(cudaEventRecord(c->ev[5], st));
    NM_CUDA(cudaEventSynchronize(c->ev[5]));
    float ms = 0;
    NM_CUDA(cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]));
    stats->ms_tets += ms;
    stats->launches += 1;
  }
}

void check_tets(const std::uint32_t* tets, std::size_t nt, std::size_t n_nodes) {
  for (std::size_t i = 0; i < 4 * nt; ++i)
    if (tets[i] >= n_nodes) throw Error("tet " + std::to_string(i / 4) + " references node " + std::to_string(tets[i]) +
                                        " >= node count " + std::to_string(n_nodes));
}

// The same validation on tets already uploaded to d_tets (k_max_index, one
// word read back); the host scan only runs to name the offending tet.
void check_tets_device(nm_ctx* c, const std::uint32_t* d_tets, const std::uint32_t* h_tets, std::size_t nt,
                       std::size_t n_nodes, cudaStream_t st) {
  if (nt == 0) return;
  auto* d_word = c->word.as<std::uint32_t>(1);
  NM_CUDA(cudaMemsetAsync(d_word, 0, sizeof(std::uint32_t), st));
  nm::k_max_index<<<grid_for(nt, 256, c->sm_count * 8), 256, 0, st>>>(reinterpret_cast<const uint4*>(d_tets), nt,
                                                                      d_word);
  NM_CUDA(cudaGetLastError());
  NM_CUDA(cudaMemcpyAsync(c->h_word, d_word, sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
  NM_CUDA(cudaStreamSynchronize(st));
  if (*c->h_word >= n_nodes) check_tets(h_tets, nt, n_nodes);
}


// Lexicographic order (k0, k1, k2) of m triples by three stable LSD radix
// passes; returns the device permutation (valid until the next call).
std::uint32_t* lex_order3(nm_ctx* c, const std::uint32_t* k0, const std::uint32_t* k1, const std::uint32_t* k2,
                          std::size_t m, cudaStream_t st) {
  auto* buf = c->lex.as<std::uint32_t>(4 * std::max<std::size_t>(m, 1));
  std::uint32_t *perm = buf, *perm2 = buf + m, *key = buf + 2 * m, *key2 = buf + 3 * m;
  nm::k_iota<<<grid_for(std::max<std::size_t>(m, 1), 256, c->sm_count * 32), 256, 0, st>>>(perm, m);
  if (m <= 1) return perm;
  std::uint32_t* cur = perm;
  std::uint32_t* alt = perm2;
  for (const std::uint32_t* k : {k2, k1, k0}) {
    nm::k_gather_key<<<grid_for(m, 256, c->sm_count * 32), 256, 0, st>>>(k, cur, m, key);
    cub::DoubleBuffer<std::uint32_t> kb(key, key2), vb(cur, alt);
    std::size_t tmp = 0;
    NM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(m), 0, 32, st));
    void* tp = c->cub_tmp.get(tmp);
    NM_CUDA(cub::DeviceRadixSort::SortPairs(tp, tmp, kb, vb, static_cast<int>(m), 0, 32, st));
    if (vb.Current() != cur) std::swap(cur, alt);
  }
  return cur;
}

// Face adjacency (mesh.hpp:68-88): nbr[4t+f] = tet across local face f, -1 on
// the mesh boundary. Sorted face triples; equal neighbours share the face.
void face_adjacency(nm_ctx* c, const uint4* t4, std::size_t nt, std::int32_t* d_nbr, cudaStream_t st) {
  const std::size_t m = 4 * nt;
  NM_CUDA(cudaMemsetAsync(d_nbr, 0xff, std::max<std::size_t>(m, 1) * sizeof(std::int32_t), st));
  if (m <= 1) return;
  auto* ka = c->fkeys.as<std::uint32_t>(4 * m);
  std::uint32_t *kb = ka + m, *kc = ka + 2 * m, *fid = ka + 3 * m;
  nm::k_face_keys<<<grid_for(m, 256, c->sm_count * 32), 256, 0, st>>>(t4, nt, ka, kb, kc, fid);
  const std::uint32_t* order = lex_order3(c, ka, kb, kc, m, st);
  nm::k_face_pairs<<<grid_for(m, 256, c->sm_count * 32), 256, 0, st>>>(order, m, ka, kb, kc, d_nbr);
  NM_CUDA(cudaGetLastError());
}

struct PredByte {
  const std::uint8_t* v;
  __device__ bool operator()(std::size_t i) const { return v[i] != 0; }
};

// Device refine_volume (refine.cuh): (nodes n, tets nt, labels) + selected
// tets -> refined mesh in the B buffers. Returns (n2, nt2).
std::pair<std::size_t, std::size_t> refine_dev(nm_ctx* c, const double* d_nodes, std::size_t n, const std::uint32_t* d_tets,
                                               std::size_t nt, const int* d_labels, const std::uint32_t* d_sel,
                                               std::uint32_t nsel, cudaStream_t st, std::uint64_t& launches) {
  const uint4* t4 = reinterpret_cast<const uint4*>(d_tets);
  auto* red = c->r_red.as<std::uint8_t>(std::max<std::size_t>(nt, 1));
  auto* touched = c->r_touched.as<std::uint8_t>(std::max<std::size_t>(n, 1));
  auto* tmask = c->r_mask.as<std::uint8_t>(std::max<std::size_t>(nt, 1));
  auto* flag = c->r_flag.as<unsigned>(4);
  auto* d_count = c->count.as<std::uint32_t>(4);
  auto* red_list = c->r_idx.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
  NM_CUDA(cudaMemsetAsync(red, 0, std::max<std::size_t>(nt, 1), st));
  NM_CUDA(cudaMemcpyAsync(d_count, &nsel, sizeof nsel, cudaMemcpyHostToDevice, st));
  nm::k_mark_list<<<grid_for(std::max<std::uint32_t>(nsel, 1), 256, c->sm_count * 8), 256, 0, st>>>(d_sel, d_count, red);
  ++launches;
  unsigned long long* S = nullptr;
  std::uint32_t m = 0;
  for (int it = 0; it < 1000; ++it) {
    select(c, PredByte{red}, nt, red_list, d_count, st, launches);
    std::uint32_t r = 0;
    NM_CUDA(cudaMemcpyAsync(&r, d_count, sizeof r, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    const std::size_t nk = 6ull * r;
    auto* keys = c->r_keys.as<unsigned long long>(std::max<std::size_t>(nk, 1));
    auto* keys2 = c->r_keys2.as<unsigned long long>(std::max<std::size_t>(nk, 1));
    nm::k_red_edges<<<grid_for(std::max<std::uint32_t>(r, 1), 256, c->sm_count * 8), 256, 0, st>>>(t4, red_list, d_count, keys);
    ++launches;
    const unsigned long long* sorted = keys;
    if (nk > 1) {
      cub::DoubleBuffer<unsigned long long> kb(keys, keys2);
      std::size_t tmp = 0;
      NM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kb, static_cast<int>(nk), 0, 64, st));
      void* tp = c->cub_tmp.get(tmp);
      NM_CUDA(cub::DeviceRadixSort::SortKeys(tp, tmp, kb, static_cast<int>(nk), 0, 64, st));
      sorted = kb.Current();
    }
    auto* uidx = c->frontier.as<std::uint32_t>(std::max<std::size_t>(nk, 1));
    select(c, nm::PredUniqueKey{sorted}, nk, uidx, d_count, st, launches);
    S = c->r_S.as<unsigned long long>(std::max<std::size_t>(nk, 1));
    nm::k_gather_keys<<<grid_for(std::max<std::size_t>(nk, 1), 256, c->sm_count * 8), 256, 0, st>>>(sorted, uidx, d_count, S);
    NM_CUDA(cudaMemsetAsync(touched, 0, std::max<std::size_t>(n, 1), st));
    nm::k_touch_nodes<<<grid_for(std::max<std::size_t>(nk, 1), 256, c->sm_count * 8), 256, 0, st>>>(S, d_count, touched);
    NM_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), st));
    nm::k_classify<<<grid_for(std::max<std::size_t>(nt, 1), 256, c->sm_count * 32), 256, 0, st>>>(t4, nt, red, touched, S,
                                                                                                 d_count, tmask, flag);
    launches += 4;
    unsigned changed = 0;
    NM_CUDA(cudaMemcpyAsync(&changed, flag, sizeof changed, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaMemcpyAsync(&m, d_count, sizeof m, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    if (!changed) break;
  }
  // children per tet -> offsets
  auto* cnt = c->r_cnt.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
  auto* offs = c->r_offs.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
  nm::k_child_count<<<grid_for(std::max<std::size_t>(nt, 1), 256, c->sm_count * 32), 256, 0, st>>>(tmask, nt, cnt);
  std::size_t tmp = 0;
  NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, offs, static_cast<int>(nt), st));
  void* tp = c->cub_tmp.get(tmp);
  NM_CUDA(cub::DeviceScan::ExclusiveSum(tp, tmp, cnt, offs, static_cast<int>(nt), st));
  std::uint32_t last[2] = {0, 0};
  if (nt) {
    NM_CUDA(cudaMemcpyAsync(&last[0], offs + nt - 1, 4, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaMemcpyAsync(&last[1], cnt + nt - 1, 4, cudaMemcpyDeviceToHost, st));
  }
  NM_CUDA(cudaStreamSynchronize(st));
  const std::size_t nt2 = static_cast<std::size_t>(last[0]) + last[1];
  const std::size_t n2 = n + m;
  if (n2 > 0xffffffffull || nt2 > 0xffffffffull) throw Error("refined mesh exceeds 32-bit ids");
  auto* nodes2 = c->meshB_nodes.as<double>(3 * std::max<std::size_t>(n2, 1));
  auto* tets2 = c->meshB_tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt2, 1));
  auto* labels2 = c->meshB_labels.as<int>(std::max<std::size_t>(nt2, 1));
  auto* parent2 = c->meshB_parent.as<std::uint32_t>(std::max<std::size_t>(nt2, 1));
  if (n) NM_CUDA(cudaMemcpyAsync(nodes2, d_nodes, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  NM_CUDA(cudaMemcpyAsync(d_count, &m, sizeof m, cudaMemcpyHostToDevice, st));
  if (m) nm::k_midpoints<<<grid_for(m, 256, c->sm_count * 8), 256, 0, st>>>(d_nodes, S, d_count, n, nodes2);
  if (nt)
    nm::k_emit_children<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(t4, nt, tmask, offs, d_labels, S, d_count, n,
                                                                             nodes2, reinterpret_cast<uint4*>(tets2),
                                                                             labels2, parent2);
  NM_CUDA(cudaGetLastError());
  launches += 3;
  return {n2, nt2};
}


#ifndef NM_CELL_AXIS
#define NM_CELL_AXIS 120
#endif
// Certified cells of every compartment (cells.cuh), built once per surface
// set from the surfaces alone, in four phases: geometry (grids + clusters),
// certification (level-1 cells and children, on the device), runs (x-runs of
// certified cells -> winding number, neighbour run or representative) and
// resolve (representatives evaluated by the sparse k_label, final codes).
// Host loops run one compartment per thread: every compartment's grid,
// blocks, runs and representatives are independent.
class CellBuild {
 public:
  // c->K, the centring frame, xyz64 / tri_idx on the device and hbox must be
  // set; prepare() may run on a host thread beside the tile packing (it uses
  // its own stream); finish() needs the tiles (representatives run k_label).
  CellBuild(nm_ctx* c, const double* xyz, const std::uint32_t* tri, const std::uint32_t* comp_off,
            const std::vector<float4>& hbox, cudaStream_t st)
      : c_(c), xyz_(xyz), tri_(tri), comp_off_(comp_off), hbox_(hbox), K_(c->K), ctr_{c->cx, c->cy, c->cz},
        st_(st), t0_(std::chrono::steady_clock::now()), tl_(t0_),
        verbose_(std::getenv("NM_CELL_VERBOSE") != nullptr) {}

  void prepare() {
    NM_CUDA(cudaSetDevice(c_->opt.device));
    geometry();
    certify();
    runs();
  }
  void finish() { resolve(); }

 private:
  // run value of a level-1 or child run: 0 / 1 known; kRep + r: the
  // compartment's local representative r; kRun + q: the value of the
  // compartment's level-1 run q; kLeft / kRight: the neighbour parent's run
  // (resolved once the row is scanned)
  static constexpr std::int64_t kUnknown = -1, kLeft = -2, kRight = -3, kRep = 1ll << 40, kRun = 1ll << 41;
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
  const int K_;
  const double ctr_[3];
  cudaStream_t st_;
  std::chrono::steady_clock::time_point t0_, tl_;
  bool verbose_;

  std::vector<nm::CellGrid> G_;
  std::vector<std::size_t> coff_;       // first cluster of each compartment
  std::size_t total_ = 0;               // level-1 cells
  std::unique_ptr<std::uint8_t[]> cert1_;
  std::unique_ptr<std::uint32_t[]> block_of_;  // local child block of each uncertified cell
  std::vector<std::size_t> boff_;       // first child block of each compartment
  std::size_t nchild_ = 0;
  std::unique_ptr<std::uint8_t[]> child_;
  std::vector<std::vector<double>> reps_;
  std::vector<std::vector<std::int64_t>> run_val_;
  std::unique_ptr<std::int32_t[]> run_of_;
  std::vector<std::vector<FineRun>> fine_;
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

  void lap(const char* what) {
    if (!verbose_) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cells] %-6s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tl_).count());
    tl_ = t;
  }
  // host arrays allocated uninitialised: every entry is written (by a copy or
  // by its compartment's thread) before it is read
  template <class T>
  static std::unique_ptr<T[]> uninit(std::size_t m) {
    return std::unique_ptr<T[]>(new T[std::max<std::size_t>(m, 1)]);
  }
  void up(DBuf& b, const void* src, std::size_t bytes) {
    void* d = b.get(std::max<std::size_t>(bytes, 1));
    if (bytes) NM_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st_));
  }
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
  void geometry() {
    const int K = K_;
    G_.assign(K, nm::CellGrid{});
    coff_.assign(K + 1, 0);
    std::vector<std::vector<float4>> clus_kv(K), tsph_kv(K);
    std::vector<std::vector<std::uint32_t>> ctri_kv(K);
    parallel_for(K, [&](int k) { compartment_geometry(k, clus_kv[k], ctri_kv[k], tsph_kv[k]); });
    std::vector<float4> clus, tsph;
    std::vector<std::uint32_t> ctri;
    for (int k = 0; k < K; ++k) {
      G_[k].off = static_cast<std::uint32_t>(total_);
      total_ += cells(k);
      if (total_ > 0xffffffffull) throw Error("certified-cell grids exceed 2^32 cells");
      coff_[k] = clus.size();
      clus.insert(clus.end(), clus_kv[k].begin(), clus_kv[k].end());
      ctri.insert(ctri.end(), ctri_kv[k].begin(), ctri_kv[k].end());
      tsph.insert(tsph.end(), tsph_kv[k].begin(), tsph_kv[k].end());
    }
    coff_[K] = clus.size();
    lap("setup");
    up(c_->clus, clus.data(), clus.size() * sizeof(float4));
    up(c_->clus_tri, ctri.data(), ctri.size() * sizeof(std::uint32_t));
    up(c_->clus_tsph, tsph.data(), tsph.size() * sizeof(float4));
  }

  void compartment_geometry(int k, std::vector<float4>& clus, std::vector<std::uint32_t>& ctri,
                            std::vector<float4>& tsph) {
    const double* ctr = ctr_;
    const double* xyz = xyz_;
    const std::uint32_t* tri = tri_;
    const std::uint32_t b = comp_off_[k], e = comp_off_[k + 1];
    nm::CellGrid g{0.0, 0.0, 0.0, 1.0, 0, 0, 0, 0u};
    if (e > b) {
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      std::vector<std::pair<std::uint32_t, std::uint32_t>> kk;
      kk.reserve(e - b);
      for (std::uint32_t t = b; t < e; ++t) {
        double m[3] = {0, 0, 0};
        for (int v = 0; v < 3; ++v)
          for (int a = 0; a < 3; ++a) {
            const double x = xyz[3 * std::size_t(tri[3 * t + v]) + a] - ctr[a];
            lo[a] = std::min(lo[a], x);
            hi[a] = std::max(hi[a], x);
            m[a] += x / 3.0;
          }
        std::uint32_t q[3];
        for (int a = 0; a < 3; ++a)
          q[a] = static_cast<std::uint32_t>(std::clamp((m[a] + ctr[a] - c_->lo[a]) / c_->span * 1024.0, 0.0, 1023.0));
        kk.emplace_back(spread10h(q[0]) | (spread10h(q[1]) << 1) | (spread10h(q[2]) << 2), t);
      }
      std::stable_sort(kk.begin(), kk.end(), [](auto& x, auto& y) { return x.first < y.first; });
      // bounding sphere of triangles kk[i0, i1) in the centred frame: fp32
      // centre of the vertex box, radius rounded up with the kernel's
      // margins (1e-6 relative + 1e-5 mm + 4e-6 |centre|)
      auto sphere = [&](std::size_t i0, std::size_t i1) {
        double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
        for (std::size_t i = i0; i < i1; ++i)
          for (int v = 0; v < 3; ++v)
            for (int a = 0; a < 3; ++a) {
              const double x = xyz[3 * std::size_t(tri[3 * kk[i].second + v]) + a] - ctr[a];
              blo[a] = std::min(blo[a], x);
              bhi[a] = std::max(bhi[a], x);
            }
        const float fc[3] = {float(0.5 * (blo[0] + bhi[0])), float(0.5 * (blo[1] + bhi[1])),
                             float(0.5 * (blo[2] + bhi[2]))};
        double rho = 0.0;
        for (std::size_t i = i0; i < i1; ++i)
          for (int v = 0; v < 3; ++v) {
            double d2 = 0.0;
            for (int a = 0; a < 3; ++a) {
              const double d = xyz[3 * std::size_t(tri[3 * kk[i].second + v]) + a] - ctr[a] - double(fc[a]);
              d2 += d * d;
            }
            rho = std::max(rho, std::sqrt(d2));
          }
        const double rel = 4e-6 * (std::fabs(fc[0]) + std::fabs(fc[1]) + std::fabs(fc[2]));
        return make_float4(fc[0], fc[1], fc[2], std::nextafter(float(rho * (1.0 + 1e-6) + 1e-5 + rel), INFINITY));
      };
      for (std::size_t i0 = 0; i0 < kk.size(); i0 += nm::kCluster) {
        const std::size_t i1 = std::min(kk.size(), i0 + nm::kCluster);
        clus.push_back(sphere(i0, i1));
        for (std::size_t i = i0; i < i0 + nm::kCluster; ++i) {
          ctri.push_back(i < i1 ? kk[i].second : 0xffffffffu);
          tsph.push_back(i < i1 ? sphere(i, i + 1) : make_float4(0.f, 0.f, 0.f, -1e30f));
        }
      }
      const double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
      g.B = std::max(ext / NM_CELL_AXIS, 1e-3);
      int n3[3];
      for (int a = 0; a < 3; ++a) n3[a] = static_cast<int>(std::ceil((hi[a] - lo[a]) / g.B)) + 2;
      g.ox = lo[0] - g.B;
      g.oy = lo[1] - g.B;
      g.oz = lo[2] - g.B;
      g.nx = n3[0];
      g.ny = n3[1];
      g.nz = n3[2];
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
    std::vector<std::size_t> sl_off(ns + 1, 0);  // global first block of each slab
    for (std::size_t i = 0; i < ns; ++i) sl_off[i + 1] = sl_off[i] + sl_cnt[i];
    boff_.assign(K + 1, 0);
    for (int k = 0; k <= K; ++k) boff_[k] = sl_off[slab_first_[k]];
    const std::size_t nblk = boff_[K];
    block_of_ = uninit<std::uint32_t>(total_);
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
    for (int k = 0; k < K; ++k) {
      const std::size_t nb = boff_[k + 1] - boff_[k];
      if (!nb) continue;
      nm::k_child_certify<<<static_cast<unsigned>((nb * 64 + 255) / 256), 256, 0, st_>>>(
          G_[k], static_cast<const std::uint32_t*>(c_->cell_blk.p) + boff_[k], nb, clus_k(k), nclus(k), ctri_k(k),
          tsph_k(k), static_cast<const double*>(c_->xyz64.p), static_cast<const std::uint32_t*>(c_->tri_idx.p), c_->cx,
          c_->cy, c_->cz, ch_d + boff_[k] * nm::kChildren);
    }
    NM_CUDA(cudaGetLastError());
    if (verbose_) {
      NM_CUDA(cudaStreamSynchronize(st_));
      lap("l2kern");
    }
    NM_CUDA(cudaMemcpyAsync(child_.get(), ch_d, nchild_, cudaMemcpyDeviceToHost, st_));
    NM_CUDA(cudaStreamSynchronize(st_));
    lap("l2");
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
    run_of_ = uninit<std::int32_t>(total_);
    parallel_for(static_cast<int>(ns), [&](int i) { slab_runs(slabs_[i], part[i]); });
    // merge: slab-local run / representative indices -> compartment-local
    std::vector<std::size_t> run_base(ns), rep_base(ns);
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
    });
    reps_.assign(K_, {});
    run_val_.assign(K_, {});
    fine_.assign(K_, {});
    parallel_for(K_, [&](int k) {
      for (std::size_t i = slab_first_[k]; i < slab_first_[k + 1]; ++i) {
        reps_[k].insert(reps_[k].end(), part[i].reps.begin(), part[i].reps.end());
        run_val_[k].insert(run_val_[k].end(), part[i].run_val.begin(), part[i].run_val.end());
        fine_[k].insert(fine_[k].end(), part[i].fine.begin(), part[i].fine.end());
      }
    });
    lap("runs");
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
            if (outside_dop(k, g.ox + (f + 0.5) * b, yy, zz) || outside_dop(k, g.ox + (e + 0.5) * b, yy, zz))
              v = 0;
            else
              v = new_rep(out, g.ox + ((f + e) / 2 + 0.5) * b, yy, zz);
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
    parallel_for(static_cast<int>(slabs_.size()), [&](int i) {
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
    });
    parallel_for(K, [&](int k) {  // fine runs write children of their own compartment only
      for (const FineRun& fr : fine_[k]) {
        const std::int64_t w = value(k, fr.v);
        if (w == kUnknown) continue;
        for (int f = fr.fx0; f <= fr.fx1; ++f) child_at(k, fr.row, f, fr.sy, fr.sz) = static_cast<std::uint8_t>(1 + w);
      }
    });
    lap("codes");
    up(c_->cell_state, code.get(), total_ * sizeof(std::uint32_t));
    up(c_->cell_child, child_.get(), nchild_);
    up(c_->cell_grids, G_.data(), G_.size() * sizeof(nm::CellGrid));
    NM_CUDA(cudaStreamSynchronize(st_));
    lap("final");
    c_->cells_total = total_ + nchild_;
    c_->cells_certified = 0;
    for (std::size_t q = 0; q < total_; ++q) c_->cells_certified += code[q] == 1 || code[q] == 2;
    for (std::size_t q = 0; q < nchild_; ++q) c_->cells_certified += child_[q] != 0;
    c_->cell_reps = nreps_;
    c_->cells = true;
    c_->ms_cells = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
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
    prm.tri = static_cast<const float4*>(c_->tri.p);
    prm.sub = static_cast<const float4*>(c_->sub.p);
    prm.edges = static_cast<const float4*>(c_->edges.p);
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


}  // namespace

extern "C" {

int nm_abi_version(void) { return NM_ABI_VERSION; }
const char* nm_last_error(void) { return g_err.c_str(); }

void nm_default_options(nm_options* o) {
  o->device = 0;
  o->tau = 1e-2f;
  o->delta_mm = 1e-3f;
  o->band = 1e-3;
  o->tie_eps = 1e-9;
  o->far_ratio = 4.0f;
  o->far_abs_mm = 0.05f;
  o->sort_points = 1;
  o->pairs_per_thread = 1;
  o->layout = 0;
  o->cull_outside = 0;
}

int nm_create(nm_ctx** out, const nm_options* opt) {
  return guarded([&] {
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    int ndev = 0;
    const cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      throw Error(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                  "); libnestmesh_label has no CPU fallback");
    auto* c = new nm_ctx;
    try {
      if (opt) c->opt = *opt;
      else nm_default_options(&c->opt);
      if (c->opt.device < 0 || c->opt.device >= ndev) throw Error("device ordinal out of range");
      if (c->opt.pairs_per_thread != 1 && c->opt.pairs_per_thread != 2) throw Error("pairs_per_thread must be 1 or 2");
      if (c->opt.layout < 0 || c->opt.layout > 2) throw Error("layout must be 0 (auto), 1 (triangles) or 2 (strips)");
      NM_CUDA(cudaSetDevice(c->opt.device));
      cudaDeviceProp p;
      NM_CUDA(cudaGetDeviceProperties(&p, c->opt.device));
      if (p.major != 10) throw Error(std::string("device ") + p.name + " is not sm_100 (Blackwell B200)");
      c->sm_count = p.multiProcessorCount;
      NM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      NM_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      for (auto& ev : c->ev) NM_CUDA(cudaEventCreate(&ev));
      NM_CUDA(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
      NM_CUDA(cudaMallocHost(&c->h_word, sizeof(std::uint32_t)));
      // result meshes are allocated from the device's default pool: keep
      // freed blocks reserved instead of returning them at every sync
      cudaMemPool_t pool;
      NM_CUDA(cudaDeviceGetDefaultMemPool(&pool, c->opt.device));
      std::uint64_t keep = ~0ull;
      NM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int nm_destroy(nm_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->opt.device);
    cudaStreamSynchronize(c->stream);
    delete c;
  });
}

int nm_set_surfaces(nm_ctx* c, const double* xyz, std::size_t nv, const std::uint32_t* tri, std::size_t nt,
                    const std::uint32_t* comp_off, int K, const int* label_ids) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (K < 1 || K > 32) throw Error("compartment count must be in [1, 32]");
    if (comp_off[0] != 0 || comp_off[K] != nt) throw Error("comp_tri_off must start at 0 and end at the triangle count");
    for (int k = 0; k < K; ++k) {
      if (comp_off[k + 1] < comp_off[k]) throw Error("comp_tri_off must be non-decreasing");
      if (label_ids[k] <= 0) throw Error("compartment label ids must be > 0 (0 is the bounding box)");
    }
    for (std::size_t i = 0; i < 3 * nt; ++i)
      if (tri[i] >= nv) throw Error("triangle index out of range");
    NM_CUDA(cudaSetDevice(c->opt.device));
    // Domain box and centring offset of the fp32 frame.
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (std::size_t i = 0; i < nv; ++i)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], xyz[3 * i + a]);
        hi[a] = std::max(hi[a], xyz[3 * i + a]);
      }
    if (nv == 0) lo[0] = lo[1] = lo[2] = hi[0] = hi[1] = hi[2] = 0.0;
    const double ctr[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-6}) * 1.5;
    for (int a = 0; a < 3; ++a) c->lo[a] = ctr[a] - 0.5 * span;
    c->span = span;
    c->cx = ctr[0];
    c->cy = ctr[1];
    c->cz = ctr[2];

    c->has_surfaces = false;
    c->cells = false;
    c->K = K;
    // fp64 originals (fix-up, cell certification) and the 13-DOP of every
    // compartment first: the certified-cell build (cull_outside = 2) starts on
    // its own host thread and stream while the tiles are packed below.
    auto up_on = [&](DBuf& b, const void* src, std::size_t bytes, cudaStream_t st) {
      void* d = b.get(bytes);
      if (bytes) NM_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st));
    };
    up_on(c->xyz64, xyz, nv * 3 * sizeof(double), c->side);
    up_on(c->tri_idx, tri, nt * 3 * sizeof(std::uint32_t), c->side);
    up_on(c->comp_off, comp_off, (K + 1) * sizeof(std::uint32_t), c->side);
    // 13-DOP: slab bounds over the vertices (centred frame), widened by 1e-3 mm
    // + 1e-5 |bound| (covers the fp32 rounding of the point and of the
    // projection in the kernel) and rounded outward.
    std::vector<float4> hbox(static_cast<std::size_t>(K) * nm::kDopF4);
    parallel_for(K, [&](int k) {
      float* dst = reinterpret_cast<float*>(&hbox[static_cast<std::size_t>(k) * nm::kDopF4]);
      for (int q = 0; q < 4 * nm::kDopF4; ++q) dst[q] = 0.0f;
      for (int j = 0; j < nm::kDopDirs; ++j) {
        double lo = 1e300, hi = -1e300;
        for (std::uint32_t t = comp_off[k]; t < comp_off[k + 1]; ++t)
          for (int v = 0; v < 3; ++v) {
            const double* X = xyz + 3 * std::size_t(tri[3 * t + v]);
            double pr = 0.0;
            for (int a = 0; a < 3; ++a) pr += double(nm::dop_dir(j, a)) * (X[a] - ctr[a]);
            lo = std::min(lo, pr);
            hi = std::max(hi, pr);
          }
        if (comp_off[k + 1] == comp_off[k]) {  // empty compartment: everything outside
          dst[2 * j] = 1e30f;
          dst[2 * j + 1] = -1e30f;
          continue;
        }
        const double m = 1e-3 + 1e-5 * std::max(std::fabs(lo), std::fabs(hi));
        dst[2 * j] = std::nextafter(float(lo - m), -INFINITY);
        dst[2 * j + 1] = std::nextafter(float(hi + m), INFINITY);
      }
    });
    std::unique_ptr<CellBuild> cells;
    std::exception_ptr cells_err;
    struct Joiner {
      std::thread t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } cells_thread;
    if (c->opt.cull_outside == 2) {
      cells = std::make_unique<CellBuild>(c, xyz, tri, comp_off, hbox, c->side);
      cells_thread.t = std::thread([&] {
        try {
          cells->prepare();
        } catch (...) {
          cells_err = std::current_exception();
        }
      });
    }

    auto morton = [&](const double* m) {
      std::uint32_t q[3];
      for (int a = 0; a < 3; ++a) {
        const double u = (m[a] - c->lo[a]) / span * 1024.0;
        q[a] = static_cast<std::uint32_t>(std::clamp(u, 0.0, 1023.0));
      }
      return spread10h(q[0]) | (spread10h(q[1]) << 1) | (spread10h(q[2]) << 2);
    };
    auto normal64 = [&](std::uint32_t t, double* N) {
      const double* A = xyz + 3 * std::size_t(tri[3 * t]);
      const double* B = xyz + 3 * std::size_t(tri[3 * t + 1]);
      const double* C = xyz + 3 * std::size_t(tri[3 * t + 2]);
      const double e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
      const double e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
      N[0] = e1[1] * e2[2] - e1[2] * e2[1];
      N[1] = e1[2] * e2[0] - e1[0] * e2[2];
      N[2] = e1[0] * e2[1] - e1[1] * e2[0];
    };

    // ---- strip decomposition --------------------------------
    // Segment = 8 consecutive strip triangles over 10 vertices; a strip's last
    // segment is padded with zero-normal triangles repeating its last vertex.
    // Segments are laid out in chunks of kGroups consecutive segments of one
    // strip (one chunk per 32-triangle subtile): full chunks first, in Morton
    // order of their centroids, then the strips' shorter tail chunks, also in
    // Morton order. Inside a subtile a segment that continues the previous one
    // (same strip, next 8 triangles) shares its first two vertices with the
    // previous segment's last two, so the far evaluator carries their
    // distances instead of recomputing them (bit-identical: same fp32 vertex,
    // same frame). cont bit = sidx * kGroups + j per tile.
    struct Seg {
      std::uint32_t v[nm::kSegTris + 2];
      std::int64_t t[nm::kSegTris];  // original triangle id, -1 = pad
      std::uint32_t strip, pos;      // strip id (within the compartment), segment index in the strip
    };
    std::vector<std::vector<Seg>> segs(K);
    std::size_t strip_slots = 0;
    const bool try_strips = c->opt.layout != 1;
    if (try_strips) {
      parallel_for(K, [&](int k) {
        const std::vector<Strip> strips = stripify(tri, comp_off[k], comp_off[k + 1]);
        struct Chunk {
          std::uint32_t key;
          bool full;
          std::size_t first, count;  // range in `all`
        };
        std::vector<Seg> all;
        std::vector<Chunk> chunks;
        for (std::uint32_t si = 0; si < strips.size(); ++si) {
          const Strip& st = strips[si];
          const std::size_t m = st.t.size();
          std::uint32_t pos = 0;
          for (std::size_t s0 = 0; s0 < m; s0 += nm::kSegTris, ++pos) {
            Seg g;
            for (int j = 0; j < nm::kSegTris + 2; ++j) g.v[j] = st.v[std::min(s0 + j, st.v.size() - 1)];
            for (int j = 0; j < nm::kSegTris; ++j) g.t[j] = s0 + j < m ? std::int64_t(st.t[s0 + j]) : -1;
            g.strip = si;
            g.pos = pos;
            if (pos % nm::kGroups == 0) chunks.push_back({0u, false, all.size(), 0});
            chunks.back().count++;
            all.push_back(g);
          }
        }
        for (Chunk& ch : chunks) {
          double cen[3] = {0, 0, 0};
          double w = 0;
          for (std::size_t q = ch.first; q < ch.first + ch.count; ++q)
            for (int j = 0; j < nm::kSegTris + 2; ++j, w += 1)
              for (int a = 0; a < 3; ++a) cen[a] += xyz[3 * std::size_t(all[q].v[j]) + a];
          for (double& x : cen) x /= w;
          ch.key = morton(cen);
          ch.full = ch.count == static_cast<std::size_t>(nm::kGroups);
        }
        std::stable_sort(chunks.begin(), chunks.end(), [](const Chunk& x, const Chunk& y) {
          return x.full != y.full ? x.full : x.key < y.key;
        });
        for (const Chunk& ch : chunks)
          for (std::size_t q = ch.first; q < ch.first + ch.count; ++q) segs[k].push_back(all[q]);
      });
      const std::size_t per_tile = nm::kTile / nm::kSegTris;
      for (int k = 0; k < K; ++k) strip_slots += (segs[k].size() + per_tile - 1) / per_tile * nm::kTile;
    }
    std::size_t soup_slots = 0;
    for (int k = 0; k < K; ++k) soup_slots += (comp_off[k + 1] - comp_off[k] + nm::kTile - 1) / nm::kTile * nm::kTile;
    // auto: strips when their padding costs less than the ~1.5x op saving
    const bool use_strips =
        c->opt.layout == 2 || (c->opt.layout == 0 && nt > 0 && strip_slots <= soup_slots + soup_slots / 4);

    std::vector<std::uint32_t> tiles(K + 1, 0);
    std::vector<std::vector<std::uint32_t>> order(K);
    for (int k = 0; k < K; ++k) {
      std::size_t units;
      if (use_strips) {
        units = (segs[k].size() * nm::kSegTris + nm::kTile - 1) / nm::kTile;
      } else {
        const std::uint32_t b = comp_off[k], e = comp_off[k + 1];
        std::vector<std::pair<std::uint32_t, std::uint32_t>> kk;
        kk.reserve(e - b);
        for (std::uint32_t t = b; t < e; ++t) {
          double m[3];
          for (int a = 0; a < 3; ++a)
            m[a] = (xyz[3 * tri[3 * t] + a] + xyz[3 * tri[3 * t + 1] + a] + xyz[3 * tri[3 * t + 2] + a]) / 3.0;
          kk.emplace_back(morton(m), t);
        }
        std::stable_sort(kk.begin(), kk.end(), [](auto& x, auto& y) { return x.first < y.first; });
        for (auto& p : kk) order[k].push_back(p.second);
        units = (e - b + nm::kTile - 1) / nm::kTile;
      }
      tiles[k + 1] = tiles[k] + static_cast<std::uint32_t>(units);
    }
    const std::size_t ntiles = tiles[K];
    const std::size_t npad = ntiles * nm::kTile;
    const int sub_f4 = use_strips ? (nm::kSub / nm::kSegTris) * nm::kSegF4 : nm::kSub * 3;
    const std::size_t tile_f4 = static_cast<std::size_t>(sub_f4) * nm::kSubPerTile;
    std::vector<float4> htri(ntiles * tile_f4);
    std::vector<float4> hsub(ntiles * nm::kSubPerTile * nm::kSubRec);
    std::vector<float4> hedge(use_strips ? ntiles * nm::kSubPerTile * nm::kGroups * nm::kEdgeF4 : 1);
    std::vector<std::uint32_t> hcont(std::max<std::size_t>(ntiles, 1), 0u);
    static_assert(nm::kSubPerTile * nm::kGroups <= 32, "continuation bits of a tile must fit a uint32");
    const double far_ratio = c->opt.far_ratio, far_abs = c->opt.far_abs_mm;
    // Each 32-triangle subtile carries an fp32 centre c (exactly representable
    // in the centred frame) and its vertices relative to c, so near-surface
    // geometry keeps ~ulp(radius) precision; the kernel forms p - c in
    // double-single per subtile.
    parallel_for(K, [&](int k) {  // compartments own disjoint tile ranges
      const std::size_t nreal = use_strips ? segs[k].size() : order[k].size();
      // fallback vertex for all-pad units: the compartment's first vertex
      const double* pad_v = comp_off[k + 1] > comp_off[k] ? xyz + 3 * std::size_t(tri[3 * comp_off[k]]) : ctr;
      for (std::uint32_t tl = tiles[k]; tl < tiles[k + 1]; ++tl) {
        for (int sidx = 0; sidx < nm::kSubPerTile; ++sidx) {
          // gather this subtile's vertices (centred frame, fp64)
          std::vector<const double*> srcv;
          const std::size_t u0 = static_cast<std::size_t>(tl - tiles[k]) * nm::kTile / (use_strips ? nm::kSegTris : 1) +
                                 sidx * (use_strips ? nm::kSub / nm::kSegTris : nm::kSub);
          const int nunits = use_strips ? nm::kSub / nm::kSegTris : nm::kSub;
          for (int j = 0; j < nunits; ++j) {
            const std::size_t u = u0 + j;
            if (use_strips) {
              for (int q = 0; q < nm::kSegTris + 2; ++q)
                srcv.push_back(u < nreal ? xyz + 3 * std::size_t(segs[k][u].v[q]) : pad_v);
            } else {
              const std::uint32_t t = u < nreal ? order[k][u] : 0;
              for (int q = 0; q < 3; ++q) srcv.push_back(u < nreal ? xyz + 3 * std::size_t(tri[3 * t + q]) : pad_v);
            }
          }
          double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
          for (const double* v : srcv)
            for (int a = 0; a < 3; ++a) {
              blo[a] = std::min(blo[a], v[a] - ctr[a]);
              bhi[a] = std::max(bhi[a], v[a] - ctr[a]);
            }
          const float fc[3] = {float(0.5 * (blo[0] + bhi[0])), float(0.5 * (blo[1] + bhi[1])),
                               float(0.5 * (blo[2] + bhi[2]))};
          double rho = 0.0;
          std::vector<float> rel(3 * srcv.size());
          for (std::size_t q = 0; q < srcv.size(); ++q) {
            for (int a = 0; a < 3; ++a) rel[3 * q + a] = float((srcv[q][a] - ctr[a]) - double(fc[a]));
            rho = std::max(rho, std::sqrt(double(rel[3 * q]) * rel[3 * q] + double(rel[3 * q + 1]) * rel[3 * q + 1] +
                                          double(rel[3 * q + 2]) * rel[3 * q + 2]));
          }
          float4* o = &htri[(static_cast<std::size_t>(tl) * nm::kSubPerTile + sidx) * sub_f4];
          for (int j = 0; j < nunits; ++j) {
            const std::size_t u = u0 + j;
            if (use_strips) {
              if (j > 0 && u < nreal && segs[k][u].strip == segs[k][u - 1].strip &&
                  segs[k][u].pos == segs[k][u - 1].pos + 1)
                hcont[tl] |= 1u << (sidx * nm::kGroups + j);
              float4* r = o + j * nm::kSegF4;
              double N[nm::kSegTris][3];
              for (int q = 0; q < nm::kSegTris; ++q) {
                if (u < nreal && segs[k][u].t[q] >= 0) normal64(static_cast<std::uint32_t>(segs[k][u].t[q]), N[q]);
                else N[q][0] = N[q][1] = N[q][2] = 0.0;
              }
              const float* rv = &rel[3 * (j * (nm::kSegTris + 2))];
              // vertices + |V|^2 (from the stored fp32 coordinates)
              for (int q = 0; q < nm::kSegTris + 2; ++q) {
                const double sv = double(rv[3 * q]) * rv[3 * q] + double(rv[3 * q + 1]) * rv[3 * q + 1] +
                                  double(rv[3 * q + 2]) * rv[3 * q + 2];
                r[q] = make_float4(2.0f * rv[3 * q], 2.0f * rv[3 * q + 1], 2.0f * rv[3 * q + 2], float(sv));
              }
              // (N_k, N_k . V_k) with the fp32 N the kernel multiplies by
              for (int q = 0; q < nm::kSegTris; ++q) {
                const float nf[3] = {float(N[q][0]), float(N[q][1]), float(N[q][2])};
                const double w = double(nf[0]) * rv[3 * q] + double(nf[1]) * rv[3 * q + 1] + double(nf[2]) * rv[3 * q + 2];
                // kRecScale (N, N.V): exact power-of-two scaling (vos.cuh seg_far)
                const float sc = nm::kRecScale;
                r[nm::kSegT + q] = make_float4(sc * nf[0], sc * nf[1], sc * nf[2], sc * float(w));
              }
              // -(vertex dot products) of each triangle (far evaluator, vos.cuh)
              auto dot3 = [&](int o, int i, int jj) {  // (v_i - v_o).(v_jj - v_o), fp64
                double acc = 0;
                for (int a = 0; a < 3; ++a)
                  acc += (double(rv[3 * i + a]) - double(rv[3 * o + a])) * (double(rv[3 * jj + a]) - double(rv[3 * o + a]));
                return acc;
              };
              float C[4 * (nm::kSegF4 - nm::kSegC)] = {0};
              for (int q = 0; q < nm::kSegTris; ++q) {
                const int ia = q, ib = q + 1, ic = q + 2;
                C[3 * q] = float(-dot3(ic, ia, ib));      // alpha at c
                C[3 * q + 1] = float(-dot3(ia, ib, ic));  // beta at a
                C[3 * q + 2] = float(-dot3(ib, ia, ic));  // gamma at b
              }
              for (int q = 0; q < nm::kSegF4 - nm::kSegC; ++q)
                r[nm::kSegC + q] = make_float4(C[4 * q], C[4 * q + 1], C[4 * q + 2], C[4 * q + 3]);
              // -|e|^2 of the consecutive (k,k+1) and skip (k,k+2) edges (near evaluator)
              float E[4 * nm::kEdgeF4] = {0};
              auto e2 = [&](int i, int jj) {
                double s2 = 0;
                for (int a = 0; a < 3; ++a) {
                  const double d = double(rv[3 * jj + a]) - double(rv[3 * i + a]);
                  s2 += d * d;
                }
                return float(-s2);
              };
              for (int q = 0; q <= nm::kSegTris; ++q) E[q] = e2(q, q + 1);
              for (int q = 0; q < nm::kSegTris; ++q) E[nm::kSegSkip + q] = e2(q, q + 2);
              float4* er = &hedge[((static_cast<std::size_t>(tl) * nm::kSubPerTile + sidx) * nm::kGroups + j) * nm::kEdgeF4];
              for (int q = 0; q < nm::kEdgeF4; ++q) er[q] = make_float4(E[4 * q], E[4 * q + 1], E[4 * q + 2], E[4 * q + 3]);
            } else {
              double N[3] = {0, 0, 0};
              if (u < nreal) normal64(order[k][u], N);
              const float* rv = &rel[9 * j];
              for (int q = 0; q < 3; ++q) o[3 * j + q] = make_float4(rv[3 * q], rv[3 * q + 1], rv[3 * q + 2], float(N[q]));
            }
          }
#ifndef NM_DIAG_SUBR
#define NM_DIAG_SUBR 1.0
#endif
          const double R = (far_ratio * rho * NM_DIAG_SUBR + far_abs) * (1.0 + 1e-5);
          float4* hs = &hsub[(static_cast<std::size_t>(tl) * nm::kSubPerTile + sidx) * nm::kSubRec];
          hs[0] = make_float4(fc[0], fc[1], fc[2], float(R * R));
          // spheres of the kGroups groups of kSegTris triangles, centres relative to fc
          const int per_group = static_cast<int>(srcv.size()) / nm::kGroups;
          for (int g = 0; g < nm::kGroups; ++g) {
            double glo[3] = {1e300, 1e300, 1e300}, ghi[3] = {-1e300, -1e300, -1e300};
            for (int q = g * per_group; q < (g + 1) * per_group; ++q)
              for (int a = 0; a < 3; ++a) {
                glo[a] = std::min(glo[a], double(rel[3 * q + a]));
                ghi[a] = std::max(ghi[a], double(rel[3 * q + a]));
              }
            const float gc[3] = {float(0.5 * (glo[0] + ghi[0])), float(0.5 * (glo[1] + ghi[1])),
                                 float(0.5 * (glo[2] + ghi[2]))};
            double rg = 0.0;
            for (int q = g * per_group; q < (g + 1) * per_group; ++q) {
              double d2 = 0.0;
              for (int a = 0; a < 3; ++a) d2 += (double(rel[3 * q + a]) - gc[a]) * (double(rel[3 * q + a]) - gc[a]);
              rg = std::max(rg, std::sqrt(d2));
            }
            // the kernel forms (p - c) - g in fp32: one more rounding, covered by the 1e-5 margin
            const double Rg = (far_ratio * rg + far_abs) * (1.0 + 1e-5);
            hs[1 + g] = make_float4(gc[0], gc[1], gc[2], float(Rg * Rg));
          }
        }
      }
    });
    c->strips = use_strips;
    auto up = [&](DBuf& b, const void* src, std::size_t bytes) { up_on(b, src, bytes, c->stream); };
    up(c->tri, htri.data(), htri.size() * sizeof(float4));
    up(c->sub, hsub.data(), hsub.size() * sizeof(float4));
    up(c->edges, hedge.data(), hedge.size() * sizeof(float4));
    up(c->cont, hcont.data(), hcont.size() * sizeof(std::uint32_t));
    up(c->comp_tiles, tiles.data(), tiles.size() * sizeof(std::uint32_t));
    up(c->comp_box, hbox.data(), hbox.size() * sizeof(float4));
    NM_CUDA(cudaStreamSynchronize(c->stream));
    if (cells_thread.t.joinable()) cells_thread.t.join();
    if (cells_err) std::rethrow_exception(cells_err);
    NM_CUDA(cudaStreamSynchronize(c->side));
    c->comp_tiles_h = tiles;
    c->n_continued = 0;
    for (std::uint32_t w : hcont) c->n_continued += static_cast<std::size_t>(__builtin_popcount(w));
    c->nt_real = nt;
    c->nt_pad = npad;
    c->nv = nv;
    for (int k = 0; k < 32; ++k) c->ids.id[k] = k < K ? label_ids[k] : 0;
    c->comp_off_h.assign(comp_off, comp_off + K + 1);
    c->has_surfaces = true;
    if (cells) cells->finish();  // representatives need the tiles: after the packing
  });
}

int nm_cell_info(nm_ctx* c, uint64_t* cells, uint64_t* certified, uint64_t* reps, double* ms_build,
                 uint64_t* last_pairs, uint64_t* last_evals) {
  return guarded([&] {
    require_surfaces(c);
    if (cells) *cells = c->cells_total;
    if (certified) *certified = c->cells_certified;
    if (reps) *reps = c->cell_reps;
    if (ms_build) *ms_build = c->ms_cells;
    if (last_pairs) *last_pairs = c->sparse_pairs;
    if (last_evals) *last_evals = c->sparse_evals;
  });
}

int nm_surface_segments(nm_ctx* c, std::size_t* segments, std::size_t* continued) {
  return guarded([&] {
    require_surfaces(c);
    if (segments) *segments = c->strips ? c->nt_pad / nm::kSegTris : 0;
    if (continued) *continued = c->strips ? c->n_continued : 0;
  });
}

int nm_surface_info(nm_ctx* c, int* K, std::size_t* triangles, std::size_t* padded, int* layout) {
  return guarded([&] {
    require_surfaces(c);
    if (K) *K = c->K;
    if (triangles) *triangles = c->nt_real;
    if (padded) *padded = c->nt_pad;
    if (layout) *layout = c->strips ? 2 : 1;
  });
}

int nm_label_nodes_shard_device(nm_ctx* c, const double* d_pts, std::size_t n, double T, std::uint32_t* d_masks,
                                int shard, int nshards, void* stream, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    if (nshards < 1 || shard < 0 || shard >= nshards) throw Error("shard must lie in [0, nshards)");
    NM_CUDA(cudaSetDevice(c->opt.device));
    label_nodes_dev(c, d_pts, n, T, d_masks, nullptr, c->pick(stream), stats, nullptr, false, shard, nshards);
  });
}

int nm_label_nodes_device(nm_ctx* c, const double* d_pts, std::size_t n, double T, std::uint32_t* d_masks,
                          double* d_s, void* stream, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    NM_CUDA(cudaSetDevice(c->opt.device));
    label_nodes_dev(c, d_pts, n, T, d_masks, d_s, c->pick(stream), stats);
  });
}

int nm_label_tets_device(nm_ctx* c, const std::uint32_t* d_tets, std::size_t nt, const std::uint32_t* d_masks,
                         int* d_labels, void* stream, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    NM_CUDA(cudaSetDevice(c->opt.device));
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, c->pick(stream), stats);
  });
}

int nm_flag_boundary_device(nm_ctx* c, const std::uint32_t* d_tets, std::size_t nt, const std::uint32_t* d_masks,
                            std::uint32_t active, std::uint32_t* d_ids, std::uint32_t* d_count, void* stream) {
  return guarded([&] {
    require_surfaces(c);
    NM_CUDA(cudaSetDevice(c->opt.device));
    std::uint64_t l = 0;
    select(c, nm::PredStraddle{reinterpret_cast<const uint4*>(d_tets), d_masks, active}, nt, d_ids, d_count,
           c->pick(stream), l);
  });
}

int nm_label_nodes(nm_ctx* c, const double* pts, std::size_t n, double T, std::uint32_t* masks_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    NM_CUDA(cudaSetDevice(c->opt.device));
    auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n, 1));
    if (n) NM_CUDA(cudaMemcpyAsync(d_pts, pts, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    label_nodes_dev(c, d_pts, n, T, d_masks, nullptr, c->stream, stats);
    if (n) NM_CUDA(cudaMemcpyAsync(masks_out, d_masks, n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nm_enclosure(nm_ctx* c, const double* pts, std::size_t n, double T, double* s_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    NM_CUDA(cudaSetDevice(c->opt.device));
    auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n, 1));
    auto* d_s = c->s_out.as<double>(std::max<std::size_t>(n * c->K, 1));
    if (n) NM_CUDA(cudaMemcpyAsync(d_pts, pts, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    label_nodes_dev(c, d_pts, n, T, d_masks, d_s, c->stream, stats);
    if (n) NM_CUDA(cudaMemcpyAsync(s_out, d_s, n * c->K * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nm_label_tets(nm_ctx* c, const std::uint32_t* tets, std::size_t nt, const std::uint32_t* masks,
                  std::size_t n_nodes, int* labels_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    if (nt && !tets) throw Error("null tets");
    NM_CUDA(cudaSetDevice(c->opt.device));
    if (stats) std::memset(stats, 0, sizeof *stats);
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n_nodes, 1));
    auto* d_labels = c->labels.as<int>(std::max<std::size_t>(nt, 1));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, c->stream));
    check_tets_device(c, d_tets, tets, nt, n_nodes, c->stream);
    if (n_nodes) NM_CUDA(cudaMemcpyAsync(d_masks, masks, n_nodes * sizeof(std::uint32_t), cudaMemcpyHostToDevice, c->stream));
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, c->stream, stats);
    if (nt) NM_CUDA(cudaMemcpyAsync(labels_out, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// Full mesh from host buffers. The node pass is enqueued first; the tet
// upload and its index validation (k_max_index) run on the side stream
// underneath it, so neither the 16 B/tet copy nor the check sits on the
// critical path. A bad index is reported with the host scan's message.
int nm_label_mesh(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, double T,
                  int* labels_out, std::uint32_t* masks_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    if (nt && !tets) throw Error("null tets");
    if (nt && n == 0) check_tets(tets, nt, n);
    NM_CUDA(cudaSetDevice(c->opt.device));
    auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n, 1));
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_labels = c->labels.as<int>(std::max<std::size_t>(nt, 1));
    auto* d_word = c->word.as<std::uint32_t>(1);
    if (n) NM_CUDA(cudaMemcpyAsync(d_pts, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    // tet upload + index validation on the side stream, enqueued first so it
    // runs under the whole node pass (which may synchronise the host once,
    // for the sparse grid of certified-cell culling)
    if (nt) {
      NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, c->side));
      NM_CUDA(cudaMemsetAsync(d_word, 0, sizeof(std::uint32_t), c->side));
      nm::k_max_index<<<grid_for(nt, 256, c->sm_count * 8), 256, 0, c->side>>>(reinterpret_cast<const uint4*>(d_tets),
                                                                               nt, d_word);
      NM_CUDA(cudaGetLastError());
      NM_CUDA(cudaMemcpyAsync(c->h_word, d_word, sizeof(std::uint32_t), cudaMemcpyDeviceToHost, c->side));
      NM_CUDA(cudaEventRecord(c->ev_side, c->side));
    }
    label_nodes_dev(c, d_pts, n, T, d_masks, nullptr, c->stream, stats, nullptr, /*stats_deferred=*/true);
    if (nt) {
      NM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_side, 0));
      NM_CUDA(cudaEventSynchronize(c->ev_side));
      if (*c->h_word >= n) {
        NM_CUDA(cudaStreamSynchronize(c->stream));
        check_tets(tets, nt, n);  // throws with the offending tet
      }
    }
    if (stats && n) read_node_stats(c, n, c->stream, stats);
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, c->stream, stats);
    if (nt) NM_CUDA(cudaMemcpyAsync(labels_out, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (masks_out && n)
      NM_CUDA(cudaMemcpyAsync(masks_out, d_masks, n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"

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
      if (nm_create(&c, &o) != 0) throw Error(g_err);
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
      if (nm_set_surfaces(c, xyz, nv, tri, nt, comp_off, K, label_ids) != 0) throw Error(g_err);
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

struct nm_boundary {
  std::vector<std::uint32_t> tri;    // 3 per triangle, outward from the region, lexicographically sorted
  std::vector<std::uint32_t> nodes;  // sorted, unique
};

// Device-resident result mesh: fresh device arrays owned by the handle,
// filled by device-to-device copies (~3 TB/s, so the context keeps its
// grown scratch buffers for the next call); nm_mesh_copy reads them straight
// into the caller's arrays. parent == nullptr: identity (no refinement).
nm_mesh* make_device_mesh(nm_ctx* c, const DBuf& nodes, const DBuf& tets, const DBuf& labels, const DBuf* parent,
                          const DBuf* masks, std::size_t nn, std::size_t nt, std::size_t n_old, cudaStream_t st) {
  std::unique_ptr<nm_mesh> m(new nm_mesh);
  m->n_old = n_old;
  m->dev.device = c->opt.device;
  m->dev.nn = nn;
  m->dev.nt = nt;
  // stream-ordered pool allocations (nm_create keeps the pool's memory
  // reserved), so repeated calls do not pay cudaMalloc/cudaFree
  auto dup = [&](void*& dst, const void* src, std::size_t bytes) {
    NM_CUDA(cudaMallocAsync(&dst, std::max<std::size_t>(bytes, 256), st));
    if (bytes) NM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  };
  dup(m->dev.nodes, nodes.p, 3 * nn * sizeof(double));
  dup(m->dev.tets, tets.p, 4 * nt * sizeof(std::uint32_t));
  dup(m->dev.labels, labels.p, nt * sizeof(int));
  if (parent) {
    dup(m->dev.parent, parent->p, nt * sizeof(std::uint32_t));
  } else {
    NM_CUDA(cudaMallocAsync(&m->dev.parent, std::max<std::size_t>(nt * sizeof(std::uint32_t), 256), st));
    if (nt) {
      nm::k_iota<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(static_cast<std::uint32_t*>(m->dev.parent), nt);
      NM_CUDA(cudaGetLastError());
    }
  }
  if (masks) dup(m->dev.masks, masks->p, nn * sizeof(std::uint32_t));
  NM_CUDA(cudaStreamSynchronize(st));
  return m.release();
}

extern "C" {

int nm_extract_boundary(nm_ctx* c, const std::uint32_t* tets, std::size_t nt, const int* labels, const int* label_set,
                        int n_set, nm_boundary** out) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    if (n_set < 1 || n_set > 32) throw Error("label set size must be in [1, 32]");
    if (4 * nt > 0xffffffffull) throw Error("mesh too large for 32-bit face ids");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    const std::size_t m = 4 * nt;
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_labels = c->labels.as<int>(std::max<std::size_t>(nt, 1));
    auto* d_region = c->region.as<std::uint8_t>(std::max<std::size_t>(nt, 1));
    auto* d_nbr = c->nbr.as<std::int32_t>(std::max<std::size_t>(m, 1));
    auto* d_count = c->count.as<std::uint32_t>(4);
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_labels, labels, nt * sizeof(int), cudaMemcpyHostToDevice, st));
    nm::LabelIds set{};
    for (int k = 0; k < n_set; ++k) set.id[k] = label_set[k];
    const uint4* t4 = reinterpret_cast<const uint4*>(d_tets);
    std::uint32_t in_count = 0;
    if (nt) {
      nm::k_region<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(d_labels, nt, set, n_set, d_region);
      std::uint64_t l = 0;
      select(c, PredByte{d_region}, nt, c->list.as<std::uint32_t>(nt), d_count, st, l);
      NM_CUDA(cudaMemcpyAsync(&in_count, d_count, sizeof in_count, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
    }
    if (n_set == 1 && in_count == 0)
      throw Error("UnknownLabel: no tetrahedron carries label " + std::to_string(label_set[0]) + " (mesh.hpp:21-24)");
    face_adjacency(c, t4, nt, d_nbr, st);
    auto* faces = c->bfaces.as<std::uint32_t>(std::max<std::size_t>(m, 1));
    std::uint64_t l = 0;
    select(c, nm::PredBoundaryFace{d_nbr, d_region}, m, faces, d_count, st, l);
    std::uint32_t nb = 0;
    NM_CUDA(cudaMemcpyAsync(&nb, d_count, sizeof nb, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    auto* tri = c->btri.as<std::uint32_t>(6 * std::max<std::size_t>(nb, 1));
    std::uint32_t *t0 = tri, *t1 = tri + nb, *t2 = tri + 2 * nb, *sorted = tri + 3 * nb;
    std::unique_ptr<nm_boundary> res(new nm_boundary);
    if (nb) {
      nm::k_face_tris<<<grid_for(nb, 256, c->sm_count * 8), 256, 0, st>>>(t4, faces, nb, t0, t1, t2);
      const std::uint32_t* order = lex_order3(c, t0, t1, t2, nb, st);
      nm::k_gather_tris<<<grid_for(nb, 256, c->sm_count * 8), 256, 0, st>>>(order, nb, t0, t1, t2, sorted);
      NM_CUDA(cudaGetLastError());
      res->tri.resize(3 * std::size_t(nb));
      NM_CUDA(cudaMemcpyAsync(res->tri.data(), sorted, 3 * std::size_t(nb) * sizeof(std::uint32_t),
                              cudaMemcpyDeviceToHost, st));
      // sorted unique node ids
      auto* ids = c->keys.as<std::uint32_t>(3 * std::size_t(nb));
      auto* ids2 = c->keys_alt.as<std::uint32_t>(3 * std::size_t(nb));
      NM_CUDA(cudaMemcpyAsync(ids, t0, 3 * std::size_t(nb) * sizeof(std::uint32_t), cudaMemcpyDeviceToDevice, st));
      cub::DoubleBuffer<std::uint32_t> kb(ids, ids2);
      std::size_t tmp = 0;
      NM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kb, static_cast<int>(3 * nb), 0, 32, st));
      void* tp = c->cub_tmp.get(tmp);
      NM_CUDA(cub::DeviceRadixSort::SortKeys(tp, tmp, kb, static_cast<int>(3 * nb), 0, 32, st));
      const std::uint32_t* sk = kb.Current();
      auto* uidx = c->frontier.as<std::uint32_t>(3 * std::size_t(nb));
      select(c, nm::PredUniqueU32{sk}, 3 * std::size_t(nb), uidx, d_count, st, l);
      std::uint32_t nu = 0;
      NM_CUDA(cudaMemcpyAsync(&nu, d_count, sizeof nu, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
      auto* un = c->order_alt.as<std::uint32_t>(std::max<std::uint32_t>(nu, 1));
      nm::k_gather_key<<<grid_for(std::max<std::uint32_t>(nu, 1), 256, c->sm_count * 8), 256, 0, st>>>(sk, uidx, nu, un);
      res->nodes.resize(nu);
      if (nu) NM_CUDA(cudaMemcpyAsync(res->nodes.data(), un, nu * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    }
    NM_CUDA(cudaStreamSynchronize(st));
    *out = res.release();
  });
}

int nm_boundary_sizes(const nm_boundary* b, std::size_t* n_tri, std::size_t* n_nodes) {
  if (!b) return 1;
  if (n_tri) *n_tri = b->tri.size() / 3;
  if (n_nodes) *n_nodes = b->nodes.size();
  return 0;
}

int nm_boundary_copy(const nm_boundary* b, std::uint32_t* tri, std::uint32_t* nodes) {
  if (!b) return 1;
  if (tri && !b->tri.empty()) std::memcpy(tri, b->tri.data(), b->tri.size() * sizeof(std::uint32_t));
  if (nodes && !b->nodes.empty()) std::memcpy(nodes, b->nodes.data(), b->nodes.size() * sizeof(std::uint32_t));
  return 0;
}

void nm_boundary_free(nm_boundary* b) { delete b; }

int nm_lattice_device(nm_ctx* c, const double* origin, double h, int nx, int ny, int nz, double* d_nodes,
                      std::uint32_t* d_tets, void* stream) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (!(h > 0.0)) throw Error("lattice cell size must be > 0 (lattice.hpp:19)");
    if (nx < 1 || ny < 1 || nz < 1) throw Error("lattice cell counts must be >= 1 (lattice.hpp:20)");
    const std::size_t nn = static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1);
    const std::size_t cells = static_cast<std::size_t>(nx) * ny * nz;
    if (nn > 0xffffffffull || 5 * cells > 0xffffffffull) throw Error("lattice exceeds 32-bit ids");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->pick(stream);
    nm::k_lattice_nodes<<<grid_for(nn, 256, c->sm_count * 32), 256, 0, st>>>(origin[0], origin[1], origin[2], h, nx, ny,
                                                                            nz, d_nodes);
    nm::k_lattice_tets<<<grid_for(cells, 128, c->sm_count * 32), 128, 0, st>>>(d_nodes, nx, ny, nz,
                                                                             reinterpret_cast<uint4*>(d_tets));
    NM_CUDA(cudaGetLastError());
  });
}

int nm_label_lattice(nm_ctx* c, const double* origin, double h, int nx, int ny, int nz, double T, int* labels_out,
                     std::uint32_t* masks_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    const std::size_t nn = static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1);
    const std::size_t nt = 5ull * nx * ny * nz;
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    auto* d_nodes = c->pts.as<double>(3 * nn);
    auto* d_tets = c->tets.as<std::uint32_t>(4 * nt);
    auto* d_masks = c->masks.as<std::uint32_t>(nn);
    auto* d_labels = c->labels.as<int>(nt);
    if (nm_lattice_device(c, origin, h, nx, ny, nz, d_nodes, d_tets, st) != 0) throw Error(g_err);
    label_nodes_dev(c, d_nodes, nn, T, d_masks, nullptr, st, stats);
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, st, stats);
    if (labels_out) NM_CUDA(cudaMemcpyAsync(labels_out, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (masks_out) NM_CUDA(cudaMemcpyAsync(masks_out, d_masks, nn * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
  });
}

int nm_point_surface_distance(nm_ctx* c, const double* pts, std::size_t n, const double* xyz, std::size_t nv,
                              const std::uint32_t* tri, std::size_t nt, double* dist_out, nm_stats* stats) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (nt == 0) throw Error("target surface has no triangle (SPEC.md:429 pre: both non-empty)");
    for (std::size_t i = 0; i < 3 * nt; ++i)
      if (tri[i] >= nv) throw Error("triangle index out of range");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    if (stats) std::memset(stats, 0, sizeof *stats);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (std::size_t v = 0; v < nv; ++v)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], xyz[3 * v + a]);
        hi[a] = std::max(hi[a], xyz[3 * v + a]);
      }
    const double ctr[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-6}) * 1.5;
    auto morton = [&](const double* m) {  // 30-bit key in the centred frame (spread10h)
      std::uint32_t q[3];
      for (int a = 0; a < 3; ++a)
        q[a] = static_cast<std::uint32_t>(std::clamp((m[a] - ctr[a]) / span * 1024.0 + 512.0, 0.0, 1023.0));
      return spread10h(q[0]) | (spread10h(q[1]) << 1) | (spread10h(q[2]) << 2);
    };
    // clusters of kDistCluster triangles in Morton order of their centroids,
    // each with a bounding sphere (the last cluster padded by repeating a
    // triangle, which cannot change a minimum)
    std::vector<std::pair<std::uint32_t, std::uint32_t>> kk(nt);
    for (std::size_t t = 0; t < nt; ++t) {
      double m[3] = {0, 0, 0};
      for (int k = 0; k < 3; ++k)
        for (int a = 0; a < 3; ++a) m[a] += xyz[3 * std::size_t(tri[3 * t + k]) + a] / 3.0;
      kk[t] = {morton(m), static_cast<std::uint32_t>(t)};
    }
    std::stable_sort(kk.begin(), kk.end(), [](auto& x, auto& y) { return x.first < y.first; });
    const std::size_t nclus = (nt + nm::kDistCluster - 1) / nm::kDistCluster;
    std::vector<float4> h32(3 * nclus * nm::kDistCluster), hclus(nclus);
    std::vector<std::uint32_t> hslot(nclus * nm::kDistCluster);
    for (std::size_t q = 0; q < nclus; ++q) {
      double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
      for (int k = 0; k < nm::kDistCluster; ++k) {
        const std::size_t slot = q * nm::kDistCluster + k;
        const std::uint32_t t = kk[std::min(slot, nt - 1)].second;
        hslot[slot] = t;
        for (int v = 0; v < 3; ++v) {
          const double* X = xyz + 3 * std::size_t(tri[3 * t + v]);
          h32[3 * slot + v] = make_float4(float(X[0] - ctr[0]), float(X[1] - ctr[1]), float(X[2] - ctr[2]), 0.0f);
          for (int a = 0; a < 3; ++a) {
            blo[a] = std::min(blo[a], X[a] - ctr[a]);
            bhi[a] = std::max(bhi[a], X[a] - ctr[a]);
          }
        }
      }
      const float fc[3] = {float(0.5 * (blo[0] + bhi[0])), float(0.5 * (blo[1] + bhi[1])), float(0.5 * (blo[2] + bhi[2]))};
      double rho = 0.0;
      for (int k = 0; k < nm::kDistCluster; ++k)
        for (int v = 0; v < 3; ++v) {
          const double* X = xyz + 3 * std::size_t(tri[3 * hslot[q * nm::kDistCluster + k] + v]);
          double d2 = 0.0;
          for (int a = 0; a < 3; ++a) d2 += (X[a] - ctr[a] - fc[a]) * (X[a] - ctr[a] - fc[a]);
          rho = std::max(rho, std::sqrt(d2));
        }
      hclus[q] = make_float4(fc[0], fc[1], fc[2], std::nextafter(float(rho * (1.0 + 1e-6) + 1e-5), INFINITY));
    }
    // evaluation order of the points: Morton (coherent warps), results by index
    std::vector<std::pair<std::uint32_t, std::uint32_t>> pk(n);
    for (std::size_t i = 0; i < n; ++i) pk[i] = {morton(pts + 3 * i), static_cast<std::uint32_t>(i)};
    std::stable_sort(pk.begin(), pk.end(), [](auto& x, auto& y) { return x.first < y.first; });
    std::vector<std::uint32_t> hord(std::max<std::size_t>(n, 1));
    for (std::size_t i = 0; i < n; ++i) hord[i] = pk[i].second;
    auto* d_t32 = c->dist_tri.as<float4>(h32.size());
    auto* d_clus = c->dist_clus.as<float4>(nclus);
    auto* d_slot = c->dist_slot.as<std::uint32_t>(hslot.size());
    auto* d_ord = c->dist_ord.as<std::uint32_t>(hord.size());
    auto* d_xyz = c->dist_xyz.as<double>(3 * std::max<std::size_t>(nv, 1));
    auto* d_idx = c->dist_idx.as<std::uint32_t>(3 * nt);
    auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_d32 = c->dist_d32.as<float>(std::max<std::size_t>(n, 1));
    auto* d_out = c->dist_out.as<double>(std::max<std::size_t>(n, 1));
    auto* counters = c->counters.as<unsigned long long>(8);
    NM_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), st));
    NM_CUDA(cudaMemcpyAsync(d_t32, h32.data(), h32.size() * sizeof(float4), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemcpyAsync(d_xyz, xyz, 3 * nv * sizeof(double), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemcpyAsync(d_idx, tri, 3 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemcpyAsync(d_clus, hclus.data(), nclus * sizeof(float4), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemcpyAsync(d_slot, hslot.data(), hslot.size() * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemcpyAsync(d_ord, hord.data(), hord.size() * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (n) NM_CUDA(cudaMemcpyAsync(d_pts, pts, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaStreamSynchronize(st));  // h32 is released at scope exit
    if (n) {
      nm::DistParams prm{d_pts, n,      d_ord,  d_t32,  d_slot, d_clus, static_cast<int>(nclus), d_xyz,
                         d_idx, ctr[0], ctr[1], ctr[2], d_d32,  d_out,  counters};
      if (stats) NM_CUDA(cudaEventRecord(c->ev[0], st));
      const unsigned grid = static_cast<unsigned>((n + 255) / 256);
      nm::k_point_surface_distance<1><<<grid, 256, 0, st>>>(prm);
      nm::k_point_surface_distance<2><<<grid, 256, 0, st>>>(prm);
      NM_CUDA(cudaGetLastError());
      if (stats) NM_CUDA(cudaEventRecord(c->ev[1], st));
      NM_CUDA(cudaMemcpyAsync(dist_out, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    NM_CUDA(cudaStreamSynchronize(st));
    if (stats && n) {
      unsigned long long h[8];
      NM_CUDA(cudaMemcpy(h, counters, sizeof h, cudaMemcpyDeviceToHost));
      stats->points = n;
      stats->triangles = nt;
      stats->evals = 2ull * n * nt;
      stats->flagged_pairs = h[4];  // fp64 candidate evaluations
      stats->far_subtiles = h[5];   // pass-1 cluster visits (of n x clusters)
      stats->launches = 2;
      NM_CUDA(cudaEventElapsedTime(&stats->ms_label, c->ev[0], c->ev[1]));
    }
  });
}

int nm_label_centroids(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt,
                       double T, int* labels_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    check_tets(tets, nt, n);
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    auto* d_nodes = c->meshA_nodes.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_cen = c->pts.as<double>(3 * std::max<std::size_t>(nt, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
    auto* d_labels = c->labels.as<int>(std::max<std::size_t>(nt, 1));
    if (n) NM_CUDA(cudaMemcpyAsync(d_nodes, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (nt)
      nm::k_centroids<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(d_nodes, reinterpret_cast<const uint4*>(d_tets),
                                                                          nt, d_cen);
    label_nodes_dev(c, d_cen, nt, T, d_masks, nullptr, st, stats);
    if (nt) {
      nm::k_mask_labels<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(d_masks, nt, d_labels, c->ids);
      NM_CUDA(cudaGetLastError());
      NM_CUDA(cudaMemcpyAsync(labels_out, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, st));
    }
    NM_CUDA(cudaStreamSynchronize(st));
  });
}

int nm_flag_boundary(nm_ctx* c, const std::uint32_t* tets, std::size_t nt, const std::uint32_t* masks,
                     std::size_t n_nodes, std::uint32_t active, std::uint32_t* ids_out, std::size_t* count) {
  return guarded([&] {
    require_surfaces(c);
    check_tets(tets, nt, n_nodes);
    NM_CUDA(cudaSetDevice(c->opt.device));
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n_nodes, 1));
    auto* d_ids = c->list.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
    auto* d_count = c->count.as<std::uint32_t>(4);
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, c->stream));
    if (n_nodes) NM_CUDA(cudaMemcpyAsync(d_masks, masks, n_nodes * sizeof(std::uint32_t), cudaMemcpyHostToDevice, c->stream));
    std::uint64_t l = 0;
    select(c, nm::PredStraddle{reinterpret_cast<const uint4*>(d_tets), d_masks, active}, nt, d_ids, d_count, c->stream, l);
    std::uint32_t hc = 0;
    NM_CUDA(cudaMemcpyAsync(&hc, d_count, sizeof hc, cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
    if (hc) NM_CUDA(cudaMemcpy(ids_out, d_ids, hc * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    *count = hc;
  });
}

int nm_relabel(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, double T,
               int max_iters, int* labels_io, int* passes, int* converged, std::uint8_t* evaluated, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    check_tets(tets, nt, n);
    if (n > 0xffffffffull || 4 * nt > 0xffffffffull) throw Error("mesh too large for 32-bit face ids");
    if (max_iters < 1) throw Error("max_iters must be >= 1");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    if (stats) std::memset(stats, 0, sizeof *stats);
    const std::size_t m = 4 * nt;
    auto* d_pts = c->pts.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_tets = c->tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_labels = c->labels.as<int>(std::max<std::size_t>(nt, 1));
    auto* d_masks = c->masks.as<std::uint32_t>(std::max<std::size_t>(n, 1));
    auto* d_known = c->known.as<std::uint8_t>(std::max<std::size_t>(n, 1));
    auto* d_want = c->want.as<std::uint8_t>(std::max<std::size_t>(n, 1));
    auto* d_nbr = c->nbr.as<std::int32_t>(std::max<std::size_t>(m, 1));
    auto* d_list = c->frontier.as<std::uint32_t>(std::max<std::size_t>(n, 1));  // frontier node ids
    auto* d_count = c->count.as<std::uint32_t>(4);
    auto* counters = c->counters.as<unsigned long long>(8);
    if (n) NM_CUDA(cudaMemcpyAsync(d_pts, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_labels, labels_io, nt * sizeof(int), cudaMemcpyHostToDevice, st));
    NM_CUDA(cudaMemsetAsync(d_known, 0, std::max<std::size_t>(n, 1), st));
    NM_CUDA(cudaMemsetAsync(d_masks, 0, std::max<std::size_t>(n, 1) * sizeof(std::uint32_t), st));
    const uint4* t4 = reinterpret_cast<const uint4*>(d_tets);
    face_adjacency(c, t4, nt, d_nbr, st);
    c->flag_cap = std::max<std::size_t>(n, 1);
    int pass = 0;
    *converged = 0;
    std::uint64_t evaluated_total = 0;
    for (pass = 1; pass <= max_iters; ++pass) {
      NM_CUDA(cudaMemsetAsync(d_want, 0, std::max<std::size_t>(n, 1), st));
      if (nt) nm::k_frontier<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(t4, nt, d_nbr, d_labels, d_want);
      std::uint64_t l = 0;
      select(c, nm::PredWantNew{d_want, d_known}, n, d_list, d_count, st, l);
      std::uint32_t todo = 0;
      NM_CUDA(cudaMemcpyAsync(&todo, d_count, sizeof todo, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
      if (todo) {
        nm_stats s{};
        label_nodes_dev(c, d_pts, todo, T, d_masks, nullptr, st, stats ? &s : nullptr, d_list);
        if (stats) {
          stats->points += s.points;
          stats->evals += s.evals;
          stats->flagged_points += s.flagged_points;
          stats->flagged_pairs += s.flagged_pairs;
          stats->ties += s.ties;
          stats->near_subtiles += s.near_subtiles;
          stats->far_subtiles += s.far_subtiles;
          stats->ms_label += s.ms_label;
          stats->ms_fixup += s.ms_fixup;
        }
        NM_CUDA(cudaMemcpyAsync(d_count, &todo, sizeof todo, cudaMemcpyHostToDevice, st));
        nm::k_mark_known<<<grid_for(todo, 256, c->sm_count * 8), 256, 0, st>>>(d_list, d_count, d_known);
        evaluated_total += todo;
      }
      NM_CUDA(cudaMemsetAsync(counters + 7, 0, sizeof(unsigned long long), st));
      if (nt)
        nm::k_relabel_tets<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(t4, nt, d_masks, d_known, d_labels,
                                                                               c->ids, counters + 7);
      unsigned long long changed = 0;
      NM_CUDA(cudaMemcpyAsync(&changed, counters + 7, sizeof changed, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
      if (changed == 0) {
        *converged = 1;
        break;
      }
    }
    *passes = std::min(pass, max_iters);
    if (nt) NM_CUDA(cudaMemcpyAsync(labels_io, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (evaluated && n) NM_CUDA(cudaMemcpyAsync(evaluated, d_known, n, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      stats->triangles = c->nt_real;
      stats->points = evaluated_total;
    }
  });
}

int nm_refine_device(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt,
                     const int* labels, const std::uint32_t* selected, std::size_t ns, nm_mesh** out) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    check_tets(tets, nt, n);
    for (std::size_t i = 0; i < ns; ++i)
      if (selected[i] >= nt) throw Error("InvalidSelection: selected tet id out of range (SPEC.md:292)");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    auto* d_nodes = c->meshA_nodes.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_tets = c->meshA_tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_labels = c->meshA_labels.as<int>(std::max<std::size_t>(nt, 1));
    auto* d_sel = c->list.as<std::uint32_t>(std::max<std::size_t>(ns, 1));
    if (n) NM_CUDA(cudaMemcpyAsync(d_nodes, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (nt) {
      if (labels) NM_CUDA(cudaMemcpyAsync(d_labels, labels, nt * sizeof(int), cudaMemcpyHostToDevice, st));
      else NM_CUDA(cudaMemsetAsync(d_labels, 0, nt * sizeof(int), st));
    }
    if (ns) NM_CUDA(cudaMemcpyAsync(d_sel, selected, ns * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    std::uint64_t l = 0;
    const auto [n2, nt2] = refine_dev(c, d_nodes, n, d_tets, nt, d_labels, d_sel, static_cast<std::uint32_t>(ns), st, l);
    *out = make_device_mesh(c, c->meshB_nodes, c->meshB_tets, c->meshB_labels, &c->meshB_parent, nullptr, n2, nt2, n,
                            st);
  });
}

int nm_refine_boundary(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt,
                       const int* labels, int label_a, int label_b, nm_mesh** out) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    check_tets(tets, nt, n);
    if (4 * nt > 0xffffffffull) throw Error("mesh too large for 32-bit face ids");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    auto* d_nodes = c->meshA_nodes.as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_tets = c->meshA_tets.as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_labels = c->meshA_labels.as<int>(std::max<std::size_t>(nt, 1));
    auto* d_nbr = c->nbr.as<std::int32_t>(4 * std::max<std::size_t>(nt, 1));
    auto* d_count = c->count.as<std::uint32_t>(4);
    if (n) NM_CUDA(cudaMemcpyAsync(d_nodes, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_labels, labels, nt * sizeof(int), cudaMemcpyHostToDevice, st));
    const uint4* t4 = reinterpret_cast<const uint4*>(d_tets);
    face_adjacency(c, t4, nt, d_nbr, st);
    auto* d_sel = c->list.as<std::uint32_t>(std::max<std::size_t>(nt, 1));
    std::uint64_t l = 0;
    select(c, nm::PredInterface{d_nbr, d_labels, label_a, label_b}, nt, d_sel, d_count, st, l);
    std::uint32_t ns = 0;
    NM_CUDA(cudaMemcpyAsync(&ns, d_count, sizeof ns, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    const auto [n2, nt2] = refine_dev(c, d_nodes, n, d_tets, nt, d_labels, d_sel, ns, st, l);
    *out = make_device_mesh(c, c->meshB_nodes, c->meshB_tets, c->meshB_labels, &c->meshB_parent, nullptr, n2, nt2, n,
                            st);
  });
}

int nm_refine_relabel(nm_ctx* c, const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt,
                      const std::uint32_t* masks_in, double T, std::uint32_t active, int levels, nm_mesh** out,
                      nm_stats* stats) {
  return guarded([&] {
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    require_surfaces(c);
    if (nt && !tets) throw Error("null tets");
    if (levels < 0) throw Error("levels must be >= 0");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    if (stats) std::memset(stats, 0, sizeof *stats);
    auto acc = [&](const nm_stats& s) {
      if (!stats) return;
      stats->points += s.points;
      stats->evals += s.evals;
      stats->flagged_points += s.flagged_points;
      stats->flagged_pairs += s.flagged_pairs;
      stats->ties += s.ties;
      stats->near_subtiles += s.near_subtiles;
      stats->far_subtiles += s.far_subtiles;
      stats->launches += s.launches;
      stats->ms_label += s.ms_label;
      stats->ms_fixup += s.ms_fixup;
      stats->ms_tets += s.ms_tets;
    };
    // Device-resident mesh A (current) / B (refined); masks M / M2.
    DBuf* An = &c->meshA_nodes;
    DBuf* At = &c->meshA_tets;
    DBuf* Al = &c->meshA_labels;
    DBuf* M = &c->masks;
    DBuf* M2 = &c->masks2;
    std::size_t cn = n, cnt_t = nt;
    auto* d_nodes = An->as<double>(3 * std::max<std::size_t>(n, 1));
    auto* d_tets = At->as<std::uint32_t>(4 * std::max<std::size_t>(nt, 1));
    if (n) NM_CUDA(cudaMemcpyAsync(d_nodes, nodes, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) NM_CUDA(cudaMemcpyAsync(d_tets, tets, 4 * nt * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    check_tets_device(c, d_tets, tets, nt, n, st);
    auto* d_masks = M->as<std::uint32_t>(std::max<std::size_t>(n, 1));
    if (masks_in) {
      if (n) NM_CUDA(cudaMemcpyAsync(d_masks, masks_in, n * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    } else if (n) {
      nm_stats s{};
      label_nodes_dev(c, d_nodes, n, T, d_masks, nullptr, st, stats ? &s : nullptr);
      acc(s);
    }
    bool have_parent = false;
    for (int lvl = 0; lvl <= levels; ++lvl) {
      auto* d_labels = Al->as<int>(std::max<std::size_t>(cnt_t, 1));
      nm_stats ts{};
      label_tets_dev(c, reinterpret_cast<const std::uint32_t*>(At->p), cnt_t, static_cast<std::uint32_t*>(M->p), d_labels,
                     st, stats ? &ts : nullptr);
      acc(ts);
      if (lvl == levels) break;
      // straddling tets (device compaction)
      auto* d_ids = c->list.as<std::uint32_t>(std::max<std::size_t>(cnt_t, 1));
      auto* d_count = c->count.as<std::uint32_t>(4);
      std::uint64_t l = 0;
      select(c, nm::PredStraddle{reinterpret_cast<const uint4*>(At->p), static_cast<const std::uint32_t*>(M->p), active},
             cnt_t, d_ids, d_count, st, l);
      std::uint32_t ns = 0;
      NM_CUDA(cudaMemcpyAsync(&ns, d_count, sizeof ns, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
      // device refinement into the B buffers (refine_dev does not touch c->list)
      cudaEvent_t h0 = c->ev[4], h1 = c->ev[5];
      NM_CUDA(cudaEventRecord(h0, st));
      std::uint64_t rl = 0;
      const auto [n2, nt2] = refine_dev(c, static_cast<const double*>(An->p), cn, static_cast<const std::uint32_t*>(At->p),
                                        cnt_t, static_cast<const int*>(Al->p), d_ids, ns, st, rl);
      NM_CUDA(cudaEventRecord(h1, st));
      NM_CUDA(cudaEventSynchronize(h1));
      if (stats) {
        float ms = 0;
        NM_CUDA(cudaEventElapsedTime(&ms, h0, h1));
        stats->ms_host += ms;  // refinement time (device, CUDA events)
        stats->launches += rl;
      }
      // masks of old nodes are kept; only the new nodes are evaluated
      auto* m2 = M2->as<std::uint32_t>(std::max<std::size_t>(n2, 1));
      if (cn) NM_CUDA(cudaMemcpyAsync(m2, M->p, cn * sizeof(std::uint32_t), cudaMemcpyDeviceToDevice, st));
      if (n2 > cn) {
        nm_stats s{};
        label_nodes_dev(c, static_cast<const double*>(c->meshB_nodes.p) + 3 * cn, n2 - cn, T, m2 + cn, nullptr, st,
                        stats ? &s : nullptr);
        acc(s);
      }
      std::swap(c->meshA_nodes, c->meshB_nodes);
      std::swap(c->meshA_tets, c->meshB_tets);
      std::swap(c->meshA_labels, c->meshB_labels);
      std::swap(c->masks, c->masks2);
      have_parent = true;
      cn = n2;
      cnt_t = nt2;
    }
    if (stats) stats->triangles = c->nt_real;
    *out = make_device_mesh(c, *An, *At, *Al, have_parent ? &c->meshB_parent : nullptr, M, cn, cnt_t, n, st);
  });
}

}  // extern "C"
