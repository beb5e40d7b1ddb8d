// libnestmesh_label.so — C ABI (include/nestmesh_label.h) over the sm_100a
// labeling kernels. One context = one device + one stream; host entry points
// are synchronous, *_device entry points are asynchronous on the caller's
// stream. There is no CPU fallback: every compute entry point fails without
// a usable device.
//
// This translation unit: contexts, nm_set_surfaces (tile packing), the node
// pass (dense, 13-DOP culled, sparse / certified-cell, sharded), tet labels
// and the labeling entry points. See context.cuh for the others.
#include "context.cuh"
#include "strips.h"

using namespace nmh;

namespace {

}  // namespace

namespace nmh {

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
                  const std::vector<std::uint32_t>* first) {
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
  // per-compartment ordered lists of the unknown pairs (counts read back:
  // one host synchronisation per list build)
  std::vector<std::uint32_t> cnt(K);
  // (all compartments in one launch per step; the counts are read back
  // before the write so the list is sized exactly)
  auto build_lists = [&]() {
    const dim3 g(static_cast<unsigned>(nb), static_cast<unsigned>(K));
    nm::k_select_count_bits<<<g, nm::kSelBlock, 0, st>>>(unk, n, chunk);
    nm::k_select_scan<<<K, 1024, 0, st>>>(chunk, nb, dcnt);
    launches += 2;
    // (through the context's pinned words: a pageable read-back would be a
    // driver-staged copy, serialised with other host threads' copies)
    NM_CUDA(cudaMemcpyAsync(c->h_pcnt, dcnt, K * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    cnt.assign(c->h_pcnt, c->h_pcnt + K);
    std::size_t total = 0;
    c->sparse_evals = 0;
    for (int k = 0; k < K; ++k) {
      total += cnt[k];
      c->sparse_evals += std::uint64_t(cnt[k]) * (c->comp_off_h[k + 1] - c->comp_off_h[k]);
    }
    if (total > 0xffffffffull) throw Error("more than 2^32 (point, compartment) pairs to evaluate in one call");
    c->sparse_pairs = total;
    auto* list = c->sp_list.as<std::uint32_t>(std::max<std::size_t>(total, 1));
    if (total) {
      nm::k_select_write_bits<<<g, nm::kSelBlock, 0, st>>>(unk, n, chunk, dcnt, list);
      ++launches;
    }
    NM_CUDA(cudaGetLastError());
    return total;
  };
  const std::size_t total = build_lists();
  if (c->cells && total && !c->no_resolve) {
    // pairs of uncertified children joined to a certified neighbour by a
    // surface-free ball (cells.cuh k_pair_resolve), then the lists again
    nm::ResolveParams rp{};
    rp.pts = d_pts;
    rp.order = order;
    rp.cx = c->cx;
    rp.cy = c->cy;
    rp.cz = c->cz;
    rp.grids = cp.grids;
    rp.code = cp.code;
    rp.child = cp.child;
    rp.K = K;
    rp.list = static_cast<const std::uint32_t*>(c->sp_list.p);
    std::uint32_t o = 0, wsum = 0;
    for (int k = 0; k < K; ++k) {
      rp.off[k] = o;
      rp.cnt[k] = cnt[k];
      rp.wfirst[k] = wsum;
      o += cnt[k];
      wsum += (cnt[k] + 31) / 32;
    }
    rp.off[K] = o;
    rp.wfirst[K] = wsum;
    rp.unk = unk;
    rp.masks = d_masks;
    rp.s_out = d_s;
    rp.write_known = preset_known ? 1 : 0;
    rp.cl.coff = static_cast<const std::uint32_t*>(c->cert_coff.p);
    rp.cl.soff = rp.cl.coff + K + 1;
    rp.cl.sup = static_cast<const float4*>(c->clus_sup.p);
    rp.cl.clus = static_cast<const float4*>(c->clus.p);
    rp.cl.clus_tri = static_cast<const std::uint32_t*>(c->clus_tri.p);
    rp.cl.tsph = static_cast<const float4*>(c->clus_tsph.p);
    rp.cl.xyz = static_cast<const double*>(c->xyz64.p);
    rp.cl.tri = static_cast<const std::uint32_t*>(c->tri_idx.p);
    rp.pend = c->pend.as<nm::PendPair>(std::max<std::size_t>(total, 1));
    rp.npend = c->pend_n.as<unsigned>(1);
    NM_CUDA(cudaMemsetAsync(rp.npend, 0, sizeof(unsigned), st));
    nm::k_pair_resolve<<<static_cast<unsigned>((std::size_t(wsum) * 32 + 255) / 256), 256, 0, st>>>(rp);
    nm::k_pair_chain<<<grid_for(total * 32, 256, c->sm_count * 64), 256, 0, st>>>(rp);
    launches += 2;
    NM_CUDA(cudaGetLastError());
    c->resolved_pairs = total - build_lists();
  } else {
    c->resolved_pairs = 0;
  }
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
                     cudaStream_t st, nm_stats* stats, const std::uint32_t* d_subset, bool stats_deferred, int shard,
                     int nshards) {
  require_surfaces(c);
  if (!(T > 0.0 && T < 1.0)) throw Error("threshold must lie in (0, 1) (SPEC.md:216)");
  NvtxRange nvtx_pass("nm node pass");
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
  auto* flagmask = c->flagmask.as<std::uint32_t>(n);  // by evaluation position
  // every scratch buffer is sized before the first launch: a growing DBuf
  // frees its old block, and cudaFree would wait for the kernels
  auto* list = c->list.as<std::uint32_t>(n);
  auto* ms = c->pos_masks.as<std::uint32_t>(n);  // dense passes: masks by evaluation position
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
  prm.n_pts = d_subset ? ~std::size_t(0) : n;
  prm.n_tiles = c->comp_tiles_h.empty() ? 0u : c->comp_tiles_h.back();
  prm.tri = static_cast<const float4*>(c->tri.p);
  prm.sub = static_cast<const float4*>(c->sub.p);
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
  prm.masks = d_masks;  // sparse passes; dense passes write ms (below)
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
  prm.masks = ms;
  const int np = prm.cull ? 1 : c->opt.pairs_per_thread;
  const std::size_t per_block = static_cast<std::size_t>(nm::kBlock) * 2 * np;
  const std::size_t nblocks = (n + per_block - 1) / per_block;
  const int csplit = compartment_split(c, nblocks, prm.split);
  if (csplit > 1) {
    nm::k_zero_masks<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(n, ms, flagmask);
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
  nm::k_unpermute<<<grid_for(n, 256, c->sm_count * 16), 256, 0, st>>>(order, n, ms, d_masks,
                                                                       d_subset ? ~std::size_t(0) : n);
  NM_CUDA(cudaGetLastError());
  ++launches;
  }
  if (stats) NM_CUDA(cudaEventRecord(c->ev[2], st));
  // compaction of flagged points, per-compartment pair lists, fp64 fix-up
  NvtxRange nvtx_fix("nm fp64 fix-up");
  select(c, nm::PredNonzero{flagmask}, n, list, d_count, st, launches);
  const int K = c->K;
  auto* pair_cnt = c->pair_cnt.as<std::uint32_t>(2 * 32);
  NM_CUDA(cudaMemsetAsync(pair_cnt, 0, 2 * 32 * sizeof(std::uint32_t), st));
  nm::k_fix_count<<<grid_for(n, 256, c->sm_count * 4), 256, 0, st>>>(list, d_count, flagmask, pair_cnt);
  NM_CUDA(cudaGetLastError());
  // one host synchronisation: the pair lists' size (the fix-up is the only
  // consumer, and its batch grid runs from the device-side counts)
  NM_CUDA(cudaMemcpyAsync(c->h_pcnt, pair_cnt, K * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
  NM_CUDA(cudaStreamSynchronize(st));
  std::size_t total = 0, nwork = 0, npart = 0;
  for (int k = 0; k < K; ++k) {
    const std::size_t ntri = c->comp_off_h[k + 1] - c->comp_off_h[k];
    const std::size_t nch = std::max<std::size_t>(1, (ntri + nm::kFixChunk - 1) / nm::kFixChunk);
    total += c->h_pcnt[k];
    nwork += (c->h_pcnt[k] + nm::kFixPairs - 1) / nm::kFixPairs * nch;
    npart += std::size_t(c->h_pcnt[k]) * nch;
  }
  auto* pairs = c->pairs.as<std::uint32_t>(std::max<std::size_t>(total, 1));
  auto* part = c->fix_part.as<double>(std::max<std::size_t>(npart, 1));
  launches += 1;
  if (total) {
    nm::k_fix_fill<<<grid_for(n, 256, c->sm_count * 4), 256, 0, st>>>(list, d_count, flagmask, pair_cnt, K,
                                                                       pair_cnt + 32, pairs);
    nm::FixupParams fp{};
    fp.pts = d_pts;
    fp.list = list;
    fp.order = order;
    fp.n_pts = d_subset ? ~std::size_t(0) : n;
    fp.n_tri = c->nt_real;
    fp.n_part = npart;
    fp.count = d_count;
    fp.flagmask = flagmask;
    fp.tri64 = static_cast<const double*>(c->tri64.p);
    fp.comp_off = static_cast<const std::uint32_t*>(c->comp_off.p);
    fp.pair_cnt = pair_cnt;
    fp.pairs = pairs;
    fp.part = part;
    fp.K = K;
    fp.T = T;
    fp.tie_eps = c->opt.tie_eps;
    fp.masks = d_masks;
    fp.s_out = d_s;
    fp.counters = counters;
    // two stages: hybrid terms (far triangles in fp32) decide the pairs whose
    // s is not within kFixExactBand of T and whose point lies in no
    // triangle's plane; the rest get the oracle-order fp64 terms throughout
    fp.exact = c->fix_exact.as<std::uint32_t>(std::max<std::size_t>(total, 1));
    NM_CUDA(cudaMemsetAsync(fp.exact, 0, total * sizeof(std::uint32_t), st));
    static_assert(nm::kFixSmem <= 48 * 1024, "k_fixup tiles must fit the default dynamic shared memory");
    for (int stage = 1; stage <= 2; ++stage) {
      fp.stage = stage;
      nm::k_fixup<<<grid_for(nwork, 1, c->sm_count * 16), nm::kFixThreads, nm::kFixSmem, st>>>(fp);
      nm::k_fix_finalize<<<grid_for(total, 256, c->sm_count * 4), 256, 0, st>>>(fp);
    }
    NM_CUDA(cudaGetLastError());
    launches += 5;
  }
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
                    cudaStream_t st, nm_stats* stats, std::size_t n_nodes) {
  require_surfaces(c);
  if (nt == 0) return;
  NvtxRange nvtx_tets("nm tet labels");
  if (stats) NM_CUDA(cudaEventRecord(c->ev[4], st));
  nm::k_label_tets<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(reinterpret_cast<const uint4*>(d_tets), nt,
                                                                        d_masks, d_labels, c->ids, n_nodes);
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

}  // namespace nmh

extern "C" {

int nm_abi_version(void) { return NM_ABI_VERSION; }
const char* nm_last_error(void) { return last_error().c_str(); }

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
  o->cell_axis = kDefaultCellAxis;
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
      if (c->opt.cell_axis == 0) c->opt.cell_axis = kDefaultCellAxis;
      if (c->opt.cell_axis < 8 || c->opt.cell_axis > 1024) throw Error("cell_axis must be 0 (default) or in [8, 1024]");
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
      NM_CUDA(cudaMallocHost(&c->h_pcnt, 32 * sizeof(std::uint32_t)));
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
    NvtxRange nvtx_surf("nm_set_surfaces");
    const auto t_entry = std::chrono::steady_clock::now();
    if (comp_off[0] != 0 || comp_off[K] != nt) throw Error("comp_tri_off must start at 0 and end at the triangle count");
    for (int k = 0; k < K; ++k) {
      if (comp_off[k + 1] < comp_off[k]) throw Error("comp_tri_off must be non-decreasing");
      if (label_ids[k] <= 0) throw Error("compartment label ids must be > 0 (0 is the bounding box)");
    }
    {
      constexpr std::size_t kChunk = std::size_t(1) << 20;
      std::atomic<bool> bad{false};
      parallel_for(static_cast<int>((3 * nt + kChunk - 1) / kChunk), [&](int ch) {
        const std::size_t i0 = static_cast<std::size_t>(ch) * kChunk, i1 = std::min(3 * nt, i0 + kChunk);
        std::uint32_t mx = 0;
        for (std::size_t i = i0; i < i1; ++i) mx = std::max(mx, tri[i]);
        if (mx >= nv) bad = true;
      });
      if (bad) throw Error("triangle index out of range");
    }
    NM_CUDA(cudaSetDevice(c->opt.device));
    const bool verbose = std::getenv("NM_CELL_VERBOSE") != nullptr;
    auto t_prev = t_entry;
    c->surf_t0 = t_entry;
    auto lap = [&](const char* what) {
      if (!verbose) return;
      const auto t = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[surfaces] %-10s %8.1f ms  (at %6.1f)\n", what,
                   std::chrono::duration<double, std::milli>(t - t_prev).count(),
                   std::chrono::duration<double, std::milli>(t - c->surf_t0).count());
      t_prev = t;
    };
    lap("validate");
    // Domain box and centring offset of the fp32 frame.
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    {
      constexpr std::size_t kChunk = std::size_t(1) << 16;  // vertices per work item (min / max: any order)
      const int nch = static_cast<int>((nv + kChunk - 1) / kChunk);
      std::vector<std::array<double, 6>> part(std::max(nch, 1), {1e300, 1e300, 1e300, -1e300, -1e300, -1e300});
      parallel_for(nch, [&](int ch) {
        auto& b = part[ch];
        for (std::size_t i = static_cast<std::size_t>(ch) * kChunk; i < std::min(nv, (ch + 1) * kChunk); ++i)
          for (int a = 0; a < 3; ++a) {
            b[a] = std::min(b[a], xyz[3 * i + a]);
            b[3 + a] = std::max(b[3 + a], xyz[3 * i + a]);
          }
      });
      for (const auto& b : part)
        for (int a = 0; a < 3; ++a) {
          lo[a] = std::min(lo[a], b[a]);
          hi[a] = std::max(hi[a], b[3 + a]);
        }
    }
    if (nv == 0) lo[0] = lo[1] = lo[2] = hi[0] = hi[1] = hi[2] = 0.0;
    const double ctr[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-6}) * 1.5;
    for (int a = 0; a < 3; ++a) c->lo[a] = ctr[a] - 0.5 * span;
    c->span = span;
    c->cx = ctr[0];
    c->cy = ctr[1];
    c->cz = ctr[2];
    lap("box");

    c->has_surfaces = false;
    c->cells = false;
    c->K = K;
    // Device prelude: the fp64 originals (fix-up, cell certification), the
    // de-indexed fp64 triangles and the 13-DOP / box of every compartment
    // (geometry.cuh: chunks of triangles per block, merged per compartment;
    // slab bounds over the vertices in the centred frame, widened by 1e-3 mm
    // + 1e-5 |bound| and rounded outward; the fp64 extents also size the cell
    // grids). With certified cells (cull_outside = 2) the prelude and then
    // the cell build run on their own host thread, stream and stager while
    // this thread packs the tiles; otherwise the prelude runs here.
    std::vector<float4> hbox(static_cast<std::size_t>(K) * nm::kDopF4);
    std::vector<double> hext(static_cast<std::size_t>(K) * nm::kExtQ);
    auto prelude = [&](bool side) {
      auto up_on = [&](DBuf& b, const void* src, std::size_t bytes) {  // pinned chunk staging
        void* d = b.get(std::max<std::size_t>(bytes, 1));
        c->h2d(d, src, bytes, c->side, side, side);
      };
      up_on(c->xyz64, xyz, nv * 3 * sizeof(double));
      up_on(c->tri_idx, tri, nt * 3 * sizeof(std::uint32_t));
      up_on(c->comp_off, comp_off, (K + 1) * sizeof(std::uint32_t));
      c->trace(side ? "cells" : "main", "prelude: uploads");
      auto* t64 = c->tri64.as<double>(std::max<std::size_t>(nm::kFixRec * nt, 1));
      if (nt)
        nm::k_deindex64<<<grid_for(nt, 256, c->sm_count * 16), 256, 0, c->side>>>(
            static_cast<const double*>(c->xyz64.p), static_cast<const std::uint32_t*>(c->tri_idx.p), nt, t64);
      constexpr std::uint32_t kExtChunk = 8192;
      std::vector<nm::ExtentItem> items;
      std::vector<std::uint32_t> item_first(K + 1, 0);
      for (int k = 0; k < K; ++k) {
        item_first[k] = static_cast<std::uint32_t>(items.size());
        for (std::uint32_t t = comp_off[k]; t < comp_off[k + 1]; t += kExtChunk)
          items.push_back({k, t, std::min(comp_off[k + 1], t + kExtChunk)});
      }
      item_first[K] = static_cast<std::uint32_t>(items.size());
      auto* d_items = c->ext_items.as<nm::ExtentItem>(std::max<std::size_t>(items.size(), 1));
      auto* d_first = c->ext_first.as<std::uint32_t>(K + 1);
      auto* d_part = c->ext_part.as<double>(std::max<std::size_t>(items.size(), 1) * nm::kExtQ);
      auto* d_ext = c->ext_val.as<double>(static_cast<std::size_t>(K) * nm::kExtQ);
      auto* d_box = c->comp_box.as<float4>(static_cast<std::size_t>(K) * nm::kDopF4);
      c->h2d(d_items, items.data(), items.size() * sizeof(nm::ExtentItem), c->side, side, side);
      c->h2d(d_first, item_first.data(), item_first.size() * sizeof(std::uint32_t), c->side, side, side);
      if (!items.empty())
        nm::k_extents_items<<<static_cast<unsigned>(items.size()), 256, 0, c->side>>>(
            d_items, static_cast<const double*>(c->xyz64.p), static_cast<const std::uint32_t*>(c->tri_idx.p), ctr[0],
            ctr[1], ctr[2], d_part);
      nm::k_extents_finalize<<<K, 32, 0, c->side>>>(d_part, d_first, static_cast<const std::uint32_t*>(c->comp_off.p),
                                                    d_ext, d_box);
      NM_CUDA(cudaGetLastError());
      c->d2h(hext.data(), d_ext, hext.size() * sizeof(double), c->side, side, side);
      c->d2h(hbox.data(), d_box, hbox.size() * sizeof(float4), c->side, side, side);
      c->trace(side ? "cells" : "main", "prelude: extents read");
    };
    std::promise<void> dop_ready;  // set by the cell thread after its prelude
    std::unique_ptr<CellBuilder> cells;
    std::exception_ptr cells_err;
    struct Joiner {
      std::thread t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } cells_thread;
    if (c->opt.cull_outside == 2) {
      cells = make_cell_builder(c, xyz, tri, comp_off, hbox, hext, c->side, dop_ready.get_future().share());
      cells_thread.t = std::thread([&] {
        try {
          NM_CUDA(cudaSetDevice(c->opt.device));
          prelude(true);
          dop_ready.set_value();
          cells->prepare();
        } catch (...) {
          cells_err = std::current_exception();
        }
      });
    } else {
      prelude(false);
    }
    lap("prelude");

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
        const std::vector<Strip> strips = stripify(tri, comp_off[k], comp_off[k + 1], nv);
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
    lap("strips");
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
    // written in full by the packing below (every float4 of every record):
    // no zero-fill of ~50 MB on this thread before the parallel pass
    const std::size_t htri_n = ntiles * tile_f4, hsub_n = ntiles * nm::kSubPerTile * nm::kSubRec;
    std::unique_ptr<float4[]> htri(new float4[std::max<std::size_t>(htri_n, 1)]);
    std::unique_ptr<float4[]> hsub(new float4[std::max<std::size_t>(hsub_n, 1)]);
    std::vector<std::uint32_t> hcont(std::max<std::size_t>(ntiles, 1), 0u);
    static_assert(nm::kSubPerTile * nm::kGroups <= 32, "continuation bits of a tile must fit a uint32");
    const double far_ratio = c->opt.far_ratio, far_abs = c->opt.far_abs_mm;
    // Watertight subtile frames. Each 32-triangle subtile
    // carries an fp32 centre c and its vertices relative to c, so the kernel
    // forms R = (v - c) - (p - c) with ~ulp(|R|) error. For the sum over a
    // closed surface to stay a winding number in fp32, every vertex must have
    // the SAME position in every subtile it appears in: vertices are snapped
    // (centred frame, fp64) to a global power-of-two grid G fine enough that
    // v - c is exactly representable in fp32 for every subtile (c on a
    // coarser power-of-two grid Gc, exact in fp32). Snapping moves a vertex by
    // <= G/2 (a few nm) consistently in every triangle, so the snapped
    // surfaces are still closed and their winding numbers are the oracle's
    // for every point not within G of a surface (such points are caught by
    // the near-face / near-vertex detector and re-evaluated in fp64 on the
    // original vertices).
    constexpr std::uint32_t kTileChunk = 8;
    auto tile_comp = [&](std::uint32_t tl) {  // compartment owning tile tl
      return static_cast<int>(std::upper_bound(tiles.begin(), tiles.end(), tl) - tiles.begin()) - 1;
    };
    auto gather = [&](int k, std::uint32_t tl, int sidx, std::vector<const double*>& srcv) {
      const std::size_t nreal = use_strips ? segs[k].size() : order[k].size();
      // fallback vertex for all-pad units: the compartment's first vertex
      const double* pad_v = comp_off[k + 1] > comp_off[k] ? xyz + 3 * std::size_t(tri[3 * comp_off[k]]) : ctr;
      srcv.clear();
      const std::size_t u0 = static_cast<std::size_t>(tl - tiles[k]) * nm::kTile / (use_strips ? nm::kSegTris : 1) +
                             sidx * (use_strips ? nm::kSub / nm::kSegTris : nm::kSub);
      const int nunits = use_strips ? nm::kSub / nm::kSegTris : nm::kSub;
      for (int j = 0; j < nunits; ++j) {
        const std::size_t u = u0 + j;
        if (use_strips) {
          for (int q = 0; q < nm::kSegTris + 2; ++q) srcv.push_back(u < nreal ? xyz + 3 * std::size_t(segs[k][u].v[q]) : pad_v);
        } else {
          const std::uint32_t t = u < nreal ? order[k][u] : 0;
          for (int q = 0; q < 3; ++q) srcv.push_back(u < nreal ? xyz + 3 * std::size_t(tri[3 * t + q]) : pad_v);
        }
      }
      return u0;
    };
    auto mid_of = [&](const std::vector<const double*>& srcv, double* mid, double* half) {
      double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
      for (const double* v : srcv)
        for (int a = 0; a < 3; ++a) {
          blo[a] = std::min(blo[a], v[a] - ctr[a]);
          bhi[a] = std::max(bhi[a], v[a] - ctr[a]);
        }
      for (int a = 0; a < 3; ++a) {
        mid[a] = 0.5 * (blo[a] + bhi[a]);
        half[a] = 0.5 * (bhi[a] - blo[a]);
      }
    };
    // grids: Gc for the centres (|c| / Gc < 2^23), G for the vertices
    // (|v - c| / G < 2^23 with c rounded to Gc)
    double cmax = 0.0, emax = 0.0;
    {
      // work items: chunks of kTileChunk tiles over all compartments (every
      // host thread busy whatever the compartment sizes)
      const int nitems = static_cast<int>((ntiles + kTileChunk - 1) / kTileChunk);
      std::vector<double> cm(std::max(nitems, 1), 0.0), em(std::max(nitems, 1), 0.0);
      parallel_for(nitems, [&](int i) {
        std::vector<const double*> srcv;
        const std::uint32_t t0 = static_cast<std::uint32_t>(i) * kTileChunk,
                            t1 = std::min<std::uint32_t>(static_cast<std::uint32_t>(ntiles), t0 + kTileChunk);
        for (std::uint32_t tl = t0; tl < t1; ++tl) {
          const int k = tile_comp(tl);
          for (int sidx = 0; sidx < nm::kSubPerTile; ++sidx) {
            gather(k, tl, sidx, srcv);
            double mid[3], half[3];
            mid_of(srcv, mid, half);
            for (int a = 0; a < 3; ++a) {
              cm[i] = std::max(cm[i], std::fabs(mid[a]));
              em[i] = std::max(em[i], half[a]);
            }
          }
        }
      });
      for (int i = 0; i < nitems; ++i) {
        cmax = std::max(cmax, cm[i]);
        emax = std::max(emax, em[i]);
      }
    }
    // (factor-2 margins: |v - c| <= emax + G/2 + Gc/2 < 2^24 G)
    lap("grid");
    double Gc = std::ldexp(1.0, std::max(-120, std::ilogb(std::max(cmax, 1e-30)) + 1 - 23));
    const double G = std::ldexp(1.0, std::max(-120, std::ilogb(std::max(emax + Gc, 1e-30)) + 1 - 22));
    Gc = std::max(Gc, G);  // centres on the vertex grid too
    c->snap_grid = G;
    std::atomic<bool> inexact{false};
    auto snap = [&](double x, double g) { return std::nearbyint(x / g) * g; };
    parallel_for(static_cast<int>((ntiles + kTileChunk - 1) / kTileChunk), [&](int item) {  // disjoint tile ranges
      std::vector<const double*> srcv;
      const std::uint32_t t0 = static_cast<std::uint32_t>(item) * kTileChunk,
                          t1 = std::min<std::uint32_t>(static_cast<std::uint32_t>(ntiles), t0 + kTileChunk);
      for (std::uint32_t tl = t0; tl < t1; ++tl) {
        const int k = tile_comp(tl);
        const std::size_t nreal = use_strips ? segs[k].size() : order[k].size();
        for (int sidx = 0; sidx < nm::kSubPerTile; ++sidx) {
          const std::size_t u0 = gather(k, tl, sidx, srcv);
          const int nunits = use_strips ? nm::kSub / nm::kSegTris : nm::kSub;
          double mid[3], half[3];
          mid_of(srcv, mid, half);
          const float fc[3] = {float(snap(mid[0], Gc)), float(snap(mid[1], Gc)), float(snap(mid[2], Gc))};
          // snapped vertex relative to the centre: exact in fp32 (checked)
          auto relv = [&](const double* v, float* out) {
            for (int a = 0; a < 3; ++a) {
              const double r = snap(v[a] - ctr[a], G) - double(fc[a]);
              out[a] = float(r);
              if (double(out[a]) != r) inexact = true;
            }
          };
          double rho = 0.0;
          std::vector<float> rel(3 * srcv.size());
          for (std::size_t q = 0; q < srcv.size(); ++q) {
            relv(srcv[q], &rel[3 * q]);
            rho = std::max(rho, std::sqrt(double(rel[3 * q]) * rel[3 * q] + double(rel[3 * q + 1]) * rel[3 * q + 1] +
                                          double(rel[3 * q + 2]) * rel[3 * q + 2]));
          }
          // N = (v2 - v1) x (v3 - v1) of the snapped ORIGINAL triangle (its own
          // vertex order: outward whatever the strip parity), fp64 from the
          // exact fp32 coordinates
          auto normal_rel = [&](std::uint32_t t, double* N) {
            float A[3], B[3], C[3];
            relv(xyz + 3 * std::size_t(tri[3 * t]), A);
            relv(xyz + 3 * std::size_t(tri[3 * t + 1]), B);
            relv(xyz + 3 * std::size_t(tri[3 * t + 2]), C);
            const double e1[3] = {double(B[0]) - A[0], double(B[1]) - A[1], double(B[2]) - A[2]};
            const double e2[3] = {double(C[0]) - A[0], double(C[1]) - A[1], double(C[2]) - A[2]};
            N[0] = e1[1] * e2[2] - e1[2] * e2[1];
            N[1] = e1[2] * e2[0] - e1[0] * e2[2];
            N[2] = e1[0] * e2[1] - e1[1] * e2[0];
          };
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
                if (u < nreal && segs[k][u].t[q] >= 0) normal_rel(static_cast<std::uint32_t>(segs[k][u].t[q]), N[q]);
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
            } else {
              double N[3] = {0, 0, 0};
              if (u < nreal) normal_rel(order[k][u], N);
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
    lap("pack");
    if (inexact) throw Error("internal: a snapped subtile coordinate is not exact in fp32");
    c->strips = use_strips;
    auto up = [&](DBuf& b, const void* src, std::size_t bytes) {  // pinned chunk staging (recycled chunks)
      void* d = b.get(std::max<std::size_t>(bytes, 1));
      c->trace("main", "  alloc");
      c->h2d(d, src, bytes, c->stream);
      c->trace("main", "  staged");
    };
    up(c->tri, htri.get(), htri_n * sizeof(float4));
    lap("up-tri");
    up(c->sub, hsub.get(), hsub_n * sizeof(float4));
    up(c->cont, hcont.data(), hcont.size() * sizeof(std::uint32_t));
    up(c->comp_tiles, tiles.data(), tiles.size() * sizeof(std::uint32_t));
    // (comp_box: written on the device by k_extents_finalize)
    NM_CUDA(cudaStreamSynchronize(c->stream));
    lap("upload");
    if (cells_thread.t.joinable()) cells_thread.t.join();
    lap("cells-join");
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
    lap("cells-fin");
    cells.reset();
    // the packing's host arrays (~160 MB at cfg5: segments, fp32 records) are
    // released on a detached thread: unmapping them took milliseconds
    std::thread([a = std::move(segs), b = std::move(order), t = std::move(htri), u = std::move(hsub)]() mutable {
      a.clear();
      b.clear();
      t.reset();
      u.reset();
    }).detach();
    lap("end");
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

int nm_cell_dump(nm_ctx* c, uint32_t* codes, size_t codes_cap, uint8_t* children, size_t children_cap, size_t* n_codes,
                 size_t* n_children) {
  return guarded([&] {
    require_surfaces(c);
    if (!c->cells) throw Error("no certified cells (cull_outside = 2)");
    NM_CUDA(cudaSetDevice(c->opt.device));
    if (n_codes) *n_codes = c->cells_l1;
    if (n_children) *n_children = c->cells_children;
    if (codes && codes_cap >= c->cells_l1 && c->cells_l1)
      NM_CUDA(cudaMemcpy(codes, c->cell_state.p, c->cells_l1 * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    if (children && children_cap >= c->cells_children && c->cells_children)
      NM_CUDA(cudaMemcpy(children, c->cell_child.p, c->cells_children, cudaMemcpyDeviceToHost));
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
    c->h2d(d_pts, pts, 3 * n * sizeof(double), c->stream);
    label_nodes_dev(c, d_pts, n, T, d_masks, nullptr, c->stream, stats);
    c->d2h(masks_out, d_masks, n * sizeof(std::uint32_t), c->stream);
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
    c->h2d(d_pts, pts, 3 * n * sizeof(double), c->stream);
    label_nodes_dev(c, d_pts, n, T, d_masks, d_s, c->stream, stats);
    c->d2h(s_out, d_s, n * c->K * sizeof(double), c->stream);
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
    c->h2d(d_tets, tets, 4 * nt * sizeof(std::uint32_t), c->stream);
    check_tets_device(c, d_tets, tets, nt, n_nodes, c->stream);
    c->h2d(d_masks, masks, n_nodes * sizeof(std::uint32_t), c->stream);
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, c->stream, stats, n_nodes);
    c->d2h(labels_out, d_labels, nt * sizeof(int), c->stream);
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
    const bool timing = std::getenv("NM_TIMING") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      NM_CUDA(cudaStreamSynchronize(c->stream));
      std::fprintf(stderr, "[nm_label_mesh] %-14s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    // The nodes first (every host copy thread on them: the node pass needs
    // all of them). The tets follow in chunks on a helper thread and the side
    // stream, under the node pass; once the node masks are done, each chunk's
    // labels are computed as soon as it is on the device and copied back
    // while the later chunks still upload (H2D and D2H run on separate copy
    // engines), so the labels' read-back hides under the tet upload. Tets
    // with a node id >= n get label 0 and are reported after the last chunk.
    c->h2d(d_pts, nodes, 3 * n * sizeof(double), c->stream);
    lap("nodes h2d");
#ifndef NM_TET_CHUNK
#define NM_TET_CHUNK (std::size_t(8) << 20)
#endif
    constexpr std::size_t kTetChunk = NM_TET_CHUNK;  // tets per chunk (128 MB of indices; profiles/r02/label_mesh_chunk_ab.txt)
    const std::size_t nch = nt ? (nt + kTetChunk - 1) / kTetChunk : 0;
    std::vector<cudaEvent_t> up_ev(nch, nullptr);
    struct EvGuard {
      std::vector<cudaEvent_t>& v;
      ~EvGuard() {
        for (cudaEvent_t e : v)
          if (e) cudaEventDestroy(e);
      }
    } ev_guard{up_ev};
    for (auto& e : up_ev) NM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    NM_CUDA(cudaMemsetAsync(d_word, 0, sizeof(std::uint32_t), c->stream));
    std::atomic<std::size_t> uploaded{0};
    std::atomic<bool> side_failed{false};
    std::exception_ptr side_err;
    std::thread side_thread;
    if (nt) {
      side_thread = std::thread([&] {
        try {
          NM_CUDA(cudaSetDevice(c->opt.device));
          for (std::size_t q = 0; q < nch; ++q) {
            const std::size_t t0 = q * kTetChunk, m = std::min(kTetChunk, nt - t0);
            // the main copy pool: the node copies are done, the main thread
            // copies labels back through the side pool
            c->h2d(d_tets + 4 * t0, tets + 4 * t0, 4 * m * sizeof(std::uint32_t), c->side, /*side=*/true,
                   /*side_pool=*/false);
            NM_CUDA(cudaEventRecord(up_ev[q], c->side));
            uploaded.store(q + 1, std::memory_order_release);
          }
        } catch (...) {
          side_err = std::current_exception();
          side_failed.store(true, std::memory_order_release);
        }
      });
    }
    struct Join {
      std::thread& t;
      ~Join() {
        if (t.joinable()) t.join();
      }
    } join{side_thread};
    label_nodes_dev(c, d_pts, n, T, d_masks, nullptr, c->stream, stats, nullptr, /*stats_deferred=*/true);
    lap("node pass");
    if (stats && n) read_node_stats(c, n, c->stream, stats);
    if (stats) NM_CUDA(cudaEventRecord(c->ev[4], c->stream));
    for (std::size_t q = 0; q < nch; ++q) {
      while (uploaded.load(std::memory_order_acquire) <= q && !side_failed.load(std::memory_order_acquire))
        std::this_thread::yield();
      if (side_failed.load(std::memory_order_acquire)) break;
      const std::size_t t0 = q * kTetChunk, m = std::min(kTetChunk, nt - t0);
      NM_CUDA(cudaStreamWaitEvent(c->stream, up_ev[q], 0));
      nm::k_label_tets<<<grid_for(m, 256, c->sm_count * 32), 256, 0, c->stream>>>(
          reinterpret_cast<const uint4*>(d_tets) + t0, m, d_masks, d_labels + t0, c->ids, n, d_word);
      NM_CUDA(cudaGetLastError());
      c->d2h(labels_out + t0, d_labels + t0, m * sizeof(int), c->stream, /*side=*/false, /*side_pool=*/true);
    }
    if (side_thread.joinable()) side_thread.join();
    if (side_err) std::rethrow_exception(side_err);
    lap("tets + labels");
    if (stats) {
      NM_CUDA(cudaEventRecord(c->ev[5], c->stream));
      NM_CUDA(cudaEventSynchronize(c->ev[5]));
      float ms = 0;
      NM_CUDA(cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]));  // labels with the tail of the upload
      stats->ms_tets += ms;
      stats->launches += static_cast<std::uint64_t>(nch);
    }
    NM_CUDA(cudaMemcpyAsync(c->h_word, d_word, sizeof(std::uint32_t), cudaMemcpyDeviceToHost, c->stream));
    NM_CUDA(cudaStreamSynchronize(c->stream));
    if (nt && *c->h_word) check_tets(tets, nt, n);  // throws with the offending tet
    if (masks_out) c->d2h(masks_out, d_masks, n * sizeof(std::uint32_t), c->stream);
    lap("d2h");
    NM_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
