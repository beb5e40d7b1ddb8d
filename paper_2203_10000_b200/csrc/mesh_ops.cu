// Mesh operations of the labeling path: face adjacency, device refinement,
// relabel_recursive, compartment-boundary extraction, lattice generation,
// point-surface distance, tet-centroid labeling.
#include "context.cuh"

using namespace nmh;

namespace nmh {

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

}  // namespace nmh

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
    if (nm_lattice_device(c, origin, h, nx, ny, nz, d_nodes, d_tets, st) != 0) throw Error(last_error());
    label_nodes_dev(c, d_nodes, nn, T, d_masks, nullptr, st, stats);
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, st, stats, nn);
    if (labels_out) c->d2h(labels_out, d_labels, nt * sizeof(int), st);
    if (masks_out) c->d2h(masks_out, d_masks, nn * sizeof(std::uint32_t), st);
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
    c->h2d(d_nodes, nodes, 3 * n * sizeof(double), st);
    c->h2d(d_tets, tets, 4 * nt * sizeof(std::uint32_t), st);
    if (nt)
      nm::k_centroids<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(d_nodes, reinterpret_cast<const uint4*>(d_tets),
                                                                          nt, d_cen);
    label_nodes_dev(c, d_cen, nt, T, d_masks, nullptr, st, stats);
    if (nt) {
      nm::k_mask_labels<<<grid_for(nt, 256, c->sm_count * 32), 256, 0, st>>>(d_masks, nt, d_labels, c->ids);
      NM_CUDA(cudaGetLastError());
      c->d2h(labels_out, d_labels, nt * sizeof(int), st);
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
    c->h2d(d_pts, nodes, 3 * n * sizeof(double), st);
    c->h2d(d_tets, tets, 4 * nt * sizeof(std::uint32_t), st);
    c->h2d(d_labels, labels_io, nt * sizeof(int), st);
    NM_CUDA(cudaMemsetAsync(d_known, 0, std::max<std::size_t>(n, 1), st));
    NM_CUDA(cudaMemsetAsync(d_masks, 0, std::max<std::size_t>(n, 1) * sizeof(std::uint32_t), st));
    const uint4* t4 = reinterpret_cast<const uint4*>(d_tets);
    face_adjacency(c, t4, nt, d_nbr, st);
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
    c->d2h(labels_io, d_labels, nt * sizeof(int), st);
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

int nm_refine_device_d(nm_ctx* c, const double* d_nodes, std::size_t n, const std::uint32_t* d_tets, std::size_t nt,
                       const int* d_labels, const std::uint32_t* d_sel, std::size_t ns, void* stream, nm_mesh** out) {
  return guarded([&] {
    if (!c) throw Error("null context");
    if (!out) throw Error("null output pointer");
    *out = nullptr;
    if (ns > nt) throw Error("InvalidSelection: more selected tets than tets (SPEC.md:292)");
    if (n > 0xffffffffull || nt > 0xffffffffull) throw Error("mesh exceeds 32-bit ids");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->pick(stream);
    // device-side validation of the inputs (the caller's arrays never reach the host)
    if (nt) {
      auto* d_word = c->word.as<std::uint32_t>(2);
      NM_CUDA(cudaMemsetAsync(d_word, 0, 2 * sizeof(std::uint32_t), st));
      nm::k_max_index<<<grid_for(nt, 256, c->sm_count * 8), 256, 0, st>>>(reinterpret_cast<const uint4*>(d_tets), nt,
                                                                          d_word);
      if (ns)
        nm::k_max_u32<<<grid_for(ns, 256, c->sm_count * 8), 256, 0, st>>>(d_sel, ns, d_word + 1);
      NM_CUDA(cudaGetLastError());
      std::uint32_t h[2];
      NM_CUDA(cudaMemcpyAsync(h, d_word, sizeof h, cudaMemcpyDeviceToHost, st));
      NM_CUDA(cudaStreamSynchronize(st));
      if (h[0] >= n) throw Error("a tet references a node >= node count");
      if (ns && h[1] >= nt) throw Error("InvalidSelection: selected tet id out of range (SPEC.md:292)");
    }
    const int* lab = d_labels;
    if (!lab) {
      auto* z = c->meshA_labels.as<int>(std::max<std::size_t>(nt, 1));
      NM_CUDA(cudaMemsetAsync(z, 0, std::max<std::size_t>(nt, 1) * sizeof(int), st));
      lab = z;
    }
    std::uint64_t l = 0;
    const auto [n2, nt2] = refine_dev(c, d_nodes, n, d_tets, nt, lab, d_sel, static_cast<std::uint32_t>(ns), st, l);
    *out = make_device_mesh(c, c->meshB_nodes, c->meshB_tets, c->meshB_labels, &c->meshB_parent, nullptr, n2, nt2, n,
                            st);
    NM_CUDA(cudaStreamSynchronize(st));  // the handle's arrays are complete for any stream that reads them
  });
}

int nm_mesh_copy_device(const nm_mesh* m, double* d_nodes, std::uint32_t* d_tets, int* d_labels, std::uint32_t* d_parent,
                        void* stream) {
  return guarded([&] {
    if (!m || m->dev.device < 0) throw Error("not a device-resident mesh");
    NM_CUDA(cudaSetDevice(m->dev.device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    const auto& d = m->dev;
    auto cp = [&](void* dst, const void* src, std::size_t bytes) {
      if (dst && bytes) NM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
    };
    cp(d_nodes, d.nodes, 3 * d.nn * sizeof(double));
    cp(d_tets, d.tets, 4 * d.nt * sizeof(std::uint32_t));
    cp(d_labels, d.labels, d.nt * sizeof(int));
    cp(d_parent, d.parent, d.nt * sizeof(std::uint32_t));
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
                     st, stats ? &ts : nullptr, cn);
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
