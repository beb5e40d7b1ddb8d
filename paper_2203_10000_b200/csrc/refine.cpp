// Host-side refinement for the recursive refine/relabel driver
// (§2.1.2, Fig. 2). CPU restatement first; the
// device version is the next item of SURVEY.md §8(f).
//
// refine_volume(mesh, selected):
//   * selected tets are split 1:8 through their edge midpoints ("red"); the
//     interior octahedron is cut along its shortest diagonal,
//     ties broken by the lowest node ids;
//   * an unselected tet whose split edges form one of the Fig. 2(c-e)
//     transition patterns — one edge, two edges of one face, the three edges
//     of one face — gets the matching conforming template ("green"); any
//     other pattern (two opposite edges, three edges not on one face, four or
//     more) escalates to the 1:8 split and the closure repeats;
//   * a face with exactly two split edges is triangulated with the diagonal
//     from the lower-id corner (deterministic and identical from both sides);
//   * old nodes keep their ids, midpoints are appended in ascending edge-key
//     order (edge_key, vec3.hpp:84-87) at (p_a + p_b) * 0.5 in fp64;
//   * children inherit the parent label and are re-oriented to
//     positive volume (mesh.hpp:44-48).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "nestmesh_label.h"

namespace {

inline std::uint64_t ekey(std::uint32_t a, std::uint32_t b) {
  return a < b ? (std::uint64_t(a) << 32 | b) : (std::uint64_t(b) << 32 | a);
}

constexpr int kEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

}  // namespace

#include "refine.h"

#include <cuda_runtime.h>

#include <memory>
#include <mutex>

#include "staging.cuh"

namespace {
thread_local std::string g_refine_err;

// Device-resident result meshes are copied into the caller's (usually
// pageable) arrays through pinned chunk buffers and a host copy pool
// (staging.cuh): ~3x the driver's pageable D2H at cfg4 sizes (4.6 GB).
struct MeshCopier {
  std::mutex m;
  std::unique_ptr<nmh::CopyPool> pool;
  nmh::Stager stager;
  bool get(int device, void* dst, const void* src, std::size_t bytes) {
    if (!dst || !bytes) return true;
    if (!src) return false;
    std::lock_guard<std::mutex> g(m);
    if (!pool) {
      const int hw = static_cast<int>(std::thread::hardware_concurrency());
      pool = std::make_unique<nmh::CopyPool>(std::max(1, std::min(11, hw - 5)));
    }
    cudaStream_t st = nullptr;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      return false;
    bool ok = true;
    try {
      stager.d2h(dst, src, bytes, st, *pool);
    } catch (...) {
      ok = false;
    }
    cudaStreamDestroy(st);
    return ok;
  }
};
MeshCopier& mesh_copier() {
  static MeshCopier c;
  return c;
}
}  // namespace

namespace nmi {

nm_mesh* refine(const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, const int* labels,
                const std::uint32_t* sel, std::size_t ns) {
  for (std::size_t i = 0; i < 4 * nt; ++i)
    if (tets[i] >= n) throw std::invalid_argument("tet references a node out of range");
  for (std::size_t i = 0; i < ns; ++i)
    if (sel[i] >= nt) throw std::invalid_argument("InvalidSelection: selected tet id out of range (SPEC.md:292)");
  // node -> tets CSR (mesh.hpp:292-308)
  std::vector<std::uint32_t> off(n + 1, 0), adj(4 * nt);
  for (std::size_t i = 0; i < 4 * nt; ++i) ++off[tets[i] + 1];
  for (std::size_t i = 0; i < n; ++i) off[i + 1] += off[i];
  {
    std::vector<std::uint32_t> cur(off.begin(), off.end() - 1);
    for (std::size_t t = 0; t < nt; ++t)
      for (int k = 0; k < 4; ++k) adj[cur[tets[4 * t + k]]++] = static_cast<std::uint32_t>(t);
  }
  std::unordered_set<std::uint64_t> split;
  split.reserve(ns * 8 + 16);
  std::vector<std::uint8_t> red(nt, 0);
  std::vector<std::uint32_t> work;
  auto add_edge = [&](std::uint32_t a, std::uint32_t b) {
    if (!split.insert(ekey(a, b)).second) return;
    for (std::uint32_t i = off[a]; i < off[a + 1]; ++i) {
      const std::uint32_t t = adj[i];
      const std::uint32_t* e = tets + 4 * std::size_t(t);
      if (!red[t] && (e[0] == b || e[1] == b || e[2] == b || e[3] == b)) work.push_back(t);
    }
  };
  auto make_red = [&](std::uint32_t t) {
    red[t] = 1;
    const std::uint32_t* e = tets + 4 * std::size_t(t);
    for (auto& ed : kEdge) add_edge(e[ed[0]], e[ed[1]]);
  };
  // pattern: 0 none, 1 one edge, 2 two edges of one face, 3 one full face, -1 escalate
  auto classify = [&](std::uint32_t t, int* which) {
    const std::uint32_t* e = tets + 4 * std::size_t(t);
    int cnt = 0;
    int ids[6];
    for (int k = 0; k < 6; ++k)
      if (split.count(ekey(e[kEdge[k][0]], e[kEdge[k][1]]))) ids[cnt++] = k;
    for (int k = 0; k < cnt; ++k) which[k] = ids[k];
    if (cnt == 0) return 0;
    if (cnt == 1) return 1;
    if (cnt == 6) return -1;
    // vertices touched
    int touched = 0;
    for (int k = 0; k < cnt; ++k) touched |= (1 << kEdge[ids[k]][0]) | (1 << kEdge[ids[k]][1]);
    const int nv = __builtin_popcount(touched);
    if (cnt == 2 && nv == 3) return 2;  // adjacent edges lie on one face
    if (cnt == 3 && nv == 3) return 3;  // a closed triangle = one face
    return -1;
  };
  for (std::size_t i = 0; i < ns; ++i)
    if (!red[sel[i]]) make_red(sel[i]);
  while (!work.empty()) {
    const std::uint32_t t = work.back();
    work.pop_back();
    if (red[t]) continue;
    int which[6];
    if (classify(t, which) < 0) make_red(t);
  }
  // midpoints in ascending edge-key order
  std::vector<std::uint64_t> keys(split.begin(), split.end());
  std::sort(keys.begin(), keys.end());
  auto* out = new nm_mesh;
  out->n_old = n;
  out->nodes.assign(nodes, nodes + 3 * n);
  out->nodes.resize(3 * (n + keys.size()));
  for (std::size_t i = 0; i < keys.size(); ++i) {
    const std::uint32_t a = static_cast<std::uint32_t>(keys[i] >> 32), b = static_cast<std::uint32_t>(keys[i]);
    for (int d = 0; d < 3; ++d) out->nodes[3 * (n + i) + d] = (nodes[3 * std::size_t(a) + d] + nodes[3 * std::size_t(b) + d]) * 0.5;
  }
  auto mid = [&](std::uint32_t a, std::uint32_t b) {
    const std::uint64_t k = ekey(a, b);
    const auto it = std::lower_bound(keys.begin(), keys.end(), k);
    return static_cast<std::uint32_t>(n + (it - keys.begin()));
  };
  const double* P = out->nodes.data();
  auto emit = [&](std::uint32_t a, std::uint32_t b, std::uint32_t c, std::uint32_t d, std::uint32_t parent) {
    std::uint32_t q[4] = {a, b, c, d};
    const double* A = P + 3 * std::size_t(a);
    const double* B = P + 3 * std::size_t(b);
    const double* C = P + 3 * std::size_t(c);
    const double* D = P + 3 * std::size_t(d);
    const double u[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
    const double v[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
    const double w[3] = {D[0] - A[0], D[1] - A[1], D[2] - A[2]};
    const double vol = (u[0] * (v[1] * w[2] - v[2] * w[1]) + u[1] * (v[2] * w[0] - v[0] * w[2]) +
                        u[2] * (v[0] * w[1] - v[1] * w[0])) / 6.0;
    if (vol < 0.0) std::swap(q[2], q[3]);
    out->tets.insert(out->tets.end(), q, q + 4);
    out->labels.push_back(labels ? labels[parent] : 0);
    out->parent.push_back(parent);
  };
  auto dist2 = [&](std::uint32_t a, std::uint32_t b) {
    double s = 0;
    for (int d = 0; d < 3; ++d) {
      const double x = P[3 * std::size_t(a) + d] - P[3 * std::size_t(b) + d];
      s += x * x;
    }
    return s;
  };
  out->tets.reserve(4 * nt + 28 * ns);
  for (std::size_t ti = 0; ti < nt; ++ti) {
    const std::uint32_t t = static_cast<std::uint32_t>(ti);
    const std::uint32_t* e = tets + 4 * ti;
    if (red[t]) {
      const std::uint32_t v0 = e[0], v1 = e[1], v2 = e[2], v3 = e[3];
      const std::uint32_t m01 = mid(v0, v1), m02 = mid(v0, v2), m03 = mid(v0, v3), m12 = mid(v1, v2),
                          m13 = mid(v1, v3), m23 = mid(v2, v3);
      emit(v0, m01, m02, m03, t);
      emit(m01, v1, m12, m13, t);
      emit(m02, m12, v2, m23, t);
      emit(m03, m13, m23, v3, t);
      // octahedron: opposite pairs (m01,m23) (m02,m13) (m03,m12); shortest diagonal
      const std::uint32_t pr[3][2] = {{m01, m23}, {m02, m13}, {m03, m12}};
      int best = 0;
      double bd = dist2(pr[0][0], pr[0][1]);
      for (int k = 1; k < 3; ++k) {
        const double d = dist2(pr[k][0], pr[k][1]);
        const auto lk = std::minmax(pr[k][0], pr[k][1]), lb = std::minmax(pr[best][0], pr[best][1]);
        if (d < bd || (d == bd && lk < lb)) {
          bd = d;
          best = k;
        }
      }
      const std::uint32_t p = pr[best][0], q = pr[best][1];
      const std::uint32_t a = pr[(best + 1) % 3][0], a2 = pr[(best + 1) % 3][1];
      const std::uint32_t b = pr[(best + 2) % 3][0], b2 = pr[(best + 2) % 3][1];
      emit(p, q, a, b, t);
      emit(p, q, b, a2, t);
      emit(p, q, a2, b2, t);
      emit(p, q, b2, a, t);
      continue;
    }
    int which[6];
    const int pat = classify(t, which);
    if (pat == 0) {
      out->tets.insert(out->tets.end(), e, e + 4);
      out->labels.push_back(labels ? labels[t] : 0);
      out->parent.push_back(t);
    } else if (pat == 1) {
      const std::uint32_t a = e[kEdge[which[0]][0]], b = e[kEdge[which[0]][1]];
      std::uint32_t o[2];
      int k = 0;
      for (int j = 0; j < 4; ++j)
        if (e[j] != a && e[j] != b) o[k++] = e[j];
      const std::uint32_t m = mid(a, b);
      emit(a, m, o[0], o[1], t);
      emit(m, b, o[0], o[1], t);
    } else if (pat == 2) {
      // split edges (a,b) and (a,c) share a; d is the apex
      const int* E0 = kEdge[which[0]];
      const int* E1 = kEdge[which[1]];
      const int ia = (E0[0] == E1[0] || E0[0] == E1[1]) ? E0[0] : E0[1];
      const int ib = E0[0] == ia ? E0[1] : E0[0];
      const int ic = E1[0] == ia ? E1[1] : E1[0];
      const int id = 6 - ia - ib - ic;
      const std::uint32_t a = e[ia], b = e[ib], c = e[ic], d = e[id];
      const std::uint32_t mab = mid(a, b), mac = mid(a, c);
      emit(d, a, mab, mac, t);
      if (c < b) {  // diagonal (mab, c)
        emit(d, mab, b, c, t);
        emit(d, mab, c, mac, t);
      } else {  // diagonal (b, mac)
        emit(d, mab, b, mac, t);
        emit(d, b, c, mac, t);
      }
    } else {
      // one face fully split, apex d
      int touched = 0;
      for (int k = 0; k < 3; ++k) touched |= (1 << kEdge[which[k]][0]) | (1 << kEdge[which[k]][1]);
      int id = 0;
      while (touched & (1 << id)) ++id;
      int f[3], k = 0;
      for (int j = 0; j < 4; ++j)
        if (j != id) f[k++] = j;
      const std::uint32_t a = e[f[0]], b = e[f[1]], c = e[f[2]], d = e[id];
      const std::uint32_t mab = mid(a, b), mbc = mid(b, c), mca = mid(c, a);
      emit(d, a, mab, mca, t);
      emit(d, mab, b, mbc, t);
      emit(d, mca, mbc, c, t);
      emit(d, mab, mbc, mca, t);
    }
  }
  return out;
}

}  // namespace nmi

extern "C" {

const char* nm_refine_last_error(void) { return g_refine_err.c_str(); }

int nm_refine(const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, const int* labels,
              const std::uint32_t* selected, std::size_t ns, nm_mesh** out) {
  try {
    *out = nmi::refine(nodes, n, tets, nt, labels, selected, ns);
    return 0;
  } catch (const std::exception& e) {
    g_refine_err = e.what();
    *out = nullptr;
    return 1;
  }
}

int nm_mesh_sizes(const nm_mesh* m, std::size_t* n_nodes, std::size_t* n_tets, std::size_t* n_old_nodes) {
  if (!m) return 1;
  if (n_nodes) *n_nodes = m->node_count();
  if (n_tets) *n_tets = m->tet_count();
  if (n_old_nodes) *n_old_nodes = m->n_old;
  return 0;
}

int nm_mesh_copy(const nm_mesh* m, double* nodes, std::uint32_t* tets, int* labels, std::uint32_t* parent) {
  if (!m) return 1;
  if (m->dev.device >= 0) {
    const auto& d = m->dev;
    if (cudaSetDevice(d.device) != cudaSuccess) return 1;
    auto get = [&](void* dst, const void* src, std::size_t bytes) { return mesh_copier().get(d.device, dst, src, bytes); };
    const bool ok = get(nodes, d.nodes, 3 * d.nn * sizeof(double)) && get(tets, d.tets, 4 * d.nt * sizeof(std::uint32_t)) &&
                    get(labels, d.labels, d.nt * sizeof(int)) && get(parent, d.parent, d.nt * sizeof(std::uint32_t));
    return ok ? 0 : 1;
  }
  if (nodes) std::memcpy(nodes, m->nodes.data(), m->nodes.size() * sizeof(double));
  if (tets) std::memcpy(tets, m->tets.data(), m->tets.size() * sizeof(std::uint32_t));
  if (labels) std::memcpy(labels, m->labels.data(), m->labels.size() * sizeof(int));
  if (parent) std::memcpy(parent, m->parent.data(), m->parent.size() * sizeof(std::uint32_t));
  return 0;
}

void nm_mesh_free(nm_mesh* m) { delete m; }

// Area-uniform samples on a triangle surface ("triangle-area-
// weighted random points with fixed seed"): splitmix64 stream; triangle by
// binary search on the fp64 cumulative area; barycentric
// (1 - sqrt(r1), sqrt(r1)(1 - r2), sqrt(r1) r2).
int nm_sample_surface(const double* xyz, const std::uint32_t* tri, std::size_t nt, std::size_t count,
                      std::uint64_t seed, double* out) {
  if (nt == 0) return 1;
  std::vector<double> cum(nt);
  double acc = 0.0;
  for (std::size_t t = 0; t < nt; ++t) {
    const double* a = xyz + 3 * std::size_t(tri[3 * t]);
    const double* b = xyz + 3 * std::size_t(tri[3 * t + 1]);
    const double* c = xyz + 3 * std::size_t(tri[3 * t + 2]);
    const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double x = u[1] * v[2] - u[2] * v[1], y = u[2] * v[0] - u[0] * v[2], z = u[0] * v[1] - u[1] * v[0];
    acc += 0.5 * std::sqrt(x * x + y * y + z * z);
    cum[t] = acc;
  }
  std::uint64_t state = seed;
  auto next = [&]() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return double(z >> 11) * (1.0 / 9007199254740992.0);
  };
  for (std::size_t i = 0; i < count; ++i) {
    const double r0 = next() * acc, r1 = next(), r2 = next();
    std::size_t t = static_cast<std::size_t>(std::upper_bound(cum.begin(), cum.end(), r0) - cum.begin());
    if (t >= nt) t = nt - 1;
    const double* a = xyz + 3 * std::size_t(tri[3 * t]);
    const double* b = xyz + 3 * std::size_t(tri[3 * t + 1]);
    const double* c = xyz + 3 * std::size_t(tri[3 * t + 2]);
    const double s1 = std::sqrt(r1);
    const double w0 = 1.0 - s1, w1 = s1 * (1.0 - r2), w2 = s1 * r2;
    for (int d = 0; d < 3; ++d) out[3 * i + d] = w0 * a[d] + w1 * b[d] + w2 * c[d];
  }
  return 0;
}

int nm_mesh_masks(const nm_mesh* m, std::uint32_t* masks) {
  if (!m) return 1;
  if (m->dev.device >= 0) {
    if (!m->dev.masks) return 1;
    return mesh_copier().get(m->dev.device, masks, m->dev.masks, m->dev.nn * sizeof(std::uint32_t)) ? 0 : 1;
  }
  if (m->masks.size() != m->nodes.size() / 3) return 1;
  std::memcpy(masks, m->masks.data(), m->masks.size() * sizeof(std::uint32_t));
  return 0;
}

}  // extern "C"

nm_mesh::~nm_mesh() {
  if (dev.device < 0) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev.device);
  for (void* p : {dev.nodes, dev.tets, dev.labels, dev.parent, dev.masks})
    if (p) cudaFreeAsync(p, cudaStreamLegacy);  // pool memory; every use completed before the handle was returned
  cudaSetDevice(prev);
}
