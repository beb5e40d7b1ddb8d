// TEST INFRASTRUCTURE ONLY — fp64 CPU restatement of refine_volume
// with the SPEC's design decisions and its
// open-question resolution. Only tests/ may load this library;
// the product path (paper_2203_10000_b200/) never does.
//
// It is written independently of the product's csrc/refine.cpp and
// csrc/refine.cuh, from the SPEC text:
//   * selection closure as a fixed point of whole-mesh sweeps (the product
//     uses a worklist over node->tet adjacency); an unselected tet is a
//     transition element iff its split edges all lie in ONE face
//     (Fig. 2(c-e): 1 edge, 2 edges of a face, the 3 edges of a face);
//     anything else — two opposite edges, an edge star or path over 4
//     vertices, >= 4 edges — escalates to the 1:8 split;
//   * midpoints: fp64 0.5*(p_a + p_b), numbered after the old nodes in
//     ascending (lo, hi) edge order (the shared numbering convention; SPEC
//     does not fix one);
//   * 1:8 split: 4 corner tets + the central octahedron cut
//     along its shortest diagonal, ties to the lexicographically smallest
//     (min id, max id) midpoint pair; the octahedron tets
//     fan around the diagonal over the equator cycle (consecutive equator
//     midpoints share an original vertex);
//   * Fig. 2(d): a face with two split edges ab, ac: corner (a, m_ab, m_ac),
//     quad (m_ab, b, c, m_ac) cut from its lower-id original corner
//     ("tie-breaks by lowest node index");
//   * Fig. 2(e): a fully split face: 4 children over the apex;
//   * children inherit the parent's label and are oriented to
//     positive fp64 volume (mesh.hpp:44-48 normalize_orientation).
// Child ORDER inside a parent is not specified by the SPEC; tests compare
// children as (parent, sorted node ids) sets.
#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

namespace {

using Id = std::uint32_t;
using EdgeKey = std::pair<Id, Id>;  // (lo, hi)

EdgeKey edge(Id a, Id b) { return a < b ? EdgeKey{a, b} : EdgeKey{b, a}; }
std::uint64_t pack(EdgeKey e) { return (std::uint64_t(e.first) << 32) | e.second; }

struct OracleMesh {
  std::vector<double> nodes;
  std::vector<Id> tets;
  std::vector<int> labels;
  std::vector<Id> parent;
  std::size_t n_old = 0;
};

thread_local std::string g_err;

// the six local edges of a tet and the local vertices of its four faces
constexpr int kLocalEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
constexpr int kFaceOmit[4] = {0, 1, 2, 3};  // face f = the three vertices other than f

double signed_volume(const double* P, Id a, Id b, Id c, Id d) {
  const double* A = P + 3 * std::size_t(a);
  const double* B = P + 3 * std::size_t(b);
  const double* C = P + 3 * std::size_t(c);
  const double* D = P + 3 * std::size_t(d);
  double u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) {
    u[k] = B[k] - A[k];
    v[k] = C[k] - A[k];
    w[k] = D[k] - A[k];
  }
  // u . (v x w) / 6 (vec3.hpp:79-81 tet_signed_volume)
  const double cx = v[1] * w[2] - v[2] * w[1];
  const double cy = v[2] * w[0] - v[0] * w[2];
  const double cz = v[0] * w[1] - v[1] * w[0];
  return (u[0] * cx + u[1] * cy + u[2] * cz) / 6.0;
}

OracleMesh* refine_oracle(const double* nodes, std::size_t n, const Id* tets, std::size_t nt, const int* labels,
                          const Id* sel, std::size_t ns) {
  for (std::size_t i = 0; i < 4 * nt; ++i)
    if (tets[i] >= n) throw std::invalid_argument("tet node index out of range");
  for (std::size_t i = 0; i < ns; ++i)
    if (sel[i] >= nt) throw std::invalid_argument("InvalidSelection");

  std::vector<char> red(nt, 0);
  std::unordered_set<std::uint64_t> split;
  auto split_all_edges = [&](std::size_t t) {
    const Id* v = tets + 4 * t;
    for (const auto& le : kLocalEdge) split.insert(pack(edge(v[le[0]], v[le[1]])));
  };
  for (std::size_t i = 0; i < ns; ++i) red[sel[i]] = 1;
  for (std::size_t t = 0; t < nt; ++t)
    if (red[t]) split_all_edges(t);

  // which local edges of t are split (bit k = kLocalEdge[k])
  auto split_bits = [&](std::size_t t) {
    const Id* v = tets + 4 * t;
    int bits = 0;
    for (int k = 0; k < 6; ++k)
      if (split.count(pack(edge(v[kLocalEdge[k][0]], v[kLocalEdge[k][1]])))) bits |= 1 << k;
    return bits;
  };
  // the face (omitted local vertex) containing every split edge, or -1
  auto face_holding = [&](int bits) {
    for (int f : kFaceOmit) {
      bool all = true;
      for (int k = 0; k < 6; ++k)
        if (((bits >> k) & 1) && (kLocalEdge[k][0] == f || kLocalEdge[k][1] == f)) all = false;
      if (all) return f;
    }
    return -1;
  };
  // closure: sweep until no unselected tet has a non-template pattern
  for (bool changed = true; changed;) {
    changed = false;
    for (std::size_t t = 0; t < nt; ++t) {
      if (red[t]) continue;
      const int bits = split_bits(t);
      if (bits == 0) continue;
      if (face_holding(bits) < 0) {
        red[t] = 1;
        split_all_edges(t);
        changed = true;
      }
    }
  }

  std::vector<EdgeKey> edges;
  edges.reserve(split.size());
  for (std::uint64_t k : split) edges.emplace_back(Id(k >> 32), Id(k & 0xffffffffu));
  std::sort(edges.begin(), edges.end());
  std::map<EdgeKey, Id> mid_id;
  auto* out = new OracleMesh;
  out->n_old = n;
  out->nodes.assign(nodes, nodes + 3 * n);
  for (std::size_t i = 0; i < edges.size(); ++i) {
    mid_id.emplace(edges[i], Id(n + i));
    const double* A = nodes + 3 * std::size_t(edges[i].first);
    const double* B = nodes + 3 * std::size_t(edges[i].second);
    for (int k = 0; k < 3; ++k) out->nodes.push_back(0.5 * (A[k] + B[k]));
  }
  const double* P = out->nodes.data();
  auto M = [&](Id a, Id b) { return mid_id.at(edge(a, b)); };
  auto child = [&](std::array<Id, 4> q, std::size_t t) {
    if (signed_volume(P, q[0], q[1], q[2], q[3]) < 0.0) std::swap(q[0], q[1]);
    out->tets.insert(out->tets.end(), q.begin(), q.end());
    out->labels.push_back(labels ? labels[t] : 0);
    out->parent.push_back(Id(t));
  };
  auto len2 = [&](Id a, Id b) {
    const double dx = P[3 * std::size_t(a)] - P[3 * std::size_t(b)];
    const double dy = P[3 * std::size_t(a) + 1] - P[3 * std::size_t(b) + 1];
    const double dz = P[3 * std::size_t(a) + 2] - P[3 * std::size_t(b) + 2];
    return dx * dx + dy * dy + dz * dz;
  };

  for (std::size_t t = 0; t < nt; ++t) {
    const Id* v = tets + 4 * t;
    if (red[t]) {
      // corner tets
      for (int i = 0; i < 4; ++i) {
        std::array<Id, 4> q;
        q[0] = v[i];
        int k = 1;
        for (int j = 0; j < 4; ++j)
          if (j != i) q[k++] = M(v[i], v[j]);
        child(q, t);
      }
      // central octahedron: opposite local edges (01|23), (02|13), (03|12)
      const int opp[3][2] = {{0, 5}, {1, 4}, {2, 3}};  // indices into kLocalEdge
      int best = -1;
      double bl = 0.0;
      EdgeKey bk{};
      for (int d = 0; d < 3; ++d) {
        const Id p = M(v[kLocalEdge[opp[d][0]][0]], v[kLocalEdge[opp[d][0]][1]]);
        const Id q = M(v[kLocalEdge[opp[d][1]][0]], v[kLocalEdge[opp[d][1]][1]]);
        const double l = len2(p, q);
        const EdgeKey k = edge(p, q);
        if (best < 0 || l < bl || (l == bl && k < bk)) {
          best = d;
          bl = l;
          bk = k;
        }
      }
      // equator: the four local edges not on the diagonal, as a cycle of
      // edges sharing an original vertex
      std::vector<int> eq;
      for (int k = 0; k < 6; ++k)
        if (k != opp[best][0] && k != opp[best][1]) eq.push_back(k);
      std::vector<int> cyc{eq[0]};
      std::vector<char> used(4, 0);
      used[0] = 1;
      while (cyc.size() < 4) {
        const int last = cyc.back();
        for (int j = 0; j < 4; ++j) {
          const int k = eq[j];
          if (used[j]) continue;
          const bool share = kLocalEdge[k][0] == kLocalEdge[last][0] || kLocalEdge[k][0] == kLocalEdge[last][1] ||
                             kLocalEdge[k][1] == kLocalEdge[last][0] || kLocalEdge[k][1] == kLocalEdge[last][1];
          if (share) {
            used[j] = 1;
            cyc.push_back(k);
            break;
          }
        }
      }
      const Id p = bk.first, q = bk.second;
      for (int j = 0; j < 4; ++j) {
        const int a = cyc[j], b = cyc[(j + 1) % 4];
        child({p, q, M(v[kLocalEdge[a][0]], v[kLocalEdge[a][1]]), M(v[kLocalEdge[b][0]], v[kLocalEdge[b][1]])}, t);
      }
      continue;
    }
    const int bits = split_bits(t);
    const int cnt = __builtin_popcount(unsigned(bits));
    if (cnt == 0) {
      out->tets.insert(out->tets.end(), v, v + 4);
      out->labels.push_back(labels ? labels[t] : 0);
      out->parent.push_back(Id(t));
      continue;
    }
    const int f = face_holding(bits);  // apex = local vertex f
    const Id d = v[f];
    std::vector<Id> face;
    for (int j = 0; j < 4; ++j)
      if (j != f) face.push_back(v[j]);
    if (cnt == 1) {  // Fig. 2(c)
      int k = 0;
      while (!((bits >> k) & 1)) ++k;
      const Id a = v[kLocalEdge[k][0]], b = v[kLocalEdge[k][1]];
      std::vector<Id> o;
      for (int j = 0; j < 4; ++j)
        if (v[j] != a && v[j] != b) o.push_back(v[j]);
      const Id m = M(a, b);
      child({a, m, o[0], o[1]}, t);
      child({m, b, o[0], o[1]}, t);
    } else if (cnt == 2) {  // Fig. 2(d)
      // a = the face vertex on both split edges; b, c the others
      Id a = 0;
      for (Id x : face) {
        int on = 0;
        for (int k = 0; k < 6; ++k)
          if (((bits >> k) & 1) && (v[kLocalEdge[k][0]] == x || v[kLocalEdge[k][1]] == x)) ++on;
        if (on == 2) a = x;
      }
      Id b = 0, c = 0;
      bool first = true;
      for (Id x : face)
        if (x != a) {
          (first ? b : c) = x;
          first = false;
        }
      const Id mab = M(a, b), mac = M(a, c);
      child({d, a, mab, mac}, t);
      const Id lo = std::min(b, c);  // quad (mab, b, c, mac): diagonal from its lower-id original corner
      if (lo == b) {
        child({d, mab, b, mac}, t);
        child({d, b, c, mac}, t);
      } else {
        child({d, mab, b, c}, t);
        child({d, mab, c, mac}, t);
      }
    } else {  // cnt == 3, Fig. 2(e)
      const Id a = face[0], b = face[1], c = face[2];
      const Id mab = M(a, b), mbc = M(b, c), mca = M(c, a);
      child({d, a, mab, mca}, t);
      child({d, b, mbc, mab}, t);
      child({d, c, mca, mbc}, t);
      child({d, mab, mbc, mca}, t);
    }
  }
  return out;
}

}  // namespace

extern "C" {

const char* oracle_refine_last_error(void) { return g_err.c_str(); }

void* oracle_refine(const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, const int* labels,
                    const std::uint32_t* sel, std::size_t ns) {
  try {
    return refine_oracle(nodes, n, tets, nt, labels, sel, ns);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void oracle_refine_sizes(const void* h, std::size_t* n_nodes, std::size_t* n_tets) {
  const auto* m = static_cast<const OracleMesh*>(h);
  *n_nodes = m->nodes.size() / 3;
  *n_tets = m->tets.size() / 4;
}

void oracle_refine_copy(const void* h, double* nodes, std::uint32_t* tets, int* labels, std::uint32_t* parent) {
  const auto* m = static_cast<const OracleMesh*>(h);
  std::memcpy(nodes, m->nodes.data(), m->nodes.size() * sizeof(double));
  std::memcpy(tets, m->tets.data(), m->tets.size() * sizeof(std::uint32_t));
  std::memcpy(labels, m->labels.data(), m->labels.size() * sizeof(int));
  std::memcpy(parent, m->parent.data(), m->parent.size() * sizeof(std::uint32_t));
}

void oracle_refine_free(void* h) { delete static_cast<OracleMesh*>(h); }

}  // extern "C"
