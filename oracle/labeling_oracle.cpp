// ============================================================================
// TEST INFRASTRUCTURE ONLY — CPU fp64 oracle for recursive solid-angle labeling.
//
// This file is the checker, never the product: only tests/, the smoke() check
// in __graft_entry__.py and the cpu_baseline / --impl reference legs of
// bench.py may load it. The product path (libnestmesh_label.so) never links
// or calls it.
//
// The reference (/root/reference, "nestmesh") specifies the labeling module
// only in SPEC.md; proj/include/nestmesh has no labeling code. This is a plain
// restatement of that specification over the reference's fp64 arithmetic:
//
//   enclosure_ratio   SPEC.md:225-233, 261  s = (1/4pi) sum_tri Omega_tri,
//                     Omega = 2*atan2(num, den) (Van Oosterom-Strackee):
//                       num = R1 . (R2 x R3)
//                       den = r1 r2 r3 + (R1.R2) r3 + (R1.R3) r2 + (R2.R3) r1
//                     with R_i = v_i - p; dot/cross/norm in the operand order
//                     of proj/include/nestmesh/vec3.hpp:32-38; triangles summed
//                     sequentially in file order.
//   inside            SPEC.md:237, 260, 263  inside_k iff s_k >= T (tie inside).
//   node mask         SPEC.md:160, 168  threshold per surface first, then
//                     priority: bit k = sequence position k (innermost first).
//   tet label         SPEC.md:237, PAPER.md:148  label = id[k] for the lowest
//                     k with all four nodes inside k, else 0.
//   relabel_recursive SPEC.md:243-251, PAPER.md:151  frontier = nodes of the
//                     tets adjacent to label-change faces; iterate until a pass
//                     changes no label; max_iters -> NonConvergence.
//   straddle flags    SPEC.md:294 (refine_boundary layer): a tet straddles an
//                     active boundary when OR != AND of its node masks on the
//                     active bits.
//   workers           SPEC.md:265  points are partitioned into contiguous
//                     ranges; every point is a pure function of its inputs, so
//                     the result is independent of the worker count.
//
// Parity pinning: SPEC.md KATs (:231-233, :240-242, :249-257) encoded in
// tests/golden/spec_kats.json and tests/test_oracle.py; analytic solid angles
// (cube face/edge/corner, single triangle closed forms) and an independent
// L'Huilier-formula cross-check. No reference golden vectors exist for this
// path.
//
// Build rules (oracle/Makefile): -O2 -ffp-contract=off, no -ffast-math, so the
// fp64 bits do not depend on FMA contraction.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

struct V3 {
  double x, y, z;
};
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
// vec3.hpp:32
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
// vec3.hpp:34-36
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// vec3.hpp:38
inline double norm(const V3& v) { return std::sqrt(dot(v, v)); }

inline V3 load(const double* xyz, std::size_t i) { return {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}; }

// One Van Oosterom-Strackee half solid angle atan2(num, den).
inline double vos_half_angle(const V3& p, const V3& a, const V3& b, const V3& c) {
  const V3 r1 = sub(a, p), r2 = sub(b, p), r3 = sub(c, p);
  const double l1 = norm(r1), l2 = norm(r2), l3 = norm(r3);
  const double num = dot(r1, cross(r2, r3));
  const double den = l1 * l2 * l3 + dot(r1, r2) * l3 + dot(r1, r3) * l2 + dot(r2, r3) * l1;
  return std::atan2(num, den);
}

// s = sum Omega / 4pi = sum atan2 / 2pi over triangles [t0, t1).
inline double enclosure(const V3& p, const double* xyz, const std::uint32_t* tri, std::size_t t0,
                        std::size_t t1) {
  double sum = 0.0;
  for (std::size_t t = t0; t < t1; ++t) {
    sum += vos_half_angle(p, load(xyz, tri[3 * t]), load(xyz, tri[3 * t + 1]), load(xyz, tri[3 * t + 2]));
  }
  return sum / (2.0 * std::numbers::pi);
}

template <class F>
void parallel_for(std::size_t n, int workers, F&& f) {
  if (workers <= 0) workers = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  workers = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(workers), std::max<std::size_t>(n, 1)));
  if (workers <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const std::size_t lo = std::min(n, w * chunk), hi = std::min(n, lo + chunk);
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

// Label of a tet from the AND of its node masks.
inline int tet_label(std::uint32_t m_and, const int* label_ids) {
  return m_and ? label_ids[__builtin_ctz(m_and)] : 0;
}

}  // namespace

extern "C" {

int oracle_version(void) { return 1; }

// s_out[i*K + k] = enclosure ratio of point i w.r.t. compartment k, whose
// triangles are tri[comp_off[k] .. comp_off[k+1]).
int oracle_enclosure(const double* pts, std::size_t n, const double* xyz, const std::uint32_t* tri,
                     const std::uint32_t* comp_off, int K, int workers, double* s_out) {
  parallel_for(n, workers, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const V3 p = load(pts, i);
      for (int k = 0; k < K; ++k) s_out[i * K + k] = enclosure(p, xyz, tri, comp_off[k], comp_off[k + 1]);
    }
  });
  return 0;
}

// masks_out[i] bit k = (s_k >= T). s_out optional (n*K).
int oracle_label_nodes(const double* pts, std::size_t n, const double* xyz, const std::uint32_t* tri,
                       const std::uint32_t* comp_off, int K, double T, int workers, std::uint32_t* masks_out,
                       double* s_out) {
  if (K < 0 || K > 32) return 1;
  parallel_for(n, workers, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const V3 p = load(pts, i);
      std::uint32_t m = 0;
      for (int k = 0; k < K; ++k) {
        const double s = enclosure(p, xyz, tri, comp_off[k], comp_off[k + 1]);
        if (s_out) s_out[i * K + k] = s;
        if (s >= T) m |= 1u << k;
      }
      masks_out[i] = m;
    }
  });
  return 0;
}

// labels_out[t] = label_ids[lowest k inside at all four nodes], else 0.
int oracle_label_tets(const std::uint32_t* tets, std::size_t nt, const std::uint32_t* masks, const int* label_ids,
                      int K, int* labels_out) {
  (void)K;
  for (std::size_t t = 0; t < nt; ++t) {
    const std::uint32_t* e = tets + 4 * t;
    labels_out[t] = tet_label(masks[e[0]] & masks[e[1]] & masks[e[2]] & masks[e[3]], label_ids);
  }
  return 0;
}

// Tets whose node masks disagree on an active compartment, in ascending order.
std::size_t oracle_flag_boundary(const std::uint32_t* tets, std::size_t nt, const std::uint32_t* masks,
                                 std::uint32_t active_mask, std::uint32_t* ids_out) {
  std::size_t c = 0;
  for (std::size_t t = 0; t < nt; ++t) {
    const std::uint32_t* e = tets + 4 * t;
    const std::uint32_t a = masks[e[0]] & masks[e[1]] & masks[e[2]] & masks[e[3]];
    const std::uint32_t o = masks[e[0]] | masks[e[1]] | masks[e[2]] | masks[e[3]];
    if ((a ^ o) & active_mask) ids_out[c++] = static_cast<std::uint32_t>(t);
  }
  return c;
}

// relabel_recursive. labels_io holds prev_labels on entry
// and the result on exit. Returns the number of passes; *converged is 1 when a
// pass changed no label within max_iters. evaluated_out (optional, n_nodes)
// receives 1 for every node whose enclosure was evaluated.
int oracle_relabel_recursive(const double* nodes, std::size_t n_nodes, const std::uint32_t* tets, std::size_t nt,
                             const double* xyz, const std::uint32_t* tri, const std::uint32_t* comp_off,
                             const int* label_ids, int K, double T, int max_iters, int workers, int* labels_io,
                             int* converged, std::uint8_t* evaluated_out, std::size_t* n_evaluated) {
  // Face adjacency (mesh.hpp:68-88): sorted node triple -> incident tets.
  struct Key {
    std::uint32_t a, b, c;
    bool operator==(const Key& o) const { return a == o.a && b == o.b && c == o.c; }
  };
  struct KeyHash {
    std::size_t operator()(const Key& k) const {
      std::uint64_t h = 1469598103934665603ull;
      for (std::uint64_t v : {k.a, k.b, k.c}) h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      return static_cast<std::size_t>(h);
    }
  };
  auto key_of = [](std::uint32_t i, std::uint32_t j, std::uint32_t k) {
    if (i > j) std::swap(i, j);
    if (j > k) std::swap(j, k);
    if (i > j) std::swap(i, j);
    return Key{i, j, k};
  };
  std::unordered_map<Key, std::int64_t, KeyHash> first;
  first.reserve(nt * 2);
  std::vector<std::int64_t> nbr(4 * nt, -1);  // face-neighbour across local face f of tet t
  static const int F[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};  // mesh.hpp:57-64
  for (std::size_t t = 0; t < nt; ++t) {
    const std::uint32_t* e = tets + 4 * t;
    for (int f = 0; f < 4; ++f) {
      const Key key = key_of(e[F[f][0]], e[F[f][1]], e[F[f][2]]);
      auto [it, ins] = first.try_emplace(key, static_cast<std::int64_t>(4 * t + f));
      if (!ins) {
        const std::int64_t o = it->second;
        nbr[4 * t + f] = o / 4;
        nbr[o] = static_cast<std::int64_t>(t);
      }
    }
  }
  std::vector<std::uint32_t> mask(n_nodes, 0);
  std::vector<std::uint8_t> known(n_nodes, 0);
  std::size_t evaluated = 0;
  int passes = 0;
  *converged = 0;
  for (int pass = 1; pass <= max_iters; ++pass) {
    passes = pass;
    // Frontier: nodes of tets adjacent to a label-change face.
    std::vector<std::uint8_t> want(n_nodes, 0);
    for (std::size_t t = 0; t < nt; ++t) {
      bool adj = false;
      for (int f = 0; f < 4 && !adj; ++f) {
        const std::int64_t o = nbr[4 * t + f];
        if (o >= 0 && labels_io[o] != labels_io[t]) adj = true;
      }
      if (!adj) continue;
      for (int v = 0; v < 4; ++v) want[tets[4 * t + v]] = 1;
    }
    std::vector<std::uint32_t> todo;
    for (std::size_t v = 0; v < n_nodes; ++v)
      if (want[v] && !known[v]) todo.push_back(static_cast<std::uint32_t>(v));
    parallel_for(todo.size(), workers, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t i = lo; i < hi; ++i) {
        const std::uint32_t v = todo[i];
        const V3 p = load(nodes, v);
        std::uint32_t m = 0;
        for (int k = 0; k < K; ++k)
          if (enclosure(p, xyz, tri, comp_off[k], comp_off[k + 1]) >= T) m |= 1u << k;
        mask[v] = m;
      }
    });
    for (std::uint32_t v : todo) known[v] = 1;
    evaluated += todo.size();
    // Label update barrier: every tet whose four nodes are evaluated.
    std::size_t changed = 0;
    for (std::size_t t = 0; t < nt; ++t) {
      const std::uint32_t* e = tets + 4 * t;
      if (!(known[e[0]] && known[e[1]] && known[e[2]] && known[e[3]])) continue;
      const int l = tet_label(mask[e[0]] & mask[e[1]] & mask[e[2]] & mask[e[3]], label_ids);
      if (l != labels_io[t]) {
        labels_io[t] = l;
        ++changed;
      }
    }
    if (changed == 0) {
      *converged = 1;
      break;
    }
  }
  if (evaluated_out) std::memcpy(evaluated_out, known.data(), n_nodes);
  if (n_evaluated) *n_evaluated = evaluated;
  return passes;
}

// quality.boundary_distance restatement: unsigned distance
// to a triangle surface = sqrt(min over triangles of the exact squared
// point-triangle distance): the plane distance when p projects inside the
// triangle (all three edge-side tests >= 0), else the nearest edge segment
// (clamped projection). Operand order of vec3.hpp:32-38, no FMA.
namespace {
inline double seg_dist2(const V3& ap, const V3& e) {
  const double ee = dot(e, e);
  double t = ee > 0.0 ? dot(ap, e) / ee : 0.0;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const V3 v{ap.x - t * e.x, ap.y - t * e.y, ap.z - t * e.z};
  return dot(v, v);
}
inline double point_tri_dist2(const V3& p, const V3& a, const V3& b, const V3& c) {
  const V3 ab = sub(b, a), bc = sub(c, b), ca = sub(a, c);
  const V3 ap = sub(p, a), bp = sub(p, b), cp = sub(p, c);
  const V3 n = cross(ab, sub(c, a));
  const double nn = dot(n, n);
  const double s0 = dot(cross(ab, ap), n), s1 = dot(cross(bc, bp), n), s2 = dot(cross(ca, cp), n);
  if (nn > 0.0 && s0 >= 0.0 && s1 >= 0.0 && s2 >= 0.0) {
    const double h = dot(ap, n);
    return (h * h) / nn;
  }
  double d = seg_dist2(ap, ab);
  const double d1 = seg_dist2(bp, bc), d2 = seg_dist2(cp, ca);
  d = d1 < d ? d1 : d;
  return d2 < d ? d2 : d;
}
}  // namespace

int oracle_point_surface_distance(const double* pts, std::size_t n, const double* xyz, const std::uint32_t* tri,
                                  std::size_t nt, int workers, double* out) {
  parallel_for(n, workers, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const V3 p = load(pts, i);
      double best = 1e300;
      for (std::size_t t = 0; t < nt; ++t) {
        const double q = point_tri_dist2(p, load(xyz, tri[3 * t]), load(xyz, tri[3 * t + 1]), load(xyz, tri[3 * t + 2]));
        best = q < best ? q : best;
      }
      out[i] = std::sqrt(best);
    }
  });
  return 0;
}

// Independent cross-check formula: L'Huilier's theorem for the solid angle of
// a spherical triangle, signed by orientation. Used only by tests to pin the
// VOS restatement (both must agree to ~1e-12 away from the surface).
double oracle_lhuilier_solid_angle(const double* p, const double* a, const double* b, const double* c) {
  const V3 P{p[0], p[1], p[2]};
  V3 u[3] = {sub(V3{a[0], a[1], a[2]}, P), sub(V3{b[0], b[1], b[2]}, P), sub(V3{c[0], c[1], c[2]}, P)};
  for (auto& w : u) {
    const double n = norm(w);
    w = {w.x / n, w.y / n, w.z / n};
  }
  auto arc = [](const V3& x, const V3& y) {
    const V3 d = sub(x, y);
    return 2.0 * std::asin(std::min(1.0, norm(d) / 2.0));
  };
  const double A = arc(u[1], u[2]), B = arc(u[0], u[2]), C = arc(u[0], u[1]);
  const double s = 0.5 * (A + B + C);
  const double t = std::tan(s / 2) * std::tan((s - A) / 2) * std::tan((s - B) / 2) * std::tan((s - C) / 2);
  const double E = 4.0 * std::atan(std::sqrt(std::max(0.0, t)));
  const double sign = dot(u[0], cross(u[1], u[2])) >= 0 ? 1.0 : -1.0;
  return sign * E;
}

}  // extern "C"
