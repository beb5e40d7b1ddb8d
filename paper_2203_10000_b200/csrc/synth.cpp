// Synthetic inputs for the labeling path: icosphere / box surfaces, the
// regular 5-tet lattice, and the five BASELINE.json configurations.
//
// These are the CALLER's side of the labeling boundary (SURVEY.md §2 #3, #5:
// lattice and surface generators stay CPU). They are re-implemented here (not
// copied) so the bench and the GPU-box tests can build inputs without
// /root/reference, and are pinned against the reference generators compiled
// in oracle/_ref (tests/test_synth.py) to produce bit-identical geometry:
//   icosphere             proj/include/nestmesh/primitives.hpp:13-54
//   box_surface           proj/include/nestmesh/primitives.hpp:75-87
//   generate_lattice_mesh proj/include/nestmesh/lattice.hpp:40-91
//   lattice_covering      proj/include/nestmesh/lattice.hpp:25-34
// Config geometry follows SURVEY.md §8(d).
//
// Compiled with -ffp-contract=off so the fp64 geometry is identical to the
// reference generators' bits.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numbers>
#include <random>
#include <string>
#include <vector>

namespace {

struct P3 {
  double x, y, z;
};

inline double dot3(const P3& a, const P3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline P3 unit(const P3& v) {
  const double n = std::sqrt(dot3(v, v));
  return n > 0.0 ? P3{v.x / n, v.y / n, v.z / n} : P3{0, 0, 0};
}

struct Mesh {
  std::vector<P3> v;
  std::vector<std::uint32_t> t;  // 3 per triangle
};

// 20-face icosahedron on the unit sphere; vertex/face order of the reference
// so that subdivision yields the same triangle sequence.
Mesh base_icosahedron() {
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  const double s = 1.0 / std::sqrt(1.0 + phi * phi);
  const double a = s, b = s * phi;
  Mesh m;
  m.v = {{-a, b, 0}, {a, b, 0},  {-a, -b, 0}, {a, -b, 0}, {0, -a, b}, {0, a, b},
         {0, -a, -b}, {0, a, -b}, {b, 0, -a},  {b, 0, a},  {-b, 0, -a}, {-b, 0, a}};
  const std::uint32_t f[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                  {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                  {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                  {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  for (auto& tri : f) m.t.insert(m.t.end(), tri, tri + 3);
  return m;
}

// Loop subdivision with midpoints pushed to the unit sphere; midpoint ids are
// assigned on first use of each undirected edge (edge key = lo<<32 | hi).
Mesh icosphere(double radius, int level, P3 c) {
  Mesh m = base_icosahedron();
  for (int l = 0; l < level; ++l) {
    std::map<std::uint64_t, std::uint32_t> mids;
    auto mid = [&](std::uint32_t u, std::uint32_t w) {
      const std::uint64_t key = u < w ? (std::uint64_t(u) << 32 | w) : (std::uint64_t(w) << 32 | u);
      auto it = mids.find(key);
      if (it != mids.end()) return it->second;
      const std::uint32_t id = static_cast<std::uint32_t>(m.v.size());
      const P3 a = m.v[u], b = m.v[w];
      const P3 s{a.x + b.x, a.y + b.y, a.z + b.z};
      m.v.push_back(unit(P3{s.x * 0.5, s.y * 0.5, s.z * 0.5}));
      mids.emplace(key, id);
      return id;
    };
    std::vector<std::uint32_t> next;
    next.reserve(m.t.size() * 4);
    for (std::size_t i = 0; i < m.t.size(); i += 3) {
      const std::uint32_t A = m.t[i], B = m.t[i + 1], C = m.t[i + 2];
      const std::uint32_t ab = mid(A, B), bc = mid(B, C), ca = mid(C, A);
      const std::uint32_t kids[12] = {A, ab, ca, B, bc, ab, C, ca, bc, ab, bc, ca};
      next.insert(next.end(), kids, kids + 12);
    }
    m.t.swap(next);
  }
  for (P3& p : m.v) {
    const P3 u = unit(p);
    p = P3{u.x * radius + c.x, u.y * radius + c.y, u.z * radius + c.z};
  }
  return m;
}

Mesh box(P3 lo, P3 hi) {
  Mesh m;
  m.v = {{lo.x, lo.y, lo.z}, {hi.x, lo.y, lo.z}, {lo.x, hi.y, lo.z}, {hi.x, hi.y, lo.z},
         {lo.x, lo.y, hi.z}, {hi.x, lo.y, hi.z}, {lo.x, hi.y, hi.z}, {hi.x, hi.y, hi.z}};
  m.t = {0, 2, 1, 1, 2, 3, 4, 5, 6, 5, 7, 6, 0, 1, 4, 1, 5, 4,
         2, 6, 3, 3, 6, 7, 0, 4, 2, 2, 4, 6, 1, 3, 5, 3, 7, 5};
  return m;
}

// Radial perturbation of a sphere about c: p = c + R * f(theta, phi) * u.
template <class F>
Mesh radial(const Mesh& unit_sphere, double R, P3 c, F f) {
  Mesh m = unit_sphere;
  for (P3& p : m.v) {
    const double th = std::acos(std::clamp(p.z, -1.0, 1.0));
    const double ph = std::atan2(p.y, p.x);
    const double r = R * f(th, ph);
    p = P3{c.x + r * p.x, c.y + r * p.y, c.z + r * p.z};
  }
  return m;
}

// Ellipsoid: unit sphere scaled by semi-axes, rotated by (yaw, pitch), shifted.
Mesh ellipsoid(const Mesh& unit_sphere, P3 ax, double yaw, double pitch, P3 c, double fold = 0.0, int fold_k = 0) {
  Mesh m = unit_sphere;
  const double cy = std::cos(yaw), sy = std::sin(yaw), cp = std::cos(pitch), sp = std::sin(pitch);
  for (P3& p : m.v) {
    double f = 1.0;
    if (fold != 0.0) {
      const double th = std::acos(std::clamp(p.z, -1.0, 1.0));
      const double ph = std::atan2(p.y, p.x);
      f = 1.0 + fold * std::sin(fold_k * th) * std::sin(fold_k * ph);
    }
    const double x = p.x * ax.x * f, y = p.y * ax.y * f, z = p.z * ax.z * f;
    // rotate about z by yaw, then about x by pitch
    const double x1 = cy * x - sy * y, y1 = sy * x + cy * y, z1 = z;
    const double y2 = cp * y1 - sp * z1, z2 = sp * y1 + cp * z1;
    p = P3{c.x + x1, c.y + y2, c.z + z2};
  }
  return m;
}

struct Compartment {
  std::string name;
  int label;
  int priority;
  bool active;
  Mesh mesh;
};

struct Config {
  std::vector<Compartment> comps;  // innermost (highest priority) first
  double origin[3];
  double h;
  int n[3];
};

void cover(Config& cfg, double h, double margin) {
  P3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
  for (auto& c : cfg.comps)
    for (auto& p : c.mesh.v) {
      lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
      hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
    }
  lo = {lo.x - margin, lo.y - margin, lo.z - margin};
  hi = {hi.x + margin, hi.y + margin, hi.z + margin};
  cfg.origin[0] = lo.x;
  cfg.origin[1] = lo.y;
  cfg.origin[2] = lo.z;
  cfg.h = h;
  const double e[3] = {hi.x - lo.x, hi.y - lo.y, hi.z - lo.z};
  for (int i = 0; i < 3; ++i) cfg.n[i] = std::max(1, static_cast<int>(std::ceil(e[i] / h - 1e-12)));  // lattice.hpp:25-34
}

Config make_config(int id) {
  Config cfg;
  const P3 O{0, 0, 0};
  if (id == 1) {
    // icosphere(10, 3) over a 32^3 lattice at h = 0.75 from (-12,-12,-12).
    cfg.comps.push_back({"sphere", 1, 1, true, icosphere(10.0, 3, O)});
    cfg.origin[0] = cfg.origin[1] = cfg.origin[2] = -12.0;
    cfg.h = 0.75;
    cfg.n[0] = cfg.n[1] = cfg.n[2] = 32;
  } else if (id == 2) {
    // 4 nested perturbed spheres (brain, CSF, skull, scalp), shared radial
    // factor 1 + 0.03 sin(3 theta) cos(2 phi), levels (5,4,4,4); h = 2 mm.
    auto f = [](double th, double ph) { return 1.0 + 0.03 * std::sin(3 * th) * std::cos(2 * ph); };
    const double R[4] = {80, 84, 92, 100};
    const int L[4] = {5, 4, 4, 4};
    const char* names[4] = {"brain", "csf", "skull", "scalp"};
    for (int i = 0; i < 4; ++i)
      cfg.comps.push_back({names[i], i + 1, i + 1, true, radial(icosphere(1.0, L[i], O), R[i], O, f)});
    cover(cfg, 2.0, 4.0);
  } else if (id == 3 || id == 4) {
    // 20-compartment head-like model (seed 2203).
    const Mesh s4 = icosphere(1.0, 4, O), s5 = icosphere(1.0, 5, O), s6 = icosphere(1.0, 6, O);
    const P3 scalp{85, 105, 100};
    std::mt19937_64 rng(2203);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<Compartment> nuclei;
    for (int i = 0; i < 15; ++i) {
      // Left/right pairs mirrored in x plus one midline nucleus; centres
      // inside the white-matter ellipsoid, semi-axes 6-15 mm.
      const int pair = i / 2;
      const bool right = (i % 2) == 1;
      P3 c;
      P3 ax{6 + 9 * U(rng), 6 + 9 * U(rng), 6 + 9 * U(rng)};
      if (i == 14) {
        c = {0.0, -20 + 40 * U(rng), -10 + 20 * U(rng)};
      } else {
        c = {(right ? 1 : -1) * (8 + 14 * U(rng)), -35 + 70 * U(rng) * (pair + 1) / 7.0, -25 + 40 * U(rng)};
      }
      const double yaw = std::numbers::pi * U(rng), pitch = std::numbers::pi * (U(rng) - 0.5);
      nuclei.push_back({"nucleus" + std::to_string(i + 1), i + 1, i + 1, true, ellipsoid(s4, ax, yaw, pitch, c)});
    }
    for (auto& n : nuclei) cfg.comps.push_back(std::move(n));
    cfg.comps.push_back({"white", 16, 16, true, ellipsoid(s6, {0.70 * scalp.x, 0.70 * scalp.y, 0.70 * scalp.z}, 0, 0, O, 0.04, 12)});
    cfg.comps.push_back({"grey", 17, 17, true, ellipsoid(s6, {0.85 * scalp.x, 0.85 * scalp.y, 0.85 * scalp.z}, 0, 0, O, 0.04, 12)});
    cfg.comps.push_back({"csf", 18, 18, true, ellipsoid(s5, {0.88 * scalp.x, 0.88 * scalp.y, 0.88 * scalp.z}, 0, 0, O)});
    cfg.comps.push_back({"skull", 19, 19, true, ellipsoid(s5, {0.93 * scalp.x, 0.93 * scalp.y, 0.93 * scalp.z}, 0, 0, O)});
    cfg.comps.push_back({"scalp", 20, 20, true, ellipsoid(s6, scalp, 0, 0, O)});
    cover(cfg, 1.0, 2.0);
  } else if (id == 5) {
    // 12 x icosphere L6 (983,040 triangles): 6 nested perturbed spheres
    // R = 50..100 and 6 intersecting ellipsoids (seed 10000), 215^3 cells.
    const Mesh s6 = icosphere(1.0, 6, O);
    auto f = [](double th, double ph) { return 1.0 + 0.02 * std::sin(4 * th) * std::cos(3 * ph); };
    std::mt19937_64 rng(10000);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    for (int i = 0; i < 6; ++i) {
      P3 c{-25 + 50 * U(rng), -25 + 50 * U(rng), -25 + 50 * U(rng)};
      P3 ax{8 + 14 * U(rng), 8 + 14 * U(rng), 8 + 14 * U(rng)};
      const double yaw = std::numbers::pi * U(rng), pitch = std::numbers::pi * (U(rng) - 0.5);
      cfg.comps.push_back({"ellipsoid" + std::to_string(i + 1), i + 1, i + 1, true, ellipsoid(s6, ax, yaw, pitch, c)});
    }
    for (int i = 0; i < 6; ++i)
      cfg.comps.push_back({"shell" + std::to_string(i + 1), 7 + i, 7 + i, true, radial(s6, 50.0 + 10.0 * i, O, f)});
    cfg.origin[0] = cfg.origin[1] = cfg.origin[2] = -107.5;
    cfg.h = 1.0;
    cfg.n[0] = cfg.n[1] = cfg.n[2] = 215;
  }
  return cfg;
}

}  // namespace

extern "C" {

struct nm_synth {
  Config cfg;
};

// ---- primitives -------------------------------------------------------------
std::size_t nm_icosphere_vertex_count(int level) { return 10ull * (1ull << (2 * level)) + 2; }
std::size_t nm_icosphere_triangle_count(int level) { return 20ull * (1ull << (2 * level)); }

void nm_icosphere(double radius, int level, const double* center, double* xyz, std::uint32_t* tri) {
  const Mesh m = icosphere(radius, level, P3{center[0], center[1], center[2]});
  std::memcpy(xyz, m.v.data(), m.v.size() * sizeof(P3));
  std::memcpy(tri, m.t.data(), m.t.size() * sizeof(std::uint32_t));
}

void nm_box_surface(const double* lo, const double* hi, double* xyz, std::uint32_t* tri) {
  const Mesh m = box(P3{lo[0], lo[1], lo[2]}, P3{hi[0], hi[1], hi[2]});
  std::memcpy(xyz, m.v.data(), m.v.size() * sizeof(P3));
  std::memcpy(tri, m.t.data(), m.t.size() * sizeof(std::uint32_t));
}

// ---- regular 5-tet lattice (lattice.hpp:40-91) -----------------------------
std::size_t nm_lattice_node_count(int nx, int ny, int nz) {
  return static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1);
}
std::size_t nm_lattice_tet_count(int nx, int ny, int nz) { return static_cast<std::size_t>(nx) * ny * nz * 5; }

void nm_lattice_nodes(const double* origin, double h, int nx, int ny, int nz, double* out) {
  std::size_t c = 0;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        out[c++] = origin[0] + i * h;
        out[c++] = origin[1] + j * h;
        out[c++] = origin[2] + k * h;
      }
}

// Five tets per cell; parity (i+j+k)&1 mirrors the split; orientation is
// normalised against the fp64 node positions (mesh.hpp:44-48, vec3.hpp:79-81).
void nm_lattice_tets(const double* nodes, int nx, int ny, int nz, std::uint32_t* out) {
  auto id = [&](int i, int j, int k) {
    return static_cast<std::uint32_t>((static_cast<std::size_t>(k) * (ny + 1) + j) * (nx + 1) + i);
  };
  auto vol_sign = [&](const std::uint32_t* t) {
    const double* a = nodes + 3 * std::size_t(t[0]);
    const double* b = nodes + 3 * std::size_t(t[1]);
    const double* c = nodes + 3 * std::size_t(t[2]);
    const double* d = nodes + 3 * std::size_t(t[3]);
    const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
    const double x[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2], v[0] * w[1] - v[1] * w[0]};
    return (u[0] * x[0] + u[1] * x[1] + u[2] * x[2]) / 6.0;
  };
  std::size_t c = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const std::uint32_t v000 = id(i, j, k), v100 = id(i + 1, j, k), v010 = id(i, j + 1, k),
                            v110 = id(i + 1, j + 1, k), v001 = id(i, j, k + 1), v101 = id(i + 1, j, k + 1),
                            v011 = id(i, j + 1, k + 1), v111 = id(i + 1, j + 1, k + 1);
        std::uint32_t q[5][4];
        if (((i + j + k) & 1) == 0) {
          const std::uint32_t e[5][4] = {{v000, v110, v101, v011}, {v100, v000, v110, v101},
                                         {v010, v000, v110, v011}, {v001, v000, v101, v011},
                                         {v111, v110, v101, v011}};
          std::memcpy(q, e, sizeof q);
        } else {
          const std::uint32_t e[5][4] = {{v100, v010, v001, v111}, {v000, v100, v010, v001},
                                         {v110, v100, v010, v111}, {v101, v100, v001, v111},
                                         {v011, v010, v001, v111}};
          std::memcpy(q, e, sizeof q);
        }
        for (auto& t : q) {
          if (vol_sign(t) < 0.0) std::swap(t[2], t[3]);
          std::memcpy(out + c, t, sizeof t);
          c += 4;
        }
      }
}

// ---- BASELINE.json configurations ------------------------------------------
nm_synth* nm_synth_config(int id) {
  if (id < 1 || id > 5) return nullptr;
  auto* s = new nm_synth;
  s->cfg = make_config(id);
  return s;
}
void nm_synth_free(nm_synth* s) { delete s; }
int nm_synth_compartments(const nm_synth* s) { return static_cast<int>(s->cfg.comps.size()); }
std::size_t nm_synth_vertex_count(const nm_synth* s) {
  std::size_t n = 0;
  for (auto& c : s->cfg.comps) n += c.mesh.v.size();
  return n;
}
std::size_t nm_synth_triangle_count(const nm_synth* s) {
  std::size_t n = 0;
  for (auto& c : s->cfg.comps) n += c.mesh.t.size() / 3;
  return n;
}
// Concatenated surfaces: global vertex array, triangles indexing it, and the
// CSR triangle offsets per compartment (sequence order = priority order).
void nm_synth_surfaces(const nm_synth* s, double* xyz, std::uint32_t* tri, std::uint32_t* comp_off, int* label_ids,
                       int* priorities, std::uint8_t* active) {
  std::size_t vo = 0, to = 0;
  comp_off[0] = 0;
  for (std::size_t k = 0; k < s->cfg.comps.size(); ++k) {
    const Compartment& c = s->cfg.comps[k];
    std::memcpy(xyz + 3 * vo, c.mesh.v.data(), c.mesh.v.size() * sizeof(P3));
    for (std::size_t i = 0; i < c.mesh.t.size(); ++i) tri[3 * to + i] = static_cast<std::uint32_t>(c.mesh.t[i] + vo);
    vo += c.mesh.v.size();
    to += c.mesh.t.size() / 3;
    comp_off[k + 1] = static_cast<std::uint32_t>(to);
    label_ids[k] = c.label;
    priorities[k] = c.priority;
    active[k] = c.active ? 1 : 0;
  }
}
const char* nm_synth_name(const nm_synth* s, int k) { return s->cfg.comps[k].name.c_str(); }
void nm_synth_lattice(const nm_synth* s, double* origin, double* h, int* n) {
  std::memcpy(origin, s->cfg.origin, sizeof s->cfg.origin);
  *h = s->cfg.h;
  std::memcpy(n, s->cfg.n, sizeof s->cfg.n);
}

}  // extern "C"
