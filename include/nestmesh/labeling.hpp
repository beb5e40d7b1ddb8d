// nestmesh/labeling.hpp — the labeling module of SPEC.md:210-272 for the
// reference library nestmesh (/root/reference/proj/include/nestmesh), as a
// header-only drop-in in the reference's own style: free inline functions in
// namespace nestmesh over TetrahedralMesh / TriangleSurface, errors as
// exceptions derived from std::runtime_error.
//
// The arithmetic runs on a B200 through libnestmesh_label.so (C ABI,
// include/nestmesh_label.h); link with -lnestmesh_label. There is no CPU
// fallback: without a usable sm_100 device every call throws LabelingError.
//
// SPEC mapping
//   SolidAngleParams        SPEC.md:215-218   (T in (0,1), default 0.5)
//   NodeEnclosure
//   CompartmentSurface
//   SurfaceSegmentation     SPEC.md:100-103   (innermost -> outermost)
//   enclosure_ratio
//   initial_label
//   relabel_recursive       SPEC.md:243-251   (NonConvergence after max_iters)
//   boundary_tets           SPEC.md:294-302   (straddle layer of refine_boundary)
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "nestmesh/mesh.hpp"
#include "nestmesh/surface.hpp"
#include "nestmesh/vec3.hpp"
#include "nestmesh_label.h"

namespace nestmesh {

struct LabelingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct SolidAngleParams {
  double threshold = 0.5;  // T; a node is inside when s >= T
  int max_iters = 64;      // relabel_recursive pass cap
};

struct NodeEnclosure {
  std::vector<double> ratio;               // s[node * K + k]
  std::vector<std::uint32_t> inside_mask;  // bit k = (s_k >= T)
  std::size_t compartments = 0;
};

struct CompartmentSurface {
  std::string name;
  int label = 1;  // > 0; 0 is the bounding box
  TriangleSurface mesh;
  double conductivity = 1.0;
  int priority = 1;  // 1 = innermost
  bool active = true;
};

struct SurfaceSegmentation {
  std::vector<CompartmentSurface> compartments;  // innermost -> outermost
  double box_margin_mm = 0.0;
};

struct RelabelResult {
  std::vector<int> labels;
  int passes = 0;
  bool converged = false;
  std::string diagnostic;
};

struct NonConvergence : std::runtime_error {
  RelabelResult best;
  explicit NonConvergence(RelabelResult r)
      : std::runtime_error("relabel_recursive: no fixed point after " + std::to_string(r.passes) + " passes"),
        best(std::move(r)) {}
};

/// Device and numerics options of the B200 path (defaults: nm_default_options).
struct GpuOptions {
  nm_options opt;
  bool validate_closed = true;  // check the SPEC.md:227 precondition with validate_closed (surface.hpp:80-104)
  std::vector<int> devices;     // > 1 entries: initial_label shards over these devices (SPEC.md:267 --label-workers)
  // Certified cells (cull_outside = 2) cost a one-off grid build per call
  // (~0.3-0.5 s at 1e6 triangles); calls with fewer point-triangle pairs
  // than this use 13-DOP culling alone. Labels are identical either way.
  double cell_min_evals = 2e12;
  GpuOptions() {
    nm_default_options(&opt);
    opt.cull_outside = 2;  // exact for closed surfaces (13-DOP + certified cells); disabled below whenever
                           // closedness is not validated
  }
};

inline int labeling_abi_version() { return nm_abi_version(); }

namespace detail {

inline void check(int rc) {
  if (rc != 0) throw LabelingError(nm_last_error());
}

/// RAII owner of one nm_ctx (one device + stream + replicated surfaces).
class Context {
 public:
  explicit Context(const GpuOptions& o = {}, double work_evals = 0.0) : validate_(o.validate_closed) {
    nm_options opt = o.opt;
    opt.cull_outside = cull_mode(o, work_evals);
    check(nm_create(&ctx_, &opt));
  }
  // culling relies on closed surfaces; certified cells only pay off on large calls
  static int cull_mode(const GpuOptions& o, double work_evals) {
    if (!o.validate_closed) return 0;
    if (o.opt.cull_outside == 2 && work_evals < o.cell_min_evals) return 1;
    return o.opt.cull_outside;
  }
  ~Context() {
    if (ctx_) nm_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  nm_ctx* get() const { return ctx_; }

  void set_segmentation(const SurfaceSegmentation& seg) {
    validate(seg);
    if (validate_) {
      for (const CompartmentSurface& c : seg.compartments) {
        const ClosednessReport r = validate_closed(c.mesh);
        if (!r.ok())
          throw LabelingError("surface '" + c.name + "' is not closed: " + std::to_string(r.open_edges.size()) +
                              " open edges, " + std::to_string(r.orientation_errors.size()) +
                              " orientation errors (SPEC.md:227)");
      }
    }
    std::vector<double> xyz;
    std::vector<std::uint32_t> tri, off{0};
    std::vector<int> ids;
    for (const CompartmentSurface& c : seg.compartments) {
      const auto base = static_cast<std::uint32_t>(xyz.size() / 3);
      for (const Vec3& p : c.mesh.positions) xyz.insert(xyz.end(), {p.x, p.y, p.z});
      for (const Triangle& t : c.mesh.triangles) tri.insert(tri.end(), {t[0] + base, t[1] + base, t[2] + base});
      off.push_back(static_cast<std::uint32_t>(tri.size() / 3));
      ids.push_back(c.label);
    }
    check(nm_set_surfaces(ctx_, xyz.data(), xyz.size() / 3, tri.data(), tri.size() / 3, off.data(),
                          static_cast<int>(ids.size()), ids.data()));
  }

  static void validate(const SurfaceSegmentation& seg) {
    if (seg.compartments.empty()) throw LabelingError("segmentation has no compartment (SPEC.md:103)");
    if (seg.compartments.size() > 32) throw LabelingError("at most 32 compartments are supported");
    for (std::size_t k = 0; k < seg.compartments.size(); ++k) {
      const auto& c = seg.compartments[k];
      if (c.label <= 0) throw LabelingError("compartment label ids must be > 0");
      if (k && c.priority <= seg.compartments[k - 1].priority)
        throw LabelingError("priorities must increase innermost -> outermost (SPEC.md:103)");
      for (std::size_t j = 0; j < k; ++j)
        if (seg.compartments[j].label == c.label) throw LabelingError("label ids must be unique (SPEC.md:99)");
    }
  }

 private:
  nm_ctx* ctx_ = nullptr;
  bool validate_ = true;
};

inline double triangles(const SurfaceSegmentation& seg) {
  double t = 0.0;
  for (const CompartmentSurface& c : seg.compartments) t += static_cast<double>(c.mesh.triangles.size());
  return t;
}

inline const double* xyz_of(const std::vector<Vec3>& v) {
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
  return reinterpret_cast<const double*>(v.data());
}
inline const std::uint32_t* idx_of(const std::vector<Tet>& t) {
  static_assert(sizeof(Tet) == 4 * sizeof(std::uint32_t), "Tet must be four packed uint32");
  return reinterpret_cast<const std::uint32_t*>(t.data());
}

}  // namespace detail

/// s = (1/4pi) * sum of signed triangle solid angles.
inline double enclosure_ratio(const Vec3& point, const TriangleSurface& surface, const GpuOptions& o = {}) {
  detail::Context ctx(o);
  SurfaceSegmentation seg;
  seg.compartments.push_back(CompartmentSurface{"surface", 1, surface, 1.0, 1, true});
  ctx.set_segmentation(seg);
  double s = 0.0;
  const double p[3] = {point.x, point.y, point.z};
  detail::check(nm_enclosure(ctx.get(), p, 1, 0.5, &s, nullptr));
  return s;
}

/// Per-node ratios and inside masks for every compartment.
inline NodeEnclosure node_enclosure(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                    const SolidAngleParams& params, const GpuOptions& o = {}) {
  detail::Context ctx(o, double(mesh.node_count()) * detail::triangles(seg));
  ctx.set_segmentation(seg);
  NodeEnclosure e;
  e.compartments = seg.compartments.size();
  e.ratio.resize(mesh.node_count() * e.compartments);
  e.inside_mask.resize(mesh.node_count());
  detail::check(nm_enclosure(ctx.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), params.threshold,
                             e.ratio.data(), nullptr));
  for (std::size_t i = 0; i < mesh.node_count(); ++i) {
    std::uint32_t m = 0;
    for (std::size_t k = 0; k < e.compartments; ++k)
      if (e.ratio[i * e.compartments + k] >= params.threshold) m |= 1u << k;
    e.inside_mask[i] = m;
  }
  return e;
}

/// initial_label: node inside k iff s_k >= T; tet label =
/// highest-priority k with all four nodes inside, else 0.
inline std::vector<int> initial_label(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                      const SolidAngleParams& params, const GpuOptions& o = {},
                                      nm_stats* stats = nullptr) {
  if (o.devices.size() > 1) {
    // validate + flatten through a single-device context, then shard over the group
    detail::Context::validate(seg);
    nm_group* g = nullptr;
    nm_options gopt = o.opt;
    gopt.cull_outside = detail::Context::cull_mode(o, double(mesh.node_count()) * detail::triangles(seg));
    detail::check(nm_group_create(&g, static_cast<int>(o.devices.size()), o.devices.data(), &gopt));
    std::unique_ptr<nm_group, int (*)(nm_group*)> guard(g, nm_group_destroy);
    std::vector<double> xyz;
    std::vector<std::uint32_t> tri, off{0};
    std::vector<int> ids;
    for (const CompartmentSurface& c : seg.compartments) {
      if (o.validate_closed && !validate_closed(c.mesh).ok())
        throw LabelingError("surface '" + c.name + "' is not closed (SPEC.md:227)");
      const auto base = static_cast<std::uint32_t>(xyz.size() / 3);
      for (const Vec3& p : c.mesh.positions) xyz.insert(xyz.end(), {p.x, p.y, p.z});
      for (const Triangle& t : c.mesh.triangles) tri.insert(tri.end(), {t[0] + base, t[1] + base, t[2] + base});
      off.push_back(static_cast<std::uint32_t>(tri.size() / 3));
      ids.push_back(c.label);
    }
    detail::check(nm_group_set_surfaces(g, xyz.data(), xyz.size() / 3, tri.data(), tri.size() / 3, off.data(),
                                        static_cast<int>(ids.size()), ids.data()));
    std::vector<int> labels(mesh.tet_count());
    detail::check(nm_group_label_mesh(g, detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra),
                                      mesh.tet_count(), params.threshold, labels.data(), nullptr, stats));
    return labels;
  }
  detail::Context ctx(o, double(mesh.node_count()) * detail::triangles(seg));
  ctx.set_segmentation(seg);
  std::vector<int> labels(mesh.tet_count());
  detail::check(nm_label_mesh(ctx.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra),
                              mesh.tet_count(), params.threshold, labels.data(), nullptr, stats));
  return labels;
}

/// relabel_recursive. Throws NonConvergence (carrying the
/// best labels) when max_iters passes do not reach a fixed point.
inline RelabelResult relabel_recursive(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                       const SolidAngleParams& params, const std::vector<int>& prev_labels,
                                       const GpuOptions& o = {}) {
  if (prev_labels.size() != mesh.tet_count()) throw LabelingError("prev_labels length != tet count");
  detail::Context ctx(o, double(mesh.node_count()) * detail::triangles(seg));
  ctx.set_segmentation(seg);
  RelabelResult r;
  r.labels = prev_labels;
  int conv = 0;
  detail::check(nm_relabel(ctx.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra),
                           mesh.tet_count(), params.threshold, params.max_iters, r.labels.data(), &r.passes, &conv,
                           nullptr, nullptr));
  r.converged = conv != 0;
  if (!r.converged) {
    r.diagnostic = "labels still changing after " + std::to_string(r.passes) + " passes";
    throw NonConvergence(std::move(r));
  }
  return r;
}

namespace detail {
inline TetrahedralMesh to_mesh(nm_mesh* m) {
  std::unique_ptr<nm_mesh, void (*)(nm_mesh*)> guard(m, nm_mesh_free);
  std::size_t nn = 0, nt = 0, nold = 0;
  check(nm_mesh_sizes(m, &nn, &nt, &nold));
  TetrahedralMesh out;
  out.nodes.resize(nn);
  out.tetrahedra.resize(nt);
  out.labels.resize(nt);
  check(nm_mesh_copy(m, reinterpret_cast<double*>(out.nodes.data()), reinterpret_cast<std::uint32_t*>(out.tetrahedra.data()),
                     out.labels.data(), nullptr));
  return out;
}
}  // namespace detail

/// refine_volume: 1:8 split of the selected tets plus
/// conforming transition templates; children inherit labels. Host code.
inline TetrahedralMesh refine_volume(const TetrahedralMesh& mesh, const std::vector<std::uint32_t>& element_set) {
  nm_mesh* m = nullptr;
  if (nm_refine(detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra), mesh.tet_count(),
                mesh.labels.size() == mesh.tet_count() ? mesh.labels.data() : nullptr, element_set.data(),
                element_set.size(), &m) != 0)
    throw LabelingError(nm_refine_last_error());
  return detail::to_mesh(m);
}

/// refine_boundary on the device: refine the layers on both
/// sides of the label_a | label_b interface (mesh.labels).
inline TetrahedralMesh refine_boundary(const TetrahedralMesh& mesh, int label_a, int label_b, const GpuOptions& o = {}) {
  if (mesh.labels.size() != mesh.tet_count()) throw LabelingError("labels length != tet count");
  detail::Context ctx(o);
  nm_mesh* m = nullptr;
  detail::check(nm_refine_boundary(ctx.get(), detail::xyz_of(mesh.nodes), mesh.node_count(),
                                   detail::idx_of(mesh.tetrahedra), mesh.tet_count(), mesh.labels.data(), label_a,
                                   label_b, &m));
  return detail::to_mesh(m);
}

/// Tets straddling an active compartment boundary (node masks disagree).
inline std::vector<std::uint32_t> boundary_tets(const TetrahedralMesh& mesh, const std::vector<std::uint32_t>& masks,
                                                std::uint32_t active_mask, const SurfaceSegmentation& seg,
                                                const GpuOptions& o = {}) {
  detail::Context ctx(o);
  ctx.set_segmentation(seg);
  std::vector<std::uint32_t> ids(mesh.tet_count());
  std::size_t n = 0;
  detail::check(nm_flag_boundary(ctx.get(), detail::idx_of(mesh.tetrahedra), mesh.tet_count(), masks.data(),
                                 masks.size(), active_mask, ids.data(), &n));
  ids.resize(n);
  return ids;
}

}  // namespace nestmesh
