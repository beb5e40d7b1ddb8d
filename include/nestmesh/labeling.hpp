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
//   Labeler                 a persistent context: surfaces (and certified
//                           cells) uploaded once, every operation above reused
//                           over it (SPEC.md:297 relabel after each refinement)
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
  // Certified cells (cull_outside = 2) cost a one-off grid build per
  // Labeler (~35 ms at 1e6 triangles, ~8 ms at 3.6e4, built on the device);
  // one-shot free-function calls with fewer point-triangle pairs than this
  // use 13-DOP culling alone (at 4.2e10 pairs, cfg2: cells 7.8 + 1.4 ms
  // against 16 ms with 13-DOP culling). Labels are identical either way.
  double cell_min_evals = 2e10;
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

inline void validate(const SurfaceSegmentation& seg) {
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

// The segmentation flattened to the C ABI's surface arrays.
struct FlatSurfaces {
  std::vector<double> xyz;
  std::vector<std::uint32_t> tri, off{0};
  std::vector<int> ids;
  explicit FlatSurfaces(const SurfaceSegmentation& seg) {
    for (const CompartmentSurface& c : seg.compartments) {
      const auto base = static_cast<std::uint32_t>(xyz.size() / 3);
      for (const Vec3& p : c.mesh.positions) xyz.insert(xyz.end(), {p.x, p.y, p.z});
      for (const Triangle& t : c.mesh.triangles) tri.insert(tri.end(), {t[0] + base, t[1] + base, t[2] + base});
      off.push_back(static_cast<std::uint32_t>(tri.size() / 3));
      ids.push_back(c.label);
    }
  }
};

// culling relies on closed surfaces; the certified-cell build (one-off per
// Labeler) pays off for persistent labelers and large one-shot calls
inline int cull_mode(const GpuOptions& o, double work_evals) {
  if (!o.validate_closed) return 0;
  if (o.opt.cull_outside == 2 && work_evals >= 0.0 && work_evals < o.cell_min_evals) return 1;
  return o.opt.cull_outside;
}

}  // namespace detail

/// A persistent labeling context: the segmentation is validated, flattened and
/// uploaded ONCE (tile packing, 13-DOP, certified cells), then every SPEC
/// operation reuses it — the relabel pass after every refinement
/// does not rebuild anything. Host arrays are passed as they
/// are (pageable std::vector storage is staged through pinned chunk buffers
/// by the library, pinned storage goes straight to DMA).
/// With GpuOptions::devices of size > 1, initial_label shards over the
/// devices (nm_group, SPEC.md:267 --label-workers); the other operations use
/// the first device.
class Labeler {
 public:
  /// work_evals < 0: persistent use, culling per o.opt.cull_outside; >= 0:
  /// a one-shot call of that many point-triangle pairs (the certified-cell
  /// build only above GpuOptions::cell_min_evals).
  explicit Labeler(const SurfaceSegmentation& seg, const GpuOptions& o = {}, double work_evals = -1.0)
      : K_(seg.compartments.size()) {
    detail::validate(seg);
    if (o.validate_closed) {
      for (const CompartmentSurface& c : seg.compartments) {
        const ClosednessReport r = validate_closed(c.mesh);
        if (!r.ok())
          throw LabelingError("surface '" + c.name + "' is not closed: " + std::to_string(r.open_edges.size()) +
                              " open edges, " + std::to_string(r.orientation_errors.size()) +
                              " orientation errors (SPEC.md:227)");
      }
    }
    nm_options opt = o.opt;
    opt.cull_outside = detail::cull_mode(o, work_evals);
    const detail::FlatSurfaces f(seg);
    if (o.devices.size() > 1) {
      nm_group* g = nullptr;
      detail::check(nm_group_create(&g, static_cast<int>(o.devices.size()), o.devices.data(), &opt));
      group_.reset(g);
      detail::check(nm_group_set_surfaces(g, f.xyz.data(), f.xyz.size() / 3, f.tri.data(), f.tri.size() / 3,
                                          f.off.data(), static_cast<int>(f.ids.size()), f.ids.data()));
      opt.device = o.devices[0];
    }
    nm_ctx* c = nullptr;
    detail::check(nm_create(&c, &opt));
    ctx_.reset(c);
    detail::check(nm_set_surfaces(c, f.xyz.data(), f.xyz.size() / 3, f.tri.data(), f.tri.size() / 3, f.off.data(),
                                  static_cast<int>(f.ids.size()), f.ids.data()));
  }

  nm_ctx* handle() const { return ctx_.get(); }
  std::size_t compartments() const { return K_; }

  /// s of one point for one compartment.
  double enclosure_ratio(const Vec3& p, std::size_t compartment = 0) {
    if (compartment >= K_) throw LabelingError("compartment index out of range");
    std::vector<double> s(K_);
    const double q[3] = {p.x, p.y, p.z};
    detail::check(nm_enclosure(ctx_.get(), q, 1, 0.5, s.data(), nullptr));
    return s[compartment];
  }
  /// s[i * K + k] for a batch of points.
  std::vector<double> enclosure_ratios(const std::vector<Vec3>& pts, nm_stats* stats = nullptr) {
    std::vector<double> s(pts.size() * K_);
    detail::check(nm_enclosure(ctx_.get(), detail::xyz_of(pts), pts.size(), 0.5, s.data(), stats));
    return s;
  }

  /// Per-node ratios and inside masks for every compartment.
  NodeEnclosure node_enclosure(const TetrahedralMesh& mesh, const SolidAngleParams& params) {
    NodeEnclosure e;
    e.compartments = K_;
    e.ratio.resize(mesh.node_count() * K_);
    e.inside_mask.resize(mesh.node_count());
    detail::check(nm_enclosure(ctx_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), params.threshold,
                               e.ratio.data(), nullptr));
    for (std::size_t i = 0; i < mesh.node_count(); ++i) {
      std::uint32_t m = 0;
      for (std::size_t k = 0; k < K_; ++k)
        if (e.ratio[i * K_ + k] >= params.threshold) m |= 1u << k;
      e.inside_mask[i] = m;
    }
    return e;
  }

  /// Node masks (bit k = s_k >= T).
  std::vector<std::uint32_t> node_masks(const TetrahedralMesh& mesh, const SolidAngleParams& params,
                                        nm_stats* stats = nullptr) {
    std::vector<std::uint32_t> m(mesh.node_count());
    detail::check(nm_label_nodes(ctx_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), params.threshold, m.data(),
                                 stats));
    return m;
  }

  /// initial_label. masks_out (nullable) receives the node masks.
  std::vector<int> initial_label(const TetrahedralMesh& mesh, const SolidAngleParams& params, nm_stats* stats = nullptr,
                                 std::vector<std::uint32_t>* masks_out = nullptr) {
    std::vector<int> labels;
    initial_label_into(mesh, params, labels, stats, masks_out);
    return labels;
  }

  /// initial_label into a caller vector (e.g. mesh.labels), reused without a
  /// new allocation when its capacity suffices: repeated labeling of large
  /// meshes does not pay the first-touch and zero-fill of a fresh 4 B/tet
  /// array per call.
  void initial_label_into(const TetrahedralMesh& mesh, const SolidAngleParams& params, std::vector<int>& labels,
                          nm_stats* stats = nullptr, std::vector<std::uint32_t>* masks_out = nullptr) {
    labels.resize(mesh.tet_count());
    std::uint32_t* m = nullptr;
    if (masks_out) {
      masks_out->resize(mesh.node_count());
      m = masks_out->data();
    }
    if (group_)
      detail::check(nm_group_label_mesh(group_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(),
                                        detail::idx_of(mesh.tetrahedra), mesh.tet_count(), params.threshold,
                                        labels.data(), m, stats));
    else
      detail::check(nm_label_mesh(ctx_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(),
                                  detail::idx_of(mesh.tetrahedra), mesh.tet_count(), params.threshold, labels.data(),
                                  m, stats));
  }

  /// Tet-centroid labeling: each tet's query point is its centroid
  /// (a+b+c+d)/4 in fp64; label = highest-priority compartment with
  /// s(centroid) >= T, else 0. The alternative query point of the north star
  /// ("tet centroids or vertices"); with it a single sphere at h = R/10 labels
  /// the volume within SPEC.md:240's [0.9, 1.0] band.
  std::vector<int> centroid_label(const TetrahedralMesh& mesh, const SolidAngleParams& params,
                                  nm_stats* stats = nullptr) {
    std::vector<int> labels(mesh.tet_count());
    detail::check(nm_label_centroids(ctx_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(),
                                     detail::idx_of(mesh.tetrahedra), mesh.tet_count(), params.threshold,
                                     labels.data(), stats));
    return labels;
  }

  /// relabel_recursive. Throws NonConvergence (carrying the
  /// best labels) when max_iters passes do not reach a fixed point.
  RelabelResult relabel_recursive(const TetrahedralMesh& mesh, const SolidAngleParams& params,
                                  const std::vector<int>& prev_labels, nm_stats* stats = nullptr) {
    if (prev_labels.size() != mesh.tet_count()) throw LabelingError("prev_labels length != tet count");
    RelabelResult r;
    r.labels = prev_labels;
    int conv = 0;
    detail::check(nm_relabel(ctx_.get(), detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra),
                             mesh.tet_count(), params.threshold, params.max_iters, r.labels.data(), &r.passes, &conv,
                             nullptr, stats));
    r.converged = conv != 0;
    if (!r.converged) {
      r.diagnostic = "labels still changing after " + std::to_string(r.passes) + " passes";
      throw NonConvergence(std::move(r));
    }
    return r;
  }

  /// Tets straddling an active compartment boundary (node masks disagree).
  std::vector<std::uint32_t> boundary_tets(const TetrahedralMesh& mesh, const std::vector<std::uint32_t>& masks,
                                           std::uint32_t active_mask = 0xffffffffu) {
    std::vector<std::uint32_t> ids(mesh.tet_count());
    std::size_t n = 0;
    detail::check(nm_flag_boundary(ctx_.get(), detail::idx_of(mesh.tetrahedra), mesh.tet_count(), masks.data(),
                                   masks.size(), active_mask, ids.data(), &n));
    ids.resize(n);
    return ids;
  }

 private:
  struct CtxDel {
    void operator()(nm_ctx* c) const { nm_destroy(c); }
  };
  struct GroupDel {
    void operator()(nm_group* g) const { nm_group_destroy(g); }
  };
  std::unique_ptr<nm_ctx, CtxDel> ctx_;
  std::unique_ptr<nm_group, GroupDel> group_;
  std::size_t K_ = 0;
};

/// s = (1/4pi) * sum of signed triangle solid angles.
inline double enclosure_ratio(const Vec3& point, const TriangleSurface& surface, const GpuOptions& o = {}) {
  SurfaceSegmentation seg;
  seg.compartments.push_back(CompartmentSurface{"surface", 1, surface, 1.0, 1, true});
  return Labeler(seg, o, 0.0).enclosure_ratio(point);
}

/// Per-node ratios and inside masks for every compartment.
inline NodeEnclosure node_enclosure(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                    const SolidAngleParams& params, const GpuOptions& o = {}) {
  return Labeler(seg, o, double(mesh.node_count()) * detail::triangles(seg)).node_enclosure(mesh, params);
}

/// initial_label: node inside k iff s_k >= T; tet label =
/// highest-priority k with all four nodes inside, else 0.
inline std::vector<int> initial_label(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                      const SolidAngleParams& params, const GpuOptions& o = {},
                                      nm_stats* stats = nullptr) {
  return Labeler(seg, o, double(mesh.node_count()) * detail::triangles(seg)).initial_label(mesh, params, stats);
}

/// relabel_recursive. One-shot: the passes evaluate only
/// the frontier (a thin shell of nodes), so no certified cells are built;
/// callers relabeling repeatedly keep a Labeler.
inline RelabelResult relabel_recursive(const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                       const SolidAngleParams& params, const std::vector<int>& prev_labels,
                                       const GpuOptions& o = {}) {
  return Labeler(seg, o, 0.0).relabel_recursive(mesh, params, prev_labels);
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
  nm_options opt = o.opt;
  opt.cull_outside = 0;
  nm_ctx* c = nullptr;
  detail::check(nm_create(&c, &opt));
  std::unique_ptr<nm_ctx, int (*)(nm_ctx*)> ctx(c, nm_destroy);
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
  GpuOptions g = o;
  g.opt.cull_outside = 0;  // no node pass: nothing to cull
  return Labeler(seg, g, 0.0).boundary_tets(mesh, masks, active_mask);
}

}  // namespace nestmesh
