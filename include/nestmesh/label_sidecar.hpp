// nestmesh/label_sidecar.hpp — a labeling result kept next to a tetmesh v1
// file as a binary sidecar (<mesh>.tetmesh.nmlabels), bit for bit: int32
// labels per tet, optional uint32 node masks, and what ties them to the mesh —
// its fingerprint, or the LatticeSpec of a generate_lattice_mesh mesh
// (lattice.hpp:40-91), which regenerates it exactly. The mesh itself stays in
// the reference's %.17g text format (save_tetmesh / load_tetmesh,
// mesh.hpp:238-289); the sidecar replaces re-writing it just to store labels.
// C ABI: nm_sidecar_* / nm_mesh_fingerprint / nm_label_lattice_sidecar
// (include/nestmesh_label.h; csrc/sidecar.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "nestmesh/labeling.hpp"
#include "nestmesh/lattice.hpp"

namespace nestmesh {

struct LabelSidecar {
  nm_sidecar_info info{};
  std::vector<int> labels;
  std::vector<std::uint32_t> masks;  // empty when the sidecar has none
};

inline std::string label_sidecar_path(const std::string& tetmesh_path) { return tetmesh_path + ".nmlabels"; }

/// Order-independent 64-bit fingerprint of the mesh's node bits and tets.
inline std::uint64_t mesh_fingerprint(const TetrahedralMesh& mesh) {
  std::uint64_t fp = 0;
  detail::check(nm_mesh_fingerprint(detail::xyz_of(mesh.nodes), mesh.node_count(), detail::idx_of(mesh.tetrahedra),
                                    mesh.tet_count(), &fp));
  return fp;
}

/// Write mesh.labels (and optional node masks) beside the mesh.
inline void write_label_sidecar(const std::string& path, const TetrahedralMesh& mesh, const SurfaceSegmentation& seg,
                                const SolidAngleParams& params, const std::vector<std::uint32_t>* masks = nullptr) {
  if (mesh.labels.size() != mesh.tet_count()) throw LabelingError("labels length != tet count");
  if (masks && masks->size() != mesh.node_count()) throw LabelingError("masks length != node count");
  nm_sidecar_info info{};
  info.n_nodes = mesh.node_count();
  info.n_tets = mesh.tet_count();
  info.mesh_fingerprint = mesh_fingerprint(mesh);
  info.K = static_cast<int>(seg.compartments.size());
  for (std::size_t k = 0; k < seg.compartments.size() && k < 32; ++k) info.label_ids[k] = seg.compartments[k].label;
  info.has_masks = masks ? 1 : 0;
  info.threshold = params.threshold;
  detail::check(nm_sidecar_write(path.c_str(), &info, mesh.labels.data(), masks ? masks->data() : nullptr));
}

inline LabelSidecar read_label_sidecar(const std::string& path) {
  LabelSidecar sc;
  detail::check(nm_sidecar_read_info(path.c_str(), &sc.info));
  sc.labels.resize(sc.info.n_tets);
  if (sc.info.has_masks) sc.masks.resize(sc.info.n_nodes);
  detail::check(nm_sidecar_read(path.c_str(), &sc.info, sc.labels.data(), sc.info.has_masks ? sc.masks.data() : nullptr));
  return sc;
}

/// Attach a sidecar's labels to the mesh it belongs to: sizes and the mesh
/// fingerprint must match (a LatticeSpec sidecar: the regenerated lattice's).
inline void apply_label_sidecar(TetrahedralMesh& mesh, const LabelSidecar& sc) {
  if (sc.info.n_tets != mesh.tet_count() || sc.info.n_nodes != mesh.node_count())
    throw LabelingError("label sidecar does not match the mesh sizes");
  if (sc.info.mesh_fingerprint != mesh_fingerprint(mesh))
    throw LabelingError("label sidecar belongs to a different mesh (fingerprint mismatch)");
  mesh.labels = sc.labels;
}

/// The LatticeSpec a lattice sidecar was written for.
inline LatticeSpec sidecar_lattice(const LabelSidecar& sc) {
  if (!sc.info.is_lattice) throw LabelingError("label sidecar does not describe a lattice");
  LatticeSpec s;
  s.origin = Vec3{sc.info.origin[0], sc.info.origin[1], sc.info.origin[2]};
  s.cell_size = sc.info.h;
  s.nx = sc.info.n[0];
  s.ny = sc.info.n[1];
  s.nz = sc.info.n[2];
  return s;
}

/// initial_label of a regular lattice straight to a sidecar: the lattice is
/// generated, labeled and fingerprinted on the device; only the labels (and
/// masks) cross to the host, into the file.
inline nm_sidecar_info label_lattice_to_sidecar(Labeler& labeler, const LatticeSpec& spec, const SolidAngleParams& params,
                                                const std::string& path, bool with_masks = true, nm_stats* stats = nullptr) {
  spec.validate();
  const double o[3] = {spec.origin.x, spec.origin.y, spec.origin.z};
  nm_sidecar_info info{};
  detail::check(nm_label_lattice_sidecar(labeler.handle(), o, spec.cell_size, spec.nx, spec.ny, spec.nz,
                                         params.threshold, path.c_str(), with_masks ? 1 : 0, &info, stats));
  return info;
}

}  // namespace nestmesh
