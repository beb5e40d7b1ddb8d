// The C++ drop-in (include/nestmesh/labeling.hpp) used exactly as a nestmesh
// maintainer would: the UNMODIFIED reference headers for the types and the
// lattice/icosphere generators, the SPEC operations from labeling.hpp.
// Built by __graft_entry__.build() where /root/reference exists (the binary
// travels to the GPU box); run by tests/test_gpu_dropin.py, which compares
// the labels it prints against the oracle.
#include <cstdio>
#include <cstdlib>

#include "nestmesh/label_sidecar.hpp"
#include "nestmesh/labeling.hpp"
#include "nestmesh/lattice.hpp"
#include "nestmesh/primitives.hpp"

using namespace nestmesh;

int main(int argc, char** argv) {
  const char* out_path = argc > 1 ? argv[1] : "labels.bin";
  SurfaceSegmentation seg;
  seg.compartments.push_back(CompartmentSurface{"inner", 3, icosphere(6.0, 3), 0.33, 1, true});
  seg.compartments.push_back(CompartmentSurface{"outer", 9, icosphere(10.0, 3), 0.0042, 2, true});
  LatticeSpec spec;
  spec.origin = Vec3{-12, -12, -12};
  spec.cell_size = 0.75;
  spec.nx = spec.ny = spec.nz = 32;
  const TetrahedralMesh mesh = generate_lattice_mesh(spec);
  SolidAngleParams params;
  nm_stats st{};
  const std::vector<int> labels = initial_label(mesh, seg, params, GpuOptions{}, &st);
  // multi-device sharding (two contexts on device 0) is bit-identical
  GpuOptions multi;
  multi.devices = {0, 0};
  if (initial_label(mesh, seg, params, multi) != labels) {
    std::fprintf(stderr, "group labels differ\n");
    return 6;
  }
  // certified cells forced on (cell_min_evals = 0), and every culling mode
  // off / 13-DOP only: the same labels
  for (int mode : {0, 1, 2}) {
    GpuOptions o;
    o.opt.cull_outside = mode;
    o.cell_min_evals = 0.0;
    if (initial_label(mesh, seg, params, o) != labels) {
      std::fprintf(stderr, "labels differ with cull_outside=%d\n", mode);
      return 9;
    }
  }
  {
    GpuOptions o;
    o.cell_min_evals = 0.0;
    const RelabelResult rc = relabel_recursive(mesh, seg, params, labels, o);
    if (rc.passes != 1 || rc.labels != labels) {
      std::fprintf(stderr, "relabel with certified cells failed\n");
      return 10;
    }
  }
  // enclosure_ratio KATs
  const double s_in = enclosure_ratio(Vec3{0, 0, 0}, seg.compartments[0].mesh);
  const double s_out = enclosure_ratio(Vec3{30, 0, 0}, seg.compartments[0].mesh);
  if (std::abs(s_in - 1.0) > 1e-6 || std::abs(s_out) > 1e-6) {
    std::fprintf(stderr, "enclosure KAT failed: %.17g %.17g\n", s_in, s_out);
    return 2;
  }
  // relabel of converged labels: one pass, no change
  const RelabelResult r = relabel_recursive(mesh, seg, params, labels);
  if (r.passes != 1 || r.labels != labels) {
    std::fprintf(stderr, "relabel fixed point failed: passes=%d\n", r.passes);
    return 3;
  }
  // invalid segmentation -> LabelingError (SPEC.md:103 priorities increasing)
  SurfaceSegmentation bad = seg;
  bad.compartments[1].priority = 0;
  try {
    (void)initial_label(mesh, bad, params);
    return 4;
  } catch (const LabelingError&) {
  }
  // open surface -> LabelingError (validate_closed)
  SurfaceSegmentation open_seg = seg;
  open_seg.compartments[0].mesh.triangles.pop_back();
  try {
    (void)initial_label(mesh, open_seg, params);
    return 5;
  } catch (const LabelingError&) {
  }
  // refine_boundary around the inner|outer interface, then relabel: the
  // recursion premise — relabel == initial labeling of the refined mesh
  TetrahedralMesh lab_mesh = mesh;
  lab_mesh.labels = labels;
  const TetrahedralMesh refined = refine_boundary(lab_mesh, 3, 9);
  if (refined.tet_count() <= mesh.tet_count() || !validate_mesh(refined).ok()) {
    std::fprintf(stderr, "refine_boundary failed\n");
    return 7;
  }
  const RelabelResult rr = relabel_recursive(refined, seg, params, refined.labels);
  if (rr.labels != initial_label(refined, seg, params)) {
    std::fprintf(stderr, "relabel != initial on the refined mesh\n");
    return 8;
  }
  // persistent Labeler: surfaces (+ certified cells) uploaded once; initial
  // labels, relabel after refinement and enclosure ratios over the same
  // context equal the free functions
  {
    Labeler lab(seg);
    std::vector<std::uint32_t> masks;
    if (lab.initial_label(mesh, params, nullptr, &masks) != labels || masks.size() != mesh.node_count()) {
      std::fprintf(stderr, "Labeler initial_label differs\n");
      return 11;
    }
    if (lab.node_masks(mesh, params) != masks) {
      std::fprintf(stderr, "Labeler node_masks differ\n");
      return 12;
    }
    const RelabelResult lr = lab.relabel_recursive(refined, params, refined.labels);
    if (lr.labels != rr.labels || lab.initial_label(refined, params) != rr.labels) {
      std::fprintf(stderr, "Labeler relabel differs\n");
      return 13;
    }
    const std::vector<double> s = lab.enclosure_ratios({Vec3{0, 0, 0}, Vec3{30, 0, 0}});
    if (std::abs(s[0] - 1.0) > 1e-6 || std::abs(s[1] - 1.0) > 1e-6 || std::abs(s[2]) > 1e-6 || std::abs(s[3]) > 1e-6) {
      std::fprintf(stderr, "Labeler enclosure_ratios KAT failed\n");
      return 14;
    }
    // centroid mode: the volume labeled inside the inner sphere (R = 6,
    // h = 0.75 = R/8) is within SPEC.md:240's [0.9, 1.0] of the sphere volume
    {
      const std::vector<int> cl = lab.centroid_label(mesh, params);
      double vol = 0.0;
      for (std::size_t t = 0; t < mesh.tet_count(); ++t)
        if (cl[t] == 3) vol += std::abs(tet_signed_volume(mesh.nodes[mesh.tetrahedra[t][0]], mesh.nodes[mesh.tetrahedra[t][1]],
                                                          mesh.nodes[mesh.tetrahedra[t][2]], mesh.nodes[mesh.tetrahedra[t][3]]));
      const double ratio = vol / (4.0 / 3.0 * 3.14159265358979323846 * 216.0);
      if (ratio < 0.9 || ratio > 1.0) {
        std::fprintf(stderr, "centroid-mode volume ratio %.4f outside [0.9, 1.0]\n", ratio);
        return 22;
      }
    }
    if (lab.boundary_tets(mesh, masks) != boundary_tets(mesh, masks, 0xffffffffu, seg)) {
      std::fprintf(stderr, "Labeler boundary_tets differ\n");
      return 15;
    }
    // NonConvergence: one pass cannot fix labels from a
    // coarse segmentation; the best labels travel with the exception
    SurfaceSegmentation coarse = seg;
    coarse.compartments[0].mesh = icosphere(6.0, 1);
    coarse.compartments[1].mesh = icosphere(10.0, 1);
    const std::vector<int> prev = initial_label(mesh, coarse, params);
    SolidAngleParams one = params;
    one.max_iters = 1;
    try {
      (void)lab.relabel_recursive(mesh, one, prev);
      std::fprintf(stderr, "NonConvergence not thrown\n");
      return 16;
    } catch (const NonConvergence& e) {
      if (e.best.passes != 1 || e.best.converged || e.best.labels.size() != prev.size()) return 17;
    }
    if (lab.relabel_recursive(mesh, params, prev).labels != labels) {
      std::fprintf(stderr, "relabel from coarse labels != initial\n");
      return 18;
    }
  }
  // label sidecar next to a tetmesh v1 file written by the reference's own
  // save_tetmesh (mesh.hpp:238-289): the lattice is labeled on the device
  // straight into the sidecar; the mesh read back by load_tetmesh matches it
  {
    Labeler lab(seg);
    const std::string mesh_path = std::string(out_path) + ".tetmesh";
    save_tetmesh(mesh_path, mesh);
    const nm_sidecar_info info = label_lattice_to_sidecar(lab, spec, params, label_sidecar_path(mesh_path));
    TetrahedralMesh back = load_tetmesh(mesh_path);
    const LabelSidecar sc = read_label_sidecar(label_sidecar_path(mesh_path));
    apply_label_sidecar(back, sc);
    if (back.labels != labels || sc.info.mesh_fingerprint != info.mesh_fingerprint ||
        generate_lattice_mesh(sidecar_lattice(sc)).nodes.size() != mesh.node_count()) {
      std::fprintf(stderr, "label sidecar round trip failed\n");
      return 19;
    }
    // an explicit (refined) mesh: sidecar tied by its fingerprint
    TetrahedralMesh r2 = refined;
    r2.labels = rr.labels;
    write_label_sidecar(mesh_path + ".refined.nmlabels", r2, seg, params);
    TetrahedralMesh other = mesh;
    try {
      apply_label_sidecar(other, read_label_sidecar(mesh_path + ".refined.nmlabels"));
      return 20;
    } catch (const LabelingError&) {
    }
    TetrahedralMesh r3 = refined;
    apply_label_sidecar(r3, read_label_sidecar(mesh_path + ".refined.nmlabels"));
    if (r3.labels != rr.labels) return 21;
  }
  FILE* f = std::fopen(out_path, "wb");
  std::fwrite(labels.data(), sizeof(int), labels.size(), f);
  std::fclose(f);
  std::printf("dropin ok: %zu tets, evals %llu\n", labels.size(), static_cast<unsigned long long>(st.evals));
  return 0;
}
