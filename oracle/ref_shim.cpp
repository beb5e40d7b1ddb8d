// TEST INFRASTRUCTURE ONLY — C shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/nestmesh/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libnestmesh_ref.so. The headers are included where they
// lie; nothing is copied. Used by tests to pin the product-side generators
// (paper_2203_10000_b200/csrc/synth.cpp) and the relabel frontier against the
// reference's own code. The reference has no labeling code (SPEC.md:210-272
// is spec-only), so this shim covers only the path's inputs and mesh plumbing.
#include <cstring>

#include "nestmesh/lattice.hpp"
#include "nestmesh/mesh.hpp"
#include "nestmesh/primitives.hpp"
#include "nestmesh/surface.hpp"

using namespace nestmesh;

extern "C" {

// primitives.hpp:29-54
void ref_icosphere(double radius, int level, const double* c, double* xyz, std::uint32_t* tri) {
  const TriangleSurface s = icosphere(radius, level, Vec3{c[0], c[1], c[2]});
  for (std::size_t i = 0; i < s.positions.size(); ++i) {
    xyz[3 * i] = s.positions[i].x;
    xyz[3 * i + 1] = s.positions[i].y;
    xyz[3 * i + 2] = s.positions[i].z;
  }
  for (std::size_t i = 0; i < s.triangles.size(); ++i) std::memcpy(tri + 3 * i, s.triangles[i].data(), 12);
}

// primitives.hpp:75-87
void ref_box_surface(const double* lo, const double* hi, double* xyz, std::uint32_t* tri) {
  Aabb b;
  b.lo = Vec3{lo[0], lo[1], lo[2]};
  b.hi = Vec3{hi[0], hi[1], hi[2]};
  const TriangleSurface s = box_surface(b);
  for (std::size_t i = 0; i < s.positions.size(); ++i) {
    xyz[3 * i] = s.positions[i].x;
    xyz[3 * i + 1] = s.positions[i].y;
    xyz[3 * i + 2] = s.positions[i].z;
  }
  for (std::size_t i = 0; i < s.triangles.size(); ++i) std::memcpy(tri + 3 * i, s.triangles[i].data(), 12);
}

// lattice.hpp:40-91
void ref_lattice_mesh(const double* origin, double h, int nx, int ny, int nz, double* nodes, std::uint32_t* tets) {
  LatticeSpec spec;
  spec.origin = Vec3{origin[0], origin[1], origin[2]};
  spec.cell_size = h;
  spec.nx = nx;
  spec.ny = ny;
  spec.nz = nz;
  const TetrahedralMesh m = generate_lattice_mesh(spec);
  for (std::size_t i = 0; i < m.nodes.size(); ++i) {
    nodes[3 * i] = m.nodes[i].x;
    nodes[3 * i + 1] = m.nodes[i].y;
    nodes[3 * i + 2] = m.nodes[i].z;
  }
  for (std::size_t i = 0; i < m.tetrahedra.size(); ++i) std::memcpy(tets + 4 * i, m.tetrahedra[i].data(), 16);
}

// lattice.hpp:25-34
void ref_lattice_covering(const double* lo, const double* hi, double h, double* origin, int* n) {
  Aabb b;
  b.lo = Vec3{lo[0], lo[1], lo[2]};
  b.hi = Vec3{hi[0], hi[1], hi[2]};
  const LatticeSpec s = lattice_covering(b, h);
  origin[0] = s.origin.x;
  origin[1] = s.origin.y;
  origin[2] = s.origin.z;
  n[0] = s.nx;
  n[1] = s.ny;
  n[2] = s.nz;
}

// surface.hpp:80-104 — returns open-edge count + orientation-error count.
int ref_validate_closed(const double* xyz, std::size_t nv, const std::uint32_t* tri, std::size_t nt) {
  TriangleSurface s;
  s.positions.resize(nv);
  for (std::size_t i = 0; i < nv; ++i) s.positions[i] = Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  s.triangles.resize(nt);
  for (std::size_t i = 0; i < nt; ++i) std::memcpy(s.triangles[i].data(), tri + 3 * i, 12);
  const ClosednessReport r = validate_closed(s);
  return static_cast<int>(r.open_edges.size() + r.orientation_errors.size());
}

// surface.hpp:40-45
double ref_signed_volume(const double* xyz, std::size_t nv, const std::uint32_t* tri, std::size_t nt) {
  TriangleSurface s;
  s.positions.resize(nv);
  for (std::size_t i = 0; i < nv; ++i) s.positions[i] = Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  s.triangles.resize(nt);
  for (std::size_t i = 0; i < nt; ++i) std::memcpy(s.triangles[i].data(), tri + 3 * i, 12);
  return s.signed_volume();
}

// mesh.hpp:134-142 — number of boundary triangles of one label; -1 on UnknownLabel.
long ref_compartment_boundary_size(const double* nodes, std::size_t nn, const std::uint32_t* tets, std::size_t nt,
                                   const int* labels, int label) {
  TetrahedralMesh m;
  m.nodes.resize(nn);
  for (std::size_t i = 0; i < nn; ++i) m.nodes[i] = Vec3{nodes[3 * i], nodes[3 * i + 1], nodes[3 * i + 2]};
  m.tetrahedra.resize(nt);
  for (std::size_t i = 0; i < nt; ++i) std::memcpy(m.tetrahedra[i].data(), tets + 4 * i, 16);
  m.labels.assign(labels, labels + nt);
  try {
    return static_cast<long>(extract_compartment_boundary(m, label).triangles.size());
  } catch (const UnknownLabel&) {
    return -1;
  }
}

// mesh.hpp:100-155 — the reference's boundary of one label (n_set == 1,
// extract_compartment_boundary) or of a label set (extract_region_boundary).
// Returns the triangle count (-1 on UnknownLabel); copies up to the given
// capacities.
long ref_boundary(const std::uint32_t* tets, std::size_t nt, const int* labels, const int* label_set, int n_set,
                  std::uint32_t* tri_out, std::size_t tri_cap, std::uint32_t* nodes_out, std::size_t nodes_cap,
                  std::size_t* n_nodes) {
  TetrahedralMesh m;
  m.tetrahedra.resize(nt);
  for (std::size_t i = 0; i < nt; ++i) std::memcpy(m.tetrahedra[i].data(), tets + 4 * i, 16);
  m.labels.assign(labels, labels + nt);
  CompartmentBoundary b;
  try {
    if (n_set == 1) b = extract_compartment_boundary(m, label_set[0]);
    else b = extract_region_boundary(m, std::vector<int>(label_set, label_set + n_set));
  } catch (const UnknownLabel&) {
    return -1;
  }
  for (std::size_t i = 0; i < b.triangles.size() && i < tri_cap; ++i) std::memcpy(tri_out + 3 * i, b.triangles[i].data(), 12);
  for (std::size_t i = 0; i < b.nodes.size() && i < nodes_cap; ++i) nodes_out[i] = b.nodes[i];
  *n_nodes = b.nodes.size();
  return static_cast<long>(b.triangles.size());
}

// mesh.hpp:194-235 — 1 when validate_mesh reports no findings.
int ref_validate_mesh_ok(const double* nodes, std::size_t nn, const std::uint32_t* tets, std::size_t nt) {
  TetrahedralMesh m;
  m.nodes.resize(nn);
  for (std::size_t i = 0; i < nn; ++i) m.nodes[i] = Vec3{nodes[3 * i], nodes[3 * i + 1], nodes[3 * i + 2]};
  m.tetrahedra.resize(nt);
  for (std::size_t i = 0; i < nt; ++i) std::memcpy(m.tetrahedra[i].data(), tets + 4 * i, 16);
  m.labels.assign(nt, 0);
  return validate_mesh(m).ok() ? 1 : 0;
}

// mesh.hpp:238-289 tetmesh v1 text export / import (the format the label
// sidecar sits next to)
int ref_save_tetmesh(const char* path, const double* nodes, std::size_t nn, const std::uint32_t* tets,
                     const int* labels, std::size_t nt) {
  try {
    TetrahedralMesh m;
    m.nodes.resize(nn);
    for (std::size_t i = 0; i < nn; ++i) m.nodes[i] = Vec3{nodes[3 * i], nodes[3 * i + 1], nodes[3 * i + 2]};
    m.tetrahedra.resize(nt);
    m.labels.assign(labels, labels + nt);
    for (std::size_t t = 0; t < nt; ++t) std::memcpy(m.tetrahedra[t].data(), tets + 4 * t, 16);
    save_tetmesh(path, m);
    return 0;
  } catch (...) {
    return 1;
  }
}

// sizes first (nodes/tets/labels null), then the arrays
int ref_load_tetmesh(const char* path, std::size_t* nn, std::size_t* nt, double* nodes, std::uint32_t* tets,
                     int* labels) {
  try {
    const TetrahedralMesh m = load_tetmesh(path);
    *nn = m.node_count();
    *nt = m.tet_count();
    if (nodes)
      for (std::size_t i = 0; i < m.node_count(); ++i) {
        nodes[3 * i] = m.nodes[i].x;
        nodes[3 * i + 1] = m.nodes[i].y;
        nodes[3 * i + 2] = m.nodes[i].z;
      }
    if (tets)
      for (std::size_t t = 0; t < m.tet_count(); ++t) std::memcpy(tets + 4 * t, m.tetrahedra[t].data(), 16);
    if (labels) std::memcpy(labels, m.labels.data(), m.tet_count() * sizeof(int));
    return 0;
  } catch (...) {
    return 1;
  }
}

}  // extern "C"
