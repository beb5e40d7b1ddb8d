// Internal: refined-mesh container shared by refine.cpp and the recursive
// driver in nestmesh_label.cu (opaque nm_mesh of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

struct nm_mesh {
  std::vector<double> nodes;          // fp64 xyz, old nodes first
  std::vector<std::uint32_t> tets;    // 4 per tet
  std::vector<int> labels;            // 1 per tet
  std::vector<std::uint32_t> parent;  // parent tet of each child (w.r.t. the last refinement)
  std::vector<std::uint32_t> masks;   // node masks (filled by the recursive driver)
  std::size_t n_old = 0;              // node count before the last refinement
};

namespace nmi {
// refine_volume; throws std::invalid_argument on bad input.
nm_mesh* refine(const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, const int* labels,
                const std::uint32_t* selected, std::size_t n_selected);
}  // namespace nmi
