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
  // Device-resident result (device refinement / recursive driver): the
  // arrays stay in the producing device's memory, owned by this handle, and
  // nm_mesh_copy / nm_mesh_masks copy them straight into the caller's
  // buffers (no host staging copy). device < 0: the vectors above hold it.
  struct Device {
    int device = -1;
    std::size_t nn = 0, nt = 0;
    void *nodes = nullptr, *tets = nullptr, *labels = nullptr, *parent = nullptr, *masks = nullptr;
  } dev;
  nm_mesh() = default;
  nm_mesh(const nm_mesh&) = delete;
  nm_mesh& operator=(const nm_mesh&) = delete;
  ~nm_mesh();
  std::size_t node_count() const { return dev.device >= 0 ? dev.nn : nodes.size() / 3; }
  std::size_t tet_count() const { return dev.device >= 0 ? dev.nt : tets.size() / 4; }
};

namespace nmi {
// refine_volume; throws std::invalid_argument on bad input.
nm_mesh* refine(const double* nodes, std::size_t n, const std::uint32_t* tets, std::size_t nt, const int* labels,
                const std::uint32_t* selected, std::size_t n_selected);
}  // namespace nmi
