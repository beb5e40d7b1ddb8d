// Host refinement (csrc/refine.cpp) under AddressSanitizer + UBSan: random
// lattice meshes and selections through the C ABI; checks conformity-free
// invariants cheaply (volume conservation, label inheritance, parent range).
// Built and run by tests/test_refine.py::test_refine_under_sanitizers (CPU).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "nestmesh_label.h"

static double tet_vol(const double* p, const uint32_t* t) {
  const double* a = p + 3 * t[0];
  const double* b = p + 3 * t[1];
  const double* c = p + 3 * t[2];
  const double* d = p + 3 * t[3];
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]},
               w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  return (u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0]) + u[2] * (v[0] * w[1] - v[1] * w[0])) / 6;
}

int main() {
  std::mt19937_64 rng(7);
  for (int round = 0; round < 6; ++round) {
    const int nx = 2 + round % 3, ny = 3, nz = 2 + round / 3;
    std::vector<double> nodes;
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
          nodes.push_back(i);
          nodes.push_back(j);
          nodes.push_back(k);
        }
    auto id = [&](int i, int j, int k) { return uint32_t((k * (ny + 1) + j) * (nx + 1) + i); };
    std::vector<uint32_t> tets;
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {  // 6-tet Kuhn split of the cell, all positively oriented
          const uint32_t v0 = id(i, j, k), v7 = id(i + 1, j + 1, k + 1);
          const uint32_t path[6][2] = {{id(i + 1, j, k), id(i + 1, j + 1, k)}, {id(i + 1, j, k), id(i + 1, j, k + 1)},
                                       {id(i, j + 1, k), id(i + 1, j + 1, k)}, {id(i, j + 1, k), id(i, j + 1, k + 1)},
                                       {id(i, j, k + 1), id(i + 1, j, k + 1)}, {id(i, j, k + 1), id(i, j + 1, k + 1)}};
          for (auto& pth : path) {
            uint32_t t[4] = {v0, pth[0], pth[1], v7};
            if (tet_vol(nodes.data(), t) < 0) std::swap(t[2], t[3]);
            tets.insert(tets.end(), t, t + 4);
          }
        }
    const size_t n = nodes.size() / 3, nt = tets.size() / 4;
    std::vector<int> labels(nt);
    for (auto& l : labels) l = int(rng() % 5);
    std::vector<uint32_t> sel;
    for (uint32_t t = 0; t < nt; ++t)
      if (rng() % 4 == 0) sel.push_back(t);
    nm_mesh* m = nullptr;
    if (nm_refine(nodes.data(), n, tets.data(), nt, labels.data(), sel.data(), sel.size(), &m) != 0) {
      std::printf("refine failed: %s\n", nm_refine_last_error());
      return 1;
    }
    size_t n2 = 0, nt2 = 0, nold = 0;
    nm_mesh_sizes(m, &n2, &nt2, &nold);
    std::vector<double> nn(3 * n2);
    std::vector<uint32_t> tt(4 * nt2), par(nt2);
    std::vector<int> ll(nt2);
    if (nm_mesh_copy(m, nn.data(), tt.data(), ll.data(), par.data()) != 0) return 2;
    nm_mesh_free(m);
    double v0 = 0, v1 = 0;
    for (size_t t = 0; t < nt; ++t) v0 += tet_vol(nodes.data(), &tets[4 * t]);
    for (size_t t = 0; t < nt2; ++t) {
      const double v = tet_vol(nn.data(), &tt[4 * t]);
      if (!(v > 0)) return 3;
      v1 += v;
      if (par[t] >= nt || ll[t] != labels[par[t]]) return 4;
      for (int q = 0; q < 4; ++q)
        if (tt[4 * t + q] >= n2) return 5;
    }
    if (std::fabs(v1 - v0) > 1e-9 * v0 || nold != n) return 6;
    // invalid input must be rejected, not crash
    const uint32_t bad = uint32_t(nt + 5);
    if (nm_refine(nodes.data(), n, tets.data(), nt, labels.data(), &bad, 1, &m) == 0) return 7;
  }
  std::printf("refine_asan ok\n");
  return 0;
}
