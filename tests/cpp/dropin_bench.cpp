// The C++ drop-in's end-to-end time, as a nestmesh user sees it: the mesh and
// segmentation live in the reference's own types (std::vector-backed,
// PAGEABLE memory), a persistent nestmesh::Labeler (include/nestmesh/
// labeling.hpp) is built once, initial_label runs `steps` times. Timed on the
// host clock around each call: H2D of the nodes and tets, the labeling, D2H
// of the labels into a std::vector.
//
// Built where the reference headers exist (paper_2203_10000_b200/build.py) as
// build/libdropin_bench.so; bench.py loads it with ctypes and passes its
// synthetic inputs (the surfaces and lattice of BASELINE configs[4]).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <vector>

#include "nestmesh/labeling.hpp"

using namespace nestmesh;

extern "C" int dropin_bench(const double* sxyz, std::size_t nv, const std::uint32_t* stri, const std::uint32_t* comp_off,
                            int K, const int* label_ids, const double* nodes, std::size_t n, const std::uint32_t* tets,
                            std::size_t nt, int cull, int steps, double* out, int* labels_out) {
  try {
    // the user's data: reference types, pageable storage
    SurfaceSegmentation seg;
    for (int k = 0; k < K; ++k) {
      TriangleSurface s;
      std::vector<std::uint32_t> remap(nv, 0xffffffffu);
      for (std::uint32_t t = comp_off[k]; t < comp_off[k + 1]; ++t) {
        Triangle tr;
        for (int a = 0; a < 3; ++a) {
          const std::uint32_t v = stri[3 * std::size_t(t) + a];
          if (remap[v] == 0xffffffffu) {
            remap[v] = static_cast<std::uint32_t>(s.positions.size());
            s.positions.push_back(Vec3{sxyz[3 * std::size_t(v)], sxyz[3 * std::size_t(v) + 1], sxyz[3 * std::size_t(v) + 2]});
          }
          tr[a] = remap[v];
        }
        s.triangles.push_back(tr);
      }
      seg.compartments.push_back(CompartmentSurface{"c" + std::to_string(k), label_ids[k], std::move(s), 1.0, k + 1, true});
    }
    TetrahedralMesh mesh;
    mesh.nodes.resize(n);
    std::memcpy(static_cast<void*>(mesh.nodes.data()), nodes, n * sizeof(Vec3));
    mesh.tetrahedra.resize(nt);
    std::memcpy(static_cast<void*>(mesh.tetrahedra.data()), tets, nt * sizeof(Tet));
    mesh.labels.assign(nt, 0);

    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    GpuOptions o;
    o.opt.cull_outside = cull;
    const auto t0 = clk::now();
    Labeler lab(seg, o);  // validate_closed + flatten + upload + tiles (+ certified cells)
    const auto t1 = clk::now();
    SolidAngleParams params;
    std::vector<int> labels = lab.initial_label(mesh, params);  // warm-up (first-use allocations)
    const auto t2 = clk::now();
    double total = 0.0, best = 1e300, total_into = 0.0, best_into = 1e300;
    for (int i = 0; i < steps; ++i) {  // by value: a fresh std::vector<int> per call
      const auto a = clk::now();
      labels = lab.initial_label(mesh, params);
      const double d = sec(a, clk::now());
      total += d;
      best = d < best ? d : best;
    }
    for (int i = 0; i < steps; ++i) {  // into mesh.labels (reused storage)
      const auto a = clk::now();
      lab.initial_label_into(mesh, params, mesh.labels);
      const double d = sec(a, clk::now());
      total_into += d;
      best_into = d < best_into ? d : best_into;
    }
    if (mesh.labels != labels) throw std::runtime_error("initial_label_into != initial_label");
    out[0] = sec(t0, t1);
    out[1] = sec(t1, t2);
    out[2] = steps ? total / steps : 0.0;
    out[3] = steps ? best : 0.0;
    out[4] = steps ? total_into / steps : 0.0;
    out[5] = steps ? best_into : 0.0;
    std::memcpy(labels_out, labels.data(), nt * sizeof(int));
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "dropin_bench: %s\n", e.what());
    return 1;
  }
}
