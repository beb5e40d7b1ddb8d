// CPU check that csrc/strips.h (exact bitset degree buckets) returns the same
// strips as the lazy-heap version it replaced (strips_heap_ref.h) on random
// triangle soups: non-manifold edges (negative degrees), degenerate triangles,
// repeated triangles, empty and partial compartment ranges. Argv: seed,
// iterations. Prints "ok <strips compared>" or the first mismatch.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "strips.h"
#include "strips_heap_ref.h"

int main(int argc, char** argv) {
  const unsigned seed = argc > 1 ? static_cast<unsigned>(std::atoi(argv[1])) : 7u;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 3000;
  std::mt19937 rng(seed);
  std::size_t compared = 0;
  for (int it = 0; it < iters; ++it) {
    const std::uint32_t nv = 3 + rng() % 60, nt = 1 + rng() % 400;
    std::vector<std::uint32_t> tri(3 * std::size_t(nt));
    if (it % 3 == 0) {  // a band of mostly edge-adjacent triangles
      for (std::uint32_t i = 0; i < nt; ++i) {
        tri[3 * i] = (i + rng() % 3) % nv;
        tri[3 * i + 1] = (i + 1) % nv;
        tri[3 * i + 2] = (i + 2 + rng() % 2) % nv;
      }
    } else {
      for (auto& x : tri) x = rng() % nv;
    }
    const std::uint32_t t0 = rng() % nt, t1 = t0 + rng() % (nt - t0 + 1);
    const auto a = nmh_heap::stripify(tri.data(), t0, t1, nv);
    const auto b = nmh::stripify(tri.data(), t0, t1, nv);
    if (a.size() != b.size()) {
      std::printf("strip count mismatch at iteration %d: %zu vs %zu\n", it, a.size(), b.size());
      return 1;
    }
    for (std::size_t i = 0; i < a.size(); ++i)
      if (a[i].v != b[i].v || a[i].t != b[i].t) {
        std::printf("strip %zu differs at iteration %d\n", i, it);
        return 1;
      }
    compared += a.size();
  }
  std::printf("ok %zu\n", compared);
  return 0;
}
