// CPU check of the strip decomposition (paper_2203_10000_b200/csrc/strips.h):
// every triangle in exactly one strip, consecutive strip triangles share an
// edge, and an order-dependent checksum of the output, so a faster stripify
// can be checked to produce the SAME strips (the packed tiles, hence every
// fp32 sum of k_label, depend on them). Input: a binary surface file
// (uint64 nv, nt, K; uint32 tri[3 nt]; uint32 comp_off[K + 1]).
// Prints: checksum, strips, triangles, milliseconds (one thread per
// compartment, sequential).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#include "strips.h"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  std::uint64_t h[3];
  if (std::fread(h, 8, 3, f) != 3) return 2;
  const std::size_t nv = h[0], nt = h[1], K = h[2];
  std::vector<std::uint32_t> tri(3 * nt), off(K + 1);
  if (std::fread(tri.data(), 4, tri.size(), f) != tri.size() || std::fread(off.data(), 4, off.size(), f) != off.size())
    return 2;
  std::fclose(f);
  std::uint64_t sum = 1469598103934665603ull, nstrips = 0, ntris = 0;
  auto mix = [&](std::uint64_t x) { sum = (sum ^ x) * 1099511628211ull; };
  double ms = 0;
  std::vector<int> seen(nt, 0);
  for (std::size_t k = 0; k < K; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<nmh::Strip> s = nmh::stripify(tri.data(), off[k], off[k + 1], nv);
    ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (const nmh::Strip& st : s) {
      if (st.v.size() != st.t.size() + 2) return 3;
      for (std::size_t i = 0; i < st.t.size(); ++i) {
        const std::uint32_t t = st.t[i];
        if (t < off[k] || t >= off[k + 1] || seen[t]++) return 4;
        const std::set<std::uint32_t> a{st.v[i], st.v[i + 1], st.v[i + 2]},
            b{tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
        if (a != b) return 5;
      }
      mix(st.v.size());
      for (std::uint32_t v : st.v) mix(v);
      for (std::uint32_t t : st.t) mix(t);
      ++nstrips;
      ntris += st.t.size();
    }
  }
  if (ntris != nt) return 6;
  std::printf("%016llx %llu %llu %.2f\n", static_cast<unsigned long long>(sum), static_cast<unsigned long long>(nstrips),
              static_cast<unsigned long long>(ntris), ms);
  return 0;
}
