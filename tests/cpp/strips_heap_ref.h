// TEST ONLY: the lazy-heap version of csrc/strips.h (before the bitset degree
// buckets), kept as the order reference for tests/cpp/strips_equiv.cpp.
// Greedy triangle-strip decomposition of one compartment,
// (Was: host code shared by nm_set_surfaces and tests/cpp/strips_check.cpp.)
#pragma once

#include <cstddef>
#include <algorithm>
#include <cstdint>
#include <functional>
#include <queue>
#include <utility>
#include <vector>

namespace nmh_heap {

// Start from the unused triangle with the fewest unused neighbours, try its
// three rotations, walk forward across (u_{k+1}, u_{k+2}) and backward from the
// reversed start, keep the longest. Returns, per strip, the vertex sequence
// u_0..u_{m+1} and the original triangle ids t_0..t_{m-1} with
// {u_k, u_{k+1}, u_{k+2}} == set(t_k). Only performance depends on the
// quality of the decomposition; every triangle appears in exactly one strip.
struct Strip {
  std::vector<std::uint32_t> v;
  std::vector<std::uint32_t> t;
};

inline std::vector<Strip> stripify(const std::uint32_t* tri, std::uint32_t t0, std::uint32_t t1, std::size_t nv) {
  const std::uint32_t m = t1 - t0;
  if (m == 0) return {};
  (void)nv;
  // edge adjacency through vertex -> incident-triangle lists (counting sort
  // over the compartment's vertex id range, linear time): adj[3 i + j] = the
  // other triangle on edge (e_j, e_{j+1}) of triangle i, -1 on a border
  std::uint32_t vlo = 0xffffffffu, vhi = 0;
  for (std::size_t q = 3 * std::size_t(t0); q < 3 * std::size_t(t1); ++q) {
    vlo = std::min(vlo, tri[q]);
    vhi = std::max(vhi, tri[q]);
  }
  const std::size_t nloc = std::size_t(vhi) - vlo + 1;
  std::vector<std::uint32_t> start(nloc + 1, 0);
  for (std::uint32_t i = 0; i < m; ++i)
    for (int j = 0; j < 3; ++j) ++start[tri[3 * std::size_t(t0 + i) + j] - vlo + 1];
  for (std::size_t v = 0; v < nloc; ++v) start[v + 1] += start[v];
  // incidence entries carry the triangle's three vertices (sequential scans
  // instead of a random triangle load per candidate)
  struct Inc {
    std::uint32_t t, v[3];
  };
  std::vector<Inc> inc(3 * std::size_t(m));
  {
    std::vector<std::uint32_t> cur(start.begin(), start.end() - 1);
    for (std::uint32_t i = 0; i < m; ++i) {
      const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
      for (int j = 0; j < 3; ++j) inc[cur[e[j] - vlo]++] = {i, {e[0], e[1], e[2]}};
    }
  }
  std::vector<std::int32_t> adj(3 * std::size_t(m), -1);
  for (std::uint32_t i = 0; i < m; ++i) {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    for (int j = 0; j < 3; ++j) {
      const std::uint32_t a = e[j] - vlo, b = e[(j + 1) % 3];
      for (std::uint32_t q = start[a]; q < start[a + 1]; ++q) {
        const Inc& o = inc[q];
        if (o.t == i) continue;
        if (o.v[0] == b || o.v[1] == b || o.v[2] == b) {
          adj[3 * std::size_t(i) + j] = static_cast<std::int32_t>(o.t);
          break;
        }
      }
    }
  }
  std::vector<std::uint8_t> used(m, 0);
  auto nbr = [&](std::uint32_t i, std::uint32_t a, std::uint32_t b) -> std::int64_t {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    for (int j = 0; j < 3; ++j) {
      const std::uint32_t x = e[j], y = e[(j + 1) % 3];
      if ((x == a && y == b) || (x == b && y == a)) return adj[3 * std::size_t(i) + j];
    }
    return -1;
  };
  std::vector<int> deg(m, 0);
  for (std::uint32_t i = 0; i < m; ++i) {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    if (e[0] != e[1] && e[1] != e[2] && e[0] != e[2]) {  // distinct vertices: edge j is the first match of itself
      deg[i] = (adj[3 * std::size_t(i)] >= 0) + (adj[3 * std::size_t(i) + 1] >= 0) + (adj[3 * std::size_t(i) + 2] >= 0);
    } else {
      for (int j = 0; j < 3; ++j) deg[i] += nbr(i, e[j], e[(j + 1) % 3]) >= 0;
    }
  }
  // Next start: the unused triangle with the smallest (degree, index).
  // Degrees only decrease, so degree 3 is a forward scan; degrees 0..2 (and
  // negative ones, possible only at non-manifold edges) are lazy min-heaps.
  using MinHeap = std::priority_queue<std::uint32_t, std::vector<std::uint32_t>, std::greater<std::uint32_t>>;
  using QE = std::pair<int, std::uint32_t>;
  MinHeap bucket[3];
  std::priority_queue<QE, std::vector<QE>, std::greater<QE>> negative;
  std::uint32_t scan3 = 0;
  for (std::uint32_t i = 0; i < m; ++i)
    if (deg[i] < 3) bucket[deg[i]].push(i);
  auto push = [&](std::uint32_t n) {
    const int d = --deg[n];
    if (d >= 0) bucket[d].push(n);
    else negative.emplace(d, n);
  };
  auto next = [&](std::uint32_t& out) {
    while (!negative.empty()) {
      const QE q = negative.top();
      if (!used[q.second] && deg[q.second] == q.first) {
        out = q.second;
        return true;
      }
      negative.pop();
    }
    for (int b = 0; b < 3; ++b)
      while (!bucket[b].empty()) {
        const std::uint32_t i = bucket[b].top();
        if (!used[i] && deg[i] == b) {
          out = i;
          return true;
        }
        bucket[b].pop();
      }
    while (scan3 < m && (used[scan3] || deg[scan3] != 3)) ++scan3;
    if (scan3 < m) {
      out = scan3;
      return true;
    }
    return false;
  };
  std::vector<std::uint32_t> mark(m, 0);
  std::uint32_t stamp = 0;
  // forward walk from triangle i with vertex order (a,b,c)
  auto walk = [&](std::uint32_t i, std::uint32_t a, std::uint32_t b, std::uint32_t c, std::vector<std::uint32_t>& vs,
                  std::vector<std::uint32_t>& ts) {
    vs.assign({a, b, c});
    ts.assign({i});
    mark[i] = stamp;
    std::uint32_t cur = i;
    for (;;) {
      const std::uint32_t u = vs[vs.size() - 2], w = vs.back();
      const std::uint32_t* ec = tri + 3 * std::size_t(t0 + cur);
      int j = 0;  // the first edge of cur on {u, w} (nbr's rule)
      while (j < 3 && !((ec[j] == u && ec[(j + 1) % 3] == w) || (ec[j] == w && ec[(j + 1) % 3] == u))) ++j;
      if (j == 3) break;
      const std::int64_t n = adj[3 * std::size_t(cur) + j];
      if (n < 0 || used[n] || mark[n] == stamp) break;
      const std::uint32_t* en = tri + 3 * std::size_t(t0 + n);
      std::uint32_t x = en[0];  // the neighbour's last vertex not on the edge
      for (int q = 0; q < 3; ++q)
        if (en[q] != u && en[q] != w) x = en[q];
      vs.push_back(x);
      ts.push_back(static_cast<std::uint32_t>(n));
      mark[n] = stamp;
      cur = static_cast<std::uint32_t>(n);
    }
  };
  std::vector<Strip> out;
  std::vector<std::uint32_t> fv, ft, bv, btt;
  Strip s;
  std::uint32_t i = 0;
  while (next(i)) {
    const std::uint32_t* e = tri + 3 * std::size_t(t0 + i);
    Strip best;
    for (int r = 0; r < 3; ++r) {
      const std::uint32_t a = e[r], b = e[(r + 1) % 3], c = e[(r + 2) % 3];
      ++stamp;
      walk(i, a, b, c, fv, ft);
      // backward: walk from the reversed start without reusing forward triangles
      walk(i, c, b, a, bv, btt);
      // bv = c,b,a,x,y,...; combined vertex sequence = reverse(bv) + fv[3:]
      if (btt.size() + ft.size() - 1 <= best.t.size()) continue;  // not longer: keep the earlier rotation
      s.v.assign(bv.rbegin(), bv.rend());
      s.v.insert(s.v.end(), fv.begin() + 3, fv.end());
      s.t.assign(btt.rbegin(), btt.rend());  // ..., i
      s.t.insert(s.t.end(), ft.begin() + 1, ft.end());
      std::swap(best, s);
    }
    for (std::uint32_t t : best.t) used[t] = 1;
    for (std::uint32_t t : best.t) {
      const std::uint32_t* f = tri + 3 * std::size_t(t0 + t);
      for (int j = 0; j < 3; ++j) {
        const std::int64_t n = nbr(t, f[j], f[(j + 1) % 3]);
        if (n >= 0 && !used[n]) push(static_cast<std::uint32_t>(n));
      }
    }
    for (auto& t : best.t) t += t0;
    out.push_back(std::move(best));
  }
  return out;
}

}  // namespace nmh_heap
