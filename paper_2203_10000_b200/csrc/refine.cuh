// Device refine_volume for the recursive driver (SPEC.md:285-293, 311-312,
// 321). Same rules, same node numbering and the same child order as the host
// restatement in refine.cpp — the two produce bit-identical meshes
// (tests/test_gpu_parity.py::test_device_refine_matches_host):
//   * closure: red tets put their 6 edges in the split set S (sorted unique
//     64-bit edge keys); a non-red tet whose split-edge pattern is not one
//     edge / two edges of one face / one full face turns red; repeat;
//   * midpoint of S[i] is node n + i at (p_a + p_b) * 0.5;
//   * children are written in parent order at scan offsets.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nm {

__device__ __forceinline__ unsigned long long ekey_d(std::uint32_t a, std::uint32_t b) {
  return a < b ? (static_cast<unsigned long long>(a) << 32 | b) : (static_cast<unsigned long long>(b) << 32 | a);
}

__device__ __forceinline__ int lower_bound_key(const unsigned long long* S, int m, unsigned long long k) {
  int lo = 0, hi = m;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool has_key(const unsigned long long* S, int m, unsigned long long k) {
  const int i = lower_bound_key(S, m, k);
  return i < m && S[i] == k;
}

static __constant__ int kEdgeD[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// 6-bit split-edge mask -> pattern: 0 none, 1 one edge, 2 two edges of one
// face, 3 one full face, -1 escalate (the host classify()).
__device__ __forceinline__ int pattern_of(unsigned mask) {
  const int cnt = __popc(mask);
  if (cnt == 0) return 0;
  if (cnt == 1) return 1;
  if (cnt == 6) return -1;
  int touched = 0;
  for (int k = 0; k < 6; ++k)
    if (mask & (1u << k)) touched |= (1 << kEdgeD[k][0]) | (1 << kEdgeD[k][1]);
  const int nv = __popc(touched);
  if (cnt == 2 && nv == 3) return 2;
  if (cnt == 3 && nv == 3) return 3;
  return -1;
}

static __global__ void k_mark_list(const std::uint32_t* ids, const std::uint32_t* count, std::uint8_t* flag) {
  const std::uint32_t n = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) flag[ids[i]] = 1;
}

static __global__ void k_red_edges(const uint4* tets, const std::uint32_t* red_list, const std::uint32_t* count,
                            unsigned long long* keys) {
  const std::uint32_t n = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint4 t = tets[red_list[i]];
    const std::uint32_t v[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int k = 0; k < 6; ++k) keys[6 * static_cast<std::size_t>(i) + k] = ekey_d(v[kEdgeD[k][0]], v[kEdgeD[k][1]]);
  }
}

struct PredUniqueKey {
  const unsigned long long* k;
  __device__ bool operator()(std::size_t i) const { return i == 0 || k[i] != k[i - 1]; }
};

static __global__ void k_gather_keys(const unsigned long long* src, const std::uint32_t* idx, const std::uint32_t* count,
                              unsigned long long* dst) {
  const std::uint32_t n = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}

static __global__ void k_touch_nodes(const unsigned long long* S, const std::uint32_t* count, std::uint8_t* touched) {
  const std::uint32_t n = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    touched[static_cast<std::uint32_t>(S[i] >> 32)] = 1;
    touched[static_cast<std::uint32_t>(S[i])] = 1;
  }
}

// Split masks of every tet; non-red tets with an escalating pattern turn red.
static __global__ void k_classify(const uint4* tets, std::size_t nt, std::uint8_t* red, const std::uint8_t* touched,
                           const unsigned long long* S, const std::uint32_t* count, std::uint8_t* mask_out,
                           unsigned* changed) {
  const int m = static_cast<int>(*count);
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    if (red[t]) {
      mask_out[t] = 0x3f;
      continue;
    }
    const uint4 e = tets[t];
    const std::uint32_t v[4] = {e.x, e.y, e.z, e.w};
    unsigned mask = 0;
    if (touched[e.x] | touched[e.y] | touched[e.z] | touched[e.w]) {
#pragma unroll
      for (int k = 0; k < 6; ++k)
        if (has_key(S, m, ekey_d(v[kEdgeD[k][0]], v[kEdgeD[k][1]]))) mask |= 1u << k;
    }
    if (pattern_of(mask) < 0) {
      red[t] = 1;
      mask_out[t] = 0x3f;
      *changed = 1u;
    } else {
      mask_out[t] = static_cast<std::uint8_t>(mask);
    }
  }
}

static __global__ void k_child_count(const std::uint8_t* mask, std::size_t nt, std::uint32_t* cnt) {
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const unsigned m = mask[t];
    const int p = m == 0x3f ? 4 : pattern_of(m);
    cnt[t] = p == 0 ? 1u : p == 1 ? 2u : p == 2 ? 3u : p == 3 ? 4u : 8u;
  }
}

static __global__ void k_midpoints(const double* nodes, const unsigned long long* S, const std::uint32_t* count,
                            std::size_t n_old, double* out) {
  const std::uint32_t m = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const std::uint32_t a = static_cast<std::uint32_t>(S[i] >> 32), b = static_cast<std::uint32_t>(S[i]);
#pragma unroll
    for (int d = 0; d < 3; ++d)
      out[3 * (n_old + i) + d] = __dmul_rn(__dadd_rn(nodes[3 * static_cast<std::size_t>(a) + d],
                                                     nodes[3 * static_cast<std::size_t>(b) + d]), 0.5);
  }
}

struct EmitCtx {
  const double* P;  // refined node array (old + midpoints)
  uint4* out;
  int* labels_out;
  std::uint32_t* parent_out;
  std::size_t pos;
  std::uint32_t parent;
  int label;
  __device__ void emit(std::uint32_t a, std::uint32_t b, std::uint32_t c, std::uint32_t d) {
    const double* A = P + 3 * static_cast<std::size_t>(a);
    const double* B = P + 3 * static_cast<std::size_t>(b);
    const double* C = P + 3 * static_cast<std::size_t>(c);
    const double* D = P + 3 * static_cast<std::size_t>(d);
    const double u0 = __dsub_rn(B[0], A[0]), u1 = __dsub_rn(B[1], A[1]), u2 = __dsub_rn(B[2], A[2]);
    const double v0 = __dsub_rn(C[0], A[0]), v1 = __dsub_rn(C[1], A[1]), v2 = __dsub_rn(C[2], A[2]);
    const double w0 = __dsub_rn(D[0], A[0]), w1 = __dsub_rn(D[1], A[1]), w2 = __dsub_rn(D[2], A[2]);
    const double x0 = __dsub_rn(__dmul_rn(v1, w2), __dmul_rn(v2, w1));
    const double x1 = __dsub_rn(__dmul_rn(v2, w0), __dmul_rn(v0, w2));
    const double x2 = __dsub_rn(__dmul_rn(v0, w1), __dmul_rn(v1, w0));
    const double vol = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(u0, x0), __dmul_rn(u1, x1)), __dmul_rn(u2, x2)), 6.0);
    out[pos] = vol < 0.0 ? make_uint4(a, b, d, c) : make_uint4(a, b, c, d);
    labels_out[pos] = label;
    parent_out[pos] = parent;
    ++pos;
  }
};

__device__ __forceinline__ double dist2_d(const double* P, std::uint32_t a, std::uint32_t b) {
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = __dsub_rn(P[3 * static_cast<std::size_t>(a) + d], P[3 * static_cast<std::size_t>(b) + d]);
    s = __dadd_rn(s, __dmul_rn(x, x));
  }
  return s;
}

static __global__ void k_emit_children(const uint4* tets, std::size_t nt, const std::uint8_t* mask, const std::uint32_t* offs,
                                const int* labels_in, const unsigned long long* S, const std::uint32_t* count,
                                std::size_t n_old, const double* P, uint4* out, int* labels_out,
                                std::uint32_t* parent_out) {
  const int m = static_cast<int>(*count);
  auto mid = [&](std::uint32_t a, std::uint32_t b) {
    return static_cast<std::uint32_t>(n_old + lower_bound_key(S, m, ekey_d(a, b)));
  };
  for (std::size_t ti = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; ti < nt;
       ti += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const uint4 e4 = tets[ti];
    const std::uint32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
    EmitCtx E{P, out, labels_out, parent_out, offs[ti], static_cast<std::uint32_t>(ti), labels_in[ti]};
    const unsigned msk = mask[ti];
    if (msk == 0x3f) {
      const std::uint32_t v0 = e[0], v1 = e[1], v2 = e[2], v3 = e[3];
      const std::uint32_t m01 = mid(v0, v1), m02 = mid(v0, v2), m03 = mid(v0, v3), m12 = mid(v1, v2),
                          m13 = mid(v1, v3), m23 = mid(v2, v3);
      E.emit(v0, m01, m02, m03);
      E.emit(m01, v1, m12, m13);
      E.emit(m02, m12, v2, m23);
      E.emit(m03, m13, m23, v3);
      const std::uint32_t pr[3][2] = {{m01, m23}, {m02, m13}, {m03, m12}};
      int best = 0;
      double bd = dist2_d(P, pr[0][0], pr[0][1]);
      for (int k = 1; k < 3; ++k) {
        const double d = dist2_d(P, pr[k][0], pr[k][1]);
        const std::uint32_t klo = min(pr[k][0], pr[k][1]), khi = max(pr[k][0], pr[k][1]);
        const std::uint32_t blo = min(pr[best][0], pr[best][1]), bhi = max(pr[best][0], pr[best][1]);
        const bool lex = klo < blo || (klo == blo && khi < bhi);
        if (d < bd || (d == bd && lex)) {
          bd = d;
          best = k;
        }
      }
      const std::uint32_t p = pr[best][0], q = pr[best][1];
      const std::uint32_t a = pr[(best + 1) % 3][0], a2 = pr[(best + 1) % 3][1];
      const std::uint32_t b = pr[(best + 2) % 3][0], b2 = pr[(best + 2) % 3][1];
      E.emit(p, q, a, b);
      E.emit(p, q, b, a2);
      E.emit(p, q, a2, b2);
      E.emit(p, q, b2, a);
      continue;
    }
    int which[6], cnt = 0;
    for (int k = 0; k < 6; ++k)
      if (msk & (1u << k)) which[cnt++] = k;
    const int pat = pattern_of(msk);
    if (pat == 0) {
      out[E.pos] = e4;
      labels_out[E.pos] = E.label;
      parent_out[E.pos] = E.parent;
    } else if (pat == 1) {
      const std::uint32_t a = e[kEdgeD[which[0]][0]], b = e[kEdgeD[which[0]][1]];
      std::uint32_t o[2];
      int k = 0;
      for (int j = 0; j < 4; ++j)
        if (e[j] != a && e[j] != b) o[k++] = e[j];
      const std::uint32_t mm = mid(a, b);
      E.emit(a, mm, o[0], o[1]);
      E.emit(mm, b, o[0], o[1]);
    } else if (pat == 2) {
      const int* E0 = kEdgeD[which[0]];
      const int* E1 = kEdgeD[which[1]];
      const int ia = (E0[0] == E1[0] || E0[0] == E1[1]) ? E0[0] : E0[1];
      const int ib = E0[0] == ia ? E0[1] : E0[0];
      const int ic = E1[0] == ia ? E1[1] : E1[0];
      const int id = 6 - ia - ib - ic;
      const std::uint32_t a = e[ia], b = e[ib], c = e[ic], d = e[id];
      const std::uint32_t mab = mid(a, b), mac = mid(a, c);
      E.emit(d, a, mab, mac);
      if (c < b) {
        E.emit(d, mab, b, c);
        E.emit(d, mab, c, mac);
      } else {
        E.emit(d, mab, b, mac);
        E.emit(d, b, c, mac);
      }
    } else {
      int touched = 0;
      for (int k = 0; k < 3; ++k) touched |= (1 << kEdgeD[which[k]][0]) | (1 << kEdgeD[which[k]][1]);
      int id = 0;
      while (touched & (1 << id)) ++id;
      int f[3], k = 0;
      for (int j = 0; j < 4; ++j)
        if (j != id) f[k++] = j;
      const std::uint32_t a = e[f[0]], b = e[f[1]], c = e[f[2]], d = e[id];
      const std::uint32_t mab = mid(a, b), mbc = mid(b, c), mca = mid(c, a);
      E.emit(d, a, mab, mca);
      E.emit(d, mab, b, mbc);
      E.emit(d, mca, mbc, c);
      E.emit(d, mab, mbc, mca);
    }
  }
}

}  // namespace nm
