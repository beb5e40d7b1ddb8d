// quality.boundary_distance kernel: unsigned distance from
// each sample point to a target triangle surface, exact point-triangle
// distance. Same N-body tile loop as the labeling kernel with a min-reduction
// instead of a sum.
//
//   (triangles are grouped in Morton-ordered clusters of 32 with bounding
//   spheres; both passes skip clusters that provably cannot matter)
//   pass 1 (fp32): d1 = min over triangles of the fp32 distance;
//   pass 2 (fp32 + fp64): every triangle whose fp32 distance is within
//     tol = 1e-3 mm + 1e-5 d1 of d1 (fp32 error at ~100 mm coordinates is
//     < 4e-5 mm) is re-evaluated in fp64 with the oracle's operand order;
//     the result is the fp64 minimum — bit-identical to the fp64 oracle's
//     min over all triangles, since the true minimiser is always a candidate.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nm {

template <class T>
struct Ops;
template <>
struct Ops<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <>
struct Ops<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

template <class T>
struct V3t {
  T x, y, z;
};

template <class T>
__device__ __forceinline__ V3t<T> vsub(V3t<T> a, V3t<T> b) {
  using O = Ops<T>;
  return {O::sub(a.x, b.x), O::sub(a.y, b.y), O::sub(a.z, b.z)};
}
template <class T>
__device__ __forceinline__ T vdot(V3t<T> a, V3t<T> b) {  // vec3.hpp:32 order
  using O = Ops<T>;
  return O::add(O::add(O::mul(a.x, b.x), O::mul(a.y, b.y)), O::mul(a.z, b.z));
}
template <class T>
__device__ __forceinline__ V3t<T> vcross(V3t<T> a, V3t<T> b) {  // vec3.hpp:34-36
  using O = Ops<T>;
  return {O::sub(O::mul(a.y, b.z), O::mul(a.z, b.y)), O::sub(O::mul(a.z, b.x), O::mul(a.x, b.z)),
          O::sub(O::mul(a.x, b.y), O::mul(a.y, b.x))};
}

// squared distance from ap = p - a to the segment a + t e, t in [0, 1]
template <class T>
__device__ __forceinline__ T seg_dist2(V3t<T> ap, V3t<T> e) {
  using O = Ops<T>;
  const T ee = vdot(e, e);
  T t = ee > T(0) ? O::div(vdot(ap, e), ee) : T(0);
  t = t < T(0) ? T(0) : (t > T(1) ? T(1) : t);
  const V3t<T> v{O::sub(ap.x, O::mul(t, e.x)), O::sub(ap.y, O::mul(t, e.y)), O::sub(ap.z, O::mul(t, e.z))};
  return vdot(v, v);
}

// Exact squared point-triangle distance: the plane distance when p projects
// inside the triangle, else the nearest of the three edges.
template <class T>
__device__ __forceinline__ T point_tri_dist2(V3t<T> p, V3t<T> a, V3t<T> b, V3t<T> c) {
  using O = Ops<T>;
  const V3t<T> ab = vsub(b, a), bc = vsub(c, b), ca = vsub(a, c);
  const V3t<T> ap = vsub(p, a), bp = vsub(p, b), cp = vsub(p, c);
  const V3t<T> n = vcross(ab, vsub(c, a));
  const T nn = vdot(n, n);
  const T s0 = vdot(vcross(ab, ap), n), s1 = vdot(vcross(bc, bp), n), s2 = vdot(vcross(ca, cp), n);
  if (nn > T(0) && s0 >= T(0) && s1 >= T(0) && s2 >= T(0)) {
    const T h = vdot(ap, n);
    return O::div(O::mul(h, h), nn);
  }
  T d = seg_dist2(ap, ab);
  const T d1 = seg_dist2(bp, bc), d2 = seg_dist2(cp, ca);
  d = d1 < d ? d1 : d;
  return d2 < d ? d2 : d;
}

constexpr int kDistCluster = 32;  // triangles per cluster (Morton order of centroids)

struct DistParams {
  const double* pts;     // n fp64 points (original frame)
  std::size_t n;
  const std::uint32_t* order;  // evaluation order of the points (Morton); results scattered back
  const float4* tri32;   // 3 float4 per triangle slot (a, b, c relative to (cx, cy, cz)), cluster order
  const std::uint32_t* slot_tri;  // original triangle of each slot (padding repeats a triangle)
  const float4* clus;    // per cluster: fp32 centre (centred frame), w = radius (rounded up)
  int nclus;
  const double* xyz;     // fp64 vertices (original frame)
  const std::uint32_t* tri;  // original triangles
  double cx, cy, cz;
  float* d32;            // pass-1 fp32 minimum distance per point
  double* out;           // fp64 distances
  unsigned long long* counters;  // [4] fp64 candidate evaluations, [5] fp32 cluster visits
};

// PASS 1: fp32 minimum; PASS 2: fp64 refinement over the candidates.
// Exact cluster culling: a cluster is skipped when the lower bound of its
// triangles' distance, |p - c| - rho, exceeds the bound (pass 1: the least
// upper bound min |p - c| + rho and the running minimum; pass 2: the
// candidate limit) by more than the fp32 error margin. A skipped cluster
// holds no triangle that could change the pass's result, so d32 and the
// candidate set — hence the fp64 minimum — are those of the full scan.
template <int PASS>
static __global__ void __launch_bounds__(256) k_point_surface_distance(const DistParams prm) {
  const std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  if (i >= prm.n) return;
  const std::size_t j = prm.order ? prm.order[i] : i;
  const double px = prm.pts[3 * j], py = prm.pts[3 * j + 1], pz = prm.pts[3 * j + 2];
  const V3t<float> p{static_cast<float>(px - prm.cx), static_cast<float>(py - prm.cy), static_cast<float>(pz - prm.cz)};
  const float margin = 1e-3f + 4e-6f * (fabsf(p.x) + fabsf(p.y) + fabsf(p.z));
  float best = 3.4e38f;
  double best64 = 1e300;
  float bound = 3.4e38f;
  if (PASS == 1) {
    for (int q = 0; q < prm.nclus; ++q) {  // least upper bound of the minimum distance
      const float4 s = __ldg(prm.clus + q);
      const float dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
      bound = fminf(bound, sqrtf(dx * dx + dy * dy + dz * dz) + s.w);
    }
  } else {
    const float d1 = prm.d32[j];
    bound = d1 + 1e-3f + 1e-5f * d1;  // candidate limit (as the full scan)
  }
  unsigned long long cand = 0, visits = 0;
  for (int q = 0; q < prm.nclus; ++q) {
    const float4 s = __ldg(prm.clus + q);
    const float dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
    const float lb = sqrtf(dx * dx + dy * dy + dz * dz) - s.w;
    if (lb > (PASS == 1 ? fminf(bound, best) : bound) + margin) continue;
    ++visits;
    for (int k = 0; k < kDistCluster; ++k) {
      const std::size_t t = static_cast<std::size_t>(q) * kDistCluster + k;
      const float4 A = __ldg(prm.tri32 + 3 * t), B = __ldg(prm.tri32 + 3 * t + 1), C = __ldg(prm.tri32 + 3 * t + 2);
      const float d = sqrtf(point_tri_dist2<float>(p, {A.x, A.y, A.z}, {B.x, B.y, B.z}, {C.x, C.y, C.z}));
      if (PASS == 1) {
        best = fminf(best, d);
      } else if (d <= bound) {
        const std::uint32_t* e = prm.tri + 3 * static_cast<std::size_t>(prm.slot_tri[t]);
        const double* a = prm.xyz + 3 * static_cast<std::size_t>(e[0]);
        const double* b = prm.xyz + 3 * static_cast<std::size_t>(e[1]);
        const double* c = prm.xyz + 3 * static_cast<std::size_t>(e[2]);
        const double q2 = point_tri_dist2<double>({px, py, pz}, {a[0], a[1], a[2]}, {b[0], b[1], b[2]},
                                                  {c[0], c[1], c[2]});
        best64 = q2 < best64 ? q2 : best64;
        ++cand;
      }
    }
  }
  if (PASS == 1) {
    prm.d32[j] = best;
    if (prm.counters) atomicAdd(prm.counters + 5, visits);
  } else {
    prm.out[j] = __dsqrt_rn(best64);
    if (prm.counters) atomicAdd(prm.counters + 4, cand);
  }
}

}  // namespace nm
