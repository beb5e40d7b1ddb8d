// Per-surface-set geometry on the device (nm_set_surfaces, round 2): the
// 13-DOP / bounding box of every compartment, and the Morton-ordered
// clusters of the certified-cell build (cells.cuh). Each kernel restates, in
// the same fp64 operations and order (explicit _rn intrinsics: no
// contraction), the host code it replaced, so its results are bit-identical:
//   * k_extents_items / k_extents_finalize: min / max over the compartment's
//     triangle corners of the 13 projections d . (x - ctr) (the first three
//     are the axis-aligned box), then the fp32 slabs of k_cull_mask, widened
//     by 1e-3 mm + 1e-5 |bound| and rounded outward;
//   * k_tri_morton: a triangle's centroid Morton key (10 bits per axis over
//     the domain box), sorted per compartment by a stable radix sort;
//   * k_cluster_spheres: one warp per cluster of kCluster consecutive sorted
//     triangles: the triangles' and the cluster's bounding spheres (fp32
//     centre of the vertex box, radius rounded up with the certification
//     margins).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nm {

constexpr int kExtQ = 2 * kDopDirs;  // per compartment: 13 minima, then 13 maxima

struct ExtentItem {
  int k;
  std::uint32_t t0, t1;  // triangle range of compartment k
};

__device__ __forceinline__ double dop_proj_rn(int j, double d0, double d1, double d2) {
  double pr = 0.0;
  pr = __dadd_rn(pr, __dmul_rn(static_cast<double>(dop_dir(j, 0)), d0));
  pr = __dadd_rn(pr, __dmul_rn(static_cast<double>(dop_dir(j, 1)), d1));
  pr = __dadd_rn(pr, __dmul_rn(static_cast<double>(dop_dir(j, 2)), d2));
  return pr;
}

// one block per item: partial min / max of the 13 projections (part[item][26])
static __global__ void __launch_bounds__(256) k_extents_items(const ExtentItem* __restrict__ items,
                                                              const double* __restrict__ xyz,
                                                              const std::uint32_t* __restrict__ tri, double cx,
                                                              double cy, double cz, double* __restrict__ part) {
  const ExtentItem it = items[blockIdx.x];
  double mn[kDopDirs], mx[kDopDirs];
#pragma unroll
  for (int j = 0; j < kDopDirs; ++j) {
    mn[j] = 1e300;
    mx[j] = -1e300;
  }
  for (std::uint32_t t = it.t0 + threadIdx.x; t < it.t1; t += blockDim.x)
    for (int v = 0; v < 3; ++v) {
      const double* X = xyz + 3 * static_cast<std::size_t>(tri[3 * static_cast<std::size_t>(t) + v]);
      const double d0 = __dsub_rn(X[0], cx), d1 = __dsub_rn(X[1], cy), d2 = __dsub_rn(X[2], cz);
#pragma unroll
      for (int j = 0; j < kDopDirs; ++j) {
        const double pr = dop_proj_rn(j, d0, d1, d2);
        mn[j] = fmin(mn[j], pr);
        mx[j] = fmax(mx[j], pr);
      }
    }
  __shared__ double red[8][kExtQ];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kDopDirs; ++j) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[j] = fmin(mn[j], __shfl_xor_sync(kFull, mn[j], o));
      mx[j] = fmax(mx[j], __shfl_xor_sync(kFull, mx[j], o));
    }
    if (lane == 0) {
      red[wid][j] = mn[j];
      red[wid][kDopDirs + j] = mx[j];
    }
  }
  __syncthreads();
  if (threadIdx.x < kExtQ) {
    const int q = threadIdx.x;
    double r = red[0][q];
    for (int w = 1; w < static_cast<int>(blockDim.x) / 32; ++w) r = q < kDopDirs ? fmin(r, red[w][q]) : fmax(r, red[w][q]);
    part[static_cast<std::size_t>(blockIdx.x) * kExtQ + q] = r;
  }
}

// one block per compartment: ext[k][26] (fp64 min / max) and the fp32 slabs
// dop4[k] (kDopF4 float4, k_cull_mask's layout; empty compartment: every
// point outside)
static __global__ void k_extents_finalize(const double* __restrict__ part, const std::uint32_t* __restrict__ item_first,
                                          const std::uint32_t* __restrict__ comp_off, double* __restrict__ ext,
                                          float4* __restrict__ dop4) {
  const int k = blockIdx.x, q = threadIdx.x;
  __shared__ double r[kExtQ];
  if (q < kExtQ) {
    double v = q < kDopDirs ? 1e300 : -1e300;
    for (std::uint32_t i = item_first[k]; i < item_first[k + 1]; ++i) {
      const double p = part[static_cast<std::size_t>(i) * kExtQ + q];
      v = q < kDopDirs ? fmin(v, p) : fmax(v, p);
    }
    r[q] = v;
    ext[static_cast<std::size_t>(k) * kExtQ + q] = v;
  }
  __syncthreads();
  float* dst = reinterpret_cast<float*>(dop4 + static_cast<std::size_t>(k) * kDopF4);
  if (q < 4 * kDopF4) dst[q] = 0.0f;
  __syncthreads();
  if (q < kDopDirs) {
    if (comp_off[k + 1] == comp_off[k]) {
      dst[2 * q] = 1e30f;
      dst[2 * q + 1] = -1e30f;
    } else {
      const double lo = r[q], hi = r[kDopDirs + q];
      const double m = __dadd_rn(1e-3, __dmul_rn(1e-5, fmax(fabs(lo), fabs(hi))));
      dst[2 * q] = nextafterf(__double2float_rn(__dsub_rn(lo, m)), -INFINITY);
      dst[2 * q + 1] = nextafterf(__double2float_rn(__dadd_rn(hi, m)), INFINITY);
    }
  }
}

struct MortonFrame {
  double cx, cy, cz;     // centring offset
  double lx, ly, lz;     // Morton box corner (original frame)
  double span;
};

// key = compartment << 30 | centroid Morton code (compartments sort apart)
static __global__ void k_tri_morton(const double* __restrict__ xyz, const std::uint32_t* __restrict__ tri,
                                    const std::uint32_t* __restrict__ comp_off, int K, std::uint32_t nt,
                                    const MortonFrame f, unsigned long long* __restrict__ keys,
                                    std::uint32_t* __restrict__ vals) {
  for (std::uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < K && t >= comp_off[k + 1]) ++k;
    const double c[3] = {f.cx, f.cy, f.cz}, l[3] = {f.lx, f.ly, f.lz};
    double m[3] = {0.0, 0.0, 0.0};
    for (int v = 0; v < 3; ++v) {
      const double* X = xyz + 3 * static_cast<std::size_t>(tri[3 * static_cast<std::size_t>(t) + v]);
      for (int a = 0; a < 3; ++a) m[a] = __dadd_rn(m[a], __ddiv_rn(__dsub_rn(X[a], c[a]), 3.0));
    }
    std::uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
      const double u = __dmul_rn(__ddiv_rn(__dsub_rn(__dadd_rn(m[a], c[a]), l[a]), f.span), 1024.0);
      q[a] = static_cast<std::uint32_t>(u < 0.0 ? 0.0 : (u > 1023.0 ? 1023.0 : u));
    }
    keys[t] = (static_cast<unsigned long long>(k) << 30) | spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
    vals[t] = t;
  }
}

// bounding sphere radius of k_cell_certify's pre-filters, from the vertex
// distances to the fp32 centre fc
__device__ __forceinline__ float sphere_radius(double rho, const float fc[3]) {
  const float sa = (fabsf(fc[0]) + fabsf(fc[1])) + fabsf(fc[2]);  // fp32 sum, as the host restatement
  const double rel = __dmul_rn(4e-6, static_cast<double>(sa));
  return nextafterf(__double2float_rn(__dadd_rn(__dadd_rn(__dmul_rn(rho, 1.0 + 1e-6), 1e-5), rel)), INFINITY);
}

// one warp per cluster q: ctri / tsph slots (pads: 0xffffffff / w = -1e30)
// and the cluster sphere
static __global__ void k_cluster_spheres(const double* __restrict__ xyz, const std::uint32_t* __restrict__ tri,
                                         const std::uint32_t* __restrict__ comp_off,
                                         const std::uint32_t* __restrict__ coff, int K, std::uint32_t nclus,
                                         double cx, double cy, double cz, const std::uint32_t* __restrict__ sorted,
                                         float4* __restrict__ clus, std::uint32_t* __restrict__ ctri,
                                         float4* __restrict__ tsph) {
  const std::uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (q >= nclus) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  int k = 0;
  while (k + 1 < K && q >= coff[k + 1]) ++k;
  const std::uint32_t i = (q - coff[k]) * kCluster + lane;
  const bool real = comp_off[k] + i < comp_off[k + 1];
  const double c[3] = {cx, cy, cz};
  double x[3][3];
  double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
  std::uint32_t t = 0xffffffffu;
  if (real) {
    t = sorted[comp_off[k] + i];
    for (int v = 0; v < 3; ++v) {
      const double* X = xyz + 3 * static_cast<std::size_t>(tri[3 * static_cast<std::size_t>(t) + v]);
      for (int a = 0; a < 3; ++a) {
        x[v][a] = __dsub_rn(X[a], c[a]);
        blo[a] = fmin(blo[a], x[v][a]);
        bhi[a] = fmax(bhi[a], x[v][a]);
      }
    }
  }
  // the triangle's own sphere
  auto rho_of = [&](const float fc[3]) {
    double rho = 0.0;
    for (int v = 0; v < 3; ++v) {
      double d2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const double d = __dsub_rn(x[v][a], static_cast<double>(fc[a]));
        d2 = __dadd_rn(d2, __dmul_rn(d, d));
      }
      rho = fmax(rho, __dsqrt_rn(d2));
    }
    return rho;
  };
  const std::size_t slot = static_cast<std::size_t>(q) * kCluster + lane;
  if (real) {
    const float fc[3] = {__double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[0], bhi[0]))),
                         __double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[1], bhi[1]))),
                         __double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[2], bhi[2])))};
    tsph[slot] = make_float4(fc[0], fc[1], fc[2], sphere_radius(rho_of(fc), fc));
  } else {
    tsph[slot] = make_float4(0.f, 0.f, 0.f, -1e30f);
  }
  ctri[slot] = t;
  // the cluster's sphere: box of all its vertices (warp min / max), then the
  // farthest vertex from the fp32 centre
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      blo[a] = fmin(blo[a], __shfl_xor_sync(kFull, blo[a], o));
      bhi[a] = fmax(bhi[a], __shfl_xor_sync(kFull, bhi[a], o));
    }
  const float fc[3] = {__double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[0], bhi[0]))),
                       __double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[1], bhi[1]))),
                       __double2float_rn(__dmul_rn(0.5, __dadd_rn(blo[2], bhi[2])))};
  double rho = real ? rho_of(fc) : 0.0;
  for (int o = 16; o > 0; o >>= 1) rho = fmax(rho, __shfl_xor_sync(kFull, rho, o));
  if (lane == 0) clus[q] = make_float4(fc[0], fc[1], fc[2], sphere_radius(rho, fc));
}

// one warp per supercluster g (32 consecutive clusters of one compartment):
// a sphere containing every cluster sphere (fp32 centre of the box of the
// cluster balls, radius from it in fp64, rounded up)
static __global__ void k_super_spheres(const float4* __restrict__ clus, const std::uint32_t* __restrict__ coff,
                                       const std::uint32_t* __restrict__ soff, int K, std::uint32_t nsup,
                                       float4* __restrict__ sup) {
  const std::uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (g >= nsup) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  int k = 0;
  while (k + 1 < K && g >= soff[k + 1]) ++k;
  const std::uint32_t q = coff[k] + (g - soff[k]) * 32 + lane;
  const bool real = q < coff[k + 1];
  float4 s = real ? clus[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  if (real) {
    const double c[3] = {s.x, s.y, s.z};
    for (int a = 0; a < 3; ++a) {
      lo[a] = c[a] - s.w;
      hi[a] = c[a] + s.w;
    }
  }
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(kFull, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(kFull, hi[a], o));
    }
  const float fc[3] = {static_cast<float>(0.5 * (lo[0] + hi[0])), static_cast<float>(0.5 * (lo[1] + hi[1])),
                       static_cast<float>(0.5 * (lo[2] + hi[2]))};
  double r = 0.0;
  if (real) {
    const double dx = double(s.x) - fc[0], dy = double(s.y) - fc[1], dz = double(s.z) - fc[2];
    r = sqrt(dx * dx + dy * dy + dz * dz) + s.w;
  }
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(kFull, r, o));
  if (lane == 0) sup[g] = make_float4(fc[0], fc[1], fc[2], nextafterf(static_cast<float>(r * (1.0 + 1e-6) + 1e-5), INFINITY));
}

}  // namespace nm
