// Exact certified-cell culling (nm_options.cull_outside = 2).
//
// The winding number of a closed surface (SPEC.md:227 closedness) is an
// integer that is constant on every connected set the surface does not meet.
// Per compartment a uniform grid of cubic cells (built once per surface set,
// from the surface alone) is classified:
//   * k_cell_certify: a cell is CERTIFIED when its circumscribed ball (centre,
//     radius B sqrt(3)/2 + margin) meets none of the compartment's triangles —
//     cluster-sphere rejection in fp32 with a 1e-3 mm margin, then the exact
//     fp64 point-triangle distance (distance.cuh) for the clusters that are
//     not rejected;
//   * every uncertified cell is split into 4^3 children, certified the same
//     way (k_child_certify), so the unresolved shell around a surface is ~4x
//     thinner;
//   * the host gives every maximal x-run of certified cells one winding
//     number: adjacent cells' balls overlap, so a run's union is connected
//     and surface-free. A run with an end cell whose centre lies outside the
//     compartment's 13-DOP (hence outside the convex hull: w = 0 exactly) is
//     0; any other run gets w = round(s) at one representative cell centre,
//     evaluated by k_label (sparse mode) — accepted only when s is within
//     1e-3 of 0 or 1, otherwise the run stays uncertified. A run of children
//     that reaches the end of its run of uncertified parents continues into
//     the certified neighbour parent (the child's ball overlaps the parent's:
//     centre distance <= 0.82 B < 0.866 B + 0.217 B) and takes its number.
// k_cell_classify then gives each point, per compartment, either a known
// bit (13-DOP outside, or inside a certified cell: s = w exactly) or leaves
// the pair to the sparse k_label pass. A point's result depends only on its
// own position and the surfaces (the grid is a function of the surfaces), so
// results stay independent of the point set and of sharding.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nm {

constexpr int kCluster = 32;  // triangles per certification cluster (Morton order)

struct CellGrid {
  double ox, oy, oz, B;  // origin of cell (0,0,0) in the centred frame, cell edge (mm)
  int nx, ny, nz;
  std::uint32_t off;     // first cell of this compartment in the state array
  double invB;           // 1 / B: point -> cell lookups multiply (an index one off at a face is
                         // harmless: the neighbour's certified ball covers the shared face)
};

// ball radius of a cube of edge B (covers the closed cube, with margin)
__host__ __device__ inline double cell_ball(double B) { return B * 0.8660254037844387 * (1.0 + 1e-9) + 1e-6; }

constexpr int kSubCells = 4;
constexpr int kChildren = kSubCells * kSubCells * kSubCells;

// Warp-cooperative certification of a BRICK of 4 x 4 x 2 cubes of edge e
// (corner O, centred frame), one cube per lane: the lanes first test 32
// clusters at a time against the brick's ball (which contains every lane's
// cube ball), then each lane tests the surviving clusters against its own
// ball (ball_hits_surface's tests). Returns this lane's "ball meets the
// surface"; inactive lanes return true.
static __device__ bool warp_certify(double Ox, double Oy, double Oz, double e, bool active, const float4* __restrict__ clus,
                             int nclus, const std::uint32_t* __restrict__ clus_tri, const float4* __restrict__ tsph,
                             const double* __restrict__ xyz, const std::uint32_t* __restrict__ tri, double cx,
                             double cy, double cz) {
  const int lane = threadIdx.x & 31;
  const double Cx = Ox + (lane % 4 + 0.5) * e, Cy = Oy + ((lane / 4) % 4 + 0.5) * e, Cz = Oz + (lane / 16 + 0.5) * e;
  const double rb = cell_ball(e);
  // brick ball: centre O + (2, 2, 1) e; radius = farthest cube centre + rb
  const float bx = static_cast<float>(Ox + 2.0 * e), by = static_cast<float>(Oy + 2.0 * e), bz = static_cast<float>(Oz + e);
  const float fbr = static_cast<float>(e * 2.1794494717703369 + rb) + 1e-3f + 4e-6f * (fabsf(bx) + fabsf(by) + fabsf(bz));
  const float fx = static_cast<float>(Cx), fy = static_cast<float>(Cy), fz = static_cast<float>(Cz);
  const float frb = static_cast<float>(rb) + 1e-3f + 4e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
  bool hit = !active;
  for (int q0 = 0; q0 < nclus; q0 += 32) {
    bool cand = false;
    if (q0 + lane < nclus) {
      const float4 s = __ldg(clus + q0 + lane);
      const float dx = bx - s.x, dy = by - s.y, dz = bz - s.z;
      const float R = fbr + s.w;
      cand = dx * dx + dy * dy + dz * dz <= R * R;
    }
    unsigned bal = __ballot_sync(kFull, cand);
    while (bal) {
      const int q = q0 + __ffs(bal) - 1;
      bal &= bal - 1;
      if (hit) continue;
      const float4 s = __ldg(clus + q);
      const float dx = fx - s.x, dy = fy - s.y, dz = fz - s.z;
      const float R = frb + s.w;
      if (dx * dx + dy * dy + dz * dz > R * R) continue;
      const V3t<double> p{Cx + cx, Cy + cy, Cz + cz};
      for (int t = 0; t < kCluster && !hit; ++t) {
        const std::uint32_t tid = __ldg(clus_tri + static_cast<std::size_t>(q) * kCluster + t);
        if (tid == 0xffffffffu) break;
        // triangle's own bounding sphere first (fp32, same margins)
        const float4 ts = __ldg(tsph + static_cast<std::size_t>(q) * kCluster + t);
        const float tx = fx - ts.x, ty = fy - ts.y, tz = fz - ts.z;
        const float TR = frb + ts.w;
        if (tx * tx + ty * ty + tz * tz > TR * TR) continue;
        const std::uint32_t* ev = tri + 3 * static_cast<std::size_t>(tid);
        const double* A = xyz + 3 * static_cast<std::size_t>(ev[0]);
        const double* Bv = xyz + 3 * static_cast<std::size_t>(ev[1]);
        const double* Cv = xyz + 3 * static_cast<std::size_t>(ev[2]);
        const double d2 = point_tri_dist2<double>(p, {A[0], A[1], A[2]}, {Bv[0], Bv[1], Bv[2]}, {Cv[0], Cv[1], Cv[2]});
        hit = !(d2 > rb * rb);  // NaN (degenerate) counts as a hit
      }
    }
    if (__all_sync(kFull, hit)) break;
  }
  return hit;
}

// Level 1: one warp per 4 x 4 x 2 brick of cells of one compartment;
// cert = 1 when no triangle of the compartment meets the cell's ball.
static __global__ void __launch_bounds__(256) k_cell_certify(const CellGrid g, const float4* __restrict__ clus, int nclus,
                                                      const std::uint32_t* __restrict__ clus_tri,
                                                      const float4* __restrict__ tsph, const double* __restrict__ xyz,
                                                      const std::uint32_t* __restrict__ tri, double cx, double cy,
                                                      double cz, std::uint8_t* __restrict__ cert) {
  const int bx = (g.nx + 3) / 4, by = (g.ny + 3) / 4, bz = (g.nz + 1) / 2;
  const std::size_t w = (blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x) / 32;
  if (w >= static_cast<std::size_t>(bx) * by * bz) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int i0 = static_cast<int>(w % bx) * 4, j0 = static_cast<int>((w / bx) % by) * 4,
            k0 = static_cast<int>(w / (static_cast<std::size_t>(bx) * by)) * 2;
  const int ix = i0 + lane % 4, iy = j0 + (lane / 4) % 4, iz = k0 + lane / 16;
  const bool active = ix < g.nx && iy < g.ny && iz < g.nz;
  const bool hit = warp_certify(g.ox + i0 * g.B, g.oy + j0 * g.B, g.oz + k0 * g.B, g.B, active, clus, nclus, clus_tri,
                                tsph, xyz, tri, cx, cy, cz);
  if (active) cert[g.off + (static_cast<std::size_t>(iz) * g.ny + iy) * g.nx + ix] = hit ? 0 : 1;
}

// Level 2: the kSubCells^3 children (edge B / kSubCells) of every
// uncertified level-1 cell, one warp per half (4 x 4 x 2 children). cells[b]
// = level-1 cell (local index) of child block b; out[b * kChildren + child]
// = 1 when certified, child = (sz * 4 + sy) * 4 + sx.
static __global__ void __launch_bounds__(256) k_child_certify(const CellGrid g, const std::uint32_t* __restrict__ cells,
                                                       std::size_t nblocks, const float4* __restrict__ clus, int nclus,
                                                       const std::uint32_t* __restrict__ clus_tri,
                                                       const float4* __restrict__ tsph, const double* __restrict__ xyz,
                                                       const std::uint32_t* __restrict__ tri, double cx, double cy,
                                                       double cz, std::uint8_t* __restrict__ out) {
  static_assert(kSubCells == 4, "one warp = 4 x 4 x 2 children");
  const std::size_t w = (blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x) / 32;
  if (w >= 2 * nblocks) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const std::uint32_t cell = cells[w / 2];
  const int half = static_cast<int>(w % 2);
  const int ix = static_cast<int>(cell % g.nx);
  const int iy = static_cast<int>((cell / g.nx) % g.ny);
  const int iz = static_cast<int>(cell / (static_cast<std::uint32_t>(g.nx) * g.ny));
  const double b = g.B / kSubCells;
  const bool hit = warp_certify(g.ox + ix * g.B, g.oy + iy * g.B, g.oz + iz * g.B + 2 * half * b, b, true, clus, nclus,
                                clus_tri, tsph, xyz, tri, cx, cy, cz);
  out[(w / 2) * kChildren + (2 * half + lane / 16) * 16 + lane % 16] = hit ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Round-2 certification (the device build; the host-run path above keeps the
// per-lane kernels, and tests compare the two builds bit for bit). Same
// decision per cube as warp_certify: "some triangle of the compartment has
// exact fp64 distance <= rb from the cube centre". Only the conservative
// fp32 pre-filters are organised differently:
//   * per candidate cluster, lane t holds triangle t's sphere and tests it
//     against all 32 cube balls of the warp at once (the cube centres lie on
//     a 4 x 4 x 2 lattice: 4 + 4 + 2 squared offsets, 32 sums), with the
//     largest lane margin — a superset of each lane's own candidates;
//   * one ballot per needing cube transposes the masks, and each cube runs
//     the exact test on its own candidate triangles.
// This replaces 32 dependent per-lane loads + tests per cluster with one
// coalesced load and a 5-stage shuffle transpose; the compartments' grids go
// in ONE launch.
// ---------------------------------------------------------------------------
struct CertifyParams {
  const CellGrid* grids;        // K
  int K;
  const unsigned long long* first;  // K + 1: first work warp of each compartment
  const std::uint32_t* coff;    // K + 1: first cluster of each compartment
  const std::uint32_t* soff;    // K + 1: first supercluster (32 clusters) of each compartment
  const float4* sup;            // supercluster spheres
  const float4* clus;           // cluster spheres (all compartments)
  const std::uint32_t* clus_tri;
  const float4* tsph;
  const double* xyz;
  const std::uint32_t* tri;
  double cx, cy, cz;
  const std::uint32_t* cells;   // level 2: global child block -> compartment-local level-1 cell
  std::uint8_t* out;            // level 1: cert flags by global cell; level 2: child flags
  unsigned long long warps;     // total work warps
};

static __device__ bool warp_certify_coop(double Ox, double Oy, double Oz, double e, bool active,
                                         const CertifyParams& p, int k) {
  const std::uint32_t c0 = p.coff[k];
  const int nclus = static_cast<int>(p.coff[k + 1] - c0);
  const float4* sup = p.sup + p.soff[k];
  const int nsup = static_cast<int>(p.soff[k + 1] - p.soff[k]);
  const int lane = threadIdx.x & 31;
  const double Cx = Ox + (lane % 4 + 0.5) * e, Cy = Oy + ((lane / 4) % 4 + 0.5) * e, Cz = Oz + (lane / 16 + 0.5) * e;
  const double rb = cell_ball(e);
  const float bx = static_cast<float>(Ox + 2.0 * e), by = static_cast<float>(Oy + 2.0 * e), bz = static_cast<float>(Oz + e);
  const float fbr = static_cast<float>(e * 2.1794494717703369 + rb) + 1e-3f + 4e-6f * (fabsf(bx) + fabsf(by) + fabsf(bz));
  const float fx = static_cast<float>(Cx), fy = static_cast<float>(Cy), fz = static_cast<float>(Cz);
  const float frb = static_cast<float>(rb) + 1e-3f + 4e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
  // the warp's cube lattice (the lanes' own fp32 centres) and the largest margin
  float X[4], Y[4], Z[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X[i] = __shfl_sync(kFull, fx, i);
    Y[i] = __shfl_sync(kFull, fy, 4 * i);
  }
  Z[0] = __shfl_sync(kFull, fz, 0);
  Z[1] = __shfl_sync(kFull, fz, 16);
  float frbm = frb;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) frbm = fmaxf(frbm, __shfl_xor_sync(kFull, frbm, o));
  const float4* clus = p.clus + c0;
  const std::uint32_t* ctri = p.clus_tri + static_cast<std::size_t>(c0) * kCluster;
  const float4* tsph = p.tsph + static_cast<std::size_t>(c0) * kCluster;
  const V3t<double> pt{Cx + p.cx, Cy + p.cy, Cz + p.cz};
  bool hit = !active;
  // superclusters (32 clusters) meeting the brick's ball, then their clusters
  for (int g0 = 0; g0 < nsup; g0 += 32) {
    bool scand = false;
    if (g0 + lane < nsup) {
      const float4 s = __ldg(sup + g0 + lane);
      const float dx = bx - s.x, dy = by - s.y, dz = bz - s.z;
      const float R = fbr + s.w;
      scand = dx * dx + dy * dy + dz * dz <= R * R;
    }
    unsigned sbal = __ballot_sync(kFull, scand);
    while (sbal) {
      const int q0 = (g0 + __ffs(sbal) - 1) * 32;
      sbal &= sbal - 1;
      bool cand = false;
      if (q0 + lane < nclus) {
        const float4 s = __ldg(clus + q0 + lane);
        const float dx = bx - s.x, dy = by - s.y, dz = bz - s.z;
        const float R = fbr + s.w;
        cand = dx * dx + dy * dy + dz * dz <= R * R;
      }
      unsigned bal = __ballot_sync(kFull, cand);
      while (bal) {
        const int q = q0 + __ffs(bal) - 1;
        bal &= bal - 1;
        // cubes (lanes) still open whose ball meets the cluster sphere
        bool need = false;
        if (!hit) {
          const float4 s = __ldg(clus + q);
          const float dx = fx - s.x, dy = fy - s.y, dz = fz - s.z;
          const float R = frb + s.w;
          need = dx * dx + dy * dy + dz * dz <= R * R;
        }
        unsigned needm = __ballot_sync(kFull, need);
        if (!needm) continue;
        // lane t: which cubes' balls meet triangle t's sphere (pads: w < 0)
        const float4 ts = __ldg(tsph + static_cast<std::size_t>(q) * kCluster + lane);
        unsigned m = 0;
        if (ts.w >= 0.0f) {
          const float R = frbm + ts.w, R2 = R * R;
          float dx2[4], dy2[4], dz2[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float dx = X[i] - ts.x, dy = Y[i] - ts.y;
            dx2[i] = dx * dx;
            dy2[i] = dy * dy;
          }
          dz2[0] = (Z[0] - ts.z) * (Z[0] - ts.z);
          dz2[1] = (Z[1] - ts.z) * (Z[1] - ts.z);
#pragma unroll
          for (int kz = 0; kz < 2; ++kz)
#pragma unroll
            for (int jy = 0; jy < 4; ++jy) {
              const float yz = dy2[jy] + dz2[kz];
#pragma unroll
              for (int ix = 0; ix < 4; ++ix) m |= (yz + dx2[ix] <= R2 ? 1u : 0u) << (ix + 4 * jy + 16 * kz);
            }
        }
        m &= needm;
        // transpose the 32 x 32 bit matrix (row t = triangle t's cube mask) so
        // that lane L holds cube L's candidate triangles: five block-swap stages
        unsigned mine = m;
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
          const unsigned M = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu : j == 2 ? 0x33333333u : 0x55555555u;
          const unsigned o = __shfl_xor_sync(kFull, mine, j);
          mine = (lane & j) ? ((mine & ~M) | ((o >> j) & M)) : ((mine & M) | ((o & M) << j));
        }
        while (mine && !hit) {
          const int t = __ffs(mine) - 1;
          mine &= mine - 1;
          const std::uint32_t tid = __ldg(ctri + static_cast<std::size_t>(q) * kCluster + t);
          const std::uint32_t* ev = p.tri + 3 * static_cast<std::size_t>(tid);
          const double* A = p.xyz + 3 * static_cast<std::size_t>(ev[0]);
          const double* Bv = p.xyz + 3 * static_cast<std::size_t>(ev[1]);
          const double* Cv = p.xyz + 3 * static_cast<std::size_t>(ev[2]);
          const double d2 = point_tri_dist2<double>(pt, {A[0], A[1], A[2]}, {Bv[0], Bv[1], Bv[2]}, {Cv[0], Cv[1], Cv[2]});
          hit = !(d2 > rb * rb);  // NaN (degenerate) counts as a hit
        }
      }
      if (__all_sync(kFull, hit)) return hit;
    }
  }
  return hit;
}

__device__ __forceinline__ int work_compartment(const CertifyParams& p, unsigned long long w) {
  int k = 0;
  while (k + 1 < p.K && w >= p.first[k + 1]) ++k;
  return k;
}

// 4 CTAs per SM: without a bound the certification kernels took 132-133
// registers, one 256-thread CTA per SM (set_surfaces at cfg5 37.5 -> ~30 ms,
// cfg3 40.7 -> 26.5 ms: profiles/r02/launch_bounds_ab.txt)
#ifndef NM_CERT_MIN_BLOCKS
#define NM_CERT_MIN_BLOCKS 4
#endif
// level 1, all compartments: one warp per 4 x 4 x 2 brick (first[] = brick prefix)
static __global__ void __launch_bounds__(256, NM_CERT_MIN_BLOCKS) k_cell_certify_all(const CertifyParams p) {
  const unsigned long long w = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) / 32;
  if (w >= p.warps) return;  // warp-uniform
  const int k = work_compartment(p, w);
  const CellGrid g = p.grids[k];
  const int lane = threadIdx.x & 31;
  const unsigned long long lw = w - p.first[k];
  const int bx = (g.nx + 3) / 4, by = (g.ny + 3) / 4;
  const int i0 = static_cast<int>(lw % bx) * 4, j0 = static_cast<int>((lw / bx) % by) * 4,
            k0 = static_cast<int>(lw / (static_cast<unsigned long long>(bx) * by)) * 2;
  const int ix = i0 + lane % 4, iy = j0 + (lane / 4) % 4, iz = k0 + lane / 16;
  const bool active = ix < g.nx && iy < g.ny && iz < g.nz;
  const bool hit = warp_certify_coop(g.ox + i0 * g.B, g.oy + j0 * g.B, g.oz + k0 * g.B, g.B, active, p, k);
  if (active) p.out[g.off + (static_cast<std::size_t>(iz) * g.ny + iy) * g.nx + ix] = hit ? 0 : 1;
}

// level 2, all compartments: one warp per half child block (first[] = 2 x block prefix)
static __global__ void __launch_bounds__(256, NM_CERT_MIN_BLOCKS) k_child_certify_all(const CertifyParams p) {
  const unsigned long long w = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) / 32;
  if (w >= p.warps) return;  // warp-uniform
  const int k = work_compartment(p, w);
  const CellGrid g = p.grids[k];
  const int lane = threadIdx.x & 31;
  const unsigned long long b = w / 2;  // global child block
  const std::uint32_t cell = p.cells[b];
  const int half = static_cast<int>(w % 2);
  const int ix = static_cast<int>(cell % g.nx);
  const int iy = static_cast<int>((cell / g.nx) % g.ny);
  const int iz = static_cast<int>(cell / (static_cast<std::uint32_t>(g.nx) * g.ny));
  const double e = g.B / kSubCells;
  const bool hit = warp_certify_coop(g.ox + ix * g.B, g.oy + iy * g.B, g.oz + iz * g.B + 2 * half * e, e, true, p, k);
  p.out[b * kChildren + (2 * half + lane / 16) * 16 + lane % 16] = hit ? 0 : 1;
}

// Per evaluation position i (point order[i]): unk bit c = pair (point, c)
// still to be evaluated; ins bit c = known inside (certified w = 1). The
// point's masks / flagmask / s entries of the known pairs are written here;
// the sparse k_label ORs the evaluated bits in.
struct ClassifyParams {
  const double* pts;
  std::size_t n;
  const std::uint32_t* order;
  double cx, cy, cz;
  const float4* dop4;  // 13-DOP slabs per compartment (k_cull_mask); nullptr: no outside culling
  const CellGrid* grids;  // nullptr: no certified cells
  const std::uint32_t* code;  // per level-1 cell: 0 unknown, 1 certified w = 0, 2 certified w = 1,
                              // 3 + b: uncertified, children in child block b
  const std::uint8_t* child;  // per child: 0 unknown, 1 w = 0, 2 w = 1
  int K;
  bool preset;  // write the known inside bits into masks (false: masks = 0; sharded passes, shard > 0)
  std::uint32_t* unk;
  std::uint32_t* masks;     // by point id
  std::uint32_t* flagmask;  // by evaluation position
  double* s_out;
};

static __global__ void k_cell_classify(const ClassifyParams prm) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < prm.n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t j = prm.order ? prm.order[i] : i;
    const double x = prm.pts[3 * j] - prm.cx, y = prm.pts[3 * j + 1] - prm.cy, z = prm.pts[3 * j + 2] - prm.cz;
    const float xf = static_cast<float>(x), yf = static_cast<float>(y), zf = static_cast<float>(z);
    std::uint32_t unk = 0, ins = 0;
    for (int c = 0; c < prm.K; ++c) {
      if (prm.dop4) {
        const float* dop = reinterpret_cast<const float*>(prm.dop4 + static_cast<std::size_t>(c) * kDopF4);
        bool o = false;
#pragma unroll
        for (int d = 0; d < kDopDirs; ++d) {
          const float pr = dop_dir(d, 0) * xf + dop_dir(d, 1) * yf + dop_dir(d, 2) * zf;
          o |= pr < __ldg(dop + 2 * d) || pr > __ldg(dop + 2 * d + 1);
        }
        if (o) continue;  // outside the convex hull: w = 0
      }
      if (!prm.grids) {
        unk |= 1u << c;
        continue;
      }
      const CellGrid g = prm.grids[c];
      const double u = (x - g.ox) * g.invB, v = (y - g.oy) * g.invB, w = (z - g.oz) * g.invB;
      std::uint32_t st = 0;
      if (u >= 0.0 && v >= 0.0 && w >= 0.0 && u < g.nx && v < g.ny && w < g.nz) {
        const int iu = static_cast<int>(u), iv = static_cast<int>(v), iw = static_cast<int>(w);
        const std::size_t cell = (static_cast<std::size_t>(iw) * g.ny + iv) * g.nx + iu;
        st = __ldg(prm.code + g.off + cell);
        if (st >= 3) {  // child cube containing the point (fractional position, fp64)
          const int a = min(static_cast<int>((u - iu) * kSubCells), kSubCells - 1);
          const int b = min(static_cast<int>((v - iv) * kSubCells), kSubCells - 1);
          const int d = min(static_cast<int>((w - iw) * kSubCells), kSubCells - 1);
          st = __ldg(prm.child + static_cast<std::size_t>(st - 3) * kChildren + (d * kSubCells + b) * kSubCells + a);
        }
      }
      if (st == 2) ins |= 1u << c;
      else if (st != 1) unk |= 1u << c;
    }
    prm.unk[i] = unk;
    prm.masks[j] = prm.preset ? ins : 0u;
    prm.flagmask[i] = 0u;  // flags are indexed by evaluation position
    if (prm.s_out)
      for (int c = 0; c < prm.K; ++c)
        if (!((unk >> c) & 1u)) prm.s_out[j * prm.K + c] = ((ins >> c) & 1u) ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Pairs left unknown by k_cell_classify (points in uncertified children),
// resolved exactly where a surface-free ball joins them to a certified
// neighbour (round 2): for the neighbour children within kResolveReach of
// the point's child (or their certified parents) with a known w,
// gap = |p - c_n| - r_n, where
// B(c_n, r_n) is the neighbour's certified ball (shrunk by a 1e-9 relative +
// 1e-9 mm margin). If the best gap < 0, p lies in that ball. Otherwise the
// pair is resolved when B(p, rho), rho just above the gap, meets no triangle
// of the compartment (the certification test with one ball per lane: warp
// ball, then superclusters, clusters, triangle spheres in fp32 with margins,
// then the exact fp64 distance > rho (1 + 1e-9)). Both balls are open,
// surface-free and overlap, so p and c_n are joined in the complement of
// the surface: w(p) = w_n exactly. Resolved pairs get their bit (when the
// caller writes known bits) and s = w, and leave the pair lists.
// ---------------------------------------------------------------------------
struct PendPair {
  std::uint32_t i, j, k, w;  // evaluation position, point id, compartment, the neighbour's w
  double p[3];               // point (centred frame)
  double t[4];               // the neighbour's certified ball: centre, radius
};

struct ResolveParams {
  const double* pts;
  const std::uint32_t* order;
  double cx, cy, cz;
  const CellGrid* grids;
  const std::uint32_t* code;
  const std::uint8_t* child;
  int K;
  const std::uint32_t* list;           // packed per-compartment lists of evaluation positions
  std::uint32_t off[33], cnt[32];      // compartment k: list[off[k] .. off[k] + cnt[k])
  std::uint32_t wfirst[33];            // first warp of compartment k
  struct PendPair* pend;               // pairs for k_pair_chain (appended)
  unsigned* npend;
  std::uint32_t* unk;                  // per position: unknown compartment bits (cleared when resolved)
  std::uint32_t* masks;                // by point id
  double* s_out;
  int write_known;
  CertifyParams cl;                    // clusters / superclusters / triangles (coff, soff, sup, clus, clus_tri, tsph, xyz, tri)
};

__device__ __forceinline__ int floor_div4(int x) { return x >= 0 ? x / 4 : -((-x + 3) / 4); }

// Exact distance from q (centred frame, the same q in every lane) to the
// nearest triangle of one compartment, or cap when none is closer; the whole
// warp works on the one query: 32 superclusters, then a candidate's 32
// clusters, then a cluster's 32 triangle spheres per step, pruned in fp32
// with the certification margins against the shrinking bound; each lane
// takes the exact fp64 distance of its candidate triangle, warp minimum.
static __device__ double warp_nearest_dist(double qx, double qy, double qz, double cap, double cx, double cy, double cz,
                                           const float4* __restrict__ sup, int nsup, const float4* __restrict__ clus,
                                           int nclus, const std::uint32_t* __restrict__ ctri,
                                           const float4* __restrict__ tsph, const double* __restrict__ xyz,
                                           const std::uint32_t* __restrict__ tri) {
  const int lane = threadIdx.x & 31;
  const float fx = static_cast<float>(qx), fy = static_cast<float>(qy), fz = static_cast<float>(qz);
  const float marg = 1e-3f + 4e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
  const V3t<double> pt{qx + cx, qy + cy, qz + cz};
  double best = cap;  // warp-uniform
  auto near = [&](const float4& s4) {
    const float dx = fx - s4.x, dy = fy - s4.y, dz = fz - s4.z;
    const float R = static_cast<float>(best) + marg + s4.w;
    return dx * dx + dy * dy + dz * dz <= R * R;
  };
  for (int g0 = 0; g0 < nsup; g0 += 32) {
    unsigned sb = __ballot_sync(kFull, g0 + lane < nsup && near(__ldg(sup + g0 + lane)));
    while (sb) {
      const int g = g0 + __ffs(sb) - 1;
      sb &= sb - 1;
      const int q = g * 32 + lane;
      unsigned cb = __ballot_sync(kFull, q < nclus && near(__ldg(clus + q)));
      while (cb) {
        const int qc = g * 32 + __ffs(cb) - 1;
        cb &= cb - 1;
        const float4 ts = __ldg(tsph + static_cast<std::size_t>(qc) * kCluster + lane);
        double d = 1e300;
        if (ts.w >= 0.0f && near(ts)) {
          const std::uint32_t tid = __ldg(ctri + static_cast<std::size_t>(qc) * kCluster + lane);
          const std::uint32_t* ev = tri + 3 * static_cast<std::size_t>(tid);
          const double* A = xyz + 3 * static_cast<std::size_t>(ev[0]);
          const double* Bv = xyz + 3 * static_cast<std::size_t>(ev[1]);
          const double* Cv = xyz + 3 * static_cast<std::size_t>(ev[2]);
          const double d2 = point_tri_dist2<double>(pt, {A[0], A[1], A[2]}, {Bv[0], Bv[1], Bv[2]}, {Cv[0], Cv[1], Cv[2]});
          d = d2 >= 0.0 ? sqrt(d2) : 0.0;  // NaN (degenerate triangle): no ball
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d = fmin(d, __shfl_xor_sync(kFull, d, o));
        best = fmin(best, d);
      }
    }
  }
  return best;
}

// balls per chain (k_pair_chain; profiles/r02/trace_ab_coop.txt)
#ifndef NM_TRACE_STEPS
#define NM_TRACE_STEPS 12
#endif
constexpr int kTraceSteps = NM_TRACE_STEPS;
#ifndef NM_TRACE_STEP
#define NM_TRACE_STEP 0.99
#endif
constexpr double kTraceStep = NM_TRACE_STEP;  // next centre at this fraction of the radius (< 1: inside the ball)

#ifndef NM_RESOLVE_REACH
#define NM_RESOLVE_REACH 1
#endif
constexpr int kResolveReach = NM_RESOLVE_REACH;  // neighbour children searched: (2 reach + 1)^3 - 1
#ifndef NM_RESOLVE_MAXGAP
#define NM_RESOLVE_MAXGAP 1.0
#endif
constexpr double kResolveMaxGap = NM_RESOLVE_MAXGAP;  // ball chains only for gaps below this many child edges

static __global__ void __launch_bounds__(256) k_pair_resolve(const ResolveParams prm) {
  const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (w >= prm.wfirst[prm.K]) return;  // warp-uniform
  int k = 0;
  while (k + 1 < prm.K && w >= prm.wfirst[k + 1]) ++k;
  const int lane = threadIdx.x & 31;
  const std::uint32_t e = (w - prm.wfirst[k]) * 32 + lane;
  const bool active = e < prm.cnt[k];
  const CellGrid g = prm.grids[k];
  std::uint32_t i = 0, j = 0;
  double x = 0.0, y = 0.0, z = 0.0;
  if (active) {
    i = prm.list[prm.off[k] + e];
    j = prm.order ? prm.order[i] : i;
    x = prm.pts[3 * static_cast<std::size_t>(j)] - prm.cx;
    y = prm.pts[3 * static_cast<std::size_t>(j) + 1] - prm.cy;
    z = prm.pts[3 * static_cast<std::size_t>(j) + 2] - prm.cz;
  }
  // the point's child cell in the compartment's fine lattice (kSubCells per cell)
  const double b = g.B / kSubCells;
  const double rl1 = cell_ball(g.B) * (1.0 - 1e-9) - 1e-9, rch = cell_ball(b) * (1.0 - 1e-9) - 1e-9;
  double best = 1e300, tx = 0.0, ty = 0.0, tz = 0.0, tr = 0.0;  // best gap and its certified ball
  int wbest = -1;
  if (active) {
    const double u = (x - g.ox) * g.invB, v = (y - g.oy) * g.invB, ww = (z - g.oz) * g.invB;
    const int iu = static_cast<int>(u), iv = static_cast<int>(v), iw = static_cast<int>(ww);
    const int fx = iu * kSubCells + min(static_cast<int>((u - iu) * kSubCells), kSubCells - 1);
    const int fy = iv * kSubCells + min(static_cast<int>((v - iv) * kSubCells), kSubCells - 1);
    const int fz = iw * kSubCells + min(static_cast<int>((ww - iw) * kSubCells), kSubCells - 1);
    for (int dz = -kResolveReach; dz <= kResolveReach; ++dz)
      for (int dy = -kResolveReach; dy <= kResolveReach; ++dy)
        for (int dx = -kResolveReach; dx <= kResolveReach; ++dx) {
          if (!dx && !dy && !dz) continue;
          const int nx = fx + dx, ny = fy + dy, nz = fz + dz;
          const int px = floor_div4(nx), py = floor_div4(ny), pz = floor_div4(nz);
          if (px < 0 || py < 0 || pz < 0 || px >= g.nx || py >= g.ny || pz >= g.nz) continue;
          const std::uint32_t st = __ldg(prm.code + g.off + (static_cast<std::size_t>(pz) * g.ny + py) * g.nx + px);
          double ccx, ccy, ccz, r;
          int wn;
          if (st == 1u || st == 2u) {  // certified parent: its ball
            wn = static_cast<int>(st) - 1;
            ccx = g.ox + (px + 0.5) * g.B;
            ccy = g.oy + (py + 0.5) * g.B;
            ccz = g.oz + (pz + 0.5) * g.B;
            r = rl1;
          } else if (st >= 3u) {
            const int sx = nx - px * kSubCells, sy = ny - py * kSubCells, sz = nz - pz * kSubCells;
            const std::uint8_t cs =
                __ldg(prm.child + static_cast<std::size_t>(st - 3u) * kChildren + (sz * kSubCells + sy) * kSubCells + sx);
            if (cs != 1 && cs != 2) continue;
            wn = cs - 1;
            ccx = g.ox + px * g.B + (sx + 0.5) * b;
            ccy = g.oy + py * g.B + (sy + 0.5) * b;
            ccz = g.oz + pz * g.B + (sz + 0.5) * b;
            r = rch;
          } else {
            continue;
          }
          const double gx = x - ccx, gy = y - ccy, gz = z - ccz;
          const double gap = sqrt(gx * gx + gy * gy + gz * gz) - r;
          if (gap < best) {
            best = gap;
            wbest = wn;
            tx = ccx;
            ty = ccy;
            tz = ccz;
            tr = r;
          }
        }
  }
  const bool resolved = active && wbest >= 0 && best < -1e-9;
  // not inside: a chain of balls towards the best neighbour (k_pair_chain),
  // one record per pending pair
  const bool pending = active && wbest >= 0 && !resolved && best < kResolveMaxGap * b;
  if (pending) {
    const unsigned r = atomicAdd(prm.npend, 1u);
    PendPair& q = prm.pend[r];
    q.i = i;
    q.j = j;
    q.k = static_cast<std::uint32_t>(k);
    q.w = static_cast<std::uint32_t>(wbest);
    q.p[0] = x;
    q.p[1] = y;
    q.p[2] = z;
    q.t[0] = tx;
    q.t[1] = ty;
    q.t[2] = tz;
    q.t[3] = tr;
  }
  if (resolved) {
    atomicAnd(prm.unk + i, ~(1u << k));
    if (prm.write_known && wbest == 1) atomicOr(prm.masks + j, 1u << k);
    if (prm.s_out) prm.s_out[static_cast<std::size_t>(j) * prm.K + k] = wbest == 1 ? 1.0 : 0.0;
  }
}

// A chain of surface-free balls from p towards the certified neighbour's
// ball, one warp per pending pair, the whole warp on each nearest-triangle
// query (warp_nearest_dist). Each ball B(q, r) has r just below q's exact
// distance to the compartment's triangles; the next centre is kTraceStep r
// further along the line to the neighbour's centre (inside the current
// ball, so consecutive balls overlap); the chain succeeds when a ball
// reaches the neighbour's ball. The first ball alone is the test "B(p, gap)
// meets no triangle". A line that runs into the surface stops (radius below
// 1e-6 child edges) or gives up after kTraceSteps balls: the pair is
// evaluated. The outcome depends only on the point and the surfaces.
// 4 CTAs per SM (64 registers, small spills): the chains are latency-bound
// dependent loads; at 116 registers (2 CTAs) the kernel ran at 14 % achieved
// occupancy and 1.5 ms at cfg5 (profiles/r02/ncu_pair_chain_final.txt,
// chain_occupancy_ab.txt)
#ifndef NM_CHAIN_MIN_BLOCKS
#define NM_CHAIN_MIN_BLOCKS 4
#endif
static __global__ void __launch_bounds__(256, NM_CHAIN_MIN_BLOCKS) k_pair_chain(const ResolveParams prm) {
  const unsigned npend = *prm.npend;
  const int lane = threadIdx.x & 31;
  for (unsigned r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < npend; r += gridDim.x * blockDim.x / 32) {
    const PendPair q = prm.pend[r];
    const int k = static_cast<int>(q.k);
    const CellGrid g = prm.grids[k];
    const double b = g.B / kSubCells, rmin = 1e-6 * b;
    const float4* sup = prm.cl.sup + prm.cl.soff[k];
    const int nsup = static_cast<int>(prm.cl.soff[k + 1] - prm.cl.soff[k]);
    const std::uint32_t c0 = prm.cl.coff[k];
    const int nclus = static_cast<int>(prm.cl.coff[k + 1] - c0);
    double qx = q.p[0], qy = q.p[1], qz = q.p[2];
    bool ok = false;  // warp-uniform
    for (int step = 0; step < kTraceSteps; ++step) {
      const double ex = q.t[0] - qx, ey = q.t[1] - qy, ez = q.t[2] - qz;
      const double len = sqrt(ex * ex + ey * ey + ez * ez);
      const double need = len - q.t[3];  // a ball of radius > need around q meets the neighbour's ball
      if (need < -1e-9) {
        ok = true;
        break;
      }
      const double d = warp_nearest_dist(qx, qy, qz, need * (1.0 + 1e-6) + 2e-9, prm.cx, prm.cy, prm.cz, sup, nsup,
                                         prm.cl.clus + c0, nclus, prm.cl.clus_tri + static_cast<std::size_t>(c0) * kCluster,
                                         prm.cl.tsph + static_cast<std::size_t>(c0) * kCluster, prm.cl.xyz, prm.cl.tri);
      const double rr = d * (1.0 - 1e-9) - 1e-9;
      if (rr > need + 1e-9) {
        ok = true;
        break;
      }
      if (rr < rmin) break;  // running into the surface
      const double f = kTraceStep * rr / len;
      qx += f * ex;
      qy += f * ey;
      qz += f * ez;
    }
    if (ok && lane == 0) {
      atomicAnd(prm.unk + q.i, ~(1u << k));
      if (prm.write_known && q.w == 1u) atomicOr(prm.masks + q.j, 1u << k);
      if (prm.s_out) prm.s_out[static_cast<std::size_t>(q.j) * prm.K + k] = q.w == 1u ? 1.0 : 0.0;
    }
  }
}

struct PredBit {
  const std::uint32_t* v;
  int bit;
  __device__ bool operator()(std::size_t i) const { return (v[i] >> bit) & 1u; }
};

// ---------------------------------------------------------------------------
// Device run logic of the certified-cell build (round 2; the host restatement
// in cell_build.cu, NM_CELLS_HOST=1, is the reference it is tested against,
// bit for bit). Same rules, same fp operations in the same order (explicit
// _rn intrinsics: no contraction), so the codes are identical:
//   * k_runs_l1, one thread per grid row: every maximal x-run of certified
//     cells gets 0 (an end at the grid edge or outside the 13-DOP) or a
//     representative at its middle cell;
//   * k_runs_fine, one thread per (row, sy, sz) child sub-row: in every
//     segment of uncertified cells, each run of certified children gets the
//     neighbour parent's value (run touching the segment's start / end), 0
//     (grid edge, 13-DOP) or a representative;
//   * the representatives are evaluated by the sparse k_label and
//     k_rep_values turns s into w (0, 1 or unresolved);
//   * k_cell_codes / k_child_codes write the final codes.
// Values: -1 unresolved, 0 / 1 known w, 2 + r representative r (global
// slot). Representative slots come from per-compartment atomic cursors: their
// numbering varies, the codes do not (each representative is evaluated on its
// own).
// ---------------------------------------------------------------------------
struct RunParams {
  const CellGrid* grids;
  int K;
  const std::uint32_t* row_first;  // K + 1: first global row of each compartment (rows = ny nz)
  const std::uint8_t* cert;        // per cell: 1 certified
  const std::uint32_t* blk;        // per cell: global child block (uncertified cells)
  const std::uint8_t* child;       // per child: 1 certified
  const float4* dop4;              // 13-DOP slabs (kDopF4 float4 per compartment)
  double ctr0, ctr1, ctr2;         // centring offset (representatives are stored in the original frame)
  std::int32_t* cellval;           // per cell (fill pass)
  std::int32_t* childval;          // per child (fill pass)
  unsigned* rep_cursor;            // K per-compartment counters
  const unsigned* rep_first;       // K slot bases (fill pass)
  double* rep_pts;                 // 3 per representative (fill pass)
  int fill;                        // 0: count representatives only
};

__device__ __forceinline__ bool outside_dop_rn(const float4* dop4, int k, double x, double y, double z) {
  const float* dop = reinterpret_cast<const float*>(dop4 + static_cast<std::size_t>(k) * kDopF4);
  const float xf = static_cast<float>(x), yf = static_cast<float>(y), zf = static_cast<float>(z);
#pragma unroll
  for (int d = 0; d < kDopDirs; ++d) {
    const float pr =
        __fadd_rn(__fadd_rn(__fmul_rn(dop_dir(d, 0), xf), __fmul_rn(dop_dir(d, 1), yf)), __fmul_rn(dop_dir(d, 2), zf));
    if (pr < __ldg(dop + 2 * d) || pr > __ldg(dop + 2 * d + 1)) return true;
  }
  return false;
}

__device__ __forceinline__ std::int32_t new_rep(const RunParams& p, int k, double x, double y, double z) {
  const unsigned slot = atomicAdd(p.rep_cursor + k, 1u);
  if (!p.fill) return 0;
  const unsigned r = p.rep_first[k] + slot;
  p.rep_pts[3 * static_cast<std::size_t>(r)] = __dadd_rn(x, p.ctr0);
  p.rep_pts[3 * static_cast<std::size_t>(r) + 1] = __dadd_rn(y, p.ctr1);
  p.rep_pts[3 * static_cast<std::size_t>(r) + 2] = __dadd_rn(z, p.ctr2);
  return 2 + static_cast<std::int32_t>(r);
}

__device__ __forceinline__ int row_compartment(const RunParams& p, std::uint32_t row) {
  int k = 0;
  while (k + 1 < p.K && row >= p.row_first[k + 1]) ++k;
  return k;
}

// ---- level-1 runs as one connected component per surface-free region ----
// Face-adjacent certified cells have overlapping balls, so all certified
// cells connected through faces lie in one surface-free connected set and
// share one winding number. The x-runs of every row are numbered (row-major,
// so within a compartment in the host restatement's order) and united with
// the runs they touch in the rows y + 1 and z + 1 (lock-free union-find,
// larger root hooked under the smaller: the root is the component's smallest
// run). A component with a run that ends at the grid edge or outside the
// 13-DOP is 0; any other component gets ONE representative, at its root
// run's middle cell. (Round 1 gave every run its own representative.)
struct L1Params {
  const CellGrid* grids;
  int K;
  const std::uint32_t* row_first;  // K + 1: first global row of each compartment
  const std::uint8_t* cert;        // per cell: 1 certified
  const float4* dop4;
  std::uint32_t* rowruns;          // per row: number of certified runs (count pass)
  const std::uint32_t* runfirst;   // per row: first run id (exclusive scan of rowruns)
  std::int32_t* cellrun;           // per certified cell: its run id
  std::uint32_t* parent;           // per run: union-find parent (flattened: the root)
  std::uint32_t* runrow;           // per run: its row
  std::uint32_t* runx;             // per run: ix0 | ix1 << 16
  std::uint32_t* zero;             // per run: 1 = 0 known (edge / 13-DOP); per root after k_l1_flatten: the component's
  std::int32_t* rootval;           // per root run: 0, or 2 + representative slot
  std::int32_t* cellval;           // per cell (k_l1_cellval)
  std::uint32_t* nruns;            // total runs (k_l1_total)
  unsigned* rep_cursor;            // K per-compartment counters
  const unsigned* rep_first;       // K slot bases (fill)
  double* rep_pts;
  double ctr0, ctr1, ctr2;
  int fill;
};

struct RowPos {
  int k, iy, iz;
  std::size_t row;  // global index of the row's cell ix = 0
};

__device__ __forceinline__ RowPos row_pos(const CellGrid* grids, const std::uint32_t* row_first, int K, std::uint32_t r) {
  int k = 0;
  while (k + 1 < K && r >= row_first[k + 1]) ++k;
  const CellGrid& g = grids[k];
  const std::uint32_t lr = r - row_first[k];
  RowPos q;
  q.k = k;
  q.iy = static_cast<int>(lr % static_cast<std::uint32_t>(g.ny));
  q.iz = static_cast<int>(lr / g.ny);
  q.row = g.off + (static_cast<std::size_t>(q.iz) * g.ny + q.iy) * g.nx;
  return q;
}

static __global__ void k_l1_count(const L1Params p, std::uint32_t nrows) {
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const RowPos q = row_pos(p.grids, p.row_first, p.K, r);
    const int nx = p.grids[q.k].nx;
    std::uint32_t n = 0;
    bool prev = false;
    for (int ix = 0; ix < nx; ++ix) {
      const bool c = p.cert[q.row + ix] != 0;
      n += c && !prev;
      prev = c;
    }
    p.rowruns[r] = n;
  }
}

static __global__ void k_l1_label(const L1Params p, std::uint32_t nrows) {
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const RowPos q = row_pos(p.grids, p.row_first, p.K, r);
    const CellGrid g = p.grids[q.k];
    const double y = __dadd_rn(g.oy, __dmul_rn(q.iy + 0.5, g.B)), z = __dadd_rn(g.oz, __dmul_rn(q.iz + 0.5, g.B));
    std::uint32_t id = p.runfirst[r];
    for (int ix = 0; ix < g.nx;) {
      const bool c1 = p.cert[q.row + ix] != 0;
      int jx = ix;
      while (jx + 1 < g.nx && (p.cert[q.row + jx + 1] != 0) == c1) ++jx;
      if (c1) {
        const bool z0 = ix == 0 || jx == g.nx - 1 ||
                        outside_dop_rn(p.dop4, q.k, __dadd_rn(g.ox, __dmul_rn(ix + 0.5, g.B)), y, z) ||
                        outside_dop_rn(p.dop4, q.k, __dadd_rn(g.ox, __dmul_rn(jx + 0.5, g.B)), y, z);
        p.zero[id] = z0 ? 1u : 0u;
        p.parent[id] = id;
        p.runrow[id] = r;
        p.runx[id] = static_cast<std::uint32_t>(ix) | (static_cast<std::uint32_t>(jx) << 16);
        for (int x = ix; x <= jx; ++x) p.cellrun[q.row + x] = static_cast<std::int32_t>(id);
        ++id;
      }
      ix = jx + 1;
    }
  }
}

__device__ __forceinline__ std::uint32_t uf_find(std::uint32_t* parent, std::uint32_t x) {
  for (;;) {
    const std::uint32_t px = __ldcg(parent + x);
    if (px == x) return x;
    const std::uint32_t gp = __ldcg(parent + px);
    if (gp != px) parent[x] = gp;  // path halving (only ever points closer to the root)
    x = px;
  }
}

__device__ __forceinline__ void uf_unite(std::uint32_t* parent, std::uint32_t a, std::uint32_t b) {
  for (;;) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const std::uint32_t t = a;
      a = b;
      b = t;
    }
    const std::uint32_t old = atomicCAS(parent + b, b, a);  // hook the larger root under the smaller
    if (old == b) return;
    b = old;
  }
}

// runs of row r with the runs they touch in the rows y + 1 and z + 1
static __global__ void k_l1_union(const L1Params p, std::uint32_t nrows) {
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const RowPos q = row_pos(p.grids, p.row_first, p.K, r);
    const CellGrid& g = p.grids[q.k];
    const std::size_t dn[2] = {static_cast<std::size_t>(g.nx), static_cast<std::size_t>(g.nx) * g.ny};
    const bool has[2] = {q.iy + 1 < g.ny, q.iz + 1 < g.nz};
    for (int ix = 0; ix < g.nx; ++ix) {
      const std::size_t c = q.row + ix;
      if (!p.cert[c]) continue;
      const std::uint32_t a = static_cast<std::uint32_t>(p.cellrun[c]);
      for (int d = 0; d < 2; ++d) {
        if (!has[d]) continue;
        const std::size_t n = c + dn[d];
        if (!p.cert[n]) continue;
        const std::int32_t b = p.cellrun[n];
        if (ix > 0 && p.cert[c - 1] && p.cert[n - 1] && p.cellrun[n - 1] == b) continue;  // same pair as at ix - 1
        uf_unite(p.parent, a, static_cast<std::uint32_t>(b));
      }
    }
  }
}

static __global__ void k_l1_total(const L1Params p, std::uint32_t nrows) {
  *p.nruns = nrows ? p.runfirst[nrows - 1] + p.rowruns[nrows - 1] : 0u;
}

// root of x without writes: during k_l1_flatten the only store to parent[i]
// must be thread i's own (a path-halving store from another thread could
// land after it and leave i pointing at a non-root)
__device__ __forceinline__ std::uint32_t uf_root(const std::uint32_t* parent, std::uint32_t x) {
  for (;;) {
    const std::uint32_t px = __ldcg(parent + x);
    if (px == x) return x;
    x = px;
  }
}

// parent = root; a component with a known-0 run is 0
static __global__ void k_l1_flatten(const L1Params p) {
  const std::uint32_t nruns = *p.nruns;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nruns; i += gridDim.x * blockDim.x)
    p.parent[i] = uf_root(p.parent, i);
}
static __global__ void k_l1_zero(const L1Params p) {
  const std::uint32_t nruns = *p.nruns;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nruns; i += gridDim.x * blockDim.x)
    if (p.zero[i] && p.parent[i] != i) atomicOr(p.zero + p.parent[i], 1u);
}

// one representative per non-zero component, at its root run's middle cell
// (count pass: per-compartment counts; fill: slot, point, rootval)
static __global__ void k_l1_roots(const L1Params p) {
  const std::uint32_t nruns = *p.nruns;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nruns; i += gridDim.x * blockDim.x) {
    if (p.parent[i] != i) continue;
    if (p.zero[i]) {
      if (p.fill) p.rootval[i] = 0;
      continue;
    }
    const RowPos q = row_pos(p.grids, p.row_first, p.K, p.runrow[i]);
    const unsigned slot = atomicAdd(p.rep_cursor + q.k, 1u);
    if (!p.fill) continue;
    const CellGrid g = p.grids[q.k];
    const int ix = static_cast<int>(p.runx[i] & 0xffffu), jx = static_cast<int>(p.runx[i] >> 16);
    const unsigned rr = p.rep_first[q.k] + slot;
    p.rep_pts[3 * static_cast<std::size_t>(rr)] = __dadd_rn(__dadd_rn(g.ox, __dmul_rn((ix + jx) / 2 + 0.5, g.B)), p.ctr0);
    p.rep_pts[3 * static_cast<std::size_t>(rr) + 1] = __dadd_rn(__dadd_rn(g.oy, __dmul_rn(q.iy + 0.5, g.B)), p.ctr1);
    p.rep_pts[3 * static_cast<std::size_t>(rr) + 2] = __dadd_rn(__dadd_rn(g.oz, __dmul_rn(q.iz + 0.5, g.B)), p.ctr2);
    p.rootval[i] = 2 + static_cast<std::int32_t>(rr);
  }
}

static __global__ void k_l1_cellval(const L1Params p, std::uint32_t nrows) {
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const RowPos q = row_pos(p.grids, p.row_first, p.K, r);
    const int nx = p.grids[q.k].nx;
    for (int ix = 0; ix < nx; ++ix)
      if (p.cert[q.row + ix]) p.cellval[q.row + ix] = p.rootval[p.parent[p.cellrun[q.row + ix]]];
  }
}

constexpr std::size_t kNoCell = ~std::size_t(0);

// The first certified level-1 cell beyond a y / z face of parents q0..q1 of
// row (iy, iz) that the child sub-row (sy, sz) lies on (order: parents in x,
// then y-, y+, z-, z+), or kNoCell. The host restatement (cell_build.cu
// segment_runs) uses the same rule and order.
__host__ __device__ inline std::size_t fine_face_neighbour(const std::uint8_t* cert, const CellGrid& g, std::size_t row,
                                                           int iy, int iz, int sy, int sz, int q0, int q1) {
  const std::size_t plane = static_cast<std::size_t>(g.nx) * g.ny;
  for (int q = q0; q <= q1; ++q) {
    if (sy == 0 && iy > 0 && cert[row - g.nx + q]) return row - g.nx + q;
    if (sy == kSubCells - 1 && iy + 1 < g.ny && cert[row + g.nx + q]) return row + g.nx + q;
    if (sz == 0 && iz > 0 && cert[row - plane + q]) return row - plane + q;
    if (sz == kSubCells - 1 && iz + 1 < g.nz && cert[row + plane + q]) return row + plane + q;
  }
  return kNoCell;
}

static __global__ void k_runs_fine(const RunParams p, std::uint32_t nrows) {
  constexpr int S = kSubCells;
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < std::size_t(nrows) * S * S;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::uint32_t r = static_cast<std::uint32_t>(t / (S * S));
    const int sy = static_cast<int>(t % S), sz = static_cast<int>((t / S) % S);
    const int k = row_compartment(p, r);
    const CellGrid g = p.grids[k];
    const std::uint32_t lr = r - p.row_first[k];
    const int iy = static_cast<int>(lr % static_cast<std::uint32_t>(g.ny)), iz = static_cast<int>(lr / g.ny);
    const std::size_t row = g.off + (static_cast<std::size_t>(iz) * g.ny + iy) * g.nx;
    const double b = g.B / S;
    const double yy = __dadd_rn(__dadd_rn(g.oy, __dmul_rn(static_cast<double>(iy), g.B)), __dmul_rn(sy + 0.5, b));
    const double zz = __dadd_rn(__dadd_rn(g.oz, __dmul_rn(static_cast<double>(iz), g.B)), __dmul_rn(sz + 0.5, b));
    auto cidx = [&](int f) {  // child index of fine x cell f in this sub-row
      return static_cast<std::size_t>(p.blk[row + f / S]) * kChildren + (sz * S + sy) * S + f % S;
    };
    for (int ix = 0; ix < g.nx;) {
      const bool c1 = p.cert[row + ix] != 0;
      int jx = ix;
      while (jx + 1 < g.nx && (p.cert[row + jx + 1] != 0) == c1) ++jx;
      if (!c1) {
        const int f_lo = S * ix, f_hi = S * jx + S - 1;
        for (int f = f_lo; f <= f_hi;) {
          if (!p.child[cidx(f)]) {
            ++f;
            continue;
          }
          int e = f;
          while (e + 1 <= f_hi && p.child[cidx(e + 1)]) ++e;
          std::int32_t v;
          if (f == f_lo) {
            v = ix == 0 ? 0 : (p.fill ? p.cellval[row + ix - 1] : 0);
          } else if (e == f_hi) {
            v = jx == g.nx - 1 ? 0 : (p.fill ? p.cellval[row + jx + 1] : 0);
          } else if (outside_dop_rn(p.dop4, k, __dadd_rn(g.ox, __dmul_rn(f + 0.5, b)), yy, zz) ||
                     outside_dop_rn(p.dop4, k, __dadd_rn(g.ox, __dmul_rn(e + 0.5, b)), yy, zz)) {
            v = 0;
          } else {
            // a run on a y / z face of its parents takes the value of a
            // certified parent beyond that face (child and parent balls
            // overlap: centre distance <= 0.82 B); else a representative
            const std::size_t nb = fine_face_neighbour(p.cert, g, row, iy, iz, sy, sz, f / S, e / S);
            if (nb != kNoCell) v = p.fill ? p.cellval[nb] : 0;
            else v = new_rep(p, k, __dadd_rn(g.ox, __dmul_rn((f + e) / 2 + 0.5, b)), yy, zz);
          }
          if (p.fill)
            for (int q = f; q <= e; ++q) p.childval[cidx(q)] = v;
          f = e + 1;
        }
      }
      ix = jx + 1;
    }
  }
}

// w of every representative: round(s) when within 1e-3 of 0 or 1, else -1
static __global__ void k_rep_values(const double* s, std::uint32_t nreps, int K, const unsigned* rep_first,
                                    std::int32_t* w_out) {
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nreps; r += gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < K && r >= rep_first[k + 1]) ++k;
    const double v = s[static_cast<std::size_t>(r) * K + k];
    const double w = round(v);
    w_out[r] = (fabs(v - w) < 1e-3 && (w == 0.0 || w == 1.0)) ? static_cast<std::int32_t>(w) : -1;
  }
}

__device__ __forceinline__ std::int32_t decode_w(std::int32_t v, const std::int32_t* rep_w) {
  return v < 0 ? -1 : (v < 2 ? v : rep_w[v - 2]);
}

static __global__ void k_cell_codes(std::size_t ncells, const std::uint8_t* cert, const std::uint32_t* blk,
                                    const std::int32_t* cellval, const std::int32_t* rep_w, std::uint32_t* code,
                                    unsigned long long* ncert) {
  unsigned long long m = 0;
  for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < ncells;
       q += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    std::uint32_t c;
    if (!cert[q]) {
      c = 3u + blk[q];
    } else {
      const std::int32_t w = decode_w(cellval[q], rep_w);
      c = w < 0 ? 0u : static_cast<std::uint32_t>(1 + w);
    }
    code[q] = c;
    m += (c == 1u || c == 2u);
  }
  m = __reduce_add_sync(kFull, static_cast<unsigned>(m));
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(ncert, m);
}

// in place: child certification flag -> child code (0 unknown, 1 + w)
static __global__ void k_child_codes(std::size_t nchild, std::uint8_t* child, const std::int32_t* childval,
                                     const std::int32_t* rep_w, unsigned long long* ncert) {
  unsigned long long m = 0;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < nchild;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    std::uint8_t c = 0;
    if (child[i]) {
      const std::int32_t w = decode_w(childval[i], rep_w);
      c = w < 0 ? 0 : static_cast<std::uint8_t>(1 + w);
    }
    child[i] = c;
    m += c != 0;
  }
  m = __reduce_add_sync(kFull, static_cast<unsigned>(m));
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(ncert, m);
}

// uncertified-cell flags (for the child-block scan) and the block list
static __global__ void k_uncert(const std::uint8_t* cert, std::size_t n, std::uint32_t* unc) {
  for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    unc[q] = cert[q] ? 0u : 1u;
}
// block b = blk[q] of uncertified cell q -> its compartment-local cell index
static __global__ void k_block_cells(const std::uint8_t* cert, const std::uint32_t* blk, std::size_t n,
                                     const CellGrid* grids, int K, std::uint32_t* blk_cells) {
  for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    if (cert[q]) continue;
    int k = 0;
    while (k + 1 < K && q >= grids[k + 1].off) ++k;
    blk_cells[blk[q]] = static_cast<std::uint32_t>(q - grids[k].off);
  }
}

}  // namespace nm
