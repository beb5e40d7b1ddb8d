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
      const double u = (x - g.ox) / g.B, v = (y - g.oy) / g.B, w = (z - g.oz) / g.B;
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

struct PredBit {
  const std::uint32_t* v;
  int bit;
  __device__ bool operator()(std::size_t i) const { return (v[i] >> bit) & 1u; }
};

}  // namespace nm
