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
//   * the host gives every maximal x-run of certified cells one winding
//     number: adjacent cells' balls overlap, so a run's union is connected
//     and surface-free. A run with an end cell whose centre lies outside the
//     compartment's 13-DOP (hence outside the convex hull: w = 0 exactly) is
//     0; any other run gets w = round(s) at one representative cell centre,
//     evaluated by k_label (sparse mode) — accepted only when s is within
//     1e-3 of 0 or 1, otherwise the run stays uncertified.
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

// One thread per cell of one compartment: cert = 1 when no triangle of the
// compartment meets the cell's ball.
__global__ void __launch_bounds__(256) k_cell_certify(const CellGrid g, const float4* __restrict__ clus, int nclus,
                                                      const std::uint32_t* __restrict__ clus_tri,
                                                      const double* __restrict__ xyz, const std::uint32_t* __restrict__ tri,
                                                      double cx, double cy, double cz, std::uint8_t* __restrict__ cert) {
  const std::size_t ncell = static_cast<std::size_t>(g.nx) * g.ny * g.nz;
  const std::size_t id = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  if (id >= ncell) return;
  const int ix = static_cast<int>(id % g.nx);
  const int iy = static_cast<int>((id / g.nx) % g.ny);
  const int iz = static_cast<int>(id / (static_cast<std::size_t>(g.nx) * g.ny));
  const double Cx = g.ox + (ix + 0.5) * g.B, Cy = g.oy + (iy + 0.5) * g.B, Cz = g.oz + (iz + 0.5) * g.B;
  const double rb = g.B * 0.8660254037844387 * (1.0 + 1e-9) + 1e-6;  // ball radius (covers the closed cube)
  const float fx = static_cast<float>(Cx), fy = static_cast<float>(Cy), fz = static_cast<float>(Cz);
  const float frb = static_cast<float>(rb) + 1e-3f;  // + fp32 margin of the cluster test
  bool hit = false;
  for (int q = 0; q < nclus && !hit; ++q) {
    const float4 s = __ldg(clus + q);
    const float dx = fx - s.x, dy = fy - s.y, dz = fz - s.z;
    const float R = frb + s.w;
    if (dx * dx + dy * dy + dz * dz > R * R) continue;
    const V3t<double> p{Cx + cx, Cy + cy, Cz + cz};
    for (int t = 0; t < kCluster; ++t) {
      const std::uint32_t tid = __ldg(clus_tri + static_cast<std::size_t>(q) * kCluster + t);
      if (tid == 0xffffffffu) break;
      const std::uint32_t* e = tri + 3 * static_cast<std::size_t>(tid);
      const double* A = xyz + 3 * static_cast<std::size_t>(e[0]);
      const double* Bv = xyz + 3 * static_cast<std::size_t>(e[1]);
      const double* Cv = xyz + 3 * static_cast<std::size_t>(e[2]);
      const double d2 = point_tri_dist2<double>(p, {A[0], A[1], A[2]}, {Bv[0], Bv[1], Bv[2]}, {Cv[0], Cv[1], Cv[2]});
      if (!(d2 > rb * rb)) {  // NaN (degenerate) counts as a hit
        hit = true;
        break;
      }
    }
  }
  cert[g.off + id] = hit ? 0 : 1;
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
  const float4* dop4;  // 13-DOP slabs per compartment (k_cull_mask)
  const CellGrid* grids;
  const std::uint8_t* state;  // 0 unknown, 1 certified w = 0, 2 certified w = 1
  int K;
  std::uint32_t* unk;
  std::uint32_t* masks;
  std::uint32_t* flagmask;
  double* s_out;
};

__global__ void k_cell_classify(const ClassifyParams prm) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < prm.n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t j = prm.order ? prm.order[i] : i;
    const double x = prm.pts[3 * j] - prm.cx, y = prm.pts[3 * j + 1] - prm.cy, z = prm.pts[3 * j + 2] - prm.cz;
    const float xf = static_cast<float>(x), yf = static_cast<float>(y), zf = static_cast<float>(z);
    std::uint32_t unk = 0, ins = 0;
    for (int c = 0; c < prm.K; ++c) {
      const float* dop = reinterpret_cast<const float*>(prm.dop4 + static_cast<std::size_t>(c) * kDopF4);
      bool o = false;
#pragma unroll
      for (int d = 0; d < kDopDirs; ++d) {
        const float pr = dop_dir(d, 0) * xf + dop_dir(d, 1) * yf + dop_dir(d, 2) * zf;
        o |= pr < __ldg(dop + 2 * d) || pr > __ldg(dop + 2 * d + 1);
      }
      if (o) continue;  // outside the convex hull: w = 0
      const CellGrid g = prm.grids[c];
      const double u = (x - g.ox) / g.B, v = (y - g.oy) / g.B, w = (z - g.oz) / g.B;
      std::uint8_t st = 0;
      if (u >= 0.0 && v >= 0.0 && w >= 0.0 && u < g.nx && v < g.ny && w < g.nz) {
        const std::size_t cell = (static_cast<std::size_t>(static_cast<int>(w)) * g.ny + static_cast<int>(v)) * g.nx +
                                 static_cast<int>(u);
        st = __ldg(prm.state + g.off + cell);
      }
      if (st == 2) ins |= 1u << c;
      else if (st != 1) unk |= 1u << c;
    }
    prm.unk[i] = unk;
    prm.masks[j] = ins;
    prm.flagmask[j] = 0u;
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
