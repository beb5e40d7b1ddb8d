// Kernels of the B200 labeling path (sm_100a). See DESIGN.md §3 for the
// roofline each one is measured against.
//
//   k_morton_keys    30-bit Morton keys of the points (performance only)
//   k_label<P>       K1: fp32 N-body tile loop over every triangle of every
//                    compartment, fp64 fold per 256-triangle tile, inside
//                    bits + near-surface flags
//   k_select_*       order-preserving stream compaction (count / scan / write)
//   k_fixup          K3: fp64 re-evaluation of flagged (point, compartment)
//   k_label_tets     K4: tet label = id[ffs(AND of 4 node masks)]
//   straddle         K4': OR != AND on active compartments
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "check.cuh"
#include "vos.cuh"

namespace nm {

constexpr int kTile = 256;              // triangles per shared-memory tile (fp64 fold granularity)
constexpr int kSub = 32;                // triangles per subtile (near/far decision unit)
constexpr int kSubPerTile = kTile / kSub;
constexpr int kGroups = kSub / kSegTris;  // near/far groups (= strip segments) per subtile
constexpr int kSubRec = 1 + kGroups;      // float4 per subtile record: sphere of the subtile + of its groups
#ifndef NM_BLOCK
#define NM_BLOCK 128
#endif
constexpr int kBlock = NM_BLOCK;        // threads per CTA of k_label
#ifndef NM_MIN_BLOCKS
#define NM_MIN_BLOCKS 4                 // resident CTAs per SM requested for k_label<1>
#endif
#ifndef NM_FAR_UNROLL
#define NM_FAR_UNROLL 4                 // strip segments per iteration of the all-far group loop
#endif
constexpr int kFarUnroll = NM_FAR_UNROLL;
#ifndef NM_SUB_UNROLL
#define NM_SUB_UNROLL 1                 // subtiles per iteration of the tile loop
#endif
constexpr int kSubUnroll = NM_SUB_UNROLL;
#ifndef NM_MIN_BLOCKS_NP2
#define NM_MIN_BLOCKS_NP2 3             // resident CTAs per SM requested for k_label<2>
#endif
#ifndef NM_STAGES
// default: the two-buffer pipeline with one CTA barrier per tile; an
// explicit NM_STAGES selects the full/empty-mbarrier pipeline of that depth
#define NM_STAGES 2
#ifndef NM_BARRIER_PIPELINE
#define NM_BARRIER_PIPELINE
#endif
#endif
constexpr int kStages = NM_STAGES;
constexpr unsigned kFull = 0xffffffffu;
constexpr double kInv2Pi = 0.15915494309189533576888376337251;

// ---- bulk-copy (TMA engine) staging helpers --------------------------------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// orders this thread's earlier generic-proxy shared accesses (made visible
// to it by a CTA barrier) before its subsequent async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "NM_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra NM_WAIT;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// 13-DOP directions (axes, cube diagonals, face diagonals; unnormalised):
// a point outside any slab [lo_j, hi_j] of p.d_j is outside the convex hull
// of the compartment's vertices, hence outside the closed surface.
constexpr int kDopDirs = 13;
constexpr int kDopF4 = 7;  // 26 floats (lo_j, hi_j) padded to 7 float4
__host__ __device__ constexpr float dop_dir(int j, int a) {
  return (j == 0)    ? (a == 0 ? 1.f : 0.f)
         : (j == 1)  ? (a == 1 ? 1.f : 0.f)
         : (j == 2)  ? (a == 2 ? 1.f : 0.f)
         : (j == 3)  ? 1.f
         : (j == 4)  ? (a == 0 ? -1.f : 1.f)
         : (j == 5)  ? (a == 1 ? -1.f : 1.f)
         : (j == 6)  ? (a == 2 ? -1.f : 1.f)
         : (j == 7)  ? (a == 2 ? 0.f : 1.f)
         : (j == 8)  ? (a == 2 ? 0.f : (a == 0 ? 1.f : -1.f))
         : (j == 9)  ? (a == 1 ? 0.f : 1.f)
         : (j == 10) ? (a == 1 ? 0.f : (a == 0 ? 1.f : -1.f))
         : (j == 11) ? (a == 0 ? 0.f : 1.f)
                     : (a == 0 ? 0.f : (a == 1 ? 1.f : -1.f));
}

struct LabelIds {
  int id[32];
};

// Label ids staged in shared memory: a dynamically indexed kernel-parameter
// array would be copied to every thread's local stack (128 B per thread).
__device__ __forceinline__ const int* stage_ids(const LabelIds& ids, int* s_ids) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 32; ++k) s_ids[k] = ids.id[k];  // constant indices: read straight from the parameter bank
  }
  __syncthreads();
  return s_ids;
}

struct LabelParams {
  const double* pts;         // fp64 xyz, original frame
  std::size_t n;
  const std::uint32_t* order;  // evaluation order (Morton); nullptr = identity
  std::size_t n_pts;           // length of pts (points), for the checked build; SIZE_MAX: unknown (subset passes)
  std::uint32_t n_tiles;       // tiles of the surface set (checked build)
  const float4* tri;         // soup: 3 float4 per triangle (a.xyz,N.x) (b.xyz,N.y) (c.xyz,N.z);
                             // strip: kSegF4 float4 per 8-triangle segment (vos.cuh)
  const std::uint32_t* cont;  // strip layout: per tile, bit sidx * kGroups + j = segment j of subtile
                              // sidx continues segment j - 1 (same strip)
  const float4* sub;         // per subtile: fp32 centre c (centred frame), w = (far radius)^2;
                             // the subtile's vertices are stored relative to c
  const std::uint32_t* comp_tiles;  // K+1 tile offsets
  int K;
  double cx, cy, cz;         // centring offset of the fp32 frame
  double T, band;
  float tau, delta;
  // Outputs. Dense modes (0, 1) write both at the EVALUATION POSITION i
  // (coalesced; the host un-permutes the masks with k_unpermute); the sparse
  // mode ORs masks into masks[point id] (preset by k_cell_classify) and flags
  // into flagmask[position]. Flags stay position-indexed for the fix-up.
  std::uint32_t* masks;
  std::uint32_t* flagmask;   // bit k: pair (point at position i, k) needs the fp64 fix-up
  const std::uint32_t* cull;  // per evaluation position: bit k = outside compartment k's 13-DOP
                              // (k_cull_mask); nullptr = off
  double* s_out;             // n*K or nullptr
  unsigned long long* counters;  // [0] near / [1] far visits of (warp, 8-triangle group)
  // Compartment split (gridDim.y > 1): CTA row y handles compartments
  // [split[y], split[y+1]) of its points and ORs its bits into masks /
  // flagmask (zeroed by k_zero_masks). Each (point, compartment) sum is still
  // one CTA's fixed-order loop, so results do not depend on the split.
  int split[33];
  // Sparse mode (k_label MODE 2, cell culling): CTA b of the 1-D grid takes
  // compartment c with sp_blk[c] <= b < sp_blk[c + 1] and evaluates the
  // positions sp_list[sp_off[c] .. sp_end[c]) (indices into `order`)
  // against that compartment only, ORing its bits in (masks pre-set by
  // k_cell_classify).
  const std::uint32_t* sp_list;
  std::uint32_t sp_off[33];
  std::uint32_t sp_end[32];  // end of compartment c's slice (= sp_off[c + 1] when the slices are packed)
  std::uint32_t sp_blk[33];
  // Split sparse mode (sp_part != nullptr): compartment c's CTAs are
  // (point chunk, fold block) pairs, sp_fb[c] fold blocks per chunk; each
  // writes its points' fold-block partial sums to sp_part[sp_po[c] + i *
  // sp_fb[c] + b] (i = position in c's slice) and its detector bits to
  // sp_det; k_sparse_finalize adds the partials in block order.
  double* sp_part;
  std::uint8_t* sp_det;
  std::uint32_t sp_po[32];
  std::uint32_t sp_fb[32];
};

// fp64 fold structure of every (point, compartment) sum: per 256-triangle
// tile an fp32 sum, added in fp64 into a fold-block sum over kFoldTiles
// consecutive tiles of the compartment, the block sums added in block order.
// The split sparse pass evaluates fold blocks in separate CTAs and adds them
// in the same order, so every pass gives the same bits.
constexpr int kFoldTiles = 32;

// NP point pairs per thread (2*NP points), packed fp32x2 arithmetic.
// STRIP = false: 3 float4 per triangle (triangle soup);
// STRIP = true : 4 strip segments of 8 triangles per subtile (vos.cuh).
// MODE 0: every point x every compartment; 1: exact 13-DOP outside culling
// (prm.cull); 2: sparse (prm.sp_*): (point, compartment) pairs left unknown
// by the certified-cell classification (k_cell_classify).
template <int NP, bool STRIP, int MODE = 0>
static __global__ void __launch_bounds__(kBlock, (NP == 1 ? NM_MIN_BLOCKS : NM_MIN_BLOCKS_NP2)) k_label(const LabelParams prm) {
  constexpr int P = 2 * NP;
  constexpr bool CULL = MODE == 1;
  constexpr bool SPARSE = MODE == 2;
  constexpr int kSubF4 = STRIP ? (kSub / kSegTris) * kSegF4 : kSub * 3;  // float4 per subtile
  constexpr int kTileF4 = kSubF4 * kSubPerTile;
  // Two tile buffers filled by the bulk-copy engine (cp.async.bulk, one
  // elected thread), completion signalled on one mbarrier per buffer: tile
  // t + 1 streams in from L2 while the CTA evaluates tile t.
  constexpr unsigned kSubF4Tile = kSubPerTile * kSubRec;
  // kStages tile buffers: "full" mbarriers (bulk-copy transaction counts)
  // and "empty" mbarriers (one arrival per warp when it is done with the
  // buffer), so warps may drift up to kStages - 1 tiles apart without a CTA
  // barrier per tile (NM_BARRIER_PIPELINE: the round-1 two-buffer scheme
  // with one __syncthreads per tile).
  __shared__ alignas(128) float4 s_tri_buf[kStages][kTileF4];
  __shared__ alignas(128) float4 s_sub_buf[kStages][kSubF4Tile];
  __shared__ alignas(8) unsigned long long s_bar[kStages];
  __shared__ alignas(8) unsigned long long s_empty[kStages];
  __shared__ unsigned s_skip;

  std::size_t base = (static_cast<std::size_t>(blockIdx.x) * kBlock + threadIdx.x) * P;
  std::size_t n_end = prm.n;
  int c_sp = 0;
  int fb = 0, t_lo = 0, t_hi = 0;  // split sparse mode: this CTA's fold block and tile range
  if (SPARSE) {
    while (c_sp + 1 < prm.K && blockIdx.x >= prm.sp_blk[c_sp + 1]) ++c_sp;
    const unsigned nfb = prm.sp_part ? prm.sp_fb[c_sp] : 1u;
    const unsigned l = blockIdx.x - prm.sp_blk[c_sp];
    fb = static_cast<int>(l % nfb);
    base = prm.sp_off[c_sp] + (static_cast<std::size_t>(l / nfb) * kBlock + threadIdx.x) * P;
    n_end = prm.sp_end[c_sp];
    t_lo = static_cast<int>(prm.comp_tiles[c_sp]);
    t_hi = static_cast<int>(prm.comp_tiles[c_sp + 1]);
    if (prm.sp_part) {
      t_lo += fb * kFoldTiles;
      t_hi = min(t_hi, t_lo + kFoldTiles);
    }
  }
  // Points in the centred frame as double-singles (hi + lo), packed in pairs;
  // per subtile the kernel forms p - c = (hi - c) + lo, exact up to one
  // rounding of |p - c| (near-surface geometry keeps ~ulp(|p - c|)).
  float2 hx[NP], hy[NP], hz[NP], lx[NP], ly[NP], lz[NP];
  std::uint32_t pid[P];
  bool valid[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const std::size_t i = base + k;
    valid[k] = i < n_end;
    std::size_t ii = valid[k] ? i : n_end - 1;
    // points, order and lists are read once: streaming loads (evict-first),
    // so they do not push the triangle tiles (re-read by every CTA) out of L2
    if (SPARSE) ii = __ldcs(prm.sp_list + ii);
    const std::uint32_t j = prm.order ? __ldcs(prm.order + ii) : static_cast<std::uint32_t>(ii);
    NM_DCHECK(j < prm.n_pts, "k_label: point id out of range");
    pid[k] = j;
    const double* pj = prm.pts + 3 * static_cast<std::size_t>(j);
    const double dx = __ldcs(pj) - prm.cx, dy = __ldcs(pj + 1) - prm.cy, dz = __ldcs(pj + 2) - prm.cz;
    const float fx = static_cast<float>(dx), fy = static_cast<float>(dy), fz = static_cast<float>(dz);
    const float gx = static_cast<float>(dx - fx), gy = static_cast<float>(dy - fy), gz = static_cast<float>(dz - fz);
    if (k & 1) {
      hx[k >> 1].y = fx; hy[k >> 1].y = fy; hz[k >> 1].y = fz;
      lx[k >> 1].y = gx; ly[k >> 1].y = gy; lz[k >> 1].y = gz;
    } else {
      hx[k >> 1].x = fx; hy[k >> 1].x = fy; hz[k >> 1].x = fz;
      lx[k >> 1].x = gx; ly[k >> 1].x = gy; lz[k >> 1].x = gz;
    }
  }
  std::uint32_t mask[P], fmask[P], cull[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    mask[k] = fmask[k] = 0u;
    cull[k] = (CULL && valid[k]) ? prm.cull[base + k] : 0u;
  }
  unsigned n_near = 0, n_far = 0;

  // Compartments every point of the CTA is outside of (exact culling) are
  // skipped by producer and consumers alike; the tile sequence is fixed here.
  if (threadIdx.x == 0) {
    for (int b = 0; b < kStages; ++b) {
      mbar_init(&s_bar[b], 1);
      mbar_init(&s_empty[b], kBlock / 32);
    }
    s_skip = ~0u;
    fence_mbar_init();
  }
  __syncthreads();
  unsigned skip = 0u;
  if (CULL) {
    unsigned mine = ~0u;
#pragma unroll
    for (int k = 0; k < P; ++k)
      if (valid[k]) mine &= cull[k];
    mine = __reduce_and_sync(kFull, mine);
    if ((threadIdx.x & 31) == 0) atomicAnd(&s_skip, mine);
    __syncthreads();
    skip = s_skip;
  }
  const int c_lo = SPARSE ? c_sp : prm.split[blockIdx.y], c_hi = SPARSE ? c_sp + 1 : prm.split[blockIdx.y + 1];
  // producer state (thread 0 only): next tile to fetch, its compartment and
  // the tiles issued so far, kept in shared memory so they take no register
  // in the consumer threads
  __shared__ int s_pf_c, s_pf_t;
  __shared__ unsigned s_issued;
  int& pf_c = s_pf_c;
  int& pf_t = s_pf_t;
  unsigned& issued = s_issued;
  // tile range of compartment c for this CTA (split sparse: one fold block)
  auto t_first = [&](int c) { return SPARSE ? t_lo : static_cast<int>(prm.comp_tiles[c]); };
  auto t_last = [&](int c) { return SPARSE ? t_hi : static_cast<int>(prm.comp_tiles[c + 1]); };
  auto pf_seek = [&](int c) {  // first tile of the first non-skipped, non-empty compartment in [c, c_hi)
    for (; c < c_hi; ++c)
      if (!((skip >> c) & 1u) && t_first(c) < t_last(c)) {
        pf_c = c;
        pf_t = t_first(c);
        return;
      }
    pf_t = -1;
  };
  auto pf_issue = [&](int b) {
    NM_DCHECK(pf_t >= 0 && static_cast<std::uint32_t>(pf_t) < prm.n_tiles, "k_label: tile out of range");
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[b], (kTileF4 + kSubF4Tile) * 16u);
    bulk_g2s(s_tri_buf[b], prm.tri + static_cast<std::size_t>(pf_t) * kTileF4, kTileF4 * 16u, &s_bar[b]);
    bulk_g2s(s_sub_buf[b], prm.sub + static_cast<std::size_t>(pf_t) * kSubF4Tile, kSubF4Tile * 16u, &s_bar[b]);
  };
  auto pf_next = [&] {  // producer: advance to the next tile of the sequence
    if (pf_t >= 0 && ++pf_t >= t_last(pf_c)) pf_seek(pf_c + 1);
  };
  if (threadIdx.x == 0) {
    issued = 0;
    pf_seek(c_lo);
#ifdef NM_BARRIER_PIPELINE
    if (pf_t >= 0) pf_issue(0);
#else
    for (int q = 0; q < kStages - 1 && pf_t >= 0; ++q) {
      pf_issue(q);
      ++issued;
      pf_next();
    }
#endif
  }
  unsigned it = 0;

  int tile = t_first(c_lo);
  for (int c = c_lo; c < c_hi; ++c) {
    const int tile_end = t_last(c);
    const int tile_c0 = static_cast<int>(prm.comp_tiles[c]);  // fold blocks count from the compartment's first tile
    double acc64[P], blk64[P];
    bool det[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      acc64[k] = blk64[k] = 0.0;
      det[k] = false;
    }
    // Exact outside culling (opt-in): a point outside a closed compartment's
    // bounding box has winding number exactly 0 (SPEC.md:227 closedness), so
    // its s is set to 0 whatever the CTA does; the CTA skips the
    // compartment's tiles when every point is outside (skip bit c).
    bool outside[P];
#pragma unroll
    for (int k = 0; k < P; ++k) outside[k] = CULL && ((cull[k] >> c) & 1u);
    if (CULL && ((skip >> c) & 1u)) tile = tile_end;
    for (; tile < tile_end; ++tile) {
#ifdef NM_BARRIER_PIPELINE
      const int buf = it & 1u;
      if (threadIdx.x == 0) {
        // buffer buf ^ 1 was released by the barrier closing the previous tile
        pf_next();
        if (pf_t >= 0) pf_issue(buf ^ 1);
      }
      mbar_wait(&s_bar[buf], (it >> 1) & 1u);
#else
      const int buf = static_cast<int>(it % kStages);
      if (threadIdx.x == 0 && pf_t >= 0) {
        // tile `issued` (= it + kStages - 1) goes to the buffer that held tile
        // issued - kStages: wait until every warp has released it
        const unsigned b = issued % kStages;
        if (issued >= static_cast<unsigned>(kStages)) mbar_wait(&s_empty[b], ((issued / kStages) - 1) & 1u);
        pf_issue(static_cast<int>(b));
        ++issued;
        pf_next();
      }
      mbar_wait(&s_bar[buf], (it / kStages) & 1u);
#endif
      ++it;
      const float4* const s_tri = s_tri_buf[buf];
      const float4* const s_sub = s_sub_buf[buf];
      NM_DCHECK(static_cast<std::uint32_t>(tile) < prm.n_tiles, "k_label: consumer tile out of range");
      const std::uint32_t tcont = STRIP ? __ldg(prm.cont + tile) : 0u;

      float2 acc[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) acc[q] = make_float2(0.0f, 0.0f);
#pragma unroll kSubUnroll
      for (int st = 0; st < kSubPerTile; ++st) {
        const float4 sb = s_sub[st * kSubRec];
        float2 mx[NP], my[NP], mz[NP], sp[NP];  // -(p - c), |p - c|^2
        bool lane_far[P];
        bool far = true;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const float2 px = add2(add2(hx[q], bc(-sb.x)), lx[q]);
          const float2 py = add2(add2(hy[q], bc(-sb.y)), ly[q]);
          const float2 pz = add2(add2(hz[q], bc(-sb.z)), lz[q]);
          mx[q] = make_float2(-px.x, -px.y);
          my[q] = make_float2(-py.x, -py.y);
          mz[q] = make_float2(-pz.x, -pz.y);
          const float2 d2 = fma2(pz, pz, fma2(py, py, mul2(px, px)));
          sp[q] = d2;
          lane_far[2 * q] = !valid[2 * q] || d2.x > sb.w;
          lane_far[2 * q + 1] = !valid[2 * q + 1] || d2.y > sb.w;
          far &= lane_far[2 * q] && lane_far[2 * q + 1];
        }
        const float4* tt = s_tri + st * kSubF4;
        if constexpr (STRIP) {
          PairFrame f[NP];
#pragma unroll
          for (int q = 0; q < NP; ++q) f[q] = PairFrame{mx[q], my[q], mz[q], sp[q]};
          float2 ra[NP], rb[NP], sab[NP];  // chain state across continued segments
          const std::uint32_t cbits = tcont >> (st * kGroups);
          if (__all_sync(kFull, far)) {
            n_far += kSub / kSegTris;
#pragma unroll kFarUnroll
            for (int g = 0; g < kSub / kSegTris; ++g)
              seg_far<NP>(tt + g * kSegF4, f, acc, ra, rb, sab, g > 0 && ((cbits >> g) & 1u));
          } else {
            // per-group decision; each lane's evaluator depends only on its
            // own point (lane_far = far from the subtile or from the group).
            // The chain state is valid when the previous group ran seg_far.
            bool chain = false;
#pragma unroll 1
            for (int g = 0; g < kSub / kSegTris; ++g) {
              const bool cont = chain && ((cbits >> g) & 1u);
              const float4 sg = s_sub[st * kSubRec + 1 + g];
              bool gf[P];
              bool all = true, any = false;
#pragma unroll
              for (int q = 0; q < NP; ++q) {
                const float2 dx = add2(mx[q], bc(sg.x)), dy = add2(my[q], bc(sg.y)), dz = add2(mz[q], bc(sg.z));
                const float2 d2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
                gf[2 * q] = lane_far[2 * q] || d2.x > sg.w;
                gf[2 * q + 1] = lane_far[2 * q + 1] || d2.y > sg.w;
                all &= gf[2 * q] && gf[2 * q + 1];
                any |= (valid[2 * q] && gf[2 * q]) || (valid[2 * q + 1] && gf[2 * q + 1]);
              }
              const float4* rec = tt + g * kSegF4;
              if (__all_sync(kFull, all)) {
                ++n_far;
                seg_far<NP>(rec, f, acc, ra, rb, sab, cont);
                chain = true;
              } else {
                ++n_near;
                float2 an[NP];
                bool dn[P], use[P];
#pragma unroll
                for (int q = 0; q < NP; ++q) an[q] = acc[q];
#pragma unroll
                for (int k = 0; k < P; ++k) {
                  dn[k] = false;
                  use[k] = valid[k] && !gf[k];
                }
                NearFrame nf[NP];
                {
                  const float4 sc = s_sub[st * kSubRec];
#pragma unroll
                  for (int q = 0; q < NP; ++q) nf[q] = near_frame(hx[q], hy[q], hz[q], lx[q], ly[q], lz[q], sc);
                }
                seg_near<NP>(rec, nf, an, dn, use, prm.tau, prm.delta);
                chain = false;
                if (__any_sync(kFull, any)) {
                  float2 af[NP];
#pragma unroll
                  for (int q = 0; q < NP; ++q) af[q] = acc[q];
                  seg_far<NP>(rec, f, af, ra, rb, sab, cont);
                  chain = true;
#pragma unroll
                  for (int q = 0; q < NP; ++q) {
                    an[q].x = gf[2 * q] ? af[q].x : an[q].x;
                    an[q].y = gf[2 * q + 1] ? af[q].y : an[q].y;
                  }
                }
#pragma unroll
                for (int q = 0; q < NP; ++q) acc[q] = an[q];
#pragma unroll
                for (int k = 0; k < P; ++k) det[k] |= dn[k] && !gf[k];
              }
            }
          }
        } else {
          // triangle-soup layout: warp-uniform loop choice, per-lane
          // evaluator (the lane's own subtile test), so a pair's value does
          // not depend on its warp mates
          if (__all_sync(kFull, far)) {
            n_far += kSub / 8;
#pragma unroll 4
            for (int t = 0; t < kSub; ++t) {
              const float4 A = tt[3 * t], B = tt[3 * t + 1], C = tt[3 * t + 2];
#pragma unroll
              for (int q = 0; q < NP; ++q) {
                const VosTerms2 v = vos_terms2(A, B, C, mx[q], my[q], mz[q]);
                acc[q] = acc_far2(acc[q], v.num, v.den);
              }
            }
          } else {
            n_near += kSub / 8;
            // far lanes keep the far-form terms (bit-identical to an all-far
            // warp); near lanes use the exact double-single frame
            NearFrame nf[NP];
#pragma unroll
            for (int q = 0; q < NP; ++q) nf[q] = near_frame(hx[q], hy[q], hz[q], lx[q], ly[q], lz[q], sb);
#pragma unroll 1
            for (int t = 0; t < kSub; ++t) {
              const float4 A = tt[3 * t], B = tt[3 * t + 1], C = tt[3 * t + 2];
#pragma unroll
              for (int q = 0; q < NP; ++q) {
                const VosTerms2 v = vos_terms2(A, B, C, mx[q], my[q], mz[q]);
                const float2 af = acc_far2(acc[q], v.num, v.den);
                const float2 m3[3] = {nf[q].mx, nf[q].my, nf[q].mz}, l3[3] = {nf[q].lx, nf[q].ly, nf[q].lz};
                const VosTerms2 w = vos_terms2x(A, B, C, m3, l3);
                const float2 aw = acc_far2(acc[q], w.num, w.den);
                bool dx = false, dy = false;
                const float nx = acc_near_lane(acc[q].x, aw.x, w.num.x, w.den.x, w.r1.x, w.r2.x, w.r3.x, prm.tau,
                                               prm.delta, dx);
                const float ny = acc_near_lane(acc[q].y, aw.y, w.num.y, w.den.y, w.r1.y, w.r2.y, w.r3.y, prm.tau,
                                               prm.delta, dy);
                acc[q].x = lane_far[2 * q] ? af.x : nx;
                acc[q].y = lane_far[2 * q + 1] ? af.y : ny;
                det[2 * q] |= dx && !lane_far[2 * q];
                det[2 * q + 1] |= dy && !lane_far[2 * q + 1];
              }
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        blk64[2 * q] += static_cast<double>(acc[q].x);
        blk64[2 * q + 1] += static_cast<double>(acc[q].y);
      }
      if ((tile - tile_c0) % kFoldTiles == kFoldTiles - 1 || tile + 1 == tile_end) {  // fold block complete
#pragma unroll
        for (int k = 0; k < P; ++k) {
          acc64[k] += blk64[k];
          blk64[k] = 0.0;
        }
      }
#ifdef NM_BARRIER_PIPELINE
      __syncthreads();  // every warp is done with buffer buf: the producer may refill it
#else
      __syncwarp();  // this warp's reads of buffer buf are done
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s_empty[buf]);
#endif
    }
    if (SPARSE && prm.sp_part) {  // split: this CTA's fold-block partials, added by k_sparse_finalize
      const unsigned nfb = prm.sp_fb[c];
#pragma unroll
      for (int k = 0; k < P; ++k)
        if (valid[k]) {
          const std::size_t slot = prm.sp_po[c] + (base + k - prm.sp_off[c]) * nfb + fb;
          prm.sp_part[slot] = acc64[k];
          prm.sp_det[slot] = det[k];
        }
      continue;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const double s = outside[k] ? 0.0 : acc64[k] * kInv2Pi;
      det[k] &= !outside[k];
      if (s >= prm.T) mask[k] |= 1u << c;
      // NaN-safe: anything not provably outside the band is re-evaluated.
      if (det[k] || !(fabs(s - prm.T) >= prm.band)) fmask[k] |= 1u << c;
      if (prm.s_out && valid[k]) prm.s_out[static_cast<std::size_t>(pid[k]) * prm.K + c] = s;
    }
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    if (valid[k] && !(SPARSE && prm.sp_part)) {
      if (SPARSE) {
        NM_DCHECK(prm.sp_list[base + k] < prm.n, "k_label: sparse position out of range");
        if (mask[k]) atomicOr(prm.masks + pid[k], mask[k]);
        if (fmask[k]) atomicOr(prm.flagmask + prm.sp_list[base + k], fmask[k]);
      } else if (gridDim.y == 1) {  // evaluation order: coalesced, streaming stores
        NM_DCHECK(base + k < prm.n, "k_label: position out of range");
        __stcs(prm.masks + base + k, mask[k]);
        __stcs(prm.flagmask + base + k, fmask[k]);
      } else {
        if (mask[k]) atomicOr(prm.masks + base + k, mask[k]);
        if (fmask[k]) atomicOr(prm.flagmask + base + k, fmask[k]);
      }
    }
  }
  if ((threadIdx.x & 31) == 0 && prm.counters) {
    atomicAdd(prm.counters + 0, static_cast<unsigned long long>(n_near));
    atomicAdd(prm.counters + 1, static_cast<unsigned long long>(n_far));
  }
}

// ---------------------------------------------------------------------------
// Morton keys (10 bits per axis) of points in [lo, lo + 1/inv) — only the
// evaluation order depends on them, never a result.
// ---------------------------------------------------------------------------
__device__ __forceinline__ std::uint32_t spread10(std::uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Split sparse pass, second half: per (point, compartment) pair the fold-block
// partials added in block order (the dense pass's order), then the same
// threshold / detector / band logic as k_label's epilogue.
struct FinalizeParams {
  const std::uint32_t* list;   // pair positions (indices into order)
  const std::uint32_t* order;  // evaluation order -> point id (nullable)
  const double* part;
  const std::uint8_t* det;
  std::uint32_t sp_off[32];    // compartment c's slice in list
  std::uint32_t qo[33];        // prefix of the slice lengths (pair index space)
  std::uint32_t po[32], fb[32];
  int K;
  double T, band;
  std::uint32_t* masks;     // by point id
  std::uint32_t* flagmask;  // by evaluation position
  double* s_out;
};

static __global__ void k_sparse_finalize(const FinalizeParams prm) {
  const std::size_t total = prm.qo[prm.K];
  for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    int c = 0;
    while (c + 1 < prm.K && q >= prm.qo[c + 1]) ++c;
    const std::size_t i = q - prm.qo[c];
    const std::size_t slot = prm.po[c] + i * prm.fb[c];
    double acc = 0.0;
    bool det = false;
    for (std::uint32_t b = 0; b < prm.fb[c]; ++b) {
      acc += prm.part[slot + b];
      det |= prm.det[slot + b] != 0;
    }
    const std::uint32_t pos = prm.list[prm.sp_off[c] + i];
    const std::uint32_t j = prm.order ? prm.order[pos] : pos;
    const double s = acc * kInv2Pi;
    if (s >= prm.T) atomicOr(prm.masks + j, 1u << c);
    if (det || !(fabs(s - prm.T) >= prm.band)) atomicOr(prm.flagmask + pos, 1u << c);
    if (prm.s_out) prm.s_out[static_cast<std::size_t>(j) * prm.K + c] = s;
  }
}


static __global__ void k_morton_keys(const double* pts, std::size_t n, const std::uint32_t* subset, double lx, double ly,
                              double lz, double inv, std::uint32_t* keys, std::uint32_t* idx) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t j = subset ? subset[i] : i;
    auto q = [&](double v, double l) {
      const double t = (v - l) * inv;
      return static_cast<std::uint32_t>(t < 0.0 ? 0.0 : (t > 1023.0 ? 1023.0 : t));
    };
    keys[i] = spread10(q(pts[3 * j], lx)) | (spread10(q(pts[3 * j + 1], ly)) << 1) |
              (spread10(q(pts[3 * j + 2], lz)) << 2);
    idx[i] = static_cast<std::uint32_t>(j);
  }
}

// ---------------------------------------------------------------------------
// Order-preserving stream compaction: out = [i for i in [0,n) if pred(i)].
// Three launches (count per chunk, scan of chunk counts, ordered write); the
// total lands in *d_count on the device, so consumers need no host sync.
// ---------------------------------------------------------------------------
constexpr int kSelBlock = 256;
constexpr int kSelItems = 8;  // per thread
constexpr int kSelChunk = kSelBlock * kSelItems;

template <class Pred>
static __global__ void __launch_bounds__(kSelBlock) k_select_count(Pred pred, std::size_t n, std::uint32_t* chunk_counts) {
  const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * kSelChunk;
  int total = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const std::size_t i = b0 + j * kSelBlock + threadIdx.x;
    total += __syncthreads_count(i < n && pred(i));
  }
  if (threadIdx.x == 0) chunk_counts[blockIdx.x] = static_cast<std::uint32_t>(total);
}

// Single-CTA exclusive scan of chunk counts; writes the grand total. With
// gridDim.x > 1, CTA k scans counts[k nb, (k + 1) nb) into d_total[k].
static __global__ void __launch_bounds__(1024) k_select_scan(std::uint32_t* counts, std::size_t nb, std::uint32_t* d_total) {
  counts += blockIdx.x * nb;
  d_total += blockIdx.x;
  __shared__ std::uint32_t warp_sums[32];
  __shared__ std::uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (std::size_t b0 = 0; b0 < nb; b0 += 1024) {
    const std::size_t i = b0 + threadIdx.x;
    const std::uint32_t v = i < nb ? counts[i] : 0u;
    // inclusive warp scan
    std::uint32_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      std::uint32_t s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(kFull, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const std::uint32_t excl = carry + (w ? warp_sums[w - 1] : 0u) + x - v;
    if (i < nb) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *d_total = carry;
}

template <class Pred>
static __global__ void __launch_bounds__(kSelBlock) k_select_write(Pred pred, std::size_t n, const std::uint32_t* chunk_offsets,
                                                            std::uint32_t* out) {
  __shared__ std::uint32_t warp_cnt[kSelBlock / 32];
  const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * kSelChunk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  std::uint32_t running = chunk_offsets[blockIdx.x];
#pragma unroll 1
  for (int j = 0; j < kSelItems; ++j) {
    const std::size_t i = b0 + j * kSelBlock + threadIdx.x;
    const bool p = i < n && pred(i);
    const unsigned bal = __ballot_sync(kFull, p);
    if (lane == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    std::uint32_t before = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < kSelBlock / 32; ++q) {
      const std::uint32_t c = warp_cnt[q];
      before += q < w ? c : 0u;
      tot += c;
    }
    if (p) out[running + before + __popc(bal & ((1u << lane) - 1u))] = static_cast<std::uint32_t>(i);
    running += tot;
    __syncthreads();
  }
}

// All compartments' lists in one launch each (gridDim.y = compartments):
// list k holds the positions with bit k of v set, lists packed in k order.
static __global__ void __launch_bounds__(kSelBlock) k_select_count_bits(const std::uint32_t* __restrict__ v,
                                                                         std::size_t n, std::uint32_t* chunk_counts) {
  const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * kSelChunk;
  const unsigned bit = 1u << blockIdx.y;
  int total = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const std::size_t i = b0 + j * kSelBlock + threadIdx.x;
    total += __syncthreads_count(i < n && (v[i] & bit));
  }
  if (threadIdx.x == 0) chunk_counts[static_cast<std::size_t>(blockIdx.y) * gridDim.x + blockIdx.x] = static_cast<std::uint32_t>(total);
}
static __global__ void __launch_bounds__(kSelBlock) k_select_write_bits(const std::uint32_t* __restrict__ v, std::size_t n,
                                                                         const std::uint32_t* chunk_offsets,
                                                                         const std::uint32_t* totals, std::uint32_t* out) {
  __shared__ std::uint32_t warp_cnt[kSelBlock / 32];
  const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * kSelChunk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned bit = 1u << blockIdx.y;
  std::uint32_t running = chunk_offsets[static_cast<std::size_t>(blockIdx.y) * gridDim.x + blockIdx.x];
  for (unsigned q = 0; q < blockIdx.y; ++q) running += totals[q];  // the lists before k
#pragma unroll 1
  for (int j = 0; j < kSelItems; ++j) {
    const std::size_t i = b0 + j * kSelBlock + threadIdx.x;
    const bool p = i < n && (v[i] & bit);
    const unsigned bal = __ballot_sync(kFull, p);
    if (lane == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    std::uint32_t before = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < kSelBlock / 32; ++q) {
      const std::uint32_t c = warp_cnt[q];
      before += q < w ? c : 0u;
      tot += c;
    }
    if (p) out[running + before + __popc(bal & ((1u << lane) - 1u))] = static_cast<std::uint32_t>(i);
    running += tot;
    __syncthreads();
  }
}

struct PredNonzero {
  const std::uint32_t* v;
  __device__ bool operator()(std::size_t i) const { return v[i] != 0u; }
};

// Dense node passes: masks[point id] = ms[evaluation position].
static __global__ void k_unpermute(const std::uint32_t* __restrict__ order, std::size_t n,
                                   const std::uint32_t* __restrict__ ms, std::uint32_t* __restrict__ masks,
                                   std::size_t n_pts) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t j = order ? __ldcs(order + i) : i;
    NM_DCHECK(j < n_pts, "k_unpermute: point id out of range");
    masks[j] = __ldcs(ms + i);
  }
}

struct PredStraddle {
  const uint4* tets;
  const std::uint32_t* masks;
  std::uint32_t active;
  __device__ bool operator()(std::size_t i) const {
    const uint4 t = tets[i];
    const std::uint32_t a = masks[t.x], b = masks[t.y], c = masks[t.z], d = masks[t.w];
    return (((a & b & c & d) ^ (a | b | c | d)) & active) != 0u;
  }
};

// ---------------------------------------------------------------------------
// K3: fp64 fix-up of flagged (point, compartment) pairs.
//
// Pairs are grouped by compartment (k_fix_count / k_fix_fill: per-compartment
// counts and lists of positions in the flagged-point list; the order inside a
// list is irrelevant, see below). k_fixup: a CTA takes a batch of kFixPairs
// pairs of ONE compartment and streams that compartment's de-indexed fp64
// triangles (72 B each, file order) through shared memory in tiles of
// kFixTile, so every triangle load feeds kFixPairs points. Each pair is
// owned by kFixLanes threads: lane l sums triangles t = l, l + kFixLanes, ...
// in increasing t into two alternating accumulators (added at the end), then
// a fixed xor-butterfly adds the lanes. That order
// depends only on the compartment's triangle count, never on which pairs
// share the batch, so s is a pure function of (point, compartment).
// ---------------------------------------------------------------------------
struct FixupParams {
  const double* pts;
  const std::uint32_t* list;    // flagged evaluation positions
  const std::uint32_t* order;   // position -> point id (nullable: identity)
  const std::uint32_t* count;   // device count of list
  const std::uint32_t* flagmask;  // by position
  const double* tri64;          // de-indexed fp64 triangles: 9 doubles per triangle, compartment ranges of comp_off
  const std::uint32_t* comp_off;  // K+1
  const std::uint32_t* pair_cnt;  // K: flagged pairs per compartment
  const std::uint32_t* pairs;     // per compartment (prefix of pair_cnt): positions into list
  double* part;                   // per pair and triangle chunk: fp64 partial sums
  std::size_t n_pts, n_tri, n_part;  // checked build: lengths of pts, tri64 (triangles), part
  int K;
  double T, tie_eps;
  std::uint32_t* masks;
  double* s_out;
  unsigned long long* counters;  // [2] pairs, [3] ties
  std::uint32_t* exact;          // per pair (packed pair index): 1 = stage 2 (the oracle's terms throughout)
  int stage;                     // 1: hybrid terms; 2: oracle-order fp64 terms for the pairs marked exact
};

constexpr int kFixThreads = 128;
constexpr int kFixLanes = 8;                          // threads per pair
constexpr int kFixPairs = kFixThreads / kFixLanes;    // pairs per batch
constexpr int kFixTile = 128;                         // triangles per shared-memory tile (two buffers, 18 KB: ~8 CTAs per SM)
constexpr int kFixChunk = 2048;                       // triangles per work item (multiple of kFixTile)
constexpr int kFixRec = 16;                           // doubles per fix-up triangle record (k_deindex64)
constexpr int kFixStride = kFixRec + 1;               // in shared memory: 136 B, so the 8 lanes of a pair
                                                      // (records u, u + 1, ...) read 8 different banks
constexpr std::size_t kFixSmem = 2 * kFixTile * kFixStride * sizeof(double);  // k_fixup dynamic shared memory
constexpr float kFixFar2f = 64.0f;                    // far term: |A - p| > 8 x the longer edge from A
constexpr double kFixExactBand = 1e-4;                // stage 1 results this close to T go to stage 2

static __global__ void k_fix_count(const std::uint32_t* list, const std::uint32_t* count, const std::uint32_t* flagmask,
                                   std::uint32_t* pair_cnt) {
  const std::uint32_t n = *count;
  for (std::uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    for (std::uint32_t fm = flagmask[list[w]]; fm; fm &= fm - 1) atomicAdd(pair_cnt + (__ffs(fm) - 1), 1u);
  }
}

// pair_fill: per-compartment cursors (zeroed); lists at the prefix of pair_cnt
static __global__ void k_fix_fill(const std::uint32_t* list, const std::uint32_t* count, const std::uint32_t* flagmask,
                                  const std::uint32_t* pair_cnt, int K,
                                  std::uint32_t* pair_fill, std::uint32_t* pairs) {
  __shared__ std::uint32_t off[33];
  if (threadIdx.x == 0) {
    std::uint32_t o = 0;
    for (int c = 0; c < K; ++c) {
      off[c] = o;
      o += pair_cnt[c];
    }
  }
  __syncthreads();
  const std::uint32_t n = *count;
  for (std::uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    for (std::uint32_t fm = flagmask[list[w]]; fm; fm &= fm - 1) {
      const int c = __ffs(fm) - 1;
      pairs[off[c] + atomicAdd(pair_fill + c, 1u)] = w;
    }
  }
}

// de-indexed fp64 triangles for the fix-up (built once by nm_set_surfaces)
// One fix-up record per triangle (kFixRec doubles, file order): the fp64
// vertex A, 14 floats for the far evaluator (A, B - A, C - A, N = (B - A) x
// (C - A) from fp64, the larger squared edge from A rounded up, a pad),
// then the fp64 vertices B and C.
static __global__ void k_deindex64(const double* xyz, const std::uint32_t* tri, std::size_t nt, double* tri64) {
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    double v[9];
    for (int r = 0; r < 9; ++r) v[r] = xyz[3 * static_cast<std::size_t>(tri[3 * t + r / 3]) + r % 3];
    double* o = tri64 + kFixRec * t;
    for (int r = 0; r < 3; ++r) o[r] = v[r];
    for (int r = 3; r < 9; ++r) o[7 + r] = v[r];  // B at 10, C at 13
    const double ba[3] = {v[3] - v[0], v[4] - v[1], v[5] - v[2]}, ca[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
    const double n[3] = {ba[1] * ca[2] - ba[2] * ca[1], ba[2] * ca[0] - ba[0] * ca[2], ba[0] * ca[1] - ba[1] * ca[0]};
    const double e2 = fmax(ba[0] * ba[0] + ba[1] * ba[1] + ba[2] * ba[2], ca[0] * ca[0] + ca[1] * ca[1] + ca[2] * ca[2]);
    float* f = reinterpret_cast<float*>(o + 3);
    f[0] = static_cast<float>(v[0]);
    f[1] = static_cast<float>(v[1]);
    f[2] = static_cast<float>(v[2]);
    f[3] = static_cast<float>(ba[0]);
    f[4] = static_cast<float>(ba[1]);
    f[5] = static_cast<float>(ba[2]);
    f[6] = static_cast<float>(ca[0]);
    f[7] = static_cast<float>(ca[1]);
    f[8] = static_cast<float>(ca[2]);
    f[9] = static_cast<float>(n[0]);
    f[10] = static_cast<float>(n[1]);
    f[11] = static_cast<float>(n[2]);
    f[12] = nextafterf(static_cast<float>(e2), INFINITY);
    f[13] = 0.0f;
  }
}

// Far term of the hybrid first stage, fp32: R_a = A - p from the rounded
// vertex and point (|R_a| > 8 edges, so ~1e-6 relative), the record's edges
// and normal; the triangle subtends < 1/128 sr, so tan of the half angle
// x = num / den < 1/256 and atan x = x - x^3/3 + x^5/5 to 1e-17.
__device__ __forceinline__ float vos_far32(const float* f, float ax, float ay, float az, float la2) {
  const float bx = ax + f[3], by = ay + f[4], bz = az + f[5];
  const float cx = ax + f[6], cy = ay + f[7], cz = az + f[8];
  const float la = sqrtf(la2), lb = sqrtf(bx * bx + by * by + bz * bz), lc = sqrtf(cx * cx + cy * cy + cz * cz);
  const float num = f[9] * ax + f[10] * ay + f[11] * az;  // a . ((a + BA) x (a + CA)) = a . (BA x CA)
  const float den = la * lb * lc + (ax * bx + ay * by + az * bz) * lc + (ax * cx + ay * cy + az * cz) * lb +
                    (bx * cx + by * cy + bz * cz) * la;
  const float x = __fdividef(num, den), x2 = x * x;
  return x * (1.0f + x2 * (-1.0f / 3.0f + x2 * 0.2f));
}

// Work item (CTA): compartment c, a batch of kFixPairs of its pairs and a
// chunk of kFixChunk of its triangles. The chunk partial of every pair goes
// to part[poff_c + j * nchunk_c + chunk]; k_fix_finalize adds the chunks in
// order. Both the chunking and the lane striding depend only on c's triangle
// count, so s is a pure function of (point, compartment).
__device__ __forceinline__ std::uint32_t fix_nchunk(std::uint32_t ntri) {
  return max(1u, (ntri + kFixChunk - 1) / kFixChunk);
}

// 8-byte asynchronous global -> shared copies (LDGSTS): the next triangle
// tile streams in while the current one is evaluated (fp64 triangles start at
// any 8-byte offset, so no bulk copy)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifndef NM_FIX_MIN_BLOCKS
#define NM_FIX_MIN_BLOCKS 1  // 8 measured equal, 12 slower (profiles/r02/launch_bounds_ab.txt)
#endif
static __global__ void __launch_bounds__(kFixThreads, NM_FIX_MIN_BLOCKS) k_fixup(const FixupParams prm) {
  extern __shared__ double s_fix[];  // two tiles of kFixTile fp64 triangles (dynamic shared memory)
  __shared__ std::uint32_t s_off[33], s_wo[33], s_po[33];
  const int K = prm.K;
  if (threadIdx.x == 0) {
    std::uint32_t o = 0, wo = 0, po = 0;
    for (int c = 0; c < K; ++c) {
      const std::uint32_t nch = fix_nchunk(prm.comp_off[c + 1] - prm.comp_off[c]);
      s_off[c] = o;
      s_wo[c] = wo;
      s_po[c] = po;
      o += prm.pair_cnt[c];
      wo += (prm.pair_cnt[c] + kFixPairs - 1) / kFixPairs * nch;
      po += prm.pair_cnt[c] * nch;
    }
    s_wo[K] = wo;
  }
  __syncthreads();
  const std::uint32_t nwork = s_wo[K];
  const int slot = threadIdx.x / kFixLanes, lane = threadIdx.x % kFixLanes;
  for (std::uint32_t wk = blockIdx.x; wk < nwork; wk += gridDim.x) {  // CTA-uniform loop
    int c = 0;
    while (c + 1 < K && wk >= s_wo[c + 1]) ++c;
    const std::uint32_t lo = prm.comp_off[c], hi = prm.comp_off[c + 1];
    const std::uint32_t nch = fix_nchunk(hi - lo);
    const std::uint32_t l = wk - s_wo[c], batch = l / nch, chunk = l % nch;
    const std::uint32_t j = batch * kFixPairs + slot;
    bool has = j < prm.pair_cnt[c];
    if (prm.stage == 2) {
      has = has && prm.exact[s_off[c] + j] != 0u;
      if (!__syncthreads_or(has)) continue;  // no pair of this batch needs the oracle's terms
    }
    double px = 0.0, py = 0.0, pz = 0.0;
    if (has) {
      const std::uint32_t w = prm.pairs[s_off[c] + j];
      const std::uint32_t i = prm.order ? prm.order[prm.list[w]] : prm.list[w];
      NM_DCHECK(i < prm.n_pts, "k_fixup: point id out of range");
      px = prm.pts[3 * static_cast<std::size_t>(i)];
      py = prm.pts[3 * static_cast<std::size_t>(i) + 1];
      pz = prm.pts[3 * static_cast<std::size_t>(i) + 2];
    }
    const std::uint32_t c0 = lo + chunk * kFixChunk, c1 = min(hi, c0 + kFixChunk);
    NM_DCHECK(c1 <= prm.n_tri && c0 <= c1, "k_fixup: triangle chunk out of range");
    double sum = 0.0, sum1 = 0.0;  // two independent chains (the fp64 atan2 / sqrt sequences are latency-bound)
    bool near_zero = false;        // stage 1: a near term with num = 0
    const float pfx = static_cast<float>(px), pfy = static_cast<float>(py), pfz = static_cast<float>(pz);
    auto load = [&](int buf, std::uint32_t t0) {
      const std::uint32_t m = min(static_cast<std::uint32_t>(kFixTile), c1 - t0);
      const double* src = prm.tri64 + kFixRec * static_cast<std::size_t>(t0);
      double* dst = s_fix + buf * (kFixTile * kFixStride);
      for (std::uint32_t q = threadIdx.x; q < kFixRec * m; q += kFixThreads)
        cp_async8(dst + (q / kFixRec) * kFixStride + q % kFixRec, src + q);
      cp_async_commit();
    };
    __syncthreads();  // both buffers are free (previous work item done)
    load(0, c0);
    int buf = 0;
    for (std::uint32_t t0 = c0; t0 < c1; t0 += kFixTile, buf ^= 1) {
      const std::uint32_t m = min(static_cast<std::uint32_t>(kFixTile), c1 - t0);
      if (t0 + kFixTile < c1) {  // next tile into the other buffer (released by the barrier below)
        load(buf ^ 1, t0 + kFixTile);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();  // tile t0 is in buffer buf for every thread
      if (has) {
        const double* tile = s_fix + buf * (kFixTile * kFixStride);
        // stage 2: the oracle's exact operand order inside every term (no
        // FMA): on-surface points (num = +-0) must get the
        // oracle's atan2 branch. Stage 1: far triangles in fp32
        // (vos_far32), the others as in stage 2; a near term with num = 0
        // (the point in a triangle's plane) sends the pair to stage 2.
        auto term = [&](const double* e) -> double {
          if (prm.stage == 1) {
            const float* f = reinterpret_cast<const float*>(e + 3);
            const float ax = f[0] - pfx, ay = f[1] - pfy, az = f[2] - pfz;
            const float d2 = ax * ax + ay * ay + az * az;
            if (d2 > kFixFar2f * f[12]) return static_cast<double>(vos_far32(f, ax, ay, az, d2));
            double num;
            const double v = vos_half_angle64(e, e + 10, e + 13, px, py, pz, &num);
            if (num == 0.0) near_zero = true;
            return v;
          }
          return vos_half_angle64(e, e + 10, e + 13, px, py, pz);
        };
        std::uint32_t u = lane;
        for (; u + kFixLanes < m; u += 2 * kFixLanes) {
          const double* e = tile + kFixStride * u;
          sum += term(e);
          sum1 += term(e + kFixStride * kFixLanes);
        }
        if (u < m) sum += term(tile + kFixStride * u);
      }
      __syncthreads();  // buffer buf is consumed: the next iteration may refill it
    }
    sum += sum1;
#pragma unroll
    for (int o = kFixLanes / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o, kFixLanes);
    NM_DCHECK(!has || s_po[c] + j * nch + chunk < prm.n_part, "k_fixup: partial slot out of range");
    if (has && lane == 0) prm.part[s_po[c] + j * nch + chunk] = sum;
    if (has && near_zero) atomicOr(prm.exact + s_off[c] + j, 1u);
  }
}

// Per pair: the chunk partials added in chunk order, then threshold, tie
// count and s (the fp64 result replaces the fp32 pass's bit).
static __global__ void k_fix_finalize(const FixupParams prm) {
  __shared__ std::uint32_t s_off[33], s_po[33], s_nch[32];
  const int K = prm.K;
  if (threadIdx.x == 0) {
    std::uint32_t o = 0, po = 0;
    for (int c = 0; c < K; ++c) {
      const std::uint32_t nch = fix_nchunk(prm.comp_off[c + 1] - prm.comp_off[c]);
      s_off[c] = o;
      s_po[c] = po;
      s_nch[c] = nch;
      o += prm.pair_cnt[c];
      po += prm.pair_cnt[c] * nch;
    }
    s_off[K] = o;
  }
  __syncthreads();
  unsigned pairs = 0, ties = 0;
  for (std::uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < s_off[K]; q += gridDim.x * blockDim.x) {
    int c = 0;
    while (c + 1 < K && q >= s_off[c + 1]) ++c;
    const std::uint32_t j = q - s_off[c], nch = s_nch[c];
    if (prm.stage == 2 && prm.exact[q] == 0u) continue;
    double tot = 0.0;
    NM_DCHECK(s_po[c] + (j + 1) * nch <= prm.n_part, "k_fix_finalize: partials out of range");
    for (std::uint32_t b = 0; b < nch; ++b) tot += prm.part[s_po[c] + j * nch + b];
    const std::uint32_t w = prm.pairs[q];
    const std::uint32_t i = prm.order ? prm.order[prm.list[w]] : prm.list[w];
    NM_DCHECK(i < prm.n_pts, "k_fix_finalize: point id out of range");
    const double s = tot / (2.0 * CUDART_PI);
    if (prm.stage == 1 && (prm.exact[q] != 0u || fabs(s - prm.T) < kFixExactBand)) {
      prm.exact[q] = 1u;  // decided by stage 2
      continue;
    }
    if (s >= prm.T) atomicOr(prm.masks + i, 1u << c);
    else atomicAnd(prm.masks + i, ~(1u << c));
    ++pairs;
    if (fabs(s - prm.T) < prm.tie_eps) ++ties;
    if (prm.s_out) prm.s_out[static_cast<std::size_t>(i) * prm.K + c] = s;
  }
  if (prm.counters) {
    pairs = __reduce_add_sync(kFull, pairs);
    ties = __reduce_add_sync(kFull, ties);
    if ((threadIdx.x & 31) == 0 && (pairs || ties)) {
      atomicAdd(prm.counters + 2, static_cast<unsigned long long>(pairs));
      atomicAdd(prm.counters + 3, static_cast<unsigned long long>(ties));
    }
  }
}

// ---------------------------------------------------------------------------
// K4: tet labels: highest-priority compartment containing all
// four nodes, else 0.
// ---------------------------------------------------------------------------
// bad (nullable): tets with a node id >= n_nodes get label 0 and set *bad
// (the caller reports them) instead of reading out of range; without it the
// ids must have been checked.
static __global__ void k_label_tets(const uint4* __restrict__ tets, std::size_t nt, const std::uint32_t* __restrict__ masks,
                             int* __restrict__ labels, const LabelIds ids, std::size_t n_nodes,
                             std::uint32_t* __restrict__ bad = nullptr) {
  __shared__ int s_ids[32];
  const int* id = stage_ids(ids, s_ids);
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < nt;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const uint4 t = __ldcs(tets + i);  // read once; the gathered masks stay in L2
    if (bad && !(t.x < n_nodes && t.y < n_nodes && t.z < n_nodes && t.w < n_nodes)) {
      atomicOr(bad, 1u);
      __stcs(labels + i, 0);
      continue;
    }
    NM_DCHECK(t.x < n_nodes && t.y < n_nodes && t.z < n_nodes && t.w < n_nodes, "k_label_tets: node id out of range");
    const std::uint32_t m = __ldg(masks + t.x) & __ldg(masks + t.y) & __ldg(masks + t.z) & __ldg(masks + t.w);
    __stcs(labels + i, m ? id[__ffs(m) - 1] : 0);
  }
}

}  // namespace nm

// ---------------------------------------------------------------------------
// relabel_recursive support
// ---------------------------------------------------------------------------
namespace nm {

// Outward face i of a tet (mesh.hpp:57-64), sorted into (a <= b <= c).
// face f of a tet in outward order (mesh.hpp:57-64: {1,2,3} {0,3,2} {0,1,3}
// {0,2,1}), by selects (no local-memory table)
__device__ __forceinline__ void face_verts(const uint4 t, int f, std::uint32_t& a, std::uint32_t& b, std::uint32_t& c) {
  a = f == 0 ? t.y : t.x;
  b = f == 0 ? t.z : (f == 1 ? t.w : (f == 2 ? t.y : t.z));
  c = f == 0 ? t.w : (f == 1 ? t.z : (f == 2 ? t.w : t.y));
}

__device__ __forceinline__ void face_key(const uint4 t, int f, std::uint32_t& a, std::uint32_t& b, std::uint32_t& c) {
  face_verts(t, f, a, b, c);
  if (a > b) { const std::uint32_t s = a; a = b; b = s; }
  if (b > c) { const std::uint32_t s = b; b = c; c = s; }
  if (a > b) { const std::uint32_t s = a; a = b; b = s; }
}

static __global__ void k_face_keys(const uint4* tets, std::size_t nt, std::uint32_t* ka, std::uint32_t* kb, std::uint32_t* kc,
                            std::uint32_t* fid) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < 4 * nt;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    std::uint32_t a, b, c;
    face_key(tets[i >> 2], static_cast<int>(i & 3), a, b, c);
    ka[i] = a;
    kb[i] = b;
    kc[i] = c;
    fid[i] = static_cast<std::uint32_t>(i);
  }
}

// out[p] = key[fid[p]] (next LSD radix key for the current face order).
static __global__ void k_gather_key(const std::uint32_t* key, const std::uint32_t* fid, std::size_t m, std::uint32_t* out) {
  for (std::size_t p = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    out[p] = key[fid[p]];
}

// Faces sorted by (a,b,c): equal neighbours are the two sides of one face.
static __global__ void k_face_pairs(const std::uint32_t* fid, std::size_t m, const std::uint32_t* ka, const std::uint32_t* kb,
                             const std::uint32_t* kc, std::int32_t* nbr) {
  for (std::size_t p = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; p + 1 < m;
       p += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::uint32_t f = fid[p], g = fid[p + 1];
    if (ka[f] == ka[g] && kb[f] == kb[g] && kc[f] == kc[g]) {
      nbr[f] = static_cast<std::int32_t>(g >> 2);
      nbr[g] = static_cast<std::int32_t>(f >> 2);
    }
  }
}

// Nodes of tets adjacent to a label-change face.
static __global__ void k_frontier(const uint4* tets, std::size_t nt, const std::int32_t* nbr, const int* labels,
                           std::uint8_t* want) {
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int l = labels[t];
    bool adj = false;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const std::int32_t o = nbr[4 * t + f];
      adj |= (o >= 0) && (labels[o] != l);
    }
    if (adj) {
      const uint4 e = tets[t];
      want[e.x] = 1;
      want[e.y] = 1;
      want[e.z] = 1;
      want[e.w] = 1;
    }
  }
}

struct PredWantNew {
  const std::uint8_t* want;
  const std::uint8_t* known;
  __device__ bool operator()(std::size_t i) const { return want[i] && !known[i]; }
};

static __global__ void k_mark_known(const std::uint32_t* ids, const std::uint32_t* count, std::uint8_t* known) {
  const std::uint32_t n = *count;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) known[ids[i]] = 1;
}

// Label update barrier: every tet whose four nodes are evaluated.
static __global__ void k_relabel_tets(const uint4* tets, std::size_t nt, const std::uint32_t* masks, const std::uint8_t* known,
                               int* labels, const LabelIds ids, unsigned long long* changed) {
  __shared__ int s_ids[32];
  const int* id = stage_ids(ids, s_ids);
  unsigned long long c = 0;
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const uint4 e = tets[t];
    if (!(known[e.x] && known[e.y] && known[e.z] && known[e.w])) continue;
    const std::uint32_t m = masks[e.x] & masks[e.y] & masks[e.z] & masks[e.w];
    const int l = m ? id[__ffs(m) - 1] : 0;
    if (l != labels[t]) {
      labels[t] = l;
      ++c;
    }
  }
  if (c) atomicAdd(changed, c);
}

}  // namespace nm

namespace nm {

// Centroid query points (a + b + c + d) * 0.25 in fp64 (the oracle's order).
static __global__ void k_centroids(const double* nodes, const uint4* tets, std::size_t nt, double* out) {
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const uint4 e = tets[t];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double s = __dadd_rn(__dadd_rn(__dadd_rn(nodes[3 * static_cast<std::size_t>(e.x) + d],
                                                     nodes[3 * static_cast<std::size_t>(e.y) + d]),
                                           nodes[3 * static_cast<std::size_t>(e.z) + d]),
                                 nodes[3 * static_cast<std::size_t>(e.w) + d]);
      out[3 * t + d] = __dmul_rn(s, 0.25);
    }
  }
}

// label = id[ffs(mask)] or 0 for point-mode labels (centroids).
static __global__ void k_mask_labels(const std::uint32_t* masks, std::size_t n, int* labels, const LabelIds ids) {
  __shared__ int s_ids[32];
  const int* id = stage_ids(ids, s_ids);
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::uint32_t m = masks[i];
    labels[i] = m ? id[__ffs(m) - 1] : 0;
  }
}

}  // namespace nm

namespace nm {

static __global__ void k_iota(std::uint32_t* p, std::size_t m) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<std::uint32_t>(i);
}

// in_region[t] = labels[t] in set (extract_region_boundary, mesh.hpp:146-155)
static __global__ void k_region(const int* labels, std::size_t nt, const LabelIds set, int n_set, std::uint8_t* in_region) {
  for (std::size_t t = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int l = labels[t];
    bool in = false;
#pragma unroll
    for (int k = 0; k < 32; ++k) in |= k < n_set && set.id[k] == l;  // constant indices: no local copy
    in_region[t] = in ? 1 : 0;
  }
}

// A face is on the region boundary when exactly one incident tet is in the
// region (mesh.hpp:100-128).
struct PredBoundaryFace {
  const std::int32_t* nbr;
  const std::uint8_t* in_region;
  __device__ bool operator()(std::size_t i) const {
    if (!in_region[i >> 2]) return false;
    const std::int32_t o = nbr[i];
    return o < 0 || !in_region[o];
  }
};

struct PredUniqueU32 {
  const std::uint32_t* k;
  __device__ bool operator()(std::size_t i) const { return i == 0 || k[i] != k[i - 1]; }
};

// outward face i of a positively oriented tet (mesh.hpp:57-64)
static __global__ void k_face_tris(const uint4* tets, const std::uint32_t* faces, std::uint32_t nb, std::uint32_t* t0,
                            std::uint32_t* t1, std::uint32_t* t2) {
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const std::uint32_t f = faces[i];
    std::uint32_t a, b, c;
    face_verts(tets[f >> 2], static_cast<int>(f & 3), a, b, c);
    t0[i] = a;
    t1[i] = b;
    t2[i] = c;
  }
}

static __global__ void k_gather_tris(const std::uint32_t* order, std::uint32_t nb, const std::uint32_t* t0,
                              const std::uint32_t* t1, const std::uint32_t* t2, std::uint32_t* out) {
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const std::uint32_t j = order[i];
    out[3 * static_cast<std::size_t>(i)] = t0[j];
    out[3 * static_cast<std::size_t>(i) + 1] = t1[j];
    out[3 * static_cast<std::size_t>(i) + 2] = t2[j];
  }
}

}  // namespace nm

namespace nm {

// Regular 5-tet lattice on the device, bit-identical to generate_lattice_mesh
// (lattice.hpp:40-91): nodes k,j,i-major at origin + (i h, j h, k h); per cell
// the central + 4 corner tets of the parity pattern; orientation normalised
// with the fp64 tet_signed_volume of vec3.hpp:79-81 (same operand order).
static __global__ void k_lattice_nodes(double ox, double oy, double oz, double h, int nx, int ny, int nz, double* nodes) {
  const std::size_t n = static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1);
  for (std::size_t v = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(v % (nx + 1));
    const int j = static_cast<int>((v / (nx + 1)) % (ny + 1));
    const int k = static_cast<int>(v / (static_cast<std::size_t>(nx + 1) * (ny + 1)));
    nodes[3 * v] = __dadd_rn(ox, __dmul_rn(static_cast<double>(i), h));
    nodes[3 * v + 1] = __dadd_rn(oy, __dmul_rn(static_cast<double>(j), h));
    nodes[3 * v + 2] = __dadd_rn(oz, __dmul_rn(static_cast<double>(k), h));
  }
}

__device__ __forceinline__ double tet_volume64(const double* P, const std::uint32_t* t) {
  const double* a = P + 3 * static_cast<std::size_t>(t[0]);
  const double* b = P + 3 * static_cast<std::size_t>(t[1]);
  const double* c = P + 3 * static_cast<std::size_t>(t[2]);
  const double* d = P + 3 * static_cast<std::size_t>(t[3]);
  const double u0 = __dsub_rn(b[0], a[0]), u1 = __dsub_rn(b[1], a[1]), u2 = __dsub_rn(b[2], a[2]);
  const double v0 = __dsub_rn(c[0], a[0]), v1 = __dsub_rn(c[1], a[1]), v2 = __dsub_rn(c[2], a[2]);
  const double w0 = __dsub_rn(d[0], a[0]), w1 = __dsub_rn(d[1], a[1]), w2 = __dsub_rn(d[2], a[2]);
  const double x0 = __dsub_rn(__dmul_rn(v1, w2), __dmul_rn(v2, w1));
  const double x1 = __dsub_rn(__dmul_rn(v2, w0), __dmul_rn(v0, w2));
  const double x2 = __dsub_rn(__dmul_rn(v0, w1), __dmul_rn(v1, w0));
  return __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(u0, x0), __dmul_rn(u1, x1)), __dmul_rn(u2, x2)), 6.0);
}

static __global__ void k_lattice_tets(const double* nodes, int nx, int ny, int nz, uint4* tets) {
  const std::size_t cells = static_cast<std::size_t>(nx) * ny * nz;
  for (std::size_t cidx = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; cidx < cells;
       cidx += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(cidx % nx);
    const int j = static_cast<int>((cidx / nx) % ny);
    const int k = static_cast<int>(cidx / (static_cast<std::size_t>(nx) * ny));
    auto id = [&](int a, int b, int c) {
      return static_cast<std::uint32_t>((static_cast<std::size_t>(c) * (ny + 1) + b) * (nx + 1) + a);
    };
    const std::uint32_t v000 = id(i, j, k), v100 = id(i + 1, j, k), v010 = id(i, j + 1, k), v110 = id(i + 1, j + 1, k),
                        v001 = id(i, j, k + 1), v101 = id(i + 1, j, k + 1), v011 = id(i, j + 1, k + 1),
                        v111 = id(i + 1, j + 1, k + 1);
    std::uint32_t q[5][4];
    if (((i + j + k) & 1) == 0) {
      const std::uint32_t e[5][4] = {{v000, v110, v101, v011}, {v100, v000, v110, v101}, {v010, v000, v110, v011},
                                     {v001, v000, v101, v011}, {v111, v110, v101, v011}};
      for (int a = 0; a < 5; ++a)
        for (int b = 0; b < 4; ++b) q[a][b] = e[a][b];
    } else {
      const std::uint32_t e[5][4] = {{v100, v010, v001, v111}, {v000, v100, v010, v001}, {v110, v100, v010, v111},
                                     {v101, v100, v001, v111}, {v011, v010, v001, v111}};
      for (int a = 0; a < 5; ++a)
        for (int b = 0; b < 4; ++b) q[a][b] = e[a][b];
    }
    for (int a = 0; a < 5; ++a) {
      if (tet_volume64(nodes, q[a]) < 0.0) {
        const std::uint32_t s = q[a][2];
        q[a][2] = q[a][3];
        q[a][3] = s;
      }
      tets[5 * cidx + a] = make_uint4(q[a][0], q[a][1], q[a][2], q[a][3]);
    }
  }
}

}  // namespace nm

namespace nm {

// refine_boundary selection: tets labeled a or b that share
// a face with a tet of the other label (the one-element-thick layers on both
// sides of the a|b interface).
struct PredInterface {
  const std::int32_t* nbr;
  const int* labels;
  int a, b;
  __device__ bool operator()(std::size_t t) const {
    const int l = labels[t];
    if (l != a && l != b) return false;
    const int other = l == a ? b : a;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const std::int32_t o = nbr[4 * t + f];
      if (o >= 0 && labels[o] == other) return true;
    }
    return false;
  }
};

}  // namespace nm

namespace nm {

// Exact outside culling, per point: bit k set when the point (fp32 centred
// coordinates, as k_label forms them) lies outside a slab of compartment k's
// 13-DOP — outside the convex hull, so its winding number is exactly 0.
static __global__ void k_cull_mask(const double* pts, const std::uint32_t* order, std::size_t n, double cx, double cy, double cz,
                            const float4* dop4, int K, std::uint32_t* out) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t j = order ? order[i] : i;
    const float x = static_cast<float>(pts[3 * j] - cx), y = static_cast<float>(pts[3 * j + 1] - cy),
                z = static_cast<float>(pts[3 * j + 2] - cz);
    std::uint32_t m = 0;
    for (int c = 0; c < K; ++c) {
      const float* dop = reinterpret_cast<const float*>(dop4 + static_cast<std::size_t>(c) * kDopF4);
      bool o = false;
#pragma unroll
      for (int j = 0; j < kDopDirs; ++j) {
        const float pr = dop_dir(j, 0) * x + dop_dir(j, 1) * y + dop_dir(j, 2) * z;
        o |= pr < __ldg(dop + 2 * j) || pr > __ldg(dop + 2 * j + 1);
      }
      if (o) m |= 1u << c;
    }
    out[i] = m;
  }
}

// Position-indexed masks / flags cleared before a compartment-split k_label
// launch (which ORs its bits in).
static __global__ void k_zero_masks(std::size_t n, std::uint32_t* masks, std::uint32_t* flagmask) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    masks[i] = 0u;
    flagmask[i] = 0u;
  }
}

// Largest node index referenced by the tets (device-side validation of the
// host mesh, overlapped with the node pass in nm_label_mesh).
static __global__ void k_max_index(const uint4* __restrict__ tets, std::size_t nt, std::uint32_t* __restrict__ out) {
  std::uint32_t m = 0;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < nt;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const uint4 t = __ldg(tets + i);
    m = max(max(m, max(t.x, t.y)), max(t.z, t.w));
  }
  m = __reduce_max_sync(kFull, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Largest value of a uint32 array (device-side range checks of caller ids).
static __global__ void k_max_u32(const std::uint32_t* __restrict__ v, std::size_t n, std::uint32_t* __restrict__ out) {
  std::uint32_t m = 0;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    m = max(m, __ldg(v + i));
  m = __reduce_max_sync(kFull, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace nm
