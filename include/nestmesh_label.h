/*
 * nestmesh_label.h — C ABI of libnestmesh_label.so, the B200 (sm_100a)
 * implementation of the recursive solid-angle labeling path of nestmesh
 * (arXiv 2203.10000).
 *
 * The reference library (/root/reference/proj/include/nestmesh) specifies the
 * labeling module only in SPEC.md:210-272; it has no labeling code and no FFI.
 * These entry points are what a maintainer binds behind the SPEC signatures
 * (see include/nestmesh/labeling.hpp for the C++ drop-in and INTEGRATION.md
 * for the binding):
 *
 *   nm_enclosure      <- enclosure_ratio(point, surface)
 *   nm_label_nodes    <- node classification of initial_label
 *   nm_label_tets     <- tet rule of initial_label
 *   nm_label_mesh     <- initial_label(mesh, seg, params)
 *   nm_flag_boundary  <- straddle layer of refine_boundary
 *   nm_relabel        <- relabel_recursive(mesh, seg, params, prev_labels)
 *                                                                SPEC.md:243-251
 *
 * Conventions
 *   - Plain pointers and sizes; no torch or STL types cross this boundary.
 *   - Host-buffer entry points borrow caller-owned buffers for the duration
 *     of the call and are synchronous. *_device entry points take device
 *     pointers and a cudaStream_t (passed as void*; NULL = the context's own
 *     non-blocking stream, cudaStreamLegacy (0x1) = the legacy default
 *     stream) and are asynchronous unless stats are requested.
 *   - Points are fp64 xyz triples (the layout of std::vector<nestmesh::Vec3>,
 *     vec3.hpp:11-28); triangles are uint32 index triples into one fp64 vertex
 *     array (std::vector<nestmesh::Triangle>, surface.hpp:16); tets are uint32
 *     quadruples (std::vector<nestmesh::Tet>, mesh.hpp:19); labels are int32
 *     (mesh.hpp:33), 0 = outside / bounding box.
 *   - Compartments are given innermost (highest priority) first, at most 32;
 *     bit k of a node mask means "inside compartment k" (s_k >= T).
 *   - Return 0 on success, non-zero on failure; nm_last_error() returns a
 *     thread-local message. There is no CPU fallback: without a usable
 *     sm_100 device every compute entry point fails.
 *   - Results are independent of the number of devices / ranks a point set is
 *     sharded over.
 */
#ifndef NESTMESH_LABEL_H
#define NESTMESH_LABEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NM_ABI_VERSION 2

typedef struct nm_ctx nm_ctx;

/* Tunables of the solid-angle kernel (defaults from nm_default_options). */
typedef struct nm_options {
  int device;            /* CUDA device ordinal */
  float tau;             /* near-face detector: |num| <= tau*r1r2r3 && den <= tau*r1r2r3 */
  float delta_mm;        /* near-vertex detector: min r_i <= delta_mm */
  double band;           /* |s - T| < band after the fp32 pass -> fp64 fix-up */
  double tie_eps;        /* |s - T| < tie_eps after fix-up -> counted as a tie */
  float far_ratio;       /* subtile is "far" for a point when d >= far_ratio * radius + far_abs_mm */
  float far_abs_mm;
  int sort_points;       /* 1: Morton-order points before the kernel (performance only) */
  int pairs_per_thread;  /* point pairs per thread of the fp32 kernel: 1 or 2 (performance only) */
  int layout;            /* triangle tiles: 0 auto, 1 independent triangles, 2 strip segments (performance only) */
  int cull_outside;      /* 1: exact culling — a point outside a closed compartment's 13-DOP (slabs on 13
                            directions around its vertices) gets s = 0 without evaluating its triangles
                            (winding number of a closed surface); 2: additionally, a point inside a
                            certified cell of the compartment's grid (a cell whose ball meets no
                            triangle; grid built by nm_set_surfaces from the surfaces alone) gets the
                            cell's exact winding number (0 or 1); 0 (default): every pair is evaluated */
  int cell_axis;         /* certified-cell grid resolution: cells along each compartment's longest bounding-box
                            side, in [8, 1024]; 0 = default (120). A finer grid takes longer to build in
                            nm_set_surfaces and leaves fewer pairs to evaluate per pass (performance only:
                            results are identical) */
} nm_options;

/* Counters of one labeling call (accumulated by the call, not across calls). */
typedef struct nm_stats {
  uint64_t points;           /* points evaluated */
  uint64_t triangles;        /* real triangles over all compartments */
  uint64_t evals;            /* points x triangles (algorithmic point-triangle evaluations) */
  uint64_t flagged_points;   /* points sent to the fp64 fix-up */
  uint64_t flagged_pairs;    /* (point, compartment) pairs re-evaluated in fp64 */
  uint64_t ties;             /* pairs with |s - T| < tie_eps after fix-up */
  uint64_t near_subtiles;    /* warp x 8-triangle group visits that took the near path */
  uint64_t far_subtiles;     /* ... that took the far path */
  uint64_t launches;         /* kernels launched by this call */
  float ms_label;            /* device time of the fp32 solid-angle kernel (CUDA events) */
  float ms_fixup;            /* device time of compaction + fp64 fix-up */
  float ms_tets;             /* device time of the tet kernels */
  float ms_total;            /* device time of the whole call */
  float ms_host;             /* refinement time inside nm_refine_relabel (device, CUDA events) */
} nm_stats;

int nm_abi_version(void);
const char* nm_last_error(void);
void nm_default_options(nm_options* opt);

int nm_create(nm_ctx** ctx, const nm_options* opt /* NULL = defaults */);
int nm_destroy(nm_ctx* ctx);

/* Replicated surface set: nv fp64 vertices, nt triangles (global indices),
 * compartment k owns triangles [comp_tri_off[k], comp_tri_off[k+1]).
 * label_ids[k] is the tet label of compartment k (> 0). */
int nm_set_surfaces(nm_ctx* ctx, const double* xyz, size_t nv, const uint32_t* tri, size_t nt,
                    const uint32_t* comp_tri_off, int K, const int* label_ids);

/* Enclosure ratios s[i*K + k] (fp64; fp32 pass + fp64 fix-up of flagged pairs). */
int nm_enclosure(nm_ctx* ctx, const double* pts, size_t n, double threshold, double* s_out, nm_stats* stats);

/* Node masks (bit k = s_k >= T). */
int nm_label_nodes(nm_ctx* ctx, const double* pts, size_t n, double threshold, uint32_t* masks_out,
                   nm_stats* stats);

/* Tet labels from node masks: label_ids[lowest k inside at all 4 nodes], else 0. */
int nm_label_tets(nm_ctx* ctx, const uint32_t* tets, size_t nt, const uint32_t* masks, size_t n_nodes,
                  int* labels_out, nm_stats* stats);

/* initial_label: host nodes + tets in, host tet labels (and optional node masks) out. */
int nm_label_mesh(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                  double threshold, int* labels_out, uint32_t* masks_out /* nullable */, nm_stats* stats);

/* Regular 5-tet lattice generated on the device, bit-identical to
 * generate_lattice_mesh (lattice.hpp:40-91): (nx+1)(ny+1)(nz+1) fp64 nodes
 * and 5 nx ny nz uint32x4 tets into caller device buffers (asynchronous). */
int nm_lattice_device(nm_ctx* ctx, const double* origin, double h, int nx, int ny, int nz, double* d_nodes,
                      uint32_t* d_tets, void* stream);
/* initial_label of a regular lattice without host mesh traffic: the lattice
 * is generated on the device, labeled, and only the tet labels (and optional
 * node masks) come back. */
int nm_label_lattice(nm_ctx* ctx, const double* origin, double h, int nx, int ny, int nz, double threshold,
                     int* labels_out /* nullable */, uint32_t* masks_out /* nullable */, nm_stats* stats);

/* Tet-centroid labeling (query point = (a+b+c+d)*0.25 in fp64): label =
 * label_ids[lowest k with s_k(centroid) >= T], else 0. The alternative query
 * point named by the north star ("tet centroids or vertices"). */
int nm_label_centroids(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                       double threshold, int* labels_out, nm_stats* stats);

/* Tets whose node masks disagree on an active compartment (OR != AND on
 * active_mask), ascending; *count receives how many were written. */
int nm_flag_boundary(nm_ctx* ctx, const uint32_t* tets, size_t nt, const uint32_t* masks, size_t n_nodes,
                     uint32_t active_mask, uint32_t* tet_ids_out, size_t* count);

/* relabel_recursive: labels_io = prev_labels in, result out. Re-evaluates only
 * nodes of tets adjacent to label-change faces, pass after pass, until a pass
 * changes no label or max_iters passes ran. Returns 0 on success; *passes and
 * *converged report the iteration; converged == 0 means NonConvergence (labels
 * are the best found). evaluated (nullable, n_nodes bytes) marks evaluated nodes. */
int nm_relabel(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
               double threshold, int max_iters, int* labels_io, int* passes, int* converged,
               uint8_t* evaluated /* nullable */, nm_stats* stats);

/* ---- single-process multi-GPU group (C/C++ hosts; SPEC.md:267 --label-workers)
 * One context per device (devices may repeat), one host thread per device,
 * contiguous node and tet shards (or, with certified cells, cost-balanced
 * shares of the pair lists). Node masks are exchanged on the devices: NCCL
 * all-gather / all-reduce over NVLink when the devices are distinct, peer
 * copies when a device repeats. Bit-identical to a single device. (torch
 * hosts use one process per GPU: paper_2203_10000_b200/distributed.py.) */
typedef struct nm_group nm_group;
int nm_group_create(nm_group** g, int n_devices, const int* devices /* NULL = 0..n-1 */, const nm_options* opt);
int nm_group_destroy(nm_group* g);
int nm_group_size(const nm_group* g);
int nm_group_set_surfaces(nm_group* g, const double* xyz, size_t nv, const uint32_t* tri, size_t nt,
                          const uint32_t* comp_tri_off, int K, const int* label_ids);
int nm_group_label_mesh(nm_group* g, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                        double threshold, int* labels_out, uint32_t* masks_out /* nullable */, nm_stats* stats);
/* 1 when the group exchanges masks through NCCL (distinct devices, libnccl found) */
int nm_group_uses_nccl(const nm_group* g);

/* ---- device-resident entry points (asynchronous on `stream`) -------------- */
int nm_label_nodes_device(nm_ctx* ctx, const double* d_pts, size_t n, double threshold, uint32_t* d_masks,
                          double* d_s_out /* nullable, n*K */, void* stream, nm_stats* stats);
/* Cost-balanced multi-GPU node pass: shard `shard` of `nshards` evaluates its
 * share of the (point, compartment) pairs of ALL n points that culling does
 * not resolve (pair i of compartment k weighs k's tile count; equal-weight
 * contiguous slices of the per-compartment lists). d_masks (n entries) gets
 * the bits this shard owns: the known bits on shard 0, the evaluated bits on
 * their owner; the shards' masks are disjoint, so their bitwise OR — or their
 * integer sum, e.g. an NCCL all-reduce — is the full result, bit-identical
 * to nm_label_nodes_device. Every shard needs all n points. */
int nm_label_nodes_shard_device(nm_ctx* ctx, const double* d_pts, size_t n, double threshold, uint32_t* d_masks,
                                int shard, int nshards, void* stream, nm_stats* stats);

int nm_label_tets_device(nm_ctx* ctx, const uint32_t* d_tets, size_t nt, const uint32_t* d_masks,
                         int* d_labels, void* stream, nm_stats* stats);
int nm_flag_boundary_device(nm_ctx* ctx, const uint32_t* d_tets, size_t nt, const uint32_t* d_masks,
                            uint32_t active_mask, uint32_t* d_ids, uint32_t* d_count, void* stream);

/* ---- refinement (host code; the recursive driver's refine step) ----------
 * refine_volume: selected tets split 1:8
 * (shortest octahedron diagonal), unselected tets with one split edge, two
 * split edges of one face or one fully split face get the conforming Fig. 2
 * templates, any other pattern escalates to 1:8. Old node ids are kept;
 * midpoints are appended in ascending edge-key order; children inherit the
 * parent's label; parent[i] = parent tet of child i. */
typedef struct nm_mesh nm_mesh;
int nm_refine(const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt, const int* labels /* nullable */,
              const uint32_t* selected, size_t n_selected, nm_mesh** out);
int nm_mesh_sizes(const nm_mesh* m, size_t* n_nodes, size_t* n_tets, size_t* n_old_nodes);
int nm_mesh_copy(const nm_mesh* m, double* nodes, uint32_t* tets, int* labels, uint32_t* parent);
void nm_mesh_free(nm_mesh* m);
const char* nm_refine_last_error(void);
int nm_mesh_masks(const nm_mesh* m, uint32_t* masks);

/* Meshes returned by the device entry points below (nm_refine_device,
 * nm_refine_boundary, nm_refine_relabel) stay in device memory owned by the
 * handle (stream-ordered pool allocations); nm_mesh_copy / nm_mesh_masks copy
 * them straight into the caller's buffers and nm_mesh_free releases them.
 * For nm_refine_relabel with levels = 0, parent is the identity. */

/* refine_volume on the device for a given selection: same rules, numbering
 * and child order as nm_refine (bit-identical result). */
int nm_refine_device(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                     const int* labels /* nullable */, const uint32_t* selected, size_t n_selected, nm_mesh** out);

/* The same on caller DEVICE arrays (asynchronous on `stream` apart from a
 * few small count reads): inputs are validated on the device; the result
 * stays on the device, nm_mesh_copy_device copies it into caller device
 * buffers (nullable). Used by the multi-rank recursive driver, whose meshes
 * never leave the GPUs. */
int nm_refine_device_d(nm_ctx* ctx, const double* d_nodes, size_t n_nodes, const uint32_t* d_tets, size_t nt,
                       const int* d_labels /* nullable */, const uint32_t* d_selected, size_t n_selected, void* stream,
                       nm_mesh** out);
int nm_mesh_copy_device(const nm_mesh* m, double* d_nodes, uint32_t* d_tets, int* d_labels, uint32_t* d_parent,
                        void* stream);

/* refine_boundary on the device: the tets labeled a or b
 * that share a face with a tet of the other label are refined with
 * refine_volume (same rules/numbering as nm_refine; children inherit labels).
 * A pair with no shared face returns the input mesh unchanged. */
int nm_refine_boundary(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                       const int* labels, int label_a, int label_b, nm_mesh** out);

/* The recursive boundary driver: `levels`
 * times { flag the tets whose node masks straddle an active compartment
 * (device compaction), refine them on the device (same rules, numbering and
 * child order as nm_refine), evaluate ONLY the new nodes, relabel the tets }. masks (nullable) are the
 * input mesh's node masks (computed when NULL). The result, with labels and
 * final node masks (nm_mesh_masks), is returned in *out (free with
 * nm_mesh_free). stats accumulates the node passes (evals of new nodes only). */
int nm_refine_relabel(nm_ctx* ctx, const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt,
                      const uint32_t* masks /* nullable */, double threshold, uint32_t active_mask, int levels,
                      nm_mesh** out, nm_stats* stats);

/* ---- compartment boundary extraction on the device ------------------------
 * extract_compartment_boundary / extract_region_boundary (mesh.hpp:100-155):
 * faces owned by exactly one tet whose label is in label_set, outward from
 * that tet (mesh.hpp:57-64), sorted lexicographically, plus the sorted unique
 * boundary node ids — the reference's output, bit for bit. With a single
 * label that no tet carries the call fails with "UnknownLabel" (mesh.hpp:21-24). */
typedef struct nm_boundary nm_boundary;
int nm_extract_boundary(nm_ctx* ctx, const uint32_t* tets, size_t nt, const int* labels, const int* label_set,
                        int n_set, nm_boundary** out);
int nm_boundary_sizes(const nm_boundary* b, size_t* n_triangles, size_t* n_nodes);
int nm_boundary_copy(const nm_boundary* b, uint32_t* triangles, uint32_t* nodes);
void nm_boundary_free(nm_boundary* b);

/* ---- quality.boundary_distance ---------------------------
 * Unsigned distance from each point to the closest point of a triangle
 * surface (exact point-triangle distance; fp32 N-body pass, then fp64 over
 * the candidates within 1e-3 mm of the fp32 minimum: equal to the fp64
 * minimum over all triangles). stats->evals counts both passes. */
int nm_point_surface_distance(nm_ctx* ctx, const double* pts, size_t n, const double* xyz, size_t nv,
                              const uint32_t* tri, size_t nt, double* dist_out, nm_stats* stats);
/* Area-uniform samples on a triangle surface with a fixed seed (host code). */
int nm_sample_surface(const double* xyz, const uint32_t* tri, size_t nt, size_t count, uint64_t seed, double* pts_out);

/* Compartment count, real and padded (evaluated) triangle slots, and the tile
 * layout (1 triangles, 2 strips) chosen for the current surfaces. */
int nm_surface_info(nm_ctx* ctx, int* K, size_t* triangles, size_t* padded_triangles, int* layout);

/* Strip layout: 8-triangle segments, and how many of them continue the
 * previous segment of their strip inside a subtile (the far evaluator
 * reuses two vertex distances there). Both 0 for the triangle layout. */
int nm_surface_segments(nm_ctx* ctx, size_t* segments, size_t* continued);

/* Certified cells (cull_outside = 2): grid cells over all compartments, how
 * many are certified, representative evaluations and host wall time of the
 * build (nm_set_surfaces); (point, compartment) pairs and point-triangle
 * evaluations of the last node pass that were not resolved by culling. */
int nm_cell_info(nm_ctx* ctx, uint64_t* cells, uint64_t* certified, uint64_t* reps, double* ms_build,
                 uint64_t* last_pairs, uint64_t* last_evals);
/* The certified-cell codes (per level-1 cell: 0 unknown, 1 / 2 winding number
 * 0 / 1, 3 + b children in block b) and child states (0 unknown, 1 / 2), for
 * tests and tools; sizes first with null buffers. */
int nm_cell_dump(nm_ctx* ctx, uint32_t* codes, size_t codes_cap, uint8_t* children, size_t children_cap,
                 size_t* n_codes, size_t* n_children);

/* ---- binary label / node-mask sidecar next to tetmesh v1 -----------------
 * The reference writes meshes as %.17g text (write_tetmesh, mesh.hpp:238-289).
 * A labeling result is kept beside it, bit for bit, in <mesh>.tetmesh.nmlabels:
 * int32 labels per tet, optional uint32 node masks, and what ties them to the
 * mesh — its fingerprint (explicit meshes) or its LatticeSpec (lattices:
 * generate_lattice_mesh, lattice.hpp:40-91, regenerates the mesh bit for bit).
 * Little-endian; the payload carries a hash checked on read. */
typedef struct nm_sidecar_info {
  uint64_t n_nodes, n_tets;
  uint64_t mesh_fingerprint; /* nm_mesh_fingerprint of the labeled mesh */
  int K;                     /* compartments (label_ids[0..K)) */
  int has_masks;             /* node masks follow the labels */
  int is_lattice;            /* origin/h/n describe the mesh (generate_lattice_mesh) */
  int reserved;
  int label_ids[32];
  double threshold;          /* T of the labeling */
  double origin[3];
  double h;
  int n[3];
  int reserved2;
} nm_sidecar_info;

/* Order-independent 64-bit fingerprint of a mesh (fp64 node bits + tet
 * indices); host and device versions give the same value. */
int nm_mesh_fingerprint(const double* nodes, size_t n_nodes, const uint32_t* tets, size_t nt, uint64_t* fp);
int nm_mesh_fingerprint_device(nm_ctx* ctx, const double* d_nodes, size_t n_nodes, const uint32_t* d_tets, size_t nt,
                               uint64_t* fp, void* stream);
int nm_sidecar_write(const char* path, const nm_sidecar_info* info, const int* labels, const uint32_t* masks /* nullable */);
int nm_sidecar_read_info(const char* path, nm_sidecar_info* info);
/* labels: n_tets entries; masks: n_nodes entries when has_masks (nullable: skipped) */
int nm_sidecar_read(const char* path, nm_sidecar_info* info, int* labels, uint32_t* masks);
/* initial_label of a regular lattice straight to a sidecar: the lattice is
 * generated, labeled and fingerprinted on the device; only labels (+ masks)
 * cross to the host, into the file. info_out (nullable) receives the header. */
int nm_label_lattice_sidecar(nm_ctx* ctx, const double* origin, double h, int nx, int ny, int nz, double threshold,
                             const char* path, int with_masks, nm_sidecar_info* info_out, nm_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* NESTMESH_LABEL_H */
