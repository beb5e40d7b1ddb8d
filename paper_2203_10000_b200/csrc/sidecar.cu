// Binary label + node-mask sidecar next to a tetmesh v1 file (SURVEY.md §8f
// row 4; the reference's mesh export is the %.17g text format of
// mesh.hpp:238-289, which stays the reference's CPU code).
//
// A labeling result is written as a small binary file beside the mesh
// (<mesh>.tetmesh.nmlabels): per-tet int32 labels and optional per-node
// uint32 masks, bit for bit, plus what ties them to their mesh:
//   * an explicit mesh: the fingerprint of its nodes and tets
//     (nm_mesh_fingerprint; host or device, same value);
//   * a regular lattice (generate_lattice_mesh, lattice.hpp:40-91): the
//     LatticeSpec, which regenerates the mesh bit for bit
//     (nm_lattice_device), so neither the 800 MB of tets nor %.17g node text
//     is written or uploaded: nm_label_lattice_sidecar generates the lattice
//     on the device, labels it, fingerprints it there and writes labels +
//     masks straight from pinned memory.
//
// File (little-endian, x86-64 layout of nm_sidecar_info):
//   "NMSIDE01" | u32 info_bytes | nm_sidecar_info | i32 labels[n_tets]
//   | u32 masks[n_nodes] (if has_masks) | u64 payload_hash
// payload_hash = the same positional hash over the label and mask words.
#include "context.cuh"

#include <cstdio>

using namespace nmh;

namespace {

constexpr char kMagic[8] = {'N', 'M', 'S', 'I', 'D', 'E', '0', '1'};
constexpr std::uint64_t kSeedNodes = 0x6e6f6465735f6e6dull, kSeedTets = 0x746574735f5f6e6dull,
                        kSeedPay = 0x7061796c6f61646dull;

// splitmix64 finaliser
__host__ __device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// positional word hash: the fingerprint is the wrapping SUM over words, so any
// reduction order (device atomics, host loop) gives the same value
__host__ __device__ __forceinline__ std::uint64_t word_hash(std::uint64_t seed, std::uint64_t i, std::uint64_t w) {
  return mix64(seed ^ mix64(i * 0x9e3779b97f4a7c15ull + w));
}

__global__ void k_hash_words(const std::uint64_t* __restrict__ w, std::size_t m, std::uint64_t seed,
                             unsigned long long* out) {
  std::uint64_t acc = 0;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    acc += word_hash(seed, i, __ldg(reinterpret_cast<const unsigned long long*>(w) + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

std::uint64_t host_hash_words(const void* p, std::size_t bytes, std::uint64_t seed) {
  const auto* b = static_cast<const unsigned char*>(p);
  std::uint64_t acc = 0;
  const std::size_t m = bytes / 8;
  for (std::size_t i = 0; i < m; ++i) {
    std::uint64_t w;
    std::memcpy(&w, b + 8 * i, 8);
    acc += word_hash(seed, i, w);
  }
  if (bytes % 8) {  // odd tail (an odd count of 4-byte words): zero-padded last word
    std::uint64_t w = 0;
    std::memcpy(&w, b + 8 * m, bytes % 8);
    acc += word_hash(seed, m, w);
  }
  return acc;
}

std::uint64_t combine(std::uint64_t hn, std::uint64_t ht, std::uint64_t n, std::uint64_t nt) {
  return mix64(hn ^ mix64(ht + 0x632be59bd9b4e019ull) ^ mix64(n * 3 + 1) ^ mix64(nt * 5 + 2));
}

std::uint64_t payload_hash(const int* labels, std::size_t nt, const std::uint32_t* masks, std::size_t nn) {
  std::uint64_t h = host_hash_words(labels, nt * sizeof(int), kSeedPay);
  if (masks) h = mix64(h) + host_hash_words(masks, nn * sizeof(std::uint32_t), kSeedPay ^ 1);
  return h;
}

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

void write_all(std::FILE* f, const void* p, std::size_t bytes, const char* path) {
  const auto* b = static_cast<const char*>(p);
  while (bytes) {
    const std::size_t chunk = std::min<std::size_t>(bytes, std::size_t(1) << 28);
    if (std::fwrite(b, 1, chunk, f) != chunk) throw Error(std::string("cannot write ") + path);
    b += chunk;
    bytes -= chunk;
  }
}
void read_all(std::FILE* f, void* p, std::size_t bytes, const char* path) {
  auto* b = static_cast<char*>(p);
  while (bytes) {
    const std::size_t chunk = std::min<std::size_t>(bytes, std::size_t(1) << 28);
    if (std::fread(b, 1, chunk, f) != chunk) throw Error(std::string("truncated sidecar ") + path);
    b += chunk;
    bytes -= chunk;
  }
}

void check_info(const nm_sidecar_info& in) {
  if (in.K < 0 || in.K > 32) throw Error("sidecar: compartment count must be in [0, 32]");
  if (in.n_tets > (std::uint64_t(1) << 40) || in.n_nodes > (std::uint64_t(1) << 40)) throw Error("sidecar: sizes out of range");
}

void write_sidecar(const char* path, const nm_sidecar_info& info, const int* labels, const std::uint32_t* masks) {
  check_info(info);
  if (info.n_tets && !labels) throw Error("sidecar: null labels");
  if (info.has_masks && info.n_nodes && !masks) throw Error("sidecar: has_masks set but masks is null");
  const std::string tmp = std::string(path) + ".tmp";
  {
    File f;
    f.f = std::fopen(tmp.c_str(), "wb");
    if (!f.f) throw Error(std::string("cannot open ") + tmp + " for writing");
    const std::uint32_t ib = sizeof(nm_sidecar_info);
    write_all(f.f, kMagic, 8, path);
    write_all(f.f, &ib, 4, path);
    write_all(f.f, &info, sizeof info, path);
    write_all(f.f, labels, info.n_tets * sizeof(int), path);
    if (info.has_masks) write_all(f.f, masks, info.n_nodes * sizeof(std::uint32_t), path);
    const std::uint64_t h = payload_hash(labels, info.n_tets, info.has_masks ? masks : nullptr, info.n_nodes);
    write_all(f.f, &h, 8, path);
    if (std::fflush(f.f) != 0) throw Error(std::string("cannot write ") + tmp);
  }
  if (std::rename(tmp.c_str(), path) != 0) throw Error(std::string("cannot rename ") + tmp + " to " + path);
}

void read_sidecar_info(std::FILE* f, const char* path, nm_sidecar_info& info) {
  char magic[8];
  std::uint32_t ib = 0;
  read_all(f, magic, 8, path);
  if (std::memcmp(magic, kMagic, 8) != 0) throw Error(std::string(path) + " is not a nestmesh label sidecar");
  read_all(f, &ib, 4, path);
  if (ib != sizeof(nm_sidecar_info)) throw Error(std::string(path) + ": unsupported sidecar header size");
  read_all(f, &info, sizeof info, path);
  check_info(info);
}

}  // namespace

extern "C" {

int nm_mesh_fingerprint(const double* nodes, size_t n, const uint32_t* tets, size_t nt, uint64_t* fp) {
  return guarded([&] {
    if (!fp) throw Error("null output");
    *fp = combine(host_hash_words(nodes, 3 * n * sizeof(double), kSeedNodes),
                  host_hash_words(tets, 4 * nt * sizeof(std::uint32_t), kSeedTets), n, nt);
  });
}

int nm_mesh_fingerprint_device(nm_ctx* c, const double* d_nodes, size_t n, const uint32_t* d_tets, size_t nt,
                               uint64_t* fp, void* stream) {
  return guarded([&] {
    if (!c || !fp) throw Error("null argument");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->pick(stream);
    auto* acc = c->word.as<unsigned long long>(2);
    NM_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), st));
    // nodes: 3n doubles = 3n words; tets: 4nt uint32 = 2nt words
    if (n)
      k_hash_words<<<grid_for(3 * n, 256, c->sm_count * 8), 256, 0, st>>>(reinterpret_cast<const std::uint64_t*>(d_nodes),
                                                                          3 * n, kSeedNodes, acc);
    if (nt)
      k_hash_words<<<grid_for(2 * nt, 256, c->sm_count * 8), 256, 0, st>>>(reinterpret_cast<const std::uint64_t*>(d_tets),
                                                                           2 * nt, kSeedTets, acc + 1);
    NM_CUDA(cudaGetLastError());
    unsigned long long h[2];
    NM_CUDA(cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, st));
    NM_CUDA(cudaStreamSynchronize(st));
    *fp = combine(h[0], h[1], n, nt);
  });
}

int nm_sidecar_write(const char* path, const nm_sidecar_info* info, const int* labels, const uint32_t* masks) {
  return guarded([&] {
    if (!path || !info) throw Error("null argument");
    write_sidecar(path, *info, labels, masks);
  });
}

int nm_sidecar_read_info(const char* path, nm_sidecar_info* info) {
  return guarded([&] {
    if (!path || !info) throw Error("null argument");
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) throw Error(std::string("cannot open ") + path);
    read_sidecar_info(f.f, path, *info);
  });
}

int nm_sidecar_read(const char* path, nm_sidecar_info* info, int* labels, uint32_t* masks) {
  return guarded([&] {
    if (!path || !info) throw Error("null argument");
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) throw Error(std::string("cannot open ") + path);
    read_sidecar_info(f.f, path, *info);
    std::vector<int> lab_tmp;
    int* lab = labels;
    if (!lab) {
      lab_tmp.resize(info->n_tets);
      lab = lab_tmp.data();
    }
    read_all(f.f, lab, info->n_tets * sizeof(int), path);
    std::vector<std::uint32_t> m_tmp;
    std::uint32_t* m = nullptr;
    if (info->has_masks) {
      m = masks;
      if (!m) {
        m_tmp.resize(info->n_nodes);
        m = m_tmp.data();
      }
      read_all(f.f, m, info->n_nodes * sizeof(std::uint32_t), path);
    }
    std::uint64_t h = 0;
    read_all(f.f, &h, 8, path);
    if (h != payload_hash(lab, info->n_tets, m, info->n_nodes))
      throw Error(std::string(path) + ": payload hash mismatch (corrupt sidecar)");
    if (std::fgetc(f.f) != EOF) throw Error(std::string(path) + ": trailing bytes after the payload");
  });
}

int nm_label_lattice_sidecar(nm_ctx* c, const double* origin, double h, int nx, int ny, int nz, double T,
                             const char* path, int with_masks, nm_sidecar_info* info_out, nm_stats* stats) {
  return guarded([&] {
    require_surfaces(c);
    if (!path || !origin) throw Error("null argument");
    if (!(h > 0.0) || nx < 1 || ny < 1 || nz < 1) throw Error("lattice cell size must be > 0 and counts >= 1");
    const std::size_t nn = static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1);
    const std::size_t nt = 5ull * nx * ny * nz;
    if (nn > 0xffffffffull) throw Error("lattice has more than 2^32 nodes");
    NM_CUDA(cudaSetDevice(c->opt.device));
    cudaStream_t st = c->stream;
    auto* d_nodes = c->pts.as<double>(3 * nn);
    auto* d_tets = c->tets.as<std::uint32_t>(4 * nt);
    auto* d_masks = c->masks.as<std::uint32_t>(nn);
    auto* d_labels = c->labels.as<int>(nt);
    if (nm_lattice_device(c, origin, h, nx, ny, nz, d_nodes, d_tets, st) != 0) throw Error(last_error());
    label_nodes_dev(c, d_nodes, nn, T, d_masks, nullptr, st, stats);
    label_tets_dev(c, d_tets, nt, d_masks, d_labels, st, stats, nn);
    nm_sidecar_info info{};
    info.n_nodes = nn;
    info.n_tets = nt;
    info.K = c->K;
    info.has_masks = with_masks ? 1 : 0;
    info.is_lattice = 1;
    for (int k = 0; k < 32; ++k) info.label_ids[k] = c->ids.id[k];
    info.threshold = T;
    for (int a = 0; a < 3; ++a) info.origin[a] = origin[a];
    info.h = h;
    info.n[0] = nx;
    info.n[1] = ny;
    info.n[2] = nz;
    if (nm_mesh_fingerprint_device(c, d_nodes, nn, d_tets, nt, &info.mesh_fingerprint, st) != 0)
      throw Error(last_error());
    // labels (and masks) into pinned staging, then straight to the file
    int* h_lab = nullptr;
    std::uint32_t* h_m = nullptr;
    NM_CUDA(cudaMallocHost(&h_lab, std::max<std::size_t>(nt, 1) * sizeof(int)));
    struct Pinned {
      void* p;
      ~Pinned() {
        if (p) cudaFreeHost(p);
      }
    } g1{h_lab}, g2{nullptr};
    NM_CUDA(cudaMemcpyAsync(h_lab, d_labels, nt * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (with_masks) {
      NM_CUDA(cudaMallocHost(&h_m, std::max<std::size_t>(nn, 1) * sizeof(std::uint32_t)));
      g2.p = h_m;
      NM_CUDA(cudaMemcpyAsync(h_m, d_masks, nn * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    }
    NM_CUDA(cudaStreamSynchronize(st));
    write_sidecar(path, info, h_lab, h_m);
    if (info_out) *info_out = info;
  });
}

}  // extern "C"
