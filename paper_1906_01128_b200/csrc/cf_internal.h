// Internal declarations shared by the libchainforge_b200 translation units.
#pragma once
#include "chainforge_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector>

namespace cf {

// Node layout of the reference (scenarios.py:20-28): 24-byte node {u32 nA@0, u32 nLnext@4,
// u64 A@8, u64 Lnext@16}; dense depth-D leaves are packed 12-byte {u32 nA@0, u64 A@4}.
constexpr uint32_t NODE_SIZE = 24, LEAF_NODE_SIZE = 12;
constexpr uint32_t OFF_NA = 0, OFF_NLNEXT = 4, OFF_A = 8, OFF_LNEXT = 16, LEAF_OFF_A = 4;
constexpr uint64_t NO_BAD = ~0ull;
// Leaf-kernel tile: 256 threads x 4 vectors x 16 B.  Host planners split work on this grain.
constexpr uint32_t SCALE_THREADS = 256;
constexpr uint32_t SCALE_UNROLL = 4;
constexpr uint64_t TILE_BYTES = uint64_t(SCALE_THREADS) * SCALE_UNROLL * 16;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void clear_error();

#define CF_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return ::cf::fail(CF_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                               \
  } while (0)

// Host<->device bulk copy whose host-side start is first brought to a 256-byte boundary by a
// small separate copy.  The copy engines lose ~13% of full-duplex throughput when a large
// transfer's host address is only 16-byte aligned, and splitting off the head recovers it
// (tools/duplex_probe.cu; profiles/r01_design_experiments.md "host alignment of DMA pieces").
inline cudaError_t copy_host_aligned(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t s) {
  const uintptr_t hp = reinterpret_cast<uintptr_t>(kind == cudaMemcpyHostToDevice ? src : dst);
  const size_t head = (256 - (hp & 255)) & 255;
  if (n < (size_t(1) << 20) || head == 0) return cudaMemcpyAsync(dst, src, n, kind, s);
  cudaError_t e = cudaMemcpyAsync(dst, src, head, kind, s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(static_cast<char*>(dst) + head, static_cast<const char*>(src) + head, n - head, kind, s);
}

#define CF_TRY(expr)            \
  do {                          \
    int r_ = (expr);            \
    if (r_ != CF_OK) return r_; \
  } while (0)

// Kernel launchers (cf_kernels.cu).  Each increments ctx->launches once per kernel launch.
int debug_info(uint64_t* out, int reset);
int launch_sm_copy(cf_ctx* ctx, void* dst, const void* src, uint64_t bytes, unsigned ctas, cudaStream_t s);
int launch_copy_list2(cf_ctx* ctx, const uint64_t* sa, const uint64_t* da, const uint64_t* ba, uint64_t na,
                      const uint64_t* sb, const uint64_t* db, const uint64_t* bb, uint64_t nb, cudaStream_t s);
int launch_check_resolved(cf_ctx* ctx, const uint64_t* ea, const uint32_t* cnt, const uint64_t* expect_off,
                          const uint32_t* cnt_plan, uint64_t image, uint64_t n, uint64_t* bad, cudaStream_t s);
int launch_copy_list(cf_ctx* ctx, const uint64_t* src, const uint64_t* dst, const uint64_t* bytes, uint64_t n,
                     cudaStream_t s);
int launch_checksum(cf_ctx* ctx, const uint64_t* addr, const uint64_t* words, const uint64_t* tile_lo, uint64_t nranges,
                    uint64_t ntiles, uint64_t* out, cudaStream_t s);
// Fault tags: a kernel that finds a bad site / chain / part raises min(tag | index) into the
// error word; the pipelined window reads one sticky word and maps the phase to the reference's
// exception (attach / detach -> AttachOutsideArena, chain walk / leaf span -> WildAccess).  The
// synchronous single-phase operations pass tag 0 (plain index).
constexpr uint64_t FAULT_SHIFT = 62;
constexpr uint64_t FAULT_ATTACH = 0ull << FAULT_SHIFT, FAULT_RESOLVE = 1ull << FAULT_SHIFT,
                   FAULT_SCALE = 2ull << FAULT_SHIFT, FAULT_DETACH = 3ull << FAULT_SHIFT;
constexpr uint64_t FAULT_INDEX_MASK = (1ull << FAULT_SHIFT) - 1;
int launch_relocate(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites,
                    uint64_t nsites, uint64_t from, uint64_t to, uint64_t* bad, cudaStream_t s,
                    const uint32_t* idx = nullptr, uint64_t tag = 0);
// One-CTA attach + resolve for small site/target counts (see SMALL_FUSED).
constexpr uint64_t SMALL_FUSED = 4096;
int launch_attach_resolve(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                          uint64_t from, uint64_t to, const cf_chain_shape& sh, const uint64_t* root, const int32_t* level,
                          const uint32_t* ordinal, uint64_t ntargets, uint64_t* ea, uint32_t* count, uint64_t* bad,
                          cudaStream_t s, uint64_t res_tag = 0);
// A resolve range whose targets are consecutive ordinals ord0, ord0 + 1, ... at one level >= 1 of a
// single dense tree, owning their A field exactly when it is misaligned (own_misaligned): the
// resolver derives level / ordinal / ownership instead of reading the tables.
struct UniTargets {
  uint32_t on, level, ord0, own_misaligned;
  uint64_t qmagic;   // floor((2^64 - 1) / q) + 1: n / q == __umul64hi(n, qmagic) for every u32 n (q >= 2)
};
// Leaf-owned relocation (one-step windows over a uniform range of dense leaf targets, RESOLVED
// mode, small equal parts): the leaf kernel's group warps find each target's leaf record from its
// parent's child block (parent table filled by k_attach_parents), attach the record's A field,
// stream the array and detach the field again -- no per-target EA table, no per-leaf sites in the
// attach / detach lists.  Part p of the step is target position p, elements [0, n_el); group g
// holds parts [g gp, min((g + 1) gp, nt)).
struct LeafOwn {
  const uint64_t* parent;   // device: child block of parent ordinal p_first + p (0 = broken chain)
  uint32_t on, level, o0, p_first, nparents, n_el, gp, nt;
  uint64_t qmagic, from, to, total;
  uint32_t keep_attached;   // diagnostics: skip the detach (CF_WIN_DEBUG_KEEP_LEAF_ATTACHED)
};
int launch_attach_parents(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                          uint64_t from, uint64_t to, const cf_chain_shape& sh, const LeafOwn& own, uint64_t* parent,
                          uint64_t* bad, cudaStream_t s);
// Attach and resolve side by side in one launch (8-byte aligned pointer fields only).
int launch_attach_resolve_wide(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                               uint64_t from, uint64_t to, const cf_chain_shape& sh, const uint64_t* root,
                               const int32_t* level, const uint32_t* ordinal, uint64_t ntargets, uint64_t* ea,
                               uint32_t* count, uint64_t* bad, cudaStream_t s, uint64_t res_tag = 0,
                               const UniTargets* uni = nullptr);
int launch_resolve(cf_ctx* ctx, const uint8_t* image, const cf_chain_shape& sh, const uint64_t* root,
                   const int32_t* level, const uint32_t* ordinal, uint64_t n, uint64_t* ea,
                   uint32_t* count, uint64_t* bad, cudaStream_t s, uint64_t tag = 0);
// A relocation job that can ride along in a leaf-kernel launch (extra CTAs).
struct RelocArgs {
  uint8_t* image;
  uint64_t total;
  const uint64_t* sites;
  const uint32_t* idx;   // optional indirection: site = sites[idx[i]]
  uint64_t n;
  uint64_t from, to;
  uint64_t tag = 0;      // fault tag (FAULT_DETACH when it rides in a window's leaf launch)
};
int launch_scale(cf_ctx* ctx, int elem, int mode, const uint8_t* image, const cf_chain_shape& sh,
                 const uint64_t* root, const int32_t* level, const uint32_t* ordinal, const uint64_t* ea,
                 const uint32_t* count, const cf_scale_work& work, double scale, uint64_t* bad,
                 cudaStream_t s, const RelocArgs* fused_reloc = nullptr, uint64_t tag = 0, bool pdl = false,
                 const LeafOwn* own = nullptr);
int launch_naive_fixup(cf_ctx* ctx, const uint64_t* field_host, const uint64_t* target_host,
                       uint64_t nsites, const uint64_t* map_host, const uint64_t* map_size,
                       const uint64_t* map_dev, uint64_t nmap, uint64_t* bad, cudaStream_t s);
int launch_fill_u64(cf_ctx* ctx, uint64_t* p, uint64_t value, uint64_t n, cudaStream_t s);
// L2 eviction by a read pass over a device buffer (clean lines: nothing to write back later).
int launch_evict_read(cf_ctx* ctx, const void* buf, uint64_t bytes, cudaStream_t s);
// (lo, hi) byte segments copied src+lo -> dst+lo by the SMs (mapped host memory allowed).
int launch_seg_copy(cf_ctx* ctx, const uint64_t* segs, uint64_t n, const uint8_t* src, uint8_t* dst, cudaStream_t s);

inline uint64_t tiles_for(uint64_t elems, int elem) {
  const uint64_t per = TILE_BYTES / uint64_t(elem);
  return (elems + per - 1) / per;
}

// Small parts (< one tile) are packed into groups of at most GROUP_BYTES / GROUP_PARTS and
// processed one warp per part, so 1M 1 KiB leaves do not become 1M mostly idle CTAs.
#ifndef CF_GROUP_KB
#define CF_GROUP_KB 32
#endif
constexpr uint64_t GROUP_BYTES = uint64_t(CF_GROUP_KB) << 10;
#ifndef CF_GROUP_PARTS
#define CF_GROUP_PARTS 32
#endif
constexpr uint32_t GROUP_PARTS = CF_GROUP_PARTS;

// Host-side builder of the leaf-kernel work list (see cf_scale_work in the header).
struct ScaleWork {
  int elem = 4;
  std::vector<uint32_t> parts;      // (target, elem_begin, elem_end) per part
  std::vector<uint64_t> tile_base;  // first tile of every big part (big parts only)
  std::vector<uint32_t> groups;     // (first part, end part) per group
  uint64_t next_tile = 0;

  uint64_t nparts() const { return parts.size() / 3; }
  uint64_t ngroups() const { return groups.size() / 2; }

  // Append one launch segment from (target, begin, end) triples: big parts first (one CTA per
  // 16 KiB tile), then the small parts packed into groups.  Device pointers are left null.
  cf_scale_work append(const std::vector<uint64_t>& tri) {
    cf_scale_work w{};
    const uint64_t tile_elems = TILE_BYTES / uint64_t(elem);
    w.big_begin = nparts();
    w.tb_begin = tile_base.size();
    w.tile_begin = next_tile;
    for (size_t i = 0; i < tri.size(); i += 3) {
      if (tri[i + 2] - tri[i + 1] < tile_elems) continue;
      parts.insert(parts.end(), {uint32_t(tri[i]), uint32_t(tri[i + 1]), uint32_t(tri[i + 2])});
      tile_base.push_back(next_tile);
      next_tile += tiles_for(tri[i + 2] - tri[i + 1], elem);
    }
    w.big_count = nparts() - w.big_begin;
    w.tile_end = next_tile;
    w.group_begin = ngroups();
    uint64_t first = nparts(), bytes = 0;
    for (size_t i = 0; i < tri.size(); i += 3) {
      const uint64_t n = tri[i + 2] - tri[i + 1];
      if (n >= tile_elems || n == 0) continue;
      const uint64_t b = n * uint64_t(elem);
      if (nparts() > first && (bytes + b > GROUP_BYTES || nparts() - first >= GROUP_PARTS)) {
        groups.insert(groups.end(), {uint32_t(first), uint32_t(nparts())});
        first = nparts();
        bytes = 0;
      }
      parts.insert(parts.end(), {uint32_t(tri[i]), uint32_t(tri[i + 1]), uint32_t(tri[i + 2])});
      bytes += b;
    }
    if (nparts() > first) groups.insert(groups.end(), {uint32_t(first), uint32_t(nparts())});
    w.group_end = ngroups();
    return w;
  }
};

}  // namespace cf

struct cf_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t compute = nullptr;
  cudaStream_t d2h = nullptr;
  std::vector<cudaStream_t> h2d;
  uint64_t* d_bad = nullptr;   // device scratch error word
  uint64_t* h_bad = nullptr;   // pinned mirror
  std::atomic<uint64_t> launches{0};
  // grow-only device scratch for the synchronous reference-named operations (avoids a
  // cudaMalloc/cudaFree -- and the implicit device sync of cudaFree -- per call)
  void* scratch = nullptr;
  uint64_t scratch_bytes = 0;
};

struct cf_tree {
  cf_spec spec{};
  uint64_t total = 0, root_off = 0, payload_bytes = 0, served = 0;
  std::vector<uint64_t> alloc_off, alloc_size;
  std::vector<int64_t> alloc_array;   // array index of an allocation, -1 for node blocks
  std::vector<uint64_t> node_off;
  std::vector<int32_t> node_level;
  std::vector<uint32_t> node_size;
  std::vector<uint32_t> node_na;      // value of the nA field
  std::vector<int64_t> node_nlnext;   // value of nLnext, -1 when the node has no such field
  std::vector<int32_t> arr_level;
  std::vector<uint64_t> arr_owner, arr_off, arr_count, arr_ordinal, arr_tree, arr_root;
  std::vector<uint64_t> site_off, site_target, site_sorted;
  std::vector<uint64_t> tree_root;
  // per tree, per level: node offsets by ordinal (pre-order within a level)
  std::vector<std::vector<std::vector<uint64_t>>> level_nodes;
  // per tree, per level: ordinal of level_nodes[tree][level][0] (non-zero below the cut level
  // of a subtree shard, whose levels hold one contiguous ordinal range)
  std::vector<std::vector<uint64_t>> level_base;
};

// RAII: make ctx's device current on this thread.
struct CfDevice {
  int prev = -1;
  explicit CfDevice(const cf_ctx* c) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (c && prev != c->device) cudaSetDevice(c->device);
  }
  ~CfDevice() {}
};
