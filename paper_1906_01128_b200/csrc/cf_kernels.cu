// sm_100a kernels of the deep-copy hot path.
//
//   k_relocate    attach / detach fix-ups over the relocation table
//                 (Machine.marshal_transfer_and_attach site loop, memory.py:316-323;
//                  Machine.demarshal site loop, memory.py:337-344)
//   k_resolve     pointerchain: walk each target chain once, emit its effective address
//                 (targeted_arrays, scenarios.py:270-284, on the device)
//   k_attach_resolve / _wide / _uni
//                 attach and resolve in one launch: one CTA (small windows), side by side
//                 (aligned fields), memory-parallel over uniform ordinal ranges (32 U targets
//                 per warp, parents walked one per lane)
//   k_attach_parents
//                 leaf-owned steps: attach the step's sites || resolve the owned range's parents
//                 into the parent table (the leaf kernel does the rest of each chain)
//   k_scale       leaf kernel x *= s (_scale_block, harness.py:307-309) in two modes:
//                   RESOLVED  reads the effective-address table (pointerchain)
//                   CHASE     re-walks the chain per 16-byte access with non-hoistable loads
//                             (Listing 2 per-iteration chain)
//                 and, for leaf-owned steps (RESOLVED), a path whose warps find each leaf record
//                 from the parent table, attach its A field, stream the array and detach it
//   k_naive_fixup per-object deep-copy fix-ups through a sorted interval map
//                 (naive_deep_copy + AddressMap.translate, memory.py:349-365, 409-419)
//   k_seg_copy / k_copy_list
//                 zero-copy moves over mapped pinned host memory: hoisted node pages of scattered
//                 layouts, and per-object copies of small objects (naive / pointerchain schemes)
//   k_checksum    per-leaf checksums for the multi-GPU result gather
//   k_sm_copy     SM-driven bulk copy (host-link experiments only)
//   k_evict_read  L2 eviction by a read pass (benchmark plumbing for L2-sized working sets)
//
// All of these are HBM/latency-bound integer or streaming work: no tensor cores.  The leaf
// kernel is the HBM-roofline kernel: 16-byte vector loads/stores with streaming cache hints,
// 4 independent vectors in flight per thread, a persistent grid sized to 148 SMs x resident
// CTAs, and a flattened (target, tile) work list so 64 huge leaves and 1M small leaves both
// balance.  Pointer fields in the packed reference layout -- and every other dense leaf record's
// A field even in aligned arenas (12-byte records) -- sit at 4 (mod 8); every 64-bit field access
// goes through ld_u64_any/st_u64_any (2 x u32 when misaligned), so a field may only be read
// concurrently with its relocation when all fields are 8-byte aligned (k_attach_resolve_wide).
// f64 arrays at 4 (mod 8) stream aligned 16-byte words (scale_f64_shifted).
#include "cf_internal.h"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

// tuning knobs (design experiments: tools/build_variants.sh)
#ifndef CF_SCALE_MINB
#define CF_SCALE_MINB 6
#endif
#ifndef CF_GROUP_MINB
#define CF_GROUP_MINB CF_SCALE_MINB
#endif
#ifndef CF_GROUP_U
#define CF_GROUP_U 4
#endif
#ifndef CF_GROUP_WARP
#define CF_GROUP_WARP 1
#endif
#ifndef CF_GROUP_WARP_U
#define CF_GROUP_WARP_U 4
#endif
#ifndef CF_RELOC_FASTMAP
#define CF_RELOC_FASTMAP 1
#endif
#ifndef CF_PDL_WAIT_ALWAYS
#define CF_PDL_WAIT_ALWAYS 0
#endif
#ifndef CF_OWN_MINB
#define CF_OWN_MINB 4
#endif
#ifndef CF_OWN_U
#define CF_OWN_U 4
#endif
#ifndef CF_OWN_CONTIG
#define CF_OWN_CONTIG 0
#endif
#ifndef CF_ROW_ALIGN
#define CF_ROW_ALIGN 128
#endif
#ifndef CF_SHIFT_ALIGN
#define CF_SHIFT_ALIGN 128
#endif


namespace cf {
namespace {

__device__ __forceinline__ uint64_t ld_u64_any(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 7) == 0) return *reinterpret_cast<const uint64_t*>(p);
  if ((a & 3) == 0) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
    return uint64_t(w[0]) | (uint64_t(w[1]) << 32);
  }
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

__device__ __forceinline__ void st_u64_any(uint8_t* p, uint64_t v) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 7) == 0) {
    *reinterpret_cast<uint64_t*>(p) = v;
  } else if ((a & 3) == 0) {
    uint32_t* w = reinterpret_cast<uint32_t*>(p);
    w[0] = uint32_t(v);
    w[1] = uint32_t(v >> 32);
  } else {
    for (int i = 0; i < 8; ++i) p[i] = uint8_t(v >> (8 * i));
  }
}

__device__ __forceinline__ uint32_t ld_u32_any(const uint8_t* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) return *reinterpret_cast<const uint32_t*>(p);
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// Non-hoistable chain loads for CHASE mode: asm volatile keeps one load per access in SASS
// (LDG.E.64.CONSTANT), the per-iteration dereference cost the paper measures.
__device__ __forceinline__ uint64_t ld_chain_u64(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 7) == 0) {
    uint64_t v;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
  }
  uint32_t lo, hi;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(lo) : "l"(p));
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(hi) : "l"(p + 4));
  return uint64_t(lo) | (uint64_t(hi) << 32);
}

__device__ __forceinline__ void raise_bad(uint64_t* bad, uint64_t idx) {
  if (bad) atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)idx);
}

// ---------------------------------------------------------------- relocation (attach/detach)
// `tag` (bits 62-63 of the error word, CF_FAULT_* << 62) names the phase that faulted, so one
// sticky word per window still maps onto the reference's exception for that phase.
__device__ __forceinline__ void relocate_one(uint8_t* __restrict__ image, uint64_t total,
                                             const uint64_t* __restrict__ sites, uint64_t i, uint64_t from,
                                             uint64_t to, uint64_t* bad, const uint32_t* __restrict__ idx = nullptr,
                                             uint64_t tag = 0) {
  const uint64_t s = sites[idx ? idx[i] : i];  // coalesced table read
  if (s + 8 > total) { raise_bad(bad, i | tag); return; }
  uint8_t* p = image + s;
  const uint64_t v = ld_u64_any(p);
  const uint64_t d = v - from;  // wraps when v < from
  if (d >= total) { raise_bad(bad, i | tag); return; }
  st_u64_any(p, to + d);
}

__global__ void __launch_bounds__(256) k_relocate(uint8_t* __restrict__ image, uint64_t total,
                                                  const uint64_t* __restrict__ sites,
                                                  const uint32_t* __restrict__ idx, uint64_t n,
                                                  uint64_t from, uint64_t to, uint64_t* bad, uint64_t tag) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    relocate_one(image, total, sites, i, from, to, bad, idx, tag);
}

// ---------------------------------------------------------------- chain walk
struct Walk {
  const uint8_t* node;  // terminal node (nullptr on failure)
  bool leaf;
};

// A pointer field read while the attach kernel may be rewriting it concurrently (8-byte aligned
// fields only: the 64-bit store is single-copy atomic): host values are translated on the fly.
__device__ __forceinline__ uint64_t xlate(uint64_t v, uint64_t from, const uint8_t* image, uint64_t bytes) {
  return (from && v - from < bytes) ? reinterpret_cast<uint64_t>(image) + (v - from) : v;
}

// A record of `size` bytes at address `next` lies wholly inside the image (a corrupted chain link
// is reported, never followed past the image's end).
__device__ __forceinline__ bool rec_inside(uint64_t next, const uint8_t* image, uint64_t bytes, uint64_t size) {
  return bytes >= size && next - reinterpret_cast<uint64_t>(image) <= bytes - size;
}

template <bool CHASE>
__device__ __forceinline__ Walk walk_chain(const uint8_t* image, const cf_chain_shape& sh, uint64_t root_off,
                                           int level, uint64_t ordinal, uint64_t xlate_from = 0) {
  const uint8_t* p = image + root_off;
  const bool dense = sh.kind == CF_DENSE;
  // base-q digits of the ordinal, most significant first: rem / q^(L-l), rem %= q^(L-l).  Ordinals
  // are u32 (window tables), so the divisions run in 32 bits -- 64-bit integer division is a long
  // emulated sequence and made the 1M-chain resolve instruction-bound (C4: 17 us).
  uint32_t qpow = 1, rem = uint32_t(ordinal) & 0x7FFFFFFFu;   // bit 31: owned-attach flag (wide kernel)
  if (dense)
    for (int l = 1; l < level; ++l) qpow *= sh.q;
  for (int l = 1; l <= level; ++l) {
    const uint64_t blk = xlate(CHASE ? ld_chain_u64(p + OFF_LNEXT) : ld_u64_any(p + OFF_LNEXT), xlate_from,
                               image, sh.image_bytes);
    uint64_t child = 0, digit = 0;
    if (dense) {
      child = (l < sh.depth) ? NODE_SIZE : LEAF_NODE_SIZE;
      const uint32_t d = rem / qpow;
      rem -= d * qpow;
      digit = d;
      qpow = qpow > 1 ? qpow / sh.q : 1;
    }
    const uint64_t next = blk + digit * child;
    if (!rec_inside(next, image, sh.image_bytes, (dense && l == sh.depth) ? LEAF_NODE_SIZE : NODE_SIZE))
      return {nullptr, false};
    p = reinterpret_cast<const uint8_t*>(next);
  }
  return {p, dense && level == sh.depth};
}

// Warp-cooperative walk (pointerchain resolve, RESOLVED mode): consecutive targets mostly share
// their parent node (C4: 100 leaves per level-2 node, targets sorted by ordinal), so the lanes of a
// warp are grouped by (root, level, parent ordinal) with __match_any_sync, one leader per group
// walks the L - 1 hops to the parent and reads its Lnext, and every lane then indexes its own
// record in that child block.  Dependent loads per chain drop from L to ~1 (the record's fields);
// the result equals walk_chain's.  All lanes of the warp must call it (inactive lanes with
// active = false); host pointers met on the way are translated as walk_chain does (xlate_from).
__device__ __forceinline__ Walk walk_chain_coop(const uint8_t* image, const cf_chain_shape& sh, uint64_t root_off,
                                                int level, uint32_t ordinal, uint64_t xlate_from, bool active) {
  const unsigned am = __ballot_sync(0xffffffffu, active);
  if (!active) return {nullptr, false};
  const unsigned lane = threadIdx.x & 31;
  const bool dense = sh.kind == CF_DENSE;
  const uint32_t q = dense ? sh.q : 1u;
  const uint32_t rem = ordinal & 0x7FFFFFFFu;   // bit 31: owned-attach flag (wide kernel)
  const uint32_t parent = level >= 1 ? rem / q : 0u;
  const unsigned grp = __match_any_sync(am, root_off) &
                       __match_any_sync(am, (uint64_t(uint32_t(level)) << 32) | parent);
  const int leader = __ffs(grp) - 1;
  uint64_t blk = 0;
  int ok = 1;
  if (int(lane) == leader && level >= 1) {
    // the parent: L - 1 hops with the parent's ordinal, then its Lnext (the child block)
    Walk pw = walk_chain<false>(image, sh, root_off, level - 1, parent, xlate_from);
    if (pw.node == nullptr || pw.leaf) {
      ok = 0;
    } else {
      blk = xlate(ld_u64_any(pw.node + OFF_LNEXT), xlate_from, image, sh.image_bytes);
    }
  }
  blk = __shfl_sync(am, blk, leader);
  ok = __shfl_sync(am, ok, leader);
  if (level < 1) return {image + root_off, dense && sh.depth == 0};
  if (!ok) return {nullptr, false};
  const uint64_t child = dense ? ((level < sh.depth) ? NODE_SIZE : LEAF_NODE_SIZE) : 0;
  const uint64_t next = blk + uint64_t(rem - parent * q) * child;
  if (!rec_inside(next, image, sh.image_bytes, (dense && level == sh.depth) ? LEAF_NODE_SIZE : NODE_SIZE))
    return {nullptr, false};
  return {reinterpret_cast<const uint8_t*>(next), dense && level == sh.depth};
}

__global__ void __launch_bounds__(128) k_resolve(const uint8_t* __restrict__ image, cf_chain_shape sh,
                                                 const uint64_t* __restrict__ root,
                                                 const int32_t* __restrict__ level,
                                                 const uint32_t* __restrict__ ordinal, uint64_t n,
                                                 uint64_t* __restrict__ ea, uint32_t* __restrict__ count,
                                                 uint64_t* bad, uint64_t tag) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool act = i < n;
  Walk w = walk_chain_coop(image, sh, act ? (root ? root[i] : sh.root_off) : 0, act ? level[i] : 0,
                           act ? ordinal[i] : 0, 0, act);
  if (!act) return;
  if (!w.node) {
    ea[i] = 0;
    count[i] = 0;
    raise_bad(bad, i | tag);
    return;
  }
  ea[i] = ld_u64_any(w.node + (w.leaf ? LEAF_OFF_A : OFF_A));
  count[i] = ld_u32_any(w.node + OFF_NA);
}

// Small windows (C2: 85 sites, 64 chains): attach and resolve in ONE CTA -- the barrier between
// them is a __syncthreads instead of a kernel boundary.
__global__ void __launch_bounds__(1024) k_attach_resolve(uint8_t* __restrict__ image, uint64_t total,
                                                         const uint64_t* __restrict__ sites, uint64_t nsites,
                                                         uint64_t from, uint64_t to, cf_chain_shape sh,
                                                         const uint64_t* __restrict__ root,
                                                         const int32_t* __restrict__ level,
                                                         const uint32_t* __restrict__ ordinal, uint64_t ntargets,
                                                         uint64_t* __restrict__ ea, uint32_t* __restrict__ count,
                                                         uint64_t* bad, uint64_t res_tag) {
  for (uint64_t i = threadIdx.x; i < nsites; i += blockDim.x) relocate_one(image, total, sites, i, from, to, bad);
  __syncthreads();
  for (uint64_t i0 = 0; i0 < ntargets; i0 += blockDim.x) {   // every lane runs every round (warp-collective walk)
    const uint64_t i = i0 + threadIdx.x;
    const bool act = i < ntargets;
    Walk w = walk_chain_coop(image, sh, act ? (root ? root[i] : sh.root_off) : 0, act ? level[i] : 0,
                             act ? ordinal[i] : 0, 0, act);
    if (!act) continue;
    if (!w.node) {
      ea[i] = 0;
      count[i] = 0;
      raise_bad(bad, i | res_tag);
      continue;
    }
    ea[i] = ld_u64_any(w.node + (w.leaf ? LEAF_OFF_A : OFF_A));
    count[i] = ld_u32_any(w.node + OFF_NA);
  }
}

// Large windows on an aligned arena (C4: 1.02M sites, 1M chains): attach and resolve in ONE
// launch, side by side -- CTAs [0, att_blocks) relocate sites, the rest resolve chains,
// translating any host pointer they meet that the attach CTAs have not rewritten yet (8-byte
// aligned fields: one atomic access).  A target whose ordinal carries bit 31 owns its A field
// (a 4-mod-8 leaf field attached in this step, left out of the attach CTAs' list): its resolver
// attaches it, so no misaligned field is ever read while another thread writes it.
// Uniform resolve range (UniTargets.on): the step's targets are consecutive ordinals ord0 + i at
// one level >= 1 of a single dense tree (C4: the 1M leaves, C2: the 64 leaves), and a target owns
// its A field exactly when that field is misaligned (own_misaligned).  The resolver then needs no
// level / ordinal table reads and no __match_any_sync: lanes sharing a parent are a contiguous
// run (leader = lane - ordinal % q, clipped to lane 0), one leader per run walks to the parent,
// every lane indexes its record in the parent's child block.
__device__ __forceinline__ Walk walk_uniform(const uint8_t* image, const cf_chain_shape& sh, const UniTargets& u,
                                             uint64_t i, uint64_t xlate_from) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t q = sh.q;
  const uint32_t ord = u.ord0 + uint32_t(i);
  const uint32_t parent = q > 1 ? uint32_t(__umul64hi(uint64_t(ord), u.qmagic)) : ord;   // ord / q
  const uint32_t j = ord - parent * q;
  const int lead = max(0, int(lane) - int(j));
  uint64_t blk = 0;
  int ok = 1;
  if (int(lane) == lead) {
    const Walk pw = walk_chain<false>(image, sh, sh.root_off, int(u.level) - 1, parent, xlate_from);
    if (pw.node == nullptr || pw.leaf) ok = 0;
    else blk = xlate(ld_u64_any(pw.node + OFF_LNEXT), xlate_from, image, sh.image_bytes);
  }
  blk = __shfl_sync(0xffffffffu, blk, lead);
  ok = __shfl_sync(0xffffffffu, ok, lead);
  if (!ok) return {nullptr, false};
  const bool leaf = int(u.level) == int(sh.depth);
  const uint64_t next = blk + uint64_t(j) * (leaf ? LEAF_NODE_SIZE : NODE_SIZE);
  if (!rec_inside(next, image, sh.image_bytes, leaf ? LEAF_NODE_SIZE : NODE_SIZE)) return {nullptr, false};
  return {reinterpret_cast<const uint8_t*>(next), leaf};
}

__global__ void __launch_bounds__(256) k_attach_resolve_wide(uint8_t* __restrict__ image, uint64_t total,
                                                             const uint64_t* __restrict__ sites, uint64_t nsites,
                                                             uint64_t from, uint64_t to, cf_chain_shape sh,
                                                             const uint64_t* __restrict__ root,
                                                             const int32_t* __restrict__ level,
                                                             const uint32_t* __restrict__ ordinal, uint64_t ntargets,
                                                             uint64_t* __restrict__ ea, uint32_t* __restrict__ count,
                                                             uint64_t* bad, unsigned att_blocks, uint64_t res_tag,
                                                             UniTargets uni) {
  if (blockIdx.x < att_blocks) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nsites) relocate_one(image, total, sites, i, from, to, bad);
    return;
  }
  const uint64_t i = uint64_t(blockIdx.x - att_blocks) * blockDim.x + threadIdx.x;
  const bool act = i < ntargets;
  uint32_t od;
  Walk w;
  if (uni.on) {   // warp-uniform branch: every lane of the warp takes it
    w = walk_uniform(image, sh, uni, i, from);
    if (!act) return;
    if (!w.node) {
      ea[i] = 0;
      count[i] = 0;
      raise_bad(bad, i | res_tag);
      return;
    }
    // the record's A field: 8-byte aligned -> one 64-bit load (an attach CTA may be rewriting
    // it); at 4 mod 8 -> this thread owns it (no other reader or writer): two u32 accesses
    uint32_t* fa = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(w.node) + (w.leaf ? LEAF_OFF_A : OFF_A));
    const bool mis = (reinterpret_cast<uintptr_t>(fa) & 7) != 0;
    uint64_t v = mis ? (uint64_t(fa[0]) | (uint64_t(fa[1]) << 32)) : *reinterpret_cast<const uint64_t*>(fa);
    if (mis && uni.own_misaligned) {   // owned field: attach it here
      const uint64_t dlt = v - from;
      if (dlt >= total) {
        ea[i] = 0;
        count[i] = 0;
        raise_bad(bad, i);
        return;
      }
      v = to + dlt;
      fa[0] = uint32_t(v);
      fa[1] = uint32_t(v >> 32);
    }
    ea[i] = xlate(v, from, image, sh.image_bytes);
    count[i] = *reinterpret_cast<const uint32_t*>(w.node + OFF_NA);
    return;
  } else {
    od = act ? ordinal[i] : 0;
    w = walk_chain_coop(image, sh, act ? (root ? root[i] : sh.root_off) : 0, act ? level[i] : 0, od, from, act);
  }
  if (!act) return;
  if (!w.node) {
    ea[i] = 0;
    count[i] = 0;
    raise_bad(bad, i | res_tag);
    return;
  }
  uint8_t* fa = const_cast<uint8_t*>(w.node) + (w.leaf ? LEAF_OFF_A : OFF_A);   // image is writable here
  uint64_t v = ld_u64_any(fa);
  if (od >> 31) {
    // owned field (4 mod 8, attached in this step): no attach CTA touches it and this thread is its
    // only reader, so the 2 x u32 read sees the untouched host value -- attach it here
    const uint64_t dlt = v - from;
    if (dlt >= total) {
      ea[i] = 0;
      count[i] = 0;
      raise_bad(bad, i);
      return;
    }
    v = to + dlt;
    st_u64_any(fa, v);
  }
  ea[i] = xlate(v, from, image, sh.image_bytes);
  count[i] = ld_u32_any(w.node + OFF_NA);
}

// Uniform resolve range (C4: 1M consecutive leaf ordinals) with memory-level parallelism: each
// warp takes a run of 32 x U consecutive targets.  Their parents are a handful of consecutive
// ordinals one level up; lane j walks parent p_first + j (all in parallel, the upper hops are L2
// hits), then every lane issues the U leaf-record loads of its targets back to back (independent,
// coalesced: consecutive records), owned A fields are attached, and the EA / count entries are
// stored.  The whole 1M-chain pass fits in about one wave with ~L + 1 dependent rounds per warp,
// against ~5 waves of one chain per thread (k_attach_resolve_wide's uniform branch).  Results are
// identical to walk_uniform's.  CTAs [0, att_blocks) relocate the other sites, as in the wide
// kernel.  The launch lets the next kernel (the leaf kernel) start its prologue early
// (programmatic dependent launch); that kernel waits for this grid's completion before reading.
constexpr int UNI_U = 8;
__global__ void __launch_bounds__(256) k_attach_resolve_uni(uint8_t* __restrict__ image, uint64_t total,
                                                            const uint64_t* __restrict__ sites, uint64_t nsites,
                                                            uint64_t from, uint64_t to, cf_chain_shape sh,
                                                            uint64_t ntargets, uint64_t* __restrict__ ea,
                                                            uint32_t* __restrict__ count, uint64_t* bad,
                                                            unsigned att_blocks, uint64_t res_tag, UniTargets uni,
                                                            unsigned per_warp_u) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x < att_blocks) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nsites) relocate_one(image, total, sites, i, from, to, bad);
    return;
  }
  const unsigned lane = threadIdx.x & 31;
  const unsigned U = per_warp_u;   // 32 U targets per warp, chosen so the run's parents fit 32 lanes
  const uint64_t wg = uint64_t(blockIdx.x - att_blocks) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t i0 = wg * 32 * U;
  if (i0 >= ntargets) return;   // warp-uniform
  const uint32_t q = sh.q;
  const uint32_t o_first = uni.ord0 + uint32_t(i0);
  const uint64_t rest = ntargets - i0;
  const uint32_t n_here = uint32_t(rest < uint64_t(32) * U ? rest : uint64_t(32) * U);
  auto divq = [&](uint32_t o) -> uint32_t { return q > 1 ? uint32_t(__umul64hi(uint64_t(o), uni.qmagic)) : o; };
  const uint32_t p_first = divq(o_first), p_last = divq(o_first + n_here - 1);
  // parents: lane j walks p_first + j
  uint64_t blk = 0;
  int ok = 1;
  if (lane <= p_last - p_first) {
    const Walk pw = walk_chain<false>(image, sh, sh.root_off, int(uni.level) - 1, p_first + lane, from);
    if (pw.node == nullptr || pw.leaf) ok = 0;
    else blk = xlate(ld_u64_any(pw.node + OFF_LNEXT), from, image, sh.image_bytes);
  }
  const bool leaf = int(uni.level) == int(sh.depth);
  const uint64_t child = leaf ? LEAF_NODE_SIZE : NODE_SIZE;
  const uint32_t off_a = leaf ? LEAF_OFF_A : OFF_A;
  const uint64_t img = reinterpret_cast<uint64_t>(image);
  uint32_t* fa[UNI_U];
  uint64_t v[UNI_U];
  uint32_t cnt[UNI_U];
  unsigned good = 0;   // bit u: target u of this lane has a record inside the image
#pragma unroll
  for (int u = 0; u < UNI_U; ++u) {
    fa[u] = nullptr;
    v[u] = 0;
    cnt[u] = 0;
    if (unsigned(u) >= U) continue;   // warp-uniform
    const uint32_t k = uint32_t(u) * 32 + lane;
    const uint32_t ord = o_first + k;
    const uint32_t par = divq(ord);
    const unsigned src = min(par - p_first, 31u);
    const uint64_t b = __shfl_sync(0xffffffffu, blk, src);
    const int pok = __shfl_sync(0xffffffffu, ok, src);
    if (k >= n_here) continue;
    const uint64_t rec = b + uint64_t(ord - par * q) * child;
    if (!pok || !rec_inside(rec, image, sh.image_bytes, child)) continue;
    fa[u] = reinterpret_cast<uint32_t*>(rec + off_a);
    good |= 1u << u;
  }
  // the U record loads of every lane, back to back (A: one 64-bit load when 8-byte aligned -- an
  // attach CTA may be rewriting it -- else 2 x u32 of an owned field)
#pragma unroll
  for (int u = 0; u < UNI_U; ++u) {
    if (!(good >> u & 1)) continue;
    const bool mis = (reinterpret_cast<uintptr_t>(fa[u]) & 7) != 0;
    v[u] = mis ? (uint64_t(fa[u][0]) | (uint64_t(fa[u][1]) << 32)) : *reinterpret_cast<const uint64_t*>(fa[u]);
    cnt[u] = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(fa[u]) - off_a + OFF_NA);
  }
#pragma unroll
  for (int u = 0; u < UNI_U; ++u) {
    const uint64_t k = uint64_t(u) * 32 + lane;
    if (unsigned(u) >= U || k >= n_here) continue;
    const uint64_t i = i0 + k;
    if (!(good >> u & 1)) {
      ea[i] = 0;
      count[i] = 0;
      raise_bad(bad, i | res_tag);
      continue;
    }
    uint64_t x = v[u];
    if (uni.own_misaligned && (reinterpret_cast<uintptr_t>(fa[u]) & 7) != 0) {   // owned field: attach it here
      const uint64_t dlt = x - from;
      if (dlt >= total) {
        ea[i] = 0;
        count[i] = 0;
        raise_bad(bad, i);
        continue;
      }
      x = to + dlt;
      fa[u][0] = uint32_t(x);
      fa[u][1] = uint32_t(x >> 32);
    }
    ea[i] = xlate(x, from, image, sh.image_bytes);
    count[i] = cnt[u];
  }
}

// Leaf-owned windows: CTAs [0, att_blocks) attach the step's non-owned sites (node-level pointer
// fields); the rest resolve each parent of the target range once -- walk to parent ordinal
// p_first + p at level L - 1 and store its child block (translated: an attach CTA may not have
// rewritten the field yet), 0 on a broken chain (fault index: the parent's first target).
__global__ void __launch_bounds__(256) k_attach_parents(uint8_t* __restrict__ image, uint64_t total,
                                                        const uint64_t* __restrict__ sites, uint64_t nsites,
                                                        uint64_t from, uint64_t to, cf_chain_shape sh, LeafOwn own,
                                                        uint64_t* __restrict__ parent, uint64_t* bad,
                                                        unsigned att_blocks) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x < att_blocks) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nsites) relocate_one(image, total, sites, i, from, to, bad);
    return;
  }
  const uint64_t p = uint64_t(blockIdx.x - att_blocks) * blockDim.x + threadIdx.x;
  if (p >= own.nparents) return;
  const uint32_t pord = own.p_first + uint32_t(p);
  const Walk pw = walk_chain<false>(image, sh, sh.root_off, int(own.level) - 1, pord, from);
  uint64_t blk = 0;
  if (pw.node != nullptr && !pw.leaf) blk = xlate(ld_u64_any(pw.node + OFF_LNEXT), from, image, sh.image_bytes);
  parent[p] = blk;
  if (blk == 0) {
    const uint64_t first = uint64_t(pord) * sh.q;
    raise_bad(bad, (first > own.o0 ? first - own.o0 : 0) | FAULT_RESOLVE);
  }
}

// ---------------------------------------------------------------- leaf kernel
template <typename T> struct Vec;
template <> struct Vec<float> {
  using V = float4;
  static constexpr int N = 4;
  __device__ static V ld(const V* p) { return __ldcs(p); }
  __device__ static void st(V* p, V v) { __stcs(p, v); }
  __device__ static V mul(V v, float s) { return make_float4(__fmul_rn(v.x, s), __fmul_rn(v.y, s), __fmul_rn(v.z, s), __fmul_rn(v.w, s)); }
};
template <> struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
  __device__ static V ld(const V* p) { return __ldcs(p); }
  __device__ static void st(V* p, V v) { __stcs(p, v); }
  __device__ static V mul(V v, double s) { return make_double2(__dmul_rn(v.x, s), __dmul_rn(v.y, s)); }
};

template <typename T>
__device__ __forceinline__ T scalar_ld(const uint8_t* p) {
  if constexpr (sizeof(T) == 8) {
    uint64_t u = ld_u64_any(p);
    return __longlong_as_double((long long)u);
  } else {
    return __uint_as_float(ld_u32_any(p));
  }
}
template <typename T>
__device__ __forceinline__ void scalar_st(uint8_t* p, T v) {
  if constexpr (sizeof(T) == 8) {
    st_u64_any(p, (uint64_t)__double_as_longlong(v));
  } else {
    if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) *reinterpret_cast<float*>(p) = v;
    else { uint32_t u = __float_as_uint(v); for (int i = 0; i < 4; ++i) p[i] = uint8_t(u >> (8 * i)); }
  }
}
template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }

// First leaf-kernel address fault seen (flag, target, address, count, image, bytes, level,
// ordinal) -- read by cf_debug_info for diagnosis.
__device__ uint64_t g_dbg[8];

struct ScaleArgs {
  const uint8_t* image;
  cf_chain_shape sh;
  const uint64_t* root;       // per-target root offsets (forests), nullptr = sh.root_off
  const int32_t* level;
  const uint32_t* ordinal;
  const uint64_t* ea;
  const uint32_t* count;
  cf_scale_work w;
  uint64_t* bad;
  uint64_t tag;      // fault tag of the leaf kernel's own checks
  RelocArgs reloc;   // optional fused relocation (reloc.n == 0: none)
  unsigned reloc_blocks;   // CTAs k * reloc_stride (k < reloc_blocks) run it, RELOC_U sites per thread
  unsigned reloc_stride;
  unsigned reloc_last;     // (reloc_blocks - 1) * reloc_stride: the last relocation CTA
  unsigned reloc_magic;    // ceil(2^32 / reloc_stride): umulhi(b, magic) is b / stride or one more
  unsigned pdl;            // launched as a programmatic dependent: wait for the primary grid
  LeafOwn own;             // PATH_OWNED launches
};

// Fused relocation: RELOC_U sites per thread, each level of the idx -> site -> field chain issued
// for all of them before the next (independent loads in flight), same checks and fault indices
// as relocate_one.
constexpr int RELOC_U = 4;
__device__ __forceinline__ void relocate_multi(const RelocArgs& r, uint64_t base, uint64_t* bad) {
  uint64_t st[RELOC_U], v[RELOC_U];
#pragma unroll
  for (int u = 0; u < RELOC_U; ++u) {
    const uint64_t i = base + uint64_t(u) * SCALE_THREADS;
    st[u] = i < r.n ? (r.idx ? r.sites[r.idx[i]] : r.sites[i]) : ~0ull;
  }
#pragma unroll
  for (int u = 0; u < RELOC_U; ++u)
    v[u] = (st[u] != ~0ull && st[u] + 8 <= r.total) ? ld_u64_any(r.image + st[u]) : 0;
#pragma unroll
  for (int u = 0; u < RELOC_U; ++u) {
    const uint64_t i = base + uint64_t(u) * SCALE_THREADS;
    if (i >= r.n) continue;
    const uint64_t d = v[u] - r.from;   // wraps when v < from
    if (st[u] + 8 > r.total || d >= r.total) { raise_bad(bad, i | r.tag); continue; }
    st_u64_any(r.image + st[u], r.to + d);
  }
}

// Array base + element count of target t: from the resolved table, or re-walked (CHASE).
template <typename T, bool CHASE>
__device__ __forceinline__ bool target_array(const ScaleArgs& a, uint64_t t, uint8_t*& arr, uint64_t& cnt) {
  if (CHASE) {
    Walk w = walk_chain<true>(a.image, a.sh, a.root ? a.root[t] : a.sh.root_off, a.level[t], a.ordinal[t]);
    if (!w.node) return false;
    arr = reinterpret_cast<uint8_t*>(ld_chain_u64(w.node + (w.leaf ? LEAF_OFF_A : OFF_A)));
    cnt = ld_u32_any(w.node + OFF_NA);
  } else {
    arr = reinterpret_cast<uint8_t*>(a.ea[t]);
    cnt = a.count[t];
  }
  if (arr == nullptr) return false;
  // never stream through an address outside the image (a corrupted chain reports, not faults):
  // the whole array [arr, arr + cnt * sizeof(T)) must lie inside it -- memory.py:139-152 raises
  // WildAccess on any span that overruns its allocation; callers then require every part to end
  // at or before cnt
  if (a.image && (arr < a.image || uint64_t(arr - a.image) > a.sh.image_bytes ||
                  cnt * sizeof(T) > a.sh.image_bytes - uint64_t(arr - a.image))) {
    if (atomicCAS(reinterpret_cast<unsigned long long*>(&g_dbg[0]), 0ull, 1ull) == 0ull) {
      g_dbg[1] = t;
      g_dbg[2] = reinterpret_cast<uint64_t>(arr);
      g_dbg[3] = cnt;
      g_dbg[4] = reinterpret_cast<uint64_t>(a.image);
      g_dbg[5] = a.sh.image_bytes;
      g_dbg[6] = a.level ? uint64_t(a.level[t]) : ~0ull;
      g_dbg[7] = a.ordinal ? uint64_t(a.ordinal[t]) : ~0ull;
    }
    return false;
  }
  return true;
}

// Re-derive the array address through the chain (CHASE: one walk per 16-byte access).
template <bool CHASE>
__device__ __forceinline__ uint8_t* chase_base(const ScaleArgs& a, uint64_t t, uint8_t* resolved) {
  if (!CHASE) return resolved;
  Walk w = walk_chain<true>(a.image, a.sh, a.root ? a.root[t] : a.sh.root_off, a.level[t], a.ordinal[t]);
  return reinterpret_cast<uint8_t*>(ld_chain_u64(w.node + (w.leaf ? LEAF_OFF_A : OFF_A)));
}

// f64 arrays at 4 (mod 8) -- the packed reference layout puts them there for odd q -- cannot use
// element-aligned vectors: every element straddles an 8-byte boundary.  One tile is streamed as
// the aligned 16-byte words over its bytes [b0, b1) instead, in ONE pass by the whole CTA: warp
// w loads SHIFT_ROWS consecutive rows of 32 words (a contiguous chunk), then a CTA barrier, then
// every thread rebuilds the three elements meeting its word A = (x0, x1, x2, x3) as u32 --
// hi(Ea) | Eb | lo(Ec) -- from its own word and its neighbours' (warp shuffles; across rows via
// lanes 0 / 31; across warps the chunk-edge u32 was loaded before the barrier) and stores A
// whole.  Straddling elements are thus computed twice, once by each word's owner, each writing
// only its own word: every u32 is written by exactly one thread, always from values read
// before any store of the tile.  Only the tile's two edge words are stored (and loaded) per
// u32, restricted to the tile's own bytes, so neighbouring tiles (other CTAs) never race.
constexpr int SHIFT_ROWS = 5;
static_assert(TILE_BYTES / 16 + CF_SHIFT_ALIGN / 16 + 1 <= uint64_t(SHIFT_ROWS) * SCALE_THREADS,
              "one pass must cover a tile");

template <bool CHASE>
#ifndef CF_F64_SHIFT_NOINLINE
#define CF_F64_SHIFT_NOINLINE 0
#endif
#if CF_F64_SHIFT_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void scale_f64_shifted(const ScaleArgs& a, uint64_t t, uint8_t* arr, uint64_t e0,
                                                  uint64_t e1, double s) {
  constexpr int U = SHIFT_ROWS;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t jw = uint64_t(warp) * (U * 32);   // the warp's first word
  uint4 x[U];
  uintptr_t A[U], b0 = 0, b1 = 0;
  uint32_t halo_lo = 0, halo_hi = 0;   // x3 of word jw-1 / x0 of word jw + 32U (chunk edges)
  uint64_t nw = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint8_t* ar = (CHASE || u == 0) ? chase_base<CHASE>(a, t, arr) : arr;   // CHASE: one walk per row
    b0 = reinterpret_cast<uintptr_t>(ar) + e0 * 8;
    b1 = reinterpret_cast<uintptr_t>(ar) + e1 * 8;
    const uintptr_t w0 = b0 & ~uintptr_t(CF_SHIFT_ALIGN - 1);
    nw = (b1 + 15 - w0) >> 4;
    const uint64_t j = jw + uint64_t(u) * 32 + lane;
    A[u] = w0 + 16 * j;
    x[u] = make_uint4(0u, 0u, 0u, 0u);
    if (j < nw) {
      const uintptr_t p = A[u];
      if (p >= b0 && p + 16 <= b1) {
        x[u] = __ldcs(reinterpret_cast<const uint4*>(p));
      } else {   // edge word: only the u32s inside the tile
        const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
        if (p >= b0 && p < b1) x[u].x = w[0];
        if (p + 4 >= b0 && p + 4 < b1) x[u].y = w[1];
        if (p + 8 >= b0 && p + 8 < b1) x[u].z = w[2];
        if (p + 12 >= b0 && p + 12 < b1) x[u].w = w[3];
      }
    }
  }
  // chunk-edge neighbours owned by other warps of this CTA, read before anyone stores
  if (lane == 0 && jw < nw && A[0] >= b0 + 4 && A[0] + 4 <= b1) halo_lo = reinterpret_cast<const uint32_t*>(A[0])[-1];
  if (lane == 31 && jw + U * 32 < nw && A[U - 1] + 20 <= b1) halo_hi = reinterpret_cast<const uint32_t*>(A[U - 1])[4];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    // x3 of word A-16 and x0 of word A+16
    uint32_t lo_prev = __shfl_up_sync(0xffffffffu, x[u].w, 1);
    uint32_t hi_next = __shfl_down_sync(0xffffffffu, x[u].x, 1);
    const uint32_t row_prev = __shfl_sync(0xffffffffu, u > 0 ? x[u > 0 ? u - 1 : 0].w : 0u, 31);
    const uint32_t row_next = __shfl_sync(0xffffffffu, u + 1 < U ? x[u + 1 < U ? u + 1 : 0].x : 0u, 0);
    if (lane == 0) lo_prev = u > 0 ? row_prev : halo_lo;
    if (lane == 31) hi_next = u + 1 < U ? row_next : halo_hi;
    const uint64_t j = jw + uint64_t(u) * 32 + lane;
    if (j >= nw) continue;
    const uintptr_t p = A[u];
    const bool own_a = p >= b0 + 4 && p + 4 <= b1;     // Ea = [A-4, A+4)
    const bool own_b = p + 4 >= b0 && p + 12 <= b1;    // Eb = [A+4, A+12)
    const bool own_c = p + 12 >= b0 && p + 20 <= b1;   // Ec = [A+12, A+20)
    const double va = __dmul_rn(__hiloint2double(int(x[u].x), int(lo_prev)), s);
    const double vb = __dmul_rn(__hiloint2double(int(x[u].z), int(x[u].y)), s);
    const double vc = __dmul_rn(__hiloint2double(int(hi_next), int(x[u].w)), s);
    const uint4 y = make_uint4(uint32_t(__double2hiint(va)), uint32_t(__double2loint(vb)),
                               uint32_t(__double2hiint(vb)), uint32_t(__double2loint(vc)));
    if (own_a && own_b && own_c) {
      __stcs(reinterpret_cast<uint4*>(p), y);
    } else {   // the tile's edge words: own u32s only
      uint32_t* w = reinterpret_cast<uint32_t*>(p);
      if (own_a) w[0] = y.x;
      if (own_b) { w[1] = y.y; w[2] = y.z; }
      if (own_c) w[3] = y.w;
    }
  }
}

// Scale elements [e0, e1) of arr with `lanes` cooperating threads (rank `me`): scalar head up to
// 128-byte alignment (so every warp's 512-byte row covers whole lines), UNROLL independent
// 128-bit loads in flight per thread, scalar tail.  Misaligned f64 (packed layouts) streams
// aligned words instead (scale_f64_shifted).
template <typename T, bool CHASE, int UNROLL>
__device__ __forceinline__ void scale_range(const ScaleArgs& a, uint64_t t, uint8_t* arr, uint64_t e0, uint64_t e1,
                                            T s, unsigned me, unsigned lanes) {
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr uint64_t VN = VT::N;
  const uintptr_t first = reinterpret_cast<uintptr_t>(arr + e0 * sizeof(T));
  if constexpr (sizeof(T) == 8) {
    if ((first & 7) == 4) {   // whole CTA on one tile (the only caller): see scale_f64_shifted
      scale_f64_shifted<CHASE>(a, t, arr, e0, e1, double(s));
      return;
    }
  }
  uint64_t v0 = e1, v1 = e1;
  if ((first % sizeof(T)) == 0) {
    const uint64_t head = ((CF_ROW_ALIGN - (first & (CF_ROW_ALIGN - 1))) & (CF_ROW_ALIGN - 1)) / sizeof(T);
    v0 = min(e1, e0 + head);
    v1 = v0 + (e1 - v0) / VN * VN;
  }
  for (uint64_t i = e0 + me; i < v0; i += lanes)
    scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
  for (uint64_t i = v1 + me; i < e1; i += lanes)
    scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
  const uint64_t nv = (v1 - v0) / VN;
  uint64_t j = me;
  if (CHASE) {
    for (; j < nv; j += lanes) {
      V* p = reinterpret_cast<V*>(chase_base<true>(a, t, arr) + v0 * sizeof(T)) + j;
      VT::st(p, VT::mul(VT::ld(p), s));
    }
    return;
  }
  V* p = reinterpret_cast<V*>(arr + v0 * sizeof(T));
  for (; j + (UNROLL - 1) * lanes < nv; j += UNROLL * lanes) {
    V r[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) r[u] = VT::ld(p + j + u * lanes);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) VT::st(p + j + u * lanes, VT::mul(r[u], s));
  }
  for (; j < nv; j += lanes) VT::st(p + j, VT::mul(VT::ld(p + j), s));
}

// A group of small parts (<= GROUP_PARTS arrays, <= 16 KiB): warp 0 loads every part's
// metadata once (one dependent-load round per group, not per part) and prefix-sums the vector
// counts into shared memory; then all 256 threads stream the group's 16-byte vectors as one
// flattened range, 4 independent loads in flight per thread.  Scalar heads/tails (only in
// packed layouts) are handled per part afterwards.
template <typename T, bool CHASE>
__device__ __forceinline__ void scale_group(const ScaleArgs& a, uint64_t g, T s) {
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr uint64_t VN = VT::N;
  __shared__ uint8_t* s_base[GROUP_PARTS];    // array base (resolved), nullptr if rejected
  __shared__ uint64_t s_v0[GROUP_PARTS];      // first 16-byte-aligned element
  __shared__ uint32_t s_pre[GROUP_PARTS + 1]; // exclusive prefix of vector counts
  __shared__ uint64_t s_t[GROUP_PARTS];
  const uint32_t p0 = a.w.groups[2 * g], p1 = a.w.groups[2 * g + 1];
  const uint32_t np = p1 - p0;
  const unsigned lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    uint32_t nv = 0;
    if (lane < np) {
      const uint64_t p = p0 + lane;
      const uint64_t t = a.w.parts[3 * p], e0 = a.w.parts[3 * p + 1], e1 = a.w.parts[3 * p + 2];
      uint8_t* arr;
      uint64_t cnt;
      s_t[lane] = t;
      if (!target_array<T, CHASE>(a, t, arr, cnt) || e1 > cnt) {
        raise_bad(a.bad, t | a.tag);
        s_base[lane] = nullptr;
        s_v0[lane] = e1;
      } else {
        const uintptr_t first = reinterpret_cast<uintptr_t>(arr + e0 * sizeof(T));
        uint64_t v0 = e1;
        if ((first % sizeof(T)) == 0) v0 = min(e1, e0 + ((16 - (first & 15)) & 15) / sizeof(T));
        nv = uint32_t((e1 - v0) / VN);
        s_base[lane] = arr;
        s_v0[lane] = v0;
      }
    }
    uint32_t inc = nv;  // warp inclusive scan -> exclusive prefix
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= unsigned(d)) inc += o;
    }
    if (lane < np) s_pre[lane] = inc - nv;
    if (lane == np - 1) s_pre[np] = inc;
  }
  __syncthreads();
  const uint32_t total = s_pre[np];
  // address of flattened vector j (CHASE: through a freshly walked chain per access)
  auto vec_ptr = [&](uint32_t j) -> V* {
    uint32_t lo = 0, hi = np;  // largest k with s_pre[k] <= j
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pre[mid] <= j) lo = mid; else hi = mid;
    }
    uint8_t* base = CHASE ? chase_base<true>(a, s_t[lo], nullptr) : s_base[lo];
    return reinterpret_cast<V*>(base + s_v0[lo] * sizeof(T)) + (j - s_pre[lo]);
  };
  constexpr int U = CF_GROUP_U;
  uint32_t j = threadIdx.x;
  for (; j + (U - 1) * SCALE_THREADS < total; j += U * SCALE_THREADS) {
    V* ptr[U];
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ptr[u] = vec_ptr(j + u * SCALE_THREADS);
      r[u] = VT::ld(ptr[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) VT::st(ptr[u], VT::mul(r[u], s));
  }
  for (; j < total; j += SCALE_THREADS) {
    V* p = vec_ptr(j);
    VT::st(p, VT::mul(VT::ld(p), s));
  }
  // scalar heads / tails (non-empty only in packed layouts); one warp per part
  const unsigned warp = threadIdx.x >> 5;
  for (uint32_t k = warp; k < np; k += SCALE_THREADS / 32) {
    uint8_t* base = s_base[k];
    if (base == nullptr) continue;
    const uint64_t p = p0 + k;
    const uint64_t e0 = a.w.parts[3 * p + 1], e1 = a.w.parts[3 * p + 2];
    const uint64_t v0 = s_v0[k], v1 = v0 + uint64_t(s_pre[k + 1] - s_pre[k]) * VN;
    for (uint64_t i = e0 + lane; i < v0; i += 32)
      scalar_st<T>(base + i * sizeof(T), mul_rn<T>(scalar_ld<T>(base + i * sizeof(T)), s));
    for (uint64_t i = v1 + lane; i < e1; i += 32)
      scalar_st<T>(base + i * sizeof(T), mul_rn<T>(scalar_ld<T>(base + i * sizeof(T)), s));
  }
}

// Small-part group, warp-local version: warp w owns parts p0+w, p0+w+8, ... (<= 4 with 32-part
// groups).  Lanes 0..3 fetch those parts' metadata in parallel (one dependent-load round per
// warp, no CTA barrier) into the warp's slots in shared memory, the warp prefix-sums their vector
// counts in registers, and then streams the flattened (part, vector) sequence with 4 independent
// 128-bit loads in flight per lane, reading each vector's part base from shared memory (an LDS:
// keeping 4 bases and the head / tail bounds in registers across the streaming loop spilled them
// to local memory under the 6-CTA/SM register budget).
template <typename T, bool CHASE>
__device__ __forceinline__ void scale_group_warp(const ScaleArgs& a, uint64_t g, T s) {
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr uint64_t VN = VT::N;
  constexpr unsigned WARPS = SCALE_THREADS / 32;
  constexpr unsigned PER = (GROUP_PARTS + WARPS - 1) / WARPS;  // parts per warp
  struct Slot { uint8_t* vbase; uint8_t* arr; uint64_t e0, e1, v0, t; };   // vbase = arr + v0 (vectors)
  __shared__ Slot slots[WARPS][PER];
  const uint32_t p0 = a.w.groups[2 * g], p1 = a.w.groups[2 * g + 1];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Slot* my = slots[warp];
  // lane j < PER: metadata of part p0 + warp + WARPS * j
  uint32_t nv = 0;
  const uint64_t pj = uint64_t(p0) + warp + uint64_t(WARPS) * lane;
  if (lane < PER) {
    uint8_t* base = nullptr;
    uint64_t v0 = 0, e0 = 0, e1 = 0, t = 0;
    if (pj < p1) {
      t = a.w.parts[3 * pj];
      e0 = a.w.parts[3 * pj + 1];
      e1 = a.w.parts[3 * pj + 2];
      uint64_t cnt;
      if (!target_array<T, CHASE>(a, t, base, cnt) || e1 > cnt) {
        raise_bad(a.bad, t | a.tag);
        base = nullptr;
        v0 = e1;
      } else {
        const uintptr_t first = reinterpret_cast<uintptr_t>(base + e0 * sizeof(T));
        v0 = e1;
        if ((first % sizeof(T)) == 0) v0 = min(e1, e0 + ((16 - (first & 15)) & 15) / sizeof(T));
        nv = uint32_t((e1 - v0) / VN);
      }
    }
    my[lane] = Slot{base + v0 * sizeof(T), base, e0, e1, v0, t};
  }
  // exclusive prefix of nv over lanes 0..PER-1, broadcast to the warp
  __syncwarp();   // the slots are visible to the whole warp
  uint32_t pre[PER + 1];
  pre[0] = 0;
#pragma unroll
  for (unsigned j = 0; j < PER; ++j) pre[j + 1] = pre[j] + __shfl_sync(0xffffffffu, nv, j);
  const uint32_t total = pre[PER];
  auto vptr = [&](uint32_t f) -> V* {
    unsigned j = 0;
#pragma unroll
    for (unsigned k = 1; k < PER; ++k) j += f >= pre[k];
    uint32_t off = pre[0];
#pragma unroll
    for (unsigned k = 1; k < PER; ++k)
      if (j == k) off = pre[k];
    uint8_t* b = CHASE ? chase_base<true>(a, my[j].t, nullptr) + my[j].v0 * sizeof(T)   // re-derived through the chain
                       : my[j].vbase;
    return reinterpret_cast<V*>(b) + (f - off);
  };
  constexpr int U = CF_GROUP_WARP_U;
  uint32_t f = lane;
  for (; f + (U - 1) * 32 < total; f += U * 32) {
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = VT::ld(vptr(f + u * 32));
#pragma unroll
    for (int u = 0; u < U; ++u) VT::st(vptr(f + u * 32), VT::mul(r[u], s));
  }
  for (; f < total; f += 32) {
    V* p = vptr(f);
    VT::st(p, VT::mul(VT::ld(p), s));
  }
  // scalar heads / tails (packed layouts only)
#pragma unroll
  for (unsigned j = 0; j < PER; ++j) {
    const Slot& sj = my[j];
    uint8_t* arr = sj.arr;
    if (arr == nullptr) continue;
    const uint64_t vj1 = sj.v0 + uint64_t(pre[j + 1] - pre[j]) * VN;
    for (uint64_t i = sj.e0 + lane; i < sj.v0; i += 32)
      scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
    for (uint64_t i = vj1 + lane; i < sj.e1; i += 32)
      scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
  }
}

// Leaf-owned group (LeafOwn): warp w owns parts g gp + w, + 8, ... (<= 4).  Lanes 0..3 find
// their part's leaf record in its parent's child block (parent table: an L2 hit), read the
// record's nA and A (one dependent DRAM round -- against groups -> parts -> EA table for the
// table-driven group), attach A (device address written into the record, memory.py:316-323),
// and check the span like target_array; the warp streams the parts' vectors as scale_group_warp
// does, then the owners write the host value back (detach, memory.py:337-344).  Fault tags:
// broken chain -> resolve, A outside the arena -> attach, span -> scale.
template <typename T>
__device__ __forceinline__ void scale_group_owned(const ScaleArgs& a, uint64_t g, T s) {
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr uint64_t VN = VT::N;
  constexpr unsigned WARPS = SCALE_THREADS / 32;
  constexpr unsigned PER = (GROUP_PARTS + WARPS - 1) / WARPS;
  // per part: the vector base, the array (nullptr: nothing to stream), its A field (attached by
  // this warp, nullptr: not attached) and host value -- in shared memory, not registers, across
  // the streaming loop (see scale_group_warp)
  struct Slot { uint8_t* vbase; uint8_t* arr; uint32_t* fa; uint64_t hv, v0; };
  __shared__ Slot slots[WARPS][PER];
  const LeafOwn& o = a.own;
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Slot* my = slots[warp];
  uint32_t nv = 0;
#if CF_OWN_CONTIG
  const uint32_t slot = warp * PER + lane;   // warp w: parts [w PER, (w + 1) PER) of the group
#else
  const uint32_t slot = warp + WARPS * lane;
#endif
  const uint64_t pj = g * o.gp + slot;
  if (lane < PER) {
    uint8_t* base = nullptr;   // attached array base (device), nullptr: nothing to stream
    uint32_t* fa = nullptr;    // the record's A field, attached by this lane
    uint64_t hv = 0, v0 = 0;
    if (slot < o.gp && pj < o.nt) {
      const uint32_t q = a.sh.q;
      const bool leaf = int(o.level) == int(a.sh.depth);
      const uint64_t child = leaf ? LEAF_NODE_SIZE : NODE_SIZE;
      const uint32_t off_a = leaf ? LEAF_OFF_A : OFF_A;
      const uint32_t ord = o.o0 + uint32_t(pj);
      const uint32_t par = q > 1 ? uint32_t(__umul64hi(uint64_t(ord), o.qmagic)) : ord;
      const uint64_t blk = o.parent[par - o.p_first];
      const uint64_t rec = blk + uint64_t(ord - par * q) * child;
      if (blk == 0 || !rec_inside(rec, a.image, a.sh.image_bytes, child)) {
        raise_bad(a.bad, pj | FAULT_RESOLVE);
      } else {
        uint32_t* f = reinterpret_cast<uint32_t*>(rec + off_a);
        const bool mis = (reinterpret_cast<uintptr_t>(f) & 7) != 0;
        hv = mis ? (uint64_t(f[0]) | (uint64_t(f[1]) << 32)) : *reinterpret_cast<const uint64_t*>(f);
        const uint64_t cnt = *reinterpret_cast<const uint32_t*>(rec + OFF_NA);
        const uint64_t d = hv - o.from;
        if (d >= o.total) {
          raise_bad(a.bad, pj | FAULT_ATTACH);
        } else {
          const uint64_t dv = o.to + d;
          if (mis) { f[0] = uint32_t(dv); f[1] = uint32_t(dv >> 32); }
          else *reinterpret_cast<uint64_t*>(f) = dv;
          fa = f;
          uint8_t* arr = reinterpret_cast<uint8_t*>(dv);
          if (uint64_t(o.n_el) > cnt || arr < a.image || uint64_t(arr - a.image) > a.sh.image_bytes ||
              cnt * sizeof(T) > a.sh.image_bytes - uint64_t(arr - a.image)) {
            raise_bad(a.bad, pj | FAULT_SCALE);
          } else {
            base = arr;
            const uintptr_t first = reinterpret_cast<uintptr_t>(arr);
            v0 = o.n_el;
            if ((first % sizeof(T)) == 0) v0 = min(uint64_t(o.n_el), uint64_t(((16 - (first & 15)) & 15) / sizeof(T)));
            nv = uint32_t((o.n_el - v0) / VN);
          }
        }
      }
    }
    my[lane] = Slot{base + v0 * sizeof(T), base, fa, hv, v0};
  }
  __syncwarp();   // the slots are visible to the whole warp
  uint32_t pre[PER + 1];
  pre[0] = 0;
#pragma unroll
  for (unsigned j = 0; j < PER; ++j) pre[j + 1] = pre[j] + __shfl_sync(0xffffffffu, nv, j);
  const uint32_t total = pre[PER];
  auto vptr = [&](uint32_t f) -> V* {
    unsigned j = 0;
#pragma unroll
    for (unsigned k = 1; k < PER; ++k) j += f >= pre[k];
    uint32_t off = pre[0];
#pragma unroll
    for (unsigned k = 1; k < PER; ++k)
      if (j == k) off = pre[k];
    return reinterpret_cast<V*>(my[j].vbase) + (f - off);
  };
  constexpr int U = CF_OWN_U;
  uint32_t f = lane;
  for (; f + (U - 1) * 32 < total; f += U * 32) {
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = VT::ld(vptr(f + u * 32));
#pragma unroll
    for (int u = 0; u < U; ++u) VT::st(vptr(f + u * 32), VT::mul(r[u], s));
  }
  for (; f < total; f += 32) {
    V* p = vptr(f);
    VT::st(p, VT::mul(VT::ld(p), s));
  }
  // scalar heads / tails (packed layouts only)
#pragma unroll
  for (unsigned j = 0; j < PER; ++j) {
    uint8_t* arr = my[j].arr;
    if (arr == nullptr) continue;
    const uint64_t vj0 = my[j].v0, vj1 = vj0 + uint64_t(pre[j + 1] - pre[j]) * VN;
    for (uint64_t i = lane; i < vj0; i += 32)
      scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
    for (uint64_t i = vj1 + lane; i < o.n_el; i += 32)
      scalar_st<T>(arr + i * sizeof(T), mul_rn<T>(scalar_ld<T>(arr + i * sizeof(T)), s));
  }
  // detach: the owners write the host value back into the record (after their warp's stores of
  // the array -- other lanes' stores are to the array, never to the record)
  if (lane < PER && my[lane].fa && !o.keep_attached) {
    uint32_t* fa = my[lane].fa;
    const uint64_t hv = my[lane].hv;
    if ((reinterpret_cast<uintptr_t>(fa) & 7) != 0) { fa[0] = uint32_t(hv); fa[1] = uint32_t(hv >> 32); }
    else *reinterpret_cast<uint64_t*>(fa) = hv;
  }
}

// One CTA per unit of work: after the fused relocation CTAs (a detach riding in the launch),
// one 16 KiB tile of a big part per CTA, then one group of small parts per CTA (one warp per
// part).  PATH specialises the kernel for launches with
// only tiles or only groups (the common cases: C2 / C4), so each gets its own register budget
// under the 6-CTA/SM launch bound instead of the union of both paths' (no spills).
enum { PATH_ALL = 0, PATH_TILES = 1, PATH_GROUPS = 2, PATH_OWNED = 3 };
template <typename T, bool CHASE, int PATH>
__global__ void __launch_bounds__(SCALE_THREADS, PATH == PATH_OWNED ? CF_OWN_MINB : PATH == PATH_GROUPS ? CF_GROUP_MINB : CF_SCALE_MINB)
    k_scale(ScaleArgs a, T s) {
  // launched as a programmatic dependent of the attach / resolve kernel: its CTAs may be resident
  // before that grid has finished -- wait for its completion (and memory) before any read
#if CF_PDL_WAIT_ALWAYS
  asm volatile("griddepcontrol.wait;" ::: "memory");
#else
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  constexpr uint64_t TILE = TILE_BYTES / sizeof(T);
  // fused relocation CTAs (the detach riding in the launch) are spread evenly through the grid --
  // CTA k * reloc_stride is relocation CTA k: in RESOLVED mode no leaf CTA reads a pointer field
  // and every resolver that reads them has completed (stream order / griddepcontrol.wait), so the
  // latency-bound relocation overlaps the streaming instead of forming a wave of its own (first)
  // or trailing the drain (last)
  unsigned b = blockIdx.x;
  if (a.reloc_blocks) {
#if CF_RELOC_FASTMAP
    // CTAs past the last relocation slot (all but a few for C2's single detach CTA) skip the
    // division; the rest divide by a multiply-high (CTA start latency matters on the tile path)
    if (b > a.reloc_last) {
      b -= a.reloc_blocks;
    } else {
      unsigned k = unsigned(__umulhi(b, a.reloc_magic));   // b / reloc_stride or one more
      if (k * a.reloc_stride > b) --k;
      if (b == k * a.reloc_stride && k < a.reloc_blocks) {
        relocate_multi(a.reloc, uint64_t(k) * (SCALE_THREADS * RELOC_U) + threadIdx.x, a.bad);
        return;
      }
      b -= min(k + 1, a.reloc_blocks);
    }
#else
    const unsigned k = b / a.reloc_stride;
    if (b % a.reloc_stride == 0 && k < a.reloc_blocks) {
      relocate_multi(a.reloc, uint64_t(k) * (SCALE_THREADS * RELOC_U) + threadIdx.x, a.bad);
      return;
    }
    b -= min(k + 1, a.reloc_blocks);
#endif
  }
  if constexpr (PATH == PATH_OWNED) {
    scale_group_owned<T>(a, b, s);
    return;
  }
  const uint64_t ntiles = a.w.tile_end - a.w.tile_begin;
  if (PATH != PATH_GROUPS && b < ntiles) {
    // lane 0 of every warp maps the tile to its part (binary search over the launch's first-tile
    // table) and reads the part and its resolved address; the warp gets them by shuffle -- one
    // search and one metadata load per warp instead of per thread
    const uint64_t tile = a.w.tile_begin + b;
    const unsigned lane = threadIdx.x & 31;
    uint64_t t = 0, e0 = 0, e1 = 0, cnt = 0;
    uintptr_t arr_u = 0;
    int ok = 0;
    if (lane == 0) {
      uint64_t lo = 0, hi = a.w.big_count;   // big part index within this launch
      const uint64_t* tb = a.w.tile_base + a.w.tb_begin;
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (tb[mid] <= tile) lo = mid; else hi = mid;
      }
      const uint32_t* pt = a.w.parts + 3 * (a.w.big_begin + lo);
      t = pt[0];
      e0 = uint64_t(pt[1]) + (tile - tb[lo]) * TILE;
      e1 = min(uint64_t(pt[2]), e0 + TILE);
      uint8_t* arr;
      ok = target_array<T, CHASE>(a, t, arr, cnt) && e1 <= cnt;
      arr_u = reinterpret_cast<uintptr_t>(arr);
      if (!ok && threadIdx.x == 0) raise_bad(a.bad, t | a.tag);
    }
    if (!__shfl_sync(0xffffffffu, ok, 0)) return;
    t = __shfl_sync(0xffffffffu, t, 0);
    e0 = __shfl_sync(0xffffffffu, e0, 0);
    e1 = __shfl_sync(0xffffffffu, e1, 0);
    arr_u = __shfl_sync(0xffffffffu, arr_u, 0);
    scale_range<T, CHASE, SCALE_UNROLL>(a, t, reinterpret_cast<uint8_t*>(arr_u), e0, e1, s, threadIdx.x, SCALE_THREADS);
    return;
  }
  if constexpr (PATH != PATH_TILES) {
    const uint64_t g = a.w.group_begin + (b - ntiles);
#if CF_GROUP_WARP
    scale_group_warp<T, CHASE>(a, g, s);
#else
    scale_group<T, CHASE>(a, g, s);
#endif
  }
}

// ---------------------------------------------------------------- naive fix-up
__device__ __forceinline__ bool translate(uint64_t addr, const uint64_t* hb, const uint64_t* sz,
                                          const uint64_t* db, uint64_t n, uint64_t* out) {
  // AddressMap.translate (memory.py:409-419): bisect_right over sorted host bases
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (hb[mid] <= addr) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return false;
  const uint64_t i = lo - 1;
  if (addr - hb[i] >= sz[i]) return false;
  *out = db[i] + (addr - hb[i]);
  return true;
}

__global__ void __launch_bounds__(256) k_naive_fixup(const uint64_t* __restrict__ field_host,
                                                     const uint64_t* __restrict__ target_host, uint64_t n,
                                                     const uint64_t* __restrict__ hb, const uint64_t* __restrict__ sz,
                                                     const uint64_t* __restrict__ db, uint64_t nmap, uint64_t* bad) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t f, tg;
    if (!translate(field_host[i], hb, sz, db, nmap, &f) || !translate(target_host[i], hb, sz, db, nmap, &tg)) {
      raise_bad(bad, i);
      continue;
    }
    st_u64_any(reinterpret_cast<uint8_t*>(f), tg);
  }
}

// Zero-copy segment copy: one warp per (lo, hi) segment, src and dst at the same offsets from
// their bases; either side may be mapped pinned host memory (PCIe loads/stores issued by the
// SMs).  Moves hundreds of scattered node records in one launch instead of one DMA each.
__global__ void __launch_bounds__(256) k_seg_copy(const uint64_t* __restrict__ segs, uint64_t n,
                                                  const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  const uint64_t wid = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  if (wid >= n) return;
  const uint64_t lo = segs[2 * wid], hi = segs[2 * wid + 1];
  uint64_t i = lo;
  if (((lo | hi) & 3) == 0) {
    for (uint64_t k = lo / 4 + lane; k < hi / 4; k += 32)
      reinterpret_cast<uint32_t*>(dst)[k] = reinterpret_cast<const uint32_t*>(src)[k];
    return;
  }
  for (i = lo + lane; i < hi; i += 32) dst[i] = src[i];
}

// Many small copies as one launch (zero-copy over mapped pinned host memory, either
// direction): warp i copies bytes[i] from src[i] to dst[i] in the widest words (16, 8 or 4 bytes)
// that both ends and the length allow.  Replaces one copy-engine command per object for the
// pointerchain scheme's small arrays (cf_selective_run).
__device__ __forceinline__ void copy_object(uint64_t s, uint64_t d, uint64_t b, unsigned lane);

__global__ void __launch_bounds__(256) k_copy_list(const uint64_t* __restrict__ src, const uint64_t* __restrict__ dst,
                                                   const uint64_t* __restrict__ bytes, uint64_t n) {
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  if (i >= n) return;
  copy_object(src[i], dst[i], bytes[i], lane);
}

// Two copy lists in one launch, their warps interleaved (A0 B0 A1 B1 ... then the longer list's
// rest): a pipelined window's copy-out of step k and copy-in of step k+1 then share every SM, so
// both link directions stay busy (zero-copy duplex) instead of one grid draining before the other.
__global__ void __launch_bounds__(256) k_copy_list2(const uint64_t* __restrict__ sa, const uint64_t* __restrict__ da,
                                                    const uint64_t* __restrict__ ba, uint64_t na,
                                                    const uint64_t* __restrict__ sb, const uint64_t* __restrict__ db,
                                                    const uint64_t* __restrict__ bb, uint64_t nb) {
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t m = na < nb ? na : nb;
  bool a;
  uint64_t i;
  if (w < 2 * m) {
    a = (w & 1) == 0;
    i = w >> 1;
  } else {
    a = na > nb;
    i = m + (w - 2 * m);
    if (i >= (a ? na : nb)) return;
  }
  if (a) copy_object(sa[i], da[i], ba[i], lane);
  else copy_object(sb[i], db[i], bb[i], lane);
}

__device__ __forceinline__ void copy_object(uint64_t s, uint64_t d, uint64_t b, unsigned lane) {
  if (((s | d | b) & 15) == 0) {
    // all loads of a 2 KiB slice first, then the stores: one PCIe round trip per slice instead
    // of one per 512 bytes (source and destination may not alias, the compiler cannot know)
    const uint4* ps = reinterpret_cast<const uint4*>(s);
    uint4* pd = reinterpret_cast<uint4*>(d);
    const uint64_t n16 = b / 16;
    for (uint64_t k = lane; k < n16; k += 128) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + 32 * u < n16) v[u] = ps[k + 32 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + 32 * u < n16) pd[k + 32 * u] = v[u];
    }
  } else if (((s | d | b) & 7) == 0) {
    const uint64_t* ps = reinterpret_cast<const uint64_t*>(s);
    uint64_t* pd = reinterpret_cast<uint64_t*>(d);
    for (uint64_t k = lane; k < b / 8; k += 32) pd[k] = ps[k];
  } else if (((s | d | b) & 3) == 0) {
    const uint32_t* ps = reinterpret_cast<const uint32_t*>(s);
    uint32_t* pd = reinterpret_cast<uint32_t*>(d);
    for (uint64_t k = lane; k < b / 4; k += 32) pd[k] = ps[k];
  } else {
    for (uint64_t k = lane; k < b; k += 32) reinterpret_cast<uint8_t*>(d)[k] = reinterpret_cast<const uint8_t*>(s)[k];
  }
}

// Naive scheme: every resolved chain must end on its array's device copy with the planned count;
// the first target that does not is reported (atomicMin on the error word).
__global__ void __launch_bounds__(256) k_check_resolved(const uint64_t* __restrict__ ea, const uint32_t* __restrict__ cnt,
                                                        const uint64_t* __restrict__ expect_off,
                                                        const uint32_t* __restrict__ cnt_plan, uint64_t image, uint64_t n,
                                                        unsigned long long* bad) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && (ea[i] != image + expect_off[i] || cnt[i] != cnt_plan[i])) atomicMin(bad, (unsigned long long)i);
}

// Bulk copy by the SMs (either side may be mapped pinned host memory): grid-stride 16-byte words,
// 4 in flight per thread.  Link experiments: SM-driven PCIe reads/writes beside the copy engines.
__global__ void __launch_bounds__(256) k_sm_copy(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t n16) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// Per-range checksum for the multi-GPU result gather: position-weighted wrapping
// u64 sum  sum_i word_i * (i + 1)  over the range's u32 words (i = word index in the range), so a
// tile written to the wrong offset or two swapped tiles change it; the terms are independent, so
// tiles still accumulate atomically.  One CTA per 64 KiB tile of a range; tile_lo[r] = first
// tile of range r.
constexpr uint64_t CK_TILE_WORDS = 16384;
__global__ void __launch_bounds__(256) k_checksum(const uint64_t* __restrict__ addr, const uint64_t* __restrict__ words,
                                                  const uint64_t* __restrict__ tile_lo, uint64_t nranges,
                                                  unsigned long long* __restrict__ out) {
  const uint64_t tile = blockIdx.x;
  uint64_t lo = 0, hi = nranges;   // largest r with tile_lo[r] <= tile
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (tile_lo[mid] <= tile) lo = mid; else hi = mid;
  }
  const uint32_t* p = reinterpret_cast<const uint32_t*>(addr[lo]);
  const uint64_t w0 = (tile - tile_lo[lo]) * CK_TILE_WORDS, w1 = min(words[lo], w0 + CK_TILE_WORDS);
  unsigned long long acc = 0;
  for (uint64_t i = w0 + threadIdx.x; i < w1; i += 256) acc += uint64_t(__ldcs(p + i)) * (i + 1);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  __shared__ unsigned long long red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < 8; ++k) t += red[k];
    atomicAdd(out + lo, t);
  }
}

// L2 eviction by a read pass (benchmark plumbing): every line of the buffer is loaded, so the L2
// ends up holding clean lines of it -- unlike a memset, whose dirty lines would be written back
// inside the next timed window.  The (never true) store keeps the loads alive.
__global__ void __launch_bounds__(256) k_evict_read(const uint4* __restrict__ p, uint64_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u && sink) *sink = acc;
}

__global__ void k_fill_u64(uint64_t* p, uint64_t v, uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

unsigned grid_for(cf_ctx* ctx, uint64_t work, unsigned threads, unsigned per_sm) {
  const uint64_t want = (work + threads - 1) / threads;
  const uint64_t cap = uint64_t(ctx->sm_count > 0 ? ctx->sm_count : 148) * per_sm;
  return unsigned(std::max<uint64_t>(1, std::min(want, cap)));
}

}  // namespace

#define CF_LAUNCHED(ctx)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(CF_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                   \
    (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                             \
  } while (0)

int launch_relocate(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t n,
                    uint64_t from, uint64_t to, uint64_t* bad, cudaStream_t s, const uint32_t* idx, uint64_t tag) {
  if (n == 0) return CF_OK;
  k_relocate<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(image, total, sites, idx, n, from, to, bad, tag);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_attach_resolve(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                          uint64_t from, uint64_t to, const cf_chain_shape& sh, const uint64_t* root, const int32_t* level,
                          const uint32_t* ordinal, uint64_t ntargets, uint64_t* ea, uint32_t* count, uint64_t* bad,
                          cudaStream_t s, uint64_t res_tag) {
  if (nsites == 0 && ntargets == 0) return CF_OK;
  const unsigned threads = unsigned(std::min<uint64_t>(1024, std::max<uint64_t>(32, ((std::max(nsites, ntargets) + 31) / 32) * 32)));
  k_attach_resolve<<<1, threads, 0, s>>>(image, total, sites, nsites, from, to, sh, root, level, ordinal, ntargets,
                                        ea, count, bad, res_tag);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_attach_resolve_wide(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                               uint64_t from, uint64_t to, const cf_chain_shape& sh, const uint64_t* root,
                               const int32_t* level, const uint32_t* ordinal, uint64_t ntargets, uint64_t* ea,
                               uint32_t* count, uint64_t* bad, cudaStream_t s, uint64_t res_tag, const UniTargets* uni) {
  const uint64_t ab = (nsites + 255) / 256;
  if (uni && uni->on && sh.q >= 2 && ntargets) {
    // memory-parallel uniform resolver: 32 U targets per warp, U as large as lets the run's
    // parents (at most (32 U - 1) / q + 2 of them) fit one lane each
    static const int u_env = getenv("CF_UNI_U") ? atoi(getenv("CF_UNI_U")) : UNI_U;   // design experiments
    unsigned U = unsigned(std::max(1, std::min(UNI_U, u_env)));
    while (U > 1 && (32 * U - 1) / sh.q + 2 > 32) U >>= 1;
    const uint64_t per_cta = uint64_t(32) * U * 8;
    const uint64_t rb = (ntargets + per_cta - 1) / per_cta;
    if (ab + rb > 0x7FFFFFFFull) return fail(CF_E_INVALID, "attach/resolve grid too large");
    k_attach_resolve_uni<<<unsigned(ab + rb), 256, 0, s>>>(image, total, sites, nsites, from, to, sh, ntargets, ea, count,
                                                          bad, unsigned(ab), res_tag, *uni, U);
    CF_LAUNCHED(ctx);
    return CF_OK;
  }
  const uint64_t rb = (ntargets + 255) / 256;
  if (ab + rb == 0) return CF_OK;
  if (ab + rb > 0x7FFFFFFFull) return fail(CF_E_INVALID, "attach/resolve grid too large");
  k_attach_resolve_wide<<<unsigned(ab + rb), 256, 0, s>>>(image, total, sites, nsites, from, to, sh, root, level,
                                                         ordinal, ntargets, ea, count, bad, unsigned(ab), res_tag,
                                                         uni ? *uni : UniTargets{0, 0, 0, 0, 0});
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_attach_parents(cf_ctx* ctx, uint8_t* image, uint64_t total, const uint64_t* sites, uint64_t nsites,
                          uint64_t from, uint64_t to, const cf_chain_shape& sh, const LeafOwn& own, uint64_t* parent,
                          uint64_t* bad, cudaStream_t s) {
  const uint64_t ab = (nsites + 255) / 256, pb = (uint64_t(own.nparents) + 255) / 256;
  if (ab + pb == 0) return CF_OK;
  k_attach_parents<<<unsigned(ab + pb), 256, 0, s>>>(image, total, sites, nsites, from, to, sh, own, parent, bad,
                                                     unsigned(ab));
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_resolve(cf_ctx* ctx, const uint8_t* image, const cf_chain_shape& sh, const uint64_t* root,
                   const int32_t* level, const uint32_t* ordinal, uint64_t n, uint64_t* ea, uint32_t* count,
                   uint64_t* bad, cudaStream_t s, uint64_t tag) {
  if (n == 0) return CF_OK;
  k_resolve<<<unsigned((n + 127) / 128), 128, 0, s>>>(image, sh, root, level, ordinal, n, ea, count, bad, tag);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_scale(cf_ctx* ctx, int elem, int mode, const uint8_t* image, const cf_chain_shape& sh,
                 const uint64_t* root, const int32_t* level, const uint32_t* ordinal, const uint64_t* ea,
                 const uint32_t* count,
                 const cf_scale_work& work, double scale, uint64_t* bad, cudaStream_t s,
                 const RelocArgs* fused_reloc, uint64_t tag, bool pdl, const LeafOwn* own) {
  const uint64_t nreloc = fused_reloc ? fused_reloc->n : 0;
  const uint64_t rblocks = (nreloc + SCALE_THREADS * RELOC_U - 1) / (SCALE_THREADS * RELOC_U);
  const uint64_t owned_groups = own ? (uint64_t(own->nt) + own->gp - 1) / own->gp : 0;
  const uint64_t units = own ? owned_groups + rblocks
                             : (work.tile_end - work.tile_begin) + (work.group_end - work.group_begin) + rblocks;
  if (units == 0) return CF_OK;
  if (units > 0x7FFFFFFFull) return fail(CF_E_INVALID, "leaf kernel: %llu work units exceed one grid",
                                         (unsigned long long)units);
  static const bool reloc_first = getenv("CF_RELOC_FIRST") != nullptr;   // design experiments
  const unsigned stride = (rblocks == 0 || reloc_first) ? 1u : unsigned(units / rblocks);
  const unsigned rlast = rblocks ? unsigned(rblocks - 1) * stride : 0u;
  const unsigned rmagic = stride > 1 ? unsigned((0x100000000ull + stride - 1) / stride) : 0u;
  ScaleArgs a{image, sh, root, level, ordinal, ea, count, work, bad, tag, RelocArgs{}, unsigned(rblocks), stride,
              rlast, rmagic, pdl ? 1u : 0u, LeafOwn{}};
  if (nreloc) a.reloc = *fused_reloc;
  if (own) {
    if (mode == CF_MODE_CHASE) return fail(CF_E_INVALID, "leaf-owned relocation needs RESOLVED mode");
    a.own = *own;
  }
  // one CTA per 16 KiB tile / small-part group: measured faster than a persistent grid-stride
  // grid on B200 (tools/scale_variants.cu: 6.7 vs 5.8 TB/s over the C2 shape) -- the hardware
  // CTA launcher keeps more independent loads in flight than a loop re-locating its part
  const unsigned grid = unsigned(units);
  const bool tiles = work.tile_end > work.tile_begin, groups = work.group_end > work.group_begin;
  const int path = own ? PATH_OWNED : (tiles && groups) ? PATH_ALL : (groups ? PATH_GROUPS : PATH_TILES);
  // pdl: the previous kernel on s is the attach / resolve launch -- let this grid launch as its
  // programmatic dependent (k_scale waits for it with griddepcontrol.wait)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SCALE_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t le = cudaSuccess;
  auto go = [&](auto tag_t, auto tag_chase) {
    using T = decltype(tag_t);
    constexpr bool C = decltype(tag_chase)::value;
    const T sc = T(scale);
    if constexpr (!C) {
      if (path == PATH_OWNED) { le = cudaLaunchKernelEx(&cfg, k_scale<T, false, PATH_OWNED>, a, sc); return; }
    }
    if (path == PATH_TILES) le = cudaLaunchKernelEx(&cfg, k_scale<T, C, PATH_TILES>, a, sc);
    else if (path == PATH_GROUPS) le = cudaLaunchKernelEx(&cfg, k_scale<T, C, PATH_GROUPS>, a, sc);
    else le = cudaLaunchKernelEx(&cfg, k_scale<T, C, PATH_ALL>, a, sc);
  };
  if (elem == 4) {
    if (mode == CF_MODE_CHASE) go(float{}, std::true_type{});
    else go(float{}, std::false_type{});
  } else {
    if (mode == CF_MODE_CHASE) go(double{}, std::true_type{});
    else go(double{}, std::false_type{});
  }
  if (le != cudaSuccess) return fail(CF_E_CUDA, "leaf kernel launch: %s", cudaGetErrorString(le));
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_naive_fixup(cf_ctx* ctx, const uint64_t* field_host, const uint64_t* target_host, uint64_t n,
                       const uint64_t* hb, const uint64_t* sz, const uint64_t* db, uint64_t nmap,
                       uint64_t* bad, cudaStream_t s) {
  if (n == 0) return CF_OK;
  k_naive_fixup<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(field_host, target_host, n, hb, sz, db, nmap, bad);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_seg_copy(cf_ctx* ctx, const uint64_t* segs, uint64_t n, const uint8_t* src, uint8_t* dst, cudaStream_t s) {
  if (n == 0) return CF_OK;
  k_seg_copy<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(segs, n, src, dst);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_sm_copy(cf_ctx* ctx, void* dst, const void* src, uint64_t bytes, unsigned ctas, cudaStream_t s) {
  if (bytes == 0) return CF_OK;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15)
    return fail(CF_E_INVALID, "sm copy needs 16-byte aligned ends");
  k_sm_copy<<<ctas ? ctas : unsigned(ctx->sm_count) * 4, 256, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src),
                                                                  bytes / 16);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_copy_list(cf_ctx* ctx, const uint64_t* src, const uint64_t* dst, const uint64_t* bytes, uint64_t n,
                     cudaStream_t s) {
  if (n == 0) return CF_OK;
  k_copy_list<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(src, dst, bytes, n);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_copy_list2(cf_ctx* ctx, const uint64_t* sa, const uint64_t* da, const uint64_t* ba, uint64_t na,
                      const uint64_t* sb, const uint64_t* db, const uint64_t* bb, uint64_t nb, cudaStream_t s) {
  if (na == 0) return launch_copy_list(ctx, sb, db, bb, nb, s);
  if (nb == 0) return launch_copy_list(ctx, sa, da, ba, na, s);
  k_copy_list2<<<unsigned(((na + nb) * 32 + 255) / 256), 256, 0, s>>>(sa, da, ba, na, sb, db, bb, nb);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_check_resolved(cf_ctx* ctx, const uint64_t* ea, const uint32_t* cnt, const uint64_t* expect_off,
                          const uint32_t* cnt_plan, uint64_t image, uint64_t n, uint64_t* bad, cudaStream_t s) {
  if (n == 0) return CF_OK;
  k_check_resolved<<<unsigned((n + 255) / 256), 256, 0, s>>>(ea, cnt, expect_off, cnt_plan, image, n,
                                                            reinterpret_cast<unsigned long long*>(bad));
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_checksum(cf_ctx* ctx, const uint64_t* addr, const uint64_t* words, const uint64_t* tile_lo, uint64_t nranges,
                    uint64_t ntiles, uint64_t* out, cudaStream_t s) {
  if (ntiles == 0) return CF_OK;
  k_checksum<<<unsigned(ntiles), 256, 0, s>>>(addr, words, tile_lo, nranges, reinterpret_cast<unsigned long long*>(out));
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int debug_info(uint64_t* out, int reset) {
  CF_CUDA(cudaMemcpyFromSymbol(out, g_dbg, sizeof(uint64_t) * 8));
  if (reset) {
    static const uint64_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    CF_CUDA(cudaMemcpyToSymbol(g_dbg, z, sizeof z));
  }
  return CF_OK;
}

int launch_evict_read(cf_ctx* ctx, const void* buf, uint64_t bytes, cudaStream_t s) {
  if (bytes < 16) return CF_OK;
  k_evict_read<<<unsigned(std::max(1, ctx->sm_count) * 8), 256, 0, s>>>(static_cast<const uint4*>(buf), bytes / 16,
                                                                           nullptr);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

int launch_fill_u64(cf_ctx* ctx, uint64_t* p, uint64_t v, uint64_t n, cudaStream_t s) {
  if (n == 0) return CF_OK;
  k_fill_u64<<<unsigned((n + 255) / 256), 256, 0, s>>>(p, v, n);
  CF_LAUNCHED(ctx);
  return CF_OK;
}

}  // namespace cf
