/*
 * chainforge_b200.h -- C ABI of libchainforge_b200.so, the B200-native deep-copy hot path.
 *
 * The reference (arxiv 1906.01128's `chainforge`, pure Python) has no FFI; its seam is the
 * Python call triple inside execute_case's metered window (harness.py:369-373).  Each entry
 * point below replaces one reference function (cited as file:line under
 * /root/reference/pkg/src/chainforge); INTEGRATION.md shows the ctypes binding a chainforge
 * maintainer would add.  Conventions:
 *   - plain C types only; every function returns int (CF_OK = 0, negative CF_E_* on failure);
 *   - cf_last_error() returns a thread-local message for the last failure on this thread;
 *   - device work is enqueued on an explicit stream (NULL = the context's compute stream);
 *   - one cf_ctx per GPU, used by one host thread (SPEC.md concurrency model).
 * Error codes map onto the reference exceptions (memory.py:44-57, harness.py:46-51):
 *   CF_E_OOM -> OutOfSimMemory, CF_E_WILD -> WildAccess,
 *   CF_E_OUTSIDE_ARENA -> AttachOutsideArena, CF_E_STATE -> SimMemoryError.
 */
#ifndef CHAINFORGE_B200_H
#define CHAINFORGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_ABI_VERSION 2   /* 2: cf_spec gained shard_rank / shard_world */

enum {
  CF_OK = 0,
  CF_E_INVALID = -1,        /* bad argument (ValueError) */
  CF_E_OOM = -2,            /* OutOfSimMemory (memory.py:48) */
  CF_E_WILD = -3,           /* WildAccess (memory.py:52) */
  CF_E_OUTSIDE_ARENA = -4,  /* AttachOutsideArena (memory.py:56) */
  CF_E_CUDA = -5,           /* CUDA runtime failure (message carries cudaGetErrorString) */
  CF_E_NODEVICE = -6,       /* no CUDA device: the product path refuses to run without one */
  CF_E_STATE = -7           /* SimMemoryError: call out of order (memory.py:333-334) */
};

/* tree kinds / layouts (scenarios.py:30-68) */
enum { CF_LINEAR = 0, CF_DENSE = 1 };
enum { CF_ALLINIT_ALLUSED = 0, CF_ALLINIT_LLUSED = 1, CF_LLINIT_LLUSED = 2 };
/* host memory kinds */
enum { CF_MEM_PAGEABLE = 0, CF_MEM_PINNED = 1, CF_MEM_MANAGED = 2 };
/* target policies: CF_TARGET_REF = targeted_arrays (scenarios.py:270-284); the other two are
 * the BASELINE configs' "consume every leaf" / "every array" policies */
enum { CF_TARGET_REF = 0, CF_TARGET_ALL_LEAVES = 1, CF_TARGET_ALL_ARRAYS = 2 };
/* leaf-kernel modes: resolved effective address (pointerchain) vs chase-per-access (Listing 2) */
enum { CF_MODE_RESOLVED = 0, CF_MODE_CHASE = 1 };

typedef struct cf_ctx cf_ctx;       /* one GPU: streams, events, scratch */
typedef struct cf_tree cf_tree;     /* planned graph layout + relocation/chain tables */
typedef struct cf_window cf_window; /* a planned, pipelined metered window */
typedef struct cf_selective cf_selective; /* a planned, pipelined pointerchain window */
typedef struct cf_kernel_plan cf_kernel_plan; /* a planned kernel_scale (eager schemes) */

/* LinearSpec / DenseSpec (scenarios.py:33-68) plus the B200 build parameters.
 * elem: 8 = float64 (reference), 4 = float32 (BASELINE configs).
 * align: 1 = packed arena (Arena.allocate, memory.py:217-227), 8 = host bump allocator
 *        (MemorySpace.allocate, memory.py:124-137), 16 = aligned production arena.
 * leaf_only: dense trees with arrays on the depth-D leaves only (BASELINE C2/C5).
 * forest / scatter_seed: BASELINE C3 -- many independent trees whose objects are scattered
 * over the slab instead of laid out in DFS order (the reference builds single trees only). */
typedef struct {
  int32_t kind;
  int32_t layout;
  int64_t k_or_q;
  int64_t n;
  int64_t depth;
  int32_t elem;
  int32_t leaf_only;
  int32_t align;
  int32_t forest;         /* number of independent trees (0 or 1: a single tree); C3 = 64 chains */
  uint64_t scatter_seed;  /* != 0: allocations placed in a seeded random order (sparse layout) */
  /* dense subtree shard: the tree is cut at the shallowest level l with
   * q^l >= shard_world; this plan materialises the replicated ancestor path plus the level-l
   * subtrees with (ordinal * shard_world / q^l) == shard_rank.  Non-owned level-l nodes keep
   * their record in the parent's block with nulled fields; arrays above level l live on rank 0
   * only.  shard_world 0 or 1: the whole tree. */
  int32_t shard_rank;
  int32_t shard_world;
} cf_spec;

typedef struct {
  uint64_t total_bytes;   /* arena bytes (== closed form when align == 1) */
  uint64_t nallocs, nnodes, narrays, nsites, ntrees;
  uint64_t root_off;      /* offset of the root node */
  uint64_t payload_bytes; /* sum of array bytes */
  uint64_t padding_bytes; /* total_bytes - sum of allocation sizes */
} cf_tree_info;

/* tables exposed by cf_tree_table (pointers stay valid until cf_tree_free) */
enum {
  CF_TAB_ALLOC_OFF = 0,   /* u64[nallocs]   allocation order (request_list)          */
  CF_TAB_ALLOC_SIZE = 1,  /* u64[nallocs]                                             */
  CF_TAB_NODE_OFF = 2,    /* u64[nnodes]    pre-order (TreeHandle.node_addrs)         */
  CF_TAB_NODE_LEVEL = 3,  /* i32[nnodes]                                              */
  CF_TAB_NODE_SIZE = 4,   /* u32[nnodes]                                              */
  CF_TAB_ARR_LEVEL = 5,   /* i32[narrays]   TreeHandle.arrays (ArrayRef)              */
  CF_TAB_ARR_OWNER = 6,   /* u64[narrays]                                             */
  CF_TAB_ARR_OFF = 7,     /* u64[narrays]                                             */
  CF_TAB_ARR_COUNT = 8,   /* u64[narrays]                                             */
  CF_TAB_SITE_OFF = 9,    /* u64[nsites]    DFS order (Arena.pointer_sites)           */
  CF_TAB_SITE_TARGET = 10,/* u64[nsites]    target offset of each pointer field      */
  CF_TAB_SITE_SORTED = 11,/* u64[nsites]    ascending offsets (the relocation table)  */
  CF_TAB_ARR_ORDINAL = 12,/* u64[narrays]   owner's ordinal among nodes of its level  */
  CF_TAB_ARR_ROOT = 13,   /* u64[narrays]   root offset of the tree owning the array   */
  CF_TAB_TREE_ROOT = 14   /* u64[ntrees]    root offset of every tree                  */
};

/* Chain shape walked by the resolve / chase kernels (kernel_scale walk, harness.py:285-304).
 * A target is (level L, ordinal): L hops through Lnext from the root; for dense trees the
 * hop at level l takes child digit_l of the ordinal written in base q. */
typedef struct {
  int32_t kind;
  int32_t depth;        /* dense D (leaf level uses 12-byte nodes); linear: k-1 */
  uint32_t q;           /* dense fan-out; 1 for linear */
  uint32_t reserved;
  uint64_t root_off;    /* root node offset inside the image */
  uint64_t image_bytes; /* every hop must stay inside [image, image + image_bytes) */
} cf_chain_shape;

/* ---------------- runtime ---------------- */
int cf_abi_version(void);
const char* cf_last_error(void);
int cf_device_count(int* count);
/* nstreams: H2D copy streams (>= 1); a compute and a D2H stream are added. */
/* NUMA placement of host arenas (no libnuma in the image): the node of the GPU's
 * PCI device (-1 if unknown), and binding the calling thread's CPUs + preferred memory to a node
 * so pinned arenas it allocates are local to that GPU's host link; node < 0 restores the default
 * memory policy (the caller restores its CPU mask). */
int cf_device_numa_node(int device, int* node);
int cf_bind_numa_node(int node);
int cf_ctx_create(int device, int nstreams, cf_ctx** out);
int cf_ctx_destroy(cf_ctx* ctx);
int cf_ctx_sync(cf_ctx* ctx);
void* cf_ctx_stream(cf_ctx* ctx);               /* compute stream (cudaStream_t) */
uint64_t cf_ctx_launches(cf_ctx* ctx);          /* kernels launched so far */
int cf_ctx_sm_count(cf_ctx* ctx);
/* Device-side phase timer (CUDA events on the context's compute stream, which every library
 * operation forks from and joins back into): _stop waits for the work enqueued since _start and
 * returns its device time in ms (execute_case's measured columns, harness.py:369-373). */
typedef struct cf_timer cf_timer;
int cf_timer_create(cf_ctx* ctx, cf_timer** out);
int cf_timer_start(cf_timer* t);
int cf_timer_stop(cf_timer* t, float* ms);
int cf_timer_free(cf_timer* t);

/* Host memory for arenas / host spaces (MemorySpace storage, memory.py:101-137).
 * PINNED = cudaHostAlloc(portable), MANAGED = cudaMallocManaged (UVM mode, memory.py:239-261),
 * PAGEABLE = page-aligned malloc (host-only builds, CPU tests). Memory is zero-filled. */
int cf_host_alloc(uint64_t bytes, int kind, void** out);
int cf_host_free(void* p, int kind);            /* PINNED / MANAGED */
int cf_host_free_sized(void* p, uint64_t bytes, int kind); /* any kind */
int cf_dev_alloc(cf_ctx* ctx, uint64_t bytes, void** out);
int cf_dev_free(cf_ctx* ctx, void* p);
/* Synchronous copy between any two spaces (Machine.transfer_range, memory.py:294-303), ordered
 * after all work already enqueued on the context's compute stream. */
int cf_memcpy(cf_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int cf_memcpy_async(cf_ctx* ctx, void* dst, const void* src, uint64_t bytes, void* stream);
int cf_memset(cf_ctx* ctx, void* dst, int value, uint64_t bytes);
/* Benchmark plumbing: evict the L2 by a read pass over `bytes` of device memory at buf (clean
 * lines, unlike a memset).  Synchronous on the context's compute stream. */
int cf_l2_evict(cf_ctx* ctx, const void* buf, uint64_t bytes);
/* Host-link roofline probe (no reference counterpart): plain cudaMemcpyAsync of
 * `bytes` between fresh pinned host buffers and HBM -- H2D alone, D2H alone, and H2D || D2H on
 * two streams -- each sample `iters` back-to-back copies, best of `reps` samples after one
 * warm-up.  GB/s of bytes moved (both directions summed for bidir).  The e2e window's link
 * fraction is graded against this, not against a copy pipeline shaped like its own. */
int cf_link_probe(cf_ctx* ctx, uint64_t bytes, int iters, int reps, double* h2d_gbs, double* d2h_gbs,
                  double* bidir_gbs);

/* ---------------- host marshaller (scenarios.py:122-267) ---------------- */
/* Plan the layout: allocation order, node/array tables, pointer sites (tree_total_bytes,
 * iter_*_allocations, scenarios.py:122-149). No payload is touched. */
int cf_tree_plan(const cf_spec* spec, cf_tree** out);
int cf_tree_info_get(const cf_tree* tree, cf_tree_info* out);
int cf_tree_table(const cf_tree* tree, int which, const void** ptr, uint64_t* count);
/* Write the graph into host memory at `host` (>= total_bytes): node fields, pointer fields
 * (= ptr_base + target offset) and payload_values(seed) (scenarios.py:152-252), multi-threaded.
 * ptr_base is normally (uint64_t)host. */
int cf_tree_build(const cf_tree* tree, void* host, uint64_t ptr_base, uint64_t seed, int nthreads);
/* targeted_arrays (scenarios.py:270-284) and the all-leaves / all-arrays policies: writes
 * array indices into out (capacity cap) and their number into *n. */
int cf_tree_targets(const cf_tree* tree, int policy, int64_t* out, uint64_t cap, uint64_t* n);
int cf_tree_chain_shape(const cf_tree* tree, cf_chain_shape* out);
/* UVM scheme, host side (harness.py:261-304 walk through memory.py:378-394 uvm_touch): the sorted
 * distinct pages of every pointer field the reference's kernel walk reads -- each target's Lnext
 * chain from root_off[i] (arena offsets; dense digits of ordinal[i] in base q), then the terminal
 * node's A field and, when count[i] > 0, its nA field -- reading the pointer values from the
 * arena at `arena`.  A chain leaving the arena contributes the page of its first outside field
 * and stops (the caller's page table then raises WildAccess).  out may be NULL to size the result. */
int cf_uvm_walk_pages(const void* arena, uint64_t total, int kind, uint32_t q, int32_t depth, const uint64_t* root_off,
                      const int32_t* level, const uint64_t* ordinal, const uint64_t* count, uint64_t n, uint64_t page,
                      uint64_t* out, uint64_t cap, uint64_t* npages);
int cf_tree_free(cf_tree* tree);

/* ---------------- device kernels (sm_100a) ---------------- */
/* Relocation (attach/detach) kernel: for each site s, v = *(u64*)(image+s);
 * require from_base <= v < from_base + image_bytes, write to_base + (v - from_base).
 * Attach: from = host arena base, to = device image (memory.py:316-323);
 * detach: from = image, to = host base (memory.py:337-344). Misaligned (4 mod 8) fields are
 * handled with 2 x u32 accesses. On a bad field, d_bad receives min(bad site index)
 * (initialise to UINT64_MAX). */
int cf_relocate(cf_ctx* ctx, void* image, uint64_t image_bytes, const uint64_t* d_sites,
                uint64_t nsites, uint64_t from_base, uint64_t to_base, uint64_t* d_bad,
                void* stream);
/* Pointerchain resolve kernel: one thread per chain (d_root: per-target root offset, NULL =
 * shape->root_off), walks it once in the relocated image and
 * writes its effective address + node count (targeted_arrays, scenarios.py:270-284, done on
 * the device; harness.py:228-238 pointerchain buffers). */
int cf_resolve(cf_ctx* ctx, const void* image, const cf_chain_shape* shape, const uint64_t* d_root,
               const int32_t* d_level, const uint32_t* d_ordinal, uint64_t ntargets,
               uint64_t* d_ea, uint32_t* d_count, uint64_t* d_bad, void* stream);
/* Leaf-kernel work list (device pointers).  A launch covers big parts
 * [big_begin, big_begin + big_count) -- one CTA per 16 KiB tile, tiles [tile_begin, tile_end), their
 * first tiles at tile_base[tb_begin ..) --
 * and small-part groups [group_begin, group_end) -- one CTA per group, one warp per part. */
typedef struct {
  const uint32_t* parts;      /* (target, elem_begin, elem_end) u32 triples (nA is u32) */
  const uint64_t* tile_base;  /* first tile number of every big part, big parts only */
  const uint32_t* groups;     /* (first part, end part) pairs */
  uint64_t big_begin, big_count; /* big parts: parts[big_begin ..), tile_base[tb_begin ..) */
  uint64_t tb_begin;
  uint64_t tile_begin, tile_end;
  uint64_t group_begin, group_end;
} cf_scale_work;

/* Leaf kernel (kernel_scale / _scale_block, harness.py:244-309): x *= scale over every part,
 * elem = 4 (f32) or 8 (f64).  mode CF_MODE_RESOLVED reads d_ea (from cf_resolve);
 * CF_MODE_CHASE re-walks the chain from the image root on every 16-byte access with
 * non-hoistable loads (d_ea unused).  d_bad is raised if a part exceeds the count read from
 * the node or the array pointer is null. */
int cf_scale(cf_ctx* ctx, int elem, int mode, const void* image, const cf_chain_shape* shape,
             const uint64_t* d_root, const int32_t* d_level, const uint32_t* d_ordinal, const uint64_t* d_ea,
             const uint32_t* d_count, const cf_scale_work* work, double scale, uint64_t* d_bad,
             void* stream);

/* ---------------- reference-named composite operations ---------------- */
/* Machine.marshal_transfer_and_attach (memory.py:307-325): chunked multi-stream H2D of the
 * pinned arena into `image`, relocation-table upload, per-chunk relocation as chunks land.
 * Synchronous; returns CF_E_OUTSIDE_ARENA with *bad_site = index into the sorted site table. */
int cf_marshal_transfer_and_attach(cf_ctx* ctx, const void* host_arena, uint64_t total,
                                   void* image, const uint64_t* h_sites_sorted, uint64_t nsites,
                                   uint64_t chunk_bytes, uint64_t* bad_site);
/* Machine.demarshal (memory.py:327-345): detach kernel on the image, then chunked D2H into
 * host_arena. Synchronous.  h_sites may come in any order; on a field outside the image,
 * CF_E_OUTSIDE_ARENA with *bad_site = the first offending index in table order (pass the
 * reversed DFS site order to get the reference's detach order, memory.py:337). */
int cf_demarshal(cf_ctx* ctx, void* host_arena, uint64_t total, void* image,
                 const uint64_t* h_sites, uint64_t nsites, uint64_t chunk_bytes,
                 uint64_t* bad_site);
/* kernel_scale over a device image (harness.py:244-304): resolve every target chain on the
 * device, then run the leaf kernel in `mode`. h_level/h_ordinal/h_count are host arrays of
 * the targets' chain keys and planned element counts. Synchronous; d_ea_out (optional,
 * device) receives the effective addresses. */
int cf_kernel_scale(cf_ctx* ctx, int elem, int mode, void* image, const cf_chain_shape* shape,
                    const uint64_t* h_root, const int32_t* h_level, const uint32_t* h_ordinal,
                    const uint64_t* h_count,
                    uint64_t ntargets, double scale, uint64_t* h_ea_out, uint64_t* bad);
/* kernel_scale planned once per target set (harness.py:244-304, repeated windows over one tree):
 * _create uploads the targets' chain keys / counts (and roots, optional) and the leaf-kernel work
 * list; _run resolves every chain on `image` and runs the leaf kernel in `mode` (same checks and
 * errors as cf_kernel_scale).  Synchronous. */
int cf_kernel_plan_create(cf_ctx* ctx, int elem, const uint64_t* h_root, const int32_t* h_level,
                          const uint32_t* h_ordinal, const uint64_t* h_count, uint64_t ntargets,
                          cf_kernel_plan** out);
int cf_kernel_plan_run(cf_kernel_plan* plan, int mode, void* image, const cf_chain_shape* shape, double scale,
                       uint64_t* bad);
/* Resolve only: walk every target chain on `image` and return the effective addresses (u64 device
 * addresses) and counts (u32 nA) to host arrays; errors as cf_kernel_scale's walk.  With h_ea and
 * h_count NULL after cf_kernel_plan_expect, the walk is checked on the device instead: every chain
 * must end at image + h_expect_off[t] with count h_count[t], else CF_E_WILD (bad = first target). */
int cf_kernel_plan_expect(cf_kernel_plan* plan, const uint64_t* h_expect_off, const uint64_t* h_count);
int cf_kernel_plan_resolve(cf_kernel_plan* plan, void* image, const cf_chain_shape* shape, uint64_t* h_ea,
                           uint32_t* h_count, uint64_t* bad);
int cf_kernel_plan_free(cf_kernel_plan* plan);
/* Pointerchain scheme leaf kernel over host-resolved buffers (harness.py:255-259): every
 * (h_ea[i], h_count[i]) names one device buffer copied by the selective pointerchain copy. */
int cf_scale_resolved(cf_ctx* ctx, int elem, const uint64_t* h_ea, const uint64_t* h_count, uint64_t n,
                      double scale);
/* naive_copy_back's host pointer restore (memory.py:368-372): write h_values[i] (8 bytes) at host
 * address h_addrs[i] (any 4-byte alignment), in parallel. */
int cf_host_write_words(const uint64_t* h_addrs, const uint64_t* h_values, uint64_t n);
/* The attach loop's bounds check (memory.py:319-321) on the host, before any transfer: every
 * site (arena offset, table order) must hold a pointer into [ptr_base, ptr_base + total).
 * Returns CF_E_OUTSIDE_ARENA with *bad_index = the first offending table index.  Lets a
 * deferred (fused) marshalling window raise AttachOutsideArena at transfer_to_device time. */
int cf_arena_check_sites(const void* host_arena, uint64_t total, const uint64_t* h_sites, uint64_t nsites,
                         uint64_t ptr_base, uint64_t* bad_index);
/* Result gather of the multi-GPU shards (no reference counterpart): per device
 * range i (h_addr[i], h_bytes[i], both 4-byte aligned) the position-weighted wrapping u64 sum
 * sum_j word_j * (j + 1) of its u32 words, into h_out[i].  Synchronous. */
int cf_checksum_ranges(cf_ctx* ctx, const uint64_t* h_addr, const uint64_t* h_bytes, uint64_t n, uint64_t* h_out);
/* Per-object transfers (naive_deep_copy / naive_copy_back, memory.py:358-361, 368-372; batched
 * selective copies): objects under 64 KiB whose both ends are SM-addressable (device, managed
 * or mapped pinned memory) are copied by one zero-copy kernel, one warp per object; the rest
 * by the copy engines (one cudaMemcpyAsync per object).  Synchronous. */
int cf_copy_objects(cf_ctx* ctx, void* const* dsts, const void* const* srcs, const uint64_t* sizes, uint64_t count);
/* Bulk copy by the SMs (16-byte aligned; either end may be mapped pinned host memory), async on
 * `stream` (NULL: the context's compute stream); ctas 0 = 4 per SM.  Host-link experiments. */
int cf_sm_copy(cf_ctx* ctx, void* dst, const void* src, uint64_t bytes, unsigned ctas, void* stream);
/* Diagnostics: the first leaf-kernel address fault caught by the bounds check (flag, target,
 * address, count, image, image bytes, level, ordinal); reset != 0 clears it. */
int cf_debug_info(cf_ctx* ctx, uint64_t* out8, int reset);
/* naive_deep_copy fixups (memory.py:349-365): per-object copies are issued by the caller with
 * cf_memcpy_batch; this kernel rewrites every site through a sorted interval map
 * (AddressMap.translate, memory.py:409-419) on the device. */
int cf_memcpy_batch(cf_ctx* ctx, void* const* dsts, const void* const* srcs,
                    const uint64_t* sizes, uint64_t count, void* stream);
int cf_naive_fixup(cf_ctx* ctx, const uint64_t* d_site_field_host, const uint64_t* d_site_target_host,
                   uint64_t nsites, const uint64_t* d_map_host_base, const uint64_t* d_map_size,
                   const uint64_t* d_map_dev_base, uint64_t nmap, uint64_t* d_bad, void* stream);
/* As cf_naive_fixup from host tables (uploaded into the context's scratch). Synchronous;
 * CF_E_WILD with *bad_site = the first site whose target was never copied. */
int cf_naive_fixup_host(cf_ctx* ctx, const uint64_t* h_site_field_host, const uint64_t* h_site_target_host,
                        uint64_t nsites, const uint64_t* h_map_host_base, const uint64_t* h_map_size,
                        const uint64_t* h_map_dev_base, uint64_t nmap, uint64_t* bad_site);

/* Pointerchain scheme as one pipelined window (transfer_to_device / kernel_scale / copy_back,
 * harness.py:228-238, 255-259, 312-325): n targeted arrays, host h_src[i] -> device buffer
 * d_buf[i], count[i] elements of elem bytes.  Steps of ~chunk_bytes; per step H2D, leaf kernel,
 * D2H, steps overlapped.  Arrays >= 64 KiB move on the copy engines, smaller ones by zero-copy
 * SM kernels over the mapped pinned host memory.  Run flags: CF_WIN_H2D | CF_WIN_SCALE |
 * CF_WIN_D2H (any subset).  cf_selective_run is synchronous. */
int cf_selective_plan(cf_ctx* ctx, uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count,
                      int elem, uint64_t chunk_bytes, cf_selective** out);
/* As cf_selective_plan, with a per-array scale mask (NULL = every array; 0 = copied in and back
 * but not scaled -- the naive scheme moves every object) and plan flags: CF_SEL_PER_OBJECT keeps
 * one transfer per object (no staged spans), the naive scheme's per-object semantics. */
enum { CF_SEL_PER_OBJECT = 1 };
int cf_selective_plan_ex(cf_ctx* ctx, uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count,
                         const uint8_t* scale_mask, uint32_t plan_flags, int elem, uint64_t chunk_bytes,
                         cf_selective** out);
int cf_selective_run(cf_selective* w, uint32_t flags, double scale);
int cf_selective_free(cf_selective* w);
/* Host-only dry run of cf_selective_plan + invariant check (no GPU): every array's bytes move
 * exactly once, to the right device address, and each step scales exactly what it moved.
 * mapped != 0 plans as if the host arrays were mapped (zero-copy for small arrays).  Returns
 * CF_E_STATE (first violation in cf_last_error) on a violation. */
int cf_selective_plan_check(uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count, int elem,
                            uint64_t chunk_bytes, int mapped, uint64_t* nsteps);

/* ---------------- unified memory (memory.py:239-261, 378-394) ---------------- */
/* Managed-memory hints for the UVM scheme. dst_device < 0 prefetches to the host (the
 * reference's copy-back re-touch of dirty pages, harness.py:321-325). advice: 0 = none,
 * 1 = SetPreferredLocation(device), 2 = SetAccessedBy(device), 3 = SetReadMostly; OR-ing
 * CF_UVM_UNSET applies the matching Unset advice. */
enum { CF_UVM_ADVISE_NONE = 0, CF_UVM_PREFERRED_DEVICE = 1, CF_UVM_ACCESSED_BY = 2, CF_UVM_READ_MOSTLY = 3,
       CF_UVM_UNSET = 0x100 };
int cf_uvm_prefetch(cf_ctx* ctx, const void* p, uint64_t bytes, int dst_device, void* stream);
int cf_uvm_advise(cf_ctx* ctx, const void* p, uint64_t bytes, int advice);

/* ---------------- pipelined metered window (harness.py:369-373) ---------------- */
/* Flags for the window */
enum {
  CF_WIN_H2D = 1u << 0,      /* upload the arena from host_src (else the image is resident) */
  CF_WIN_TABLES = 1u << 1,   /* upload the relocation / chain tables every run */
  CF_WIN_ATTACH = 1u << 2,   /* relocation kernel (attach) */
  CF_WIN_RESOLVE = 1u << 3,  /* pointerchain resolve kernel */
  CF_WIN_SCALE = 1u << 4,    /* leaf kernel */
  CF_WIN_DETACH = 1u << 5,   /* inverse relocation before copy-back */
  CF_WIN_D2H = 1u << 6,      /* copy the image back to host_dst */
  CF_WIN_GRAPH = 1u << 7,    /* capture the enqueue sequence into a CUDA graph once, replay */
  CF_WIN_UVM = 1u << 8,      /* managed-memory tree (image == host_src == host_dst): the H2D / D2H
                                steps become chunked cudaMemPrefetchAsync to the GPU / back to the
                                CPU on the copy streams, pipelined with resolve and leaf kernel
                                (the UVM scheme with prefetch hints, memory.py:239-261) */
  CF_WIN_TABLE_RESOLVE = 1u << 9  /* plan-time: no leaf-owned steps -- every target is resolved
                                     into the EA table and every site is listed (the table-driven
                                     design the leaf-owned path is measured against) */
};

typedef struct {
  const cf_tree* tree;        /* layout, relocation table and chain tables */
  const int64_t* h_targets;   /* array indices to consume (cf_tree_targets) */
  uint64_t ntargets;
  const void* host_src;       /* pinned arena (input) */
  void* host_dst;             /* pinned copy-back destination (may equal host_src) */
  uint64_t host_base;         /* pointer base used inside the arena (cf_tree_build ptr_base) */
  void* image;                /* device image, >= total bytes */
  int32_t mode;               /* CF_MODE_RESOLVED / CF_MODE_CHASE */
  uint32_t flags;             /* CF_WIN_* */
  double scale;
  uint64_t chunk_bytes;       /* pipeline granularity (0 = whole arena in one chunk) */
} cf_window_desc;

typedef struct {
  float ms_total;             /* device time from first enqueue to last completion */
  float ms_kernel;            /* sum of leaf-kernel launches (events around each) */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t launches;          /* kernels launched by this run */
  uint64_t bad;               /* UINT64_MAX if no error */
  uint64_t nchunks, nsteps;
} cf_window_stats;

/* Window faults: stats->bad (and the run's return code) carry one sticky word, min over the
 * window's kernels of (CF_FAULT_* << 62 | index): CF_FAULT_ATTACH (relocation-table index) and
 * CF_FAULT_DETACH (detach-list index) return CF_E_OUTSIDE_ARENA (AttachOutsideArena,
 * memory.py:319-321 / 337-343); CF_FAULT_RESOLVE (a chain hop leaves the image) and
 * CF_FAULT_SCALE (a leaf array [A, A + nA * elem) overruns the image, or a part runs past nA)
 * return CF_E_WILD (WildAccess, memory.py:139-152).  UINT64_MAX = no fault. */
enum { CF_FAULT_ATTACH = 0, CF_FAULT_RESOLVE = 1, CF_FAULT_SCALE = 2, CF_FAULT_DETACH = 3 };
#define CF_FAULT_KIND(bad) ((int)((bad) >> 62))
#define CF_FAULT_INDEX(bad) ((bad) & ((1ull << 62) - 1))
int cf_window_plan(cf_ctx* ctx, const cf_window_desc* desc, cf_window** out);
/* Host-only dry run of cf_window_plan (no GPU needed; host_src / image may be NULL) followed by
 * an invariant check of the schedule, re-derived independently where possible: segments
 * partition the arena; every site is attached once, in the step that uploads it; every target's
 * chain -- walked through the tree's site table -- has landed by its resolve step and ends at its
 * array's owner; the leaf-kernel parts tile each target's elements once, after their bytes land;
 * no segment is detached or copied back before its last reader or writer.  Leaf-owned ranges
 * (steps whose whole small leaf arrays form one run of consecutive ordinals: the leaf kernel
 * attaches, streams and detaches them, and they appear in no table) are checked too: table sites
 * plus owned A fields are every site exactly once, each owned target lies in its step's range
 * with that range's count, after its bytes and chain, and its record stays on the device until
 * its leaf kernel ran.  Returns CF_E_STATE (first violation in cf_last_error) if any invariant
 * fails. */
typedef struct {
  uint64_t nsteps, nsegments, nsites, ntargets, nparts, ngroups, ntiles, table_bytes, zero_copy_node_segments;
  int32_t violations;
  int32_t leaf_owned;   /* 1: the leaf kernel owns the targets' A-field relocation (one-step uniform windows) */
  double plan_ms;
} cf_plan_check;
int cf_window_plan_check(const cf_window_desc* desc, cf_plan_check* out);
/* Enqueue one window; if sync != 0 wait and fill stats (ms from CUDA events). */
int cf_window_run(cf_window* w, int sync, cf_window_stats* stats);
/* Enqueue nruns windows back to back (scale alternating scale_even / scale_odd, e.g. 2.0 / 0.5
 * so the data stays bounded), then wait: stats cover the whole sequence (benchmark timing). */
int cf_window_run_n(cf_window* w, int nruns, double scale_even, double scale_odd, cf_window_stats* stats);
/* As cf_window_run_n, alternating two windows planned alike over different images / copy-back
 * buffers: window r+1 starts copying in while window r is still copying out (each window runs on
 * its own stream; the copy engines' streams are shared). */
int cf_window_run_pair(cf_window* w0, cf_window* w1, int nruns, double scale_even, double scale_odd,
                       cf_window_stats* stats);
/* As cf_window_run_pair over a ring of nw windows planned alike (own images / copy-back buffers,
 * own streams): run r uses ws[r % nw].  Small graphs rotate over images whose total exceeds the
 * L2, so no step finds its data cached by an earlier one while the steps still overlap. */
int cf_window_run_ring(cf_window* const* ws, int nw, int nruns, double scale_even, double scale_odd,
                       cf_window_stats* stats);
/* As cf_window_run_n for working sets that fit the L2: before every window, a read pass over
 * flush_bytes at flush_buf (device) evicts the L2 (clean lines: nothing of the flush is written
 * back inside the timed window); stats->ms_total is the sum of the windows' own intervals (CUDA
 * events after each flush and after each window), flushes excluded. */
int cf_window_run_n_flushed(cf_window* w, int nruns, double scale_even, double scale_odd, void* flush_buf,
                            uint64_t flush_bytes, cf_window_stats* stats);
int cf_window_set_scale(cf_window* w, double scale);
/* Diagnostics (tests): CF_WIN_DEBUG_KEEP_LEAF_ATTACHED makes the leaf kernel of leaf-owned steps
 * skip the detach of the A fields it attached, so the image (and a copy-back) shows the device
 * addresses it wrote -- evidence that leaf-owned relocation attaches.  Drops the window's cached
 * graphs.  0 restores normal windows. */
enum { CF_WIN_DEBUG_KEEP_LEAF_ATTACHED = 1 };
int cf_window_debug(cf_window* w, uint32_t flags);
int cf_window_free(cf_window* w);

#ifdef __cplusplus
}
#endif
#endif /* CHAINFORGE_B200_H */
