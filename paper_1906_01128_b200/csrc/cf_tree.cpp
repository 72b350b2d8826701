// Host marshaller: plans the graph layout (allocation order, node/array tables, relocation
// table) and writes the graph into a host arena with multi-threaded payload initialisation.
//
// Semantics follow the reference builders exactly so that a packed (align = 1) plan is
// byte-identical to the reference arena (pinned by tests against tests/golden):
//   iter_linear_allocations / iter_dense_allocations / tree_total_bytes  scenarios.py:122-149
//   build_linear_tree / build_dense_tree (field writes, site order)      scenarios.py:164-252
//   payload_values                                                        scenarios.py:152-155
//   Arena.allocate (packed) / MemorySpace.allocate (8-byte bump)          memory.py:217-227, 124-137
//   targeted_arrays                                                       scenarios.py:270-284
// The planner is an explicit-stack traversal over the tree shape; the builder writes node
// records and pointer fields from the plan tables and fills payload in parallel (OpenMP),
// which is what takes seconds in the reference (10-18 s at C2/C4).
#include "cf_internal.h"

#include <algorithm>
#include <cstring>
#include <new>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace cf;

namespace {

uint64_t round_up(uint64_t x, uint64_t a) { return a <= 1 ? x : (x + a - 1) / a * a; }

struct Planner {
  cf_tree* t;
  uint64_t cursor = 0;
  uint64_t tree = 0;   // index of the tree being planned
  uint64_t root = 0;   // its root offset

  uint64_t alloc(uint64_t size, int64_t array_index) {
    uint64_t off = round_up(cursor, uint64_t(t->spec.align));
    cursor = off + size;
    t->alloc_off.push_back(off);
    t->alloc_size.push_back(size);
    t->alloc_array.push_back(array_index);
    t->served += size;
    return off;
  }

  void node(uint64_t off, int level, uint32_t size, uint32_t na, int64_t nlnext, uint64_t ordinal = 0) {
    t->node_off.push_back(off);
    t->node_level.push_back(level);
    t->node_size.push_back(size);
    t->node_na.push_back(na);
    t->node_nlnext.push_back(nlnext);
    auto& ln = t->level_nodes[tree];
    auto& lb = t->level_base[tree];
    if (int(ln.size()) <= level) { ln.resize(level + 1); lb.resize(level + 1, 0); }
    if (ln[level].empty()) lb[level] = ordinal;
    ln[level].push_back(off);
  }

  int64_t array(int level, uint64_t owner, uint64_t count, uint64_t ordinal) {
    int64_t idx = int64_t(t->arr_off.size());
    uint64_t off = alloc(uint64_t(t->spec.elem) * count, idx);
    t->arr_level.push_back(level);
    t->arr_owner.push_back(owner);
    t->arr_off.push_back(off);
    t->arr_count.push_back(count);
    t->arr_ordinal.push_back(ordinal);
    t->arr_tree.push_back(tree);
    t->arr_root.push_back(root);
    t->payload_bytes += uint64_t(t->spec.elem) * count;
    return idx;
  }

  void site(uint64_t field, uint64_t target) {
    t->site_off.push_back(field);
    t->site_target.push_back(target);
  }

  // Linear: allocations (node, then its array) level by level; fields afterwards.
  void linear() {
    const cf_spec& s = t->spec;
    const int64_t k = s.k_or_q;
    const bool allinit = s.layout != CF_LLINIT_LLUSED;
    std::vector<uint64_t> nodes(k);
    std::vector<int64_t> arr(k, -1);
    for (int64_t lv = 0; lv < k; ++lv) {
      nodes[lv] = alloc(NODE_SIZE, -1);
      if (lv == 0) root = nodes[0];
      if (s.n > 0 && (allinit || lv == k - 1)) arr[lv] = array(int(lv), nodes[lv], uint64_t(s.n), 0);
    }
    for (int64_t lv = 0; lv < k; ++lv) {
      node(nodes[lv], int(lv), NODE_SIZE, arr[lv] >= 0 ? uint32_t(s.n) : 0u, lv < k - 1 ? 1 : 0);
      if (arr[lv] >= 0) site(nodes[lv] + OFF_A, t->arr_off[arr[lv]]);
      if (lv < k - 1) site(nodes[lv] + OFF_LNEXT, nodes[lv + 1]);
    }
  }

  // Dense: explicit-stack pre-order traversal.  A frame is a node whose array/block have not
  // been emitted yet; children are pushed in reverse so they pop in order.
  void dense() {
    const cf_spec& s = t->spec;
    const int64_t D = s.depth;
    const uint64_t q = uint64_t(s.k_or_q);
    struct Frame { uint64_t off; int level; uint64_t ordinal; };
    std::vector<Frame> stack;
    // subtree shard: cut level sl = shallowest with q^sl >= world (sl = 0, width 1: whole tree)
    const uint64_t world = s.shard_world > 1 ? uint64_t(s.shard_world) : 1, rank = uint64_t(s.shard_rank);
    int sl = 0;
    uint64_t width = 1;   // q^sl
    while (width < world) { width *= q; ++sl; }
    root = alloc(D > 0 ? NODE_SIZE : LEAF_NODE_SIZE, -1);
    stack.push_back({root, 0, 0});
    while (!stack.empty()) {
      Frame f = stack.back();
      stack.pop_back();
      const bool leaf = f.level == D;
      if (world > 1 && f.level == sl && f.ordinal * world / width != rank) {
        // another rank's subtree: the record stays in its parent's block, fields nulled
        node(f.off, f.level, leaf ? LEAF_NODE_SIZE : NODE_SIZE, 0u, leaf ? -1 : 0, f.ordinal);
        continue;
      }
      const bool has_array = s.n > 0 && (!s.leaf_only || leaf) && (f.level >= sl || rank == 0);
      node(f.off, f.level, leaf ? LEAF_NODE_SIZE : NODE_SIZE, has_array ? uint32_t(s.n) : 0u,
           leaf ? -1 : int64_t(q), f.ordinal);
      if (has_array) {
        int64_t a = array(f.level, f.off, uint64_t(s.n), f.ordinal);
        site(f.off + (leaf ? LEAF_OFF_A : OFF_A), t->arr_off[a]);
      }
      if (!leaf) {
        const uint64_t child = (f.level + 1 < D) ? NODE_SIZE : LEAF_NODE_SIZE;
        uint64_t block = alloc(q * child, -1);
        site(f.off + OFF_LNEXT, block);
        for (uint64_t j = q; j-- > 0;)
          stack.push_back({block + j * child, f.level + 1, f.ordinal * q + j});
      }
    }
  }
};

uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Sparse layout: place the allocations in a seeded random order (same sizes / alignment) and
// move every recorded offset with its allocation.
void scatter(cf_tree* t, uint64_t seed) {
  const size_t m = t->alloc_off.size();
  std::vector<size_t> perm(m);
  for (size_t i = 0; i < m; ++i) perm[i] = i;
  uint64_t st = seed;
  for (size_t i = m; i > 1; --i) std::swap(perm[i - 1], perm[splitmix(st) % i]);
  std::vector<uint64_t> neu(m);
  uint64_t cur = 0;
  for (size_t k = 0; k < m; ++k) {
    const size_t i = perm[k];
    const uint64_t off = round_up(cur, uint64_t(t->spec.align));
    neu[i] = off;
    cur = off + t->alloc_size[i];
  }
  const std::vector<uint64_t> old = t->alloc_off;  // ascending (bump order)
  auto remap = [&](uint64_t off) {
    const size_t i = size_t(std::upper_bound(old.begin(), old.end(), off) - old.begin()) - 1;
    return neu[i] + (off - old[i]);
  };
  for (auto* v : {&t->node_off, &t->arr_owner, &t->arr_off, &t->arr_root, &t->site_off, &t->site_target,
                  &t->tree_root})
    for (auto& x : *v) x = remap(x);
  for (auto& tree : t->level_nodes)
    for (auto& lv : tree)
      for (auto& x : lv) x = remap(x);
  t->root_off = remap(t->root_off);
  t->alloc_off = neu;
  t->total = cur;
}

void fill_payload(uint8_t* host, const cf_tree* t, uint64_t seed31, int nthreads) {
  // payload_values (scenarios.py:152-155): raw_i = (seed*16777619 + level*1000003 + i) mod 2^31,
  // stored as f64 or as the round-to-nearest f32 of raw_i.  Work is split into 1 MiB pieces
  // across all arrays so that both 64 huge leaves and 1M small arrays balance.
  const uint64_t M = (1ull << 31) - 1;
  const int e = t->spec.elem;
  const uint64_t piece = (1ull << 20) / uint64_t(e);
  std::vector<uint64_t> first_piece(t->arr_off.size() + 1, 0);
  for (size_t a = 0; a < t->arr_off.size(); ++a)
    first_piece[a + 1] = first_piece[a] + (t->arr_count[a] + piece - 1) / piece;
  const int64_t npieces = int64_t(first_piece.back());
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int64_t p = 0; p < npieces; ++p) {
    size_t a = size_t(std::upper_bound(first_piece.begin(), first_piece.end(), uint64_t(p)) -
                      first_piece.begin()) - 1;
    uint64_t i0 = (uint64_t(p) - first_piece[a]) * piece;
    uint64_t i1 = std::min(t->arr_count[a], i0 + piece);
    uint64_t b = (seed31 * 16777619ull + uint64_t(t->arr_level[a]) * 1000003ull) & M;
    uint8_t* dst = host + t->arr_off[a];
    if (e == 8) {
      if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
        double* d = reinterpret_cast<double*>(dst);
        for (uint64_t i = i0; i < i1; ++i) d[i] = double((b + i) & M);
      } else {
        for (uint64_t i = i0; i < i1; ++i) { double v = double((b + i) & M); memcpy(dst + 8 * i, &v, 8); }
      }
    } else {
      float* d = reinterpret_cast<float*>(dst);
      for (uint64_t i = i0; i < i1; ++i) d[i] = float(int64_t((b + i) & M));
    }
  }
}

}  // namespace

extern "C" {

int cf_tree_plan(const cf_spec* spec, cf_tree** out) {
  if (!spec || !out) return fail(CF_E_INVALID, "null argument");
  const cf_spec& s = *spec;
  if (s.kind != CF_LINEAR && s.kind != CF_DENSE) return fail(CF_E_INVALID, "unknown kind %d", s.kind);
  if (s.kind == CF_LINEAR && s.k_or_q < 1) return fail(CF_E_INVALID, "k must be >= 1");
  if (s.kind == CF_DENSE && s.k_or_q < 1) return fail(CF_E_INVALID, "q must be >= 1");
  if (s.n < 0) return fail(CF_E_INVALID, "n must be >= 0");
  if (s.kind == CF_DENSE && s.depth < 0) return fail(CF_E_INVALID, "depth must be >= 0");
  if (s.kind == CF_LINEAR && (s.layout < 0 || s.layout > 2)) return fail(CF_E_INVALID, "unknown layout");
  if (s.elem != 4 && s.elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  if (s.align != 1 && s.align != 4 && s.align != 8 && s.align != 16 && s.align != 64 && s.align != 128)
    return fail(CF_E_INVALID, "align must be 1, 4, 8, 16, 64 or 128");
  if (s.shard_world > 1) {
    if (s.kind != CF_DENSE || s.forest > 1 || s.scatter_seed)
      return fail(CF_E_INVALID, "subtree shards are defined for single dense trees");
    if (s.shard_rank < 0 || s.shard_rank >= s.shard_world) return fail(CF_E_INVALID, "shard rank out of range");
    double leaves = 1;
    for (int64_t l = 0; l < s.depth; ++l) leaves *= double(s.k_or_q);
    if (leaves < double(s.shard_world))
      return fail(CF_E_INVALID, "q^depth = %.0f subtrees cannot be split over %d shards", leaves, s.shard_world);
  }
  if (s.kind == CF_DENSE) {
    // guard the node count: sum q^l for l <= D must fit comfortably in memory
    double nodes = 0, p = 1;
    for (int64_t l = 0; l <= s.depth; ++l, p *= double(s.k_or_q)) nodes += p;
    if (nodes > 4e8) return fail(CF_E_OOM, "dense tree with %.3g nodes is too large to plan", nodes);
  }
  cf_tree* t = new (std::nothrow) cf_tree();
  if (!t) return fail(CF_E_OOM, "out of host memory");
  t->spec = s;
  const uint64_t ntrees = s.forest > 1 ? uint64_t(s.forest) : 1;
  t->level_nodes.resize(ntrees);
  t->level_base.resize(ntrees);
  Planner pl{t};
  for (uint64_t f = 0; f < ntrees; ++f) {
    pl.tree = f;
    if (s.kind == CF_LINEAR) pl.linear();
    else pl.dense();
    t->tree_root.push_back(pl.root);
  }
  t->root_off = t->tree_root[0];
  t->total = pl.cursor;
  if (s.scatter_seed) scatter(t, s.scatter_seed);
  t->site_sorted = t->site_off;
  std::sort(t->site_sorted.begin(), t->site_sorted.end());
  *out = t;
  return CF_OK;
}

int cf_tree_info_get(const cf_tree* t, cf_tree_info* out) {
  if (!t || !out) return fail(CF_E_INVALID, "null argument");
  out->total_bytes = t->total;
  out->nallocs = t->alloc_off.size();
  out->nnodes = t->node_off.size();
  out->narrays = t->arr_off.size();
  out->nsites = t->site_off.size();
  out->ntrees = t->tree_root.size();
  out->root_off = t->root_off;
  out->payload_bytes = t->payload_bytes;
  out->padding_bytes = t->total - t->served;
  return CF_OK;
}

int cf_tree_table(const cf_tree* t, int which, const void** ptr, uint64_t* count) {
  if (!t || !ptr || !count) return fail(CF_E_INVALID, "null argument");
#define TAB(id, vec)            \
  case id:                      \
    *ptr = (vec).data();        \
    *count = (vec).size();      \
    return CF_OK;
  switch (which) {
    TAB(CF_TAB_ALLOC_OFF, t->alloc_off)
    TAB(CF_TAB_ALLOC_SIZE, t->alloc_size)
    TAB(CF_TAB_NODE_OFF, t->node_off)
    TAB(CF_TAB_NODE_LEVEL, t->node_level)
    TAB(CF_TAB_NODE_SIZE, t->node_size)
    TAB(CF_TAB_ARR_LEVEL, t->arr_level)
    TAB(CF_TAB_ARR_OWNER, t->arr_owner)
    TAB(CF_TAB_ARR_OFF, t->arr_off)
    TAB(CF_TAB_ARR_COUNT, t->arr_count)
    TAB(CF_TAB_SITE_OFF, t->site_off)
    TAB(CF_TAB_SITE_TARGET, t->site_target)
    TAB(CF_TAB_SITE_SORTED, t->site_sorted)
    TAB(CF_TAB_ARR_ORDINAL, t->arr_ordinal)
    TAB(CF_TAB_ARR_ROOT, t->arr_root)
    TAB(CF_TAB_TREE_ROOT, t->tree_root)
    default:
      return fail(CF_E_INVALID, "unknown table %d", which);
  }
#undef TAB
}

int cf_tree_build(const cf_tree* t, void* host, uint64_t ptr_base, uint64_t seed, int nthreads) {
  if (!t || !host) return fail(CF_E_INVALID, "null argument");
  uint8_t* h = static_cast<uint8_t*>(host);
  // 1. zero everything that is not array payload: node blocks and alignment gaps
  //    (the reference storage is zero-filled, memory.py:135)
  std::vector<size_t> order(t->alloc_off.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return t->alloc_off[x] < t->alloc_off[y]; });
  uint64_t prev_end = 0;
  for (size_t i : order) {
    const uint64_t off = t->alloc_off[i];
    if (off > prev_end) memset(h + prev_end, 0, off - prev_end);
    if (t->alloc_array[i] < 0) memset(h + off, 0, t->alloc_size[i]);
    prev_end = off + t->alloc_size[i];
  }
  // 2. node scalar fields (nA always; nLnext where the node has one)
  for (size_t i = 0; i < t->node_off.size(); ++i) {
    const uint64_t off = t->node_off[i];
    memcpy(h + off + OFF_NA, &t->node_na[i], 4);
    if (t->node_nlnext[i] >= 0) {
      uint32_t v = uint32_t(t->node_nlnext[i]);
      memcpy(h + off + OFF_NLNEXT, &v, 4);
    }
  }
  // 3. pointer fields: host addresses of their targets
  for (size_t i = 0; i < t->site_off.size(); ++i) {
    uint64_t v = ptr_base + t->site_target[i];
    memcpy(h + t->site_off[i], &v, 8);
  }
  // 4. payload
  fill_payload(h, t, seed & ((1ull << 31) - 1), nthreads);
  return CF_OK;
}

int cf_tree_targets(const cf_tree* t, int policy, int64_t* out, uint64_t cap, uint64_t* n) {
  if (!t || !n) return fail(CF_E_INVALID, "null argument");
  std::vector<int64_t> idx;
  const cf_spec& s = t->spec;
  const size_t na = t->arr_off.size();
  if (policy == CF_TARGET_ALL_ARRAYS) {
    for (size_t i = 0; i < na; ++i) idx.push_back(int64_t(i));
  } else if (s.kind == CF_LINEAR) {
    for (size_t i = 0; i < na; ++i)
      if (s.layout == CF_ALLINIT_ALLUSED || t->arr_level[i] == s.k_or_q - 1) idx.push_back(int64_t(i));
  } else if (policy == CF_TARGET_ALL_LEAVES) {
    for (size_t i = 0; i < na; ++i)
      if (t->arr_level[i] == s.depth) idx.push_back(int64_t(i));
  } else if (policy == CF_TARGET_REF) {
    // per tree: the leaf reached by always taking the last child (scenarios.py:277-284)
    for (size_t f = 0; f < t->tree_root.size(); ++f) {
      const auto& leaves = t->level_nodes[f][s.depth];
      const uint64_t node = leaves.back();
      if (s.shard_world > 1) {   // the reference target lives on the shard owning the last leaf
        uint64_t last = 1;
        for (int64_t l = 0; l < s.depth; ++l) last *= uint64_t(s.k_or_q);
        bool mine = false;
        for (size_t i = 0; i < na; ++i)
          if (t->arr_owner[i] == node && t->arr_ordinal[i] == last - 1) mine = true;
        if (!mine) continue;
      }
      for (size_t i = 0; i < na; ++i)
        if (t->arr_tree[i] == f && t->arr_owner[i] == node) idx.push_back(int64_t(i));
    }
  } else {
    return fail(CF_E_INVALID, "unknown target policy %d", policy);
  }
  *n = idx.size();
  if (out) {
    if (cap < idx.size()) return fail(CF_E_INVALID, "target buffer too small (%llu < %zu)",
                                      (unsigned long long)cap, idx.size());
    std::copy(idx.begin(), idx.end(), out);
  }
  return CF_OK;
}

int cf_tree_chain_shape(const cf_tree* t, cf_chain_shape* out) {
  if (!t || !out) return fail(CF_E_INVALID, "null argument");
  memset(out, 0, sizeof *out);
  out->kind = t->spec.kind;
  out->depth = t->spec.kind == CF_DENSE ? int32_t(t->spec.depth) : int32_t(t->spec.k_or_q - 1);
  out->q = t->spec.kind == CF_DENSE ? uint32_t(t->spec.k_or_q) : 1u;
  out->root_off = t->root_off;
  out->image_bytes = t->total;
  return CF_OK;
}

int cf_uvm_walk_pages(const void* arena, uint64_t total, int kind, uint32_t q, int32_t depth, const uint64_t* root_off,
                      const int32_t* level, const uint64_t* ordinal, const uint64_t* count, uint64_t n, uint64_t page,
                      uint64_t* out, uint64_t cap, uint64_t* npages) {
  if (!npages || (n && (!arena || !root_off || !level || !ordinal || !count)) || page == 0)
    return fail(CF_E_INVALID, "bad arguments");
  const uint8_t* a = static_cast<const uint8_t*>(arena);
  const uint64_t base = reinterpret_cast<uint64_t>(arena);
  const bool dense = kind == CF_DENSE;
  const uint64_t p0 = base / page, np = (base + total + page - 1) / page - p0;
  std::vector<uint8_t> hit(np, 0);          // pages inside the arena (benign same-value races)
  std::vector<std::vector<uint64_t>> wild;   // per thread: pages of fields outside the arena
  int nthr = 1;
#ifdef _OPENMP
  nthr = n > (1u << 14) ? omp_get_max_threads() : 1;
#endif
  wild.resize(size_t(nthr));
#pragma omp parallel num_threads(nthr)
  {
    int me = 0;
#ifdef _OPENMP
    me = omp_get_thread_num();
#endif
    auto mark = [&](uint64_t off) {   // the page of the 8-byte field at arena offset off
      const uint64_t pg = (base + off) / page;
      if (pg >= p0 && pg - p0 < np) hit[pg - p0] = 1;
      else wild[size_t(me)].push_back(pg);
    };
#pragma omp for schedule(static)
    for (int64_t ii = 0; ii < int64_t(n); ++ii) {
      const uint64_t i = uint64_t(ii);
      const int L = level[i];
      uint64_t node = root_off[i];
      uint64_t pw = 1;
      if (dense)
        for (int l = 1; l < L; ++l) pw *= q;
      bool ok = true;
      for (int l = 1; l <= L && ok; ++l) {
        const uint64_t f = node + OFF_LNEXT;
        mark(f);
        if (f + 8 > total) { ok = false; break; }   // a wild chain: its next field is outside
        uint64_t v;
        memcpy(&v, a + f, 8);
        const uint64_t blk = v - base;   // wraps for values below the arena
        if (dense) {
          const uint64_t digit = (ordinal[i] / pw) % q;
          pw = pw >= q ? pw / q : 1;
          node = blk + digit * ((l == depth) ? LEAF_NODE_SIZE : NODE_SIZE);
        } else {
          node = blk;
        }
      }
      if (!ok) continue;
      const bool leaf = dense && L == depth;
      mark(node + (leaf ? LEAF_OFF_A : OFF_A));
      if (count[i]) mark(node + OFF_NA);
    }
  }
  uint64_t k = 0;
  std::vector<uint64_t> extra;
  for (auto& v : wild) extra.insert(extra.end(), v.begin(), v.end());
  std::sort(extra.begin(), extra.end());
  extra.erase(std::unique(extra.begin(), extra.end()), extra.end());
  // sorted output: wild pages below the arena, the arena's pages, wild pages above
  auto emit = [&](uint64_t pg) { if (out && k < cap) out[k] = pg; ++k; };
  size_t x = 0;
  for (; x < extra.size() && extra[x] < p0; ++x) emit(extra[x]);
  for (uint64_t j = 0; j < np; ++j)
    if (hit[j]) emit(p0 + j);
  for (; x < extra.size(); ++x) emit(extra[x]);
  *npages = k;
  return (out && k > cap) ? fail(CF_E_INVALID, "page buffer too small (%llu needed)", (unsigned long long)k) : CF_OK;
}

int cf_tree_free(cf_tree* t) {
  delete t;
  return CF_OK;
}

}  // extern "C"
