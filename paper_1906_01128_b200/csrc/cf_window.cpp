// Pipelined metered window: the reference's transfer_to_device -> kernel_scale -> copy_back
// (harness.py:369-373, marshalling scheme + device pointerchain) as one planned, multi-stream
// schedule on a B200.
//
// The arena is cut into segments (boundaries never split a pointer field) grouped into steps
// that are uploaded in order.  When the graph has few node allocations, all node records are
// hoisted into step 0 (tiny copies) so every chain is resolvable before the first array chunk
// lands, whatever the placement (scattered C3 layouts); array data follows in 16 MiB chunks.
// Step c of the schedule, on the compute stream, after step c's segments have landed:
//   1. relocate (attach) the sites inside them                          memory.py:316-323
//   2. resolve the targets whose chain fields have all landed            scenarios.py:270-284
//   3. scale the array pieces that are ready at step c                   harness.py:307-309
//   4. detach every segment whose last reader ran at step <= c, then
//      copy it home on the D2H stream                                    memory.py:327-345
// H2D copies alternate over the context's copy streams, D2H runs concurrently on its own
// stream, so copy-in, compute and copy-out overlap over the full-duplex host link.  All
// dependency bookkeeping (ready / release steps) is computed once here on the host; a run is
// only enqueues.  The tables the device needs are packed into one pinned block and uploaded
// at the start of every run (CF_WIN_TABLES), since in a real deep copy they travel with the
// arena.
#include "cf_internal.h"

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

using namespace cf;

struct cf_window {
  cf_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;       // the window's own compute stream (pairs overlap)
  cudaEvent_t ev_fan = nullptr;        // fan-in/fan-out with the context's compute stream
  cf_window_desc d{};
  cf_chain_shape sh{};
  int elem = 8;
  uint64_t total = 0;
  uint64_t nsteps = 0;
  std::vector<uint64_t> seg_lo, seg_hi;          // segments in upload order
  std::vector<uint64_t> step_seg_lo;             // segments of step k: [step_seg_lo[k], step_seg_lo[k+1])
  std::vector<uint64_t> reloc_lo;      // attach-site ranges per step (sites grouped by step)
  // per step: how many of the step's sites the attach CTAs of a one-launch attach || resolve take;
  // the rest (misaligned leaf A fields of targets resolved at the same step) are attached by their
  // own resolver thread, the only reader of that field in the launch
  std::vector<uint64_t> attach_n;
  bool owned_attach = false;
  std::vector<uint64_t> res_lo;        // resolve-target ranges per step
  std::vector<UniTargets> uni;         // per step: the resolve range is uniform (no table reads)
  // leaf-owned relocation (LeafOwn): per step, a consecutive range of leaf targets whose whole
  // arrays are scaled at that step; the leaf kernel attaches / detaches their A fields itself, so
  // they appear in no table (no site, no resolve entry, no part).  Planned only when the window
  // runs all four device phases (flags are fixed at plan time).
  bool own_any = false;
  std::vector<LeafOwn> own_step;       // per step (on == 0: none)
  uint64_t parent_base = 0;            // parent ordinal of d_parent[0]
  uint64_t own_parents = 0;            // d_parent entries
  uint32_t debug = 0;                  // CF_WIN_DEBUG_* (cf_window_debug)
  uint64_t* d_parent = nullptr;
  std::vector<cf_scale_work> seg;      // leaf-kernel work per step (device pointers set at plan)
  std::vector<uint64_t> det_lo;        // detach-site ranges per step
  std::vector<std::vector<uint32_t>> released;  // segments whose copy-back may start after step k
  // zero-copy node transfers (scattered layouts): step 0's node segments are pulled from the
  // mapped host arena by one kernel, and pushed back by one kernel per release step
  bool zc = false;
  uint64_t zc_n = 0;                   // node segments in step 0
  std::vector<uint64_t> zc_rel_lo;     // per step: range in the release-ordered node-seg list
  uint64_t off_zc_h2d = 0, off_zc_d2h = 0;
  // one pinned table block and its device mirror
  uint8_t* h_tab = nullptr;
  uint8_t* d_tab = nullptr;
  uint64_t tab_bytes = 0;
  uint64_t off_sites = 0, off_det = 0, off_level = 0, off_ord = 0, off_root = 0, off_parts = 0, off_tb = 0,
           off_grp = 0;
  uint64_t* d_ea = nullptr;
  uint32_t* d_count = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_rel;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_join = nullptr, ev_first = nullptr, ev_tables = nullptr;
  std::vector<cudaEvent_t> ev_k0, ev_k1;   // leaf-kernel timing per step
  uint64_t nsites = 0;
  bool has_roots = false;
  // every pointer field 8-byte aligned: a field read while the attach rewrites it is then one
  // single-copy-atomic 64-bit access, so attach || resolve in one launch is safe.  Not implied
  // by an aligned arena: 12-byte dense leaf records put every other leaf's A field at 4 mod 8
  // (2 x u32 accesses, which a concurrent attach can tear).
  bool aligned8 = false;
  bool wide_ok = false;    // aligned8, or every misaligned field is a leaf A field (owned attach)
  // CF_WIN_GRAPH: one instantiated graph per scale value (run_n alternates two scales)
  struct Graph { double scale; cudaGraphExec_t exec; uint64_t h2d, d2h, launches; };
  std::vector<Graph> graphs;
  // dry run (cf_window_plan_check): the host plan kept for the invariant checker, no CUDA state
  struct Dry {
    std::vector<uint64_t> reloc, torder, ready, release, seg_step, part_step;
    std::vector<uint32_t> det;
    std::vector<uint8_t> owned;   // per target (desc order): resolver attaches its own A field
    std::vector<uint64_t> lown;   // per target: step whose leaf kernel owns its relocation (nsteps: none)
    cf::ScaleWork sw;
  };
  Dry* dry = nullptr;
};

namespace {

// Address -> segment lookup over segments sorted by start address.
struct SegIndex {
  std::vector<uint64_t> lo;    // sorted starts
  std::vector<uint32_t> seg;   // segment id of each start
  uint32_t at(uint64_t off) const {
    return seg[size_t(std::upper_bound(lo.begin(), lo.end(), off) - lo.begin()) - 1];
  }
};

// Hoist node records into their own leading step when there are few node allocations.
constexpr uint64_t HOIST_MAX_NODE_ALLOCS = 4096;
constexpr uint64_t HOIST_MERGE_GAP = 64;
#ifndef CF_HOIST_PAGE
#define CF_HOIST_PAGE 4096
#endif
constexpr uint64_t HOIST_PAGE = CF_HOIST_PAGE;
// More hoisted node segments than this move by zero-copy kernels instead of one DMA each.
constexpr uint64_t ZC_MIN_SEGS = 16;

// One piece of a target's array: elements [b, e) of target t, scaled at upload step `step`.
struct Part { uint64_t t, b, e, step; };

// Stable bucket order of [0, key.size()) by key (< nk): order = indices grouped by key, lo[c] =
// first position whose key >= c (lo has nk + 1 entries).
void bucket_order(const std::vector<uint64_t>& key, uint64_t nk, std::vector<uint64_t>& order,
                  std::vector<uint64_t>& lo) {
  lo.assign(nk + 1, 0);
  for (uint64_t k : key) ++lo[k + 1];
  for (uint64_t c = 0; c < nk; ++c) lo[c + 1] += lo[c];
  std::vector<uint64_t> at(lo.begin(), lo.end() - 1);
  order.resize(key.size());
  for (uint64_t i = 0; i < key.size(); ++i) order[at[key[i]]++] = i;
}

void destroy(cf_window* w) {
  if (!w) return;
  if (w->dry) {   // host-only plan: no CUDA resources were created
    delete w->dry;
    delete w;
    return;
  }
  CfDevice g(w->ctx);
  if (w->h_tab) cudaFreeHost(w->h_tab);
  if (w->d_tab) cudaFree(w->d_tab);
  if (w->d_ea) cudaFree(w->d_ea);
  if (w->d_count) cudaFree(w->d_count);
  if (w->d_parent) cudaFree(w->d_parent);
  for (auto e : w->ev_h2d) cudaEventDestroy(e);
  for (auto e : w->ev_rel) cudaEventDestroy(e);
  for (auto e : w->ev_k0) cudaEventDestroy(e);
  for (auto e : w->ev_k1) cudaEventDestroy(e);
  if (w->ev_start) cudaEventDestroy(w->ev_start);
  if (w->ev_end) cudaEventDestroy(w->ev_end);
  if (w->ev_join) cudaEventDestroy(w->ev_join);
  if (w->ev_first) cudaEventDestroy(w->ev_first);
  if (w->ev_tables) cudaEventDestroy(w->ev_tables);
  for (auto& gr : w->graphs) cudaGraphExecDestroy(gr.exec);
  if (w->ev_fan) cudaEventDestroy(w->ev_fan);
  if (w->stream) cudaStreamDestroy(w->stream);
  delete w;
}

}  // namespace

extern "C" {

namespace {
int plan_impl(cf_ctx* ctx, const cf_window_desc* desc, cf_window** out, bool dry);
}

int cf_window_plan(cf_ctx* ctx, const cf_window_desc* desc, cf_window** out) {
  if (!ctx) return fail(CF_E_INVALID, "null argument");
  return plan_impl(ctx, desc, out, false);
}

namespace {
int plan_impl(cf_ctx* ctx, const cf_window_desc* desc, cf_window** out, bool dry) {
  if (!desc || !out || !desc->tree) return fail(CF_E_INVALID, "null argument");
  const cf_tree* t = desc->tree;
  const uint32_t fl = desc->flags;
  if ((fl & CF_WIN_UVM) && (desc->host_src != desc->image || desc->host_dst != desc->image || (fl & (CF_WIN_ATTACH | CF_WIN_DETACH | CF_WIN_GRAPH))))
    return fail(CF_E_INVALID, "UVM window: one managed buffer for host and image, no relocation, no graph capture");
  if ((fl & CF_WIN_H2D) && !desc->host_src && !dry) return fail(CF_E_INVALID, "H2D needs host_src");
  if ((fl & CF_WIN_D2H) && !desc->host_dst && !dry) return fail(CF_E_INVALID, "D2H needs host_dst");
  if (!desc->image && !dry) return fail(CF_E_INVALID, "null image");
  if (desc->ntargets && !desc->h_targets) return fail(CF_E_INVALID, "null targets");
  CfDevice g(dry ? nullptr : ctx);
  // CF_PLAN_PROFILE=1: phase times of the planner on stderr
  static const bool prof = getenv("CF_PLAN_PROFILE") != nullptr;
  auto tp0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!prof) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[cf_window_plan] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - tp0).count());
    tp0 = now;
  };
  cf_window* w = new cf_window();
  w->ctx = ctx;
  w->d = *desc;
  if (dry) w->dry = new cf_window::Dry();
  w->elem = t->spec.elem;
  cf_tree_chain_shape(t, &w->sh);
  const uint64_t total = t->total;
  const uint64_t nsites = t->site_sorted.size();
  w->nsites = nsites;
  const uint64_t* sites = t->site_sorted.data();

  // ---- segments and steps (no pointer field straddles a segment boundary)
  w->total = total;
  const uint64_t ch = desc->chunk_bytes;
  std::vector<std::pair<uint64_t, uint64_t>> node_ranges;
  for (size_t i = 0; i < t->alloc_off.size(); ++i)
    if (t->alloc_array[i] < 0) node_ranges.push_back({t->alloc_off[i], t->alloc_off[i] + t->alloc_size[i]});
  // hoist only when address order would make arrays wait for their chains, i.e. some chain
  // node lies after the array it leads to (scattered layouts; DFS layouts never do)
  bool late_nodes = false;
  for (uint64_t i = 0; i < desc->ntargets && !late_nodes; ++i) {
    const int64_t a = desc->h_targets[i];
    if (a < 0 || uint64_t(a) >= t->arr_off.size()) break;
    late_nodes = t->arr_owner[a] > t->arr_off[a] || t->arr_root[a] > t->arr_off[a];
  }
  const bool hoist = ch && ch < total && late_nodes && !node_ranges.empty() &&
                     node_ranges.size() <= HOIST_MAX_NODE_ALLOCS;
  auto cut = [&](uint64_t a, uint64_t b, bool check_sites) {   // [a, b) into <= ch pieces, one step each
    uint64_t x = a;
    while (x < b) {
      uint64_t y = (ch && ch < total) ? std::min(b, (x / ch + 1) * ch) : b;
      // a 4-mod-8 pointer field may straddle the grid point: end the segment just before the
      // field, or -- when the field opens this segment (the previous cut moved down to it) --
      // run on to the next grid point, so every field lands whole in one segment
      while (check_sites && y < b) {
        const uint64_t* it = std::lower_bound(sites, sites + nsites, y >= 7 ? y - 7 : 0);
        if (it == sites + nsites || *it >= y || *it + 8 <= y) break;
        if (*it > x) { y = *it; break; }
        y = std::min(b, y + ch);
      }
      w->seg_lo.push_back(x);
      w->seg_hi.push_back(y);
      w->step_seg_lo.push_back(w->seg_lo.size() - 1);
      x = y;
    }
  };
  if (hoist) {
    std::sort(node_ranges.begin(), node_ranges.end());
    // widen node ranges to whole pages so the bulk data copies stay page-aligned (the copy
    // engines lose full-duplex overlap on many unaligned pieces)
    // 64 KiB pages when that moves < 1/32 of the arena through the node step, else 4 KiB
    const uint64_t pa = (HOIST_PAGE > 1 && node_ranges.size() * 65536 <= total / 32) ? 65536 : HOIST_PAGE;
    for (auto& r : node_ranges) {
      r.first = r.first / pa * pa;
      r.second = std::min(total, (r.second + pa - 1) / pa * pa);
    }
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    for (auto& r : node_ranges) {
      if (!merged.empty() && r.first <= merged.back().second + HOIST_MERGE_GAP) merged.back().second = std::max(merged.back().second, r.second);
      else merged.push_back(r);
    }
    w->step_seg_lo.push_back(0);                       // step 0: every node segment
    for (auto& r : merged) { w->seg_lo.push_back(r.first); w->seg_hi.push_back(r.second); }
    // then the data between them: pieces on the chunk grid, consecutive pieces packed into
    // steps of about one chunk (a scattered layout leaves many short gaps)
    uint64_t x = 0, acc = ch;
    auto add = [&](uint64_t a, uint64_t b) {
      while (a < b) {
        const uint64_t y = std::min(b, (a / ch + 1) * ch);
        if (acc + (y - a) > ch) { w->step_seg_lo.push_back(w->seg_lo.size()); acc = 0; }
        w->seg_lo.push_back(a);
        w->seg_hi.push_back(y);
        acc += y - a;
        a = y;
      }
    };
    for (auto& r : merged) { if (r.first > x) add(x, r.first); x = r.second; }
    if (x < total) add(x, total);
  } else {
    cut(0, total, true);
  }
  const uint64_t nseg = w->seg_lo.size();
  const uint64_t nch = w->step_seg_lo.size();
  w->nsteps = nch;
  w->step_seg_lo.push_back(nseg);
  std::vector<uint64_t> seg_step(nseg);
  for (uint64_t k = 0; k < nch; ++k)
    for (uint64_t j = w->step_seg_lo[k]; j < w->step_seg_lo[k + 1]; ++j) seg_step[j] = k;
  SegIndex six;
  {
    std::vector<uint32_t> ord(nseg);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) { return w->seg_lo[x] < w->seg_lo[y]; });
    for (uint32_t j : ord) { six.lo.push_back(w->seg_lo[j]); six.seg.push_back(j); }
  }
  mark("segments");
  auto step_of = [&](uint64_t off) { return seg_step[six.at(off)]; };
  // Every ordering below is a stable bucket order on a step number (< nch), so planning is
  // linear in sites + targets (a C4 tree has a million of each); per-item work runs in parallel.
  // attach sites grouped by the step that uploads them (address order within a step)
  std::vector<uint64_t> site_step(nsites);
#pragma omp parallel for schedule(static) if (nsites > (1u << 15))
  for (int64_t k = 0; k < int64_t(nsites); ++k) site_step[k] = step_of(sites[k]);
  std::vector<uint64_t> reloc_order;
  bucket_order(site_step, nch, reloc_order, w->reloc_lo);
  std::vector<uint64_t> reloc(nsites);
  for (uint64_t k = 0; k < nsites; ++k) reloc[k] = sites[reloc_order[k]];

  mark("sites");
  // ---- per target: chain fields -> ready step (fields as (segment) pairs in CSR form)
  const uint64_t nt = desc->ntargets;
  const bool dense = t->spec.kind == CF_DENSE;
  const uint64_t q = dense ? uint64_t(t->spec.k_or_q) : 1;
  for (uint64_t i = 0; i < nt; ++i) {
    const int64_t a = desc->h_targets[i];
    if (a < 0 || uint64_t(a) >= t->arr_off.size()) { destroy(w); return fail(CF_E_INVALID, "target %lld out of range", (long long)a); }
  }
  std::vector<uint64_t> ready(nt, 0), max_step(nt, 0), fld_lo(nt + 1, 0);
  for (uint64_t i = 0; i < nt; ++i) fld_lo[i + 1] = fld_lo[i] + 2 * uint64_t(t->arr_level[desc->h_targets[i]] + 1);
  std::vector<uint32_t> fld_seg(fld_lo[nt]);
#pragma omp parallel for schedule(static) if (nt > (1u << 12))
  for (int64_t ii = 0; ii < int64_t(nt); ++ii) {
    const uint64_t i = uint64_t(ii);
    const int64_t a = desc->h_targets[i];
    const int L = t->arr_level[a];
    const uint64_t ord = t->arr_ordinal[a];
    const auto& lnodes = t->level_nodes[t->arr_tree[a]];
    const auto& lbase = t->level_base[t->arr_tree[a]];
    uint64_t r = 0, f = fld_lo[i];
    uint64_t pw = 1;   // q^(L-l): q^L at the root, divided by q per level down
    if (dense)
      for (int l = 0; l < L; ++l) pw *= q;
    for (int l = 0; l <= L; ++l, pw = (dense && pw >= q) ? pw / q : 1) {
      // ancestor at level l: ordinal prefix ord / q^(L-l) (pre-order within a level)
      const uint64_t node = lnodes[size_t(l)][dense ? ord / pw - lbase[size_t(l)] : 0];
      const bool leaf = dense && l == t->spec.depth;
      uint64_t lo, hi;  // byte range read at this level
      if (l < L) { lo = node + OFF_LNEXT; hi = lo + 8; }
      else { lo = node + OFF_NA; hi = node + (leaf ? LEAF_NODE_SIZE : OFF_LNEXT); }
      for (uint64_t x : {lo, hi - 1}) {
        const uint32_t sg = six.at(x);
        fld_seg[f++] = sg;
        r = std::max(r, seg_step[sg]);
      }
    }
    ready[i] = r;
  }
  mark("targets");
  // ---- parts: each target's array cut at segment boundaries; element i belongs to the
  //      segment holding its last byte
  const uint64_t e = uint64_t(w->elem);
  std::vector<Part> parts;
  // per segment: the last step that reads or writes it (thread-local maxima, merged below)
  std::vector<uint64_t> release(seg_step);
  {
    int nthr = 1;
#ifdef _OPENMP
    nthr = nt > (1u << 12) ? omp_get_max_threads() : 1;
#endif
    std::vector<std::vector<Part>> tparts(static_cast<size_t>(nthr));
    std::vector<std::vector<uint64_t>> trel(static_cast<size_t>(nthr), std::vector<uint64_t>(nseg, 0));
#pragma omp parallel num_threads(nthr)
    {
      int me = 0;
#ifdef _OPENMP
      me = omp_get_thread_num();
#endif
      auto& P = tparts[size_t(me)];
      auto& R = trel[size_t(me)];
      P.reserve(nt / size_t(nthr) + 64);
#pragma omp for schedule(static)
      for (int64_t ii = 0; ii < int64_t(nt); ++ii) {
        const uint64_t i = uint64_t(ii);
        const int64_t a = desc->h_targets[i];
        const uint64_t off = t->arr_off[a], n = t->arr_count[a];
        if (n == 0) continue;
        const uint64_t end = off + e * n;
        // first element whose last byte lies at or after byte x
        auto first_i = [&](uint64_t x) -> uint64_t {
          if (x <= off + e - 1) return 0;
          return std::min(n, (x - (off + e - 1) + e - 1) / e);
        };
        // walk the segments under the array in address order
        size_t pos = size_t(std::upper_bound(six.lo.begin(), six.lo.end(), off + e - 1) - six.lo.begin()) - 1;
        {
          // common case: the whole array inside one segment (one piece)
          const uint32_t sg = six.seg[pos];
          if (w->seg_lo[sg] <= off && w->seg_hi[sg] >= end) {
            const uint64_t step = std::max(ready[i], seg_step[sg]);
            P.push_back({i, 0, n, step});
            R[sg] = std::max(R[sg], step);
            max_step[i] = step;
            continue;
          }
        }
        uint64_t ms = 0;
        for (; pos < six.lo.size() && six.lo[pos] < end; ++pos) {
          const uint32_t sg = six.seg[pos];
          const uint64_t i0 = first_i(w->seg_lo[sg]);
          const uint64_t i1 = (w->seg_hi[sg] >= end) ? n : first_i(w->seg_hi[sg]);
          if (i1 <= i0) continue;
          // the piece's bytes may reach into neighbouring segments (elements straddling a
          // boundary): it runs once all of them have landed and its chain is resolved
          const size_t pb = size_t(std::upper_bound(six.lo.begin(), six.lo.end(), off + e * i0) - six.lo.begin()) - 1;
          const size_t pe = size_t(std::upper_bound(six.lo.begin(), six.lo.end(), off + e * i1 - 1) - six.lo.begin()) - 1;
          uint64_t step = ready[i];
          for (size_t x = pb; x <= pe; ++x) step = std::max(step, seg_step[six.seg[x]]);
          P.push_back({i, i0, i1, step});
          ms = std::max(ms, step);
          // every segment this piece touches is copied back no earlier than its step
          for (size_t x = pb; x <= pe; ++x) R[six.seg[x]] = std::max(R[six.seg[x]], step);
        }
        max_step[i] = ms;
      }
    }
    for (auto& v : tparts) parts.insert(parts.end(), v.begin(), v.end());
    for (auto& v : trel)
      for (uint64_t sg = 0; sg < nseg; ++sg) release[sg] = std::max(release[sg], v[sg]);
  }
  const bool chase = desc->mode == CF_MODE_CHASE;
  // attach || resolve in one launch: safe when every field a resolver may read while the attach
  // CTAs rewrite it is 8-byte aligned (one atomic 64-bit access).  Dense 12-byte leaf records put
  // every other leaf's A field at 4 mod 8; a resolver is that field's only reader, so when the
  // field is attached in the step that resolves its target, the resolver attaches it itself.
  w->aligned8 = std::all_of(sites, sites + nsites, [](uint64_t o) { return (o & 7) == 0; });
  {
    bool misaligned_only_leaf_a = dense && !chase;
    if (misaligned_only_leaf_a && !w->aligned8) {
      std::vector<uint64_t> leafs;
      for (const auto& tr : t->level_nodes)
        if (tr.size() > size_t(t->spec.depth)) leafs.insert(leafs.end(), tr[size_t(t->spec.depth)].begin(), tr[size_t(t->spec.depth)].end());
      std::sort(leafs.begin(), leafs.end());
      for (uint64_t i = 0; i < nsites && misaligned_only_leaf_a; ++i)
        if (sites[i] & 7) misaligned_only_leaf_a = std::binary_search(leafs.begin(), leafs.end(), sites[i] - LEAF_OFF_A);
    }
    w->wide_ok = w->aligned8 || misaligned_only_leaf_a;
    w->owned_attach = w->wide_ok && !w->aligned8;
  }
  // ---- leaf-owned relocation (LeafOwn): a leaf target whose whole, group-sized array is scaled in
  //      one step is owned by that step's leaf kernel when the step's such targets are one run of
  //      consecutive ordinals with equal counts (dense single tree, RESOLVED, aligned node fields)
  std::vector<uint64_t> lown(nt, nch);
  w->own_step.assign(nch, LeafOwn{});
  {
    static const bool no_leaf_own = getenv("CF_NO_LEAF_OWN") != nullptr;   // A/B switch (design experiments)
    constexpr uint32_t PHASES = CF_WIN_ATTACH | CF_WIN_RESOLVE | CF_WIN_SCALE | CF_WIN_DETACH;
    if (!no_leaf_own && !(fl & CF_WIN_TABLE_RESOLVE) && (fl & PHASES) == PHASES && !(fl & CF_WIN_UVM) && dense && !chase && w->wide_ok &&
        t->tree_root.size() <= 1 && q >= 2 && t->spec.depth >= 1 && nt > 0 && nt < (1ull << 31)) {
      std::vector<uint32_t> npc(nt, 0);
      std::vector<uint64_t> pst(nt, 0);
      std::vector<uint8_t> whole(nt, 0);
      for (const Part& pp : parts) {
        ++npc[pp.t];
        pst[pp.t] = pp.step;
        whole[pp.t] = pp.b == 0 && pp.e == t->arr_count[desc->h_targets[pp.t]];
      }
      std::vector<std::vector<std::pair<uint64_t, uint64_t>>> cand(nch);   // per step: (ordinal, target)
      for (uint64_t i = 0; i < nt; ++i) {
        const int64_t a = desc->h_targets[i];
        const uint64_t n = t->arr_count[a];
        if (t->arr_level[a] != int(t->spec.depth) || npc[i] != 1 || !whole[i] || n == 0 || n * e >= TILE_BYTES) continue;
        cand[pst[i]].push_back({t->arr_ordinal[a], i});
      }
      for (uint64_t k = 0; k < nch; ++k) {
        auto& c = cand[k];
        if (c.empty()) continue;
        std::sort(c.begin(), c.end());
        const uint64_t n_el = t->arr_count[desc->h_targets[c[0].second]];
        bool ok = c.back().first - c.front().first + 1 == c.size() && c.back().first < (1ull << 31);
        for (size_t j = 0; j < c.size() && ok; ++j) ok = t->arr_count[desc->h_targets[c[j].second]] == n_el;
        if (!ok) continue;
        // the table path's grouping rule (ScaleWork::append): <= GROUP_PARTS parts, <= GROUP_BYTES
        const uint64_t gp = std::max<uint64_t>(1, std::min<uint64_t>(GROUP_PARTS, GROUP_BYTES / (n_el * e)));
        const uint32_t o0 = uint32_t(c.front().first), cn = uint32_t(c.size());
        w->own_step[k] = LeafOwn{nullptr, 1u, uint32_t(t->spec.depth), o0, uint32_t(o0 / q),
                                 uint32_t((uint64_t(o0) + cn - 1) / q - o0 / q + 1), uint32_t(n_el), uint32_t(gp), cn,
                                 ~0ull / q + 1, 0, 0, 0};
        for (auto& pr : c) lown[pr.second] = k;
        w->own_any = true;
      }
    }
  }
  if (w->own_any) {
    // owned targets leave every table: their parts, their resolve entries, their A-field sites
    parts.erase(std::remove_if(parts.begin(), parts.end(), [&](const Part& pp) { return lown[pp.t] < nch; }), parts.end());
    std::vector<uint64_t> ofa;
    for (uint64_t i = 0; i < nt; ++i)
      if (lown[i] < nch) ofa.push_back(t->arr_owner[desc->h_targets[i]] + LEAF_OFF_A);
    std::sort(ofa.begin(), ofa.end());
    std::vector<uint64_t> nrl, nlo(nch + 1, 0);
    nrl.reserve(reloc.size() - ofa.size());
    for (uint64_t k = 0; k < nch; ++k) {
      nlo[k] = nrl.size();
      for (uint64_t r = w->reloc_lo[k]; r < w->reloc_lo[k + 1]; ++r)
        if (!std::binary_search(ofa.begin(), ofa.end(), reloc[r])) nrl.push_back(reloc[r]);
    }
    nlo[nch] = nrl.size();
    reloc.swap(nrl);
    w->reloc_lo.swap(nlo);
    uint64_t p0 = ~0ull, p1 = 0;
    for (const LeafOwn& o : w->own_step)
      if (o.on) { p0 = std::min<uint64_t>(p0, o.p_first); p1 = std::max<uint64_t>(p1, uint64_t(o.p_first) + o.nparents); }
    w->parent_base = p0;
    w->own_parents = p1 - p0;
  }
  const uint64_t nrel = reloc.size();   // sites in the tables (all sites but the leaf-owned A fields)
  {   // chain fields are read until the target's resolve (chase: until its last piece; leaf-owned:
      // until its leaf kernel, which reads and writes the record)
    int nthr = 1;
#ifdef _OPENMP
    nthr = nt > (1u << 14) ? omp_get_max_threads() : 1;
#endif
    std::vector<std::vector<uint64_t>> trel(static_cast<size_t>(nthr), std::vector<uint64_t>(nseg, 0));
#pragma omp parallel num_threads(nthr)
    {
      int me = 0;
#ifdef _OPENMP
      me = omp_get_thread_num();
#endif
      auto& R = trel[size_t(me)];
#pragma omp for schedule(static)
      for (int64_t ii = 0; ii < int64_t(nt); ++ii) {
        const uint64_t i = uint64_t(ii);
        const uint64_t v = chase ? std::max(ready[i], max_step[i]) : lown[i] < nch ? std::max(ready[i], lown[i]) : ready[i];
        for (uint64_t f = fld_lo[i]; f < fld_lo[i + 1]; ++f) R[fld_seg[f]] = std::max(R[fld_seg[f]], v);
      }
    }
    for (auto& v : trel)
      for (uint64_t sg = 0; sg < nseg; ++sg) release[sg] = std::max(release[sg], v[sg]);
  }

  mark("parts");
  // ---- order targets by ready step, parts by step, detach sites by release step
  // (leaf-owned targets go to a bucket past the last step: they are never resolved from tables)
  std::vector<uint64_t> torder;
  {
    std::vector<uint64_t> rkey(nt);
    for (uint64_t i = 0; i < nt; ++i) rkey[i] = lown[i] < nch ? nch : ready[i];
    bucket_order(rkey, nch + 1, torder, w->res_lo);
  }
  const uint64_t nt_tab = w->res_lo[nch];   // targets with table entries (resolved from tables)
  std::vector<uint64_t> tpos(nt);
  for (uint64_t k = 0; k < nt; ++k) tpos[torder[k]] = k;
  std::vector<uint8_t> owned_target(nt, 0);
  w->attach_n.assign(nch, 0);
  for (uint64_t k = 0; k < nch; ++k) w->attach_n[k] = w->reloc_lo[k + 1] - w->reloc_lo[k];
  if (w->owned_attach) {
    std::vector<uint8_t> owned_site(nrel, 0);
    for (uint64_t i = 0; i < nt; ++i) {
      const int64_t a = desc->h_targets[i];
      if (t->arr_level[a] != int(t->spec.depth) || lown[i] < nch) continue;   // table-resolved leaf records only
      const uint64_t fa = t->arr_owner[a] + LEAF_OFF_A;
      if ((fa & 7) == 0 || step_of(fa) != ready[i]) continue;        // aligned, or attached earlier
      const uint64_t r = uint64_t(std::lower_bound(reloc.begin() + w->reloc_lo[ready[i]], reloc.begin() + w->reloc_lo[ready[i] + 1], fa) -
                                  reloc.begin());
      if (r < w->reloc_lo[ready[i] + 1] && reloc[r] == fa) {
        owned_site[r] = 1;
        owned_target[i] = 1;
      }
    }
    // within each step: sites the attach CTAs take first, owned sites after (address order kept)
    for (uint64_t k = 0; k < nch; ++k) {
      auto b = reloc.begin() + w->reloc_lo[k], e = reloc.begin() + w->reloc_lo[k + 1];
      std::vector<uint64_t> keep, own;
      for (auto it = b; it != e; ++it) (owned_site[size_t(it - reloc.begin())] ? own : keep).push_back(*it);
      std::copy(keep.begin(), keep.end(), b);
      std::copy(own.begin(), own.end(), b + keep.size());
      w->attach_n[k] = keep.size();
    }
  }
  // uniform resolve ranges: one tree, consecutive ordinals at one level >= 1, ownership == misalignment
  w->uni.assign(nch, UniTargets{0, 0, 0, 0, 0});
  if (dense && t->tree_root.size() <= 1) {
    for (uint64_t k = 0; k < nch; ++k) {
      const uint64_t lo = w->res_lo[k], hi = w->res_lo[k + 1];
      if (hi == lo) continue;
      const int64_t a0 = desc->h_targets[torder[lo]];
      const int L = t->arr_level[a0];
      const uint64_t o0 = t->arr_ordinal[a0];
      bool ok = L >= 1 && o0 + (hi - lo) < (1ull << 31);
      for (uint64_t p2 = lo; p2 < hi && ok; ++p2) {
        const uint64_t i = torder[p2];
        const int64_t a = desc->h_targets[i];
        const uint64_t fa = t->arr_owner[a] + (L == int(t->spec.depth) ? LEAF_OFF_A : OFF_A);
        ok = t->arr_level[a] == L && t->arr_ordinal[a] == o0 + (p2 - lo) &&
             bool(owned_target[i]) == (w->owned_attach && (fa & 7) != 0);
      }
      if (ok) w->uni[k] = UniTargets{1, uint32_t(L), uint32_t(o0), w->owned_attach ? 1u : 0u, q > 1 ? ~0ull / q + 1 : 0};
    }
  }
  mark("o:targets");
  // per step: the pieces ready at that step, as one leaf-kernel launch (big tiles + small groups)
  std::vector<uint64_t> pstep(parts.size()), porder, plo;
  for (size_t k = 0; k < parts.size(); ++k) pstep[k] = parts[k].step;
  bucket_order(pstep, nch, porder, plo);
  mark("o:pstep");
  ScaleWork sw;
  sw.elem = w->elem;
  sw.parts.reserve(3 * parts.size());
  sw.groups.reserve(2 * (parts.size() / 8 + nch + 1));
  w->seg.resize(nch);
  std::vector<uint64_t> tri;
  for (uint64_t c = 0; c < nch; ++c) {
    tri.clear();
    tri.reserve(3 * (plo[c + 1] - plo[c]));
    for (uint64_t k = plo[c]; k < plo[c + 1]; ++k) {
      const Part& pp = parts[porder[k]];
      tri.insert(tri.end(), {tpos[pp.t], pp.b, pp.e});
    }
    w->seg[c] = sw.append(tri);
  }
  mark("o:work");
  // detach order: positions in the (step-ordered) relocation table, grouped by release step
  std::vector<uint32_t> det(nrel);
  {
    std::vector<uint64_t> srel(nrel), sidx;
#pragma omp parallel for schedule(static) if (nrel > (1u << 15))
    for (int64_t k = 0; k < int64_t(nrel); ++k) srel[k] = release[six.at(reloc[k])];
    bucket_order(srel, nch, sidx, w->det_lo);
    for (uint64_t k = 0; k < nrel; ++k) det[k] = uint32_t(sidx[k]);
  }
  mark("orders");
  w->released.assign(nch, {});
  const uint64_t nnode_seg = hoist ? w->step_seg_lo[1] : 0;
  if (!dry) {
    void* dp = nullptr;
    const bool mapped = desc->host_src && cudaHostGetDevicePointer(&dp, const_cast<void*>(desc->host_src), 0) == cudaSuccess &&
                        dp == desc->host_src &&
                        (!desc->host_dst || (cudaHostGetDevicePointer(&dp, desc->host_dst, 0) == cudaSuccess && dp == desc->host_dst));
    cudaGetLastError();
    w->zc = hoist && mapped && nnode_seg > ZC_MIN_SEGS;
  } else {
    w->zc = hoist && nnode_seg > ZC_MIN_SEGS;   // dry runs plan as if the arena were mapped
  }
  std::vector<uint64_t> zc_rel;   // node segments ordered by release step
  for (uint64_t sg = 0; sg < nseg; ++sg) {
    if (w->zc && sg < nnode_seg) continue;
    w->released[release[sg]].push_back(uint32_t(sg));
  }
  if (w->zc) {
    w->zc_n = nnode_seg;
    std::vector<uint64_t> ids(nnode_seg);
    std::iota(ids.begin(), ids.end(), 0);
    std::stable_sort(ids.begin(), ids.end(), [&](uint64_t x, uint64_t y) { return release[x] < release[y]; });
    w->zc_rel_lo.assign(nch + 1, 0);
    for (uint64_t c = 0, k = 0; c <= nch; ++c) {
      while (k < nnode_seg && release[ids[k]] < c) ++k;
      w->zc_rel_lo[c] = k;
    }
    for (uint64_t id : ids) zc_rel.insert(zc_rel.end(), {w->seg_lo[id], w->seg_hi[id]});
  }

  if (getenv("CF_PLAN_DUMP")) {   // design experiments: the step schedule, one line per step
    for (uint64_t k = 0; k < nch; ++k) {
      uint64_t up = 0, down = 0;
      for (uint64_t j = w->step_seg_lo[k]; j < w->step_seg_lo[k + 1]; ++j) up += w->seg_hi[j] - w->seg_lo[j];
      for (uint32_t r : w->released[k]) down += w->seg_hi[r] - w->seg_lo[r];
      fprintf(stderr, "step %llu up %llu down %llu nrel %zu\n", (unsigned long long)k, (unsigned long long)up,
              (unsigned long long)down, w->released[k].size());
    }
  }
  mark("released");
  // ---- table block: sites | det | level | ordinal | parts | tile_base | groups
  auto al8 = [](uint64_t x) { return (x + 7) & ~7ull; };
  w->has_roots = t->tree_root.size() > 1;   // single trees use the shape's root
  w->off_sites = 0;
  w->off_det = al8(w->off_sites + nrel * 8);
  w->off_level = al8(w->off_det + nrel * 4);
  w->off_ord = al8(w->off_level + nt_tab * 4);
  w->off_root = al8(w->off_ord + nt_tab * 4);
  w->off_parts = al8(w->off_root + (w->has_roots ? nt_tab * 8 : 0));
  w->off_tb = al8(w->off_parts + sw.parts.size() * 4);
  w->off_grp = al8(w->off_tb + sw.tile_base.size() * 8);
  w->off_zc_h2d = al8(w->off_grp + sw.groups.size() * 4 + 8);
  w->off_zc_d2h = w->off_zc_h2d + (w->zc ? w->zc_n * 16 : 0);
  w->tab_bytes = al8(w->off_zc_d2h + (w->zc ? w->zc_n * 16 : 0) + 8);
  if (dry) {
    auto& D = *w->dry;
    D.reloc = std::move(reloc);
    D.det = std::move(det);
    D.torder = std::move(torder);
    D.ready = std::move(ready);
    D.release = std::move(release);
    D.seg_step = std::move(seg_step);
    D.part_step = std::move(pstep);
    D.owned = std::move(owned_target);
    D.lown = std::move(lown);
    D.sw = std::move(sw);
    mark("tables");
    *out = w;
    return CF_OK;
  }
  cudaError_t ce = cudaHostAlloc(&w->h_tab, w->tab_bytes, cudaHostAllocPortable);
  if (ce == cudaSuccess) ce = cudaMalloc(&w->d_tab, w->tab_bytes);
  if (ce == cudaSuccess) ce = cudaMalloc(&w->d_ea, std::max<uint64_t>(nt, 1) * 8);
  if (ce == cudaSuccess) ce = cudaMalloc(&w->d_count, std::max<uint64_t>(nt, 1) * 4);
  if (ce == cudaSuccess && w->own_any) ce = cudaMalloc(&w->d_parent, w->own_parents * 8);
  if (ce != cudaSuccess) { cudaGetLastError(); destroy(w); return fail(CF_E_OOM, "window tables: %s", cudaGetErrorString(ce)); }
  if (nrel) memcpy(w->h_tab + w->off_sites, reloc.data(), nrel * 8);
  if (nrel) memcpy(w->h_tab + w->off_det, det.data(), nrel * 4);
  int32_t* lv = reinterpret_cast<int32_t*>(w->h_tab + w->off_level);
  uint32_t* od = reinterpret_cast<uint32_t*>(w->h_tab + w->off_ord);
  uint64_t* rt = reinterpret_cast<uint64_t*>(w->h_tab + w->off_root);
  for (uint64_t k = 0; k < nt_tab; ++k) {
    const int64_t a = desc->h_targets[torder[k]];
    lv[k] = t->arr_level[a];
    od[k] = uint32_t(t->arr_ordinal[a]) | (owned_target[torder[k]] ? 0x80000000u : 0u);   // bit 31: attach own A field
    if (w->has_roots) rt[k] = t->arr_root[a];
  }
  if (!sw.parts.empty()) memcpy(w->h_tab + w->off_parts, sw.parts.data(), sw.parts.size() * 4);
  if (!sw.tile_base.empty()) memcpy(w->h_tab + w->off_tb, sw.tile_base.data(), sw.tile_base.size() * 8);
  if (!sw.groups.empty()) memcpy(w->h_tab + w->off_grp, sw.groups.data(), sw.groups.size() * 4);
  if (w->zc) {
    uint64_t* zh = reinterpret_cast<uint64_t*>(w->h_tab + w->off_zc_h2d);
    for (uint64_t j = 0; j < w->zc_n; ++j) { zh[2 * j] = w->seg_lo[j]; zh[2 * j + 1] = w->seg_hi[j]; }
    memcpy(w->h_tab + w->off_zc_d2h, zc_rel.data(), zc_rel.size() * 8);
  }
  for (auto& sg : w->seg) {
    sg.parts = reinterpret_cast<const uint32_t*>(w->d_tab + w->off_parts);
    sg.tile_base = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_tb);
    sg.groups = reinterpret_cast<const uint32_t*>(w->d_tab + w->off_grp);
  }
  // the device mirror starts valid so runs without CF_WIN_TABLES work
  ce = cudaMemcpyAsync(w->d_tab, w->h_tab, w->tab_bytes, cudaMemcpyHostToDevice, ctx->compute);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->compute);
  if (ce != cudaSuccess) { cudaGetLastError(); destroy(w); return fail(CF_E_CUDA, "table upload: %s", cudaGetErrorString(ce)); }

  mark("tables");
  // ---- events
  auto mk = [](cudaEvent_t* e, unsigned f) { return cudaEventCreateWithFlags(e, f); };
  w->ev_h2d.resize(nch);
  w->ev_rel.resize(nch);
  w->ev_k0.resize(nch);
  w->ev_k1.resize(nch);
  bool ok = mk(&w->ev_start, cudaEventDefault) == cudaSuccess && mk(&w->ev_end, cudaEventDefault) == cudaSuccess &&
            mk(&w->ev_join, cudaEventDisableTiming) == cudaSuccess && mk(&w->ev_first, cudaEventDefault) == cudaSuccess &&
            mk(&w->ev_tables, cudaEventDisableTiming) == cudaSuccess &&
            mk(&w->ev_fan, cudaEventDisableTiming) == cudaSuccess &&
            cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking) == cudaSuccess;
  for (uint64_t c = 0; c < nch && ok; ++c)
    ok = mk(&w->ev_h2d[c], cudaEventDisableTiming) == cudaSuccess && mk(&w->ev_rel[c], cudaEventDisableTiming) == cudaSuccess &&
         mk(&w->ev_k0[c], cudaEventDefault) == cudaSuccess && mk(&w->ev_k1[c], cudaEventDefault) == cudaSuccess;
  if (!ok) { cudaGetLastError(); destroy(w); return fail(CF_E_CUDA, "event creation failed"); }
  mark("events");
  *out = w;
  return CF_OK;
}
}  // namespace

}  // extern "C"

namespace {
// Invariants of a planned window, re-derived independently of the planner where possible (the
// chain of every target is walked through the tree's site table, not its level tables).
struct Checker {
  const cf_tree* t;
  const cf_window_desc* d;
  const cf_window* w;
  int violations = 0;
  template <typename... A>
  void bad(const char* fmt, A... a) {
    if (violations++ == 0) fail(CF_E_STATE, fmt, a...);
  }
  uint32_t seg_at(uint64_t off) const {   // segment holding byte off (segments partition [0, total))
    return sorted_seg[size_t(std::upper_bound(sorted_lo.begin(), sorted_lo.end(), off) - sorted_lo.begin()) - 1];
  }
  std::vector<uint64_t> sorted_lo;
  std::vector<uint32_t> sorted_seg;

  void run() {
    const auto& D = *w->dry;
    const uint64_t total = t->total, nseg = w->seg_lo.size(), nch = w->nsteps, nt = d->ntargets;
    const uint64_t e = uint64_t(t->spec.elem);
    // 1. segments partition [0, total)
    std::vector<uint32_t> ord(nseg);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return w->seg_lo[a] < w->seg_lo[b]; });
    uint64_t x = 0;
    for (uint32_t j : ord) {
      if (w->seg_lo[j] != x || w->seg_hi[j] <= w->seg_lo[j]) bad("segment %u [%llu, %llu) breaks the partition at %llu", j,
                                                              (unsigned long long)w->seg_lo[j], (unsigned long long)w->seg_hi[j], (unsigned long long)x);
      x = w->seg_hi[j];
      sorted_lo.push_back(w->seg_lo[j]);
      sorted_seg.push_back(j);
    }
    if (x != total) bad("segments end at %llu, arena is %llu bytes", (unsigned long long)x, (unsigned long long)total);
    if (w->step_seg_lo.size() != nch + 1 || w->step_seg_lo.back() != nseg) bad("step table malformed");
    // 2. sites: each once, in the step that uploads both its ends
    // (leaf-owned targets' A fields are relocated by their leaf kernel, not from the table)
    std::vector<uint64_t> rs(D.reloc);
    for (uint64_t i = 0; i < nt; ++i)
      if (D.lown[i] < nch) rs.push_back(t->arr_owner[d->h_targets[i]] + LEAF_OFF_A);
    std::sort(rs.begin(), rs.end());
    if (rs != t->site_sorted) bad("relocation table + leaf-owned fields are not a permutation of the sites");
    for (uint64_t k = 0; k < nch; ++k)
      for (uint64_t i = w->reloc_lo[k]; i < w->reloc_lo[k + 1]; ++i) {
        const uint64_t s0 = D.reloc[i];
        const uint32_t a = seg_at(s0), b = seg_at(s0 + 7);
        if (a != b) bad("site %llu straddles segments %u / %u", (unsigned long long)s0, a, b);
        if (D.seg_step[a] != k) bad("site %llu attached at step %llu, uploaded at %llu", (unsigned long long)s0,
                                    (unsigned long long)k, (unsigned long long)D.seg_step[a]);
      }
    // 3. chains, walked through the site table: ready = last upload step of every byte read
    std::vector<std::pair<uint64_t, uint64_t>> fmap(t->site_off.size());
    for (size_t i = 0; i < fmap.size(); ++i) fmap[i] = {t->site_off[i], t->site_target[i]};
    std::sort(fmap.begin(), fmap.end());
    auto target_of = [&](uint64_t field, bool& ok) -> uint64_t {
      auto it = std::lower_bound(fmap.begin(), fmap.end(), std::make_pair(field, uint64_t(0)));
      ok = it != fmap.end() && it->first == field;
      return ok ? it->second : 0;
    };
    const bool dense = t->spec.kind == CF_DENSE;
    const uint64_t q = dense ? uint64_t(t->spec.k_or_q) : 1;
    const bool chase = d->mode == CF_MODE_CHASE;
    std::vector<uint64_t> need_release(nseg, 0);
    for (uint64_t sg = 0; sg < nseg; ++sg) need_release[sg] = D.seg_step[sg];
    std::vector<std::vector<uint32_t>> chain_segs(nt);
    std::vector<std::vector<uint64_t>> chain_fields(nt);   // pointer fields each resolver reads
    for (uint64_t i = 0; i < nt; ++i) {
      const int64_t a = d->h_targets[i];
      const int L = t->arr_level[a];
      uint64_t node = t->arr_root[a], r = 0;
      auto touch = [&](uint64_t lo, uint64_t hi) {
        for (uint64_t y : {lo, hi - 1}) {
          const uint32_t sg = seg_at(y);
          r = std::max(r, D.seg_step[sg]);
          chain_segs[i].push_back(sg);
        }
      };
      for (int l = 1; l <= L; ++l) {
        bool ok = false;
        const uint64_t blk = target_of(node + OFF_LNEXT, ok);
        if (!ok) { bad("target %llu: no Lnext site at level %d", (unsigned long long)i, l); break; }
        touch(node + OFF_LNEXT, node + OFF_LNEXT + 8);
        chain_fields[i].push_back(node + OFF_LNEXT);
        uint64_t pw = 1;
        for (int m = l; m < L; ++m) pw *= q;
        const uint64_t digit = dense ? (uint64_t(t->arr_ordinal[a]) / pw) % q : 0;
        node = blk + digit * ((dense && l == int(t->spec.depth)) ? LEAF_NODE_SIZE : NODE_SIZE);
      }
      if (node != t->arr_owner[a]) bad("target %llu: chain ends at %llu, array owner is %llu", (unsigned long long)i,
                                       (unsigned long long)node, (unsigned long long)t->arr_owner[a]);
      const bool leaf = dense && L == int(t->spec.depth);
      touch(node + OFF_NA, node + (leaf ? LEAF_NODE_SIZE : OFF_LNEXT));
      chain_fields[i].push_back(node + (leaf ? LEAF_OFF_A : OFF_A));
      if (D.ready[i] != r) bad("target %llu ready at step %llu, its chain lands at %llu", (unsigned long long)i,
                               (unsigned long long)D.ready[i], (unsigned long long)r);
    }
    for (uint64_t c = 0; c < nch; ++c)
      for (uint64_t k = w->res_lo[c]; k < w->res_lo[c + 1]; ++k) {
        if (D.ready[D.torder[k]] != c) bad("target resolved at step %llu is ready at %llu", (unsigned long long)c,
                                           (unsigned long long)D.ready[D.torder[k]]);
        if (D.lown[D.torder[k]] < nch) bad("leaf-owned target %llu also resolved from the tables", (unsigned long long)D.torder[k]);
      }
    for (uint64_t k = w->res_lo[nch]; k < nt; ++k)
      if (D.lown[D.torder[k]] >= nch) bad("target %llu is neither resolved nor leaf-owned", (unsigned long long)D.torder[k]);
    // 3b. one-launch attach || resolve: no misaligned field in the attach CTAs' list is read by a
    //     resolver of the same step; every owned field sits in its target's step's owned tail
    if (w->wide_ok) {
      std::vector<std::vector<uint64_t>> read_at(nch);   // misaligned fields read by resolvers, per step
      for (uint64_t i = 0; i < nt; ++i)
        for (uint64_t f : chain_fields[i])
          if (f & 7) read_at[D.ready[i]].push_back(f);
      for (auto& v : read_at) std::sort(v.begin(), v.end());
      for (uint64_t k = 0; k < nch; ++k) {
        for (uint64_t j = w->reloc_lo[k]; j < w->reloc_lo[k] + w->attach_n[k]; ++j)
          if ((D.reloc[j] & 7) && std::binary_search(read_at[k].begin(), read_at[k].end(), D.reloc[j]))
            bad("misaligned site %llu attached by the attach CTAs while a resolver reads it (step %llu)",
                (unsigned long long)D.reloc[j], (unsigned long long)k);
        std::vector<uint64_t> tail(D.reloc.begin() + w->reloc_lo[k] + w->attach_n[k], D.reloc.begin() + w->reloc_lo[k + 1]);
        std::sort(tail.begin(), tail.end());
        uint64_t owners = 0;
        for (uint64_t p2 = w->res_lo[k]; p2 < w->res_lo[k + 1]; ++p2) {
          const uint64_t i = D.torder[p2];
          if (!D.owned[i]) continue;
          ++owners;
          const uint64_t fa = t->arr_owner[d->h_targets[i]] + LEAF_OFF_A;
          if (!std::binary_search(tail.begin(), tail.end(), fa)) bad("owned A field of target %llu not in step %llu's tail",
                                                                     (unsigned long long)i, (unsigned long long)k);
        }
        if (owners != tail.size()) bad("step %llu: %llu owned sites, %llu owning resolvers", (unsigned long long)k,
                                       (unsigned long long)tail.size(), (unsigned long long)owners);
      }
    }
    // 4. parts: tile every target's [0, count) once, each after its bytes and its chain
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> cover(nt);
    std::vector<uint64_t> max_part(nt, 0);
    const auto& P = D.sw.parts;
    auto part = [&](uint64_t k, uint64_t p) {
      const uint64_t tp = P[3 * p], e0 = P[3 * p + 1], e1 = P[3 * p + 2];
      if (tp >= nt) { bad("part %llu names target position %llu", (unsigned long long)p, (unsigned long long)tp); return; }
      const uint64_t i = D.torder[tp];
      const int64_t a = d->h_targets[i];
      if (k < D.ready[i]) bad("part of target %llu scaled at step %llu before its chain (step %llu)", (unsigned long long)i,
                              (unsigned long long)k, (unsigned long long)D.ready[i]);
      const uint64_t b0 = t->arr_off[a] + e0 * e, b1 = t->arr_off[a] + e1 * e;
      for (size_t z = size_t(std::upper_bound(sorted_lo.begin(), sorted_lo.end(), b0) - sorted_lo.begin()) - 1;
           z < sorted_lo.size() && sorted_lo[z] < b1; ++z) {
        const uint32_t sg = sorted_seg[z];
        if (D.seg_step[sg] > k) bad("part of target %llu scaled at step %llu before segment %u lands (%llu)",
                                    (unsigned long long)i, (unsigned long long)k, sg, (unsigned long long)D.seg_step[sg]);
        need_release[sg] = std::max(need_release[sg], k);
      }
      cover[i].push_back({e0, e1});
      max_part[i] = std::max(max_part[i], k);
    };
    for (uint64_t k = 0; k < nch; ++k) {
      const cf_scale_work& sw = w->seg[k];
      uint64_t tiles = 0;
      for (uint64_t p = sw.big_begin; p < sw.big_begin + sw.big_count; ++p) {
        part(k, p);
        // the kernel maps tile -> big part by tile_base: consecutive, one tile per 16 KiB
        if (D.sw.tile_base[sw.tb_begin + (p - sw.big_begin)] != sw.tile_begin + tiles) bad("tile base of part %llu is off", (unsigned long long)p);
        tiles += tiles_for(P[3 * p + 2] - P[3 * p + 1], int(e));
      }
      if (sw.tile_end - sw.tile_begin != tiles) bad("step %llu launches %llu tiles for %llu", (unsigned long long)k,
                                                    (unsigned long long)(sw.tile_end - sw.tile_begin), (unsigned long long)tiles);
      for (uint64_t g = sw.group_begin; g < sw.group_end; ++g) {
        const uint64_t p0 = D.sw.groups[2 * g], p1 = D.sw.groups[2 * g + 1];
        // the group kernel holds at most GROUP_PARTS parts (warp-local metadata)
        if (p1 <= p0 || p1 - p0 > GROUP_PARTS) bad("group %llu holds %llu parts", (unsigned long long)g, (unsigned long long)(p1 - p0));
        for (uint64_t p = p0; p < p1; ++p) {
          part(k, p);
          if (P[3 * p + 2] - P[3 * p + 1] >= TILE_BYTES / e) bad("big part %llu packed into a group", (unsigned long long)p);
        }
      }
    }
    // 4b. leaf-owned ranges: step k's range [o0, o0 + nt) is exactly its owned targets (leaf level,
    //     count n_el), each whole and after its bytes and its chain; group / parent shape as the
    //     kernel derives them
    {
      std::vector<std::vector<uint64_t>> by_step(nch);
      for (uint64_t i = 0; i < nt; ++i)
        if (D.lown[i] < nch) by_step[D.lown[i]].push_back(i);
      for (uint64_t k = 0; k < nch; ++k) {
        const LeafOwn& o = w->own_step[k];
        if (!o.on) { if (!by_step[k].empty()) bad("step %llu owns targets without a range", (unsigned long long)k); continue; }
        if (by_step[k].size() != o.nt) bad("step %llu: %u owned range, %zu owned targets", (unsigned long long)k, o.nt, by_step[k].size());
        const uint64_t gp_rule = std::max<uint64_t>(1, std::min<uint64_t>(GROUP_PARTS, GROUP_BYTES / (uint64_t(o.n_el) * e)));
        if (o.gp != gp_rule || o.level != uint32_t(t->spec.depth) || o.level < 1 || uint64_t(o.p_first) != o.o0 / q ||
            uint64_t(o.p_first) + o.nparents != (uint64_t(o.o0) + o.nt - 1) / q + 1)
          bad("step %llu: leaf-owned range shape (gp %u, level %u, parents [%u, +%u))", (unsigned long long)k, o.gp, o.level,
              o.p_first, o.nparents);
        if (uint64_t(o.p_first) < w->parent_base || uint64_t(o.p_first) + o.nparents > w->parent_base + w->own_parents)
          bad("step %llu: parents outside the parent table", (unsigned long long)k);
        std::vector<uint8_t> hit(o.nt, 0);
        for (uint64_t i : by_step[k]) {
          const int64_t a = d->h_targets[i];
          const uint64_t od = t->arr_ordinal[a];
          if (t->arr_level[a] != int(t->spec.depth) || od < o.o0 || od - o.o0 >= o.nt || hit[od - o.o0]++ ||
              t->arr_count[a] != o.n_el) {
            bad("leaf-owned target %llu (ordinal %llu) outside step %llu's range", (unsigned long long)i, (unsigned long long)od,
                (unsigned long long)k);
            continue;
          }
          if (D.ready[i] > k) bad("leaf-owned target %llu scaled at step %llu before its chain (step %llu)", (unsigned long long)i,
                                  (unsigned long long)k, (unsigned long long)D.ready[i]);
          const uint64_t b0 = t->arr_off[a], b1 = b0 + uint64_t(o.n_el) * e;
          for (size_t z = size_t(std::upper_bound(sorted_lo.begin(), sorted_lo.end(), b0) - sorted_lo.begin()) - 1;
               z < sorted_lo.size() && sorted_lo[z] < b1; ++z) {
            const uint32_t sg = sorted_seg[z];
            if (D.seg_step[sg] > k) bad("leaf-owned target %llu scaled at step %llu before segment %u lands", (unsigned long long)i,
                                        (unsigned long long)k, sg);
            need_release[sg] = std::max(need_release[sg], k);
          }
          cover[i].push_back({0, o.n_el});
          max_part[i] = std::max(max_part[i], k);
        }
      }
    }
    for (uint64_t i = 0; i < nt; ++i) {
      const uint64_t n = t->arr_count[d->h_targets[i]];
      auto& cv = cover[i];
      std::sort(cv.begin(), cv.end());
      uint64_t y = 0;
      for (auto& iv : cv) {
        if (iv.first != y || iv.second <= iv.first) { bad("target %llu: parts do not tile [0, %llu)", (unsigned long long)i, (unsigned long long)n); break; }
        y = iv.second;
      }
      if (y != n) bad("target %llu: parts cover [0, %llu) of %llu elements", (unsigned long long)i, (unsigned long long)y,
                      (unsigned long long)n);
      // a leaf-owned target's record is read and written by its leaf kernel
      for (uint32_t sg : chain_segs[i])
        need_release[sg] = std::max(need_release[sg], (chase || D.lown[i] < nch) ? std::max(D.ready[i], max_part[i]) : D.ready[i]);
    }
    // 5. release: no segment goes home before its last reader / writer
    for (uint64_t sg = 0; sg < nseg; ++sg)
      if (D.release[sg] < need_release[sg] || D.release[sg] >= nch)
        bad("segment %llu released at step %llu, needed until %llu", (unsigned long long)sg, (unsigned long long)D.release[sg],
            (unsigned long long)need_release[sg]);
    // 6. detach: every site once, at its segment's release step
    std::vector<uint8_t> seen(D.det.size(), 0);
    for (uint64_t c = 0; c < nch; ++c)
      for (uint64_t j = w->det_lo[c]; j < w->det_lo[c + 1]; ++j) {
        const uint32_t r = D.det[j];
        if (r >= D.reloc.size() || seen[r]++) { bad("detach list repeats or overflows at %llu", (unsigned long long)j); continue; }
        const uint32_t sg = seg_at(D.reloc[r]);
        if (D.release[sg] != c) bad("site %llu detached at step %llu, its segment is released at %llu",
                                    (unsigned long long)D.reloc[r], (unsigned long long)c, (unsigned long long)D.release[sg]);
      }
    for (uint64_t r = 0; r < seen.size(); ++r)
      if (!seen[r]) bad("site %llu never detached", (unsigned long long)D.reloc[r]);
    // 7. copy-back: every segment exactly once, at its release step
    std::vector<uint8_t> home(nseg, 0);
    for (uint64_t c = 0; c < nch; ++c)
      for (uint32_t sg : w->released[c]) {
        if (home[sg]++) bad("segment %u copied back twice", sg);
        if (D.release[sg] != c) bad("segment %u copied back at %llu, released at %llu", sg, (unsigned long long)c,
                                    (unsigned long long)D.release[sg]);
      }
    if (w->zc) {   // hoisted node segments go home by zero-copy kernels, in release order
      for (uint64_t c = 0; c < nch; ++c)
        if (w->zc_rel_lo[c + 1] < w->zc_rel_lo[c]) bad("zero-copy release table not monotone");
      if (w->zc_rel_lo[nch] != w->zc_n) bad("zero-copy release table covers %llu of %llu node segments",
                                            (unsigned long long)w->zc_rel_lo[nch], (unsigned long long)w->zc_n);
      for (uint64_t sg = 0; sg < w->zc_n; ++sg) {
        if (D.seg_step[sg] != 0) bad("hoisted node segment %llu not in step 0", (unsigned long long)sg);
        home[sg]++;
      }
    }
    for (uint64_t sg = 0; sg < nseg; ++sg)
      if (!home[sg]) bad("segment %llu never copied back", (unsigned long long)sg);
  }
};
}  // namespace

extern "C" {

int cf_window_plan_check(const cf_window_desc* desc, cf_plan_check* out) {
  if (!desc || !out) return fail(CF_E_INVALID, "null argument");
  memset(out, 0, sizeof *out);
  const auto t0 = std::chrono::steady_clock::now();
  cf_window* w = nullptr;
  CF_TRY(plan_impl(nullptr, desc, &w, true));
  out->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  out->nsteps = w->nsteps;
  out->nsegments = w->seg_lo.size();
  out->nsites = w->nsites;
  out->ntargets = desc->ntargets;
  out->nparts = w->dry->sw.nparts();
  out->ngroups = w->dry->sw.ngroups();
  out->ntiles = w->dry->sw.next_tile;
  out->table_bytes = w->tab_bytes;
  out->zero_copy_node_segments = w->zc ? w->zc_n : 0;
  out->leaf_owned = 0;
  for (const LeafOwn& o : w->own_step) out->leaf_owned += o.on ? 1 : 0;   // steps with a leaf-owned range
  Checker ck{desc->tree, desc, w};
  ck.run();
  out->violations = ck.violations;
  destroy(w);
  return ck.violations ? CF_E_STATE : CF_OK;
}

int cf_window_debug(cf_window* w, uint32_t flags) {
  if (!w) return fail(CF_E_INVALID, "null window");
  CfDevice g(w->ctx);
  if (!w->graphs.empty()) {   // captured with the old setting
    CF_CUDA(cudaStreamSynchronize(w->stream));
    for (auto& gr : w->graphs) CF_CUDA(cudaGraphExecDestroy(gr.exec));
    w->graphs.clear();
  }
  w->debug = flags;
  return CF_OK;
}

int cf_window_set_scale(cf_window* w, double scale) {
  if (!w) return fail(CF_E_INVALID, "null window");
  w->d.scale = scale;
  return CF_OK;
}

namespace {
int enqueue(cf_window* w, bool timing, uint64_t* h2d_out, uint64_t* d2h_out);
int one_run(cf_window* w, bool timing, uint64_t* h2d, uint64_t* d2h);
int finish(cf_window* w, cf_window_stats* st, uint64_t launches0, uint64_t h2d, uint64_t d2h, bool kernel_times,
           cudaEvent_t first);
}  // namespace

namespace {
// Batch prologue/epilogue on the context's compute stream: the windows' own streams fan out
// from it (ordered after earlier context work) and join back (ordered before later work).
int batch_begin(cf_ctx* c, cf_window* const* ws, int nw, cudaEvent_t first) {
  CF_CUDA(cudaEventRecord(first, c->compute));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, c->compute));
  CF_CUDA(cudaEventRecord(ws[0]->ev_fan, c->compute));
  for (int i = 0; i < nw; ++i) CF_CUDA(cudaStreamWaitEvent(ws[i]->stream, ws[0]->ev_fan, 0));
  return CF_OK;
}
int batch_end(cf_ctx* c, cf_window* const* ws, int nw, uint64_t* d2h, cudaEvent_t end) {
  for (int i = 0; i < nw; ++i) {
    CF_CUDA(cudaEventRecord(ws[i]->ev_fan, ws[i]->stream));
    CF_CUDA(cudaStreamWaitEvent(c->compute, ws[i]->ev_fan, 0));
  }
  // the error word (sticky over the batch) is read back once, after the last window
  CF_CUDA(cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, c->compute));
  *d2h += 8;
  CF_CUDA(cudaEventRecord(end, c->compute));
  return CF_OK;
}
}  // namespace

int cf_window_run(cf_window* w, int sync, cf_window_stats* st) {
  if (!w) return fail(CF_E_INVALID, "null window");
  CfDevice g(w->ctx);
  const uint64_t launches0 = w->ctx->launches.load();
  uint64_t h2d = 0, d2h = 0;
  const bool timing = sync != 0 && st != nullptr && !(w->d.flags & CF_WIN_GRAPH);
  CF_TRY(batch_begin(w->ctx, &w, 1, w->ev_first));
  CF_TRY(one_run(w, timing, &h2d, &d2h));
  CF_TRY(batch_end(w->ctx, &w, 1, &d2h, w->ev_end));
  if (!sync) return CF_OK;
  return finish(w, st, launches0, h2d, d2h, timing, w->ev_first);
}

int cf_window_run_n(cf_window* w, int nruns, double scale_even, double scale_odd, cf_window_stats* st) {
  return cf_window_run_pair(w, nullptr, nruns, scale_even, scale_odd, st);
}

int cf_window_run_pair(cf_window* w0, cf_window* w1, int nruns, double scale_even, double scale_odd,
                       cf_window_stats* st) {
  cf_window* ws[2] = {w0, w1};
  return cf_window_run_ring(ws, w1 ? 2 : 1, nruns, scale_even, scale_odd, st);
}

int cf_window_run_ring(cf_window* const* ws, int nw, int nruns, double scale_even, double scale_odd,
                       cf_window_stats* st) {
  if (!ws || nw < 1 || !ws[0] || nruns < 1) return fail(CF_E_INVALID, "bad arguments");
  cf_window* w0 = ws[0];
  for (int i = 1; i < nw; ++i)
    if (!ws[i] || ws[i]->ctx != w0->ctx || ws[i]->d.flags != w0->d.flags) return fail(CF_E_INVALID, "mismatched window ring");
  CfDevice g(w0->ctx);
  const uint64_t launches0 = w0->ctx->launches.load();
  uint64_t h2d = 0, d2h = 0;
  CF_TRY(batch_begin(w0->ctx, ws, nw, w0->ev_first));
  for (int r = 0; r < nruns; ++r) {
    cf_window* w = ws[r % nw];
    w->d.scale = (r & 1) ? scale_odd : scale_even;
    uint64_t a = 0, b = 0;
    CF_TRY(one_run(w, false, &a, &b));
    h2d += a;
    d2h += b;
  }
  CF_TRY(batch_end(w0->ctx, ws, nw, &d2h, w0->ev_end));
  return finish(w0, st, launches0, h2d, d2h, false, w0->ev_first);
}

int cf_window_run_n_flushed(cf_window* w, int nruns, double scale_even, double scale_odd, void* flush_buf,
                            uint64_t flush_bytes, cf_window_stats* st) {
  if (!w || nruns < 1 || (flush_bytes && !flush_buf)) return fail(CF_E_INVALID, "bad arguments");
  CfDevice g(w->ctx);
  std::vector<cudaEvent_t> ev(2 * size_t(nruns), nullptr);
  struct Guard { std::vector<cudaEvent_t>& e; ~Guard() { for (auto x : e) if (x) cudaEventDestroy(x); } } guard{ev};
  for (auto& e : ev) CF_CUDA(cudaEventCreate(&e));
  const uint64_t launches0 = w->ctx->launches.load();
  uint64_t h2d = 0, d2h = 0;
  CF_TRY(batch_begin(w->ctx, &w, 1, w->ev_first));
  for (int r = 0; r < nruns; ++r) {
    // evict the working set from L2 (outside the timed interval) with a read pass -- clean lines,
    // so no write-back of the flush lands inside the window -- then time this window alone
    if (flush_bytes) CF_TRY(launch_evict_read(w->ctx, flush_buf, flush_bytes, w->stream));
    CF_CUDA(cudaEventRecord(ev[2 * r], w->stream));
    w->d.scale = (r & 1) ? scale_odd : scale_even;
    uint64_t a = 0, b = 0;
    CF_TRY(one_run(w, false, &a, &b));
    CF_CUDA(cudaEventRecord(ev[2 * r + 1], w->stream));
    h2d += a;
    d2h += b;
  }
  CF_TRY(batch_end(w->ctx, &w, 1, &d2h, w->ev_end));
  CF_TRY(finish(w, st, launches0, h2d, d2h, false, w->ev_first));
  if (st) {
    float total = 0;
    for (int r = 0; r < nruns; ++r) {
      float ms = 0;
      CF_CUDA(cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]));
      total += ms;
    }
    st->ms_total = total;   // sum of the windows' own intervals (flushes excluded)
  }
  return CF_OK;
}

namespace {
// Direct enqueue, or (CF_WIN_GRAPH) capture the whole multi-stream sequence once per scale value
// into a CUDA graph and replay it: one launch call instead of ~100 per window.
int one_run(cf_window* w, bool timing, uint64_t* h2d, uint64_t* d2h) {
  if (!(w->d.flags & CF_WIN_GRAPH)) return enqueue(w, timing, h2d, d2h);
  cf_ctx* c = w->ctx;
  cf_window::Graph* gr = nullptr;
  for (auto& g : w->graphs)
    if (g.scale == w->d.scale) gr = &g;
  if (!gr) {
    // bounded cache: run_n alternates two scales; a caller cycling through more scales recaptures
    // instead of accumulating executable graphs (the evicted one may still be in flight: drain
    // this window's stream first)
    constexpr size_t MAX_GRAPHS = 4;
    if (w->graphs.size() >= MAX_GRAPHS) {
      CF_CUDA(cudaStreamSynchronize(w->stream));
      CF_CUDA(cudaGraphExecDestroy(w->graphs.front().exec));
      w->graphs.erase(w->graphs.begin());
    }
    cf_window::Graph g{w->d.scale, nullptr, 0, 0, 0};
    const uint64_t l0 = c->launches.load();
    CF_CUDA(cudaStreamBeginCapture(w->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue(w, false, &g.h2d, &g.d2h);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(w->stream, &graph);
    if (rc != CF_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (ce != cudaSuccess) return fail(CF_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(CF_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    g.launches = c->launches.load() - l0;
    c->launches.fetch_sub(g.launches);  // counted when the graph actually runs
    w->graphs.push_back(g);
    gr = &w->graphs.back();
  }
  CF_CUDA(cudaGraphLaunch(gr->exec, w->stream));
  c->launches.fetch_add(gr->launches);
  *h2d = gr->h2d;
  *d2h = gr->d2h;
  return CF_OK;
}

int enqueue(cf_window* w, bool timing, uint64_t* h2d_out, uint64_t* d2h_out) {
  cf_ctx* c = w->ctx;
  const cf_window_desc& d = w->d;
  const uint32_t fl = d.flags;
  const uint64_t nch = w->nsteps;
  uint8_t* img = static_cast<uint8_t*>(d.image);
  const uint8_t* src = static_cast<const uint8_t*>(d.host_src);
  uint8_t* dst = static_cast<uint8_t*>(d.host_dst);
  const uint64_t dimg = reinterpret_cast<uint64_t>(d.image);
  cudaStream_t cs = w->stream;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;

  // copy streams join only when this window copies anything (a resident window is kernels only)
  const bool copies = (fl & (CF_WIN_H2D | CF_WIN_D2H | CF_WIN_TABLES)) != 0;
  if (copies) {
    CF_CUDA(cudaEventRecord(w->ev_start, cs));
    for (auto s : c->h2d) CF_CUDA(cudaStreamWaitEvent(s, w->ev_start, 0));
    CF_CUDA(cudaStreamWaitEvent(c->d2h, w->ev_start, 0));
  }
  if (fl & CF_WIN_TABLES) {
    // the relocation / chain tables travel with the arena, first on the H2D copy stream
    // (an H2D copy on the compute stream serialises badly against the D2H engine)
    cudaStream_t s0 = c->h2d[0];
    CF_CUDA(cudaMemcpyAsync(w->d_tab, w->h_tab, w->tab_bytes, cudaMemcpyHostToDevice, s0));
    CF_CUDA(cudaEventRecord(w->ev_tables, s0));
    CF_CUDA(cudaStreamWaitEvent(cs, w->ev_tables, 0));
    h2d_bytes += w->tab_bytes;
  }
  const uint64_t* dsites = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_sites);
  const uint32_t* ddet = reinterpret_cast<const uint32_t*>(w->d_tab + w->off_det);
  const int32_t* dlv = reinterpret_cast<const int32_t*>(w->d_tab + w->off_level);
  const uint32_t* dod = reinterpret_cast<const uint32_t*>(w->d_tab + w->off_ord);
  const uint64_t* drt = w->has_roots ? reinterpret_cast<const uint64_t*>(w->d_tab + w->off_root) : nullptr;
  const bool chase = d.mode == CF_MODE_CHASE;
  static const bool no_uni = getenv("CF_NO_UNI") != nullptr;   // A/B switch (design experiments)

  for (uint64_t k = 0; k < nch; ++k) {
    if ((fl & CF_WIN_H2D) && k == 0 && w->zc) {
      // node records straight from the mapped host arena, one kernel for all of them
      CF_TRY(launch_seg_copy(c, reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zc_h2d), w->zc_n, src, img, cs));
      for (uint64_t j = 0; j < w->zc_n; ++j) h2d_bytes += w->seg_hi[j] - w->seg_lo[j];
    } else if (fl & CF_WIN_H2D) {
      cudaStream_t s = c->h2d[k % c->h2d.size()];
      for (uint64_t j = w->step_seg_lo[k]; j < w->step_seg_lo[k + 1]; ++j) {
        const uint64_t lo = w->seg_lo[j], hi = w->seg_hi[j];
        if (fl & CF_WIN_UVM) CF_CUDA(cudaMemPrefetchAsync(img + lo, hi - lo, c->device, s));   // migrate ahead
        else CF_CUDA(copy_host_aligned(img + lo, src + lo, hi - lo, cudaMemcpyHostToDevice, s));
        h2d_bytes += hi - lo;
      }
      CF_CUDA(cudaEventRecord(w->ev_h2d[k], s));
      CF_CUDA(cudaStreamWaitEvent(cs, w->ev_h2d[k], 0));
    }
    const uint64_t ns = w->reloc_lo[k + 1] - w->reloc_lo[k], nr = w->res_lo[k + 1] - w->res_lo[k];
    const bool do_attach = (fl & CF_WIN_ATTACH) && ns, do_resolve = (fl & CF_WIN_RESOLVE) && !chase && nr;
    bool resolved_last = false;   // the last op on cs is the attach / resolve launch
    // leaf-owned step (planned only when the window runs all four device phases, RESOLVED)
    const bool owned_step = w->own_any && w->own_step[k].on;
    LeafOwn own{};
    if (owned_step) {
      own = w->own_step[k];
      own.parent = w->d_parent + (own.p_first - w->parent_base);
      own.from = d.host_base;
      own.to = dimg;
      own.total = w->total;
      own.keep_attached = (w->debug & CF_WIN_DEBUG_KEEP_LEAF_ATTACHED) ? 1u : 0u;
      // every site of the step attached (the resolver-owned tail too: its resolvers run after)
      // || the owned range's parents resolved into the parent table
      CF_TRY(launch_attach_parents(c, img, w->total, dsites + w->reloc_lo[k], ns, d.host_base, dimg, w->sh, own,
                                   w->d_parent + (own.p_first - w->parent_base), c->d_bad, cs));
      if (nr)   // the step's other targets, from the tables (their fields are attached by now)
        CF_TRY(launch_resolve(c, img, w->sh, drt ? drt + w->res_lo[k] : nullptr, dlv + w->res_lo[k], dod + w->res_lo[k], nr,
                              w->d_ea + w->res_lo[k], w->d_count + w->res_lo[k], c->d_bad, cs, FAULT_RESOLVE));
      resolved_last = true;
    } else if (do_attach && do_resolve && ns <= SMALL_FUSED && nr <= SMALL_FUSED) {
      CF_TRY(launch_attach_resolve(c, img, w->total, dsites + w->reloc_lo[k], ns, d.host_base, dimg, w->sh,
                                   drt ? drt + w->res_lo[k] : nullptr, dlv + w->res_lo[k], dod + w->res_lo[k], nr, w->d_ea + w->res_lo[k],
                                   w->d_count + w->res_lo[k], c->d_bad, cs, FAULT_RESOLVE));
    } else if (do_attach && do_resolve && w->wide_ok) {
      CF_TRY(launch_attach_resolve_wide(c, img, w->total, dsites + w->reloc_lo[k], w->attach_n[k], d.host_base, dimg, w->sh,
                                        drt ? drt + w->res_lo[k] : nullptr, dlv + w->res_lo[k], dod + w->res_lo[k], nr,
                                        w->d_ea + w->res_lo[k], w->d_count + w->res_lo[k], c->d_bad, cs, FAULT_RESOLVE,
                                        w->uni[k].on && !no_uni ? &w->uni[k] : nullptr));
      resolved_last = true;
    } else {
      if (do_attach)
        CF_TRY(launch_relocate(c, img, w->total, dsites + w->reloc_lo[k], ns, d.host_base, dimg, c->d_bad, cs, nullptr,
                               FAULT_ATTACH));
      if (do_resolve)
        CF_TRY(launch_resolve(c, img, w->sh, drt ? drt + w->res_lo[k] : nullptr, dlv + w->res_lo[k], dod + w->res_lo[k], nr,
                              w->d_ea + w->res_lo[k],
                              w->d_count + w->res_lo[k], c->d_bad, cs, FAULT_RESOLVE));
    }
    // In RESOLVED mode the leaf kernel never reads pointer fields, and every resolve that reads
    // the fields detached at this step has already run: the detach rides in the same launch.
    const bool fuse_detach = ((fl & CF_WIN_DETACH) && (fl & CF_WIN_SCALE) && !chase && !timing) || owned_step;
    if (fl & CF_WIN_SCALE) {
      const cf_scale_work& sg = w->seg[k];
      const bool table_parts = sg.tile_end > sg.tile_begin || sg.group_end > sg.group_begin;
      const uint64_t nd = fuse_detach ? w->det_lo[k + 1] - w->det_lo[k] : 0;
      // programmatic dependent launch behind the attach / resolve launch (its CTAs are resident
      // and waiting when the resolver's last wave drains)
      static const bool no_pdl = getenv("CF_NO_PDL") != nullptr;   // A/B switch (design experiments)
      const bool pdl = resolved_last && !timing && !no_pdl;
      RelocArgs det{img, w->total, dsites, ddet + w->det_lo[k], nd, dimg, d.host_base, FAULT_DETACH};
      if (owned_step) {
        // the owned range (with the step's detach riding along), then any table-driven parts
        if (timing) CF_CUDA(cudaEventRecord(w->ev_k0[k], cs));
        CF_TRY(launch_scale(c, w->elem, d.mode, img, w->sh, drt, dlv, dod, w->d_ea, w->d_count, sg, d.scale, c->d_bad, cs,
                            nd ? &det : nullptr, FAULT_SCALE, pdl, &own));
        if (table_parts)
          CF_TRY(launch_scale(c, w->elem, d.mode, img, w->sh, drt, dlv, dod, w->d_ea, w->d_count, sg, d.scale, c->d_bad, cs,
                              nullptr, FAULT_SCALE));
        if (timing) CF_CUDA(cudaEventRecord(w->ev_k1[k], cs));
      } else if (table_parts || nd) {
        if (timing) CF_CUDA(cudaEventRecord(w->ev_k0[k], cs));
        CF_TRY(launch_scale(c, w->elem, d.mode, img, w->sh, drt, dlv, dod, w->d_ea, w->d_count, sg, d.scale, c->d_bad, cs,
                            nd ? &det : nullptr, FAULT_SCALE, pdl));
        if (timing) CF_CUDA(cudaEventRecord(w->ev_k1[k], cs));
      }
    }
    if ((fl & CF_WIN_DETACH) && !fuse_detach)
      CF_TRY(launch_relocate(c, img, w->total, dsites, w->det_lo[k + 1] - w->det_lo[k], dimg, d.host_base, c->d_bad, cs,
                             ddet + w->det_lo[k], FAULT_DETACH));
    if ((fl & CF_WIN_D2H) && w->zc && w->zc_rel_lo[k + 1] > w->zc_rel_lo[k]) {
      const uint64_t* zs = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zc_d2h) + 2 * w->zc_rel_lo[k];
      CF_TRY(launch_seg_copy(c, zs, w->zc_rel_lo[k + 1] - w->zc_rel_lo[k], img, dst, cs));
      for (uint64_t j = w->zc_rel_lo[k]; j < w->zc_rel_lo[k + 1]; ++j) {
        const uint64_t* hz = reinterpret_cast<const uint64_t*>(w->h_tab + w->off_zc_d2h);
        d2h_bytes += hz[2 * j + 1] - hz[2 * j];
      }
    }
    if ((fl & CF_WIN_D2H) && !w->released[k].empty()) {
      CF_CUDA(cudaEventRecord(w->ev_rel[k], cs));
      CF_CUDA(cudaStreamWaitEvent(c->d2h, w->ev_rel[k], 0));
      for (uint32_t r : w->released[k]) {
        const uint64_t rlo = w->seg_lo[r], rhi = w->seg_hi[r];
        if (fl & CF_WIN_UVM) CF_CUDA(cudaMemPrefetchAsync(img + rlo, rhi - rlo, cudaCpuDeviceId, c->d2h));   // migrate home
        else CF_CUDA(copy_host_aligned(dst + rlo, img + rlo, rhi - rlo, cudaMemcpyDeviceToHost, c->d2h));
        d2h_bytes += rhi - rlo;
      }
    }
  }
  // join the copy streams back into the compute stream
  if (copies) {
    for (auto s : c->h2d) {
      CF_CUDA(cudaEventRecord(w->ev_join, s));
      CF_CUDA(cudaStreamWaitEvent(cs, w->ev_join, 0));
    }
    CF_CUDA(cudaEventRecord(w->ev_join, c->d2h));
    CF_CUDA(cudaStreamWaitEvent(cs, w->ev_join, 0));
  }
  *h2d_out = h2d_bytes;
  *d2h_out = d2h_bytes;
  return CF_OK;
}

int finish(cf_window* w, cf_window_stats* st, uint64_t launches0, uint64_t h2d, uint64_t d2h, bool kernel_times,
           cudaEvent_t first) {
  cf_ctx* c = w->ctx;
  CF_CUDA(cudaEventSynchronize(w->ev_end));
  const uint64_t bad = c->h_bad[0];
  const uint64_t nch = w->nsteps;
  if (st) {
    memset(st, 0, sizeof *st);
    CF_CUDA(cudaEventElapsedTime(&st->ms_total, first, w->ev_end));
    float ks = 0;
    if (kernel_times) {
      for (uint64_t k = 0; k < nch; ++k) {
        const cf_scale_work& sg = w->seg[k];
        const bool launched = sg.tile_end > sg.tile_begin || sg.group_end > sg.group_begin ||
                              (w->own_any && w->own_step[k].on);
        if (!(w->d.flags & CF_WIN_SCALE) || !launched) continue;
        float ms = 0;
        CF_CUDA(cudaEventElapsedTime(&ms, w->ev_k0[k], w->ev_k1[k]));
        ks += ms;
      }
    }
    st->ms_kernel = ks;
    st->h2d_bytes = h2d;
    st->d2h_bytes = d2h;
    st->launches = c->launches.load() - launches0;
    st->bad = bad;
    st->nchunks = w->seg_lo.size();
    st->nsteps = nch;
  }
  if (bad != NO_BAD) {
    // the tag names the phase (the lowest-tagged fault wins: the reference's phase order)
    const uint64_t idx = bad & FAULT_INDEX_MASK;
    switch (bad & ~FAULT_INDEX_MASK) {
      case FAULT_ATTACH:   // memory.py:319-321
        return fail(CF_E_OUTSIDE_ARENA, "window attach: relocation-table entry %llu targets outside the arena",
                    (unsigned long long)idx);
      case FAULT_RESOLVE:  // a chain hop leaves the image (harness.py:285-304 walk -> WildAccess)
        return fail(CF_E_WILD, "window resolve: chain of target %llu leaves the device image", (unsigned long long)idx);
      case FAULT_SCALE:    // leaf span outside the image / beyond nA (memory.py:139-152)
        return fail(CF_E_WILD, "window leaf kernel: array of target %llu overruns the device image or its nA",
                    (unsigned long long)idx);
      default:             // demarshal's check, memory.py:337-343
        return fail(CF_E_OUTSIDE_ARENA, "window detach: pointer field (detach entry %llu) holds a value outside the device image",
                    (unsigned long long)idx);
    }
  }
  return CF_OK;
}
}  // namespace

int cf_window_free(cf_window* w) {
  destroy(w);
  return CF_OK;
}

}  // extern "C"
