// Pipelined pointerchain window: the reference's selective-copy scheme
//   transfer_to_device (pointerchain branch)  harness.py:228-238  one bulk copy per target array
//   kernel_scale       (pointerchain branch)  harness.py:255-259  scale through resolved addresses
//   copy_back          (pointerchain branch)  harness.py:312-325  one bulk copy back per array
// as one planned schedule.  The targeted arrays (host address, device buffer, count) are cut
// into steps of about one chunk.  Step k: its arrays' bytes go host -> device, the leaf kernel
// scales them, and they go back -- while step k+1 is already copying in.  Arrays of at least
// DMA_MIN bytes move on the copy engines (one H2D and one D2H stream, so the two directions
// overlap over the full-duplex link); smaller ones move by zero-copy SM kernels over the mapped
// pinned host memory, one warp per array, which avoids one copy-engine command per object (the
// C4 shape has a million 1 KiB arrays).  When a step's small arrays fill most of the host span
// they lie in (address-ordered layouts: C4's leaf arrays sit between 1.2 KB leaf blocks), that
// span goes in as ONE copy-engine DMA into a device staging area and a device-side copy list
// moves each array into its buffer: copy engine H2D beside SM-store D2H runs the full-duplex link
// at 88 GB/s where SM traffic both ways reaches 77 (profiles/r01_design_experiments.md).  The
// span goes back the same way (arrays packed into the staging slice, ONE D2H DMA) only when no
// other data shares it: no DMA-moved array of any step and no small array of another step may
// overlap it, or the span's stale staging bytes would land on their results.  All bookkeeping is
// planned once; a run only enqueues.
#include "cf_internal.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

using namespace cf;

namespace {
constexpr uint64_t DMA_MIN = 64 << 10;
// a step's small arrays are staged through one span DMA when they fill at least this share of it
constexpr double SPAN_MIN_FILL = 0.75;
}

struct cf_selective {
  cf_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;   // compute stream of this window
  int elem = 4;
  uint64_t n = 0, nsteps = 0;
  struct Piece { uint64_t src, dst, bytes; };
  std::vector<Piece> dma;                  // DMA pieces, grouped by step
  std::vector<uint64_t> dma_lo;            // per step: range in dma
  std::vector<uint64_t> zc_lo;             // per step: range in the zero-copy list
  std::vector<cf_scale_work> work;         // per step: leaf-kernel work (device pointers set)
  uint64_t nzc = 0;
  std::vector<Piece> span;                 // per step: staged host span (bytes 0 = none); dst = staging offset
  std::vector<uint8_t> span_out;           // per step: the span also goes back as one DMA (see sel_plan)
  uint8_t* d_stage = nullptr;              // staging area (device) for the span DMAs
  uint64_t stage_bytes = 0;
  // one pinned table block + device mirror: ea u64[n] | count u32[n] | zc src u64[nzc] |
  // zc dst u64[nzc] | zc bytes u64[nzc] | zc in-source u64[nzc] | parts | tile_base | groups
  // (in-source: where the H2D copy list reads an entry -- its host address, or its place in the
  // staging area when its step's span is staged)
  uint8_t* h_tab = nullptr;
  uint8_t* d_tab = nullptr;
  uint64_t tab_bytes = 0, off_cnt = 0, off_zs = 0, off_zd = 0, off_zb = 0, off_zi = 0;
  std::vector<cudaEvent_t> ev_in, ev_out;
  cudaEvent_t ev_start = nullptr, ev_tab = nullptr, ev_join = nullptr;
  // dry run (cf_selective_plan_check): the host plan, no CUDA state
  struct Dry { std::vector<uint64_t> zsrc, zdst, zbytes; ScaleWork sw; };
  Dry* dry = nullptr;
};

namespace {
void destroy(cf_selective* w) {
  if (!w) return;
  if (w->dry) {
    delete w->dry;
    delete w;
    return;
  }
  CfDevice g(w->ctx);
  if (w->h_tab) cudaFreeHost(w->h_tab);
  if (w->d_tab) cudaFree(w->d_tab);
  if (w->d_stage) cudaFree(w->d_stage);
  for (auto e : w->ev_in) cudaEventDestroy(e);
  for (auto e : w->ev_out) cudaEventDestroy(e);
  for (auto e : {w->ev_start, w->ev_tab, w->ev_join})
    if (e) cudaEventDestroy(e);
  if (w->stream) cudaStreamDestroy(w->stream);
  delete w;
}
}  // namespace

namespace {
int sel_plan(cf_ctx* ctx, uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count, int elem,
             uint64_t chunk_bytes, cf_selective** out, bool dry, bool dry_mapped, const uint8_t* scale_mask = nullptr,
             uint32_t plan_flags = 0) {
  if (!out || (n && (!h_src || !d_buf || !count))) return fail(CF_E_INVALID, "null argument");
  if (elem != 4 && elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  CfDevice g(dry ? nullptr : ctx);
  cf_selective* w = new cf_selective();
  w->ctx = ctx;
  w->elem = elem;
  w->n = n;
  if (dry) w->dry = new cf_selective::Dry();
  const uint64_t ch = std::max<uint64_t>(chunk_bytes ? chunk_bytes : (16ull << 20), TILE_BYTES);
  // zero-copy needs every small array's host memory mapped at the same address (UVA pinned)
  bool mapped = true;
  if (dry) {
    mapped = dry_mapped;
  } else {
    for (uint64_t i = 0; i < n && mapped; ++i) {
      if (count[i] * uint64_t(elem) >= DMA_MIN) continue;
      void* dp = nullptr;
      mapped = cudaHostGetDevicePointer(&dp, reinterpret_cast<void*>(h_src[i]), 0) == cudaSuccess &&
               reinterpret_cast<uint64_t>(dp) == h_src[i];
    }
    cudaGetLastError();
  }
  std::vector<uint64_t> zsrc, zdst, zbytes;
  ScaleWork sw;
  sw.elem = elem;
  std::vector<uint64_t> tri;
  uint64_t acc = 0;
  auto close_step = [&]() {
    w->work.push_back(sw.append(tri));
    tri.clear();
    w->dma_lo.push_back(w->dma.size());
    w->zc_lo.push_back(zsrc.size());
    acc = 0;
  };
  w->dma_lo.push_back(0);
  w->zc_lo.push_back(0);
  const uint64_t piece_elems = ch / uint64_t(elem);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bytes = count[i] * uint64_t(elem);
    if (bytes == 0) continue;
    if (bytes < DMA_MIN && mapped) {
      if (acc + bytes > ch && acc) close_step();
      zsrc.push_back(h_src[i]);
      zdst.push_back(d_buf[i]);
      zbytes.push_back(bytes);
      if (!scale_mask || scale_mask[i]) tri.insert(tri.end(), {i, 0, count[i]});
      acc += bytes;
      continue;
    }
    for (uint64_t e0 = 0; e0 < count[i]; e0 += piece_elems) {
      const uint64_t e1 = std::min(count[i], e0 + piece_elems);
      const uint64_t pb = (e1 - e0) * uint64_t(elem);
      if (acc + pb > ch && acc) close_step();
      w->dma.push_back({h_src[i] + e0 * uint64_t(elem), d_buf[i] + e0 * uint64_t(elem), pb});
      if (!scale_mask || scale_mask[i]) tri.insert(tri.end(), {i, e0, e1});
      acc += pb;
    }
  }
  if (acc || w->work.empty()) close_step();
  w->nsteps = w->work.size();
  w->nzc = zsrc.size();
  // staged spans: per step, the host range its zero-copy entries lie in, when they fill it densely
  // (staging offsets keep the host address mod 256, so the copy list's 16-byte paths still apply)
  w->span.assign(w->nsteps, cf_selective::Piece{0, 0, 0});
  for (uint64_t k = 0; k < w->nsteps && !(plan_flags & CF_SEL_PER_OBJECT); ++k) {
    const uint64_t z0 = w->zc_lo[k], z1 = w->zc_lo[k + 1];
    if (z1 - z0 < 2) continue;
    uint64_t lo = ~uint64_t(0), hi = 0, fill = 0;
    for (uint64_t j = z0; j < z1; ++j) {
      lo = std::min(lo, zsrc[j]);
      hi = std::max(hi, zsrc[j] + zbytes[j]);
      fill += zbytes[j];
    }
    if (hi - lo < DMA_MIN || double(fill) < SPAN_MIN_FILL * double(hi - lo)) continue;
    const uint64_t off = (w->stage_bytes + 255) / 256 * 256 + (lo & 255);
    w->span[k] = cf_selective::Piece{lo, off, hi - lo};
    w->stage_bytes = off + (hi - lo);
  }
  // Copy-back through the staged span too (arrays packed into the staging slice on the device,
  // then ONE D2H DMA of the span: copy engines both ways run the link at 99 GB/s where SM stores
  // beside a DMA reach 88) -- only when that cannot disturb anything: every selected array that
  // overlaps the span is one of this step's own zero-copy entries, which are packed into the
  // slice before the DMA (the bytes between them go back exactly as they were read at the start
  // of this window, which no one can change before copy_back returns).  A DMA-moved array inside
  // the span -- even one of step k -- is scaled in its own buffer and goes home by its own DMA;
  // the span DMA would then overwrite it with the unscaled staging bytes, so it disqualifies.
  w->span_out.assign(w->nsteps, 0);
  {
    constexpr uint64_t DMA_PIECE = ~uint64_t(0);   // step tag of DMA pieces: overlap always disqualifies
    struct Iv { uint64_t lo, hi, step; };
    std::vector<Iv> iv;
    iv.reserve(zsrc.size() + w->dma.size());
    for (uint64_t k = 0; k < w->nsteps; ++k) {
      for (uint64_t j = w->zc_lo[k]; j < w->zc_lo[k + 1]; ++j) iv.push_back({zsrc[j], zsrc[j] + zbytes[j], k});
      for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j)
        iv.push_back({w->dma[j].src, w->dma[j].src + w->dma[j].bytes, DMA_PIECE});
    }
    std::sort(iv.begin(), iv.end(), [](const Iv& a, const Iv& b) { return a.lo < b.lo; });
    uint64_t maxlen = 0;
    for (const Iv& v : iv) maxlen = std::max(maxlen, v.hi - v.lo);
    for (uint64_t k = 0; k < w->nsteps && !(plan_flags & CF_SEL_PER_OBJECT); ++k) {
      const cf_selective::Piece& sp = w->span[k];
      if (!sp.bytes) continue;
      const uint64_t lo = sp.src, hi = sp.src + sp.bytes;
      // intervals starting in [lo - maxlen, hi) are the only ones that can overlap
      auto it = std::lower_bound(iv.begin(), iv.end(), lo > maxlen ? lo - maxlen : 0,
                                 [](const Iv& a, uint64_t x) { return a.lo < x; });
      bool ok = true;
      for (; it != iv.end() && it->lo < hi && ok; ++it)
        if (it->hi > lo && it->step != k) ok = false;
      w->span_out[k] = ok;
    }
  }
  // table block
  auto al8 = [](uint64_t x) { return (x + 7) & ~7ull; };
  w->off_cnt = al8(n * 8);
  w->off_zs = al8(w->off_cnt + n * 4);
  w->off_zd = w->off_zs + w->nzc * 8;
  w->off_zb = w->off_zd + w->nzc * 8;
  w->off_zi = w->off_zb + w->nzc * 8;
  const uint64_t off_parts = w->off_zi + w->nzc * 8;
  const uint64_t off_tb = al8(off_parts + sw.parts.size() * 4);
  const uint64_t off_grp = al8(off_tb + sw.tile_base.size() * 8);
  w->tab_bytes = al8(off_grp + sw.groups.size() * 4 + 8);
  if (dry) {
    w->dry->zsrc = std::move(zsrc);
    w->dry->zdst = std::move(zdst);
    w->dry->zbytes = std::move(zbytes);
    w->dry->sw = std::move(sw);
    *out = w;
    return CF_OK;
  }
  cudaError_t ce = cudaHostAlloc(&w->h_tab, w->tab_bytes, cudaHostAllocPortable);
  if (ce == cudaSuccess) ce = cudaMalloc(&w->d_tab, w->tab_bytes);
  if (ce == cudaSuccess && w->stage_bytes) ce = cudaMalloc(&w->d_stage, w->stage_bytes);
  if (ce != cudaSuccess) { cudaGetLastError(); destroy(w); return fail(CF_E_OOM, "selective tables: %s", cudaGetErrorString(ce)); }
  uint32_t* cnt32 = reinterpret_cast<uint32_t*>(w->h_tab + w->off_cnt);
  for (uint64_t i = 0; i < n; ++i) {
    if (count[i] >> 32) { destroy(w); return fail(CF_E_INVALID, "count %llu does not fit the u32 nA field", (unsigned long long)count[i]); }
    cnt32[i] = uint32_t(count[i]);
  }
  if (n) memcpy(w->h_tab, d_buf, n * 8);
  if (w->nzc) {
    memcpy(w->h_tab + w->off_zs, zsrc.data(), w->nzc * 8);
    memcpy(w->h_tab + w->off_zd, zdst.data(), w->nzc * 8);
    memcpy(w->h_tab + w->off_zb, zbytes.data(), w->nzc * 8);
    uint64_t* zi = reinterpret_cast<uint64_t*>(w->h_tab + w->off_zi);
    for (uint64_t k = 0; k < w->nsteps; ++k)
      for (uint64_t j = w->zc_lo[k]; j < w->zc_lo[k + 1]; ++j)
        zi[j] = w->span[k].bytes ? reinterpret_cast<uint64_t>(w->d_stage) + w->span[k].dst + (zsrc[j] - w->span[k].src)
                                 : zsrc[j];
  }
  if (!sw.parts.empty()) memcpy(w->h_tab + off_parts, sw.parts.data(), sw.parts.size() * 4);
  if (!sw.tile_base.empty()) memcpy(w->h_tab + off_tb, sw.tile_base.data(), sw.tile_base.size() * 8);
  if (!sw.groups.empty()) memcpy(w->h_tab + off_grp, sw.groups.data(), sw.groups.size() * 4);
  for (auto& k : w->work) {
    k.parts = reinterpret_cast<const uint32_t*>(w->d_tab + off_parts);
    k.tile_base = reinterpret_cast<const uint64_t*>(w->d_tab + off_tb);
    k.groups = reinterpret_cast<const uint32_t*>(w->d_tab + off_grp);
  }
  bool ok = cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&w->ev_start, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&w->ev_tab, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming) == cudaSuccess;
  w->ev_in.resize(w->nsteps, nullptr);
  w->ev_out.resize(w->nsteps, nullptr);
  for (uint64_t k = 0; k < w->nsteps && ok; ++k)
    ok = cudaEventCreateWithFlags(&w->ev_in[k], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&w->ev_out[k], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) { cudaGetLastError(); destroy(w); return fail(CF_E_CUDA, "selective window streams/events"); }
  *out = w;
  return CF_OK;
}

}  // namespace

extern "C" {

int cf_selective_plan(cf_ctx* ctx, uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count,
                      int elem, uint64_t chunk_bytes, cf_selective** out) {
  if (!ctx) return fail(CF_E_INVALID, "null argument");
  return sel_plan(ctx, n, h_src, d_buf, count, elem, chunk_bytes, out, false, false);
}

int cf_selective_plan_ex(cf_ctx* ctx, uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count,
                         const uint8_t* scale_mask, uint32_t plan_flags, int elem, uint64_t chunk_bytes, cf_selective** out) {
  if (!ctx) return fail(CF_E_INVALID, "null argument");
  return sel_plan(ctx, n, h_src, d_buf, count, elem, chunk_bytes, out, false, false, scale_mask, plan_flags);
}

int cf_selective_plan_check(uint64_t n, const uint64_t* h_src, const uint64_t* d_buf, const uint64_t* count, int elem,
                            uint64_t chunk_bytes, int mapped, uint64_t* nsteps) {
  // invariants: every array's bytes move exactly once (DMA pieces or one zero-copy entry) from its
  // host address to its device buffer, and the leaf kernel of step k scales exactly the elements
  // that moved in step k -- each array's [0, count) once
  cf_selective* w = nullptr;
  CF_TRY(sel_plan(nullptr, n, h_src, d_buf, count, elem, chunk_bytes, &w, true, mapped != 0));
  const auto& D = *w->dry;
  const uint64_t e = uint64_t(elem);
  int bad = 0;
  auto report = [&](const char* msg, uint64_t a, uint64_t b) {
    if (bad++ == 0) fail(CF_E_STATE, "%s (%llu, %llu)", msg, (unsigned long long)a, (unsigned long long)b);
  };
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> moved(n), scaled(n);   // element ranges per array
  // address -> array lookup over the host ranges (sorted by host address)
  std::vector<std::pair<uint64_t, uint64_t>> by_host;
  for (uint64_t i = 0; i < n; ++i)
    if (count[i]) by_host.push_back({h_src[i], i});
  std::sort(by_host.begin(), by_host.end());
  auto owner = [&](uint64_t host) -> int64_t {
    auto it = std::upper_bound(by_host.begin(), by_host.end(), std::make_pair(host, ~uint64_t(0)));
    if (it == by_host.begin()) return -1;
    --it;
    const uint64_t i = it->second;
    return host < h_src[i] + count[i] * e ? int64_t(i) : -1;
  };
  uint64_t stage_end = 0;
  for (uint64_t k = 0; k < w->nsteps; ++k) {
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> step_moved(n);
    auto move = [&](uint64_t src, uint64_t dst, uint64_t bytes) {
      const int64_t i = owner(src);
      if (i < 0) { report("copy from outside every array", src, bytes); return; }
      const uint64_t off = src - h_src[i];
      if (dst != d_buf[i] + off || off % e || bytes % e || off + bytes > count[i] * e) { report("copy misplaced", src, dst); return; }
      step_moved[i].push_back({off / e, (off + bytes) / e});
      moved[i].push_back({off / e, (off + bytes) / e});
    };
    for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j) move(w->dma[j].src, w->dma[j].dst, w->dma[j].bytes);
    for (uint64_t j = w->zc_lo[k]; j < w->zc_lo[k + 1]; ++j) move(D.zsrc[j], D.zdst[j], D.zbytes[j]);
    // a staged span holds every zero-copy entry of its step, in its own slice of the staging area
    const auto& sp = w->span[k];
    if (sp.bytes) {
      if (sp.dst < stage_end || sp.dst % 256 != sp.src % 256) report("staging slice misplaced", k, sp.dst);
      stage_end = sp.dst + sp.bytes;
      for (uint64_t j = w->zc_lo[k]; j < w->zc_lo[k + 1]; ++j)
        if (D.zsrc[j] < sp.src || D.zsrc[j] + D.zbytes[j] > sp.src + sp.bytes) report("entry outside its staged span", k, j);
    }
    const cf_scale_work& ws = w->work[k];
    auto part = [&](uint64_t p) {
      const uint64_t i = D.sw.parts[3 * p], e0 = D.sw.parts[3 * p + 1], e1 = D.sw.parts[3 * p + 2];
      if (i >= n) { report("part names array", p, i); return; }
      bool in = false;   // the part's elements moved in this very step
      for (auto& r : step_moved[i]) in |= r.first <= e0 && e1 <= r.second;
      if (!in) report("part scaled in a step that did not move it", i, k);
      scaled[i].push_back({e0, e1});
    };
    for (uint64_t p = ws.big_begin; p < ws.big_begin + ws.big_count; ++p) part(p);
    for (uint64_t gr = ws.group_begin; gr < ws.group_end; ++gr)
      for (uint64_t p = D.sw.groups[2 * gr]; p < D.sw.groups[2 * gr + 1]; ++p) part(p);
  }
  for (uint64_t i = 0; i < n; ++i)
    for (auto* v : {&moved[i], &scaled[i]}) {
      std::sort(v->begin(), v->end());
      uint64_t y = 0;
      for (auto& r : *v) {
        if (r.first != y) { report("array not tiled exactly once", i, r.first); break; }
        y = r.second;
      }
      if (y != count[i]) report("array covered up to", i, y);
    }
  if (stage_end > w->stage_bytes) report("staging area too small", stage_end, w->stage_bytes);
  // a span copied back whole must not overlap any array moved by another step, nor any DMA piece
  // of any step -- its own included: that piece is scaled in its buffer and goes home by its own
  // DMA, which the span DMA would overwrite with unscaled staging bytes (quadratic, small n)
  for (uint64_t k = 0; k < w->nsteps; ++k) {
    if (!w->span_out[k]) continue;
    if (!w->span[k].bytes) { report("span copied back without a span", k, 0); continue; }
    const uint64_t lo = w->span[k].src, hi = lo + w->span[k].bytes;
    for (uint64_t j = 0; j < w->nsteps; ++j) {
      for (uint64_t q = w->dma_lo[j]; q < w->dma_lo[j + 1]; ++q)
        if (w->dma[q].src < hi && w->dma[q].src + w->dma[q].bytes > lo) report("copied-back span overlaps a DMA piece", k, j);
      if (j == k) continue;
      for (uint64_t q = w->zc_lo[j]; q < w->zc_lo[j + 1]; ++q)
        if (D.zsrc[q] < hi && D.zsrc[q] + D.zbytes[q] > lo) report("copied-back span overlaps another step's array", k, j);
    }
  }
  if (nsteps) *nsteps = w->nsteps;
  destroy(w);
  return bad ? CF_E_STATE : CF_OK;
}

int cf_selective_run(cf_selective* w, uint32_t flags, double scale) {
  if (!w) return fail(CF_E_INVALID, "null window");
  cf_ctx* c = w->ctx;
  CfDevice g(c);
  cudaStream_t cs = w->stream, hs = c->h2d[0], ds = c->d2h;
  const uint64_t* ea = reinterpret_cast<const uint64_t*>(w->d_tab);
  const uint32_t* cnt = reinterpret_cast<const uint32_t*>(w->d_tab + w->off_cnt);
  const uint64_t* zs = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zs);
  const uint64_t* zd = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zd);
  const uint64_t* zb = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zb);
  const uint64_t* zi = reinterpret_cast<const uint64_t*>(w->d_tab + w->off_zi);
  // fan out from the context's compute stream (ordered after earlier work on this context)
  CF_CUDA(cudaEventRecord(w->ev_start, c->compute));
  for (cudaStream_t s : {cs, hs, ds}) CF_CUDA(cudaStreamWaitEvent(s, w->ev_start, 0));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, cs));
  // the resolved-address / work tables travel with the data, first on the H2D stream
  CF_CUDA(cudaMemcpyAsync(w->d_tab, w->h_tab, w->tab_bytes, cudaMemcpyHostToDevice, hs));
  CF_CUDA(cudaEventRecord(w->ev_tab, hs));
  CF_CUDA(cudaStreamWaitEvent(cs, w->ev_tab, 0));
  cf_chain_shape sh;
  memset(&sh, 0, sizeof sh);
  // Full windows: the zero-copy copy-out of step k and copy-in of step k+1 run as ONE launch on
  // the compute stream (warps interleaved), so both link directions share every SM; the DMA
  // pieces keep their own H2D / D2H copy-engine streams.
  const bool duplex = (flags & CF_WIN_H2D) && (flags & CF_WIN_D2H) && (flags & CF_WIN_SCALE) && w->nzc &&
                      !getenv("CF_SEL_NO_DUPLEX");
  if (duplex) {
    auto zin = [&](uint64_t k) { return w->zc_lo[k]; };
    auto nz = [&](uint64_t k) { return w->zc_lo[k + 1] - w->zc_lo[k]; };
    auto dma_in = [&](uint64_t k) -> int {
      for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j)
        CF_CUDA(copy_host_aligned(reinterpret_cast<void*>(w->dma[j].dst), reinterpret_cast<const void*>(w->dma[j].src),
                                  w->dma[j].bytes, cudaMemcpyHostToDevice, hs));
      const cf_selective::Piece& sp = w->span[k];
      if (sp.bytes)
        CF_CUDA(copy_host_aligned(w->d_stage + sp.dst, reinterpret_cast<const void*>(sp.src), sp.bytes, cudaMemcpyHostToDevice, hs));
      CF_CUDA(cudaEventRecord(w->ev_in[k], hs));
      return CF_OK;
    };
    for (uint64_t k = 0; k < w->nsteps; ++k) CF_TRY(dma_in(k));   // the copy engine streams run ahead
    if (w->span[0].bytes) CF_CUDA(cudaStreamWaitEvent(cs, w->ev_in[0], 0));
    CF_TRY(launch_copy_list(c, zi + zin(0), zd + zin(0), zb + zin(0), nz(0), cs));
    for (uint64_t k = 0; k < w->nsteps; ++k) {
      CF_CUDA(cudaStreamWaitEvent(cs, w->ev_in[k], 0));
      CF_TRY(launch_scale(c, w->elem, CF_MODE_RESOLVED, nullptr, sh, nullptr, nullptr, nullptr, ea, cnt, w->work[k], scale,
                          c->d_bad, cs));
      CF_CUDA(cudaEventRecord(w->ev_out[k], cs));
      CF_CUDA(cudaStreamWaitEvent(ds, w->ev_out[k], 0));
      for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j)
        CF_CUDA(copy_host_aligned(reinterpret_cast<void*>(w->dma[j].src), reinterpret_cast<const void*>(w->dma[j].dst),
                                  w->dma[j].bytes, cudaMemcpyDeviceToHost, ds));
      // copy-out of step k (device buffers -> host, or packed into its staged span) beside the
      // copy-in of step k+1
      const bool packed = w->span_out[k];
      const uint64_t* out_dst = packed ? zi : zs;
      if (k + 1 < w->nsteps) {
        if (w->span[k + 1].bytes) CF_CUDA(cudaStreamWaitEvent(cs, w->ev_in[k + 1], 0));   // staged copy-in source
        CF_TRY(launch_copy_list2(c, zd + zin(k), out_dst + zin(k), zb + zin(k), nz(k), zi + zin(k + 1), zd + zin(k + 1),
                                 zb + zin(k + 1), nz(k + 1), cs));
      } else {
        CF_TRY(launch_copy_list(c, zd + zin(k), out_dst + zin(k), zb + zin(k), nz(k), cs));
      }
      if (packed) {   // the whole span back in one DMA once its arrays are packed
        const cf_selective::Piece& sp = w->span[k];
        CF_CUDA(cudaEventRecord(w->ev_out[k], cs));
        CF_CUDA(cudaStreamWaitEvent(ds, w->ev_out[k], 0));
        CF_CUDA(copy_host_aligned(reinterpret_cast<void*>(sp.src), w->d_stage + sp.dst, sp.bytes, cudaMemcpyDeviceToHost, ds));
      }
    }
  }
  for (uint64_t k = 0; k < w->nsteps && !duplex; ++k) {
    if (flags & CF_WIN_H2D) {
      for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j)
        CF_CUDA(copy_host_aligned(reinterpret_cast<void*>(w->dma[j].dst), reinterpret_cast<const void*>(w->dma[j].src),
                                w->dma[j].bytes, cudaMemcpyHostToDevice, hs));
      const cf_selective::Piece& sp = w->span[k];
      if (sp.bytes)
        CF_CUDA(copy_host_aligned(w->d_stage + sp.dst, reinterpret_cast<const void*>(sp.src), sp.bytes, cudaMemcpyHostToDevice, hs));
      CF_CUDA(cudaEventRecord(w->ev_in[k], hs));
      CF_CUDA(cudaStreamWaitEvent(cs, w->ev_in[k], 0));
      // small arrays: one warp per array pulls it over the mapped host memory, or out of the
      // staged span in HBM
      CF_TRY(launch_copy_list(c, zi + w->zc_lo[k], zd + w->zc_lo[k], zb + w->zc_lo[k], w->zc_lo[k + 1] - w->zc_lo[k], cs));
    }
    if (flags & CF_WIN_SCALE)
      CF_TRY(launch_scale(c, w->elem, CF_MODE_RESOLVED, nullptr, sh, nullptr, nullptr, nullptr, ea, cnt, w->work[k], scale,
                          c->d_bad, cs));
    if (flags & CF_WIN_D2H) {
      CF_CUDA(cudaEventRecord(w->ev_out[k], cs));
      CF_CUDA(cudaStreamWaitEvent(ds, w->ev_out[k], 0));
      for (uint64_t j = w->dma_lo[k]; j < w->dma_lo[k + 1]; ++j)
        CF_CUDA(copy_host_aligned(reinterpret_cast<void*>(w->dma[j].src), reinterpret_cast<const void*>(w->dma[j].dst),
                                w->dma[j].bytes, cudaMemcpyDeviceToHost, ds));
      // small arrays pushed back by SM stores into mapped host memory, on the D2H stream
      CF_TRY(launch_copy_list(c, zd + w->zc_lo[k], zs + w->zc_lo[k], zb + w->zc_lo[k], w->zc_lo[k + 1] - w->zc_lo[k], ds));
    }
  }
  for (cudaStream_t s : {hs, ds}) {
    CF_CUDA(cudaEventRecord(w->ev_join, s));
    CF_CUDA(cudaStreamWaitEvent(cs, w->ev_join, 0));
  }
  CF_CUDA(cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, cs));
  CF_CUDA(cudaEventRecord(w->ev_join, cs));
  CF_CUDA(cudaStreamWaitEvent(c->compute, w->ev_join, 0));
  CF_CUDA(cudaStreamSynchronize(cs));
  if (c->h_bad[0] != NO_BAD)
    return fail(CF_E_WILD, "leaf kernel: buffer %llu rejected", (unsigned long long)c->h_bad[0]);
  return CF_OK;
}

int cf_selective_free(cf_selective* w) {
  destroy(w);
  return CF_OK;
}

}  // extern "C"
