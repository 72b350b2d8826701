// C-ABI entry points for the device kernels and the reference-named composite operations:
//   cf_marshal_transfer_and_attach  <- Machine.marshal_transfer_and_attach  memory.py:307-325
//   cf_demarshal                    <- Machine.demarshal                    memory.py:327-345
//   cf_kernel_scale                 <- kernel_scale (marshalling/naive walk) harness.py:244-304
//   cf_naive_fixup                  <- naive_deep_copy fix-up loop         memory.py:362-364
//   cf_arena_check_sites            <- the attach loop's bounds check      memory.py:319-321
//   cf_checksum_ranges              <- result gather of the multi-GPU shards
//   cf_copy_objects                 <- per-object transfers (naive_deep_copy / copy-back and
//                                      the selective copies, memory.py:358-361, 368-372)
#include "cf_internal.h"

#include <algorithm>
#include <cstring>
#include <vector>

using namespace cf;

namespace {

cudaStream_t pick(cf_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->compute; }

// Device scratch taken from the context's grow-only buffer (callers are synchronous, one
// operation at a time per context).
struct DevBuf {
  cf_ctx* c;
  void* p = nullptr;
  explicit DevBuf(cf_ctx* ctx) : c(ctx) {}
  int alloc(uint64_t bytes) {
    if (bytes == 0) bytes = 8;
    if (bytes > c->scratch_bytes) {
      if (c->scratch) {
        cudaStreamSynchronize(c->compute);
        cudaFree(c->scratch);
        c->scratch = nullptr;
        c->scratch_bytes = 0;
      }
      const uint64_t want = std::max<uint64_t>(bytes, 1ull << 20);
      cudaError_t e = cudaMalloc(&c->scratch, want);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA, "cudaMalloc(%llu): %s",
                    (unsigned long long)want, cudaGetErrorString(e));
      }
      c->scratch_bytes = want;
    }
    p = c->scratch;
    return CF_OK;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

struct EventSet {
  std::vector<cudaEvent_t> ev;
  ~EventSet() { for (auto e : ev) cudaEventDestroy(e); }
  int make(size_t n) {
    ev.resize(n, nullptr);
    for (auto& e : ev) CF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return CF_OK;
  }
};

// Chunk boundaries over [0, total) at multiples of chunk, moved down so that no 8-byte pointer
// field straddles two chunks (packed layouts put fields at 4 mod 8).
std::vector<uint64_t> chunk_bounds(uint64_t total, uint64_t chunk, const uint64_t* sites, uint64_t nsites) {
  std::vector<uint64_t> b{0};
  if (chunk == 0 || chunk >= total) {
    b.push_back(total);
    return b;
  }
  for (uint64_t x = chunk; x < total; x += chunk) {
    uint64_t y = x;
    if (nsites) {
      const uint64_t* it = std::lower_bound(sites, sites + nsites, x >= 7 ? x - 7 : 0);
      if (it != sites + nsites && *it < x && *it + 8 > x) y = *it;
    }
    if (y > b.back()) b.push_back(y);
  }
  b.push_back(total);
  return b;
}

// Upload a host ScaleWork into `dst` (device) and point `w` at it.
uint64_t work_bytes(const ScaleWork& sw) {
  return ((sw.parts.size() * 4 + 7) / 8) * 8 + sw.tile_base.size() * 8 + sw.groups.size() * 4 + 8;
}
int upload_work(const ScaleWork& sw, uint8_t* dst, cudaStream_t s, cf_scale_work* w) {
  const uint64_t n1 = ((sw.parts.size() * 4 + 7) / 8) * 8, n2 = sw.tile_base.size() * 8, n3 = sw.groups.size() * 4;
  if (!sw.parts.empty()) CF_CUDA(cudaMemcpyAsync(dst, sw.parts.data(), sw.parts.size() * 4, cudaMemcpyHostToDevice, s));
  if (n2) CF_CUDA(cudaMemcpyAsync(dst + n1, sw.tile_base.data(), n2, cudaMemcpyHostToDevice, s));
  if (n3) CF_CUDA(cudaMemcpyAsync(dst + n1 + n2, sw.groups.data(), n3, cudaMemcpyHostToDevice, s));
  w->parts = reinterpret_cast<const uint32_t*>(dst);
  w->tile_base = reinterpret_cast<const uint64_t*>(dst + n1);
  w->groups = reinterpret_cast<const uint32_t*>(dst + n1 + n2);
  return CF_OK;
}

int read_bad(cf_ctx* c, const uint64_t* d_bad, cudaStream_t s, uint64_t* out) {
  CF_CUDA(cudaMemcpyAsync(c->h_bad, d_bad, 8, cudaMemcpyDeviceToHost, s));
  CF_CUDA(cudaStreamSynchronize(s));
  *out = c->h_bad[0];
  return CF_OK;
}

}  // namespace

extern "C" {

int cf_relocate(cf_ctx* c, void* image, uint64_t image_bytes, const uint64_t* d_sites, uint64_t nsites,
                uint64_t from_base, uint64_t to_base, uint64_t* d_bad, void* stream) {
  if (!c || (!image && nsites)) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  return launch_relocate(c, static_cast<uint8_t*>(image), image_bytes, d_sites, nsites, from_base, to_base,
                         d_bad, pick(c, stream));
}

int cf_resolve(cf_ctx* c, const void* image, const cf_chain_shape* shape, const uint64_t* d_root,
               const int32_t* d_level, const uint32_t* d_ordinal, uint64_t ntargets, uint64_t* d_ea,
               uint32_t* d_count, uint64_t* d_bad, void* stream) {
  if (!c || !shape) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  return launch_resolve(c, static_cast<const uint8_t*>(image), *shape, d_root, d_level, d_ordinal, ntargets, d_ea,
                        d_count, d_bad, pick(c, stream));
}

int cf_scale(cf_ctx* c, int elem, int mode, const void* image, const cf_chain_shape* shape,
             const uint64_t* d_root, const int32_t* d_level, const uint32_t* d_ordinal, const uint64_t* d_ea,
             const uint32_t* d_count,
             const cf_scale_work* work, double scale, uint64_t* d_bad, void* stream) {
  if (!c || !shape || !work) return fail(CF_E_INVALID, "null argument");
  if (elem != 4 && elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  if (!work->parts || (work->big_count && !work->tile_base) || (work->group_end > work->group_begin && !work->groups))
    return fail(CF_E_INVALID, "incomplete work list");
  CfDevice g(c);
  return launch_scale(c, elem, mode, static_cast<const uint8_t*>(image), *shape, d_root, d_level, d_ordinal, d_ea,
                      d_count, *work, scale, d_bad, pick(c, stream));
}

int cf_marshal_transfer_and_attach(cf_ctx* c, const void* host_arena, uint64_t total, void* image,
                                   const uint64_t* h_sites, uint64_t nsites, uint64_t chunk_bytes,
                                   uint64_t* bad_site) {
  if (!c || !host_arena || !image || (nsites && !h_sites)) return fail(CF_E_INVALID, "null argument");
  if (total == 0) return fail(CF_E_INVALID, "empty arena");
  CfDevice g(c);
  if (bad_site) *bad_site = NO_BAD;
  DevBuf d_sites(c);
  CF_TRY(d_sites.alloc(nsites * 8));
  const uint64_t base = reinterpret_cast<uint64_t>(host_arena);
  const uint64_t dimg = reinterpret_cast<uint64_t>(image);
  // relocation table + error word first, on the compute stream
  if (nsites) CF_CUDA(cudaMemcpyAsync(d_sites.p, h_sites, nsites * 8, cudaMemcpyHostToDevice, c->compute));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, c->compute));
  std::vector<uint64_t> b = chunk_bounds(total, chunk_bytes, h_sites, nsites);
  const size_t nch = b.size() - 1;
  EventSet ev;
  CF_TRY(ev.make(nch + 1));
  CF_CUDA(cudaEventRecord(ev.ev[nch], c->compute));
  for (size_t i = 0; i < nch; ++i) {
    cudaStream_t s = c->h2d[i % c->h2d.size()];
    if (i < c->h2d.size()) CF_CUDA(cudaStreamWaitEvent(s, ev.ev[nch], 0));
    CF_CUDA(copy_host_aligned(static_cast<uint8_t*>(image) + b[i], static_cast<const uint8_t*>(host_arena) + b[i],
                            b[i + 1] - b[i], cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaEventRecord(ev.ev[i], s));
    // sites whose field lies in this chunk are relocated as soon as it lands
    const uint64_t s0 = uint64_t(std::lower_bound(h_sites, h_sites + nsites, b[i]) - h_sites);
    const uint64_t s1 = uint64_t(std::lower_bound(h_sites, h_sites + nsites, b[i + 1]) - h_sites);
    CF_CUDA(cudaStreamWaitEvent(c->compute, ev.ev[i], 0));
    CF_TRY(launch_relocate(c, static_cast<uint8_t*>(image), total, d_sites.as<uint64_t>() + s0, s1 - s0, base,
                           dimg, c->d_bad, c->compute));
  }
  uint64_t bad = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, c->compute, &bad));
  if (bad != NO_BAD) {
    // the device flags chunk-relative indices; the host arena is untouched, so report the
    // first offending field in table order (memory.py:319-321 raises on the first one)
    const uint8_t* h = static_cast<const uint8_t*>(host_arena);
    for (uint64_t i = 0; i < nsites; ++i) {
      uint64_t v;
      memcpy(&v, h + h_sites[i], 8);
      if (v - base >= total) {
        if (bad_site) *bad_site = i;
        return fail(CF_E_OUTSIDE_ARENA, "pointer field at arena offset %llu targets 0x%llx outside the arena",
                    (unsigned long long)h_sites[i], (unsigned long long)v);
      }
    }
    return fail(CF_E_OUTSIDE_ARENA, "relocation kernel reported a field outside the arena");
  }
  return CF_OK;
}

int cf_demarshal(cf_ctx* c, void* host_arena, uint64_t total, void* image, const uint64_t* h_sites,
                 uint64_t nsites, uint64_t chunk_bytes, uint64_t* bad_site) {
  if (!c || !host_arena || !image || (nsites && !h_sites)) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  if (bad_site) *bad_site = NO_BAD;
  DevBuf d_sites(c);
  CF_TRY(d_sites.alloc(nsites * 8));
  const uint64_t base = reinterpret_cast<uint64_t>(host_arena);
  const uint64_t dimg = reinterpret_cast<uint64_t>(image);
  if (nsites) CF_CUDA(cudaMemcpyAsync(d_sites.p, h_sites, nsites * 8, cudaMemcpyHostToDevice, c->compute));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, c->compute));
  // detach on the device (memory.py:337-344), then copy the image home
  CF_TRY(launch_relocate(c, static_cast<uint8_t*>(image), total, d_sites.as<uint64_t>(), nsites, dimg, base,
                         c->d_bad, c->compute));
  EventSet ev;
  CF_TRY(ev.make(1));
  CF_CUDA(cudaEventRecord(ev.ev[0], c->compute));
  CF_CUDA(cudaStreamWaitEvent(c->d2h, ev.ev[0], 0));
  // every field is detached before the first chunk leaves, so chunks need not respect fields
  // and the table may come in any order (the drop-in passes the reference's detach order)
  std::vector<uint64_t> b = chunk_bounds(total, chunk_bytes, nullptr, 0);
  for (size_t i = 0; i + 1 < b.size(); ++i)
    CF_CUDA(copy_host_aligned(static_cast<uint8_t*>(host_arena) + b[i], static_cast<const uint8_t*>(image) + b[i],
                            b[i + 1] - b[i], cudaMemcpyDeviceToHost, c->d2h));
  CF_CUDA(cudaStreamSynchronize(c->d2h));
  uint64_t bad = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, c->compute, &bad));
  if (bad != NO_BAD) {
    if (bad_site) *bad_site = bad;
    return fail(CF_E_OUTSIDE_ARENA, "pointer field at arena offset %llu holds a value outside the device image",
                (unsigned long long)h_sites[bad]);
  }
  return CF_OK;
}

int cf_kernel_scale(cf_ctx* c, int elem, int mode, void* image, const cf_chain_shape* shape,
                    const uint64_t* h_root, const int32_t* h_level, const uint32_t* h_ordinal,
                    const uint64_t* h_count, uint64_t ntargets, double scale, uint64_t* h_ea_out, uint64_t* bad) {
  if (!c || !shape || (ntargets && (!h_level || !h_ordinal || !h_count))) return fail(CF_E_INVALID, "null argument");
  if (elem != 4 && elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  CfDevice g(c);
  if (bad) *bad = NO_BAD;
  if (ntargets == 0) return CF_OK;
  // parts: whole arrays with their planned counts
  ScaleWork sw;
  sw.elem = elem;
  std::vector<uint64_t> tri;
  for (uint64_t t = 0; t < ntargets; ++t)
    if (h_count[t]) tri.insert(tri.end(), {t, 0, h_count[t]});
  cf_scale_work work = sw.append(tri);
  // one device block: level | ordinal | ea | count | roots | work list
  const uint64_t off_ord = ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_ea = off_ord + ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_cnt = off_ea + ntargets * 8;
  const uint64_t off_root = off_cnt + ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_work = off_root + (h_root ? ntargets * 8 : 0);
  DevBuf blk(c);
  CF_TRY(blk.alloc(off_work + work_bytes(sw) + 8));
  uint8_t* d = blk.as<uint8_t>();
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemcpyAsync(d, h_level, ntargets * 4, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemcpyAsync(d + off_ord, h_ordinal, ntargets * 4, cudaMemcpyHostToDevice, s));
  if (h_root) CF_CUDA(cudaMemcpyAsync(d + off_root, h_root, ntargets * 8, cudaMemcpyHostToDevice, s));
  const uint64_t* droot = h_root ? reinterpret_cast<const uint64_t*>(d + off_root) : nullptr;
  CF_TRY(upload_work(sw, d + off_work, s, &work));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  const int32_t* lv = reinterpret_cast<const int32_t*>(d);
  const uint32_t* od = reinterpret_cast<const uint32_t*>(d + off_ord);
  uint64_t* ea = reinterpret_cast<uint64_t*>(d + off_ea);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(d + off_cnt);
  CF_TRY(launch_resolve(c, static_cast<const uint8_t*>(image), *shape, droot, lv, od, ntargets, ea, cnt, c->d_bad, s));
  uint64_t rb = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) {
    if (bad) *bad = rb;
    return fail(CF_E_WILD, "chain walk for target %llu left the device image", (unsigned long long)rb);
  }
  CF_TRY(launch_scale(c, elem, mode, static_cast<const uint8_t*>(image), *shape, droot, lv, od, ea, cnt, work, scale,
                      c->d_bad, s));
  if (h_ea_out) CF_CUDA(cudaMemcpyAsync(h_ea_out, ea, ntargets * 8, cudaMemcpyDeviceToHost, s));
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) {
    if (bad) *bad = rb;
    return fail(CF_E_WILD, "leaf kernel: target %llu count/address mismatch", (unsigned long long)rb);
  }
  return CF_OK;
}

}  // extern "C"

// A planned kernel_scale: the targets' chain keys, counts and leaf-kernel work list uploaded
// once (C4: 1M targets, 24 MB of tables and a 1M-part work list planned on the host), then
// every eager kernel_scale over the same targets only launches resolve + leaf kernel.
struct cf_kernel_plan {
  cf_ctx* ctx = nullptr;
  int elem = 4;
  uint64_t ntargets = 0;
  uint8_t* d = nullptr;
  int32_t* lv = nullptr;
  uint32_t* od = nullptr;
  uint64_t* ea = nullptr;
  uint32_t* cnt = nullptr;
  uint64_t* root = nullptr;
  uint64_t* expect = nullptr;     // cf_kernel_plan_expect: where each chain must end (image offsets)
  uint32_t* cnt_plan = nullptr;   // ... and with which count
  cf_scale_work work{};
};

extern "C" {

int cf_kernel_plan_create(cf_ctx* c, int elem, const uint64_t* h_root, const int32_t* h_level,
                          const uint32_t* h_ordinal, const uint64_t* h_count, uint64_t ntargets, cf_kernel_plan** out) {
  if (!c || !out || (ntargets && (!h_level || !h_ordinal || !h_count))) return fail(CF_E_INVALID, "null argument");
  if (elem != 4 && elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  CfDevice g(c);
  ScaleWork sw;
  sw.elem = elem;
  std::vector<uint64_t> tri;
  tri.reserve(3 * ntargets);
  for (uint64_t t = 0; t < ntargets; ++t)
    if (h_count[t]) tri.insert(tri.end(), {t, 0, h_count[t]});
  cf_kernel_plan* k = new cf_kernel_plan();
  k->ctx = c;
  k->elem = elem;
  k->ntargets = ntargets;
  k->work = sw.append(tri);
  const uint64_t off_ord = ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_ea = off_ord + ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_cnt = off_ea + ntargets * 8;
  const uint64_t off_root = off_cnt + ((ntargets * 4 + 7) / 8) * 8;
  const uint64_t off_work = off_root + (h_root ? ntargets * 8 : 0);
  cudaError_t e = cudaMalloc(&k->d, off_work + work_bytes(sw) + 8);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete k;
    return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA, "kernel plan: %s", cudaGetErrorString(e));
  }
  k->lv = reinterpret_cast<int32_t*>(k->d);
  k->od = reinterpret_cast<uint32_t*>(k->d + off_ord);
  k->ea = reinterpret_cast<uint64_t*>(k->d + off_ea);
  k->cnt = reinterpret_cast<uint32_t*>(k->d + off_cnt);
  k->root = h_root ? reinterpret_cast<uint64_t*>(k->d + off_root) : nullptr;
  cudaStream_t s = c->compute;
  int rc = CF_OK;
  auto up = [&](void* dst, const void* src, uint64_t n) {
    if (rc == CF_OK && n && cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s) != cudaSuccess)
      rc = fail(CF_E_CUDA, "kernel plan upload: %s", cudaGetErrorString(cudaGetLastError()));
  };
  up(k->lv, h_level, ntargets * 4);
  up(k->od, h_ordinal, ntargets * 4);
  if (h_root) up(k->root, h_root, ntargets * 8);
  if (rc == CF_OK) rc = upload_work(sw, k->d + off_work, s, &k->work);
  if (rc == CF_OK && cudaStreamSynchronize(s) != cudaSuccess)   // host tables go out of scope
    rc = fail(CF_E_CUDA, "kernel plan upload: %s", cudaGetErrorString(cudaGetLastError()));
  if (rc != CF_OK) {
    cudaFree(k->d);
    delete k;
    return rc;
  }
  *out = k;
  return CF_OK;
}

int cf_kernel_plan_run(cf_kernel_plan* k, int mode, void* image, const cf_chain_shape* shape, double scale,
                       uint64_t* bad) {
  if (!k || !shape) return fail(CF_E_INVALID, "null argument");
  cf_ctx* c = k->ctx;
  CfDevice g(c);
  if (bad) *bad = NO_BAD;
  if (k->ntargets == 0) return CF_OK;
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  CF_TRY(launch_resolve(c, static_cast<const uint8_t*>(image), *shape, k->root, k->lv, k->od, k->ntargets, k->ea, k->cnt,
                        c->d_bad, s));
  uint64_t rb = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) {
    if (bad) *bad = rb;
    return fail(CF_E_WILD, "chain walk for target %llu left the device image", (unsigned long long)rb);
  }
  CF_TRY(launch_scale(c, k->elem, mode, static_cast<const uint8_t*>(image), *shape, k->root, k->lv, k->od, k->ea, k->cnt,
                      k->work, scale, c->d_bad, s));
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) {
    if (bad) *bad = rb;
    return fail(CF_E_WILD, "leaf kernel: target %llu count/address mismatch", (unsigned long long)rb);
  }
  return CF_OK;
}

int cf_kernel_plan_expect(cf_kernel_plan* k, const uint64_t* h_expect_off, const uint64_t* h_count) {
  if (!k || (k->ntargets && (!h_expect_off || !h_count))) return fail(CF_E_INVALID, "null argument");
  CfDevice g(k->ctx);
  if (k->ntargets == 0) return CF_OK;
  std::vector<uint32_t> c32(k->ntargets);
  for (uint64_t t = 0; t < k->ntargets; ++t) {
    if (h_count[t] >> 32) return fail(CF_E_INVALID, "count does not fit the u32 nA field");
    c32[t] = uint32_t(h_count[t]);
  }
  if (!k->expect) {
    cudaError_t e = cudaMalloc(&k->expect, k->ntargets * 12);
    if (e != cudaSuccess) {
      cudaGetLastError();
      k->expect = nullptr;
      return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA, "kernel plan expect: %s", cudaGetErrorString(e));
    }
    k->cnt_plan = reinterpret_cast<uint32_t*>(k->expect + k->ntargets);
  }
  CF_CUDA(cudaMemcpyAsync(k->expect, h_expect_off, k->ntargets * 8, cudaMemcpyHostToDevice, k->ctx->compute));
  CF_CUDA(cudaMemcpyAsync(k->cnt_plan, c32.data(), k->ntargets * 4, cudaMemcpyHostToDevice, k->ctx->compute));
  CF_CUDA(cudaStreamSynchronize(k->ctx->compute));
  return CF_OK;
}

int cf_kernel_plan_resolve(cf_kernel_plan* k, void* image, const cf_chain_shape* shape, uint64_t* h_ea,
                           uint32_t* h_count, uint64_t* bad) {
  if (!k || !shape || (k->ntargets && (!h_ea || !h_count) && !k->expect)) return fail(CF_E_INVALID, "null argument");
  cf_ctx* c = k->ctx;
  CfDevice g(c);
  if (bad) *bad = NO_BAD;
  if (k->ntargets == 0) return CF_OK;
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  CF_TRY(launch_resolve(c, static_cast<const uint8_t*>(image), *shape, k->root, k->lv, k->od, k->ntargets, k->ea, k->cnt,
                        c->d_bad, s));
  if (h_ea) CF_CUDA(cudaMemcpyAsync(h_ea, k->ea, k->ntargets * 8, cudaMemcpyDeviceToHost, s));
  if (h_count) CF_CUDA(cudaMemcpyAsync(h_count, k->cnt, k->ntargets * 4, cudaMemcpyDeviceToHost, s));
  uint64_t rb = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) {
    if (bad) *bad = rb;
    return fail(CF_E_WILD, "chain walk for target %llu left the device image", (unsigned long long)rb);
  }
  if (!h_ea && k->expect) {   // check on the device: every chain ends where it must
    CF_TRY(launch_check_resolved(c, k->ea, k->cnt, k->expect, k->cnt_plan, reinterpret_cast<uint64_t>(image),
                                 k->ntargets, c->d_bad, s));
    CF_TRY(read_bad(c, c->d_bad, s, &rb));
    if (rb != NO_BAD) {
      if (bad) *bad = rb;
      return fail(CF_E_WILD, "chain of target %llu does not end on its array's device copy", (unsigned long long)rb);
    }
  }
  return CF_OK;
}

int cf_kernel_plan_free(cf_kernel_plan* k) {
  if (!k) return CF_OK;
  CfDevice g(k->ctx);
  cudaStreamSynchronize(k->ctx->compute);
  cudaFree(k->d);
  if (k->expect) cudaFree(k->expect);
  delete k;
  return CF_OK;
}

int cf_scale_resolved(cf_ctx* c, int elem, const uint64_t* h_ea, const uint64_t* h_count, uint64_t n,
                      double scale) {
  if (!c || (n && (!h_ea || !h_count))) return fail(CF_E_INVALID, "null argument");
  if (elem != 4 && elem != 8) return fail(CF_E_INVALID, "elem must be 4 or 8");
  CfDevice g(c);
  std::vector<uint32_t> cnt(n);
  ScaleWork sw;
  sw.elem = elem;
  std::vector<uint64_t> tri;
  for (uint64_t t = 0; t < n; ++t) {
    if (h_count[t] >> 32) return fail(CF_E_INVALID, "count does not fit the u32 nA field");
    cnt[t] = uint32_t(h_count[t]);
    if (h_count[t] == 0 || h_ea[t] == 0) continue;
    tri.insert(tri.end(), {t, 0, h_count[t]});
  }
  cf_scale_work work = sw.append(tri);
  if (sw.nparts() == 0) return CF_OK;
  const uint64_t off_cnt = n * 8, off_work = off_cnt + ((n * 4 + 7) / 8) * 8;
  DevBuf blk(c);
  CF_TRY(blk.alloc(off_work + work_bytes(sw) + 8));
  uint8_t* d = blk.as<uint8_t>();
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemcpyAsync(d, h_ea, n * 8, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemcpyAsync(d + off_cnt, cnt.data(), n * 4, cudaMemcpyHostToDevice, s));
  CF_TRY(upload_work(sw, d + off_work, s, &work));
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  cf_chain_shape sh;
  memset(&sh, 0, sizeof sh);
  CF_TRY(launch_scale(c, elem, CF_MODE_RESOLVED, nullptr, sh, nullptr, nullptr, nullptr, reinterpret_cast<const uint64_t*>(d),
                      reinterpret_cast<const uint32_t*>(d + off_cnt), work, scale, c->d_bad, s));
  uint64_t rb = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, s, &rb));
  if (rb != NO_BAD) return fail(CF_E_WILD, "leaf kernel: buffer %llu rejected", (unsigned long long)rb);
  return CF_OK;
}

int cf_host_write_words(const uint64_t* h_addrs, const uint64_t* h_values, uint64_t n) {
  if (n && (!h_addrs || !h_values)) return fail(CF_E_INVALID, "null argument");
#pragma omp parallel for schedule(static) if (n > (1u << 16))
  for (int64_t i = 0; i < int64_t(n); ++i) memcpy(reinterpret_cast<void*>(h_addrs[i]), &h_values[i], 8);
  return CF_OK;
}

int cf_arena_check_sites(const void* host_arena, uint64_t total, const uint64_t* h_sites, uint64_t nsites,
                         uint64_t ptr_base, uint64_t* bad_index) {
  if (!host_arena || (nsites && !h_sites)) return fail(CF_E_INVALID, "null argument");
  if (bad_index) *bad_index = NO_BAD;
  const uint8_t* h = static_cast<const uint8_t*>(host_arena);
  uint64_t first = NO_BAD;   // smallest offending index in table order
#pragma omp parallel for schedule(static) reduction(min : first) if (nsites > (1u << 16))
  for (int64_t i = 0; i < int64_t(nsites); ++i) {
    const uint64_t s = h_sites[i];
    uint64_t v;
    if (s > total || total - s < 8) { first = std::min<uint64_t>(first, uint64_t(i)); continue; }
    memcpy(&v, h + s, 8);
    if (v - ptr_base >= total) first = std::min<uint64_t>(first, uint64_t(i));
  }
  if (first == NO_BAD) return CF_OK;
  if (bad_index) *bad_index = first;
  uint64_t v = 0;
  if (h_sites[first] <= total && total - h_sites[first] >= 8) memcpy(&v, h + h_sites[first], 8);
  return fail(CF_E_OUTSIDE_ARENA, "pointer field at arena offset %llu targets 0x%llx outside the arena",
              (unsigned long long)h_sites[first], (unsigned long long)v);
}

int cf_checksum_ranges(cf_ctx* c, const uint64_t* h_addr, const uint64_t* h_bytes, uint64_t n, uint64_t* h_out) {
  if (!c || (n && (!h_addr || !h_bytes || !h_out))) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  if (n == 0) return CF_OK;
  constexpr uint64_t TW = 16384;   // words per tile (k_checksum)
  std::vector<uint64_t> words(n), tile_lo(n);
  uint64_t ntiles = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if ((h_addr[i] | h_bytes[i]) & 3) return fail(CF_E_INVALID, "range %llu is not 4-byte aligned", (unsigned long long)i);
    words[i] = h_bytes[i] / 4;
    tile_lo[i] = ntiles;
    ntiles += (words[i] + TW - 1) / TW;
  }
  DevBuf blk(c);
  CF_TRY(blk.alloc(32 * n));
  uint64_t* d = blk.as<uint64_t>();
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemcpyAsync(d, h_addr, 8 * n, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemcpyAsync(d + n, words.data(), 8 * n, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemcpyAsync(d + 2 * n, tile_lo.data(), 8 * n, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemsetAsync(d + 3 * n, 0, 8 * n, s));
  CF_TRY(launch_checksum(c, d, d + n, d + 2 * n, n, ntiles, d + 3 * n, s));
  CF_CUDA(cudaMemcpyAsync(h_out, d + 3 * n, 8 * n, cudaMemcpyDeviceToHost, s));
  CF_CUDA(cudaStreamSynchronize(s));
  return CF_OK;
}

int cf_copy_objects(cf_ctx* c, void* const* dsts, const void* const* srcs, const uint64_t* sizes, uint64_t count) {
  if (!c || (count && (!dsts || !srcs || !sizes))) return fail(CF_E_INVALID, "null argument");
  if (count == 0) return CF_OK;
  CfDevice g(c);
  constexpr uint64_t SMALL = 64 << 10;
  // zero-copy needs both ends addressable by the SMs (device, managed or mapped pinned memory)
  auto dev_ok = [](const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type != cudaMemoryTypeUnregistered && a.devicePointer == p;
  };
  // fast path: every object small and both ends SM-addressable -- the caller's own address and
  // size arrays are the copy list (no per-object host work beyond one scan)
  {
    bool all_small = true;
    for (uint64_t i = 0; i < count && all_small; ++i) all_small = sizes[i] < SMALL;
    if (all_small && dev_ok(srcs[0]) && dev_ok(dsts[0])) {
      cudaStream_t s = c->compute;
      DevBuf blk(c);
      CF_TRY(blk.alloc(24 * count));
      uint64_t* d = blk.as<uint64_t>();
      CF_CUDA(cudaMemcpyAsync(d, srcs, 8 * count, cudaMemcpyHostToDevice, s));
      CF_CUDA(cudaMemcpyAsync(d + count, dsts, 8 * count, cudaMemcpyHostToDevice, s));
      CF_CUDA(cudaMemcpyAsync(d + 2 * count, sizes, 8 * count, cudaMemcpyHostToDevice, s));
      CF_TRY(launch_copy_list(c, d, d + count, d + 2 * count, count, s));
      CF_CUDA(cudaStreamSynchronize(s));
      return CF_OK;
    }
  }
  std::vector<uint64_t> zs, zd, zb;
  std::vector<void*> bd;
  std::vector<const void*> bs;
  std::vector<uint64_t> bz;
  zs.reserve(count);
  zd.reserve(count);
  zb.reserve(count);
  bool zc = true;
  bool checked = false;
  for (uint64_t i = 0; i < count; ++i) {
    if (sizes[i] < SMALL && zc) {
      if (!checked) { zc = dev_ok(srcs[i]) && dev_ok(dsts[i]); checked = true; }
      if (zc) {
        zs.push_back(reinterpret_cast<uint64_t>(srcs[i]));
        zd.push_back(reinterpret_cast<uint64_t>(dsts[i]));
        zb.push_back(sizes[i]);
        continue;
      }
    }
    bd.push_back(dsts[i]);
    bs.push_back(srcs[i]);
    bz.push_back(sizes[i]);
  }
  cudaStream_t s = c->compute;
  if (!bz.empty()) CF_TRY(cf_memcpy_batch(c, bd.data(), bs.data(), bz.data(), bz.size(), s));
  if (!zb.empty()) {
    const uint64_t m = zb.size();
    DevBuf blk(c);
    CF_TRY(blk.alloc(24 * m));
    uint64_t* d = blk.as<uint64_t>();
    CF_CUDA(cudaMemcpyAsync(d, zs.data(), 8 * m, cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaMemcpyAsync(d + m, zd.data(), 8 * m, cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaMemcpyAsync(d + 2 * m, zb.data(), 8 * m, cudaMemcpyHostToDevice, s));
    CF_TRY(launch_copy_list(c, d, d + m, d + 2 * m, m, s));
  }
  CF_CUDA(cudaStreamSynchronize(s));
  return CF_OK;
}

int cf_sm_copy(cf_ctx* c, void* dst, const void* src, uint64_t bytes, unsigned ctas, void* stream) {
  if (!c || !dst || !src) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  return launch_sm_copy(c, dst, src, bytes, ctas, pick(c, stream));
}

int cf_debug_info(cf_ctx* c, uint64_t* out8, int reset) {
  if (!c || !out8) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  return debug_info(out8, reset);
}

int cf_naive_fixup_host(cf_ctx* c, const uint64_t* h_field_host, const uint64_t* h_target_host, uint64_t nsites,
                        const uint64_t* h_map_host_base, const uint64_t* h_map_size, const uint64_t* h_map_dev_base,
                        uint64_t nmap, uint64_t* bad_site) {
  if (!c || (nsites && (!h_field_host || !h_target_host)) || (nmap && (!h_map_host_base || !h_map_size || !h_map_dev_base)))
    return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  if (bad_site) *bad_site = NO_BAD;
  if (nsites == 0) return CF_OK;
  DevBuf blk(c);
  CF_TRY(blk.alloc(8 * (2 * nsites + 3 * nmap)));
  uint64_t* d = blk.as<uint64_t>();
  cudaStream_t s = c->compute;
  CF_CUDA(cudaMemcpyAsync(d, h_field_host, 8 * nsites, cudaMemcpyHostToDevice, s));
  CF_CUDA(cudaMemcpyAsync(d + nsites, h_target_host, 8 * nsites, cudaMemcpyHostToDevice, s));
  uint64_t* m = d + 2 * nsites;
  if (nmap) {
    CF_CUDA(cudaMemcpyAsync(m, h_map_host_base, 8 * nmap, cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaMemcpyAsync(m + nmap, h_map_size, 8 * nmap, cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaMemcpyAsync(m + 2 * nmap, h_map_dev_base, 8 * nmap, cudaMemcpyHostToDevice, s));
  }
  CF_CUDA(cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  CF_TRY(launch_naive_fixup(c, d, d + nsites, nsites, m, m + nmap, m + 2 * nmap, nmap, c->d_bad, s));
  uint64_t bad = NO_BAD;
  CF_TRY(read_bad(c, c->d_bad, s, &bad));
  if (bad != NO_BAD) {
    if (bad_site) *bad_site = bad;
    return fail(CF_E_WILD, "fixup target 0x%llx was never copied to the device", (unsigned long long)h_target_host[bad]);
  }
  return CF_OK;
}

int cf_naive_fixup(cf_ctx* c, const uint64_t* d_field_host, const uint64_t* d_target_host, uint64_t nsites,
                   const uint64_t* d_map_host_base, const uint64_t* d_map_size, const uint64_t* d_map_dev_base,
                   uint64_t nmap, uint64_t* d_bad, void* stream) {
  if (!c) return fail(CF_E_INVALID, "null ctx");
  CfDevice g(c);
  return launch_naive_fixup(c, d_field_host, d_target_host, nsites, d_map_host_base, d_map_size, d_map_dev_base,
                            nmap, d_bad, pick(c, stream));
}

}  // extern "C"
