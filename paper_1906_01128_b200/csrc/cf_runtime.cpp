// Runtime plumbing behind the C ABI: errors, per-GPU context, host/device memory, copies.
// Replaces the simulated Machine/MemorySpace storage of the reference (memory.py:101-303) with
// real pinned host memory, HBM and CUDA streams.
#include "cf_internal.h"

#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <fstream>
#include <sstream>
#include <string>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace cf {
namespace {
thread_local char g_err[1024] = "";
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
void clear_error() { g_err[0] = 0; }
const char* last_error() { return g_err; }

}  // namespace cf

using namespace cf;

extern "C" {

int cf_abi_version(void) { return CF_ABI_VERSION; }
const char* cf_last_error(void) { return cf::last_error(); }

int cf_device_count(int* count) {
  if (!count) return fail(CF_E_INVALID, "null count");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return CF_OK;
  }
  *count = n;
  return CF_OK;
}

int cf_device_numa_node(int device, int* node) {
  if (!node) return fail(CF_E_INVALID, "null node");
  *node = -1;
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return fail(CF_E_NODEVICE, "no PCI bus id for device %d", device);
  }
  std::string id(bus);
  for (auto& ch : id) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  // sysfs uses a 4-hex-digit domain; the runtime may print 8
  if (id.size() > 12 && id.find(':') == 8) id = id.substr(4);
  std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
  int n = -1;
  if (f >> n) *node = n;
  return CF_OK;
}

int cf_bind_numa_node(int node) {
  // Pin the calling thread to the node's CPUs and prefer its memory, so pinned arenas allocated
  // and first-touched by this thread sit next to the GPU's host link (no libnuma in the image:
  // sysfs cpulist + raw set_mempolicy).
  if (node < 0) {   // back to the default memory policy (the caller restores its CPU mask)
    syscall(SYS_set_mempolicy, 0 /* MPOL_DEFAULT */, nullptr, 0);
    return CF_OK;
  }
  std::ifstream f("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
  std::string list;
  if (!(f >> list)) return fail(CF_E_INVALID, "no cpulist for NUMA node %d", node);
  cpu_set_t set;
  CPU_ZERO(&set);
  std::stringstream ss(list);
  std::string part;
  int ncpu = 0;
  while (std::getline(ss, part, ',')) {
    const size_t dash = part.find('-');
    const int lo = std::stoi(part.substr(0, dash));
    const int hi = dash == std::string::npos ? lo : std::stoi(part.substr(dash + 1));
    for (int c = lo; c <= hi && c < CPU_SETSIZE; ++c, ++ncpu) CPU_SET(c, &set);
  }
  if (ncpu == 0) return fail(CF_E_INVALID, "empty cpulist for NUMA node %d", node);
  if (sched_setaffinity(0, sizeof set, &set) != 0) return fail(CF_E_INVALID, "sched_setaffinity failed");
  unsigned long mask[16] = {0};
  if (node < int(sizeof mask * 8)) {
    mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
    constexpr int MPOL_PREFERRED_ = 1;
    syscall(SYS_set_mempolicy, MPOL_PREFERRED_, mask, sizeof mask * 8);   // best effort
  }
  return CF_OK;
}

int cf_ctx_create(int device, int nstreams, cf_ctx** out) {
  if (!out || nstreams < 1 || nstreams > 16) return fail(CF_E_INVALID, "bad ctx arguments");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(CF_E_NODEVICE, "no CUDA device visible: the chainforge_b200 path requires a GPU");
  }
  if (device < 0 || device >= n) return fail(CF_E_INVALID, "device %d out of range (%d)", device, n);
  CF_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CF_CUDA(cudaGetDeviceProperties(&prop, device));
  cf_ctx* c = new cf_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  CF_CUDA(cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking));
  CF_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  c->h2d.resize(nstreams);
  for (auto& s : c->h2d) CF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CF_CUDA(cudaMalloc(&c->d_bad, 64));
  CF_CUDA(cudaHostAlloc(&c->h_bad, 64, cudaHostAllocPortable));
  *out = c;
  return CF_OK;
}

int cf_ctx_destroy(cf_ctx* c) {
  if (!c) return CF_OK;
  CfDevice g(c);
  cudaDeviceSynchronize();
  cudaStreamDestroy(c->compute);
  cudaStreamDestroy(c->d2h);
  for (auto s : c->h2d) cudaStreamDestroy(s);
  cudaFree(c->d_bad);
  cudaFreeHost(c->h_bad);
  if (c->scratch) cudaFree(c->scratch);
  delete c;
  return CF_OK;
}

int cf_ctx_sync(cf_ctx* c) {
  if (!c) return fail(CF_E_INVALID, "null ctx");
  CfDevice g(c);
  CF_CUDA(cudaDeviceSynchronize());
  return CF_OK;
}

void* cf_ctx_stream(cf_ctx* c) { return c ? (void*)c->compute : nullptr; }

}  // extern "C"

// Device timer over the context's compute stream: every operation of the library forks from and
// joins back into that stream, so an event pair on it brackets all the device work in between.
struct cf_timer {
  cf_ctx* c = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
};

extern "C" {

int cf_timer_create(cf_ctx* c, cf_timer** out) {
  if (!c || !out) return fail(CF_E_INVALID, "null argument");
  CfDevice g(c);
  cf_timer* t = new cf_timer();
  t->c = c;
  if (cudaEventCreate(&t->a) != cudaSuccess || cudaEventCreate(&t->b) != cudaSuccess) {
    cudaGetLastError();
    if (t->a) cudaEventDestroy(t->a);
    delete t;
    return fail(CF_E_CUDA, "timer events");
  }
  *out = t;
  return CF_OK;
}

int cf_timer_start(cf_timer* t) {
  if (!t) return fail(CF_E_INVALID, "null timer");
  CfDevice g(t->c);
  CF_CUDA(cudaEventRecord(t->a, t->c->compute));
  return CF_OK;
}

int cf_timer_stop(cf_timer* t, float* ms) {
  if (!t || !ms) return fail(CF_E_INVALID, "null argument");
  CfDevice g(t->c);
  CF_CUDA(cudaEventRecord(t->b, t->c->compute));
  CF_CUDA(cudaEventSynchronize(t->b));
  CF_CUDA(cudaEventElapsedTime(ms, t->a, t->b));
  return CF_OK;
}

int cf_timer_free(cf_timer* t) {
  if (!t) return CF_OK;
  CfDevice g(t->c);
  cudaEventDestroy(t->a);
  cudaEventDestroy(t->b);
  delete t;
  return CF_OK;
}
uint64_t cf_ctx_launches(cf_ctx* c) { return c ? c->launches.load() : 0; }
int cf_ctx_sm_count(cf_ctx* c) { return c ? c->sm_count : 0; }

int cf_host_alloc(uint64_t bytes, int kind, void** out) {
  if (!out) return fail(CF_E_INVALID, "null out");
  if (bytes == 0) return fail(CF_E_INVALID, "allocation size must be positive");
  void* p = nullptr;
  if (kind == CF_MEM_PAGEABLE) {
    // page-aligned, zero-filled (anonymous mmap)
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return fail(CF_E_OOM, "host mmap of %llu bytes failed", (unsigned long long)bytes);
  } else if (kind == CF_MEM_PINNED) {
    // mapped: under UVA the same pointer is usable by kernels (zero-copy node transfers)
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA,
                  "cudaHostAlloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    }
    // zero-fill in parallel: the reference's storage is zero-initialised (memory.py:135)
    const uint64_t CH = 8ull << 20;
    int64_t nch = (int64_t)((bytes + CH - 1) / CH);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nch; ++i) {
      uint64_t o = uint64_t(i) * CH;
      memset((char*)p + o, 0, bytes - o < CH ? bytes - o : CH);
    }
  } else if (kind == CF_MEM_MANAGED) {
    cudaError_t e = cudaMallocManaged(&p, bytes, cudaMemAttachGlobal);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA,
                  "cudaMallocManaged(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    }
    memset(p, 0, bytes);
  } else {
    return fail(CF_E_INVALID, "unknown memory kind %d", kind);
  }
  *out = p;
  return CF_OK;
}

int cf_host_free(void* p, int kind) {
  if (!p) return CF_OK;
  if (kind == CF_MEM_PAGEABLE) return fail(CF_E_INVALID, "pageable blocks are freed by size: use cf_host_free_sized");
  if (kind == CF_MEM_PINNED) CF_CUDA(cudaFreeHost(p));
  else if (kind == CF_MEM_MANAGED) CF_CUDA(cudaFree(p));
  else return fail(CF_E_INVALID, "unknown memory kind %d", kind);
  return CF_OK;
}

int cf_host_free_sized(void* p, uint64_t bytes, int kind) {
  if (!p) return CF_OK;
  if (kind == CF_MEM_PAGEABLE) {
    munmap(p, bytes);
    return CF_OK;
  }
  return cf_host_free(p, kind);
}

int cf_dev_alloc(cf_ctx* c, uint64_t bytes, void** out) {
  if (!c || !out) return fail(CF_E_INVALID, "null argument");
  if (bytes == 0) return fail(CF_E_INVALID, "allocation size must be positive");
  CfDevice g(c);
  cudaError_t e = cudaMalloc(out, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA, "cudaMalloc(%llu): %s",
                (unsigned long long)bytes, cudaGetErrorString(e));
  }
  return CF_OK;
}

int cf_dev_free(cf_ctx* c, void* p) {
  if (!p) return CF_OK;
  CfDevice g(c);
  CF_CUDA(cudaFree(p));
  return CF_OK;
}

int cf_memcpy(cf_ctx* c, void* dst, const void* src, uint64_t bytes) {
  if (bytes == 0) return CF_OK;
  if (!c) return fail(CF_E_INVALID, "null ctx");
  CfDevice g(c);
  // ordered after everything already on the compute stream (the context's streams are
  // non-blocking, so the legacy default stream would not order against them), then waited for
  CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->compute));
  CF_CUDA(cudaStreamSynchronize(c->compute));
  return CF_OK;
}

int cf_memcpy_async(cf_ctx* c, void* dst, const void* src, uint64_t bytes, void* stream) {
  if (!c) return fail(CF_E_INVALID, "null ctx");
  if (bytes == 0) return CF_OK;
  CfDevice g(c);
  CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream ? (cudaStream_t)stream : c->compute));
  return CF_OK;
}

int cf_l2_evict(cf_ctx* c, const void* buf, uint64_t bytes) {
  if (!c || (bytes && !buf)) return fail(CF_E_INVALID, "bad arguments");
  CfDevice g(c);
  CF_TRY(launch_evict_read(c, buf, bytes, c->compute));
  CF_CUDA(cudaStreamSynchronize(c->compute));
  return CF_OK;
}

int cf_memset(cf_ctx* c, void* dst, int value, uint64_t bytes) {
  if (!c) return fail(CF_E_INVALID, "null ctx");
  CfDevice g(c);
  CF_CUDA(cudaMemsetAsync(dst, value, bytes, c->compute));
  CF_CUDA(cudaStreamSynchronize(c->compute));
  return CF_OK;
}

int cf_memcpy_batch(cf_ctx* c, void* const* dsts, const void* const* srcs, const uint64_t* sizes,
                    uint64_t count, void* stream) {
  if (!c) return fail(CF_E_INVALID, "null ctx");
  if (count == 0) return CF_OK;
  CfDevice g(c);
  cudaStream_t s = stream ? (cudaStream_t)stream : c->compute;
  // one cudaMemcpyAsync per object (naive_deep_copy, memory.py:358-361), all on one non-blocking
  // stream; the driver's batched submission call is not used (it is closed on the GPU pool)
  for (uint64_t i = 0; i < count; ++i)
    CF_CUDA(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, s));
  return CF_OK;
}

int cf_uvm_prefetch(cf_ctx* c, const void* p, uint64_t bytes, int dst_device, void* stream) {
  if (!c || !p) return fail(CF_E_INVALID, "null argument");
  if (bytes == 0) return CF_OK;
  CfDevice g(c);
  cudaStream_t s = stream ? (cudaStream_t)stream : c->compute;
#if CUDART_VERSION >= 12080
  cudaMemLocation loc;
  loc.type = dst_device < 0 ? cudaMemLocationTypeHost : cudaMemLocationTypeDevice;
  loc.id = dst_device < 0 ? 0 : c->device;
  CF_CUDA(cudaMemPrefetchAsync_v2(p, bytes, loc, 0, s));
#else
  CF_CUDA(cudaMemPrefetchAsync(p, bytes, dst_device < 0 ? cudaCpuDeviceId : c->device, s));
#endif
  return CF_OK;
}

int cf_uvm_advise(cf_ctx* c, const void* p, uint64_t bytes, int advice) {
  if (!c || !p) return fail(CF_E_INVALID, "null argument");
  const bool unset = (advice & CF_UVM_UNSET) != 0;
  advice &= ~CF_UVM_UNSET;
  if (advice == CF_UVM_ADVISE_NONE || bytes == 0) return CF_OK;
  if (advice < CF_UVM_PREFERRED_DEVICE || advice > CF_UVM_READ_MOSTLY) return fail(CF_E_INVALID, "unknown advice %d", advice);
  CfDevice g(c);
  cudaMemoryAdvise a = advice == CF_UVM_PREFERRED_DEVICE
                           ? (unset ? cudaMemAdviseUnsetPreferredLocation : cudaMemAdviseSetPreferredLocation)
                       : advice == CF_UVM_ACCESSED_BY ? (unset ? cudaMemAdviseUnsetAccessedBy : cudaMemAdviseSetAccessedBy)
                                                      : (unset ? cudaMemAdviseUnsetReadMostly : cudaMemAdviseSetReadMostly);
#if CUDART_VERSION >= 12080
  cudaMemLocation loc;
  loc.type = cudaMemLocationTypeDevice;
  loc.id = c->device;
  CF_CUDA(cudaMemAdvise_v2(p, bytes, a, loc));
#else
  CF_CUDA(cudaMemAdvise(p, bytes, a, c->device));
#endif
  return CF_OK;
}

}  // extern "C"

// Independent host-link roofline probe: plain cudaMemcpyAsync between fresh
// pinned host buffers and device buffers -- no chunking, no window -- so the e2e fraction is not
// measured against a copy pipeline shaped like the one it grades.  Each sample is `iters`
// back-to-back copies of `bytes` (H2D alone, D2H alone, or H2D || D2H on two streams); the best
// of `reps` samples is reported as GB/s of bytes moved (both directions summed for bidir).
extern "C" int cf_link_probe(cf_ctx* c, uint64_t bytes, int iters, int reps, double* h2d_gbs, double* d2h_gbs,
                             double* bidir_gbs) {
  if (!c || bytes == 0 || iters < 1 || reps < 1) return fail(CF_E_INVALID, "bad arguments");
  CfDevice g(c);
  void *h_src = nullptr, *h_dst = nullptr, *d_a = nullptr, *d_b = nullptr;
  cudaStream_t s1 = nullptr, s2 = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, ej = nullptr;
  auto cleanup = [&]() {
    if (h_src) cudaFreeHost(h_src);
    if (h_dst) cudaFreeHost(h_dst);
    if (d_a) cudaFree(d_a);
    if (d_b) cudaFree(d_b);
    for (auto s : {s1, s2}) if (s) cudaStreamDestroy(s);
    for (auto e : {e0, e1, ej}) if (e) cudaEventDestroy(e);
  };
  cudaError_t ce = cudaHostAlloc(&h_src, bytes, cudaHostAllocPortable);
  if (ce == cudaSuccess) ce = cudaHostAlloc(&h_dst, bytes, cudaHostAllocPortable);
  if (ce == cudaSuccess) ce = cudaMalloc(&d_a, bytes);
  if (ce == cudaSuccess) ce = cudaMalloc(&d_b, bytes);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaEventCreate(&e0);
  if (ce == cudaSuccess) ce = cudaEventCreate(&e1);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ej, cudaEventDisableTiming);
  if (ce != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    return fail(ce == cudaErrorMemoryAllocation ? CF_E_OOM : CF_E_CUDA, "link probe setup: %s", cudaGetErrorString(ce));
  }
  memset(h_src, 0x5A, bytes);   // touch every page once before timing
  memset(h_dst, 0xA5, bytes);
  double out[3] = {0, 0, 0};
  for (int mode = 0; mode < 3 && ce == cudaSuccess; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < reps + 1 && ce == cudaSuccess; ++r) {   // sample 0 is a warm-up
      ce = cudaEventRecord(e0, s1);
      if (ce == cudaSuccess && mode == 2) ce = cudaStreamWaitEvent(s2, e0, 0);
      for (int i = 0; i < iters && ce == cudaSuccess; ++i) {
        if (mode != 1) ce = cudaMemcpyAsync(d_a, h_src, bytes, cudaMemcpyHostToDevice, s1);
        if (ce == cudaSuccess && mode != 0)
          ce = cudaMemcpyAsync(h_dst, d_b, bytes, cudaMemcpyDeviceToHost, mode == 2 ? s2 : s1);
      }
      if (ce == cudaSuccess && mode == 2) ce = cudaEventRecord(ej, s2);
      if (ce == cudaSuccess && mode == 2) ce = cudaStreamWaitEvent(s1, ej, 0);
      if (ce == cudaSuccess) ce = cudaEventRecord(e1, s1);
      if (ce == cudaSuccess) ce = cudaEventSynchronize(e1);
      float ms = 0;
      if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
      if (ce == cudaSuccess && r > 0 && ms < best) best = ms;
    }
    out[mode] = double(mode == 2 ? 2 : 1) * double(bytes) * iters / (double(best) * 1e-3) / 1e9;
  }
  cleanup();
  if (ce != cudaSuccess) return fail(CF_E_CUDA, "link probe: %s", cudaGetErrorString(ce));
  if (h2d_gbs) *h2d_gbs = out[0];
  if (d2h_gbs) *d2h_gbs = out[1];
  if (bidir_gbs) *bidir_gbs = out[2];
  return CF_OK;
}
