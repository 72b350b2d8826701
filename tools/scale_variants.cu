// Design experiment (not product code): streaming leaf-kernel variants on B200 over the C2
// shape (64 arrays x 16 MiB float32 = 1 GiB), timed with CUDA events.  Used to pick the
// k_scale design; results are summarised in profiles/.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Parts { const uint64_t* base; const uint64_t* ea; uint64_t nparts; uint64_t ntiles; };

template <int UNROLL, bool HINT>
__global__ void __launch_bounds__(256) k_tiles(Parts a, float s) {
  constexpr uint64_t TILE = 256ull * UNROLL * 4;  // floats
  for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    uint64_t lo = 0, hi = a.nparts;
    while (hi - lo > 1) { uint64_t mid = (lo + hi) >> 1; if (a.base[mid] <= tile) lo = mid; else hi = mid; }
    float4* p = reinterpret_cast<float4*>(a.ea[lo]) + (tile - a.base[lo]) * (TILE / 4);
    float4 r[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) r[u] = HINT ? __ldcs(p + threadIdx.x + u * 256) : p[threadIdx.x + u * 256];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      float4 v = r[u];
      v.x *= s; v.y *= s; v.z *= s; v.w *= s;
      if (HINT) __stcs(p + threadIdx.x + u * 256, v); else p[threadIdx.x + u * 256] = v;
    }
  }
}

template <int UNROLL>
__global__ void __launch_bounds__(256) k_flat(float4* p, uint64_t nvec, float s) {
  uint64_t stride = uint64_t(gridDim.x) * 256 * UNROLL;
  for (uint64_t i = uint64_t(blockIdx.x) * 256 * UNROLL + threadIdx.x; i < nvec; i += stride) {
    float4 r[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) r[u] = __ldcs(p + i + u * 256);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { float4 v = r[u]; v.x *= s; v.y *= s; v.z *= s; v.w *= s; __stcs(p + i + u * 256, v); }
  }
}

// TMA bulk-copy pipeline: STAGES x CHUNK bytes ring in shared memory per CTA.
template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(256) k_bulk(Parts a, float s, uint64_t tile_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // each CTA owns tiles blockIdx.x + k*gridDim.x; tile = CHUNK bytes
  const uint64_t ntiles = a.ntiles;
  uint64_t my = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) ++my;
  auto tile_ptr = [&](uint64_t tile) -> uint8_t* {
    uint64_t lo = 0, hi = a.nparts;
    while (hi - lo > 1) { uint64_t mid = (lo + hi) >> 1; if (a.base[mid] <= tile) lo = mid; else hi = mid; }
    return reinterpret_cast<uint8_t*>(a.ea[lo]) + (tile - a.base[lo]) * CHUNK;
  };
  auto issue = [&](uint64_t k) {
    const int st = int(k % STAGES);
    uint8_t* g = tile_ptr(blockIdx.x + k * gridDim.x);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[st]);
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + st * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bar), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(g), "r"(CHUNK), "r"(bar) : "memory");
  };
  if (tid == 0) for (uint64_t k = 0; k < my && k < STAGES; ++k) issue(k);
  for (uint64_t k = 0; k < my; ++k) {
    const int st = int(k % STAGES);
    const uint32_t phase = uint32_t((k / STAGES) & 1);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[st]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(bar), "r"(phase));
    float4* b = reinterpret_cast<float4*>(smem + st * CHUNK);
    for (int i = tid; i < CHUNK / 16; i += 256) { float4 v = b[i]; v.x *= s; v.y *= s; v.z *= s; v.w *= s; b[i] = v; }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      uint8_t* g = tile_ptr(blockIdx.x + k * gridDim.x);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"((uint32_t)__cvta_generic_to_shared(smem + st * CHUNK)), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      // before refilling stage st (used again at k+STAGES) the store reading it must be done
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (k + STAGES < my) issue(k + STAGES);
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const uint64_t NARR = 64, PER = 16ull << 20, TOTAL = NARR * PER;
  uint8_t* buf;
  CK(cudaMalloc(&buf, TOTAL + 4096));
  CK(cudaMemset(buf, 0, TOTAL));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto make_parts = [&](uint64_t tile_bytes, uint64_t** d_base, uint64_t** d_ea, uint64_t* ntiles) {
    std::vector<uint64_t> base(NARR), ea(NARR);
    uint64_t t = 0;
    for (uint64_t i = 0; i < NARR; ++i) { base[i] = t; ea[i] = (uint64_t)(buf + i * PER); t += PER / tile_bytes; }
    CK(cudaMalloc(d_base, NARR * 8)); CK(cudaMalloc(d_ea, NARR * 8));
    CK(cudaMemcpy(*d_base, base.data(), NARR * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(*d_ea, ea.data(), NARR * 8, cudaMemcpyHostToDevice));
    *ntiles = t;
  };
  auto timeit = [&](const char* name, auto&& launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9, sum = 0; int n = 10;
    for (int i = 0; i < n; ++i) {
      CK(cudaEventRecord(a)); launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = ms < best ? ms : best; sum += ms;
    }
    CK(cudaGetLastError());
    printf("%-34s best %.4f ms (%.1f GB/s)  mean %.4f ms (%.1f GB/s)\n", name, best, 2.0 * TOTAL / best / 1e6,
           sum / n, 2.0 * TOTAL / (sum / n) / 1e6);
  };
  float s = 1.0f;
  timeit("cudaMemcpy D2D (r+w)", [&] { CK(cudaMemcpyAsync(buf + TOTAL / 2, buf, TOTAL / 2, cudaMemcpyDeviceToDevice)); });
  for (int per : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "flat U4 grid=%dx%d", sms, per);
    timeit(nm, [&] { k_flat<4><<<sms * per, 256>>>((float4*)buf, TOTAL / 16, s); });
  }
  timeit("flat U8 grid=148x8", [&] { k_flat<8><<<sms * 8, 256>>>((float4*)buf, TOTAL / 16, s); });
  {
    uint64_t *db, *de, nt; make_parts(16384, &db, &de, &nt);
    Parts p{db, de, NARR, nt};
    timeit("tiles U4 hint grid=148x8", [&] { k_tiles<4, true><<<sms * 8, 256>>>(p, s); });
    timeit("tiles U4 nohint grid=148x8", [&] { k_tiles<4, false><<<sms * 8, 256>>>(p, s); });
    timeit("tiles U4 hint grid=ntiles", [&] { k_tiles<4, true><<<(unsigned)nt, 256>>>(p, s); });
    timeit("tiles U4 hint grid=148x16", [&] { k_tiles<4, true><<<sms * 16, 256>>>(p, s); });
  }
  {
    uint64_t *db, *de, nt; make_parts(32768, &db, &de, &nt);
    Parts p{db, de, NARR, nt};
    timeit("tiles U8 hint grid=148x8", [&] { k_tiles<8, true><<<sms * 8, 256>>>(p, s); });
    timeit("tiles U8 hint grid=ntiles", [&] { k_tiles<8, true><<<(unsigned)nt, 256>>>(p, s); });
  }
  {
    constexpr int CH = 16384, ST = 4;
    uint64_t *db, *de, nt; make_parts(CH, &db, &de, &nt);
    Parts p{db, de, NARR, nt};
    CK(cudaFuncSetAttribute(k_bulk<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
    for (int per : {2, 3}) {
      char nm[64]; snprintf(nm, 64, "bulk 4x16K grid=148x%d", per);
      timeit(nm, [&] { k_bulk<ST, CH><<<sms * per, 256, ST * CH>>>(p, s, CH); });
    }
  }
  {
    constexpr int CH = 32768, ST = 3;
    uint64_t *db, *de, nt; make_parts(CH, &db, &de, &nt);
    Parts p{db, de, NARR, nt};
    CK(cudaFuncSetAttribute(k_bulk<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
    timeit("bulk 3x32K grid=148x2", [&] { k_bulk<ST, CH><<<sms * 2, 256, ST * CH>>>(p, s, CH); });
  }
  return 0;
}
