// Experiment: 16-byte (LDG/STG.128) vs 32-byte (LDG/STG.E.ENL2.256, ld.global.v8.f32) vectors for
// the leaf kernel's streaming x *= s over 1 GiB, one CTA per tile (the shipped scheme).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/v8_probe tools/v8_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

template <int U>
__global__ void __launch_bounds__(256, 6) k16(float4* p, float s) {
  const size_t base = size_t(blockIdx.x) * 256 * U;
  float4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) r[u] = __ldcs(p + base + u * 256 + threadIdx.x);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float4 v = r[u];
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    __stcs(p + base + u * 256 + threadIdx.x, v);
  }
}

struct f8 { float a[8]; };
__device__ __forceinline__ f8 ld8(const float* q) {
  f8 v;
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v.a[0]), "=f"(v.a[1]), "=f"(v.a[2]), "=f"(v.a[3]), "=f"(v.a[4]), "=f"(v.a[5]), "=f"(v.a[6]), "=f"(v.a[7])
               : "l"(q));
  return v;
}
__device__ __forceinline__ void st8(float* q, const f8& v) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(q), "f"(v.a[0]), "f"(v.a[1]), "f"(v.a[2]),
               "f"(v.a[3]), "f"(v.a[4]), "f"(v.a[5]), "f"(v.a[6]), "f"(v.a[7])
               : "memory");
}

template <int U>
__global__ void __launch_bounds__(256, 6) k32(float* p, float s) {
  const size_t base = (size_t(blockIdx.x) * 256 * U) * 8;
  f8 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) r[u] = ld8(p + base + (u * 256 + threadIdx.x) * 8);
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[u].a[k] *= s;
    st8(p + base + (u * 256 + threadIdx.x) * 8, r[u]);
  }
}

int main() {
  const size_t bytes = size_t(1) << 30;
  float* p;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMemset(p, 0, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9f;
    for (int it = 0; it < 12; ++it) {
      cudaEventRecord(a);
      launch(it & 1 ? 0.5f : 2.0f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it >= 2 && ms < best) best = ms;
    }
    printf("%-28s %.4f ms  %.1f GB/s (r+w)\n", name, best, 2.0 * bytes / (best * 1e-3) / 1e9);
  };
  run("16B x4 (16 KiB tile)", [&](float s) { k16<4><<<bytes / (256 * 4 * 16), 256>>>((float4*)p, s); });
  run("16B x8 (32 KiB tile)", [&](float s) { k16<8><<<bytes / (256 * 8 * 16), 256>>>((float4*)p, s); });
  run("32B x2 (16 KiB tile)", [&](float s) { k32<2><<<bytes / (256 * 2 * 32), 256>>>(p, s); });
  run("32B x4 (32 KiB tile)", [&](float s) { k32<4><<<bytes / (256 * 4 * 32), 256>>>(p, s); });
  run("32B x1 (8 KiB tile)", [&](float s) { k32<1><<<bytes / (256 * 1 * 32), 256>>>(p, s); });
  CK(cudaGetLastError());
  return 0;
}
