// Host-link experiment: can SM-driven PCIe traffic (kernels loading from / storing to mapped
// pinned host memory) add to the copy engines' full-duplex bandwidth?
//   CE: cudaMemcpyAsync on a copy stream; SM: a grid-stride 16-byte copy kernel over mapped memory.
// Modes: H2D / D2H alone (CE, SM), and both directions at once in every CE/SM combination.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smlink_probe tools/smlink_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void smcopy(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

int main(int argc, char** argv) {
  const size_t bytes = size_t(argc > 1 ? atoll(argv[1]) : 1024) << 20;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaHostAlloc(&h2, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  memset(h1, 1, bytes); memset(h2, 2, bytes);
  CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&d2, bytes));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, j;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  const char* names[] = {"H2D CE", "D2H CE", "H2D SM", "D2H SM", "both CE+CE", "both CE(H2D)+SM(D2H)", "both SM(H2D)+CE(D2H)", "both SM+SM"};
  for (int ctas_per_sm : {2, 4, 8}) {
    const unsigned grid = unsigned(sms * ctas_per_sm);
    for (int mode = 0; mode < 8; ++mode) {
      if (ctas_per_sm != 4 && (mode < 2 || mode == 4)) continue;   // CE-only modes once
      float best = 1e30f;
      for (int it = 0; it < 5; ++it) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, s1));
        CK(cudaStreamWaitEvent(s2, a, 0));
        const bool h2d = mode == 0 || mode == 2 || mode >= 4, d2h = mode == 1 || mode == 3 || mode >= 4;
        const bool h2d_sm = mode == 2 || mode == 6 || mode == 7, d2h_sm = mode == 3 || mode == 5 || mode == 7;
        if (h2d) {
          if (h2d_sm) smcopy<<<grid, 256, 0, s1>>>((uint4*)d1, (const uint4*)h1, bytes / 16);
          else CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1));
        }
        if (d2h) {
          if (d2h_sm) smcopy<<<grid, 256, 0, s2>>>((uint4*)h2, (const uint4*)d2, bytes / 16);
          else CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2));
        }
        CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s1, j, 0));
        CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
      }
      const double mult = mode >= 4 ? 2.0 : 1.0;
      printf("%-24s ctas/SM=%d  %.3f ms  %.2f GB/s\n", names[mode], ctas_per_sm, best, mult * bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
