// Does write-combined pinned host memory change the copy engines' rates?  H2D alone and both
// directions at once (1 GiB each), source / destination pinned with and without
// cudaHostAllocWriteCombined.  Design experiment (round 2).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
static float timed(void* d1, const void* h1, void* h2, const void* d2, size_t bytes, int both, cudaStream_t s1,
                   cudaStream_t s2, cudaEvent_t a, cudaEvent_t b, cudaEvent_t j) {
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, s1));
    CK(cudaStreamWaitEvent(s2, a, 0));
    CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1));
    if (both) CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2));
    CK(cudaEventRecord(j, s2));
    CK(cudaStreamWaitEvent(s1, j, 0));
    CK(cudaEventRecord(b, s1));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}
int main() {
  const size_t bytes = size_t(1) << 30;
  void *hn, *hw, *on, *ow, *d1, *d2;
  CK(cudaHostAlloc(&hn, bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&hw, bytes, cudaHostAllocPortable | cudaHostAllocWriteCombined));
  CK(cudaHostAlloc(&on, bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&ow, bytes, cudaHostAllocPortable | cudaHostAllocWriteCombined));
  memset(hn, 1, bytes); memset(hw, 1, bytes); memset(on, 2, bytes); memset(ow, 2, bytes);
  CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&d2, bytes));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, j;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&j));
  for (int rep = 0; rep < 2; ++rep) {
    printf("H2D normal src      %.2f GB/s\n", bytes / (timed(d1, hn, on, d2, bytes, 0, s1, s2, a, b, j) * 1e-3) / 1e9);
    printf("H2D WC src          %.2f GB/s\n", bytes / (timed(d1, hw, on, d2, bytes, 0, s1, s2, a, b, j) * 1e-3) / 1e9);
    printf("both, normal/normal %.2f GB/s\n", 2 * bytes / (timed(d1, hn, on, d2, bytes, 1, s1, s2, a, b, j) * 1e-3) / 1e9);
    printf("both, WC src        %.2f GB/s\n", 2 * bytes / (timed(d1, hw, on, d2, bytes, 1, s1, s2, a, b, j) * 1e-3) / 1e9);
    printf("both, WC src + dst  %.2f GB/s\n", 2 * bytes / (timed(d1, hw, ow, d2, bytes, 1, s1, s2, a, b, j) * 1e-3) / 1e9);
  }
  return 0;
}
