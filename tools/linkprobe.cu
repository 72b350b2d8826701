// Host-link probe: pinned H2D / D2H / bidirectional cudaMemcpyAsync bandwidth.
// Used once per box to establish the copy roofline denominator.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
int main(int argc, char** argv) {
  size_t bytes = (argc > 1 ? atoll(argv[1]) : 1024) << 20;
  void *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&h2, bytes, cudaHostAllocPortable));
  memset(h1, 1, bytes); memset(h2, 2, bytes);
  CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&d2, bytes));
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      if (mode == 0 || mode == 2) CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1));
      if (mode == 1 || mode == 2) {
        if (mode == 2) { cudaEvent_t f; CK(cudaEventCreate(&f)); CK(cudaEventRecord(f, s1)); }
        CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, mode == 2 ? s2 : s1));
      }
      if (mode == 2) { cudaEvent_t j; CK(cudaEventCreate(&j)); CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s1, j, 0)); }
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    double gbs = (mode == 2 ? 2.0 : 1.0) * bytes / (best * 1e-3) / 1e9;
    printf("%s bytes=%zu best_ms=%.3f GB/s=%.2f\n", mode == 0 ? "H2D" : mode == 1 ? "D2H" : "BIDIR(sum)", bytes, best, gbs);
  }
  // chunked H2D 32 MiB on 4 streams
  {
    cudaStream_t ss[4]; for (int i = 0; i < 4; ++i) CK(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
    size_t ch = 32 << 20; float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      CK(cudaDeviceSynchronize()); CK(cudaEventRecord(a, 0));
      int i = 0; for (size_t o = 0; o < bytes; o += ch, ++i) CK(cudaMemcpyAsync((char*)d1 + o, (char*)h1 + o, ch, cudaMemcpyHostToDevice, ss[i % 4]));
      CK(cudaDeviceSynchronize()); CK(cudaEventRecord(b, 0)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    printf("H2D chunked32MiBx4streams GB/s=%.2f\n", bytes / (best * 1e-3) / 1e9);
  }
  // pageable H2D
  { void* p = malloc(bytes); memset(p, 3, bytes); float best = 1e30f;
    for (int it = 0; it < 3; ++it) { CK(cudaDeviceSynchronize()); CK(cudaEventRecord(a, s1)); CK(cudaMemcpyAsync(d1, p, bytes, cudaMemcpyHostToDevice, s1)); CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms; }
    printf("H2D pageable GB/s=%.2f\n", bytes / (best * 1e-3) / 1e9); }
  // D2D copy
  { float best = 1e30f; for (int it = 0; it < 5; ++it) { CK(cudaEventRecord(a, s1)); CK(cudaMemcpyAsync(d2, d1, bytes, cudaMemcpyDeviceToDevice, s1)); CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms; }
    printf("D2D r+w GB/s=%.2f\n", 2.0 * bytes / (best * 1e-3) / 1e9); }
  return 0;
}
