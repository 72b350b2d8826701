// Experiment: full-duplex pipelining of 1 GiB in steps (H2D of step k+1 while D2H of step k),
// with each step moved as one DMA or as several smaller DMAs per direction, and with host pieces
// at page-aligned vs 272-byte-offset addresses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/duplex_probe tools/duplex_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

int main() {
  const size_t G = size_t(1) << 30, step = 32 << 20;
  char *h, *d;
  CK(cudaHostAlloc((void**)&h, G + (1 << 20), cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaMalloc((void**)&d, G + (1 << 20)));
  cudaStream_t hs, ds;
  CK(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
  const int nst = int(G / step);
  std::vector<cudaEvent_t> ev(nst);
  for (auto& x : ev) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  cudaEvent_t a, b, j;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
  struct Case { int pieces; size_t hoff, doff; int split; };
  std::vector<Case> cases = {{1,0,0,0},{1,16,16,0},{1,16,16,1},{1,272,272,1},{1,4080,4080,1},{1,16,16,2},{1,272,272,2},
                             {1,4080,4080,2},{1,16,16,3},{1,272,272,3},{1,4080,4080,3},{1,16,0,3},{2,16,16,3},{1,0,0,0}};
  for (const Case& c : cases) {
    float best = 1e9f;
    for (int it = 0; it < 5; ++it) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, hs));
      CK(cudaStreamWaitEvent(ds, a, 0));
      for (int k = 0; k < nst; ++k) {
        const size_t ps = step / c.pieces;
        auto copy = [&](bool h2d, size_t off, size_t n) {
          char* hp = h + c.hoff + off; char* dp = d + c.doff + off;
          const size_t al = c.split == 1 ? 4096 : 256;
          size_t head = c.split ? ((al - (uintptr_t(hp) & (al - 1))) & (al - 1)) : 0;
          if (head > n) head = n;
          size_t tail = c.split == 3 ? (uintptr_t(hp + n) & (al - 1)) : 0;
          if (head + tail > n) tail = 0;
          cudaStream_t s = h2d ? hs : ds;
          if (head) CK(cudaMemcpyAsync(h2d ? (void*)dp : (void*)hp, h2d ? (void*)hp : (void*)dp, head,
                                       h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s));
          CK(cudaMemcpyAsync(h2d ? (void*)(dp + head) : (void*)(hp + head), h2d ? (void*)(hp + head) : (void*)(dp + head),
                             n - head - tail, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s));
          if (tail) CK(cudaMemcpyAsync(h2d ? (void*)(dp + n - tail) : (void*)(hp + n - tail), h2d ? (void*)(hp + n - tail) : (void*)(dp + n - tail),
                                       tail, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s));
        };
        for (int p = 0; p < c.pieces; ++p) copy(true, k * step + p * ps, ps);
        CK(cudaEventRecord(ev[k], hs));
        CK(cudaStreamWaitEvent(ds, ev[k], 0));
        for (int p = 0; p < c.pieces; ++p) copy(false, k * step + p * ps, ps);
      }
      CK(cudaEventRecord(j, ds)); CK(cudaStreamWaitEvent(hs, j, 0));
      CK(cudaEventRecord(b, hs)); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("pieces/step %d host off %4zu dev off %4zu split %d: %.2f ms\n", c.pieces, c.hoff, c.doff, c.split, best);
  }
  return 0;
}
