// host_ce_probe.cu — how fast can a store-and-forward host path be on copy
// engines?  GPU -> pinned host -> GPU of `total` bytes (one B200, loopback):
//   alone   : one D2H, one H2D, and both at once (separate buffers)
//   staged  : chunks of `c` bytes, D2H of chunk i on stream 0, event, H2D of
//             chunk i on stream 1 (D2H of i+1 overlaps H2D of i) — 1-D copies
//   staged2d: the same with each op a 2-D copy of `rows` chunks at a stride
//             (the engine's grouped CE host path)
// Prints: mode total chunk rows GB/s (total / time, best of 5)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_ce_probe host_ce_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  const size_t total = 64ull << 20, span = 8 * total;
  uint8_t *src, *dst, *h, *h2;
  CK(cudaMalloc(&src, span));
  CK(cudaMalloc(&dst, span));
  CK(cudaHostAlloc((void**)&h, total, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaHostAlloc((void**)&h2, total, cudaHostAllocPortable | cudaHostAllocMapped));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev(512);
  for (auto& ev_i : ev) CK(cudaEventCreateWithFlags(&ev_i, cudaEventDisableTiming));
  cudaEvent_t t0, t1, j;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  auto timeit = [&](auto&& body) -> double {
    double best = 1e30;
    for (int r = 0; r < 6; ++r) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, s0));
      CK(cudaStreamWaitEvent(s1, t0, 0));
      body();
      CK(cudaEventRecord(j, s1));
      CK(cudaStreamWaitEvent(s0, j, 0));
      CK(cudaEventRecord(t1, s0));
      CK(cudaEventSynchronize(t1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, t0, t1));
      if (r) best = ms < best ? ms : best;
    }
    return total / (best * 1e-3) / 1e9;
  };
  printf("alone_d2h %zu 0 0 %.1f\n", total, timeit([&] { cudaMemcpyAsync(h, src, total, cudaMemcpyDeviceToHost, s0); }));
  printf("alone_h2d %zu 0 0 %.1f\n", total, timeit([&] { cudaMemcpyAsync(dst, h, total, cudaMemcpyHostToDevice, s1); }));
  printf("duplex_per_dir %zu 0 0 %.1f\n", total, timeit([&] {
           cudaMemcpyAsync(h, src, total, cudaMemcpyDeviceToHost, s0);
           cudaMemcpyAsync(dst, h2, total, cudaMemcpyHostToDevice, s1);
         }));
  const size_t chunks[] = {256ull << 10, 1ull << 20, 2ull << 20, 4ull << 20, 8ull << 20, 16ull << 20};
  for (size_t c : chunks) {
    const int n = (int)(total / c);
    double g = timeit([&] {
      for (int i = 0; i < n; ++i) {
        cudaMemcpyAsync(h + i * c, src + i * c, c, cudaMemcpyDeviceToHost, s0);
        cudaEventRecord(ev[i], s0);
        cudaStreamWaitEvent(s1, ev[i], 0);
        cudaMemcpyAsync(dst + i * c, h + i * c, c, cudaMemcpyHostToDevice, s1);
      }
    });
    printf("staged %zu %zu 1 %.1f\n", total, c, g);
    for (int rows : {2, 4}) {
      if (n % rows) continue;
      const int ng = n / rows;
      const size_t pitch = 8 * c;  // the chunk stride of a k-path round-robin plan
      double g2 = timeit([&] {
        for (int i = 0; i < ng; ++i) {
          uint8_t* hs = h + (size_t)i * rows * c;
          cudaMemcpy2DAsync(hs, c, src + (size_t)i * rows * pitch, pitch, c, rows, cudaMemcpyDeviceToHost, s0);
          cudaEventRecord(ev[i], s0);
          cudaStreamWaitEvent(s1, ev[i], 0);
          cudaMemcpy2DAsync(dst + (size_t)i * rows * pitch, pitch, hs, c, c, rows, cudaMemcpyHostToDevice, s1);
        }
      });
      printf("staged2d %zu %zu %d %.1f\n", total, c, rows, g2);
    }
  }
  return 0;
}
