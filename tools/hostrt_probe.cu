// hostrt_probe.cu — what does a small host round trip cost inside a copy kernel?
//
// A grid-stride HBM->HBM copy (148 x 4 CTAs x 256 threads, 16-byte LDG/STG)
// launched back to back, with CTA 0's warps 1.. also doing, per mode:
//   0  nothing (baseline)
//   1  store H bytes to mapped pinned host memory
//   2  store H bytes, CTA barrier, load them back into device memory (roundtrip)
//   3  like 2, with __threadfence_system() after the stores
//   4  store H bytes to a DEVICE buffer, barrier, load back (no PCIe at all)
// Plain and programmatic-dependent (PDL) launches.  Prints one line per case:
//   bytes host_bytes mode pdl us_per_kernel
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostrt_probe hostrt_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void __launch_bounds__(256) copyk(const int4* __restrict__ s, int4* __restrict__ d, size_t n16,
                                             int4* host, int4* back, int hn16, int mode) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x >= 32 && mode > 0) {
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    for (int i = t; i < hn16; i += nt) host[i] = s[i];
    if (mode == 3) __threadfence_system();
    if (mode >= 2) {
      asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
      for (int i = t; i < hn16; i += nt) {
        int4 v;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(host + i));
        back[i] = v;
      }
    }
  } else {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = s[i + u * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) d[i + u * stride] = v[u];
    }
    for (; i < n16; i += stride) d[i] = s[i];
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main() {
  const size_t maxb = 256ull << 20;
  int4 *s, *d, *back, *dev_stage;
  uint8_t* h;
  CK(cudaMalloc(&s, maxb));
  CK(cudaMalloc(&d, maxb));
  CK(cudaMalloc(&back, 1 << 20));
  CK(cudaMalloc(&dev_stage, 1 << 20));
  CK(cudaHostAlloc((void**)&h, 1 << 20, cudaHostAllocMapped | cudaHostAllocPortable));
  int4* hd = nullptr;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  CK(cudaMemset(s, 7, maxb));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t sizes[] = {4096, 64ull << 10, 4ull << 20, 16ull << 20, 64ull << 20, 128ull << 20};
  const int hbytes[] = {64, 5 << 10, 64 << 10};
  for (size_t bytes : sizes)
    for (int hb : hbytes)
      for (int mode = 0; mode <= 4; ++mode)
        for (int pdl = 0; pdl <= 1; ++pdl) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(148 * 4);
          lc.blockDim = dim3(256);
          lc.stream = st;
          cudaLaunchAttribute a[1];
          a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          a[0].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = a;
          lc.numAttrs = pdl;
          int4* stage = mode == 4 ? dev_stage : hd;
          const int reps = 200;
          for (int w = 0; w < 20; ++w)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, stage, back, hb / 16, mode));
          CK(cudaEventRecord(e0, st));
          for (int r = 0; r < reps; ++r)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, stage, back, hb / 16, mode));
          CK(cudaEventRecord(e1, st));
          CK(cudaEventSynchronize(e1));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          printf("%zu %d %d %d %.3f\n", bytes, hb, mode, pdl, ms * 1e3 / reps);
        }
  return 0;
}
