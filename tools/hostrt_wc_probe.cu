// hostrt_wc_probe.cu — does the host staging allocation change the latency
// of a small host round trip (hop1 write to pinned host memory, barrier,
// hop2 read back) inside a copy kernel?
//
// Host slots allocated as (a) cached pinned memory (cudaHostAllocMapped |
// Portable: the engine's allocation) or (b) write-combined
// (| cudaHostAllocWriteCombined: not snooped by the CPU caches on GPU reads).
// Each of `nrt` CTAs (0..nrt-1) has its warps 1.. do one roundtrip of
// `hb` bytes on its own 128-byte-aligned slot while every CTA's warp 0 and
// the other CTAs copy `bytes` HBM->HBM (grid-stride, 16-byte LDG/STG).
// Back-to-back PDL launches; also a latency-only kernel (1 CTA, roundtrip,
// no copy).  Prints: alloc bytes hb nrt us_per_kernel
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostrt_wc_probe hostrt_wc_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

__global__ void __launch_bounds__(256) copyk(const int4* __restrict__ s, int4* __restrict__ d, size_t n16,
                                             int4* host, int4* back, int hn16, int nrt, int per,
                                             int slot16) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if ((int)blockIdx.x < nrt && threadIdx.x >= 32) {
    // `per` chunks of hn16 vectors each (slots slot16 apart): every hop1
    // write of the CTA's chunks, one barrier, every hop2 read
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    // hop1 flattened over (chunk, vector): every load of a thread before
    // its stores, so `per` chunks cost one HBM load latency, not `per`
    int4 v[8];
    const int tot = per * hn16;
    for (int b = 0; b < tot; b += 8 * nt) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = b + t + u * nt;
        if (k < tot) v[u] = s[(size_t)(blockIdx.x * per + k / hn16) * slot16 + k % hn16];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = b + t + u * nt;
        if (k < tot) host[(size_t)(blockIdx.x * per + k / hn16) * slot16 + k % hn16] = v[u];
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    for (int b = 0; b < tot; b += 8 * nt) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = b + t + u * nt;
        if (k < tot) {
          const size_t o = (size_t)(blockIdx.x * per + k / hn16) * slot16 + k % hn16;
          asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(host + o));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = b + t + u * nt;
        if (k < tot) back[(size_t)(blockIdx.x * per + k / hn16) * slot16 + k % hn16] = v[u];
      }
    }
  } else if (n16) {
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
  const size_t maxb = 64ull << 20;
  int4 *s, *d, *back;
  CK(cudaMalloc(&s, maxb));
  CK(cudaMalloc(&d, maxb));
  CK(cudaMalloc(&back, 4 << 20));
  CK(cudaMemset(s, 7, maxb));
  int4* hd[2];
  for (int a = 0; a < 2; ++a) {
    uint8_t* h;
    unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable | (a ? cudaHostAllocWriteCombined : 0);
    CK(cudaHostAlloc((void**)&h, 4 << 20, fl));
    CK(cudaHostGetDevicePointer((void**)&hd[a], h, 0));
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t sizes[] = {0, 4ull << 20, 16ull << 20};
  const int hbytes[] = {256, 2048};
  const int shapes[][2] = {{0, 0}, {1, 1}, {8, 1}, {4, 2}, {2, 4}, {1, 8}, {1, 16}, {16, 1}};
  const int spacings[] = {0};  // slot stride in bytes (0: hb, contiguous)
  for (int rep = 0; rep < 2; ++rep)
  for (size_t bytes : sizes)
    for (int hb : hbytes)
      for (auto& sh : shapes)
        for (int sp : spacings)
        for (int a = 0; a < 1; ++a) {
          const int nrt = sh[0], per = sh[1];
          if (nrt == 0 && (sp || hb != 256)) continue;
          if (nrt * per == 1 && sp) continue;
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(bytes ? 148 * 4 : (nrt ? nrt : 1));
          lc.blockDim = dim3(256);
          lc.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          const int reps = 400, slot16 = (sp ? sp : hb) / 16;
          for (int w = 0; w < 40; ++w)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, hd[a], back, hb / 16, nrt, per,
                                  slot16));
          CK(cudaEventRecord(e0, st));
          for (int r = 0; r < reps; ++r)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, hd[a], back, hb / 16, nrt, per,
                                  slot16));
          CK(cudaEventRecord(e1, st));
          CK(cudaEventSynchronize(e1));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          printf("%s %zu %d %dx%d stride %d %.3f\n", a ? "wc" : "cached", bytes, hb, nrt, per, sp ? sp : hb,
                 ms * 1e3 / reps);
        }
  return 0;
}
