// hoststore_probe.cu — does the kind of store a kernel uses to write mapped
// pinned host memory change the cost of its completion under programmatic
// dependent launch?  A grid-stride HBM copy (148 x 4 CTAs x 256 threads)
// launched back to back with PDL; CTA 0's warps 1.. store `hb` bytes to host
// memory with one of:
//   0 none   1 st.global (default)   2 st.global.wt   3 st.global.cs
//   4 st.volatile   5 st.global + fence.sc.sys by the storing warps
//   6 st.global.wt + read back (roundtrip)   7 st.global + read back
//   8 st.release.sys of the last vector (release at system scope)
//   9 st.global, fence.sc.sys, barrier, read back (fence BEFORE hop2)
//  10 st.global, barrier, read back, fence.sc.sys (fence after hop2)
//  15 hop1 as a TMA bulk store (smem -> host, cp.async.bulk + wait_group 0)
//     then read back;  16: the same with wait_group.read only (no write wait)
//  12-14: the roundtrip on an EXTRA CTA (grid + 1) that does no copy work:
//  12 no fence, 13 fence.sc.sys after the stores (before the read back),
//  14 fence.sc.sys after the read back
// Prints: bytes hb mode us_per_kernel
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hoststore_probe hoststore_probe.cu
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

__device__ __forceinline__ void st_mode(int4* p, const int4& v, int mode) {
  switch (mode) {
    case 2:
    case 6:
      asm volatile("st.global.wt.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
      break;
    case 3:
      asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
      break;
    case 4:
      asm volatile("st.volatile.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                   "r"(v.w)
                   : "memory");
      break;
    default:
      asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
  }
}

__global__ void __launch_bounds__(256) copyk(const int4* __restrict__ s, int4* __restrict__ d, size_t n16,
                                             int4* host, int4* back, int hn16, int mode) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode >= 12) {
    if (blockIdx.x == gridDim.x - 1) {  // the extra CTA: the roundtrip only
      const int t = threadIdx.x, nt = blockDim.x;
      for (int i = t; i < hn16; i += nt) st_mode(host + i, s[i], 1);
      if (mode == 13) asm volatile("fence.sc.sys;" ::: "memory");
      __syncthreads();
      for (int i = t; i < hn16; i += nt) {
        int4 v;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(host + i));
        back[i] = v;
      }
      if (mode == 14) asm volatile("fence.sc.sys;" ::: "memory");
    } else {
      const size_t stride = (size_t)(gridDim.x - 1) * blockDim.x;
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
    return;
  }
  if ((mode == 15 || mode == 16) && blockIdx.x == 0 && threadIdx.x >= 32) {
    __shared__ __align__(128) int4 sbuf[256];  // <= 4 KiB
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    for (int i = t; i < hn16; i += nt) sbuf[i] = s[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    if (t == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(host),
                   "r"((unsigned)__cvta_generic_to_shared(sbuf)), "r"(hn16 * 16)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (mode == 15) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    if (mode == 15)
      for (int i = t; i < hn16; i += nt) {
        int4 v;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(host + i));
        back[i] = v;
      }
  } else if (blockIdx.x == 0 && threadIdx.x >= 32 && mode > 0 && mode < 15) {
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    for (int i = t; i < hn16; i += nt) st_mode(host + i, s[i], mode);
    if (mode == 5 || mode == 9) asm volatile("fence.sc.sys;" ::: "memory");
    if (mode == 8 && t == 0) {
      const int x = 1;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(host + hn16), "r"(x) : "memory");
    }
    if (mode == 6 || mode == 7 || mode == 9 || mode == 10) {
      asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
      for (int i = t; i < hn16; i += nt) {
        int4 v;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(host + i));
        back[i] = v;
      }
      if (mode == 10) asm volatile("fence.sc.sys;" ::: "memory");
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
  const size_t maxb = 64ull << 20;
  int4 *s, *d, *back;
  CK(cudaMalloc(&s, maxb));
  CK(cudaMalloc(&d, maxb));
  CK(cudaMalloc(&back, 1 << 20));
  CK(cudaMemset(s, 7, maxb));
  uint8_t* h;
  int4* hd;
  CK(cudaHostAlloc((void**)&h, 1 << 20, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t sizes[] = {4ull << 20, 8ull << 20, 16ull << 20, 32ull << 20};
  for (int rep = 0; rep < 2; ++rep)
    for (size_t bytes : sizes)
      for (int hb : {512, 4096})
        for (int mode : {0, 1, 7, 10, 15, 16}) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(148 * 4 + (mode >= 12 ? 1 : 0));
          lc.blockDim = dim3(256);
          lc.stream = st;
          cudaLaunchAttribute a[1];
          a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          a[0].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = a;
          lc.numAttrs = 1;
          const int reps = 400;
          for (int w = 0; w < 40; ++w)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, hd, back, hb / 16, mode));
          CK(cudaEventRecord(e0, st));
          for (int r = 0; r < reps; ++r)
            CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, bytes / 16, hd, back, hb / 16, mode));
          CK(cudaEventRecord(e1, st));
          CK(cudaEventSynchronize(e1));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          printf("%zu %d %d %.3f\n", bytes, hb, mode, ms * 1e3 / reps);
        }
  return 0;
}
