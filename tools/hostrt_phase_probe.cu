// hostrt_phase_probe.cu — where does a small host round trip spend its time
// inside a saturating HBM copy?
//
// A grid-stride 16-byte LDG/STG copy of `bytes` (148 x 4 CTAs x 256
// threads) launched back to back (PDL); CTA 0's warps 1.. do one roundtrip
// of `hb` bytes: hop1 loads from device memory (t0 -> t1: loads returned),
// stores to mapped pinned host memory, named barrier (t2), hop2 loads from
// host (t3: returned), stores to device memory (t4).  %globaltimer stamps of
// thread 32 averaged over the timed launches, relative to t0.  The copy
// CTAs (and warp 0 of CTA 0) optionally sleep `delay` ns before copying,
// letting the roundtrip's loads reach HBM first.
// Prints: bytes hb delay us_per_kernel t1 t2 t3 t4 (ns after t0)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostrt_phase_probe hostrt_phase_probe.cu
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

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) copyk(const int4* __restrict__ s, int4* __restrict__ d, size_t n16,
                                             int4* host, int4* back, int hn16, int delay,
                                             unsigned long long* acc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x >= 32) {
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    const uint64_t t0 = gt();
    int4 v = make_int4(0, 0, 0, 0);
    if (t < hn16) v = s[n16 + (size_t)t * 8];  // source lines outside the copy's range
    unsigned x = 0;
    if (t < hn16) asm volatile("mov.b32 %0, %1;" : "=r"(x) : "r"(v.x));  // waits for the load
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    const uint64_t t1 = gt();
    v.y ^= (int)(x & 0u);
    if (t < hn16) host[t] = v;
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    const uint64_t t2 = gt();
    int4 w = make_int4(0, 0, 0, 0);
    if (t < hn16)
      asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                   : "l"(host + t));
    unsigned y = 0;
    if (t < hn16) asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(w.x));  // waits for the load
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    const uint64_t t3 = gt();
    w.y ^= (int)(y & 0u);
    if (t < hn16) back[t] = w;
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    const uint64_t t4 = gt();
    if (t == 0) {
      atomicAdd(&acc[0], t1 - t0);
      atomicAdd(&acc[1], t2 - t0);
      atomicAdd(&acc[2], t3 - t0);
      atomicAdd(&acc[3], t4 - t0);
      atomicAdd(&acc[4], 1ull);
    }
  } else {
    if (delay) __nanosleep(delay);
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
  unsigned long long* acc;
  CK(cudaMalloc(&s, maxb + (1 << 20)));
  CK(cudaMalloc(&d, maxb));
  CK(cudaMalloc(&back, 1 << 20));
  CK(cudaMalloc(&acc, 64));
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
  const size_t sizes[] = {0, 4ull << 20, 16ull << 20, 64ull << 20};
  const int hbytes[] = {256, 2048};
  const int delays[] = {0, 250, 500, 1000};
  for (size_t bytes : sizes)
    for (int hb : hbytes)
      for (int dl : delays) {
        if (bytes == 0 && dl) continue;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(bytes ? 148 * 4 : 1);
        lc.blockDim = dim3(256);
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        const int reps = 400;
        const size_t n16 = bytes ? bytes / 16 : 0;
        for (int w = 0; w < 40; ++w)
          CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, n16, hd, back, hb / 16, dl, acc));
        CK(cudaMemsetAsync(acc, 0, 64, st));
        CK(cudaEventRecord(e0, st));
        for (int r = 0; r < reps; ++r)
          CK(cudaLaunchKernelEx(&lc, copyk, (const int4*)s, d, n16, hd, back, hb / 16, dl, acc));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long a[5];
        CK(cudaMemcpy(a, acc, sizeof(a), cudaMemcpyDeviceToHost));
        printf("%zu %d %d %.3f %llu %llu %llu %llu\n", bytes, hb, dl, ms * 1e3 / reps, a[0] / a[4], a[1] / a[4],
               a[2] / a[4], a[3] / a[4]);
      }
  return 0;
}
