// host_api_cost.cu — host cost (ns per call) of the CUDA runtime calls an
// mp_send makes, next to mp_send itself, on this box's host CPU.
//
// Batches of 200 calls are timed with CLOCK_MONOTONIC; the stream is drained
// between batches outside the timed region (so a full launch queue never
// blocks a timed call).  Loopback: logical GPU0/GPU1 on cuda:0.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/host_api_cost.cu \
//       -o _build/host_api_cost -L paper_2604_22228_b200 -lmpb200 \
//       -Xlinker -rpath,'$ORIGIN/../paper_2604_22228_b200'
// Prints: name ns_per_call (median of batches)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include <algorithm>
#include <functional>
#include <string>
#include <vector>

#include <cuda.h>

#include "mpb200.h"

static double now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e9 + ts.tv_nsec;
}

struct Params {
  uint64_t w[40];  // 320 bytes, the small-message kernel's parameter block
};
__global__ void empty_kernel(const __grid_constant__ Params p) {
  if (p.w[0] == 12345 && threadIdx.x == 1000) asm volatile("trap;");
}
__global__ void empty_small(uint64_t x) {
  if (x == 12345 && threadIdx.x == 1000) asm volatile("trap;");
}

__global__ void spin_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) break;
  }
}

static bool g_blocked = false;  // a 3 ms spin kernel ahead of every batch: the timed calls only queue

static void measure(const char* name, cudaStream_t s, const std::function<void()>& call, int batches = 60) {
  std::vector<double> per;
  for (int b = 0; b < batches; ++b) {
    cudaStreamSynchronize(s);
    if (g_blocked) spin_kernel<<<1, 32, 0, s>>>(3000000);
    const double t0 = now_ns();
    for (int i = 0; i < 200; ++i) call();
    per.push_back((now_ns() - t0) / 200);
  }
  cudaStreamSynchronize(s);
  std::sort(per.begin() + 5, per.end());  // the first 5 batches are warm-up
  printf("%-40s %8.1f\n", (std::string(name) + (g_blocked ? " [queued]" : "")).c_str(), per[5 + (per.size() - 5) / 2]);
  fflush(stdout);
}

int main() {
  cudaSetDevice(0);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (int pass = 0; pass < 2; ++pass) {
  g_blocked = pass == 1;
  Params p{};
    int dev = 0;
    measure("busy loop baseline (clock only)", s, [] {});
    measure("cudaGetDevice", s, [&] { cudaGetDevice(&dev); });
    measure("cudaSetDevice(same)", s, [&] { cudaSetDevice(0); });
    measure("cudaEventRecord", s, [&] { cudaEventRecord(ev, s); });
    measure("cudaStreamWaitEvent", s, [&] { cudaStreamWaitEvent(s2, ev, 0); });
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(16);
    lc.blockDim = dim3(256);
    lc.stream = s;
    measure("cudaLaunchKernelEx 320B", s, [&] { cudaLaunchKernelEx(&lc, empty_kernel, p); });
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = a;
    lc.numAttrs = 1;
    measure("cudaLaunchKernelEx 320B + PDL", s, [&] { cudaLaunchKernelEx(&lc, empty_kernel, p); });
    measure("launch PDL + eventRecord", s, [&] {
      cudaLaunchKernelEx(&lc, empty_kernel, p);
      cudaEventRecord(ev, s);
    });
    measure("<<<>>> 320B", s, [&] { empty_kernel<<<16, 256, 0, s>>>(p); });
    measure("<<<>>> 8B", s, [&] { empty_small<<<16, 256, 0, s>>>(7); });
    uint64_t x8 = 7;
    measure("cudaLaunchKernelEx 8B + PDL", s, [&] { cudaLaunchKernelEx(&lc, empty_small, x8); });
    // driver API: cuLaunchKernelEx on the same function
    {
      CUfunction f;
      cudaGetFuncBySymbol(&f, (const void*)empty_kernel);
      CUlaunchConfig cc = {};
      cc.gridDimX = 16; cc.gridDimY = 1; cc.gridDimZ = 1;
      cc.blockDimX = 256; cc.blockDimY = 1; cc.blockDimZ = 1;
      cc.hStream = (CUstream)s;
      CUlaunchAttribute ca[1];
      ca[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      ca[0].value.programmaticStreamSerializationAllowed = 1;
      cc.attrs = ca;
      cc.numAttrs = 1;
      void* args[] = {&p};
      measure("cuLaunchKernelEx 320B + PDL", s, [&] { cuLaunchKernelEx(&cc, f, args, nullptr); });
      void* extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, &p, CU_LAUNCH_PARAM_BUFFER_SIZE, nullptr, CU_LAUNCH_PARAM_END};
      size_t psz = sizeof p;
      extra[3] = &psz;
      measure("cuLaunchKernelEx 320B + PDL (extra)", s, [&] { cuLaunchKernelEx(&cc, f, nullptr, extra); });
      cc.numAttrs = 0;
      measure("cuLaunchKernelEx 320B", s, [&] { cuLaunchKernelEx(&cc, f, args, nullptr); });
    }
    // a one-kernel graph replay
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s2, cudaStreamCaptureModeThreadLocal);
    empty_kernel<<<16, 256, 0, s2>>>(p);
    cudaStreamEndCapture(s2, &g);
    cudaGraphInstantiate(&ge, g, 0);
    measure("cudaGraphLaunch (1 kernel)", s, [&] { cudaGraphLaunch(ge, s); });
  
  
  }
  // mp_send: single path, cached; 1 MiB (small kernel, PDL) and 16 MiB (static TMA, PDL)
  const char* topo_text =
      "name loop\n[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 3.2e12 2e-06 full 1\n"
      "[hostlink]\n0 1e9 1e-05 full\n1 1e9 1e-05 full\n";
  mp_topology* topo = nullptr;
  if (mp_topology_load(topo_text, "loop", &topo)) { printf("topology: %s\n", mp_last_error()); return 1; }
  int32_t dmap[2] = {0, 0};
  mp_ctx* ctx = nullptr;
  if (mp_ctx_create(2, dmap, &ctx) || mp_ctx_set_topology(ctx, topo)) { printf("ctx: %s\n", mp_last_error()); return 1; }
  uint8_t *a1, *b1;
  cudaMalloc(&a1, 16 << 20);
  cudaMalloc(&b1, 16 << 20);
  mp_config cfg = {1, 0, 1, 1, 16, 0};
  for (uint64_t n : {(uint64_t)1 << 20, (uint64_t)16 << 20}) {
    char name[64];
    snprintf(name, sizeof name, "mp_send %llu MiB (graph, cached)", (unsigned long long)(n >> 20));
    measure(name, s, [&] { mp_send(ctx, a1, b1, n, 0, 1, &cfg, s); });
  }
  mp_config host = {1, 1, 8, 1, 16, 0};
  measure("mp_send 4 MiB direct+host k=8", s, [&] { mp_send(ctx, a1, b1, 4 << 20, 0, 1, &host, s); });
  g_blocked = true;
  for (uint64_t n : {(uint64_t)1 << 20, (uint64_t)16 << 20}) {
    char name[64];
    snprintf(name, sizeof name, "mp_send %llu MiB (graph, cached)", (unsigned long long)(n >> 20));
    measure(name, s, [&] { mp_send(ctx, a1, b1, n, 0, 1, &cfg, s); });
  }
  mp_ctx_destroy(ctx);
  mp_topology_destroy(topo);
  return 0;
}
