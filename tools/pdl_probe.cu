// pdl_probe.cu — does programmatic dependent launch (PDL) shrink the ~2 us
// per-kernel slot of back-to-back dependent copies on B200?  Per-kernel GPU
// time of a 148-CTA copy kernel, stream-ordered, for: plain launches, PDL
// launches (griddepcontrol.wait before touching memory), each inside one
// graph of K kernels (GPU-side cost, no host in the loop) and as K separate
// one-kernel graph launches (the engine's per-send shape).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pdl_probe.cu -o _build/pdl_probe
#include <cuda_runtime.h>
#include <stdio.h>

#include <chrono>

__global__ void __launch_bounds__(256) copy_k(const int4* __restrict__ s, int4* __restrict__ d,
                                              unsigned n16, int pdl) {
  // pdl 1: trigger dependents at entry; pdl 2: trigger after the copy loop
  if (pdl == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
    d[i] = s[i];
  if (pdl == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static void launch(cudaStream_t s, const int4* a, int4* b, unsigned n16, int pdl) {
  cudaLaunchConfig_t cfg = {};
  unsigned grid = (n16 + 255) / 256;
  cfg.gridDim = dim3(grid < 148 ? grid : 148);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, copy_k, a, b, n16, pdl);
}

static double per_kernel_us(cudaStream_t s, const int4* a, int4* b, unsigned n16, int pdl,
                            int per_graph, int graphs) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < per_graph; ++i) launch(s, a, b, n16, pdl);
  cudaStreamEndCapture(s, &g);
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1;
  for (int i = 0; i < 50; ++i) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < graphs; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms * 1e3 / ((double)per_graph * graphs);
}

// K launches straight onto the stream (no graph): host launch cost vs GPU
static double per_launch_direct_us(cudaStream_t s, const int4* a, int4* b, unsigned n16, int pdl,
                                   int iters, double* host_us) {
  for (int i = 0; i < 200; ++i) launch(s, a, b, n16, pdl);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) launch(s, a, b, n16, pdl);
  auto t1 = std::chrono::steady_clock::now();
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  *host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
  return ms * 1e3 / iters;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t N = 64 << 20;
  int4 *a, *b;
  cudaMalloc(&a, N);
  cudaMalloc(&b, N);
  cudaMemset(a, 1, N);
  printf("bytes,plain_in_graph_us,pdl_in_graph_us,plain_graph_per_send_us,pdl_graph_per_send_us,"
         "plain_direct_us,plain_direct_host_us,pdl_direct_us,pdl_direct_host_us,pdl_late_direct_us,"
         "pdl_late_direct_host_us\n");
  for (size_t n : {4096ul, 65536ul, 262144ul, 1ul << 20, 2ul << 20, 3ul << 20, 4ul << 20, 16ul << 20}) {
    unsigned n16 = (unsigned)(n / 16);
    double p1 = per_kernel_us(s, a, b, n16, 0, 32, 300);
    double q1 = per_kernel_us(s, a, b, n16, 1, 32, 300);
    double p2 = per_kernel_us(s, a, b, n16, 0, 1, 10000);
    double q2 = per_kernel_us(s, a, b, n16, 1, 1, 10000);
    double hp, hq;
    double p3 = per_launch_direct_us(s, a, b, n16, 0, 20000, &hp);
    double q3 = per_launch_direct_us(s, a, b, n16, 1, 20000, &hq);
    double hr;
    double r3 = per_launch_direct_us(s, a, b, n16, 2, 20000, &hr);
    printf("%zu,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f\n", n, p1, q1, p2, q2, p3, hp, q3, hq,
           r3, hr);
  }
  return 0;
}
