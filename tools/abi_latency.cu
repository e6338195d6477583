/* abi_latency.cu — a plain-C consumer of include/mpb200.h: host cost per
 * mp_send call (cached-graph replay and per-call stream launch) and the GPU
 * time per message of back-to-back sends, with no Python in the loop.
 *
 *   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/abi_latency.cu \
 *       -o _build/abi_latency -L paper_2604_22228_b200 -lmpb200 \
 *       -Xlinker -rpath,'$ORIGIN/../paper_2604_22228_b200'
 * Baselines in the same process: an empty kernel (stream launch and
 * single-node graph replay) and a plain cudaMemcpyAsync per message.
 *   ./_build/abi_latency [iters]
 *
 * Prints one JSON line per (size, mode).  Loopback: logical GPU0/GPU1 on cuda:0.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <time.h>

#include "mpb200.h"

static double now_us(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

#define CHECK(x)                                                        \
  do {                                                                  \
    int rc_ = (x);                                                      \
    if (rc_ != 0) {                                                     \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, mp_last_error()); \
      exit(1);                                                          \
    }                                                                   \
  } while (0)

// Pseudo-random bytes (splitmix-style hash of the index): copy rates are
// data-dependent on B200 — constant data (e.g. a fresh cudaMalloc) copies
// ~1% faster at 512 MiB and a launch slot faster at 16 MiB than random data.
__global__ void fill_random(uint8_t* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 8;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    reinterpret_cast<unsigned long long*>(p)[i] = z ^ (z >> 31);
  }
}

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 0) *p = 0;
}

static int cmp_d(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : x > y;
}

int main(int argc, char** argv) {
  int iters = argc > 1 ? atoi(argv[1]) : 10000;
  const char* topo_text =
      "name loop\n[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 3000000000000.0 2e-06 full 1\n"
      "[hostlink]\n0 6000000000.0 1e-05 full\n1 6000000000.0 1e-05 full\n";
  mp_topology* topo = NULL;
  CHECK(mp_topology_load(topo_text, "loop", &topo));
  int32_t dmap[2] = {0, 0};
  mp_ctx* ctx = NULL;
  CHECK(mp_ctx_create(2, dmap, &ctx));
  CHECK(mp_ctx_set_topology(ctx, topo));
  size_t max_bytes = 512u << 20;
  void *src = NULL, *dst = NULL;
  if (cudaMalloc(&src, max_bytes) || cudaMalloc(&dst, max_bytes)) return 1;
  if (!getenv("ZERO_DATA")) fill_random<<<1184, 256>>>((uint8_t*)src, max_bytes);
  else cudaMemset(src, 0, max_bytes);
  cudaMemset(dst, 0, max_bytes);
  cudaDeviceSynchronize();
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* per = (double*)malloc(sizeof(double) * iters);
  /* baselines: GPU time per launch of an empty kernel, stream and graph */
  {
    for (int i = 0; i < 100; ++i) empty_kernel<<<1, 128, 0, s>>>(NULL);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) empty_kernel<<<1, 128, 0, s>>>(NULL);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"mode\": \"empty_kernel_stream\", \"gpu_us_per_msg\": %.3f}\n", ms * 1e3 / iters);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    empty_kernel<<<1, 128, 0, s>>>(NULL);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 100; ++i) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"mode\": \"empty_kernel_graph\", \"gpu_us_per_msg\": %.3f}\n", ms * 1e3 / iters);
    for (int i = 0; i < 100; ++i) cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) cudaMemcpyAsync(dst, src, 4096, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"mode\": \"memcpy_async_4k\", \"gpu_us_per_msg\": %.3f}\n", ms * 1e3 / iters);
    fflush(stdout);
  }
  const uint64_t sizes[] = {4096, 65536, 1u << 20, 4u << 20, 16u << 20, 32u << 20, 64u << 20,
                           128u << 20, 256u << 20, 512u << 20};
  mp_engine_opts base;
  CHECK(mp_ctx_get_engine(ctx, &base));
  const char* variant = getenv("ENGINE");
  mp_engine_opts o = base;
  if (variant && variant[0] == 'v') { o.copy_kind = MP_COPY_VEC; o.threads = 256; }
  if (variant && variant[0] == 'r') { o.copy_kind = MP_COPY_TMA; o.threads = 128; o.ctas_per_sm = 1; }
  if (variant && variant[0] == 'c') o.direct_engine = MP_ENGINE_CE;
  if (variant && variant[0] == 'p') o.tma_peer = -1; /* the NVLink-peer LDG/STG kernel */
  if (variant && variant[0] == 'h') o.host_engine = MP_ENGINE_SM; /* SM host path */
  if (getenv("TILE")) o.tile_bytes = atoll(getenv("TILE"));
  if (getenv("STAGES")) o.tma_stages = atoi(getenv("STAGES"));
  if (getenv("BLOCK")) o.tma_block = atoi(getenv("BLOCK"));
  if (getenv("CTAS")) o.ctas_per_sm = atoi(getenv("CTAS"));
  if (getenv("UNROLL")) o.unroll = atoi(getenv("UNROLL"));
  if (getenv("SMALL")) o.small_max_bytes = atoll(getenv("SMALL"));
  const char* sched = getenv("SCHED");
  if (sched && sched[0] == 'd') o.sched = MP_SCHED_DYNAMIC;
  CHECK(mp_ctx_set_engine(ctx, &o));
  const int modes = getenv("MODES") ? atoi(getenv("MODES")) : 3;
  for (int mode = 0; mode < modes; ++mode) {
    /* 0: single path, graph replay; 1: direct + host, graph replay; 2: single path,
       stream; 3: direct + host, stream */
    mp_config cfg = {1, mode == 1 || mode == 3, 1, mode < 2, 16, MP_SHARE_BANDWIDTH};
    for (size_t k = 0; k < sizeof sizes / sizeof sizes[0]; ++k) {
      uint64_t n = sizes[k];
      int it = n >= (128u << 20) ? iters / 100 : n >= (16u << 20) ? iters / 10 : iters;
      if (it < 10) it = 10;
      for (int i = 0; i < 20; ++i) CHECK(mp_send(ctx, src, dst, n, 0, 1, &cfg, s));
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int i = 0; i < it; ++i) {
        double t0 = now_us();
        CHECK(mp_send(ctx, src, dst, n, 0, 1, &cfg, s));
        per[i] = now_us() - t0;
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      double sum = 0;
      for (int i = 0; i < it; ++i) sum += per[i];
      qsort(per, it, sizeof(double), cmp_d);
      mp_send_stats st;
      CHECK(mp_send_stats_get(ctx, &st));
      printf("{\"engine\": \"%s%s small<=%lld\", \"mode\": \"%s\", \"bytes\": %llu, \"host_us_mean\": %.3f, \"host_us_p50\": %.3f, "
             "\"host_us_p99\": %.3f, \"gpu_us_per_msg\": %.3f, \"gbs\": %.3f, \"launch_us\": %.3f}\n",
             variant ? variant : "default", o.sched == MP_SCHED_DYNAMIC ? "+dynamic" : "", (long long)o.small_max_bytes, mode == 0 ? "single_graph" : mode == 1 ? "multi_graph" : mode == 2 ? "single_stream" : "multi_stream",
             (unsigned long long)n, sum / it, per[it / 2], per[(int)(it * 0.99)],
             ms * 1e3 / it, n / (ms * 1e-3 / it) / 1e9, st.launch_us);
      fflush(stdout);
    }
  }
  CHECK(mp_sync(ctx));
  mp_ctx_destroy(ctx);
  mp_topology_destroy(topo);
  return 0;
}
