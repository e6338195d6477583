// kexp.cu — per-launch GPU cost of the transfer kernel in isolation (graph
// replay, back-to-back), against an empty kernel and a minimal copy kernel:
// where does a small message's time go?
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        -I paper_2604_22228_b200/csrc tools/kexp.cu -o _build/kexp && ./_build/kexp
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>

#include "mp_kernels.cuh"

__global__ void empty_kernel() {}

__global__ void plain_copy(const int4* __restrict__ s, int4* __restrict__ d, unsigned n16) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) d[i] = s[i];
}

// bisection kernels: copy_range alone, + descriptor from params, + from global
__global__ void k_range(const uint8_t* s, uint8_t* d, uint64_t len) {
  mpk::copy_range<8, false>(s, d, len);
}
__global__ void k_range_param(const __grid_constant__ mpk::Tile t) {
  mpk::copy_range<8, false>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len);
}
__global__ void k_range_global(const mpk::Tile* tiles) {
  __shared__ mpk::Tile st;
  if (threadIdx.x == 0) st = tiles[blockIdx.x];
  __syncthreads();
  mpk::copy_range<8, false>((const uint8_t*)st.src, (uint8_t*)st.dst, st.len);
}
__global__ void k_plain_global(const mpk::Tile* tiles) {
  const mpk::Tile t = tiles[blockIdx.x];
  const int4* s = (const int4*)t.src;
  int4* d = (int4*)t.dst;
  for (unsigned i = threadIdx.x; i < t.len / 16; i += blockDim.x) d[i] = s[i];
}

__global__ void k_spin(unsigned ns) {
  const uint64_t t0 = mpk::globaltimer();
  while (mpk::globaltimer() - t0 < ns) {
  }
}

template <class F>
static double per_launch_us(cudaStream_t s, F launch, int iters = 20000) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  launch();
  cudaStreamEndCapture(s, &g);
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1;
  for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms * 1e3 / iters;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t N = 64 << 20;
  uint8_t *src, *dst;
  cudaMalloc(&src, N);
  cudaMalloc(&dst, N);
  mpk::Ctl* ctl;
  cudaMalloc(&ctl, sizeof(mpk::Ctl));
  cudaMemset(ctl, 0, sizeof(mpk::Ctl));
  auto k_tma = mpk::transfer_kernel<1, 8>;
  auto k_vec = mpk::transfer_kernel<0, 8>;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  mpk::GroupSync gs{};
  printf("empty<<<1,128>>>           %.3f us\n", per_launch_us(s, [&] { empty_kernel<<<1, 128, 0, s>>>(); }));
  printf("empty<<<148,128>>>         %.3f us\n", per_launch_us(s, [&] { empty_kernel<<<148, 128, 0, s>>>(); }));
  printf("empty<<<1,128,128K smem>>> %.3f us\n", per_launch_us(s, [&] {
           cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
           empty_kernel<<<1, 128, 131072, s>>>();
         }));
  for (unsigned bytes : {4096u, 65536u, 1u << 20, 4u << 20}) {
    unsigned n16 = bytes / 16;
    unsigned grid = bytes <= 4096 ? 1 : 146;
    printf("plain_copy %8u B grid %3u  %.3f us\n", bytes, grid,
           per_launch_us(s, [&] { plain_copy<<<grid, 256, 0, s>>>((const int4*)src, (int4*)dst, n16); }));
  }
  for (unsigned ns : {0u, 200u, 400u, 600u, 800u, 1000u, 1200u, 1500u, 2000u, 3000u})
    printf("k_spin %4u ns        %.3f us\n", ns, per_launch_us(s, [&] { k_spin<<<1, 32, 0, s>>>(ns); }));
  {
    mpk::Tile t{};
    t.src = (uint64_t)src;
    t.dst = (uint64_t)dst;
    t.len = 4096;
    mpk::Tile* dt;
    cudaMalloc(&dt, sizeof t);
    cudaMemcpy(dt, &t, sizeof t, cudaMemcpyHostToDevice);
    printf("k_range 4K          %.3f us\n", per_launch_us(s, [&] { k_range<<<1, 256, 0, s>>>(src, dst, 4096); }));
    printf("k_range_param 4K    %.3f us\n", per_launch_us(s, [&] { k_range_param<<<1, 256, 0, s>>>(t); }));
    printf("k_range_global 4K   %.3f us\n", per_launch_us(s, [&] { k_range_global<<<1, 256, 0, s>>>(dt); }));
    printf("k_plain_global 4K   %.3f us\n", per_launch_us(s, [&] { k_plain_global<<<1, 256, 0, s>>>(dt); }));
  }
  for (unsigned bytes : {4096u, 16384u, 65536u, 131072u, 1u << 20, 4u << 20}) {
    // one tile per CTA, as the static schedule cuts it
    unsigned ntiles = bytes <= (128u << 10) ? (bytes + 4095) / 4096 : 146;
    size_t tb = ((bytes + ntiles - 1) / ntiles + 15) & ~(size_t)15;
    std::vector<mpk::Tile> tv;
    for (size_t o = 0; o < bytes; o += tb) {
      mpk::Tile t{};
      t.src = (uint64_t)(src + o);
      t.dst = (uint64_t)(dst + o);
      t.len = std::min<size_t>(tb, bytes - o);
      tv.push_back(t);
    }
    mpk::Tile* dt;
    cudaMalloc(&dt, tv.size() * sizeof(mpk::Tile));
    cudaMemcpy(dt, tv.data(), tv.size() * sizeof(mpk::Tile), cudaMemcpyHostToDevice);
    unsigned nt = (unsigned)tv.size();
    printf("tma %8u B %3u tiles       %.3f us\n", bytes, nt, per_launch_us(s, [&] {
             k_tma<<<nt, 128, 4 * 32768, s>>>(dt, nt, ctl, 4, 32768, nt, nullptr, gs, nullptr);
           }));
    printf("tma %8u B %3u tiles, 2 stages x 16K %.3f us\n", bytes, nt, per_launch_us(s, [&] {
             k_tma<<<nt, 128, 2 * 16384, s>>>(dt, nt, ctl, 2, 16384, nt, nullptr, gs, nullptr);
           }));
    printf("vec %8u B %3u tiles       %.3f us\n", bytes, nt, per_launch_us(s, [&] {
             k_vec<<<nt, 256, 0, s>>>(dt, nt, ctl, 4, 32768, nt, nullptr, gs, nullptr);
           }));
    {
      static mpk::SmallTable<mpk::kSmallMaxTiles> st;
      for (unsigned i = 0; i < nt; ++i) {
        st.src[i] = tv[i].src;
        st.dst[i] = tv[i].dst;
        st.len[i] = (uint32_t)tv[i].len;
      }
      printf("small %8u B %3u tiles     %.3f us\n", bytes, nt,
             per_launch_us(s, [&] { mpk::small_copy_kernel<4, mpk::kSmallMaxTiles><<<nt, 256, 0, s>>>(st); }));
    }
    printf("tma %8u B ntiles=0        %.3f us\n", bytes, per_launch_us(s, [&] {
             k_tma<<<nt, 128, 4 * 32768, s>>>(dt, 0, ctl, 4, 32768, 0, nullptr, gs, nullptr);
           }));
    cudaFree(dt);
  }
  return 0;
}
