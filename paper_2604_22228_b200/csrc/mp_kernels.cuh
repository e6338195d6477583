// mp_kernels.cuh — sm_100a copy kernels of the multi-path transfer engine.
//
// One persistent "transfer kernel" runs per participating physical device and
// drains that device's tile table.  A tile is a byte range of one chunk-hop of
// the reference's chunk plan (pipeline.py:51-78): a Direct chunk, the hop1
// (src -> relay staging) or hop2 (relay staging -> dst) half of a GPU-staged
// chunk.  Tiles are claimed dynamically (atomic counter) in plan order, so a
// hop2 tile is only ever claimed after every hop1 tile it waits on was claimed
// by a resident CTA — the wait cannot deadlock, even when the relay and the
// source share one physical GPU.
//
// Ordering (the reference's hop1(i) -> hop2(i) edge, graph.py:115-117,
// sim.py:182-191): every hop1 tile of chunk i does a system-scope release
// increment on flag[i] (which lives in the relay's memory); hop2 tiles of
// chunk i acquire-spin until flag[i] reaches the hop1 tile count.  The last
// hop2 tile to pass resets the flag, so a cached CUDA graph can be replayed
// without a memset node.
#pragma once
#include <cstdint>

namespace mpk {

struct __align__(16) Tile {
  uint64_t src;          // byte address (local, peer-mapped or host-mapped)
  uint64_t dst;
  uint64_t len;          // bytes, >= 1
  uint32_t* signal;      // hop1: flag to release-increment after the copy
  uint32_t* wait;        // hop2: flag to acquire-wait on
  uint32_t* pass;        // hop2: pass counter next to the flag
  uint32_t wait_count;   // hop1 tiles of the chunk
  uint32_t pass_count;   // hop2 tiles of the chunk
  uint32_t flags;        // TILE_* bits
  uint32_t pad;
};

enum : uint32_t {
  TILE_SRC_MUTABLE = 1u,  // source written during this launch (staging): no .nc loads
};

struct __align__(16) Ctl {
  unsigned int work;     // next tile to claim
  unsigned int exit;     // CTAs finished
  unsigned int error;    // 1 = a wait timed out
  unsigned int launches;
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte loads: read-only non-coherent path for immutable sources, L2-only
// (.cg) for staging written during the launch.
__device__ __forceinline__ int4 ld16_nc(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld16_cg(const void* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(void* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Copy `len` bytes with 16-byte vectors when src and dst agree modulo 16
// (the reference keeps src offset == dst offset, pipeline.py:24), peeling an
// unaligned head and tail bytewise.  UNROLL independent 16-byte loads per
// thread are in flight before the matching stores.
template <int UNROLL, bool MUTABLE>
__device__ __forceinline__ void copy_range(const uint8_t* __restrict__ src,
                                           uint8_t* __restrict__ dst, uint64_t len) {
  const unsigned tid = threadIdx.x, nt = blockDim.x;
  if ((((uintptr_t)src ^ (uintptr_t)dst) & 15u) == 0) {
    uint64_t head = (16u - ((uintptr_t)dst & 15u)) & 15u;
    if (head > len) head = len;
    if (tid < head) dst[tid] = MUTABLE ? *(volatile const uint8_t*)(src + tid) : src[tid];
    const uint8_t* s = src + head;
    uint8_t* d = dst + head;
    const uint64_t nvec = (len - head) >> 4;
    const int4* s4 = reinterpret_cast<const int4*>(s);
    int4* d4 = reinterpret_cast<int4*>(d);
    const uint64_t step = (uint64_t)nt * UNROLL;
    uint64_t i = tid;
    for (; i + (uint64_t)(UNROLL - 1) * nt < nvec; i += step) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = MUTABLE ? ld16_cg(s4 + i + u * nt) : ld16_nc(s4 + i + u * nt);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) st16(d4 + i + u * nt, v[u]);
    }
    for (; i < nvec; i += nt) st16(d4 + i, MUTABLE ? ld16_cg(s4 + i) : ld16_nc(s4 + i));
    const uint64_t done = head + (nvec << 4);
    const uint64_t tail = len - done;
    if (tid < tail) dst[done + tid] = MUTABLE ? *(volatile const uint8_t*)(src + done + tid) : src[done + tid];
  } else if ((((uintptr_t)src ^ (uintptr_t)dst) & 3u) == 0) {
    uint64_t head = (4u - ((uintptr_t)dst & 3u)) & 3u;
    if (head > len) head = len;
    if (tid < head) dst[tid] = src[tid];
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src + head);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + head);
    const uint64_t nw = (len - head) >> 2;
    for (uint64_t i = tid; i < nw; i += nt) d[i] = MUTABLE ? *(volatile const uint32_t*)(s + i) : s[i];
    const uint64_t done = head + (nw << 2);
    if (tid < len - done) dst[done + tid] = src[done + tid];
  } else {
    for (uint64_t i = tid; i < len; i += nt) dst[i] = MUTABLE ? *(volatile const uint8_t*)(src + i) : src[i];
  }
}

constexpr uint64_t kWaitTimeoutNs = 4000000000ull;  // 4 s: never hang the GPU

template <int UNROLL>
__global__ void __launch_bounds__(256) transfer_kernel(const Tile* __restrict__ tiles,
                                                       unsigned ntiles, Ctl* ctl) {
  __shared__ unsigned s_claim[2];
  __shared__ Tile s_tile;
  if (threadIdx.x == 0) s_claim[0] = atomicAdd(&ctl->work, 1u);
  __syncthreads();
  unsigned w = s_claim[0];
  unsigned parity = 1;
  while (w < ntiles) {
    if (threadIdx.x == 0) {
      s_claim[parity] = atomicAdd(&ctl->work, 1u);  // prefetch the next claim
      s_tile = tiles[w];
      if (s_tile.wait) {
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(s_tile.wait) < s_tile.wait_count) {
          if (globaltimer() - t0 > kWaitTimeoutNs) {
            atomicExch(&ctl->error, 1u);
            break;
          }
          __nanosleep(64);
        }
        // last hop2 tile of the chunk to pass re-arms the flag for replay
        if (atomicAdd(s_tile.pass, 1u) + 1u == s_tile.pass_count) {
          *(volatile uint32_t*)s_tile.pass = 0u;
          *(volatile uint32_t*)s_tile.wait = 0u;
        }
      }
    }
    __syncthreads();
    const Tile& t = s_tile;
    if (t.flags & TILE_SRC_MUTABLE)
      copy_range<UNROLL, true>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len);
    else
      copy_range<UNROLL, false>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len);
    __syncthreads();  // every thread's stores precede the release below
    if (threadIdx.x == 0 && t.signal) {
      __threadfence_system();
      red_release_sys_add(t.signal, 1u);
    }
    w = s_claim[parity];
    parity ^= 1u;
    __syncthreads();  // s_tile / s_claim reuse
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->exit, 1u) + 1u == gridDim.x) {  // last CTA re-arms the counters
      ctl->work = 0u;
      ctl->exit = 0u;
      ctl->launches += 1u;
      __threadfence();
    }
  }
}

}  // namespace mpk
