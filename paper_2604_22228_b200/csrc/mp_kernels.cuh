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
  union {
    uint32_t* pass;      // hop2: pass counter next to the flag
    uint8_t* stage;      // TILE_ROUNDTRIP: the staging slot (mapped pinned host memory)
  };
  uint32_t wait_count;   // hop1 tiles of the chunk (TILE_ROUNDTRIP: source bytes hop1 adds
                         // before the chunk to write whole host lines)
  uint32_t pass_count;   // hop2 tiles of the chunk (TILE_ROUNDTRIP: bytes added after it)
  uint32_t flags;        // TILE_* bits
  uint32_t node;        // logical graph node (chunk-hop) id, for traces
};

enum : uint32_t {
  TILE_SRC_MUTABLE = 1u,  // source written during this launch (staging): no .nc loads
  TILE_SIGNAL_BYTES = 2u, // signal is a u64 byte counter (+len), not a u32 tile count (+1)
  // A whole host-staged chunk in ONE CTA (source and destination on one
  // device): hop1 src -> stage, a CTA barrier, hop2 stage -> dst.  The
  // barrier orders hop2 after hop1 (graph.py:115-117) with no flag and no
  // system-scope fence; trace nodes `node` (hop1) and `node + 1` (hop2).
  TILE_ROUNDTRIP = 4u,
  // signal / wait at GPU scope: producer and consumer tiles run on the same
  // device (a relay or host chunk in loopback), so no system-scope release
  TILE_SCOPE_GPU = 8u,
  // a helper-warp roundtrip ends with a system-scope fence (messages long
  // enough for the fence to finish inside the direct stream): the host
  // writes then retire before the grid completes, instead of in its flush,
  // which a programmatic-dependent next launch waits for (~0.7 us at
  // 32-64 MiB, tools/hoststore_probe.cu)
  TILE_FENCE = 16u,
};

// Cross-process ordering of consecutive group transfers (multi-process mode):
// every rank's kernel for transfer n starts once every rank finished n-1
// (gen[q] >= *seq), and its last CTA bumps *seq and its own gen.  All state is
// in device memory, so a captured graph replays it unchanged.  n == 0: off.
constexpr int kMaxRanks = 16;
struct GroupSync {
  uint32_t* gen[kMaxRanks];  // every rank's generation counter (IPC-mapped)
  uint32_t* seq;             // this rank's transfer sequence number (local)
  uint32_t* self_gen;        // this rank's generation counter (local)
  int n;
};

// Claim counters of one cached program (stored right after its tile table).
// Launch L of the program claims from work[L & 1]; L = (arrival ticket) /
// gridDim.x because every launch of a program has the same grid and launches
// are stream-ordered.  The first CTA of launch L zeroes work[(L + 1) & 1] for
// the next launch (the previous user of that slot, launch L-1, has finished),
// so dynamic tables need no exit protocol (fence + atomic per CTA + a reset
// by the last CTA) to be replayable.
struct __align__(16) Sched {
  unsigned long long arrive;
  unsigned int work[2];
};

struct __align__(16) Ctl {
  unsigned int work;     // next tile to claim
  unsigned int exit;     // CTAs finished
  unsigned int error;    // non-zero: a wait timed out (1 relay flag, 2 group barrier, 3 receiver)
  unsigned int launches;
  unsigned int* herr;    // the same code, in mapped pinned host memory: the host sees a
                         // timeout with a plain load and fails every later send (sticky)
  unsigned long long timeout_ns;  // flag / barrier wait limit (0: kWaitTimeoutNs)
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

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
                                           uint8_t* __restrict__ dst, uint64_t len,
                                           unsigned tid, unsigned nt) {
  if ((((uintptr_t)src ^ (uintptr_t)dst) & 15u) == 0) {
    uint64_t head = (16u - ((uintptr_t)dst & 15u)) & 15u;
    if (head > len) head = len;
    const uint8_t* s = src + head;
    uint8_t* d = dst + head;
    const uint64_t nvec = (len - head) >> 4;
    const uint64_t done = head + (nvec << 4);
    const uint64_t tail = len - done;
    // the peel's byte loads are issued before the vector loop and stored
    // after it: an unaligned chunk boundary (most reference chunk offsets
    // are unaligned) never adds a serial memory latency to its tile
    const bool hv = tid < head, tv = tid < tail;
    uint8_t hb = 0, tb = 0;
    if (hv) hb = MUTABLE ? *(volatile const uint8_t*)(src + tid) : src[tid];
    if (tv) tb = MUTABLE ? *(volatile const uint8_t*)(src + done + tid) : src[done + tid];
    const int4* s4 = reinterpret_cast<const int4*>(s);
    int4* d4 = reinterpret_cast<int4*>(d);
    // up to 7 leading vectors reach a 128-byte destination line, so every
    // warp of the main loop writes (and, src == dst mod 16, reads) whole
    // lines: a misaligned chunk start costs partial-line traffic in one
    // tile only (loaded first, stored last, like the byte peel)
    const uint64_t pre = min(nvec, (uint64_t)(((128u - ((uintptr_t)d & 127u)) & 127u) >> 4));
    const bool pv = tid < pre;
    int4 pvec;
    if (pv) pvec = MUTABLE ? ld16_cg(s4 + tid) : ld16_nc(s4 + tid);
    s4 += pre;
    d4 += pre;
    const uint64_t nmain = nvec - pre;
    const uint64_t step = (uint64_t)nt * UNROLL;
    uint64_t i = tid;
    for (; i + (uint64_t)(UNROLL - 1) * nt < nmain; i += step) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = MUTABLE ? ld16_cg(s4 + i + u * nt) : ld16_nc(s4 + i + u * nt);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) st16(d4 + i + u * nt, v[u]);
    }
    // the remainder (< UNROLL vectors per thread) as ONE round, every load
    // before any store (loads clamped to the last vector, stores predicated):
    // a tile that is not a multiple of UNROLL x 16 x threads bytes — every
    // tile cut from an unaligned chunk — otherwise ended in up to UNROLL-1
    // serial load -> store round trips on a few threads, and the last tile
    // of a table set the kernel's end (+1.7 us at 128 MiB over 9 chunks)
    if (i < nmain) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint64_t k = min(i + (uint64_t)u * nt, nmain - 1);
        v[u] = MUTABLE ? ld16_cg(s4 + k) : ld16_nc(s4 + k);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (i + (uint64_t)u * nt < nmain) st16(d4 + i + u * nt, v[u]);
    }
    if (pv) st16(d4 - pre + tid, pvec);
    if (hv) dst[tid] = hb;
    if (tv) dst[done + tid] = tb;
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

// A wait timed out: record the code on the device and in host memory (the
// host checks the mapped word before every send, so the error is sticky
// until mp_sync clears it).  The first error wins.
__device__ __forceinline__ void raise_error(Ctl* ctl, unsigned code) {
  if (atomicCAS(&ctl->error, 0u, code) == 0u && ctl->herr) {
    *(volatile unsigned*)ctl->herr = code;
    __threadfence_system();
  }
}

// A wait gives up at the limit, or at once when another wait of this device
// already failed (every later wait would time out behind it).
__device__ __forceinline__ bool wait_expired(const Ctl* ctl, uint64_t t0) {
  const uint64_t lim = ctl->timeout_ns ? ctl->timeout_ns : kWaitTimeoutNs;
  return globaltimer() - t0 > lim || *(volatile const unsigned*)&ctl->error != 0u;
}

// ---------------------------------------------------------------------------
// TMA bulk path: cp.async.bulk global -> shared -> global through a ring of
// `stages` shared-memory blocks, driven by one thread; completion of each load
// is tracked by an mbarrier (complete_tx), reuse of a stage by bulk-group
// read completion.  The body must be 16-byte aligned on both sides.
// ---------------------------------------------------------------------------
struct TmaRing {
  uint8_t* buf;         // stages * block bytes of dynamic shared memory
  uint64_t* bar;        // one mbarrier per stage
  uint32_t phase;       // bit s = parity to wait for on stage s
  uint32_t stages;
  uint32_t block;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load(void* smem, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store(void* gdst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Acquire-wait on a hop2 tile's flag; the last hop2 tile of the chunk to pass
// re-arms flag and pass counter so a cached graph replays without a memset.
// Returns false on a timeout: the caller skips the tile (staging is never
// copied unsignalled — the destination keeps its old bytes) and leaves the
// flag state for mp_sync to re-zero.
__device__ __forceinline__ bool wait_tile_flag(const Tile& t, Ctl* ctl) {
  const uint64_t t0 = globaltimer();
  const bool gpu = t.flags & TILE_SCOPE_GPU;
  while ((gpu ? ld_acquire_gpu(t.wait) : ld_acquire_sys(t.wait)) < t.wait_count) {
    if (wait_expired(ctl, t0)) {
      raise_error(ctl, 1u);
      return false;
    }
    __nanosleep(64);
  }
  if (atomicAdd(t.pass, 1u) + 1u == t.pass_count) {
    *(volatile uint32_t*)t.pass = 0u;
    *(volatile uint32_t*)t.wait = 0u;
  }
  return true;
}

// A tile's completion signal is ONE system-scope release reduction by thread
// 0 after the CTA barrier (VEC) or after the bulk stores completed and
// fence.proxy.async (TMA): bar.sync orders every thread's stores before thread
// 0's release, and release is cumulative, so an acquirer that observes the
// flag observes the tile (the libcu++ pattern of __syncthreads + a
// memory_order_release store at thread_scope_system).  No separate
// fence.sc.sys: it cost ~9% of relay throughput (tools/exp_relay.py).
__device__ __forceinline__ void release_signal(uint32_t* sig) {
  red_release_sys_add(sig, 1u);
}

// Completion signal of a tile, by mode (sig_bytes): 0 = +1 on a u32 flag at
// system scope, kSigGpu = +1 at GPU scope (TILE_SCOPE_GPU), else +bytes on a
// u64 byte counter (TILE_SIGNAL_BYTES, group mode).
constexpr uint64_t kSigGpu = ~0ull;
__device__ __forceinline__ void signal_tile(uint32_t* sig, uint64_t mode) {
  if (mode == 0) {
    release_signal(sig);
  } else if (mode == kSigGpu) {
    red_release_gpu_add(sig, 1u);
  } else {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(sig), "l"(mode) : "memory");
  }
}

__device__ __forceinline__ uint64_t sig_bytes(const Tile& t) {
  return (t.flags & TILE_SIGNAL_BYTES) ? t.len : (t.flags & TILE_SCOPE_GPU) ? kSigGpu : 0ull;
}

// Bytes [lo, hi) of the 16-byte vector v to d[lo..hi) (d 16-byte aligned).
__device__ __forceinline__ void st_bytes16(uint8_t* d, const int4& v, unsigned lo, unsigned hi) {
  const unsigned w[4] = {(unsigned)v.x, (unsigned)v.y, (unsigned)v.z, (unsigned)v.w};
#pragma unroll
  for (unsigned j = 0; j < 16; ++j)
    if (j >= lo && j < hi) d[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
}

// hop2 of a roundtrip: the slot's bytes read back from host memory as
// whole aligned 16-byte vectors (one request shape per line, every load of
// the thread before its stores), stored to dst clipped to the chunk.  A
// chunk's unaligned head / tail as separate byte loads measured up to
// +1.5 us per 4 MiB message (33-492-byte chunks vs 4-9-byte ones).
template <int UNROLL>
__device__ __forceinline__ void hop2_vectors(const uint8_t* s, uint8_t* d, uint64_t len, unsigned tid,
                                             unsigned nt) {
  const uint64_t lead = (uintptr_t)s & 15u;
  const int4* s4 = reinterpret_cast<const int4*>(s - lead);
  uint8_t* d0 = d - lead;  // 16-byte aligned: d == s mod 16
  const uint64_t nv = (lead + len + 15) >> 4, end = lead + len;
  for (uint64_t base = 0; base < nv; base += (uint64_t)nt * UNROLL) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t k = base + tid + (uint64_t)u * nt;
      if (k < nv) v[u] = ld16_cg(s4 + k);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t k = base + tid + (uint64_t)u * nt;
      if (k >= nv) continue;
      const uint64_t b = k << 4;
      if (b >= lead && b + 16 <= end) st16(d0 + b, v[u]);
      else st_bytes16(d0 + b, v[u], b < lead ? (unsigned)(lead - b) : 0u,
                      b + 16 <= end ? 16u : (unsigned)(end - b));
    }
  }
}

// A TILE_ROUNDTRIP tile by threads [tid0, tid0 + nt) of the CTA: hop1 into
// the staging slot (the source lines around the chunk, so the PCIe writes
// are whole lines; wait_count / pass_count = bytes before / after it), a barrier over exactly those threads (named barrier
// `bar`, or the CTA barrier when bar == 0), hop2 out of it with L2 loads.
// `fence`: a system-scope fence after hop2.  hop2 has read back every line
// hop1 wrote (a PCIe read does not pass an earlier posted write), so the
// fence is cheap here — and it retires the CTA's host writes early instead
// of leaving them to the grid-completion flush, which queues behind any
// saturating H2D DMA (an e2e window's 512 MiB upload: +20 us per 512 MiB
// message, sends 11.5 -> 10.3 ms per window) and that a programmatic-
// dependent next launch waits for (~0.7 us).  Dynamic tables (large
// messages, roundtrips far off the critical path) fence; the static TMA
// table's helper warps fence when the tile carries TILE_FENCE (programs
// from 20 MiB; below, the roundtrip is the message's tail and the fence
// adds to it: 8 MiB 0.82 -> 0.65 of single path).
template <int UNROLL>
__device__ __forceinline__ void roundtrip(const Tile& t, unsigned tid, unsigned nt, unsigned bar,
                                          unsigned long long* trace, bool lead, bool fence) {
  // hop1 widened by wait_count / pass_count bytes (whole host lines)
  copy_range<UNROLL, false>((const uint8_t*)t.src - t.wait_count, t.stage - t.wait_count,
                            t.len + t.wait_count + t.pass_count, tid, nt);
  if (bar) asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory");
  else __syncthreads();
  if (lead && trace) {
    atomicMax(&trace[2 * t.node + 1], (unsigned long long)globaltimer());
    atomicMin(&trace[2 * (t.node + 1)], (unsigned long long)globaltimer());
  }
  if ((((uintptr_t)t.stage ^ (uintptr_t)t.dst) & 15u) == 0)
    hop2_vectors<(UNROLL > 4 ? 4 : UNROLL)>(t.stage, (uint8_t*)t.dst, t.len, tid, nt);
  else
    copy_range<UNROLL, true>(t.stage, (uint8_t*)t.dst, t.len, tid, nt);
  if (fence) __threadfence_system();
}

// Group barrier prologue (thread 0 of every CTA) with the 4 s safety timeout.
__device__ __forceinline__ void group_wait(const GroupSync& g, Ctl* ctl) {
  if (g.n == 0) return;
  const uint32_t want = *(volatile uint32_t*)g.seq;
  const uint64_t t0 = globaltimer();
  for (int q = 0; q < g.n; ++q)
    while (ld_acquire_sys(g.gen[q]) < want) {
      if (wait_expired(ctl, t0)) {
        raise_error(ctl, 2u);
        return;
      }
      __nanosleep(128);
    }
}

__device__ __forceinline__ void group_done(const GroupSync& g) {
  if (g.n == 0) return;
  *(volatile uint32_t*)g.seq = *(volatile uint32_t*)g.seq + 1u;
  release_signal(g.self_gen);
}

// Trace stamps (trace mode only): per logical node, the first tile start and
// the last tile completion in %globaltimer ns (array pre-set to {max, 0}).
__device__ __forceinline__ void trace_start(unsigned long long* tr, uint32_t node) {
  if (tr) atomicMin(&tr[2 * node], (unsigned long long)globaltimer());
}
__device__ __forceinline__ void trace_end(unsigned long long* tr, uint32_t node) {
  if (tr) atomicMax(&tr[2 * node + 1], (unsigned long long)globaltimer());
}

// Per-stage bookkeeping of the TMA block stream.
struct BlockMeta {
  uint8_t* dst;
  uint32_t bytes;
  uint32_t node_end;  // node + 1 on a tile's last block (trace mode), else 0
  uint32_t* signal;   // set on a tile's last block when the tile signals
  uint64_t sig_bytes; // 0: +1 on a u32 flag; else +bytes on a u64 counter
};

// The TMA engine: thread 0 streams 16-byte-aligned tile bodies through the
// shared-memory ring as ONE continuous block sequence that spans tiles, so the
// ring stays full across tile boundaries (no per-tile drain).  Loads run up to
// `stages` blocks ahead of stores; stage s is refilled once the store that
// last used it has read shared memory (bulk-group .read completion, lagging
// one store).  Tiles that must wait on a relay flag, or whose src/dst disagree
// mod 16, drain the stream first (a waited-on hop1 tile may be one this CTA
// still holds); misaligned tiles are handed back to the whole CTA.
// Returns 0 when the tile table is exhausted, 1 with *coop = a tile for the CTA.
struct TmaEngine {
  TmaRing r;
  BlockMeta* meta;
  const Tile* tiles;
  unsigned ntiles;
  Ctl* ctl;
  unsigned next_claim;
  unsigned long long* trace;
  // loader cursor
  const uint8_t* ls = nullptr;
  uint8_t* ld = nullptr;
  uint64_t lrem = 0;
  uint32_t* lsig = nullptr;
  uint64_t lsig_bytes = 0;
  uint32_t lnode_end = 0;
  int blocked = -1;  // -1 none, 0 table exhausted, 1 misaligned tile, 2 flag wait
  bool peel_help = false;  // all-static table, CTA >= 64 threads: warps 1.. copy plain tiles' peels
  Tile pending;
  uint64_t g_load = 0, g_store = 0;

  __device__ void start_tile(const Tile& t) {
    const uint8_t* src = (const uint8_t*)t.src;
    uint8_t* dst = (uint8_t*)t.dst;
    const bool mut = t.flags & TILE_SRC_MUTABLE;
    uint64_t head = (16u - ((uintptr_t)dst & 15u)) & 15u;
    if (head > t.len) head = t.len;
    const uint64_t body = (t.len - head) & ~(uint64_t)15;
    const uint64_t tail_at = head + body;
    const uint64_t tail = t.len - tail_at;
    trace_start(trace, t.node);
    // a static table's plain tile leaves its peel to warps 1.. (kernel
    // prologue), so no scalar load latency precedes the bulk stream
    if ((head | tail) && !(peel_help && !t.signal)) {  // < 16 + 16 bytes: every load before any store
      uint8_t hb[15], tb[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) {
        if ((uint64_t)k < head) hb[k] = mut ? *(volatile const uint8_t*)(src + k) : src[k];
        if ((uint64_t)k < tail)
          tb[k] = mut ? *(volatile const uint8_t*)(src + tail_at + k) : src[tail_at + k];
      }
#pragma unroll
      for (int k = 0; k < 15; ++k) {
        if ((uint64_t)k < head) dst[k] = hb[k];
        if ((uint64_t)k < tail) dst[tail_at + k] = tb[k];
      }
    }
    if (body == 0) {
      trace_end(trace, t.node);  // stamped before the release: hop2 cannot precede it
      if (t.signal) signal_tile(t.signal, sig_bytes(t));
      return;
    }
    if (mut) fence_proxy_async();  // staged bytes were written by the generic proxy
    ls = src + head;
    ld = dst + head;
    lrem = body;
    lsig = t.signal;
    lsig_bytes = sig_bytes(t);
    lnode_end = trace ? t.node + 1 : 0;
  }

  // Make the loader cursor non-empty; false when blocked.  Claims run two
  // deep: when tile k starts, tile k+1's descriptor is already in registers
  // (`ahead`, loaded at the previous fetch) and the atomic for k+2 is issued
  // now but only consumed at the next fetch — neither latency is exposed.
  Tile ahead;
  unsigned claim2;
  unsigned nstatic;  // tiles [0, nstatic) go to CTA blockIdx.x without a claim
  unsigned* ctr;  // this launch's claim counter (thread 0)
  __device__ unsigned claim() {
    return nstatic >= ntiles ? ntiles : atomicAdd(ctr, 1u) + nstatic;
  }
  __device__ void prime() {
    next_claim = blockIdx.x < nstatic ? blockIdx.x : claim();
    claim2 = claim();
    if (next_claim < ntiles) ahead = tiles[next_claim];
  }
  __device__ bool fetch() {
    while (lrem == 0) {
      if (blocked >= 0) return false;
      const unsigned w = next_claim;
      if (w >= ntiles) {
        blocked = 0;
        return false;
      }
      const Tile t = ahead;
      next_claim = claim2;
      claim2 = next_claim < ntiles ? claim() : ntiles;
      if (next_claim < ntiles) ahead = tiles[next_claim];
      const bool aligned = (((uintptr_t)t.src ^ (uintptr_t)t.dst) & 15u) == 0;
      if (t.wait || !aligned || (t.flags & TILE_ROUNDTRIP)) {  // roundtrips: the whole CTA
        pending = t;
        blocked = t.wait ? 2 : 1;
        return false;
      }
      start_tile(t);
    }
    return true;
  }

  __device__ bool issue_load() {
    if (!fetch()) return false;
    const uint32_t n = (uint32_t)(lrem < r.block ? lrem : r.block);
    const uint32_t s = (uint32_t)(g_load % r.stages);
    meta[s] = BlockMeta{ld, n, lrem == n ? lnode_end : 0u, lrem == n ? lsig : nullptr, lsig_bytes};
    mbar_expect_tx(&r.bar[s], n);
    tma_load(r.buf + (size_t)s * r.block, ls, n, &r.bar[s]);
    ls += n;
    ld += n;
    lrem -= n;
    ++g_load;
    return true;
  }

  __device__ int run(Tile* coop) {
    for (;;) {
      const uint64_t seg = g_store;  // every stage is free here
      for (uint32_t i = 0; i < r.stages && issue_load(); ++i) {
      }
      while (g_store < g_load) {
        const uint32_t s = (uint32_t)(g_store % r.stages);
        mbar_wait(&r.bar[s], (r.phase >> s) & 1u);
        r.phase ^= 1u << s;
        tma_store(meta[s].dst, r.buf + (size_t)s * r.block, meta[s].bytes);
        bulk_commit();
        const uint64_t b = g_store++;
        if (meta[s].signal || meta[s].node_end) {  // tile complete: its bytes land first
          bulk_wait_all();
          fence_proxy_async();
          if (meta[s].node_end) trace_end(trace, meta[s].node_end - 1);
          if (meta[s].signal) signal_tile(meta[s].signal, meta[s].sig_bytes);
        }
        if (b > seg) {  // refill the stage of block b-1 once its store has read smem
          bulk_wait_read<1>();
          issue_load();
        }
      }
      bulk_wait_read<0>();
      if (blocked == 0) return 0;
      const Tile t = pending;
      const int why = blocked;
      blocked = -1;
      if (t.wait && !wait_tile_flag(t, ctl)) continue;  // timed out: skip, never copy staging
      if (why == 1 || (((uintptr_t)t.src ^ (uintptr_t)t.dst) & 15u) != 0 || (t.flags & TILE_ROUNDTRIP)) {
        *coop = t;
        return 1;
      }
      start_tile(t);
    }
  }
};

// ---------------------------------------------------------------------------
// Small-message kernel.  Back-to-back launches on one stream complete in
// ~2.05 us "slots" (tools/kexp.cu: an empty kernel takes one slot, a kernel
// whose body runs >~0.7 us takes two).  A small message therefore has a
// budget of about one L2 round trip: its descriptor comes from the kernel
// parameters (constant bank, no dependent global load), every thread issues
// all its 16-byte loads before any store, and there is no shared memory, no
// barrier, no claim and no exit protocol.  Used for static tables of direct
// tiles only (no flags, no host memory), one tile per CTA.
//
// Programmatic dependent launch: the "slots" are a property of ordinary
// stream-ordered launches (one-kernel graph replays and plain launches
// alike retire in 2.048 us quanta on B200).  Launched with programmatic
// stream serialization (engine option pdl) the next send's kernel is
// processed while this one runs and back-to-back sends cost ~1.9 us up to
// 2 MiB (tools/pdl_probe.cu).  Stream order is kept on the device:
// griddepcontrol.wait (before ANY global access) returns once the previous
// grid has completed and its memory is visible — a no-op for a normal
// launch — and each CTA allows the dependent launch only after its stores
// are issued (an early trigger leaves the dependent's waiting CTAs resident
// beside a long body: 4 MiB 5.9 vs 2.5 us).
// ---------------------------------------------------------------------------
constexpr unsigned kSmallMaxTiles = 148;
template <unsigned N>
struct SmallTable {
  uint64_t src[N];
  uint64_t dst[N];
  uint32_t len[N];
};
// Parameter block sizes: a launch copies its parameters, so tables of up to
// 16 tiles (messages <= 64 KiB at 4 KiB tiles) use a 320-byte block.
constexpr unsigned kSmallTilesLo = 16;

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int V>
__device__ __forceinline__ void small_copy_body(uint64_t src_addr, uint64_t dst_addr, uint32_t len) {
  const uint8_t* src = (const uint8_t*)src_addr;
  uint8_t* dst = (uint8_t*)dst_addr;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  if ((((uintptr_t)src ^ (uintptr_t)dst) & 15u) != 0) {
    copy_range<4, false>(src, dst, len, threadIdx.x, blockDim.x);
    return;
  }
  uint32_t head = (16u - ((uint32_t)(uintptr_t)dst & 15u)) & 15u;
  if (head > len) head = len;
  const uint32_t nvec = (len - head) >> 4;
  const uint32_t tail_at = head + (nvec << 4);
  const int4* s4 = reinterpret_cast<const int4*>(src + head);
  int4* d4 = reinterpret_cast<int4*>(dst + head);
  const bool hv = tid < head, tv = tid < len - tail_at;
  uint8_t hb = 0, tb = 0;
  if (hv) hb = src[tid];
  if (tv) tb = src[tail_at + tid];
  for (uint32_t base = tid; base < nvec; base += V * nt) {
    int4 v[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (base + k * nt < nvec) v[k] = ld16_nc(s4 + base + k * nt);
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (base + k * nt < nvec) st16(d4 + base + k * nt, v[k]);
  }
  if (hv) dst[tid] = hb;
  if (tv) dst[tail_at + tid] = tb;
}

template <int V, unsigned N>
__global__ void __launch_bounds__(256) small_copy_kernel(const __grid_constant__ SmallTable<N> tab) {
  griddep_wait();
  small_copy_body<V>(tab.src[blockIdx.x], tab.dst[blockIdx.x], tab.len[blockIdx.x]);
  griddep_launch_dependents();
}

// Time base of a traced send: %globaltimer at the fork point of this device.
__global__ void stamp_kernel(unsigned long long* out) { *out = globaltimer(); }

// (LDG/STG at 4 CTAs x 256 threads per SM: 76 registers, 3 CTAs resident,
// the 4th wave claims what is left.  Forcing 4 resident CTAs (64 registers,
// spills) measured 174 vs 161 us at 512 MiB.)
template <int KIND, int UNROLL>
__global__ void __launch_bounds__(256) transfer_kernel(const Tile* __restrict__ tiles,
                                                       unsigned ntiles, Ctl* ctl,
                                                       unsigned stages, unsigned block,
                                                       unsigned nstatic,
                                                       unsigned long long* trace,
                                                       GroupSync gsync, Sched* sched,
                                                       unsigned nhelp) {
  // programmatic dependent launch (static tables, engine option pdl): no
  // global access before the previous grid has completed (a no-op otherwise)
  griddep_wait();
  // Helper tiles (TMA kernel, static tables only): the last `nhelp` tiles are
  // host-path tiles worked by warps 1.. of CTA (j mod gridDim.x) while thread
  // 0 streams the CTA's own tile through the TMA ring — PCIe latency overlaps
  // the HBM/NVLink stream inside one launch, and the table stays static.
  ntiles -= nhelp;
  // Tiles [0, nstatic) (a prefix with no flag waits, nstatic <= gridDim.x) are
  // taken by CTA blockIdx.x without a claim; the rest are claimed dynamically.
  // A fully static table (nstatic == ntiles: one tile per CTA, no waits) runs
  // with no atomics and no exit protocol at all: the control block is
  // untouched, so a small message costs one launch and one copy.
  const bool all_static = nstatic >= ntiles && gsync.n == 0;
  // per-program counters (no exit protocol) unless a group barrier needs the
  // last CTA anyway; thread 0 takes its arrival ticket here
  const bool use_sched = sched != nullptr && gsync.n == 0 && !all_static;
  unsigned* ctr = &ctl->work;
  if (threadIdx.x == 0 && use_sched) {
    const unsigned long long a = atomicAdd(&sched->arrive, 1ull);
    const unsigned long long launch = a / gridDim.x;
    if (a % gridDim.x == 0) sched->work[(launch + 1) & 1] = 0u;
    ctr = &sched->work[launch & 1];
  }
  __shared__ Tile s_tile;
  __shared__ int s_cmd;
  __shared__ uint64_t s_bar[16];
  __shared__ BlockMeta s_meta[16];
  extern __shared__ __align__(128) uint8_t s_ring[];
  if (threadIdx.x == 0) group_wait(gsync, ctl);
  __syncthreads();
  if (KIND == 1) {
    // ---- TMA: thread 0 streams; the CTA helps only with misaligned tiles ----
    TmaEngine eng{TmaRing{s_ring, s_bar, 0u, stages, block}, s_meta, tiles, ntiles, ctl, 0u,
                  trace};
    eng.nstatic = nstatic;
    eng.ctr = ctr;
    eng.peel_help = all_static && blockDim.x >= 64;
    if (threadIdx.x == 0) {
      for (unsigned s = 0; s < stages; ++s) mbar_init(&s_bar[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      eng.prime();
    }
    if (threadIdx.x >= 32) {
      // warps 1..: (a) the unaligned head / tail bytes (< 16 each) of this
      // CTA's own plain tile, loaded first and stored last, while thread 0
      // streams its 16-byte-aligned body; (b) the helper tiles of this CTA
      const unsigned htid = threadIdx.x - 32, hnt = blockDim.x - 32;
      uint8_t* peel_dst = nullptr;
      uint8_t peel = 0;
      if (all_static && blockIdx.x < ntiles) {
        const Tile t = tiles[blockIdx.x];
        if (!t.signal && (((uintptr_t)t.src ^ (uintptr_t)t.dst) & 15u) == 0) {
          uint64_t head = (16u - ((uintptr_t)t.dst & 15u)) & 15u;
          if (head > t.len) head = t.len;
          const uint64_t tail_at = head + ((t.len - head) & ~(uint64_t)15);
          uint64_t o = ~0ull;
          if (htid < head) o = htid;
          else if (htid >= 16 && htid - 16 < t.len - tail_at) o = tail_at + htid - 16;
          if (o != ~0ull) {
            peel = ((const uint8_t*)t.src)[o];
            peel_dst = (uint8_t*)t.dst + o;
          }
        }
      }
      for (unsigned j = blockIdx.x; j < nhelp; j += gridDim.x) {
        const Tile t = tiles[ntiles + j];
        if (htid == 0) trace_start(trace, t.node);
        if (t.flags & TILE_ROUNDTRIP) {
          roundtrip<UNROLL>(t, htid, hnt, 1, trace, htid == 0, (t.flags & TILE_FENCE) != 0);
          asm volatile("bar.sync 1, %0;" ::"r"(hnt) : "memory");
          if (htid == 0) trace_end(trace, t.node + 1);
        } else {  // hop1 to host memory (the destination GPU's kernel runs hop2)
          copy_range<UNROLL, false>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len, htid, hnt);
          asm volatile("bar.sync 1, %0;" ::"r"(hnt) : "memory");
          if (htid == 0) {
            trace_end(trace, t.node);
            if (t.signal) signal_tile(t.signal, sig_bytes(t));
          }
        }
      }
      if (peel_dst) *peel_dst = peel;
    }
    for (;;) {
      if (threadIdx.x == 0) {
        s_cmd = eng.run(&s_tile);
        if (s_cmd) trace_start(trace, s_tile.node);
      }
      __syncthreads();
      if (s_cmd == 0) break;
      const Tile& t = s_tile;
      const bool rt = t.flags & TILE_ROUNDTRIP;
      if (rt)
        roundtrip<UNROLL>(t, threadIdx.x, blockDim.x, 0, trace, threadIdx.x == 0, true);
      else if (t.flags & TILE_SRC_MUTABLE)
        copy_range<UNROLL, true>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len, threadIdx.x, blockDim.x);
      else
        copy_range<UNROLL, false>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len, threadIdx.x, blockDim.x);
      __syncthreads();  // every thread's stores precede the release
      if (threadIdx.x == 0) {
        trace_end(trace, rt ? t.node + 1 : t.node);
        if (t.signal) signal_tile(t.signal, sig_bytes(t));
      }
    }
    // smem must outlive the last bulk store's reads; its global writes are
    // complete at grid completion (tiles that signal waited for them above)
    if (threadIdx.x == 0) bulk_wait_read<0>();
  } else {
    // ---- vector LDG/STG: the whole CTA copies each claimed tile ----
    // Control is pipelined off the copy's critical path: thread 0 loads the
    // NEXT tile's descriptor (claimed one tile earlier) into registers before
    // copying its share of the current tile, and the completion signal of a
    // tile (a system-scope release, which stalls its thread until the tile's
    // stores are visible) is issued by thread 32 (second warp) at the start of
    // the next tile while the other warps already copy — or by thread 0 before
    // it waits on a flag, so a CTA never holds back a signal while it waits.
    // Two barriers per tile.
    __shared__ Tile s_tiles[2];
    __shared__ unsigned s_w[2];
    __shared__ int s_skip;  // the tile's flag wait timed out: skip it
    const unsigned sig_tid = blockDim.x > 32 ? 32u : 0u;  // a thread of the second warp
    unsigned c1 = ntiles;  // thread 0: claim of the tile after the next one
    if (threadIdx.x == 0) {
      const unsigned w0 = blockIdx.x < nstatic ? blockIdx.x
                                               : (all_static ? ntiles : atomicAdd(ctr, 1u) + nstatic);
      s_w[0] = w0;
      if (w0 < ntiles) {
        s_tiles[0] = tiles[w0];
        c1 = all_static ? ntiles : atomicAdd(ctr, 1u) + nstatic;
      }
    }
    __syncthreads();
    unsigned slot = 0;
    uint32_t* pend_sig = nullptr;  // thread 32: the previous tile's signal
    uint64_t pend_bytes = 0;
    uint32_t pend_node = 0;
    bool pend = false;
    while (s_w[slot] < ntiles) {
      const Tile t = s_tiles[slot];
      Tile next{};
      unsigned wn = ntiles;
      if (threadIdx.x == 0) {
        wn = c1;
        if (wn < ntiles) {
          next = tiles[wn];  // in flight during the copy below
          c1 = all_static ? ntiles : atomicAdd(ctr, 1u) + nstatic;
        }
        if (t.wait) {
          // release the previous tile BEFORE waiting: the flag may be its own
          if (pend) {
            trace_end(trace, pend_node);
            if (pend_sig) signal_tile(pend_sig, pend_bytes);
          }
          s_skip = !wait_tile_flag(t, ctl);
        }
        trace_start(trace, t.node);
      }
      __syncthreads();  // B1: the tile's flag wait is done
      if (threadIdx.x == sig_tid && pend && !t.wait) {  // deferred completion of the previous tile
        trace_end(trace, pend_node);
        if (pend_sig) signal_tile(pend_sig, pend_bytes);
      }
      const bool skip = t.wait && s_skip;  // s_skip is only written for waiting tiles
      if (skip) {
      } else if (t.flags & TILE_ROUNDTRIP)  // <= 64 KiB, latency-bound: a narrow unroll (no spills)
        roundtrip<4>(t, threadIdx.x, blockDim.x, 0, trace, threadIdx.x == 0, true);
      else if (t.flags & TILE_SRC_MUTABLE)
        copy_range<UNROLL, true>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len, threadIdx.x, blockDim.x);
      else
        copy_range<UNROLL, false>((const uint8_t*)t.src, (uint8_t*)t.dst, t.len, threadIdx.x, blockDim.x);
      if (threadIdx.x == 0) {
        s_tiles[slot ^ 1u] = next;
        s_w[slot ^ 1u] = wn;
      }
      __syncthreads();  // B2: every store of the tile precedes its (deferred) release
      pend = true;
      pend_sig = skip ? nullptr : t.signal;  // a skipped tile never reports bytes
      pend_bytes = sig_bytes(t);
      pend_node = (t.flags & TILE_ROUNDTRIP) ? t.node + 1 : t.node;
      slot ^= 1u;
    }
    if (threadIdx.x == sig_tid && pend) {
      trace_end(trace, pend_node);
      if (pend_sig) signal_tile(pend_sig, pend_bytes);
    }
  }
  if (threadIdx.x == 0 && !all_static && !use_sched) {
    __threadfence();
    if (atomicAdd(&ctl->exit, 1u) + 1u == gridDim.x) {  // last CTA re-arms the counters
      ctl->work = 0u;
      ctl->exit = 0u;
      ctl->launches += 1u;
      __threadfence();
      group_done(gsync);
    }
  }
  griddep_launch_dependents();
}

// Receiver side of a group transfer: wait until `expected` bytes have landed
// (direct and hop2 tiles add their sizes to *done), re-arm, finish the barrier.
// ONE thread does the protocol (the kernels launch as one warp): with every
// thread of the warp in it, each bumped this rank's generation — 32 per
// transfer — so a sender ran ahead and its bytes landed before the previous
// wait re-armed the counter (a back-to-back timeout found in round 2,
// tests/test_gpu_group.py::test_group_back_to_back_transfers).
__global__ void group_recv_kernel(GroupSync gsync, unsigned long long* done,
                                  unsigned long long expected, Ctl* ctl) {
  if (threadIdx.x != 0) return;
  group_wait(gsync, ctl);
  const uint64_t t0 = globaltimer();
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(done) : "memory");
    if (v >= expected) break;
    if (wait_expired(ctl, t0)) {
      raise_error(ctl, 3u);
      break;
    }
    __nanosleep(128);
  }
  *(volatile unsigned long long*)done = 0ull;
  __threadfence_system();
  group_done(gsync);
}

// A rank with no part in a group transfer still takes part in its barrier.
__global__ void group_noop_kernel(GroupSync gsync, Ctl* ctl) {
  if (threadIdx.x != 0) return;  // one thread: one generation bump per transfer
  group_wait(gsync, ctl);
  group_done(gsync);
}

}  // namespace mpk
