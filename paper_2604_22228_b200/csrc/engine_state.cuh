// engine_state.cuh — internal to mp_engine.cu (included once, in order):
// kernel launch policy, the context's physical/logical devices, cached
// entries (programs + copy-engine ops), group-mode state, and the arenas
// (relay staging, flags, pinned host staging) that programs point into.
#pragma once

namespace {

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw Error{MP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)};     \
  } while (0)

using KernelFn = void (*)(const mpk::Tile*, unsigned, mpk::Ctl*, unsigned, unsigned, unsigned,
                          unsigned long long*, mpk::GroupSync, mpk::Sched*, unsigned);

KernelFn pick_kernel(const mp_engine_opts& o) {
  if (o.copy_kind == MP_COPY_TMA) return mpk::transfer_kernel<1, 8>;
  switch (o.unroll) {
    case 4: return mpk::transfer_kernel<0, 4>;
    case 16: return mpk::transfer_kernel<0, 16>;
    default: return mpk::transfer_kernel<0, 8>;
  }
}

size_t kernel_smem(const mp_engine_opts& o) {
  return o.copy_kind == MP_COPY_TMA ? (size_t)o.tma_stages * (size_t)o.tma_block : 0;
}

// Kernel choice per tile table (measured, tools/abi_latency.cu, loopback):
//  * PROG_SMALL       static table <= small_max_bytes of plain direct tiles:
//                     small_copy_kernel, descriptors in the kernel parameters
//                     (one ~2 us launch slot up to 64 KiB);
//  * PROG_STATIC_TMA  static table (one tile per CTA, <= kStaticMaxPerCta):
//                     the TMA ring kernel, 1 CTA x 128 threads per SM, no
//                     claims and no exit protocol (16-64 MiB: 10% ahead);
//  * PROG_DYNAMIC     everything else: the configured kernel with atomic tile
//                     claims — by default the 16-byte LDG/STG kernel at
//                     4 CTAs x 256 threads per SM over 64 KiB tiles, which
//                     copies 512 MiB at 100% of the measured HBM peak (the TMA
//                     ring, copy_kind = MP_COPY_TMA, reaches 98%).
// Tables that touch another GPU's memory never run TMA unless tma_peer allows
// it (TMA bulk copies on peer addresses are unverified on this 1-GPU pool).
enum ProgKind { PROG_DYNAMIC = 0, PROG_STATIC_TMA = 1, PROG_SMALL = 2 };
// Small-message tables from this size launch with programmatic dependent
// launch when opts.pdl is set (see pdl_replay in mp_engine.cu).
constexpr uint64_t kPdlMinBytesDefault = 1 << 20;
inline uint64_t pdl_min_bytes() {  // MP_PDL_MIN: experiments only
  static const uint64_t v = [] {
    const char* e = std::getenv("MP_PDL_MIN");
    return e ? (uint64_t)std::strtoull(e, nullptr, 10) : kPdlMinBytesDefault;
  }();
  return v;
}
constexpr int kPeerCtasPerSm = 4;
constexpr uint64_t kVecTileBytes = 64 << 10;
// ... and of GPU-relay hops on it (lowering.cuh lower_relay)
constexpr uint64_t kRelayTileBytes = 128 << 10;
bool tma_ok(const mp_engine_opts& o, bool peer) {
  return !(o.tma_peer < 0 || (peer && o.tma_peer == 0));
}
bool vec_peer(const mp_engine_opts& o, bool peer) { return o.copy_kind == MP_COPY_TMA && !tma_ok(o, peer); }

// Raise a kernel's dynamic shared-memory limit on the current device once
// (cudaFuncSetAttribute costs microseconds; a per-launch call would dominate
// a small message's host time).
void allow_smem(KernelFn fn, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, KernelFn>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{dev, fn}];
  if (have >= smem) return;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  have = smem;
}

// Which kernel launch_transfer runs for a table (MP_KERNEL_*, untraced).
int kernel_of(const mp_engine_opts& o, int kind, bool peer) {
  if (kind == PROG_SMALL) return MP_KERNEL_SMALL;
  if (kind != PROG_DYNAMIC) return tma_ok(o, peer) ? MP_KERNEL_TMA : MP_KERNEL_VEC;
  if (vec_peer(o, peer)) return MP_KERNEL_VEC;
  return o.copy_kind == MP_COPY_TMA ? MP_KERNEL_TMA : MP_KERNEL_VEC;
}

// Launch the transfer kernel (mp_kernels.cuh) over one tile table.
// `nstatic` > 0 only for tables without flag waits: static first tiles must
// never be waited on by another CTA (residency of every CTA is not guaranteed).
void launch_transfer(const mp_engine_opts& o_in, unsigned grid, cudaStream_t s, const mpk::Tile* tiles,
                     unsigned ntiles, mpk::Ctl* ctl, unsigned nstatic,
                     unsigned long long* trace = nullptr, const mpk::GroupSync* gsync = nullptr,
                     bool peer = false, int sms = 148, const mpk::SmallTable<mpk::kSmallMaxTiles>* small = nullptr,
                     int kind = PROG_DYNAMIC, mpk::Sched* sched = nullptr, unsigned nhelp = 0) {
  if (kind == PROG_SMALL && small && !trace && !gsync) {
    // programmatic dependent launch (opts.pdl) from kPdlMinBytes: the kernel
    // waits on griddepcontrol before any memory access, so stream order holds
    uint64_t bytes = 0;
    for (unsigned i = 0; i < ntiles; ++i) bytes += small->len[i];
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(ntiles);
    lc.blockDim = dim3(256);
    lc.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = o_in.pdl && bytes >= pdl_min_bytes() ? 1 : 0;
    if (ntiles <= mpk::kSmallTilesLo) {
      mpk::SmallTable<mpk::kSmallTilesLo> lo;
      std::copy(small->src, small->src + ntiles, lo.src);
      std::copy(small->dst, small->dst + ntiles, lo.dst);
      std::copy(small->len, small->len + ntiles, lo.len);
      CK(cudaLaunchKernelEx(&lc, mpk::small_copy_kernel<4, mpk::kSmallTilesLo>, lo));
    } else {
      CK(cudaLaunchKernelEx(&lc, mpk::small_copy_kernel<4, mpk::kSmallMaxTiles>, *small));
    }
    return;
  }
  mp_engine_opts o = o_in;
  if (kind != PROG_DYNAMIC && tma_ok(o, peer)) {
    // static table (a traced small one too): the TMA ring, one CTA per tile
    o.copy_kind = MP_COPY_TMA;
    o.threads = 128;
  } else if (kind != PROG_DYNAMIC || vec_peer(o, peer)) {
    // LDG/STG kernel at the measured shape (tma_peer < 0 forces it: testing)
    o.copy_kind = MP_COPY_VEC;
    o.unroll = 8;
    o.threads = 256;
    grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sms * kPeerCtasPerSm);
    nstatic = nstatic ? grid : 0;
  }
  KernelFn fn = pick_kernel(o);
  size_t smem = kernel_smem(o);
  if (smem > 48 * 1024) allow_smem(fn, smem);
  mpk::GroupSync g{};
  if (gsync) g = *gsync;
  // static tables (one tile per CTA, no waits, no control block) launch with
  // programmatic dependent launch like the small-message kernel
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(o.threads);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = (o_in.pdl >= 3 || (o_in.pdl >= 2 && kind != PROG_DYNAMIC)) && !trace && !gsync ? 1 : 0;
  CK(cudaLaunchKernelEx(&lc, fn, tiles, ntiles, ctl, (unsigned)o.tma_stages, (unsigned)o.tma_block,
                        nstatic, trace, g, sched, nhelp));
}

double now_us() {
  using namespace std::chrono;
  return duration<double, std::micro>(steady_clock::now().time_since_epoch()).count();
}

// cudaSetDevice costs ~55 ns of host time even to the current device,
// cudaGetDevice ~25 ns (tools/host_api_cost.cu): switch only on a change
inline void set_device(int ordinal) {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != ordinal) CK(cudaSetDevice(ordinal));
}

struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Physical CUDA device owned by the context.
struct Phys {
  int ordinal = 0;
  int sms = 148;
  mpk::Ctl* ctl = nullptr;               // transfer-kernel control block
  unsigned* herr_dev = nullptr;          // device view of this device's sticky error word
  cudaStream_t kstream = nullptr;        // SM transfer-kernel stream
  cudaStream_t capture = nullptr;        // graph-capture origin
  std::vector<cudaStream_t> lanes;       // copy-engine lane streams
  std::vector<cudaEvent_t> events;       // handoff / fork / join events
  size_t next_event = 0;
  cudaEvent_t kt0 = nullptr, kt1 = nullptr;  // kernel timing
};

// Logical accelerator (several may map to one physical device: loopback).
struct Logi {
  int phys = 0;
  uint8_t* stage = nullptr;  // relay staging arena
  size_t stage_cap = 0;
  uint32_t* flags = nullptr;  // [flag_cap] chunk flags + [flag_cap] pass counters
  int flag_cap = 0;
};

struct CeOp {
  int phys;        // device whose lane stream runs it
  int lane;        // lane stream index on that device
  void* dst;
  const void* src;
  size_t len;      // bytes per row
  int wait_ev;     // index into the op-event list to wait on, -1 none
  int record_ev;   // index into the op-event list to record, -1 none
  uint32_t node;   // logical graph node (chunk-hop) id, for traces
  // 2-D batch: `rows` rows of `len` bytes at pitches spitch / dpitch (one
  // cudaMemcpy2DAsync moving several equal, evenly strided chunks), whose
  // logical nodes are `nodes` (traces give each the op's interval)
  size_t rows = 1, spitch = 0, dpitch = 0;
  std::vector<uint32_t> nodes;
  CeOp(int ph, int ln, void* d, const void* s, size_t n, int w, int r, uint32_t nd)
      : phys(ph), lane(ln), dst(d), src(s), len(n), wait_ev(w), record_ev(r), node(nd) {}
};

struct Program {
  int phys;
  mpk::Tile* d_tiles = nullptr;   // tile table, followed by the program's claim counters
  mpk::Sched* d_sched = nullptr;  // (same allocation)
  unsigned ntiles = 0;
  unsigned grid = 0;
  unsigned nstatic = 0;  // = grid when the table has no flag waits
  bool peer = false;     // some tile reads or writes another GPU's memory
  int kind = PROG_DYNAMIC;                 // ProgKind
  std::shared_ptr<mpk::SmallTable<mpk::kSmallMaxTiles>> small;  // PROG_SMALL: the table as kernel params
  uint64_t bytes = 0;    // PROG_SMALL: bytes the table moves
  unsigned nhelp = 0;    // PROG_STATIC_TMA: trailing host-path tiles worked by helper warps
};

// Hash of a cache key (raw bytes: pointers, sizes, devices, config; up to
// 64 transfers for a program): 8 bytes per step, a few ns per transfer —
// std::hash<std::string> costs ~1 us on a 64-transfer key.
struct KeyHash {
  size_t operator()(const std::string& k) const noexcept {
    const char* p = k.data();
    size_t n = k.size();
    uint64_t h = 0x9E3779B97F4A7C15ull ^ n;
    for (; n >= 8; p += 8, n -= 8) {
      uint64_t w;
      memcpy(&w, p, 8);
      h = (h ^ w) * 0xff51afd7ed558ccdull;
      h ^= h >> 32;
    }
    uint64_t w = 0;
    memcpy(&w, p, n);
    h = (h ^ w) * 0xc4ceb9fe1a85ec53ull;
    return (size_t)(h ^ (h >> 29));
  }
};

struct Entry {
  std::string key;
  std::vector<mp_path> paths;
  std::vector<mp_chunk> chunks;
  int nodes_logical = 0;
  std::vector<Program> progs;
  std::vector<CeOp> ce;
  std::vector<int> ev_phys;  // device of each op event
  int src_phys = 0;
  cudaGraphExec_t exec = nullptr;
  int nodes_physical = 0;
  bool graph = false;
  int grole = 0;                  // group mode: 0 none, 1 sender, 2 relay, 3 receiver
  unsigned long long expected = 0;  // group receiver: bytes that must land
  // recorded into a caller's CUDA graph (a send inside a stream capture):
  // that graph's nodes point at this entry's tile tables, so LRU eviction
  // skips it (clear_cache / set_topology / arena growth / close still free
  // it, and with it the validity of those captured graphs)
  bool pinned = false;
};

// Multi-process ("group") mode: one process per GPU.  Each rank owns a
// resource block — relay staging arena, relay flags, and a sync block
// {gen u32, seq u32, done u64} — exported as CUDA-IPC handles and mapped by
// every other rank (peer access over NVLink).
struct GroupState {
  int rank = -1, nranks = 0;
  uint8_t* stage = nullptr;
  size_t stage_cap = 0;
  uint32_t* flags = nullptr;  // [flag_cap] chunk flags + [flag_cap] pass counters
  int flag_cap = 0;
  uint8_t* sync = nullptr;    // gen @0, seq @4, done @8
  std::vector<uint8_t*> peer_stage, peer_sync;
  std::vector<uint32_t*> peer_flags;
  std::vector<size_t> peer_stage_cap;
  std::map<std::string, void*> opened;  // IPC-opened peer buffers by handle
  // host inboxes (host-staged path): POSIX shm, pinned + mapped in every rank
  uint8_t* host = nullptr;       // this rank's inbox (host address)
  uint8_t* host_dev = nullptr;   // ... as the device addresses it
  size_t host_cap = 0;
  std::string host_name;         // shm name (unlinked by the owner at destroy)
  std::vector<uint8_t*> peer_host, peer_host_dev;
  std::vector<size_t> peer_host_cap;
  uint32_t* gen(int q) { return (uint32_t*)(q == rank ? sync : peer_sync[q]); }
  unsigned long long* done(int q) { return (unsigned long long*)((q == rank ? sync : peer_sync[q]) + 8); }
};

}  // namespace

struct mp_ctx {
  GroupState* group = nullptr;  // non-null: multi-process group context
  std::vector<Phys> phys;
  std::vector<Logi> logi;
  std::vector<int> peer;  // n_phys x n_phys can-access matrix
  bool has_topo = false;
  Topology topo;
  mp_engine_opts opts{};
  uint8_t* host_stage = nullptr;
  size_t host_cap = 0;
  // sticky wait-timeout codes, one per physical device, in mapped pinned
  // memory: kernels write them (mpk::raise_error), every send reads them
  // with a plain load before it enqueues anything; mp_sync clears them
  unsigned* herr = nullptr;
  std::list<Entry*> lru;  // least recent first
  std::unordered_map<std::string, std::list<Entry*>::iterator, KeyHash> index;
  mp_send_stats stats{};
  std::vector<mp_path> last_paths;
  std::vector<mp_chunk> last_chunks;
  // resend fast path of mp_send_many: the last program's raw arguments and
  // its entry, valid while no entry has been destroyed since (cache_epoch)
  uint64_t cache_epoch = 0;
  struct {
    std::vector<mp_xfer> xfers;
    mp_config cfg{};
    int32_t joint = -1;
    Entry* entry = nullptr;
    std::list<Entry*>::iterator lru_pos;
    uint64_t epoch = 0;
  } last_many;
  // the same for mp_send: the last single send's key bytes and entry
  struct {
    std::string key;
    Entry* entry = nullptr;
    std::list<Entry*>::iterator lru_pos;
    uint64_t epoch = 0;
  } last_one;
  // mp_last_plan's source: copied from the entry only when it changes
  const void* last_plan_of = nullptr;
  uint64_t last_plan_epoch = ~0ull;
  cudaEvent_t last_done = nullptr;  // serialises sends issued on different streams
  void* last_stream = nullptr;
  bool have_last = false;
  int timed_phys = -1;  // device whose kt0/kt1 events bracket the last timed kernel
  bool kernel_timing = false;  // streamed sends bracket the kernel with kt0/kt1
  struct SizeRule {
    uint64_t max_bytes;
    int direct, host;  // MP_ENGINE_*, host -1 = opts.host_engine
  };
  std::vector<SizeRule> size_policy;
  std::mutex mu;
};

namespace {

cudaEvent_t take_event(Phys& p) {
  if (p.next_event >= p.events.size()) {
    DeviceGuard g;
    CK(cudaSetDevice(p.ordinal));
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p.events.push_back(e);
  }
  return p.events[p.next_event++];
}

cudaStream_t lane_stream(Phys& p, int lane) {
  while ((int)p.lanes.size() <= lane) {
    DeviceGuard g;
    CK(cudaSetDevice(p.ordinal));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    p.lanes.push_back(s);
  }
  return p.lanes[lane];
}

void destroy_entry(mp_ctx* ctx, Entry* e) {
  if (!e) return;
  ctx->cache_epoch++;  // invalidates every remembered Entry* (mp_send_many fast path)
  for (auto& pr : e->progs) {
    cudaSetDevice(ctx->phys[pr.phys].ordinal);
    if (pr.d_tiles) cudaFree(pr.d_tiles);
  }
  if (e->exec) cudaGraphExecDestroy(e->exec);
  delete e;
}

void clear_cache(mp_ctx* ctx) {
  for (auto& p : ctx->phys) {
    cudaSetDevice(p.ordinal);
    cudaDeviceSynchronize();
  }
  for (Entry* e : ctx->lru) destroy_entry(ctx, e);
  ctx->lru.clear();
  ctx->index.clear();
  ctx->cache_epoch++;
}

// Grow staging arenas; cached programs point into them, so growth drops the cache.
void ensure_arenas(mp_ctx* ctx, const std::vector<size_t>& stage_need,
                   const std::vector<char>& flag_devs, int flags_need, size_t host_need) {
  bool grow = host_need > ctx->host_cap;
  for (size_t i = 0; i < ctx->logi.size(); ++i)
    if (stage_need[i] > ctx->logi[i].stage_cap || (flag_devs[i] && flags_need > ctx->logi[i].flag_cap))
      grow = true;
  if (!grow) return;
  // growth frees the arenas every cached program points into; programs
  // recorded into a caller's CUDA graph (pinned) would be left dangling in
  // that graph, so refuse instead of corrupting a later replay
  const auto pinned = std::count_if(ctx->lru.begin(), ctx->lru.end(), [](const Entry* x) { return x->pinned; });
  if (pinned)
    throw Error{MP_ERR_STATE, "this send needs larger staging arenas, which would free " + std::to_string(pinned) +
                                  " program(s) captured into CUDA graphs: send the largest transfers once before "
                                  "capturing, or clear_cache() and re-capture"};
  clear_cache(ctx);
  DeviceGuard g;
  for (size_t i = 0; i < ctx->logi.size(); ++i) {
    Logi& L = ctx->logi[i];
    if (stage_need[i] == 0 && !flag_devs[i]) continue;
    CK(cudaSetDevice(ctx->phys[L.phys].ordinal));
    if (stage_need[i] > L.stage_cap) {
      if (L.stage) CK(cudaFree(L.stage));
      size_t cap = std::max(stage_need[i], (size_t)2 * L.stage_cap);
      cap = (cap + 4095) & ~(size_t)4095;
      CK(cudaMalloc(&L.stage, cap));
      L.stage_cap = cap;
    }
    if (flag_devs[i] && flags_need > L.flag_cap) {
      if (L.flags) CK(cudaFree(L.flags));
      int cap = std::max(flags_need, 2 * L.flag_cap);
      CK(cudaMalloc(&L.flags, (size_t)cap * 2 * sizeof(uint32_t)));
      CK(cudaMemset(L.flags, 0, (size_t)cap * 2 * sizeof(uint32_t)));
      CK(cudaDeviceSynchronize());
      L.flag_cap = cap;
    }
  }
  if (host_need > ctx->host_cap) {
    if (ctx->host_stage) CK(cudaFreeHost(ctx->host_stage));
    size_t cap = std::max(host_need, (size_t)2 * ctx->host_cap);
    cap = (cap + 4095) & ~(size_t)4095;
    CK(cudaHostAlloc((void**)&ctx->host_stage, cap, cudaHostAllocPortable | cudaHostAllocMapped));
    ctx->host_cap = cap;
  }
}

}  // namespace
