// mp_engine.cu — the B200 execution engine behind mp_send.
//
// Replaces the reference's simulated execution (sim.py:152-292) with real
// data movement, keeping its semantics:
//   * the chunk plan is the reference planner's, bit-exact (core.hpp);
//   * a staged chunk's hop2 starts only after its hop1 finished
//     (graph.py:115-117, sim.py:182-191) — a device flag for SM lanes, a
//     CUDA event / graph edge for copy-engine lanes;
//   * copy-engine lanes are FIFO streams, one per (path, hop)
//     (pipeline.py:102-125, "two separate CUDA streams");
//   * graph mode captures the whole multi-path workflow once and replays it
//     from an LRU cache keyed by (src, dst, size, devices, path set)
//     (graph.py:121-186).
//
// Physical layout of one send on B200:
//   * every NVLink/HBM path (direct, relay hop1, relay hop2) handled by the SM
//     engine becomes tiles of ONE persistent transfer kernel per physical
//     device (mp_kernels.cuh): one launch per device regardless of chunk count;
//   * copy-engine paths (host-staged always; direct/relay when configured)
//     become cudaMemcpyAsync on lane streams with per-chunk events;
//   * fork/join events tie all lanes to the caller's stream.
//
// Files (one translation unit): engine_state.cuh (launch policy, devices,
// cache entries, arenas), lowering.cuh (transfers -> tile tables + copy-
// engine ops), this file (enqueue / capture / cache lookup, group mode,
// traces, probes, and the C ABI).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <functional>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "core.hpp"
#include "mp_kernels.cuh"

using namespace mp;

#include "engine_state.cuh"
#include "lowering.cuh"

namespace {

// Enqueue the entry's work after `origin`, then make `origin` wait for it.
// Trace-mode resources (mp_send_trace): per physical device a stamp array
// {first start, last end} per logical node plus a %globaltimer base, and
// timing events around every copy-engine op.
struct Trace {
  int nodes = 0;
  std::vector<unsigned long long*> stamps;  // per phys, 2 * nodes
  std::vector<unsigned long long*> base;    // per phys, 1
  std::vector<cudaEvent_t> base_ev;         // per phys, timing event at the fork
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ce_ev;  // per CE op
};

mpk::GroupSync group_sync(mp_ctx* ctx) {
  GroupState* G = ctx->group;
  mpk::GroupSync g{};
  g.n = G->nranks;
  for (int q = 0; q < G->nranks; ++q) g.gen[q] = G->gen(q);
  g.seq = (uint32_t*)(G->sync + 4);
  g.self_gen = G->gen(G->rank);
  return g;
}

// Group mode: this rank's single kernel for the transfer — its tiles (sender
// / relay), the completion wait (receiver) or just the barrier (others).
void enqueue_group(mp_ctx* ctx, Entry* e, cudaStream_t origin) {
  Phys& P = ctx->phys[0];
  P.next_event = 0;
  CK(cudaSetDevice(P.ordinal));
  cudaEvent_t fork = take_event(P);
  CK(cudaEventRecord(fork, origin));
  CK(cudaStreamWaitEvent(P.kstream, fork, 0));
  mpk::GroupSync g = group_sync(ctx);
  if (!e->progs.empty()) {
    const Program& pr = e->progs[0];
    // the receiver's own tiles (host-path hop2) run first, outside the
    // barrier protocol; its byte-count wait below closes the transfer
    const bool recv = e->grole == 3;
    const mpk::GroupSync none{};  // n = 0: no barrier (non-null: no PDL either)
    launch_transfer(ctx->opts, pr.grid, P.kstream, pr.d_tiles, pr.ntiles, P.ctl, pr.nstatic, nullptr,
                    recv ? &none : &g, pr.peer, P.sms, pr.small.get(), pr.kind, pr.d_sched, pr.nhelp);
    if (recv) {
      mpk::group_recv_kernel<<<1, 32, 0, P.kstream>>>(g, ctx->group->done(ctx->group->rank), e->expected,
                                                      P.ctl);
      CK(cudaGetLastError());
    }
  } else if (e->grole == 3) {
    mpk::group_recv_kernel<<<1, 32, 0, P.kstream>>>(g, ctx->group->done(ctx->group->rank), e->expected,
                                                    P.ctl);
    CK(cudaGetLastError());
  } else {
    mpk::group_noop_kernel<<<1, 32, 0, P.kstream>>>(g, P.ctl);
    CK(cudaGetLastError());
  }
  cudaEvent_t j = take_event(P);
  CK(cudaEventRecord(j, P.kstream));
  CK(cudaStreamWaitEvent(origin, j, 0));
}

// A cached single send whose whole program is ONE kernel on the caller's
// device — the small-message kernel from kPdlMinBytes (opts.pdl >= 1), a
// static one-tile-per-CTA TMA table (>= 2) or a dynamic table (3, the
// default; also relay tables whose flags stay on one device) — replays as
// a direct programmatic-dependent launch of that kernel instead of its
// one-node graph: back-to-back graph launches retire in 2.048 us quanta
// (1-4 MiB: 4.1 us, 16 MiB: 8.2 us) while PDL launches overlap the next
// launch's processing with the running kernel: 1-4 MiB 4.1 -> 2.5-3.4 us,
// 8 MiB 6.1 -> 3.8, 16 MiB 8.2 -> 5.4, 32 MiB 10.2 -> 8.0
// (tools/exp_pdl.py).  Below ~512 KiB the graph replay often takes one
// quantum and its host path is cheaper, so it stays.  The graph is still
// captured and instantiated (lifecycle phases; pdl = 0 replays it).
bool pdl_replay(const mp_ctx* ctx, const Entry* e) {
  if (!ctx->opts.pdl || ctx->group || !e->ce.empty() || e->progs.size() != 1 ||
      e->progs[0].phys != e->src_phys)
    return false;
  const Program& pr = e->progs[0];
  if (pr.kind == PROG_SMALL) return pr.small && pr.bytes >= pdl_min_bytes();
  if (pr.kind == PROG_STATIC_TMA) return ctx->opts.pdl >= 2;
  return ctx->opts.pdl >= 3;  // dynamic tables: 128 MiB 45.8 -> 44.0 us, 512 MiB 162.4 -> 160.8 us
}

void enqueue(mp_ctx* ctx, Entry* e, cudaStream_t origin, bool timing, Trace* tr = nullptr) {
  if (ctx->group) {
    enqueue_group(ctx, e, origin);
    return;
  }
  Phys& S = ctx->phys[e->src_phys];
  set_device(S.ordinal);
  if (!tr && e->ce.empty() && e->progs.size() == 1 && e->progs[0].phys == e->src_phys) {
    // one kernel on the caller's device and nothing else: no fork/join, the
    // kernel goes straight onto the caller's stream (per-call launch ~= one
    // kernel launch; a captured graph is the single kernel node either way)
    const Program& pr = e->progs[0];
    if (timing) ctx->timed_phys = pr.phys;
    if (timing) CK(cudaEventRecord(S.kt0, origin));
    launch_transfer(ctx->opts, pr.grid, origin, pr.d_tiles, pr.ntiles, S.ctl, pr.nstatic, nullptr,
                    nullptr, pr.peer, S.sms, pr.small.get(), pr.kind, pr.d_sched, pr.nhelp);
    if (timing) CK(cudaEventRecord(S.kt1, origin));
    return;
  }
  for (auto& p : ctx->phys) p.next_event = 0;
  cudaEvent_t fork = take_event(S);
  CK(cudaEventRecord(fork, origin));
  std::vector<std::pair<int, cudaStream_t>> used;
  auto use = [&](int ph, cudaStream_t s) {
    for (auto& u : used)
      if (u.second == s) return;
    CK(cudaSetDevice(ctx->phys[ph].ordinal));
    CK(cudaStreamWaitEvent(s, fork, 0));
    used.push_back({ph, s});
  };
  if (tr) {  // time base of every device: a timing event + a %globaltimer stamp
    for (size_t ph = 0; ph < ctx->phys.size(); ++ph) {
      Phys& P = ctx->phys[ph];
      use((int)ph, P.kstream);
      CK(cudaSetDevice(P.ordinal));
      CK(cudaEventRecord(tr->base_ev[ph], P.kstream));
      mpk::stamp_kernel<<<1, 1, 0, P.kstream>>>(tr->base[ph]);
      CK(cudaGetLastError());
    }
  }
  // SM transfer kernels, one per physical device; the caller's device runs
  // its kernel straight on the caller's stream (no fork/join for it)
  for (auto& pr : e->progs) {
    Phys& P = ctx->phys[pr.phys];
    const bool on_origin = !tr && pr.phys == e->src_phys;
    cudaStream_t ks = on_origin ? origin : P.kstream;
    if (!on_origin) use(pr.phys, P.kstream);
    CK(cudaSetDevice(P.ordinal));
    bool t = timing && pr.phys == e->src_phys;
    if (t) ctx->timed_phys = pr.phys;
    if (t) CK(cudaEventRecord(P.kt0, ks));
    launch_transfer(ctx->opts, pr.grid, ks, pr.d_tiles, pr.ntiles, P.ctl, pr.nstatic,
                    tr ? tr->stamps[pr.phys] : nullptr, nullptr, pr.peer, P.sms, pr.small.get(), pr.kind, pr.d_sched, pr.nhelp);
    if (t) CK(cudaEventRecord(P.kt1, ks));
  }
  // copy-engine lanes
  std::vector<cudaEvent_t> evs(e->ev_phys.size());
  for (size_t i = 0; i < evs.size(); ++i) evs[i] = take_event(ctx->phys[e->ev_phys[i]]);
  for (size_t i = 0; i < e->ce.size(); ++i) {
    const CeOp& op = e->ce[i];
    Phys& P = ctx->phys[op.phys];
    cudaStream_t s = lane_stream(P, op.lane);
    use(op.phys, s);
    CK(cudaSetDevice(P.ordinal));
    if (op.wait_ev >= 0) CK(cudaStreamWaitEvent(s, evs[op.wait_ev], 0));
    if (tr) CK(cudaEventRecord(tr->ce_ev[i].first, s));
    if (op.rows > 1)
      CK(cudaMemcpy2DAsync(op.dst, op.dpitch, op.src, op.spitch, op.len, op.rows, cudaMemcpyDefault, s));
    else
      CK(cudaMemcpyAsync(op.dst, op.src, op.len, cudaMemcpyDefault, s));
    if (tr) CK(cudaEventRecord(tr->ce_ev[i].second, s));
    if (op.record_ev >= 0) CK(cudaEventRecord(evs[op.record_ev], s));
  }
  // join
  for (auto& u : used) {
    Phys& P = ctx->phys[u.first];
    CK(cudaSetDevice(P.ordinal));
    cudaEvent_t j = take_event(P);
    CK(cudaEventRecord(j, u.second));
    CK(cudaSetDevice(S.ordinal));
    CK(cudaStreamWaitEvent(origin, j, 0));
  }
  CK(cudaSetDevice(S.ordinal));
}

void capture(mp_ctx* ctx, Entry* e) {
  Phys& S = ctx->phys[e->src_phys];
  CK(cudaSetDevice(S.ordinal));
  double t0 = now_us();
  CK(cudaStreamBeginCapture(S.capture, cudaStreamCaptureModeThreadLocal));
  double t1 = now_us();
  try {
    enqueue(ctx, e, S.capture, false);
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(S.capture, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t graph = nullptr;
  CK(cudaStreamEndCapture(S.capture, &graph));
  double t2 = now_us();
  size_t n = 0;
  cudaGraphGetNodes(graph, nullptr, &n);
  e->nodes_physical = (int)n;
  cudaError_t ie = cudaGraphInstantiate(&e->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) throw Error{MP_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie)};
  double t3 = now_us();
  ctx->stats.creation_us = t1 - t0;
  ctx->stats.construction_us = t2 - t1;
  ctx->stats.instantiation_us = t3 - t2;
}

void append_key(std::string& key, const void* src, void* dst, uint64_t size, int sd, int dd,
                const mp_config& c) {
  struct {
    uint64_t s, d, n;
    int32_t sd, dd, g, h, m, gm, pol, pad;  // explicit pad: every key byte is defined
  } k{(uint64_t)(uintptr_t)src, (uint64_t)(uintptr_t)dst, size, sd, dd,
      c.num_gpu_paths, c.host_path_enabled, c.max_chunks, c.graph_mode ? 1 : 0, c.share_policy, 0};
  static_assert(sizeof k == 3 * 8 + 8 * 4, "key has no implicit padding");
  key.append((const char*)&k, sizeof k);
}

std::string make_key(const void* src, void* dst, uint64_t size, int sd, int dd, const mp_config& c) {
  std::string key;
  append_key(key, src, dst, size, sd, dd, c);
  return key;
}

// LRU lookup; a miss plans, lowers and (graph mode) captures + instantiates
// the entry, then evicts the least recent one past cfg.cache_capacity
// (graph.py:173-186).  Updates the lifecycle stats.
Entry* lookup_entry(mp_ctx* ctx, const void* src, void* dst, uint64_t size, int src_dev, int dst_dev,
                    const mp_config& cfg, cudaStream_t user,
                    const std::function<Entry*(const std::string&)>& builder = nullptr,
                    const std::string* key_override = nullptr) {
  double t_start = now_us();
  std::string own;
  const std::string& key = key_override ? *key_override : (own = make_key(src, dst, size, src_dev, dst_dev, cfg));
  mp_send_stats& st = ctx->stats;
  auto it = ctx->index.find(key);
  if (it != ctx->index.end()) {
    ctx->lru.splice(ctx->lru.end(), ctx->lru, it->second);
    st.hit = 1;
    st.cache_hits++;
    st.creation_us = st.construction_us = st.instantiation_us = st.plan_us = 0.0;
    return *it->second;
  }
  validate_config(cfg);
  Entry* e = builder ? builder(key) : build_entry(ctx, key, src, dst, size, src_dev, dst_dev, cfg);
  st.plan_us = now_us() - t_start;
  st.creation_us = st.construction_us = st.instantiation_us = 0.0;
  if (cfg.graph_mode) {
    try {
      capture(ctx, e);
      e->graph = true;
    } catch (...) {
      destroy_entry(ctx, e);
      throw;
    }
  }
  ctx->lru.push_back(e);
  ctx->index[key] = std::prev(ctx->lru.end());
  while ((int)ctx->lru.size() > cfg.cache_capacity) {  // graph.py:184-185
    // the least recent entry not pinned by a caller's captured graph
    auto victim = std::find_if(ctx->lru.begin(), ctx->lru.end(), [](const Entry* x) { return !x->pinned; });
    if (victim == ctx->lru.end() || *victim == e) break;
    Entry* old = *victim;
    ctx->lru.erase(victim);
    ctx->index.erase(old->key);
    CK(cudaSetDevice(ctx->phys[old->src_phys].ordinal));
    // the old entry may still be replaying on `user` or on the stream of the
    // previous send (which `user` has not been made to wait for yet)
    CK(cudaStreamSynchronize(user));
    if (ctx->have_last) CK(cudaEventSynchronize(ctx->last_done));
    destroy_entry(ctx, old);
    st.cache_evictions++;
  }
  st.hit = 0;
  st.cache_misses++;
  return e;
}


// Group mode: tile sizes of relay hops (128 KiB: half the system-scope flag
// traffic, as kRelayTileBytes) and host hops (64 KiB: parallelism while the
// PCIe path is the bottleneck), agreed by construction across ranks.
constexpr uint64_t kGroupRelayTileBytes = 128 << 10;
constexpr uint64_t kGroupHostTileBytes = 64 << 10;

// Serialized CUDA-IPC handles of one rank's group resource block.
struct GroupBlob {
  uint64_t stage_cap;
  int32_t flag_cap;
  int32_t rank;
  cudaIpcMemHandle_t stage, flags, sync;
  uint64_t host_cap;   // 0: no host inbox
  char host_name[40];  // POSIX shm name of the inbox
};
static_assert(sizeof(GroupBlob) <= MP_GROUP_BLOB_BYTES, "group blob size");

// Group mode: lower the plan to THIS rank's part (every rank computes the same
// plan, node ids, staging offsets and tile cuts deterministically).
Entry* build_group_entry(mp_ctx* ctx, const std::string& key, const void* src, uint32_t src_align,
                         void* dst, uint64_t size, int sr, int dr, const mp_config& cfg) {
  GroupState* G = ctx->group;
  std::unique_ptr<Entry> e(new Entry());
  e->key = key;
  e->paths = plan_paths(ctx->topo, sr, dr, cfg);
  for (const mp_path& p : e->paths)
    if (p.kind == MP_PATH_HOST && ((dr == G->rank && !G->host) || (dr != G->rank && !G->peer_host[dr])))
      throw Error{MP_ERR_STATE, "the host-staged path needs the destination rank's host inbox "
                                "(mp_group_host_arena before mp_group_export)"};
  e->chunks = make_chunk_plan(e->paths.data(), (int)e->paths.size(), (int64_t)size, cfg.max_chunks);
  const int np = (int)e->paths.size(), nc = (int)e->chunks.size();
  for (const mp_chunk& c : e->chunks) e->nodes_logical += e->paths[c.path_index].nhops;
  e->src_phys = 0;
  const int me = G->rank;
  e->grole = me == sr ? 1 : me == dr ? 3 : 0;
  for (const mp_path& p : e->paths)
    if (p.kind == MP_PATH_GPU && p.stage == me) e->grole = 2;
  e->expected = size;
  if (nc > G->flag_cap) throw Error{MP_ERR_STATE, "group flag array too small for the chunk plan"};
  std::vector<uint64_t> path_bytes(np, 0);
  for (const mp_chunk& c : e->chunks) path_bytes[c.path_index] += c.length;
  const int sms = ctx->phys[0].sms;
  const uint64_t s0 = (uint64_t)(uintptr_t)src, d0 = (uint64_t)(uintptr_t)dst;
  std::vector<std::pair<std::pair<uint64_t, uint64_t>, mpk::Tile>> tiles;
  std::vector<uint64_t> stage_off(np, 0);
  uint32_t node = 0;
  for (int c = 0; c < nc; ++c) {
    const mp_chunk& ch = e->chunks[c];
    const mp_path& P = e->paths[ch.path_index];
    const int p = ch.path_index;
    const uint64_t round = (uint64_t)ch.seq;
    const uint32_t n_a = node, n_b = node + 1;
    node += (uint32_t)P.nhops;
    if (P.kind == MP_PATH_DIRECT) {
      if (e->grole != 1) continue;
      mpk::Tile t{};
      t.node = n_a;
      t.signal = (uint32_t*)G->done(dr);  // bytes landed at the receiver
      t.flags = mpk::TILE_SIGNAL_BYTES;
      append_tiles(tiles, 2 * round, s0 + ch.offset, d0 + ch.offset, ch.length,
                   auto_tile_bytes(ctx, path_bytes[p], sms), t);
      continue;
    }
    if (P.kind == MP_PATH_HOST) {
      // the destination rank's host inbox: the sender's hop1 tiles write the
      // chunk there and release its flag in the destination's HBM (system
      // scope), the destination's hop2 tiles load it back once the flag
      // counts every hop1 tile; offsets / cuts agree across ranks by
      // construction (congruent to the source mod 16, fixed tile size)
      stage_off[p] += (((uint64_t)src_align + ch.offset) - stage_off[p]) & 15u;
      const uint64_t so = stage_off[p];
      stage_off[p] += ch.length;
      const size_t cap = dr == me ? G->host_cap : G->peer_host_cap[dr];
      if (stage_off[p] > cap) throw Error{MP_ERR_STATE, "group host inbox too small for the host share"};
      const uint64_t th = kGroupHostTileBytes;
      if (e->grole == 1) {
        uint8_t* slot = G->peer_host_dev[dr] + so;
        mpk::Tile h1{};
        h1.node = n_a;
        h1.signal = G->peer_flags[dr] + c;
        append_tiles(tiles, 2 * round, s0 + ch.offset, (uint64_t)(uintptr_t)slot, ch.length, th, h1);
      } else if (me == dr) {
        uint8_t* slot = G->host_dev + so;
        mpk::Tile h2{};
        h2.node = n_b;
        h2.wait = G->flags + c;
        h2.pass = G->flags + G->flag_cap + c;
        h2.wait_count = (uint32_t)ntiles_of((uint64_t)(uintptr_t)slot, ch.length, th);
        h2.pass_count = (uint32_t)ntiles_of(d0 + ch.offset, ch.length, th);
        h2.signal = (uint32_t*)G->done(dr);
        h2.flags = mpk::TILE_SRC_MUTABLE | mpk::TILE_SIGNAL_BYTES;
        append_tiles(tiles, 2 * round + 3, (uint64_t)(uintptr_t)slot, d0 + ch.offset, ch.length, th, h2);
      }
      continue;
    }
    const int k = P.stage;
    stage_off[p] += (((uint64_t)src_align + ch.offset) - stage_off[p]) & 15u;
    const uint64_t so = stage_off[p];
    stage_off[p] += ch.length;
    const size_t cap = k == me ? G->stage_cap : G->peer_stage_cap[k];
    if (stage_off[p] > cap) throw Error{MP_ERR_STATE, "group staging arena too small for the relay share"};
    // relay tiles are cut identically on the sender (hop1 signals) and the
    // relay rank (hop2 waits for that many signals): a size that depends on
    // nothing rank-local (not the SM count, not the engine options)
    const uint64_t t1 = kGroupRelayTileBytes;
    if (e->grole == 1) {
      uint8_t* stage = G->peer_stage[k] + so;
      mpk::Tile h1{};
      h1.node = n_a;
      h1.signal = G->peer_flags[k] + c;
      append_tiles(tiles, 2 * round, s0 + ch.offset, (uint64_t)(uintptr_t)stage, ch.length, t1, h1);
    } else if (e->grole == 2 && k == me) {
      uint8_t* stage = G->stage + so;
      mpk::Tile h2{};
      h2.node = n_b;
      h2.wait = G->flags + c;
      h2.pass = G->flags + G->flag_cap + c;
      h2.wait_count = (uint32_t)ntiles_of((uint64_t)(uintptr_t)stage, ch.length, t1);
      h2.pass_count = (uint32_t)ntiles_of(d0 + ch.offset, ch.length, t1);
      h2.signal = (uint32_t*)G->done(dr);
      h2.flags = mpk::TILE_SRC_MUTABLE | mpk::TILE_SIGNAL_BYTES;
      append_tiles(tiles, 2 * round + 3, (uint64_t)(uintptr_t)stage, d0 + ch.offset, ch.length, t1, h2);
    }
  }
  if (!tiles.empty()) {
    std::stable_sort(tiles.begin(), tiles.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<mpk::Tile> flat;
    for (auto& kv : tiles) flat.push_back(kv.second);
    Program pr;
    pr.phys = 0;
    pr.ntiles = (unsigned)flat.size();
    pr.grid = (unsigned)std::min<uint64_t>(flat.size(), (uint64_t)sms * std::max(1, ctx->opts.ctas_per_sm));
    bool waits = false;
    for (const auto& t : flat) waits |= t.wait != nullptr;
    pr.nstatic = waits ? 0u : pr.grid;
    // IPC-mapped buffers of another physical GPU make this an NVLink table
    const int here = ctx->phys[0].ordinal;
    std::set<uint64_t> seen;  // one query per 16 MiB region
    for (const auto& t : flat)
      for (uint64_t a : {t.src, t.dst}) {
        if (!seen.insert(a >> 24).second) continue;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, (const void*)(uintptr_t)a) == cudaSuccess &&
            at.type == cudaMemoryTypeDevice && at.device != here)
          pr.peer = true;
        else
          cudaGetLastError();
      }
    CK(cudaSetDevice(ctx->phys[0].ordinal));
    CK(cudaMalloc(&pr.d_tiles, flat.size() * sizeof(mpk::Tile)));
    CK(cudaMemcpy(pr.d_tiles, flat.data(), flat.size() * sizeof(mpk::Tile), cudaMemcpyHostToDevice));
    CK(cudaStreamSynchronize(cudaStreamLegacy));  // the upload lands before any launch
    e->progs.push_back(pr);
  }
  return e.release();
}

// A group host inbox: `bytes` of POSIX shared memory (created by its owner,
// opened by every peer), pinned and mapped for this process's device.
void map_host_inbox(const char* name, size_t bytes, bool create, uint8_t** host, uint8_t** dev) {
  const int fd = shm_open(name, create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) throw Error{MP_ERR_CUDA, std::string("shm_open ") + name + ": " + strerror(errno)};
  // reserve the pages now: a /dev/shm smaller than the inbox fails here
  // (ENOSPC) instead of with SIGBUS when the pages are first touched
  int fe = 0;
  if (create && (ftruncate(fd, (off_t)bytes) != 0 || (fe = posix_fallocate(fd, 0, (off_t)bytes)) != 0)) {
    const std::string why = strerror(fe ? fe : errno);
    close(fd);
    shm_unlink(name);
    throw Error{MP_ERR_CUDA, "host inbox of " + std::to_string(bytes) + " bytes in /dev/shm: " + why};
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    if (create) shm_unlink(name);
    throw Error{MP_ERR_CUDA, std::string("mmap host inbox: ") + strerror(errno)};
  }
  const cudaError_t r = cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (r != cudaSuccess) {
    munmap(p, bytes);
    if (create) shm_unlink(name);
    throw Error{MP_ERR_CUDA, std::string("cudaHostRegister host inbox: ") + cudaGetErrorString(r)};
  }
  CK(cudaHostGetDevicePointer((void**)dev, p, 0));
  *host = (uint8_t*)p;
}

void unmap_host_inbox(uint8_t* host, size_t bytes) {
  cudaHostUnregister(host);
  munmap(host, bytes);
}

// Base address of the allocation holding `p` (driver entry point, resolved at
// run time so the library loads without libcuda on GPU-less hosts).
uint64_t allocation_base(const void* p) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = nullptr;
  if (!fn) {
    void* sym = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q));
    if (!sym) throw Error{MP_ERR_CUDA, "cuMemGetAddressRange unavailable"};
    fn = (Fn)sym;
  }
  unsigned long long base = 0;
  size_t sz = 0;
  if (fn(&base, &sz, (unsigned long long)(uintptr_t)p) != 0)
    throw Error{MP_ERR_CUDA, "cuMemGetAddressRange failed"};
  return base;
}

const char* wait_what(unsigned code) {
  static const char* what[] = {"wait", "relay flag wait", "group barrier wait", "receiver byte-count wait"};
  return code <= 3 ? what[code] : what[0];
}

// A kernel's wait timed out since the last mp_sync: fail every later send
// (the error word is in mapped host memory, so this is a plain load).
void check_sticky(const mp_ctx* ctx) {
  if (!ctx->herr) return;
  for (size_t i = 0; i < ctx->phys.size(); ++i) {
    const unsigned c = ((volatile const unsigned*)ctx->herr)[i];
    if (c)
      throw Error{MP_ERR_CUDA, std::string(wait_what(c)) + " timed out on device " +
                                   std::to_string(ctx->phys[i].ordinal) +
                                   ": a transfer was not delivered (its staged bytes were never copied); "
                                   "mp_sync reports and clears the error"};
  }
}

// mp_last_plan's copy of an entry's plan, refreshed only when the entry
// changes (a resend of the same entry copies nothing)
void remember_plan(mp_ctx* ctx, const Entry* e) {
  if (ctx->last_plan_of == e && ctx->last_plan_epoch == ctx->cache_epoch) return;
  ctx->last_paths = e->paths;
  ctx->last_chunks = e->chunks;
  ctx->last_plan_of = e;
  ctx->last_plan_epoch = ctx->cache_epoch;
}

// A send enqueued into a CUDA stream capture (the caller building its own
// graph): the cached program is recorded as nodes of that graph (enqueue,
// never a nested cudaGraphLaunch), no engine event is recorded or waited on
// (an event recorded inside a capture is unusable outside it — it broke
// every later cross-stream send), and a cache miss is refused (building a
// program allocates and uploads, which a capture forbids).
bool stream_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

const char* const kCaptureMiss =
    "a send inside a CUDA stream capture must hit the plan cache: send it once outside the capture first";

uint64_t timeout_ns(const mp_engine_opts& o) { return (uint64_t)o.wait_timeout_ms * 1000000ull; }

// (Re)initialise a device's control block: zero counters and error word,
// the host error word's device address and the wait limit.
void init_ctl(mp_ctx* ctx, Phys& P) {
  mpk::Ctl c{};
  c.herr = P.herr_dev;
  c.timeout_ns = timeout_ns(ctx->opts);
  DeviceGuard g;
  CK(cudaSetDevice(P.ordinal));
  CK(cudaMemcpy(P.ctl, &c, sizeof c, cudaMemcpyHostToDevice));
  CK(cudaDeviceSynchronize());  // lands before any launch on a non-blocking stream
}

}  // namespace


// ===========================================================================
// C ABI
// ===========================================================================
#define GUARD_BEGIN try {
#define GUARD_END                                      \
  }                                                    \
  catch (const Error& e) {                             \
    return fail(e.code, e.msg);                        \
  }                                                    \
  catch (const std::exception& e) {                    \
    return fail(MP_ERR_VALUE, e.what());               \
  }

extern "C" {

int mp_ctx_create(int32_t n_logical, const int32_t* device_map, mp_ctx** out) {
  GUARD_BEGIN
  if (!out || n_logical < 1 || !device_map) return fail(MP_ERR_VALUE, "bad context arguments");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  DeviceGuard g;
  auto ctx = std::make_unique<mp_ctx>();
  ctx->opts.direct_engine = MP_ENGINE_SM;
  ctx->opts.relay_engine = MP_ENGINE_SM;
  // measured defaults (tools/abi_latency.cu, profiles/): dynamic tables run
  // the LDG/STG kernel, 4 CTAs x 256 threads per SM, 64 KiB tiles (100% of
  // the measured HBM copy peak at 512 MiB); static tables run the TMA ring
  // (4 x 32 KiB per SM) and small ones the small-message kernel
  ctx->opts.copy_kind = MP_COPY_VEC;
  ctx->opts.ctas_per_sm = 4;
  ctx->opts.threads = 256;
  ctx->opts.tile_bytes = 0;
  ctx->opts.host_slots = 0;
  ctx->opts.pull = 0;
  ctx->opts.sm_min_bytes = 0;
  // the SM kernels move a small host-staged share (mapped pinned memory): a
  // host chunk <= 64 KiB is one roundtrip tile worked beside the direct
  // stream inside the same launch, so direct + host stays ONE kernel (a PDL
  // replay); the copy-engine variant (2-D copies, fork/join events) costs a
  // multi-node graph per send: 64 MiB 27.9 vs 21.0 us, 16 MiB 20.8 vs 6.3 us
  // (profiles/r02_multifree.jsonl).  Larger host chunks go to copy engines.
  ctx->opts.host_engine = MP_ENGINE_AUTO;
  ctx->opts.unroll = 8;
  ctx->opts.tma_stages = 4;
  ctx->opts.tma_block = 32768;
  ctx->opts.sched = MP_SCHED_AUTO;
  ctx->opts.small_max_bytes = kSmallMaxBytes;
  ctx->opts.pdl = 3;
  std::map<int, int> phys_of;
  for (int i = 0; i < n_logical; ++i) {
    int ord = device_map[i];
    if (ord < 0 || ord >= ndev)
      return fail(MP_ERR_VALUE, "device_map[" + std::to_string(i) + "] = " + std::to_string(ord) +
                                    " is not a CUDA device (have " + std::to_string(ndev) + ")");
    if (!phys_of.count(ord)) {
      phys_of[ord] = (int)ctx->phys.size();
      Phys p;
      p.ordinal = ord;
      ctx->phys.push_back(p);
    }
    Logi L;
    L.phys = phys_of[ord];
    ctx->logi.push_back(L);
  }
  const int np = (int)ctx->phys.size();
  ctx->peer.assign(np * np, 0);
  for (int a = 0; a < np; ++a) {
    Phys& P = ctx->phys[a];
    CK(cudaSetDevice(P.ordinal));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, P.ordinal));
    P.sms = prop.multiProcessorCount;
    CK(cudaMalloc(&P.ctl, sizeof(mpk::Ctl)));
    CK(cudaStreamCreateWithFlags(&P.kstream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&P.capture, cudaStreamNonBlocking));
    CK(cudaEventCreate(&P.kt0));
    CK(cudaEventCreate(&P.kt1));
    for (int b = 0; b < np; ++b) {
      if (a == b) {
        ctx->peer[a * np + b] = 1;
        continue;
      }
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, P.ordinal, ctx->phys[b].ordinal));
      if (can) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(ctx->phys[b].ordinal, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (pe != cudaSuccess) throw Error{MP_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(pe)};
      }
      ctx->peer[a * np + b] = can;
    }
  }
  CK(cudaSetDevice(ctx->phys[0].ordinal));
  CK(cudaHostAlloc((void**)&ctx->herr, np * sizeof(unsigned), cudaHostAllocPortable | cudaHostAllocMapped));
  for (int a = 0; a < np; ++a) {
    ctx->herr[a] = 0u;
    CK(cudaHostGetDevicePointer((void**)&ctx->phys[a].herr_dev, ctx->herr + a, 0));
    init_ctl(ctx.get(), ctx->phys[a]);
  }
  CK(cudaEventCreateWithFlags(&ctx->last_done, cudaEventDisableTiming));
  CK(cudaDeviceSynchronize());
  *out = ctx.release();
  return MP_OK;
  GUARD_END
}

void mp_ctx_destroy(mp_ctx* ctx) {
  if (!ctx) return;
  clear_cache(ctx);
  if (GroupState* G = ctx->group) {
    cudaSetDevice(ctx->phys[0].ordinal);
    for (auto& kv : G->opened) cudaIpcCloseMemHandle(kv.second);
    for (int q = 0; q < G->nranks; ++q) {
      if (q == G->rank) continue;
      if (G->peer_stage[q]) cudaIpcCloseMemHandle(G->peer_stage[q]);
      if (G->peer_flags[q]) cudaIpcCloseMemHandle(G->peer_flags[q]);
      if (G->peer_sync[q]) cudaIpcCloseMemHandle(G->peer_sync[q]);
    }
    cudaFree(G->stage);
    cudaFree(G->flags);
    cudaFree(G->sync);
    for (int q = 0; q < G->nranks; ++q)
      if (G->peer_host[q]) unmap_host_inbox(G->peer_host[q], G->peer_host_cap[q]);
    if (G->host) {
      unmap_host_inbox(G->host, G->host_cap);
      shm_unlink(G->host_name.c_str());
    }
    delete G;
    ctx->group = nullptr;
  }
  for (auto& L : ctx->logi) {
    if (L.phys < 0) continue;
    cudaSetDevice(ctx->phys[L.phys].ordinal);
    if (L.stage) cudaFree(L.stage);
    if (L.flags) cudaFree(L.flags);
  }
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  if (ctx->herr) cudaFreeHost(ctx->herr);
  for (auto& P : ctx->phys) {
    cudaSetDevice(P.ordinal);
    for (auto s : P.lanes) cudaStreamDestroy(s);
    for (auto e : P.events) cudaEventDestroy(e);
    cudaStreamDestroy(P.kstream);
    cudaStreamDestroy(P.capture);
    cudaEventDestroy(P.kt0);
    cudaEventDestroy(P.kt1);
    cudaFree(P.ctl);
  }
  cudaEventDestroy(ctx->last_done);
  delete ctx;
}

int mp_ctx_set_topology(mp_ctx* ctx, const mp_topology* topo) {
  GUARD_BEGIN
  if (!ctx || !topo) return fail(MP_ERR_VALUE, "null argument");
  if (topo->t.n_accel != (int)ctx->logi.size())
    return fail(MP_ERR_STATE, "topology has " + std::to_string(topo->t.n_accel) +
                                  " accelerators but the context maps " +
                                  std::to_string(ctx->logi.size()));
  std::lock_guard<std::mutex> lk(ctx->mu);
  clear_cache(ctx);
  ctx->topo = topo->t;
  ctx->has_topo = true;
  return MP_OK;
  GUARD_END
}

int mp_ctx_set_engine(mp_ctx* ctx, const mp_engine_opts* o) {
  GUARD_BEGIN
  if (!ctx || !o) return fail(MP_ERR_VALUE, "null argument");
  if (o->threads < 32 || o->threads > 256 || o->threads % 32)
    return fail(MP_ERR_VALUE, "threads must be a multiple of 32 in [32, 256]");
  if (o->ctas_per_sm < 1 || o->ctas_per_sm > 8) return fail(MP_ERR_VALUE, "ctas_per_sm must be in [1, 8]");
  if (o->host_slots == 1) return fail(MP_ERR_VALUE, "host_slots must be 0 (all) or >= 2");
  if (o->unroll != 4 && o->unroll != 8 && o->unroll != 16) return fail(MP_ERR_VALUE, "unroll must be 4, 8 or 16");
  if (o->copy_kind != MP_COPY_VEC && o->copy_kind != MP_COPY_TMA) return fail(MP_ERR_VALUE, "unknown copy kind");
  if (o->tma_stages < 2 || o->tma_stages > 16) return fail(MP_ERR_VALUE, "tma_stages must be in [2, 16]");
  if (o->tma_block < 16 || o->tma_block % 16 || (int64_t)o->tma_block * o->tma_stages > 227 * 1024)
    return fail(MP_ERR_VALUE, "tma_block must be a multiple of 16 with stages*block <= 227 KiB");
  if (o->direct_engine < 0 || o->direct_engine > 1 || o->relay_engine < 0 || o->relay_engine > 1 ||
      o->host_engine < 0 || o->host_engine > 2)
    return fail(MP_ERR_VALUE, "unknown engine");
  if (o->sched != MP_SCHED_AUTO && o->sched != MP_SCHED_DYNAMIC) return fail(MP_ERR_VALUE, "unknown sched");
  if (o->small_max_bytes < 0 || o->small_max_bytes > (int64_t)1 << 31)
    return fail(MP_ERR_VALUE, "small_max_bytes must be in [0, 2^31]");
  if (o->pdl < 0 || o->pdl > 3) return fail(MP_ERR_VALUE, "pdl must be 0..3");
  if (o->wait_timeout_ms < 0) return fail(MP_ERR_VALUE, "wait_timeout_ms must be >= 0");
  if (o->fault_inject < 0 || o->fault_inject > 3) return fail(MP_ERR_VALUE, "fault_inject must be 0..3");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  clear_cache(ctx);
  ctx->opts = *o;
  const unsigned long long lim = timeout_ns(*o);
  for (auto& P : ctx->phys) {  // the wait limit lives in the control block
    CK(cudaSetDevice(P.ordinal));
    CK(cudaMemcpy(&P.ctl->timeout_ns, &lim, sizeof lim, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
  }
  return MP_OK;
  GUARD_END
}

int mp_ctx_set_size_policy(mp_ctx* ctx, const uint64_t* max_bytes, const int32_t* direct_engine,
                           const int32_t* host_engine, int32_t n) {
  GUARD_BEGIN
  if (!ctx || n < 0 || (n > 0 && (!max_bytes || !direct_engine)))
    return fail(MP_ERR_VALUE, "bad size policy arguments");
  std::vector<mp_ctx::SizeRule> rules;
  auto ok = [](int e) { return e == MP_ENGINE_SM || e == MP_ENGINE_CE; };
  for (int i = 0; i < n; ++i) {
    if (!ok(direct_engine[i]) || (host_engine && !ok(host_engine[i])))
      return fail(MP_ERR_VALUE, "unknown engine in size policy");
    if (i > 0 && max_bytes[i] <= max_bytes[i - 1])
      return fail(MP_ERR_VALUE, "size policy bounds must increase");
    rules.push_back(mp_ctx::SizeRule{max_bytes[i], direct_engine[i], host_engine ? host_engine[i] : -1});
  }
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  clear_cache(ctx);
  ctx->size_policy = rules;
  return MP_OK;
  GUARD_END
}

int mp_ctx_get_engine(const mp_ctx* ctx, mp_engine_opts* o) {
  if (!ctx || !o) return fail(MP_ERR_VALUE, "null argument");
  *o = ctx->opts;
  return MP_OK;
}

int mp_ctx_peer_matrix(const mp_ctx* ctx, int32_t* out, int32_t cap) {
  if (!ctx || !out) return fail(MP_ERR_VALUE, "null argument");
  if (cap < (int)ctx->peer.size()) return fail(MP_ERR_CAPACITY, "peer matrix capacity too small");
  for (size_t i = 0; i < ctx->peer.size(); ++i) out[i] = ctx->peer[i];
  return MP_OK;
}

int mp_send(mp_ctx* ctx, const void* src, void* dst, uint64_t size, int32_t src_dev,
            int32_t dst_dev, const mp_config* cfg, void* stream) {
  GUARD_BEGIN
  if (!ctx || !cfg) return fail(MP_ERR_VALUE, "null argument");
  if (!ctx->has_topo) return fail(MP_ERR_STATE, "context has no topology (mp_ctx_set_topology)");
  if (ctx->group) return fail(MP_ERR_STATE, "group context: use mp_group_send");
  if (src_dev < 0 || src_dev >= (int)ctx->logi.size() || dst_dev < 0 || dst_dev >= (int)ctx->logi.size()) {
    if (src_dev == dst_dev)
      return fail(MP_ERR_PLAN, "source and destination are the same device (" + device_label(src_dev) + ")");
    return fail(MP_ERR_PLAN, "transfers run between accelerators");
  }
  if (size == 0) return fail(MP_ERR_CHUNK, "message size must be >= 1 byte, got 0");
  if (!src || !dst) return fail(MP_ERR_VALUE, "null buffer");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  cudaStream_t user = (cudaStream_t)stream;
  const bool capturing = stream_capturing(user);
  // resend of the last single send (back-to-back messages on one buffer
  // pair): the same key bytes and its entry still cached — a hit without
  // the hash lookup (the key buffer is reused: a hit allocates nothing)
  auto& lo = ctx->last_one;
  thread_local std::string key;
  key.clear();
  append_key(key, src, dst, size, src_dev, dst_dev, *cfg);
  Entry* e = nullptr;
  if (lo.entry && lo.epoch == ctx->cache_epoch && lo.key == key) {
    e = lo.entry;
    ctx->lru.splice(ctx->lru.end(), ctx->lru, lo.lru_pos);
    mp_send_stats& hs = ctx->stats;
    hs.hit = 1;
    hs.cache_hits++;
    hs.creation_us = hs.construction_us = hs.instantiation_us = hs.plan_us = 0.0;
  } else {
    if (capturing && ctx->index.find(key) == ctx->index.end()) throw Error{MP_ERR_STATE, kCaptureMiss};
    e = lookup_entry(ctx, src, dst, size, src_dev, dst_dev, *cfg, user, nullptr, &key);
    lo.key = key;
    lo.entry = e;
    lo.lru_pos = ctx->index.find(key)->second;
    lo.epoch = ctx->cache_epoch;
  }
  mp_send_stats& st = ctx->stats;
  Phys& S = ctx->phys[e->src_phys];
  set_device(S.ordinal);
  // serialise with a send issued on another stream (shared counters/arenas)
  if (!capturing && ctx->have_last && ctx->last_stream != stream)
    CK(cudaStreamWaitEvent(user, ctx->last_done, 0));
  double t_launch = now_us();
  bool timing = !cfg->graph_mode && ctx->kernel_timing && !capturing;
  if (capturing) e->pinned = true;
  if (cfg->graph_mode && e->graph && !pdl_replay(ctx, e) && !capturing) {
    CK(cudaGraphLaunch(e->exec, user));
    st.ce_copies = (int)e->ce.size();
  } else {
    enqueue(ctx, e, user, timing);
    st.ce_copies = (int)e->ce.size();
  }
  if (!capturing) {
    CK(cudaEventRecord(ctx->last_done, user));
    ctx->have_last = true;
    ctx->last_stream = stream;
  }
  st.launch_us = now_us() - t_launch;
  st.graph_mode = cfg->graph_mode ? 1 : 0;
  st.nodes_logical = e->nodes_logical;
  st.nodes_physical = e->nodes_physical;
  st.kernels = (int)e->progs.size();
  st.kernel = MP_KERNEL_NONE;
  for (const Program& pr : e->progs)
    if (pr.phys == e->src_phys) st.kernel = kernel_of(ctx->opts, pr.kind, pr.peer);
  remember_plan(ctx, e);
  return MP_OK;
  GUARD_END
}

int mp_send_many(mp_ctx* ctx, const mp_xfer* xfers, int32_t n, const mp_config* cfg, int32_t joint,
                 void* stream) {
  GUARD_BEGIN
  if (!ctx || !cfg || !xfers || n < 1 || n > 64) return fail(MP_ERR_VALUE, "need 1..64 transfers");
  if (!ctx->has_topo) return fail(MP_ERR_STATE, "context has no topology (mp_ctx_set_topology)");
  if (ctx->group) return fail(MP_ERR_STATE, "group context: use mp_group_send");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  cudaStream_t user = (cudaStream_t)stream;
  const bool capturing = stream_capturing(user);  // see mp_send
  auto& lm = ctx->last_many;
  Entry* e = nullptr;
  if (lm.entry && lm.epoch == ctx->cache_epoch && lm.joint == joint && (int)lm.xfers.size() == n &&
      memcmp(&lm.cfg, cfg, sizeof *cfg) == 0 && memcmp(lm.xfers.data(), xfers, n * sizeof *xfers) == 0) {
    // resend of the last program (windows, halo exchanges): the same raw
    // arguments, already validated, and its entry is still cached — a hit
    // without rebuilding and hashing the key (~20 ns per transfer)
    e = lm.entry;
    ctx->lru.splice(ctx->lru.end(), ctx->lru, lm.lru_pos);
    mp_send_stats& hs = ctx->stats;
    hs.hit = 1;
    hs.cache_hits++;
    hs.creation_us = hs.construction_us = hs.instantiation_us = hs.plan_us = 0.0;
  }
  // otherwise the key is built in a reused buffer (a cached-graph hit
  // allocates nothing)
  thread_local std::string key;
  if (!e) {
    key.assign(1, joint ? 'J' : 'I');
    for (int i = 0; i < n; ++i) {
      const mp_xfer& x = xfers[i];
      if (x.src_dev < 0 || x.src_dev >= (int)ctx->logi.size() || x.dst_dev < 0 ||
          x.dst_dev >= (int)ctx->logi.size())
        return fail(MP_ERR_PLAN, "transfers run between accelerators");
      if (x.size == 0) return fail(MP_ERR_CHUNK, "message size must be >= 1 byte, got 0");
      if (!x.src || !x.dst) return fail(MP_ERR_VALUE, "null buffer");
      append_key(key, x.src, x.dst, x.size, x.src_dev, x.dst_dev, *cfg);
    }
  }
  if (!e) {
    if (capturing && ctx->index.find(key) == ctx->index.end()) throw Error{MP_ERR_STATE, kCaptureMiss};
    e = lookup_entry(
      ctx, xfers[0].src, xfers[0].dst, xfers[0].size, xfers[0].src_dev, xfers[0].dst_dev, *cfg, user,
      [&](const std::string& k) {
        std::vector<Xfer> xs;
        for (int i = 0; i < n; ++i)
          xs.push_back(Xfer{xfers[i].src, xfers[i].dst, xfers[i].size, xfers[i].src_dev, xfers[i].dst_dev, {}});
        if (joint) {  // channel-disjoint staging across the transfers (paths.py:210-242)
          std::vector<std::pair<int, int>> tr;
          for (auto& x : xs) tr.emplace_back(x.sd, x.dd);
          int shared = 0;
          auto sets = plan_contention_free_sets(ctx->topo, tr, *cfg, &shared);
          for (size_t i = 0; i < xs.size(); ++i) xs[i].paths = sets[i];
        }
        return build_entry_multi(ctx, k, xs, *cfg);
      },
      &key);
    lm.xfers.assign(xfers, xfers + n);
    lm.cfg = *cfg;
    lm.joint = joint;
    lm.entry = e;
    lm.lru_pos = ctx->index.find(key)->second;
    lm.epoch = ctx->cache_epoch;
  }
  mp_send_stats& st = ctx->stats;
  Phys& S = ctx->phys[e->src_phys];
  set_device(S.ordinal);
  if (!capturing && ctx->have_last && ctx->last_stream != stream)
    CK(cudaStreamWaitEvent(user, ctx->last_done, 0));
  double t0 = now_us();
  if (capturing) e->pinned = true;
  if (cfg->graph_mode && e->graph && !capturing) CK(cudaGraphLaunch(e->exec, user));
  else enqueue(ctx, e, user, false);
  if (!capturing) {
    CK(cudaEventRecord(ctx->last_done, user));
    ctx->have_last = true;
    ctx->last_stream = stream;
  }
  st.launch_us = now_us() - t0;
  st.graph_mode = cfg->graph_mode ? 1 : 0;
  st.nodes_logical = e->nodes_logical;
  st.nodes_physical = e->nodes_physical;
  st.kernels = (int)e->progs.size();
  st.ce_copies = (int)e->ce.size();
  st.kernel = MP_KERNEL_NONE;
  for (const Program& pr : e->progs)
    if (pr.phys == e->src_phys) st.kernel = kernel_of(ctx->opts, pr.kind, pr.peer);
  remember_plan(ctx, e);
  return MP_OK;
  GUARD_END
}

int mp_send_trace(mp_ctx* ctx, const void* src, void* dst, uint64_t size, int32_t src_dev,
                  int32_t dst_dev, const mp_config* cfg, mp_trace_rec* out, int32_t cap,
                  int32_t* n_out) {
  GUARD_BEGIN
  if (!ctx || !cfg || !n_out) return fail(MP_ERR_VALUE, "null argument");
  if (!ctx->has_topo) return fail(MP_ERR_STATE, "context has no topology (mp_ctx_set_topology)");
  if (ctx->group) return fail(MP_ERR_STATE, "group context: use mp_group_send");
  if (src_dev < 0 || src_dev >= (int)ctx->logi.size() || dst_dev < 0 || dst_dev >= (int)ctx->logi.size())
    return fail(MP_ERR_PLAN, "transfers run between accelerators");
  if (size == 0) return fail(MP_ERR_CHUNK, "message size must be >= 1 byte, got 0");
  if (!src || !dst) return fail(MP_ERR_VALUE, "null buffer");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  mp_config c = *cfg;
  c.graph_mode = 0;  // traced sends run the streamed program
  Phys& S0 = ctx->phys[ctx->logi[src_dev].phys];
  Entry* e = lookup_entry(ctx, src, dst, size, src_dev, dst_dev, c, S0.capture);
  *n_out = e->nodes_logical;
  if (cap < e->nodes_logical || !out) return fail(MP_ERR_CAPACITY, "trace capacity too small");
  Trace tr;
  tr.nodes = e->nodes_logical;
  const size_t np = ctx->phys.size();
  tr.stamps.assign(np, nullptr);
  tr.base.assign(np, nullptr);
  tr.base_ev.assign(np, nullptr);
  std::vector<unsigned long long> init(2 * (size_t)tr.nodes);
  for (int i = 0; i < tr.nodes; ++i) {
    init[2 * i] = ~0ull;
    init[2 * i + 1] = 0ull;
  }
  auto cleanup = [&]() {
    for (size_t ph = 0; ph < np; ++ph) {
      cudaSetDevice(ctx->phys[ph].ordinal);
      if (tr.stamps[ph]) cudaFree(tr.stamps[ph]);
      if (tr.base[ph]) cudaFree(tr.base[ph]);
      if (tr.base_ev[ph]) cudaEventDestroy(tr.base_ev[ph]);
    }
    for (auto& p : tr.ce_ev) {
      if (p.first) cudaEventDestroy(p.first);
      if (p.second) cudaEventDestroy(p.second);
    }
  };
  try {
    for (size_t ph = 0; ph < np; ++ph) {
      CK(cudaSetDevice(ctx->phys[ph].ordinal));
      CK(cudaMalloc(&tr.stamps[ph], init.size() * sizeof(unsigned long long)));
      CK(cudaMemcpy(tr.stamps[ph], init.data(), init.size() * sizeof(unsigned long long),
                    cudaMemcpyHostToDevice));
      CK(cudaMalloc(&tr.base[ph], sizeof(unsigned long long)));
      CK(cudaEventCreate(&tr.base_ev[ph]));
    }
    for (const CeOp& op : e->ce) {
      CK(cudaSetDevice(ctx->phys[op.phys].ordinal));
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      tr.ce_ev.push_back({a, b});
    }
    Phys& S = ctx->phys[e->src_phys];
    CK(cudaSetDevice(S.ordinal));
    if (ctx->have_last) CK(cudaStreamWaitEvent(S.capture, ctx->last_done, 0));
    enqueue(ctx, e, S.capture, false, &tr);
    CK(cudaEventRecord(ctx->last_done, S.capture));
    ctx->have_last = true;
    ctx->last_stream = (void*)S.capture;
    CK(cudaStreamSynchronize(S.capture));
    for (int i = 0; i < tr.nodes; ++i) out[i] = mp_trace_rec{i, -1, -1, 0, 0.0, 0.0};
    for (size_t ph = 0; ph < np; ++ph) {
      CK(cudaSetDevice(ctx->phys[ph].ordinal));
      std::vector<unsigned long long> st(init.size());
      unsigned long long base = 0;
      CK(cudaMemcpy(st.data(), tr.stamps[ph], st.size() * sizeof(unsigned long long),
                    cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&base, tr.base[ph], sizeof base, cudaMemcpyDeviceToHost));
      for (int i = 0; i < tr.nodes; ++i)
        if (st[2 * i] != ~0ull) {
          out[i].engine = MP_ENGINE_SM;
          out[i].device = (int32_t)ph;
          out[i].start_us = ((double)st[2 * i] - (double)base) * 1e-3;
          out[i].end_us = ((double)st[2 * i + 1] - (double)base) * 1e-3;
        }
    }
    for (size_t i = 0; i < e->ce.size(); ++i) {
      const CeOp& op = e->ce[i];
      CK(cudaSetDevice(ctx->phys[op.phys].ordinal));
      float a = 0.f, b = 0.f;
      CK(cudaEventElapsedTime(&a, tr.base_ev[op.phys], tr.ce_ev[i].first));
      CK(cudaEventElapsedTime(&b, tr.base_ev[op.phys], tr.ce_ev[i].second));
      std::vector<uint32_t> nodes = op.nodes.empty() ? std::vector<uint32_t>{op.node} : op.nodes;
      for (uint32_t nd : nodes) {
        mp_trace_rec& r = out[nd];
        r.engine = MP_ENGINE_CE;
        r.device = op.phys;
        r.start_us = a * 1e3;
        r.end_us = b * 1e3;
      }
    }
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  remember_plan(ctx, e);
  return MP_OK;
  GUARD_END
}

int mp_wait(mp_ctx* ctx, void* stream) {
  GUARD_BEGIN
  if (!ctx) return fail(MP_ERR_VALUE, "null argument");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  // inside a caller's capture the sends recorded there are already ordered
  // on the capturing stream, and waiting on the engine's (eager) event
  // would break the capture: nothing to do
  if (stream_capturing((cudaStream_t)stream)) return MP_OK;
  if (ctx->have_last) CK(cudaStreamWaitEvent((cudaStream_t)stream, ctx->last_done, 0));
  return MP_OK;
  GUARD_END
}

int mp_send_stats_get(const mp_ctx* ctx, mp_send_stats* out) {
  if (!ctx || !out) return fail(MP_ERR_VALUE, "null argument");
  *out = ctx->stats;
  return MP_OK;
}

int mp_last_plan(const mp_ctx* ctx, mp_path* paths, int32_t paths_cap, int32_t* n_paths,
                 mp_chunk* chunks, int32_t chunks_cap, int32_t* n_chunks) {
  if (!ctx) return fail(MP_ERR_VALUE, "null argument");
  if (n_paths) *n_paths = (int32_t)ctx->last_paths.size();
  if (n_chunks) *n_chunks = (int32_t)ctx->last_chunks.size();
  if (paths_cap < (int)ctx->last_paths.size() || chunks_cap < (int)ctx->last_chunks.size())
    return fail(MP_ERR_CAPACITY, "plan capacity too small");
  if (paths && !ctx->last_paths.empty())
    memcpy(paths, ctx->last_paths.data(), ctx->last_paths.size() * sizeof(mp_path));
  if (chunks && !ctx->last_chunks.empty())
    memcpy(chunks, ctx->last_chunks.data(), ctx->last_chunks.size() * sizeof(mp_chunk));
  return MP_OK;
}

int mp_cache_clear(mp_ctx* ctx) {
  GUARD_BEGIN
  if (!ctx) return fail(MP_ERR_VALUE, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  clear_cache(ctx);
  return MP_OK;
  GUARD_END
}

int mp_sync(mp_ctx* ctx) {
  GUARD_BEGIN
  if (!ctx) return fail(MP_ERR_VALUE, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  unsigned code = 0;
  int where = -1;
  for (auto& P : ctx->phys) {
    CK(cudaSetDevice(P.ordinal));
    CK(cudaDeviceSynchronize());
    mpk::Ctl c;
    CK(cudaMemcpy(&c, P.ctl, sizeof c, cudaMemcpyDeviceToHost));
    const unsigned h = ((volatile unsigned*)ctx->herr)[&P - ctx->phys.data()];
    if ((c.error || h) && !code) {
      code = c.error ? c.error : h;
      where = P.ordinal;
    }
  }
  if (!code) return MP_OK;
  // Clear the error: a timed-out wait left its chunk's flag / pass counters
  // (and a late hop1 signal may still have landed) — re-zero every flag
  // array and control block so the next program starts from a clean state.
  for (auto& L : ctx->logi)
    if (L.phys >= 0 && L.flags) {
      CK(cudaSetDevice(ctx->phys[L.phys].ordinal));
      CK(cudaMemset(L.flags, 0, (size_t)L.flag_cap * 2 * sizeof(uint32_t)));
    }
  if (GroupState* G = ctx->group) {
    CK(cudaSetDevice(ctx->phys[0].ordinal));
    CK(cudaMemset(G->flags, 0, (size_t)G->flag_cap * 2 * sizeof(uint32_t)));
    CK(cudaMemset(G->sync + 8, 0, 8));  // receiver byte counter
  }
  for (auto& P : ctx->phys) {
    CK(cudaSetDevice(P.ordinal));
    CK(cudaDeviceSynchronize());
    ((volatile unsigned*)ctx->herr)[&P - ctx->phys.data()] = 0u;
    init_ctl(ctx, P);
  }
  return fail(MP_ERR_CUDA, std::string(wait_what(code)) + " timed out on device " + std::to_string(where) +
                               (ctx->group ? " (group barrier state may be inconsistent: recreate the group)" : ""));
  GUARD_END
}

int mp_ctx_set_kernel_timing(mp_ctx* ctx, int32_t on) {
  if (!ctx) return fail(MP_ERR_VALUE, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->kernel_timing = on != 0;
  return MP_OK;
}

int mp_kernel_time_ms(const mp_ctx* ctx, double* ms) {
  GUARD_BEGIN
  if (!ctx || !ms) return fail(MP_ERR_VALUE, "null argument");
  DeviceGuard g;
  if (ctx->timed_phys < 0) return fail(MP_ERR_STATE, "no timed kernel yet (streamed-mode SM send)");
  const Phys& S = ctx->phys[ctx->timed_phys];
  CK(cudaSetDevice(S.ordinal));
  float f = 0.f;
  CK(cudaEventSynchronize(S.kt1));
  CK(cudaEventElapsedTime(&f, S.kt0, S.kt1));
  *ms = f;
  return MP_OK;
  GUARD_END
}

int mp_kernel_bench(mp_ctx* ctx, const void* src, void* dst, uint64_t size, int32_t src_dev,
                    int32_t dst_dev, const mp_config* cfg, int32_t reps, double* ms_per_launch) {
  GUARD_BEGIN
  if (!ctx || !cfg || !ms_per_launch || reps < 1) return fail(MP_ERR_VALUE, "bad arguments");
  if (!ctx->has_topo) return fail(MP_ERR_STATE, "context has no topology (mp_ctx_set_topology)");
  if (ctx->group) return fail(MP_ERR_STATE, "group context");
  if (src_dev < 0 || src_dev >= (int)ctx->logi.size() || dst_dev < 0 || dst_dev >= (int)ctx->logi.size())
    return fail(MP_ERR_PLAN, "transfers run between accelerators");
  if (!src || !dst || size == 0) return fail(MP_ERR_VALUE, "null buffer or empty message");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  mp_config c = *cfg;
  c.graph_mode = 0;
  Phys& S0 = ctx->phys[ctx->logi[src_dev].phys];
  Entry* e = lookup_entry(ctx, src, dst, size, src_dev, dst_dev, c, S0.capture);
  const Program* pr = nullptr;
  for (const auto& p : e->progs)
    if (p.phys == e->src_phys) pr = &p;
  if (!pr) return fail(MP_ERR_STATE, "no SM transfer kernel on the source device for this transfer");
  Phys& S = ctx->phys[e->src_phys];
  CK(cudaSetDevice(S.ordinal));
  CK(cudaDeviceSynchronize());
  // ordinary launches: the kernel's own duration, launch gap included (PDL
  // would overlap each launch with the previous kernel's tail)
  mp_engine_opts o = ctx->opts;
  o.pdl = 0;
  launch_transfer(o, pr->grid, S.kstream, pr->d_tiles, pr->ntiles, S.ctl, pr->nstatic, nullptr,
                  nullptr, pr->peer, S.sms, pr->small.get(), pr->kind, pr->d_sched, pr->nhelp);  // warm
  CK(cudaEventRecord(S.kt0, S.kstream));
  for (int i = 0; i < reps; ++i)
    launch_transfer(o, pr->grid, S.kstream, pr->d_tiles, pr->ntiles, S.ctl, pr->nstatic, nullptr,
                    nullptr, pr->peer, S.sms, pr->small.get(), pr->kind, pr->d_sched, pr->nhelp);
  CK(cudaEventRecord(S.kt1, S.kstream));
  CK(cudaEventSynchronize(S.kt1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, S.kt0, S.kt1));
  *ms_per_launch = ms / reps;
  return MP_OK;
  GUARD_END
}

int mp_measure_paths(mp_ctx* ctx, int32_t src_dev, int32_t dst_dev, uint64_t bytes, int32_t iters,
                     double* out_gbps, int32_t cap) {
  GUARD_BEGIN
  if (!ctx || !out_gbps || cap < 4) return fail(MP_ERR_VALUE, "need 4 output slots");
  if (src_dev < 0 || dst_dev < 0 || src_dev >= (int)ctx->logi.size() || dst_dev >= (int)ctx->logi.size())
    return fail(MP_ERR_VALUE, "device out of range");
  if (bytes == 0 || iters < 1) return fail(MP_ERR_VALUE, "bytes and iters must be positive");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  Phys& S = ctx->phys[ctx->logi[src_dev].phys];
  Phys& D = ctx->phys[ctx->logi[dst_dev].phys];
  uint8_t *a = nullptr, *b = nullptr, *h = nullptr;
  CK(cudaSetDevice(S.ordinal));
  CK(cudaMalloc(&a, bytes));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(D.ordinal));
  CK(cudaMalloc(&b, bytes));
  CK(cudaHostAlloc((void**)&h, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  auto time_it = [&](Phys& P, auto&& fn) {
    CK(cudaSetDevice(P.ordinal));
    fn(P.kstream);  // warm-up
    CK(cudaEventRecord(P.kt0, P.kstream));
    for (int i = 0; i < iters; ++i) fn(P.kstream);
    CK(cudaEventRecord(P.kt1, P.kstream));
    CK(cudaEventSynchronize(P.kt1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, P.kt0, P.kt1));
    return (double)bytes * iters / (ms * 1e-3) / 1e9;
  };
  // direct: the SM transfer kernel over one tile table (same code as mp_send)
  std::vector<mpk::Tile> flat;
  uint64_t tile = auto_tile_bytes(ctx, bytes, S.sms);
  for (uint64_t o = 0; o < bytes; o += tile) {
    mpk::Tile t{};
    t.src = (uint64_t)(uintptr_t)(a + o);
    t.dst = (uint64_t)(uintptr_t)(b + o);
    t.len = std::min(tile, bytes - o);
    flat.push_back(t);
  }
  mpk::Tile* dt = nullptr;
  CK(cudaSetDevice(S.ordinal));
  CK(cudaMalloc(&dt, flat.size() * sizeof(mpk::Tile)));
  CK(cudaMemcpy(dt, flat.data(), flat.size() * sizeof(mpk::Tile), cudaMemcpyHostToDevice));
  CK(cudaStreamSynchronize(cudaStreamLegacy));
  unsigned grid = (unsigned)std::min<uint64_t>(flat.size(), (uint64_t)S.sms * ctx->opts.ctas_per_sm);
  out_gbps[0] = time_it(S, [&](cudaStream_t s) {
    launch_transfer(ctx->opts, grid, s, dt, (unsigned)flat.size(), S.ctl, grid);
  });
  out_gbps[1] = time_it(S, [&](cudaStream_t s) { cudaMemcpyAsync(h, a, bytes, cudaMemcpyDeviceToHost, s); });
  out_gbps[2] = time_it(D, [&](cudaStream_t s) { cudaMemcpyAsync(b, h, bytes, cudaMemcpyHostToDevice, s); });
  out_gbps[3] = time_it(S, [&](cudaStream_t s) { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDefault, s); });
  if (cap >= 8) {
    // out[6] / out[7]: the SM transfer kernel writing to / reading from mapped
    // pinned host memory over PCIe (the SM variant of the host-staged hops)
    uint8_t* hd = nullptr;
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    auto sm_copy = [&](uint8_t* from, uint8_t* to) {
      std::vector<mpk::Tile> ft;
      uint64_t tl = std::min<uint64_t>(auto_tile_bytes(ctx, bytes, S.sms), kHostTileBytes);
      for (uint64_t o = 0; o < bytes; o += tl) {
        mpk::Tile t{};
        t.src = (uint64_t)(uintptr_t)(from + o);
        t.dst = (uint64_t)(uintptr_t)(to + o);
        t.len = std::min(tl, bytes - o);
        ft.push_back(t);
      }
      mpk::Tile* d = nullptr;
      CK(cudaSetDevice(S.ordinal));
      CK(cudaMalloc(&d, ft.size() * sizeof(mpk::Tile)));
      CK(cudaMemcpy(d, ft.data(), ft.size() * sizeof(mpk::Tile), cudaMemcpyHostToDevice));
      CK(cudaStreamSynchronize(cudaStreamLegacy));
      unsigned gr = (unsigned)std::min<uint64_t>(ft.size(), (uint64_t)S.sms * ctx->opts.ctas_per_sm);
      double r = time_it(S, [&](cudaStream_t s) {
        launch_transfer(ctx->opts, gr, s, d, (unsigned)ft.size(), S.ctl, gr);
      });
      cudaFree(d);
      return r;
    };
    out_gbps[6] = sm_copy(a, hd);
    out_gbps[7] = sm_copy(hd, b);
  }
  if (cap >= 6) {
    // out[4]: D2H and H2D running at the same time (full duplex), per direction
    // out[5]: the host-staged path as the engine runs it: 8 pipelined chunks,
    //         D2H on one lane, H2D on another after a per-chunk event
    cudaStream_t l0 = lane_stream(S, 0), l1 = lane_stream(D, 1);
    const int kc = 8;
    const uint64_t chunk = (bytes / kc + 15) & ~(uint64_t)15;
    std::vector<cudaEvent_t> ev(kc);
    for (auto& e : ev) e = take_event(S);
    cudaEvent_t fork = take_event(S), join = take_event(D);
    auto round = [&](bool staged) {
      CK(cudaSetDevice(S.ordinal));
      CK(cudaEventRecord(fork, S.kstream));
      CK(cudaStreamWaitEvent(l0, fork, 0));
      CK(cudaSetDevice(D.ordinal));
      CK(cudaStreamWaitEvent(l1, fork, 0));
      for (int c = 0; c < kc; ++c) {
        uint64_t off = (uint64_t)c * chunk;
        if (off >= bytes) break;
        uint64_t n = std::min(chunk, bytes - off);
        CK(cudaSetDevice(S.ordinal));
        CK(cudaMemcpyAsync(h + off, a + off, n, cudaMemcpyDeviceToHost, l0));
        CK(cudaEventRecord(ev[c], l0));
        CK(cudaSetDevice(D.ordinal));
        if (staged) CK(cudaStreamWaitEvent(l1, ev[c], 0));
        // full-duplex probe: H2D reads a different half-buffer region concurrently
        CK(cudaMemcpyAsync(b + off, staged ? h + off : h + (bytes - off - n), n,
                           cudaMemcpyHostToDevice, l1));
      }
      CK(cudaEventRecord(join, l1));
      CK(cudaSetDevice(S.ordinal));
      CK(cudaStreamWaitEvent(S.kstream, join, 0));
      CK(cudaStreamWaitEvent(S.kstream, ev[kc - 1], 0));
    };
    S.next_event = 0;
    double duplex = time_it(S, [&](cudaStream_t) { round(false); });
    double staged = time_it(S, [&](cudaStream_t) { round(true); });
    out_gbps[4] = duplex;
    out_gbps[5] = staged;
    S.next_event = 0;
    D.next_event = 0;
  }
  CK(cudaGetLastError());
  CK(cudaSetDevice(S.ordinal));
  CK(cudaDeviceSynchronize());
  cudaFree(dt);
  cudaFree(a);
  cudaSetDevice(D.ordinal);
  cudaFree(b);
  cudaFreeHost(h);
  return MP_OK;
  GUARD_END
}

int mp_ipc_export(const void* dev_ptr, int32_t device, uint8_t* handle_out, uint64_t* offset_out) {
  GUARD_BEGIN
  if (!dev_ptr || !handle_out) return fail(MP_ERR_VALUE, "null argument");
  DeviceGuard g;
  CK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == MP_IPC_HANDLE_BYTES, "ipc handle size");
  memcpy(handle_out, &h, sizeof h);
  if (offset_out) *offset_out = (uint64_t)(uintptr_t)dev_ptr - allocation_base(dev_ptr);
  return MP_OK;
  GUARD_END
}

int mp_ipc_import(const uint8_t* handle, int32_t device, void** dev_ptr_out) {
  GUARD_BEGIN
  if (!handle || !dev_ptr_out) return fail(MP_ERR_VALUE, "null argument");
  DeviceGuard g;
  CK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  CK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return MP_OK;
  GUARD_END
}

int mp_ipc_close(void* dev_ptr, int32_t device) {
  GUARD_BEGIN
  DeviceGuard g;
  CK(cudaSetDevice(device));
  CK(cudaIpcCloseMemHandle(dev_ptr));
  return MP_OK;
  GUARD_END
}

int mp_group_create(int32_t nranks, int32_t rank, int32_t device, uint64_t stage_bytes,
                    int32_t flag_cap, mp_ctx** out) {
  GUARD_BEGIN
  if (!out || nranks < 1 || nranks > mpk::kMaxRanks || rank < 0 || rank >= nranks || flag_cap < 1)
    return fail(MP_ERR_VALUE, "bad group arguments (1 <= nranks <= 16, 0 <= rank < nranks)");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MP_ERR_VALUE, "device is not a CUDA device");
  DeviceGuard g;
  std::vector<int32_t> map(1, device);
  mp_ctx* ctx = nullptr;
  int rc = mp_ctx_create(1, map.data(), &ctx);
  if (rc) return rc;
  Logi local = ctx->logi[0];
  ctx->logi.assign(nranks, Logi{});
  for (auto& L : ctx->logi) L.phys = -1;
  ctx->logi[rank] = local;
  auto* G = new GroupState();
  ctx->group = G;
  G->rank = rank;
  G->nranks = nranks;
  G->flag_cap = flag_cap;
  G->stage_cap = stage_bytes ? stage_bytes : 1;
  G->peer_stage.assign(nranks, nullptr);
  G->peer_sync.assign(nranks, nullptr);
  G->peer_flags.assign(nranks, nullptr);
  G->peer_stage_cap.assign(nranks, 0);
  G->peer_host.assign(nranks, nullptr);
  G->peer_host_dev.assign(nranks, nullptr);
  G->peer_host_cap.assign(nranks, 0);
  try {
    CK(cudaSetDevice(device));
    CK(cudaMalloc(&G->stage, G->stage_cap));
    CK(cudaMalloc(&G->flags, (size_t)flag_cap * 2 * sizeof(uint32_t)));
    CK(cudaMemset(G->flags, 0, (size_t)flag_cap * 2 * sizeof(uint32_t)));
    CK(cudaMalloc(&G->sync, 256));
    CK(cudaMemset(G->sync, 0, 256));
    CK(cudaDeviceSynchronize());
  } catch (...) {
    mp_ctx_destroy(ctx);
    throw;
  }
  *out = ctx;
  return MP_OK;
  GUARD_END
}

int mp_group_host_arena(mp_ctx* ctx, uint64_t bytes) {
  GUARD_BEGIN
  if (!ctx || !ctx->group) return fail(MP_ERR_VALUE, "not a group context");
  GroupState* G = ctx->group;
  if (bytes == 0) return fail(MP_ERR_VALUE, "host inbox size must be >= 1 byte");
  if (G->host) return fail(MP_ERR_STATE, "the host inbox is already set up");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  CK(cudaSetDevice(ctx->phys[0].ordinal));
  static std::atomic<unsigned> serial{0};
  const std::string name = "/mpb200_" + std::to_string((long)getpid()) + "_" + std::to_string(G->rank) +
                           "_" + std::to_string(serial++);
  map_host_inbox(name.c_str(), bytes, true, &G->host, &G->host_dev);
  G->host_cap = bytes;
  G->host_name = name;
  return MP_OK;
  GUARD_END
}

int mp_group_export(const mp_ctx* ctx, uint8_t* blob) {
  GUARD_BEGIN
  if (!ctx || !ctx->group || !blob) return fail(MP_ERR_VALUE, "not a group context");
  const GroupState* G = ctx->group;
  DeviceGuard g;
  CK(cudaSetDevice(ctx->phys[0].ordinal));
  GroupBlob b{};
  b.stage_cap = G->stage_cap;
  b.flag_cap = G->flag_cap;
  b.rank = G->rank;
  CK(cudaIpcGetMemHandle(&b.stage, G->stage));
  CK(cudaIpcGetMemHandle(&b.flags, G->flags));
  CK(cudaIpcGetMemHandle(&b.sync, G->sync));
  b.host_cap = G->host_cap;
  snprintf(b.host_name, sizeof b.host_name, "%s", G->host_name.c_str());
  memset(blob, 0, MP_GROUP_BLOB_BYTES);
  memcpy(blob, &b, sizeof b);
  return MP_OK;
  GUARD_END
}

int mp_group_import(mp_ctx* ctx, int32_t rank, const uint8_t* blob) {
  GUARD_BEGIN
  if (!ctx || !ctx->group || !blob) return fail(MP_ERR_VALUE, "not a group context");
  GroupState* G = ctx->group;
  if (rank < 0 || rank >= G->nranks) return fail(MP_ERR_VALUE, "rank out of range");
  if (rank == G->rank) return MP_OK;
  GroupBlob b;
  memcpy(&b, blob, sizeof b);
  if (b.rank != rank) return fail(MP_ERR_VALUE, "blob belongs to another rank");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  CK(cudaSetDevice(ctx->phys[0].ordinal));
  clear_cache(ctx);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, b.stage, cudaIpcMemLazyEnablePeerAccess));
  G->peer_stage[rank] = (uint8_t*)p;
  CK(cudaIpcOpenMemHandle(&p, b.flags, cudaIpcMemLazyEnablePeerAccess));
  G->peer_flags[rank] = (uint32_t*)p;
  CK(cudaIpcOpenMemHandle(&p, b.sync, cudaIpcMemLazyEnablePeerAccess));
  G->peer_sync[rank] = (uint8_t*)p;
  G->peer_stage_cap[rank] = b.stage_cap;
  G->flag_cap = std::min(G->flag_cap, (int)b.flag_cap);
  if (b.host_cap && !G->peer_host[rank]) {
    b.host_name[sizeof b.host_name - 1] = 0;
    map_host_inbox(b.host_name, b.host_cap, false, &G->peer_host[rank], &G->peer_host_dev[rank]);
    G->peer_host_cap[rank] = b.host_cap;
  }
  return MP_OK;
  GUARD_END
}

int mp_group_open(mp_ctx* ctx, const uint8_t* handle, uint64_t offset, void** ptr) {
  GUARD_BEGIN
  if (!ctx || !ctx->group || !handle || !ptr) return fail(MP_ERR_VALUE, "not a group context");
  GroupState* G = ctx->group;
  std::lock_guard<std::mutex> lk(ctx->mu);
  std::string k((const char*)handle, MP_IPC_HANDLE_BYTES);
  auto it = G->opened.find(k);
  if (it == G->opened.end()) {
    DeviceGuard g;
    CK(cudaSetDevice(ctx->phys[0].ordinal));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    it = G->opened.emplace(k, base).first;
  }
  *ptr = (uint8_t*)it->second + offset;
  return MP_OK;
  GUARD_END
}

int mp_group_send(mp_ctx* ctx, const void* src, uint32_t src_align, void* dst, uint64_t size,
                  int32_t src_rank, int32_t dst_rank, const mp_config* cfg, void* stream) {
  GUARD_BEGIN
  if (!ctx || !ctx->group || !cfg) return fail(MP_ERR_VALUE, "not a group context");
  GroupState* G = ctx->group;
  if (!ctx->has_topo) return fail(MP_ERR_STATE, "context has no topology (mp_ctx_set_topology)");
  if (src_rank < 0 || src_rank >= G->nranks || dst_rank < 0 || dst_rank >= G->nranks)
    return fail(MP_ERR_PLAN, "transfers run between accelerators");
  if (size == 0) return fail(MP_ERR_CHUNK, "message size must be >= 1 byte, got 0");
  if (G->rank == src_rank && !src) return fail(MP_ERR_VALUE, "the sender needs its source buffer");
  for (int q = 0; q < G->nranks; ++q)
    if (q != G->rank && !G->peer_sync[q]) return fail(MP_ERR_STATE, "group peers not imported");
  check_sticky(ctx);
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g;
  cudaStream_t user = (cudaStream_t)stream;
  // the device-side barrier counts transfers as they run; a captured
  // transfer replayed out of step with the other ranks would desynchronise it
  if (stream_capturing(user))
    return fail(MP_ERR_STATE, "group transfers cannot be captured into a CUDA graph (the ranks' device barrier "
                              "counts transfers as they run)");
  const void* ksrc = G->rank == src_rank ? src : nullptr;
  Entry* e = lookup_entry(ctx, ksrc, dst, size ^ ((uint64_t)src_align << 58), src_rank, dst_rank, *cfg,
                          user, [&](const std::string& key) {
                            return build_group_entry(ctx, key, ksrc, src_align & 15u, dst, size,
                                                     src_rank, dst_rank, *cfg);
                          });
  mp_send_stats& st = ctx->stats;
  CK(cudaSetDevice(ctx->phys[0].ordinal));
  if (ctx->have_last && ctx->last_stream != stream) CK(cudaStreamWaitEvent(user, ctx->last_done, 0));
  double t0 = now_us();
  if (cfg->graph_mode && e->graph) CK(cudaGraphLaunch(e->exec, user));
  else enqueue(ctx, e, user, false);
  CK(cudaEventRecord(ctx->last_done, user));
  ctx->have_last = true;
  ctx->last_stream = stream;
  st.launch_us = now_us() - t0;
  st.graph_mode = cfg->graph_mode ? 1 : 0;
  st.nodes_logical = e->nodes_logical;
  st.nodes_physical = e->nodes_physical;
  st.kernels = 1;
  st.ce_copies = 0;
  st.kernel = e->progs.empty() ? MP_KERNEL_NONE : kernel_of(ctx->opts, e->progs[0].kind, e->progs[0].peer);
  remember_plan(ctx, e);
  return MP_OK;
  GUARD_END
}

int mp_group_role(const mp_ctx* ctx, int32_t* role) {
  if (!ctx || !ctx->group || !role) return fail(MP_ERR_VALUE, "not a group context");
  std::lock_guard<std::mutex> lk(const_cast<mp_ctx*>(ctx)->mu);
  *role = ctx->lru.empty() ? -1 : ctx->lru.back()->grole;
  return MP_OK;
}

}  // extern "C"
