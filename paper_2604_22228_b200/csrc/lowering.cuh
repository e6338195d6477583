// lowering.cuh — internal to mp_engine.cu (included once, after
// engine_state.cuh): tiling constants and tile cuts, and the Lowering of one
// or more transfers into per-device tile tables (SM kernels) and copy-engine
// ops, uploaded as the programs of a cache entry.
#pragma once

namespace {

// Host-path tiles stay small so many CTAs keep PCIe requests in flight.
constexpr uint64_t kHostTileBytes = 64 << 10;
// A host-staged chunk up to this size, with source and destination on one
// device, moves as ONE roundtrip tile (mpk::TILE_ROUNDTRIP: hop1, CTA
// barrier, hop2 in one CTA) — no flag, no system-scope release, no wait, so
// the table keeps its static schedule; larger chunks are cut into hop1 /
// hop2 tiles handed off through the chunk's flag (chunk-level hop ordering
// of the reference's trace needs the whole chunk's hop1 before any hop2).
constexpr uint64_t kRoundtripMaxBytes = 64 << 10;

// Rounds between a relay chunk's hop1 and hop2 tiles in one table (loopback,
// or a relay sharing the source GPU): hop2 of round r queues after round
// r + kHop2Delay.  Round 1 (system-scope flags) measured delay 3 ahead of 1;
// with GPU-scope flags and the batched copy remainder, delay 1 is ahead of
// 0 / 2 / 3 / 5 by 0.5-1.2% across 1-6 relays (tools/exp_relay2.py: 0.971 /
// 0.972 / 0.963 of the loopback roofline at 1 / 2 / 3 relays, delay 0
// 0.81-0.92: hop2 tiles then wait).  Cross-device relays are unaffected
// (the relay's table holds only hop2 tiles).
constexpr uint64_t kHop2Delay = 1;

// Helper-warp roundtrips of messages from this size on end with a
// system-scope fence (mpk::TILE_FENCE): the host writes retire inside the
// direct stream instead of in the grid-completion flush the next
// (programmatic-dependent) launch waits for.  Below it the fence outlasts
// the message's copy.  Direct + host k=8 over single path, fence off -> on
// (tools/exp_rtfence.py, profiles/r02_exp_rtfence.jsonl): 8 MiB 0.82 ->
// 0.65, 16 MiB 0.78-0.85 -> 0.74-0.85 (box-dependent), 20 MiB even,
// 24 MiB 0.82 -> 0.96, 32 MiB 0.97 -> 0.99, 48-92 MiB 0.99 -> 1.00.
// MP_RT_FENCE_MIN overrides it (experiments).
constexpr uint64_t kRoundtripFenceMinBytes = 20ull << 20;
inline uint64_t rt_fence_min_bytes() {
  const char* e = std::getenv("MP_RT_FENCE_MIN");
  return e ? (uint64_t)std::strtoull(e, nullptr, 10) : kRoundtripFenceMinBytes;
}

// cudaMemcpy2D pitches stay below the device's maximum pitch (2^31 - 1 class)
constexpr uint64_t kMaxCopyPitch = 1ull << 30;

// CE host path batching: the host chunks of a transfer move as
// ceil(host bytes / kHostGroupBytes) (<= kHostMaxGroups) 2-D copy groups,
// D2H of group g+1 overlapping H2D of group g.  Measured (tools/
// exp_hostlanes.py, direct + host k=8, window 64): one group instead of 8
// per-chunk D2H/H2D pairs lifts 16 MiB 340 -> 720 GB/s and 128 MiB 1912 ->
// 2856; a 4-group pipeline pays off only when the host share is large.
constexpr uint64_t kHostGroupBytes = 2 << 20;
constexpr int kHostMaxGroups = 4;

// Smallest tile of a static (one-tile-per-CTA) table: below this a message
// spreads over fewer CTAs rather than into sub-4 KiB slivers.
constexpr uint64_t kStaticMinTile = 4096;
// Largest per-CTA share of a static table.  Measured crossover (loopback,
// tools/abi_latency.cu): static wins up to 64 MiB (16 MiB: 6.2 vs 10.2 us per
// message), dynamic claims win from 128 MiB (512 MiB: 166.8 vs 178.2 us) —
// per-SM copy rates are not uniform enough for one fixed share per CTA.
constexpr uint64_t kStaticMaxPerCta = 640 << 10;
// Default ceiling of the small-message kernel (engine opts small_max_bytes):
// measured 1 launch slot up to 64 KiB, 3.0 us at 1 MiB (TMA kernel 4.1),
// a tie at 4 MiB, and 8.2 vs 6.2 us at 16 MiB (tools/abi_latency.cu).
constexpr int64_t kSmallMaxBytes = 4 << 20;

uint64_t auto_tile_bytes(const mp_ctx* ctx, uint64_t path_bytes, int sms) {
  if (ctx->opts.tile_bytes > 0) return (uint64_t)ctx->opts.tile_bytes;
  // aim for >= 12 tiles per resident CTA (the tail is at most one tile),
  // 32 .. 256 KiB, multiple of 4 KiB; the TMA stream is continuous across
  // tiles so small tiles cost only a claim + a prefetched descriptor
  uint64_t ctas = (uint64_t)sms * std::max(1, ctx->opts.ctas_per_sm);
  uint64_t t = path_bytes / (ctas * 12);
  t = std::max<uint64_t>(t, 32 << 10);
  t = std::min<uint64_t>(t, 256 << 10);
  return (t + 4095) & ~(uint64_t)4095;
}

// Interior tile boundaries of [0, len): every `tile` bytes, moved down to a
// 128-byte-aligned destination address (a whole L2 line) so only a chunk's
// first and last tiles carry an unaligned head/tail and every interior tile
// moves whole lines (chunk offsets are mostly unaligned, pipeline.py:66-77;
// 16-byte cuts measured +2.6% at 128 MiB over 9 chunks).
std::vector<uint64_t> tile_cuts(uint64_t dst, uint64_t len, uint64_t tile) {
  std::vector<uint64_t> cuts{0};
  uint64_t o = 0;
  while (len - o > tile) {
    uint64_t next = o + tile;
    uint64_t adj = next - ((dst + next) & 127u);
    if (adj > o) next = adj;
    cuts.push_back(next);
    o = next;
  }
  cuts.push_back(len);
  return cuts;
}

// Split [src, src+len) -> dst into tiles appended to `out`.
void append_tiles(std::vector<std::pair<std::pair<uint64_t, uint64_t>, mpk::Tile>>& out,
                  uint64_t order, uint64_t src, uint64_t dst, uint64_t len, uint64_t tile,
                  const mpk::Tile& proto) {
  auto cuts = tile_cuts(dst, len, tile);
  for (size_t i = 0; i + 1 < cuts.size(); ++i) {
    mpk::Tile t = proto;
    t.src = src + cuts[i];
    t.dst = dst + cuts[i];
    t.len = cuts[i + 1] - cuts[i];
    out.push_back({{order, out.size()}, t});
  }
}

uint64_t ntiles_of(uint64_t dst, uint64_t len, uint64_t tile) {
  return tile_cuts(dst, len, tile).size() - 1;
}

// One transfer of a (possibly multi-transfer) program.
struct Xfer {
  const void* src;
  void* dst;
  uint64_t size;
  int sd, dd;                  // logical source / destination
  std::vector<mp_path> paths;  // pre-planned (joint planning) or empty
};

// Lowering of one or more transfers to device programs and copy-engine ops:
// ONE tile table (one kernel) per physical device for every NVLink/HBM
// chunk-hop of every transfer, interleaved round by round so concurrent
// transfers progress together; copy-engine lanes per (transfer, path, hop).
// Steps: plan (chunk plans, per-path sizes, engines, arenas) -> schedule
// (peer tables, static vs dynamic tables) -> lower every chunk-hop -> upload.
class Lowering {
 public:
  Lowering(mp_ctx* ctx, const std::string& key, std::vector<Xfer> xs)
      : ctx_(ctx), o_(ctx->opts), xs_(std::move(xs)), e_(new Entry()) {
    e_->key = key;
  }
  ~Lowering() {  // frees a half-built entry (and its device tables) on error
    if (e_) destroy_entry(ctx_, e_);
  }
  Lowering(const Lowering&) = delete;
  Lowering& operator=(const Lowering&) = delete;
  Entry* build(const mp_config& cfg) {
    plan(cfg);
    schedule();
    tiles_.assign(ctx_->phys.size(), {});
    helpers_.assign(ctx_->phys.size(), {});
    stage_cursor_.assign(ctx_->logi.size(), 0);
    for (int t = 0; t < (int)xs_.size(); ++t) lower_transfer(t);
    upload();
    Entry* r = e_;
    e_ = nullptr;
    return r;
  }

 private:
  struct PathInfo {
    uint64_t bytes = 0, nominal = 0;
    int count = 0;
  };
  struct Engines {
    bool direct_sm, relay_sm, host_sm;
    int host_slots;
  };
  // one CE host-path chunk, batched into 2-D copies (emit_host_groups)
  struct HostRow {
    uint64_t off, len;
    int seq;
    uint32_t n_a, n_b;
    int p;
  };
  using TileList = std::vector<std::pair<std::pair<uint64_t, uint64_t>, mpk::Tile>>;

  mp_ctx* ctx_;
  const mp_engine_opts& o_;
  std::vector<Xfer> xs_;
  Entry* e_;
  std::vector<std::vector<mp_chunk>> chunks_;
  std::vector<int> chunk_base_;
  std::vector<std::vector<PathInfo>> info_;
  std::vector<Engines> eng_;
  std::vector<char> peer_phys_;
  std::vector<uint64_t> static_tile_;
  std::vector<int> static_kind_;
  std::vector<TileList> tiles_;
  // host-path tiles of a static TMA table, worked by the helper warps
  // (transfer_kernel nhelp); folded into the front of the table otherwise
  std::vector<std::vector<mpk::Tile>> helpers_;
  std::vector<uint64_t> stage_cursor_;  // shared relay arenas
  uint64_t host_cursor_ = 0;            // shared pinned arena
  uint32_t node_ = 0;  // logical node id of a chunk's first hop (graph.py:97-117), global
  int lane_next_ = 0;
  bool faulted_ = false;  // opts.fault_inject: one staged chunk's hop1 already muted

  // Testing only (opts.fault_inject & 2): lower as if every logical device
  // had its own GPU — system-scope flags, host chunks as hop1 / hop2 tiles
  // (no roundtrip tiles) — so the cross-device mechanics run on one GPU.
  bool same_gpu(int a, int b) const { return a == b && (o_.fault_inject & 2) == 0; }

  // Testing only (opts.fault_inject & 1): the first staged chunk's hop1
  // tiles never signal, so its hop2 wait times out (sticky-error tests).
  uint32_t* hop1_signal(uint32_t* flag) {
    if ((o_.fault_inject & 1) == 0 || faulted_) return flag;
    faulted_ = true;
    return nullptr;
  }

  int phys_of(int logical) const { return ctx_->logi[logical].phys; }
  int new_event(int phys) {
    e_->ev_phys.push_back(phys);
    return (int)e_->ev_phys.size() - 1;
  }

  // Chunk plans (bit-exact planner), per-path byte counts, the measured
  // per-size engine choice, and the relay / host / flag arenas they need.
  void plan(const mp_config& cfg) {
    const int T = (int)xs_.size();
    if (T < 1 || T > 64) throw Error{MP_ERR_VALUE, "1..64 transfers per program"};
    chunks_.resize(T);
    chunk_base_.assign(T, 0);
    int total_chunks = 0;
    for (int t = 0; t < T; ++t) {
      if (xs_[t].paths.empty()) xs_[t].paths = plan_paths(ctx_->topo, xs_[t].sd, xs_[t].dd, cfg);
      chunks_[t] = make_chunk_plan(xs_[t].paths.data(), (int)xs_[t].paths.size(),
                                   (int64_t)xs_[t].size, cfg.max_chunks);
      chunk_base_[t] = total_chunks;
      total_chunks += (int)chunks_[t].size();
      for (const mp_chunk& c : chunks_[t]) e_->nodes_logical += xs_[t].paths[c.path_index].nhops;
    }
    e_->paths = xs_[0].paths;
    e_->chunks = chunks_[0];
    e_->src_phys = phys_of(xs_[0].sd);

    info_.resize(T);
    eng_.resize(T);
    std::vector<size_t> stage_need(ctx_->logi.size(), 0);
    std::vector<char> flag_devs(ctx_->logi.size(), 0);
    size_t host_need = 0;
    for (int t = 0; t < T; ++t) {
      const auto& paths = xs_[t].paths;
      info_[t].assign(paths.size(), PathInfo{});
      for (const mp_chunk& c : chunks_[t]) {
        PathInfo& pi = info_[t][c.path_index];
        pi.bytes += c.length;
        pi.nominal = std::max<uint64_t>(pi.nominal, c.length);
        pi.count += 1;
      }
      // engines per path type for this message size (measured policy)
      const bool sm_ok = xs_[t].size >= (uint64_t)o_.sm_min_bytes;
      int direct_engine = o_.direct_engine, host_engine = o_.host_engine;
      for (const auto& rule : ctx_->size_policy)
        if (xs_[t].size <= rule.max_bytes) {
          direct_engine = rule.direct;
          if (rule.host >= 0) host_engine = rule.host;
          break;
        }
      // MP_ENGINE_AUTO (the default) for the host path: the SM kernels when
      // every host chunk is one roundtrip tile (<= kRoundtripMaxBytes: the
      // hops ride inside the direct stream's launch), copy engines for
      // larger host chunks (a bandwidth-sized PCIe share: 2-D CE copies
      // measured ~10% ahead of SM-driven PCIe at 128-256 MiB)
      uint64_t host_nominal = 0;
      for (size_t p = 0; p < xs_[t].paths.size(); ++p)
        if (xs_[t].paths[p].kind == MP_PATH_HOST) host_nominal = info_[t][p].nominal;
      const bool host_sm = host_engine == MP_ENGINE_SM ||
                           (host_engine == MP_ENGINE_AUTO && host_nominal <= kRoundtripMaxBytes);
      eng_[t] = Engines{direct_engine == MP_ENGINE_SM && sm_ok, o_.relay_engine == MP_ENGINE_SM && sm_ok,
                        host_sm && sm_ok, 0};
      for (size_t p = 0; p < paths.size(); ++p) {
        const PathInfo& pi = info_[t][p];
        if (paths[p].kind == MP_PATH_GPU) {
          stage_need[paths[p].stage] += pi.bytes + 128 * (size_t)pi.count;
          if (eng_[t].relay_sm) flag_devs[paths[p].stage] = 1;
        }
        if (paths[p].kind == MP_PATH_HOST) {
          // the SM host path keeps every chunk resident (its share is a few MB)
          eng_[t].host_slots = (o_.host_slots > 0 && !eng_[t].host_sm) ? std::min(o_.host_slots, pi.count)
                                                                       : pi.count;
          host_need += eng_[t].host_slots < pi.count ? (size_t)eng_[t].host_slots * pi.nominal
                                                     : pi.bytes + 256 * (size_t)pi.count;
          if (eng_[t].host_sm) flag_devs[xs_[t].dd] = 1;
        }
      }
    }
    ensure_arenas(ctx_, stage_need, flag_devs, total_chunks, host_need);
  }

  // CTAs of a device's dynamic kernel.
  uint64_t grid_of(size_t ph) const {
    const bool vp = vec_peer(o_, peer_phys_[ph] != 0);
    int per_sm = vp ? kPeerCtasPerSm : std::max(1, o_.ctas_per_sm);
    if (o_.copy_kind == MP_COPY_TMA && !vp)  // rings that fit one SM
      per_sm = std::min<int>(per_sm, std::max<int>(1, (int)((227u << 10) / kernel_smem(o_))));
    return (uint64_t)ctx_->phys[ph].sms * per_sm;
  }

  // Tile bytes of a chunk-hop executed on device `ph`.
  uint64_t tile_for(int ph, uint64_t path_bytes) const {
    if (static_tile_[ph]) return static_tile_[ph];
    if (o_.tile_bytes == 0 && (o_.copy_kind == MP_COPY_VEC || vec_peer(o_, peer_phys_[ph] != 0)))
      return kVecTileBytes;
    return auto_tile_bytes(ctx_, path_bytes, ctx_->phys[ph].sms);
  }

  // Peer tables (tiles that touch another GPU's memory over NVLink, see
  // launch_transfer) and the static schedule (MP_SCHED_AUTO): a device whose
  // tiles never wait on a flag and never touch host memory, and whose share
  // is <= kStaticMaxPerCta per SM, gets ONE tile per SM — tile bytes = its SM
  // bytes over (SMs - 2 x segments), so cutting every chunk-hop segment still
  // yields <= SMs tiles.  Those kernels run with no claim atomics and no exit
  // protocol.  Devices with waits or PCIe tiles keep dynamic claims.
  void schedule() {
    const size_t nph = ctx_->phys.size();
    const int T = (int)xs_.size();
    peer_phys_.assign(nph, 0);
    for (int t = 0; t < T; ++t) {
      const int sp = phys_of(xs_[t].sd), dp = phys_of(xs_[t].dd);
      if (sp != dp) peer_phys_[o_.pull ? dp : sp] = 1;
      for (const mp_path& P : xs_[t].paths)
        if (P.kind == MP_PATH_GPU) {
          const int rp = phys_of(P.stage);
          if (rp != sp) peer_phys_[sp] = 1;
          if (rp != dp) peer_phys_[rp] = 1;
        }
    }
    static_tile_.assign(nph, 0);
    static_kind_.assign(nph, PROG_DYNAMIC);
    if (o_.sched != MP_SCHED_AUTO || o_.tile_bytes != 0) return;
    std::vector<uint64_t> sm_bytes(nph, 0);
    std::vector<int> segs(nph, 0);
    std::vector<char> dyn(nph, 0), relayed(nph, 0), helped(nph, 0);
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> direct_segs(nph);  // (dst, len)
    for (int t = 0; t < T; ++t) {
      const int sp = phys_of(xs_[t].sd), dp = phys_of(xs_[t].dd);
      for (const mp_chunk& c : chunks_[t]) {
        const mp_path& P = xs_[t].paths[c.path_index];
        if (P.kind == MP_PATH_DIRECT && eng_[t].direct_sm) {
          const int ex = o_.pull ? dp : sp;
          sm_bytes[ex] += c.length;
          segs[ex] += 1;
          direct_segs[ex].emplace_back((uint64_t)(uintptr_t)xs_[t].dst + c.offset, c.length);
        } else if (P.kind == MP_PATH_GPU && eng_[t].relay_sm) {
          sm_bytes[sp] += c.length;
          segs[sp] += 1;
          relayed[sp] = 1;
          dyn[phys_of(P.stage)] = 1;
        } else if (P.kind == MP_PATH_HOST && eng_[t].host_sm) {
          // same device: roundtrip tiles (helpers) unless the chunk needs
          // the flag handoff; two devices: hop1 helpers on the source, the
          // destination's table waits on flags
          if (sp != dp) {
            helped[sp] = 1;
            dyn[dp] = 1;
          } else if (c.length <= kRoundtripMaxBytes) {
            helped[sp] = 1;
          } else {
            dyn[sp] = 1;
          }
        }
      }
    }
    for (size_t ph = 0; ph < nph; ++ph) {
      const uint64_t grid = (uint64_t)ctx_->phys[ph].sms;
      if (dyn[ph] || segs[ph] == 0) continue;
      if ((uint64_t)segs[ph] * 4 > grid) {
        // many small direct segments (a posting window sent as one program,
        // mp_send_many): the small-message kernel still takes them in ONE
        // launch slot if a tile size keeps the table within one tile per
        // SM — the smallest 16-byte multiple that does, counted exactly
        if (relayed[ph] || helped[ph] || (uint64_t)segs[ph] > grid ||
            sm_bytes[ph] > (uint64_t)o_.small_max_bytes)
          continue;
        uint64_t tb = std::max<uint64_t>((sm_bytes[ph] + grid - 1) / grid, kStaticMinTile);
        for (;; tb += tb / 4) {
          tb = (tb + 15) & ~(uint64_t)15;
          uint64_t n = 0;
          for (const auto& sg : direct_segs[ph]) n += ntiles_of(sg.first, sg.second, tb);
          if (n <= grid) break;
        }
        static_tile_[ph] = tb;
        static_kind_[ph] = PROG_SMALL;
        continue;
      }
      // host-path helper tiles need the TMA kernel's idle warps
      const bool small = sm_bytes[ph] <= (uint64_t)o_.small_max_bytes && !helped[ph];
      const bool tma = sm_bytes[ph] <= grid * kStaticMaxPerCta && tma_ok(o_, peer_phys_[ph] != 0);
      if (!small && !tma) continue;
      uint64_t tb = (sm_bytes[ph] + (grid - 2 * segs[ph]) - 1) / (grid - 2 * segs[ph]);
      if (!relayed[ph]) {
        // direct segments only: the smallest tile whose exact cut count fits
        // one tile per SM, so no SM idles (8 segments at 64 MiB: 136 -> 148
        // tiles; the closed form above reserves two cuts per segment)
        uint64_t x = std::max<uint64_t>((sm_bytes[ph] + grid - 1) / grid, kStaticMinTile);
        for (int it = 0; it < 256 && x < tb; ++it, x += std::max<uint64_t>(x / 256, 128)) {
          x = (x + 15) & ~(uint64_t)15;
          uint64_t n = 0;
          for (const auto& sg : direct_segs[ph]) n += ntiles_of(sg.first, sg.second, x);
          if (n <= grid) {
            tb = x;
            break;
          }
        }
      }
      tb = std::max<uint64_t>(tb, kStaticMinTile);
      static_tile_[ph] = (tb + 15) & ~(uint64_t)15;
      static_kind_[ph] = small ? PROG_SMALL : PROG_STATIC_TMA;
    }
  }

  // Every chunk-hop of transfer t: tiles for the SM kernels, copy-engine ops
  // for CE paths.  Queue position of a tile: round-robin rounds, transfers
  // interleaved; key 0 is reserved for the SM host path's hop1 tiles, which
  // go first so their latency-bound PCIe writes overlap the whole HBM/NVLink
  // stream instead of forming a tail.
  void lower_transfer(int t) {
    const Xfer& x = xs_[t];
    const auto& paths = x.paths;
    const int np = (int)paths.size(), nc = (int)chunks_[t].size();
    std::vector<int> lane_base(np, 0);
    for (int p = 0; p < np; ++p) {
      lane_base[p] = lane_next_;
      lane_next_ += paths[p].nhops;
    }
    std::vector<int> hop2_done_ev(nc, -1);  // host WAR: event recorded after hop2 of chunk
    std::vector<int> host_chunk_of_seq;
    std::vector<HostRow> host_rows;  // CE host chunks in seq order (all resident)
    const uint64_t host_base = host_cursor_;
    for (int c = 0; c < nc; ++c) {
      const mp_chunk& ch = chunks_[t][c];
      const mp_path& P = paths[ch.path_index];
      const int p = ch.path_index;
      const uint32_t n_a = node_, n_b = node_ + 1;
      node_ += (uint32_t)P.nhops;
      const PathInfo& pi = info_[t][p];
      const Engines& en = eng_[t];
      if (P.kind == MP_PATH_DIRECT) {
        lower_direct(t, ch, pi, n_a, lane_base[p]);
      } else if (P.kind == MP_PATH_GPU) {
        lower_relay(t, c, ch, P, pi, n_a, n_b, lane_base[p]);
      } else if (en.host_sm) {
        lower_host_sm(t, c, ch, pi, n_a, n_b);
      } else if (en.host_slots >= pi.count) {
        host_rows.push_back(HostRow{ch.offset, ch.length, ch.seq, n_a, n_b, p});  // batched below
      } else {
        lower_host_ce_slots(t, c, ch, pi, n_a, n_b, lane_base[p], host_base, hop2_done_ev,
                            host_chunk_of_seq);
      }
    }
    if (!host_rows.empty()) emit_host_groups(t, host_rows, lane_base);
    for (int p = 0; p < np; ++p)  // reserve the slot ring of a WAR-reusing host path
      if (paths[p].kind == MP_PATH_HOST && !eng_[t].host_sm && eng_[t].host_slots < info_[t][p].count)
        host_cursor_ = std::max<uint64_t>(host_cursor_,
                                          host_base + (uint64_t)eng_[t].host_slots * info_[t][p].nominal);
  }

  uint64_t order(int t, uint64_t k) const { return (k + 1) * 64 + (uint64_t)t; }

  void lower_direct(int t, const mp_chunk& ch, const PathInfo& pi, uint32_t n_a, int lane) {
    const Xfer& x = xs_[t];
    const int sp = phys_of(x.sd), dp = phys_of(x.dd);
    if (eng_[t].direct_sm) {
      const int exec = o_.pull ? dp : sp;
      mpk::Tile proto{};
      proto.node = n_a;
      append_tiles(tiles_[exec], order(t, 2 * (uint64_t)ch.seq), (uint64_t)(uintptr_t)x.src + ch.offset,
                   (uint64_t)(uintptr_t)x.dst + ch.offset, ch.length, tile_for(exec, pi.bytes), proto);
    } else {
      e_->ce.push_back(CeOp{sp, lane, (uint8_t*)x.dst + ch.offset, (const uint8_t*)x.src + ch.offset,
                            (size_t)ch.length, -1, -1, n_a});
    }
  }

  // GPU relay: hop1 src -> relay staging, hop2 staging -> dst.  SM tables
  // hand off through the chunk's flag in the relay's memory (hop2 of round r
  // queued after round r + kHop2Delay); CE lanes through an event.
  void lower_relay(int t, int c, const mp_chunk& ch, const mp_path& P, const PathInfo& pi, uint32_t n_a,
                   uint32_t n_b, int lane) {
    const Xfer& x = xs_[t];
    const int sp = phys_of(x.sd);
    const uint64_t s0 = (uint64_t)(uintptr_t)x.src, d0 = (uint64_t)(uintptr_t)x.dst;
    Logi& L = ctx_->logi[P.stage];
    const int rp = L.phys;
    const int g = chunk_base_[t] + c;  // flag index, unique across the program
    // staging offset congruent to the source mod 128 keeps hop1 on whole lines
    uint64_t& cur = stage_cursor_[P.stage];
    cur += ((s0 + ch.offset) - ((uint64_t)(uintptr_t)L.stage + cur)) & 127u;
    uint8_t* stage = L.stage + cur;
    cur += ch.length;
    if (!eng_[t].relay_sm) {
      const int ev = new_event(sp);
      e_->ce.push_back(CeOp{sp, lane, stage, (const uint8_t*)x.src + ch.offset, (size_t)ch.length, -1, ev,
                            n_a});
      e_->ce.push_back(CeOp{rp, lane + 1, (uint8_t*)x.dst + ch.offset, stage, (size_t)ch.length, ev, -1,
                            n_b});
      return;
    }
    // relay hops on the LDG/STG kernel: 128 KiB tiles (half the flag
    // releases / acquires of the 64 KiB direct tiles) — 512 MiB through 1 / 2
    // / 6 relays +1-5% in loopback and +12-17% with system-scope flags (the
    // cross-device lowering, fault_inject=2; tools/exp_relay_tiles.py)
    uint64_t t1 = tile_for(sp, pi.bytes);
    uint64_t t2 = tile_for(rp, pi.bytes);
    if (o_.tile_bytes == 0 && t1 == kVecTileBytes && !static_tile_[sp]) t1 = kRelayTileBytes;
    if (o_.tile_bytes == 0 && t2 == kVecTileBytes && !static_tile_[rp]) t2 = kRelayTileBytes;
    if (const char* e = std::getenv("MP_RELAY_TILE")) {  // experiment knob
      const uint64_t v = std::strtoull(e, nullptr, 10);
      if (v && !static_tile_[sp]) t1 = v;
      if (v && !static_tile_[rp]) t2 = v;
    }
    // hop1 and hop2 on one device (loopback): release / acquire at GPU scope
    const uint32_t scope = same_gpu(sp, rp) ? mpk::TILE_SCOPE_GPU : 0u;
    mpk::Tile h1{};
    h1.signal = hop1_signal(L.flags + g);
    h1.node = n_a;
    h1.flags = scope;
    const uint64_t r2 = 2 * (uint64_t)ch.seq;
    append_tiles(tiles_[sp], order(t, r2), s0 + ch.offset, (uint64_t)(uintptr_t)stage, ch.length, t1, h1);
    mpk::Tile h2{};
    h2.wait = L.flags + g;
    h2.pass = L.flags + L.flag_cap + g;
    h2.wait_count = (uint32_t)ntiles_of((uint64_t)(uintptr_t)stage, ch.length, t1);
    h2.pass_count = (uint32_t)ntiles_of(d0 + ch.offset, ch.length, t2);
    h2.flags = mpk::TILE_SRC_MUTABLE | scope;
    h2.node = n_b;
    append_tiles(tiles_[rp], order(t, r2 + 1 + 2 * kHop2Delay), (uint64_t)(uintptr_t)stage, d0 + ch.offset,
                 ch.length, t2, h2);
  }

  // Host-staged by the SM kernels over mapped pinned memory.  Source and
  // destination on one device and a chunk <= kRoundtripMaxBytes: ONE
  // roundtrip tile (hop1, CTA barrier, hop2 in one CTA).  Otherwise hop1
  // tiles (src device) store into the slot and release the chunk's flag (in
  // dst memory); hop2 tiles (dst device) load it back once the flag counts
  // every hop1 tile.  On a static TMA table the host tiles of the source
  // device go to the helper warps; elsewhere they lead the table (key t),
  // hop2 tiles right behind their hop1 (a hop2 tile waits only on hop1
  // tiles claimed before it by resident CTAs).
  void lower_host_sm(int t, int c, const mp_chunk& ch, const PathInfo& pi, uint32_t n_a, uint32_t n_b) {
    const Xfer& x = xs_[t];
    const int sp = phys_of(x.sd), dp = phys_of(x.dd);
    const uint64_t s0 = (uint64_t)(uintptr_t)x.src, d0 = (uint64_t)(uintptr_t)x.dst;
    const int g = chunk_base_[t] + c;
    Logi& L = ctx_->logi[x.dd];
    uint8_t* host_dev = nullptr;
    CK(cudaHostGetDevicePointer((void**)&host_dev, ctx_->host_stage, 0));
    // every slot starts on a fresh 128-byte line of the arena (no two
    // chunks share a host cache line: partial-line PCIe writes from two
    // CTAs to one line serialise in the root complex — 8 x 1310-byte
    // roundtrips at 8 MiB measured 12.2 -> 7.1 us), congruent to its source
    // mod 128 so the copies stay 16-byte vectors
    host_cursor_ = (host_cursor_ + 127u) & ~(uint64_t)127u;
    host_cursor_ += ((s0 + ch.offset) - ((uint64_t)(uintptr_t)host_dev + host_cursor_)) & 127u;
    uint8_t* slot = host_dev + host_cursor_;
    host_cursor_ += ch.length;
    const bool help = static_kind_[sp] == PROG_STATIC_TMA;
    (void)n_b;
    if (same_gpu(sp, dp) && ch.length <= kRoundtripMaxBytes) {
      mpk::Tile rt{};
      rt.src = s0 + ch.offset;
      rt.dst = d0 + ch.offset;
      rt.stage = slot;
      rt.len = ch.length;
      // fence when the source device's whole program (every transfer of a
      // send_many window) is long enough to hide it
      uint64_t on_src = 0;
      for (const Xfer& y : xs_)
        if (phys_of(y.sd) == sp) on_src += y.size;
      rt.flags = mpk::TILE_ROUNDTRIP | (on_src >= rt_fence_min_bytes() ? mpk::TILE_FENCE : 0u);
      rt.node = n_a;  // hop2 is n_a + 1 == n_b
      // hop1 writes whole 128-byte lines into the slot (the chunk widened
      // to its source lines, clipped to the message): a partial-line PCIe
      // write costs the root complex a read-modify-write; hop2 reads back
      // only the chunk's bytes
      const uint64_t a = s0 + ch.offset, e = a + ch.length;
      rt.wait_count = (uint32_t)std::min<uint64_t>(a & 127u, ch.offset);
      rt.pass_count = (uint32_t)std::min<uint64_t>((0 - e) & 127u, x.size - (ch.offset + ch.length));
      if (help) helpers_[sp].push_back(rt);
      else tiles_[sp].push_back({{(uint64_t)t, tiles_[sp].size()}, rt});
      return;
    }
    const uint32_t scope = same_gpu(sp, dp) ? mpk::TILE_SCOPE_GPU : 0u;
    const uint64_t th = std::min<uint64_t>(auto_tile_bytes(ctx_, pi.bytes, ctx_->phys[sp].sms), kHostTileBytes);
    mpk::Tile h1{};
    h1.signal = hop1_signal(L.flags + g);
    h1.node = n_a;
    h1.flags = scope;
    TileList h1t;
    append_tiles(h1t, (uint64_t)t, s0 + ch.offset, (uint64_t)(uintptr_t)slot, ch.length, th, h1);
    for (auto& kv : h1t) {
      if (help && sp != dp) helpers_[sp].push_back(kv.second);
      else tiles_[sp].push_back({{(uint64_t)t, tiles_[sp].size()}, kv.second});
    }
    mpk::Tile h2{};
    h2.wait = L.flags + g;
    h2.pass = L.flags + L.flag_cap + g;
    h2.wait_count = (uint32_t)h1t.size();
    h2.pass_count = (uint32_t)ntiles_of(d0 + ch.offset, ch.length, th);
    h2.flags = mpk::TILE_SRC_MUTABLE | scope;
    h2.node = n_b;
    append_tiles(tiles_[dp], (uint64_t)t, (uint64_t)(uintptr_t)slot, d0 + ch.offset, ch.length, th, h2);
  }

  // Host-staged by copy engines through `host_slots` reused staging slots:
  // per-chunk D2H then H2D (event), slot reuse guarded by a WAR event.
  void lower_host_ce_slots(int t, int c, const mp_chunk& ch, const PathInfo& pi, uint32_t n_a,
                           uint32_t n_b, int lane, uint64_t host_base, std::vector<int>& hop2_done_ev,
                           std::vector<int>& host_chunk_of_seq) {
    const Xfer& x = xs_[t];
    const int sp = phys_of(x.sd), dp = phys_of(x.dd);
    const int seq = ch.seq;
    const int slots = eng_[t].host_slots;
    host_chunk_of_seq.push_back(c);
    uint8_t* slot = ctx_->host_stage + host_base + (size_t)(seq % slots) * pi.nominal;
    const int war = seq >= slots ? hop2_done_ev[host_chunk_of_seq[seq - slots]] : -1;
    const int ev1 = new_event(sp);
    e_->ce.push_back(CeOp{sp, lane, slot, (const uint8_t*)x.src + ch.offset, (size_t)ch.length, war, ev1,
                          n_a});
    const int ev2 = new_event(dp);
    hop2_done_ev[c] = ev2;
    e_->ce.push_back(CeOp{dp, lane + 1, (uint8_t*)x.dst + ch.offset, slot, (size_t)ch.length, ev1, ev2,
                          n_b});
  }

  // The round-robin plan puts a path's full chunks at a constant stride
  // (pipeline.py:68-77), so the host path's chunks are rows of a 2-D copy:
  // split them into consecutive groups and move each group with ONE 2-D D2H
  // into packed pinned staging and ONE 2-D H2D out of it (event handoff per
  // group; D2H of group g+1 overlaps H2D of group g).  Rows that break the
  // stride (the truncated last chunk) form their own group.
  void emit_host_groups(int t, const std::vector<HostRow>& host_rows, const std::vector<int>& lane_base) {
    const Xfer& x = xs_[t];
    const int sp = phys_of(x.sd), dp = phys_of(x.dd);
    uint64_t hbytes = 0;
    for (const HostRow& r : host_rows) hbytes += r.len;
    const int ngroups = (int)std::max<uint64_t>(
        1, std::min<uint64_t>({host_rows.size(), (uint64_t)kHostMaxGroups,
                               (hbytes + kHostGroupBytes - 1) / kHostGroupBytes}));
    const size_t per = (host_rows.size() + ngroups - 1) / ngroups;
    std::vector<std::vector<HostRow>> groups;
    for (const HostRow& r : host_rows) {
      bool fresh = groups.empty() || groups.back().size() >= per;
      if (!fresh) {
        const auto& gv = groups.back();
        const HostRow& f = gv.front();
        const uint64_t stride = gv.size() >= 2 ? gv[1].off - gv[0].off : r.off - f.off;
        fresh = r.len != f.len || r.off - gv.back().off != stride || stride < r.len || stride > kMaxCopyPitch;
      }
      if (fresh) groups.emplace_back();
      groups.back().push_back(r);
    }
    for (const auto& gv : groups) {
      const HostRow& f = gv.front();
      const uint64_t stride = gv.size() >= 2 ? gv[1].off - gv[0].off : f.len;
      uint8_t* slot = ctx_->host_stage + host_cursor_;
      host_cursor_ += f.len * gv.size();
      const int lane = lane_base[f.p];  // one D2H / H2D stream pair: groups pipeline
      CeOp d2h{sp, lane, slot, (const uint8_t*)x.src + f.off, (size_t)f.len, -1, new_event(sp), f.n_a};
      CeOp h2d{dp, lane + 1, (uint8_t*)x.dst + f.off, slot, (size_t)f.len, d2h.record_ev, -1, f.n_b};
      d2h.rows = h2d.rows = gv.size();
      d2h.spitch = h2d.dpitch = stride;
      d2h.dpitch = h2d.spitch = f.len;
      for (const HostRow& r : gv) {
        d2h.nodes.push_back(r.n_a);
        h2d.nodes.push_back(r.n_b);
      }
      e_->ce.push_back(d2h);
      e_->ce.push_back(h2d);
    }
  }

  // One tile table per physical device, sorted by queue key, its kernel kind
  // (ProgKind), grid and static prefix, uploaded with the program's claim
  // counters right behind it.
  void upload() {
    DeviceGuard dg;
    for (size_t ph = 0; ph < tiles_.size(); ++ph) {
      auto& v = tiles_[ph];
      auto& hv = helpers_[ph];
      if (v.empty() && hv.empty()) continue;
      std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      std::vector<mpk::Tile> flat;
      flat.reserve(v.size() + hv.size());
      for (auto& kv : v) flat.push_back(kv.second);
      Program pr;
      pr.phys = (int)ph;
      Phys& P = ctx_->phys[ph];
      // helper tiles ride behind a static TMA table's own tiles; if the
      // table is not (or no longer) static they lead it as ordinary tiles
      const bool as_helpers = !hv.empty() && !flat.empty() && static_tile_[ph] &&
                              static_kind_[ph] == PROG_STATIC_TMA && flat.size() <= (size_t)P.sms;
      if (!hv.empty() && !as_helpers) flat.insert(flat.begin(), hv.begin(), hv.end());
      bool waits = false, plain = true;
      for (const auto& tl : flat) {
        waits |= tl.wait != nullptr;
        plain = plain && !tl.wait && !tl.signal && tl.flags == 0;
      }
      pr.peer = peer_phys_[ph] != 0;
      pr.kind = static_tile_[ph] && flat.size() <= (size_t)P.sms ? static_kind_[ph] : PROG_DYNAMIC;
      if (pr.kind == PROG_SMALL && (!plain || flat.size() > mpk::kSmallMaxTiles))
        pr.kind = tma_ok(o_, pr.peer) ? PROG_STATIC_TMA : PROG_DYNAMIC;  // e.g. relay hop1 tiles
      if (!hv.empty() && !as_helpers) pr.kind = PROG_DYNAMIC;
      pr.grid = (unsigned)std::min<uint64_t>(flat.size(), pr.kind == PROG_DYNAMIC ? grid_of(ph) : P.sms);
      pr.nstatic = waits ? 0u : pr.grid;
      if (as_helpers) {
        flat.insert(flat.end(), hv.begin(), hv.end());
        pr.nhelp = (unsigned)hv.size();
      }
      pr.ntiles = (unsigned)flat.size();
      CK(cudaSetDevice(P.ordinal));
      CK(cudaMalloc(&pr.d_tiles, flat.size() * sizeof(mpk::Tile) + sizeof(mpk::Sched)));
      pr.d_sched = reinterpret_cast<mpk::Sched*>(pr.d_tiles + flat.size());
      e_->progs.push_back(pr);  // owned by the entry from here (freed on error)
      // tiles and zeroed claim counters in ONE upload, completed below before
      // any launch (an unsynchronised legacy-stream cudaMemset once zeroed
      // the arrival counter under a running first launch on a non-blocking
      // caller stream, shifting every later launch's index)
      flat.resize(flat.size() + (sizeof(mpk::Sched) + sizeof(mpk::Tile) - 1) / sizeof(mpk::Tile));
      std::memset(static_cast<void*>(flat.data() + pr.ntiles), 0, (flat.size() - pr.ntiles) * sizeof(mpk::Tile));
      CK(cudaMemcpy(pr.d_tiles, flat.data(), pr.ntiles * sizeof(mpk::Tile) + sizeof(mpk::Sched),
                    cudaMemcpyHostToDevice));
      flat.resize(pr.ntiles);
      if (pr.kind == PROG_SMALL) {
        auto sm = std::make_shared<mpk::SmallTable<mpk::kSmallMaxTiles>>();
        uint64_t bytes = 0;
        for (size_t i = 0; i < flat.size(); ++i) {
          sm->src[i] = flat[i].src;
          sm->dst[i] = flat[i].dst;
          sm->len[i] = (uint32_t)flat[i].len;
          bytes += flat[i].len;
        }
        e_->progs.back().small = sm;
        e_->progs.back().bytes = bytes;
      }
    }
    // A pageable-memory cudaMemcpy may return before its DMA reaches the
    // device, and it runs on the legacy stream, which the non-blocking
    // caller streams do not wait for: finish the uploads before any launch.
    for (const Program& pr : e_->progs) {
      CK(cudaSetDevice(ctx_->phys[pr.phys].ordinal));
      CK(cudaStreamSynchronize(cudaStreamLegacy));
    }
  }
};

Entry* build_entry_multi(mp_ctx* ctx, const std::string& key, std::vector<Xfer> xs,
                         const mp_config& cfg) {
  return Lowering(ctx, key, std::move(xs)).build(cfg);
}

Entry* build_entry(mp_ctx* ctx, const std::string& key, const void* src, void* dst, uint64_t size,
                   int src_dev, int dst_dev, const mp_config& cfg) {
  return build_entry_multi(ctx, key, {Xfer{src, dst, size, src_dev, dst_dev, {}}}, cfg);
}

}  // namespace
