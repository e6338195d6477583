/*
 * mpb200.h — C ABI of the B200-native multi-path intra-node transfer engine.
 *
 * This is the drop-in boundary for the reference package `mpsim`
 * (/root/reference/pkg/src/mpsim).  Every entry point below replaces one
 * reference interface; the citation after each declaration names it.
 * Plain pointers, sizes and PODs only — no torch or C++ types cross here.
 *
 * Conventions
 *   - Every function returns an int status: MP_OK (0) or a negative MP_ERR_*.
 *     The message of the last failure on the calling thread is available from
 *     mp_last_error(); its text matches the reference's exception messages so
 *     the Python layer can re-raise TopologyError / PlanError / ChunkError
 *     with identical wording.
 *   - Devices are accelerator indices 0..n-1 of the topology; the implicit
 *     host device is MP_HOST (-1).
 *   - Output arrays are caller-allocated with a capacity; when the capacity
 *     is too small the call fails with MP_ERR_CAPACITY and writes the needed
 *     count to *n_out, so "call with cap=0, allocate, call again" works.
 */
#ifndef MPB200_H
#define MPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_ABI_VERSION 4

/* ---- status codes -------------------------------------------------------- */
#define MP_OK 0
#define MP_ERR_TOPOLOGY -1   /* reference TopologyError   topology.py:25  */
#define MP_ERR_PLAN -2       /* reference PlanError       paths.py:33     */
#define MP_ERR_CHUNK -3      /* reference ChunkError      pipeline.py:17  */
#define MP_ERR_VALUE -4      /* reference ValueError (graph/cache)        */
#define MP_ERR_CAPACITY -5   /* output array too small; *n_out = needed   */
#define MP_ERR_CUDA -6       /* CUDA runtime/driver failure               */
#define MP_ERR_STATE -7      /* misuse: no topology, closed context, ...  */

#define MP_HOST (-1)

/* ---- path kinds / roles / policies (reference string constants) ---------- */
#define MP_PATH_DIRECT 0     /* paths.py:17 DIRECT = "direct"      */
#define MP_PATH_GPU 1        /* paths.py:18 GPU_STAGED = "gpu"     */
#define MP_PATH_HOST 2       /* paths.py:19 HOST_STAGED = "host"   */

#define MP_ROLE_DIRECT 0     /* graph.py:20 "direct"      */
#define MP_ROLE_HOP1 1       /* graph.py:21 "stage_hop1"  */
#define MP_ROLE_HOP2 2       /* graph.py:22 "stage_hop2"  */

#define MP_SHARE_BANDWIDTH 0 /* paths.py:22 "bandwidth_proportional" */
#define MP_SHARE_EQUAL 1     /* paths.py:21 "equal"                  */

#define MP_DUPLEX_FULL 0
#define MP_DUPLEX_HALF 1

/* ---- plain data ---------------------------------------------------------- */

/* PathConfig (paths.py:67-86). */
typedef struct {
  int32_t num_gpu_paths;     /* >= 1, path 0 is always Direct          */
  int32_t host_path_enabled; /* 0/1                                   */
  int32_t max_chunks;        /* >= 1                                  */
  int32_t graph_mode;        /* 0 = per-call stream launch, 1 = graph */
  int32_t cache_capacity;    /* >= 1                                  */
  int32_t share_policy;      /* MP_SHARE_*                            */
} mp_config;

/* LinkSpec (topology.py:69-90), bandwidth already aggregated over sublinks. */
typedef struct {
  int32_t a, b;              /* device indices, MP_HOST for the host  */
  double bandwidth;          /* bytes/s per direction channel         */
  double latency;            /* seconds per copy                      */
  int32_t duplex;            /* MP_DUPLEX_*                           */
  int32_t sublinks;
} mp_link;

/* Channel (topology.py:57-66). */
typedef struct {
  char id[32];               /* "0->1", "0<->host", ...               */
  double bandwidth;
  double latency;
  int32_t a, b;              /* creation endpoints                    */
} mp_channel;

/* Hop (paths.py:37-43). */
typedef struct {
  int32_t channel;           /* index into the topology's channels    */
  int32_t src, dst;          /* device indices / MP_HOST              */
} mp_hop;

/* Path (paths.py:46-64). */
typedef struct {
  int32_t kind;              /* MP_PATH_*                             */
  int32_t stage;             /* staging device, MP_HOST, or -2 = none */
  double share;
  int32_t nhops;             /* 1 (direct) or 2 (staged)              */
  mp_hop hops[2];
} mp_path;

#define MP_NO_STAGE (-2)

/* ChunkAssignment (pipeline.py:21-32). */
typedef struct {
  uint64_t offset;           /* same offset in src and dst buffers    */
  uint64_t length;
  int32_t path_index;
  int32_t seq;
} mp_chunk;

/* Lane (pipeline.py:81-88): members are chunk ids in members[first..first+count). */
typedef struct {
  int32_t lane_id;
  int32_t path_index;
  int32_t hop;
  int32_t first;
  int32_t count;
} mp_lane;

/* LaneSchedule dependency (pipeline.py:96-97): (lane1,pos1) -> (lane2,pos2). */
typedef struct {
  int32_t lane1, pos1, lane2, pos2;
} mp_lane_dep;

/* CopyNode (graph.py:28-39). */
typedef struct {
  int32_t id;
  int32_t src_dev, dst_dev;
  int32_t channel;
  uint64_t offset, length;
  int32_t lane;
  int32_t role;              /* MP_ROLE_*                             */
  int32_t chunk_index;
  int32_t path_index;
} mp_node;

typedef struct {
  int32_t from, to;
} mp_edge;

/* Measured graph lifecycle of the last mp_send on a context: the four phases
 * of the reference's OverheadModel (graph.py:194-236, PHASES graph.py:24),
 * measured on the host clock instead of modelled. */
typedef struct {
  int32_t hit;               /* 1 = cached executable replayed        */
  int32_t graph_mode;
  int32_t nodes_logical;     /* reference node count (graph.py:91)    */
  int32_t nodes_physical;    /* nodes in the CUDA graph               */
  int32_t kernels;           /* our kernels launched by this send     */
  int32_t ce_copies;         /* copy-engine memcpys issued            */
  double creation_us;
  double construction_us;
  double instantiation_us;
  double launch_us;          /* host time of the enqueue call         */
  double plan_us;            /* plan + key on a miss                  */
  uint64_t cache_hits, cache_misses, cache_evictions;
  int32_t kernel;            /* MP_KERNEL_*: the source device's copy kernel */
  int32_t pad;
} mp_send_stats;
#define MP_KERNEL_NONE (-1)  /* copy engines only                           */
#define MP_KERNEL_VEC 0      /* transfer_kernel<0,U>: 16-byte LDG/STG        */
#define MP_KERNEL_TMA 1      /* transfer_kernel<1,8>: TMA bulk ring          */
#define MP_KERNEL_SMALL 2    /* small_copy_kernel: descriptors in params     */

/* Engine knobs (choice of copy mechanism per path type; measured defaults). */
#define MP_ENGINE_SM 0       /* hand-written sm_100a copy kernel       */
#define MP_ENGINE_CE 1       /* copy engine cudaMemcpyAsync            */
#define MP_ENGINE_AUTO 2     /* host path only (default): SM kernels while
                                every host chunk fits one roundtrip tile
                                (<= 64 KiB), copy engines above          */
#define MP_COPY_VEC 0        /* 16-byte vector LDG/STG                 */
#define MP_COPY_TMA 1        /* cp.async.bulk staged through smem      */
#define MP_SCHED_AUTO 0      /* static one-tile-per-CTA tables where no
                                tile waits or touches host memory (no
                                atomics, no exit protocol); else dynamic */
#define MP_SCHED_DYNAMIC 1   /* always claim tiles dynamically          */

typedef struct {
  int32_t direct_engine;     /* MP_ENGINE_*                           */
  int32_t relay_engine;      /* MP_ENGINE_*                           */
  int32_t copy_kind;         /* MP_COPY_*                             */
  int32_t ctas_per_sm;       /* persistent grid = SMs * ctas_per_sm   */
  int32_t threads;           /* threads per CTA                       */
  int64_t tile_bytes;        /* 0 = automatic                         */
  int32_t host_slots;        /* pinned host staging slots (>=2), 0=all */
  int32_t pull;              /* 1: direct copies run on the dst device */
  int64_t sm_min_bytes;      /* below this a path uses CE even if SM  */
  int32_t unroll;            /* VEC: 16-byte loads in flight / thread (4, 8, 16) */
  int32_t tma_stages;        /* TMA: shared-memory ring stages (2..16)  */
  int32_t tma_block;         /* TMA: bytes per bulk copy (multiple of 16) */
  int32_t host_engine;       /* MP_ENGINE_*: host-staged path by the SM
                                kernels (mapped pinned memory), by CEs,
                                or MP_ENGINE_AUTO (default)              */
  int32_t tma_peer;          /* 1: TMA bulk copies also on tables that touch
                                another GPU over NVLink; 0 (default): such
                                tables run the 16-byte LDG/STG kernel;
                                -1: every table does (testing)        */
  int32_t sched;             /* MP_SCHED_*: tile scheduling of the SM kernel */
  int64_t small_max_bytes;   /* static direct tables up to this size run the
                                one-launch-slot small-message kernel (0 = off) */
  int32_t pdl;               /* programmatic dependent launch of sends whose
                                program is ONE kernel (the kernel waits on
                                griddepcontrol before touching memory),
                                graph mode included: B200 retires
                                back-to-back one-kernel graph launches in
                                2.048 us quanta, PDL launches do not
                                (tools/pdl_probe.cu).  0: off (graph
                                replay); 1: small-message kernel >= 1 MiB;
                                2: also static TMA tables; 3 (default):
                                also dynamic tables                      */
  int32_t wait_timeout_ms;   /* limit of a relay-flag / group-barrier wait
                                (0 = 4000).  A wait that times out skips
                                its tile (staging is never copied
                                unsignalled) and makes the error sticky:
                                every later mp_send / mp_send_many /
                                mp_wait / mp_group_send fails until
                                mp_sync reports and clears it            */
  int32_t fault_inject;      /* testing only, bits: 1 = the first staged
                                chunk's hop1 tiles never signal (forces a
                                timeout); 2 = lower loopback devices as
                                separate GPUs (system-scope flags, host
                                chunks as hop1 / hop2 tiles) */
} mp_engine_opts;

/* ---- errors / version ---------------------------------------------------- */
const char* mp_last_error(void);
int mp_abi_version(void);

/* ---- topology (replaces topology.py:164-240 load_topology, :93-154 Topology) */
typedef struct mp_topology mp_topology;

int mp_topology_load(const char* text, const char* default_name, mp_topology** out);
int mp_topology_create(const char* name, int32_t n_accel, const mp_link* links,
                       int32_t n_links, mp_topology** out);
void mp_topology_destroy(mp_topology* topo);
int mp_topology_info(const mp_topology* topo, int32_t* n_accel, int32_t* n_links,
                     int32_t* n_channels);
int mp_topology_name(const mp_topology* topo, char* buf, size_t cap);
int mp_topology_link(const mp_topology* topo, int32_t i, mp_link* out);
int mp_topology_channel(const mp_topology* topo, int32_t i, mp_channel* out);
/* topology.py:136-143 channel_for */
int mp_topology_channel_for(const mp_topology* topo, int32_t src, int32_t dst,
                            int32_t* channel);

/* ---- planner (replaces paths.py:144-187, pipeline.py:51-125, graph.py:91-144) */
int mp_config_validate(const mp_config* cfg);                   /* paths.py:78-86 */
/* paths.py:170-187 plan_paths (+_build_path_set :160-167, _assign_shares :144-150) */
int mp_plan_paths(const mp_topology* topo, int32_t src, int32_t dst,
                  const mp_config* cfg, mp_path* out, int32_t cap, int32_t* n_out);
/* paths.py:210-242 plan_contention_free: out holds n_transfers path sets of
 * paths_per_set paths each; *shared = shared channel count. */
int mp_plan_contention_free(const mp_topology* topo, const int32_t* srcs,
                            const int32_t* dsts, int32_t n_transfers,
                            const mp_config* cfg, mp_path* out, int32_t cap,
                            int32_t* paths_per_set, int32_t* shared);
/* paths.py:125-132 PathSet.__post_init__ */
int mp_pathset_validate(const mp_path* paths, int32_t n);
/* pipeline.py:51-78 make_chunk_plan */
int mp_make_chunk_plan(const mp_path* paths, int32_t n_paths, uint64_t size,
                       int32_t max_chunks, mp_chunk* out, int32_t cap, int32_t* n_out);
/* pipeline.py:102-125 lane_schedule */
int mp_lane_schedule(const mp_path* paths, int32_t n_paths, const mp_chunk* chunks,
                     int32_t n_chunks, mp_lane* lanes, int32_t lanes_cap,
                     int32_t* n_lanes, int32_t* members, int32_t members_cap,
                     int32_t* n_members, mp_lane_dep* deps, int32_t deps_cap,
                     int32_t* n_deps);
/* graph.py:91-118 build_graph */
int mp_build_graph(const mp_path* paths, int32_t n_paths, const mp_chunk* chunks,
                   int32_t n_chunks, mp_node* nodes, int32_t nodes_cap,
                   int32_t* n_nodes, mp_edge* edges, int32_t edges_cap,
                   int32_t* n_edges, int32_t* lane_count);
/* graph.py:132-144 _digest / graph_key: hex sha256 of the reference's repr
 * tuple, byte-identical to the reference.  Hop channel fields index
 * `channel_ids` (the Channel.id strings).  out_hex must hold 65 bytes. */
int mp_graph_digest(const mp_config* cfg, int32_t src, int32_t dst,
                    const mp_path* paths, int32_t n_paths,
                    const char* const* channel_ids, int32_t n_channels,
                    char* out_hex);
/* LinkSpec.__post_init__ (topology.py:79-90); duplex -1 = not full/half. */
int mp_link_validate(const mp_link* link);
/* Python float repr (shortest round trip), used by the digest and plan dumps. */
int mp_format_double(double x, char* buf, size_t cap);

/* ---- LRU cache (replaces graph.py:147-191 GraphCache) -------------------- */
typedef struct mp_cache mp_cache;
int mp_cache_create(int32_t capacity, mp_cache** out);
void mp_cache_destroy(mp_cache* cache);
/* graph.py:173-186 get_or_build: on a hit *hit=1 and *value=stored value;
 * on a miss the key is inserted with *value (caller-chosen) and up to
 * evicted_cap evicted values are returned (oldest first). */
int mp_cache_access(mp_cache* cache, const void* key, size_t key_len, int32_t* hit,
                    uint64_t* value, uint64_t* evicted, int32_t evicted_cap,
                    int32_t* n_evicted);
int mp_cache_len(const mp_cache* cache, int32_t* n);
int mp_cache_contains(const mp_cache* cache, const void* key, size_t key_len,
                      int32_t* yes);
/* values in LRU order, least recently used first */
int mp_cache_values(const mp_cache* cache, uint64_t* out, int32_t cap, int32_t* n_out);

/* ---- engine (replaces sim.py:272-292 simulate_* with real execution) ----- */
typedef struct mp_ctx mp_ctx;

/* device_map[i] = physical CUDA ordinal of logical accelerator i (several
 * logical devices may share one ordinal: "loopback"). Enables peer access
 * between every pair of distinct physical devices. */
int mp_ctx_create(int32_t n_logical, const int32_t* device_map, mp_ctx** out);
void mp_ctx_destroy(mp_ctx* ctx);
int mp_ctx_set_topology(mp_ctx* ctx, const mp_topology* topo);
int mp_ctx_set_engine(mp_ctx* ctx, const mp_engine_opts* opts);
int mp_ctx_get_engine(const mp_ctx* ctx, mp_engine_opts* opts);
/* Per-message-size choice of the direct-path and host-path mechanisms, from
 * measurement (tuner.tune_engines): a message of S bytes uses
 * direct_engine[i] / host_engine[i] for the first i with S <= max_bytes[i]
 * (host_engine may be NULL: keep opts.host_engine); sizes past the table (or
 * n = 0) use opts. */
int mp_ctx_set_size_policy(mp_ctx* ctx, const uint64_t* max_bytes,
                           const int32_t* direct_engine, const int32_t* host_engine,
                           int32_t n);
int mp_ctx_peer_matrix(const mp_ctx* ctx, int32_t* out, int32_t cap);

/* The multi-path transfer: size bytes from src (on logical src_dev) to dst
 * (on logical dst_dev).  Ordered after prior work on `stream` (a
 * cudaStream_t of the src device, NULL = legacy default) and makes `stream`
 * wait for completion.  graph_mode selects cached CUDA-graph replay
 * (key = src, dst, size, devices, path set; LRU of cudaGraphExec_t) or
 * per-call stream launch.  This is the B200 counterpart of the reference's
 * plan_paths -> make_chunk_plan -> graph_key -> GraphCache.get_or_build ->
 * simulate_graph chain (sim.py:272-277).  On a stream being captured into
 * the caller's CUDA graph, a cached program is recorded into that graph
 * (and pinned against LRU eviction); a cache miss fails with MP_ERR_STATE. */
int mp_send(mp_ctx* ctx, const void* src, void* dst, uint64_t size,
            int32_t src_dev, int32_t dst_dev, const mp_config* cfg, void* stream);
/* One transfer of a concurrent batch. */
typedef struct {
  const void* src;
  void* dst;
  uint64_t size;
  int32_t src_dev, dst_dev;
} mp_xfer;

/* Concurrent transfers (windows, bidirectional flows, ring halo exchanges —
 * the reference's simulate_concurrent, sim.py:287-292) as ONE program: the
 * tiles of every transfer share one persistent kernel per device,
 * interleaved round by round, and the whole batch is one cached graph.
 * joint = 1 chooses staging devices with plan_contention_free
 * (paths.py:210-242); 0 plans each transfer with plan_paths.  1..64
 * transfers.  Resending the previous call's exact arguments while its
 * entry is cached skips the key rebuild (the osu_bw / halo-exchange loop). */
int mp_send_many(mp_ctx* ctx, const mp_xfer* xfers, int32_t n, const mp_config* cfg,
                 int32_t joint, void* stream);

/* One executed chunk-hop of a traced send (the GPU counterpart of the
 * reference's SimTask, sim.py:32-49): first tile start / last tile
 * completion (%globaltimer, SM lanes) or CE timing events, in microseconds
 * from the send's fork on that device. */
typedef struct {
  int32_t node;              /* logical node id, build_graph order      */
  int32_t engine;            /* MP_ENGINE_SM / MP_ENGINE_CE             */
  int32_t device;            /* physical device index in the context    */
  int32_t pad;
  double start_us;
  double end_us;
} mp_trace_rec;

/* Synchronous traced send (streamed program): writes one record per logical
 * node (cap >= nodes; *n_out = nodes) — the real Timeline the reference's
 * check_timeline (integrity.py:63-101) verifies. */
int mp_send_trace(mp_ctx* ctx, const void* src, void* dst, uint64_t size,
                  int32_t src_dev, int32_t dst_dev, const mp_config* cfg,
                  mp_trace_rec* out, int32_t cap, int32_t* n_out);

/* Receiver side: make `stream` (any device) wait for the last mp_send. */
int mp_wait(mp_ctx* ctx, void* stream);
int mp_send_stats_get(const mp_ctx* ctx, mp_send_stats* out);
/* Chunk plan used by the last mp_send (for parity checks against the oracle). */
int mp_last_plan(const mp_ctx* ctx, mp_path* paths, int32_t paths_cap,
                 int32_t* n_paths, mp_chunk* chunks, int32_t chunks_cap,
                 int32_t* n_chunks);
int mp_cache_clear(mp_ctx* ctx);
/* Wait for every transfer of the context.  If a wait timed out (see
 * mp_engine_opts.wait_timeout_ms) it fails with the error and clears it:
 * flag arrays and control blocks are re-zeroed, later sends run again. */
int mp_sync(mp_ctx* ctx);

/* Per-path bandwidth probe: times `iters` copies of `bytes` over each path
 * type between src and dst and writes GB/s (1e9 B/s): out[0] = direct by the
 * SM transfer kernel, out[1] = D2H, out[2] = H2D, out[3] = direct by a CE
 * copy; with cap >= 6 also out[4] = D2H and H2D concurrently (per direction)
 * and out[5] = the host-staged path as executed (8 pipelined chunks); with
 * cap >= 8 also out[6] / out[7] = the SM transfer kernel writing to / reading
 * from mapped pinned host memory (the SM variant of the host hops). */
int mp_measure_paths(mp_ctx* ctx, int32_t src_dev, int32_t dst_dev, uint64_t bytes,
                     int32_t iters, double* out_gbps, int32_t cap);

/* Device time of the transfer kernel of the last streamed-mode send (CUDA
 * events on its stream around that one launch, launch latency included).
 * Off by default (timing events cost ~2 launch slots per send): enable with
 * mp_ctx_set_kernel_timing(ctx, 1). */
int mp_ctx_set_kernel_timing(mp_ctx* ctx, int32_t on);
int mp_kernel_time_ms(const mp_ctx* ctx, double* ms);
/* Average duration of the src device's transfer kernel for this transfer's
 * program over `reps` back-to-back launches between two CUDA events on its
 * stream (launch gaps amortised): the roofline denominator.  Only the kernel
 * runs (copy-engine lanes are not enqueued); synchronous. */
int mp_kernel_bench(mp_ctx* ctx, const void* src, void* dst, uint64_t size, int32_t src_dev,
                    int32_t dst_dev, const mp_config* cfg, int32_t reps, double* ms_per_launch);

/* ---- CUDA IPC (multi-process mode) --------------------------------------- */
#define MP_IPC_HANDLE_BYTES 64
/* Handle of the allocation holding dev_ptr, and dev_ptr's offset in it. */
int mp_ipc_export(const void* dev_ptr, int32_t device, uint8_t* handle_out,
                  uint64_t* offset_out);
int mp_ipc_import(const uint8_t* handle, int32_t device, void** dev_ptr_out);
int mp_ipc_close(void* dev_ptr, int32_t device);

/* ---- multi-process group mode (one process per GPU) ------------------------
 * The paper's UCX cuda_ipc setting: ranks exchange CUDA-IPC
 * handles once (rendezvous, cached) and every transfer is issued collectively:
 * the source rank pushes Direct and hop1 tiles into IPC-mapped peer memory,
 * each relay rank runs its hop2 tiles, the destination rank waits until all
 * bytes landed.  A device-side generation barrier orders consecutive
 * transfers, so cached CUDA graphs replay without host synchronisation.
 * The host-staged path needs every rank's host inbox (mp_group_host_arena):
 * the sender's kernel writes a host chunk into the destination rank's inbox
 * (shared pinned memory) and releases the chunk's flag in the destination's
 * HBM; the destination's kernel loads it back. */
#define MP_GROUP_BLOB_BYTES 256
int mp_group_create(int32_t nranks, int32_t rank, int32_t device, uint64_t stage_bytes,
                    int32_t flag_cap, mp_ctx** out);
/* This rank's host inbox for the host-staged path (paths.py:165-166): `bytes`
 * of POSIX shared memory, pinned and mapped (cudaHostRegister) here and in
 * every peer at mp_group_import.  Call before mp_group_export; optional
 * (without it a host-staged plan fails with MP_ERR_STATE). */
int mp_group_host_arena(mp_ctx* ctx, uint64_t bytes);
int mp_group_export(const mp_ctx* ctx, uint8_t* blob);
int mp_group_import(mp_ctx* ctx, int32_t rank, const uint8_t* blob);
/* Map a peer buffer (handle from mp_ipc_export) into this process, cached. */
int mp_group_open(mp_ctx* ctx, const uint8_t* handle, uint64_t offset, void** ptr);
/* Collective: every rank calls it for every transfer, in the same order.
 * src: the sender's buffer (NULL elsewhere); src_align = src address mod 16
 * (all ranks); dst: the destination buffer as mapped in this process. */
int mp_group_send(mp_ctx* ctx, const void* src, uint32_t src_align, void* dst, uint64_t size,
                  int32_t src_rank, int32_t dst_rank, const mp_config* cfg, void* stream);
/* Role of this rank in the last transfer: 1 sender, 2 relay, 3 receiver, 0 none. */
int mp_group_role(const mp_ctx* ctx, int32_t* role);

#ifdef __cplusplus
}
#endif
#endif /* MPB200_H */
