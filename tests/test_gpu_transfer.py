"""GPU parity: bytes delivered by the CUDA engine equal the oracle's, and the
chunk plan the engine executed equals the oracle's plan, on the same inputs.

Every multi-GPU path runs on one B200 through loopback: logical GPUs 0..n-1
of the topology all map to cuda:0 (device_map), so direct, relay (with the
cross-CTA flag handoff) and host-staged paths execute for real.
dst is pre-poisoned with ~src so any byte not written fails the comparison.
"""

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MiB = 1 << 20


def _topo_text(n, link=2.0e12, host=50e9):
    from paper_2604_22228_b200 import mesh_text
    return mesh_text("loop", n, link, 1, 2e-6, host, 10e-6, "full")


def _engine(n=4, **opts):
    from paper_2604_22228_b200 import Engine, load_topology
    text = _topo_text(n)
    eng = Engine(load_topology(text), [0] * n)
    if opts:
        eng.configure(**opts)
    return eng, text


def _check(eng, text, size, *, gpu_paths=1, host=False, chunks=1, graph=False,
           src_off=0, dst_off=0, seed=None, policy="bandwidth_proportional", reps=1,
           cache=16):
    from paper_2604_22228_b200 import PathConfig
    cfg = PathConfig(num_gpu_paths=gpu_paths, host_path_enabled=host, max_chunks=chunks,
                     graph_mode=graph, share_policy=policy, cache_capacity=cache)
    src_buf = torch.empty(size + src_off + 64, dtype=torch.uint8, device="cuda:0")
    dst_buf = torch.empty(size + dst_off + 64, dtype=torch.uint8, device="cuda:0")
    src = src_buf[src_off:src_off + size]
    dst = dst_buf[dst_off:dst_off + size]
    t = op.parse_topology(text)
    opaths = op.plan_paths(t, 0, 1, gpu_paths, host, policy)
    ochunks = op.make_chunk_plan([p["share"] for p in opaths], size, chunks)
    for r in range(reps):
        data = ot.pattern(size, seed=None if seed is None else seed + r)
        src.copy_(torch.from_numpy(data))
        dst_buf.fill_(0x5A)  # guard bytes around dst: never written
        dst.copy_(torch.bitwise_not(src))
        eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
        eng.sync()
        torch.cuda.synchronize()
        assert bool((dst_buf[:dst_off] == 0x5A).all()) and bool((dst_buf[dst_off + size:] == 0x5A).all()), \
            "bytes outside the destination range were written"
        expect = np.empty_like(data)
        ot.run(data, expect, [p["kind"] for p in opaths], ochunks, threads=4)
        got = dst.cpu().numpy()
        assert np.array_equal(got, expect), f"byte mismatch at rep {r}: first bad index " \
            f"{int(np.nonzero(got != expect)[0][0])}"
    paths, chunks_done = eng.last_plan()
    assert [(c.path_index, c.offset, c.length, c.seq) for c in chunks_done] == ochunks
    assert [p.share for p in paths] == [p["share"] for p in opaths]
    return eng.stats()


@pytest.mark.parametrize("copy", ["vec", "tma"])
@pytest.mark.parametrize("size", [1, 15, 16, 17, 4095, 65536 + 3, MiB + 7, 16 * MiB])
@pytest.mark.parametrize("graph", [False, True])
def test_direct_sizes(size, graph, copy):
    eng, text = _engine(2, copy=copy)
    _check(eng, text, size, graph=graph)
    eng.close()


@pytest.mark.parametrize("direct,host", [("sm", "ce"), ("ce", "ce"), ("sm", "sm")])
@pytest.mark.parametrize("k", [1, 2, 4, 8, 16, 32])
def test_config1_direct_plus_host_64mib(direct, host, k):
    """BASELINE config 1: 64 MiB over direct + host-staged, K chunks per path
    (host hops by copy engines or by the SM kernels over mapped memory)."""
    eng, text = _engine(2, direct=direct, host=host)
    st = _check(eng, text, 64 * MiB, host=True, chunks=k, graph=True)
    assert st.nodes_logical == sum(1 if p == 0 else 2 for p, *_ in
                                   op.make_chunk_plan(
                                       [q["share"] for q in op.plan_paths(
                                           op.parse_topology(text), 0, 1, 1, True)],
                                       64 * MiB, k))
    eng.close()


@pytest.mark.parametrize("relay,copy", [("sm", "vec"), ("sm", "tma"), ("ce", "vec")])
@pytest.mark.parametrize("gpu_paths", [2, 3, 4])
@pytest.mark.parametrize("graph", [False, True])
def test_gpu_relays(relay, copy, gpu_paths, graph):
    """Direct + 1..3 GPU relays (+host): relay flags / events order hop2 after hop1."""
    eng, text = _engine(gpu_paths + 1, relay=relay, copy=copy, tile_bytes=256 << 10)
    _check(eng, text, 8 * MiB + 12345, gpu_paths=gpu_paths, host=True, chunks=4, graph=graph,
           policy="equal", reps=2)
    eng.close()


def test_eight_logical_gpus_six_relays():
    """BASELINE config 4 shape: direct + 6 relays + host, max_chunks 16."""
    eng, text = _engine(8)
    _check(eng, text, 32 * MiB + 1, gpu_paths=7, host=True, chunks=16, graph=True,
           policy="equal")
    eng.close()


@pytest.mark.parametrize("copy", ["vec", "tma"])
@pytest.mark.parametrize("offs", [(0, 0), (5, 5), (3, 7), (8, 0), (1, 2), (2, 6)])
def test_misaligned_buffers(offs, copy):
    eng, text = _engine(3, copy=copy)
    _check(eng, text, 3 * MiB + 11, gpu_paths=2, host=True, chunks=5, src_off=offs[0],
           dst_off=offs[1], policy="equal")
    eng.close()


@pytest.mark.parametrize("copy", ["vec", "tma"])
def test_graph_replay_fresh_data_every_time(copy):
    """A cached graph replayed many times with new source bytes: relay flags
    must re-arm themselves (no memset node)."""
    eng, text = _engine(4, copy=copy, tile_bytes=64 << 10)
    st = _check(eng, text, 4 * MiB + 99, gpu_paths=3, host=True, chunks=8, graph=True,
                seed=7, reps=12, policy="equal")
    assert st.hit and st.cache_hits >= 11
    eng.close()


def test_host_double_buffer_war():
    """2 pinned slots for many host chunks: slot reuse waits for the H2D (WAR)."""
    eng, text = _engine(2, host_slots=2)
    _check(eng, text, 16 * MiB + 5, host=True, chunks=16, graph=True, policy="equal", reps=3,
           seed=3)
    _check(eng, text, 16 * MiB + 5, host=True, chunks=16, graph=False, policy="equal", reps=2,
           seed=5)
    eng.close()


def test_lru_eviction_counts():
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(2)
    cfg = PathConfig(max_chunks=2, graph_mode=True, cache_capacity=2)
    src = torch.arange(4096, dtype=torch.int32, device="cuda:0").view(torch.uint8)
    dsts = [torch.zeros_like(src) for _ in range(3)]
    hits = []
    for i in [0, 1, 0, 2, 1]:
        eng.send(src, dsts[i], None, cfg, src_dev=0, dst_dev=1)
        hits.append(eng.stats().hit)
    eng.sync()
    assert hits == [False, False, True, False, False]  # oracle LRU: 1 evicted by 2
    lru = op.LRU(2)
    assert [lru.access(k) for k in [0, 1, 0, 2, 1]] == hits
    for d in dsts:
        assert torch.equal(d, src)
    eng.close()


def test_streams_and_events_order_with_user_work():
    """send is asynchronous on the caller's stream: work queued before it is
    seen by the copy, work queued after it sees the delivered bytes."""
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(3)
    cfg = PathConfig(num_gpu_paths=2, host_path_enabled=True, max_chunks=4, graph_mode=True)
    s = torch.cuda.Stream()
    n = 8 * MiB
    src = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    with torch.cuda.stream(s):
        for v in range(1, 6):
            src.fill_(v)
            eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
            total = dst.sum(dtype=torch.int64)
            assert int(total) == v * n
    eng.close()


def test_full_size_512mib_multipath_bytes_exact():
    """BASELINE size: 512 MiB + 7 over direct + 2 relays + host, compared on
    the device (size-independent property: dst == src everywhere)."""
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(4)
    n = 512 * MiB + 7
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0",
                        generator=torch.Generator(device="cuda:0").manual_seed(20261017))
    dst = torch.bitwise_not(src)
    for graph in (False, True):
        cfg = PathConfig(num_gpu_paths=3, host_path_enabled=True, max_chunks=8, graph_mode=graph)
        eng.send(src, dst, n, cfg, src_dev=0, dst_dev=1)
        eng.sync()
        assert torch.equal(src, dst)
        dst.bitwise_not_()
    eng.close()


def test_probe_node_writes_a_plannable_topology():
    import paper_2604_22228_b200 as mp
    eng, _ = _engine(3)
    text = eng.probe_node(64 * MiB, 3, name="probed3")
    topo = mp.load_topology(text)
    assert topo.name == "probed3" and len(topo.accelerators) == 3
    assert all(ch.bandwidth > 1e9 for ch in topo.channels())
    ps = mp.plan_paths(topo, topo.device(0), topo.device(1),
                       mp.PathConfig(num_gpu_paths=2, host_path_enabled=True))
    assert abs(sum(p.share for p in ps.paths) - 1.0) < 1e-12
    eng.close()


@pytest.mark.parametrize("graph", [False, True])
def test_peer_table_fallback_kernel(graph):
    """Tables touching another GPU run the LDG/STG kernel (tma_peer = 0);
    tma_peer = -1 forces that launch path on one GPU so it is exercised."""
    eng, text = _engine(4, tma_peer=-1)
    _check(eng, text, 8 * MiB + 333, gpu_paths=3, host=True, chunks=4, graph=graph,
           policy="equal", src_off=3, dst_off=3, reps=2, seed=9)
    eng.close()


@pytest.mark.parametrize("mode", ["small", "static", "dynamic"])
@pytest.mark.parametrize("size,chunks,host,offs", [
    (1, 1, False, (0, 0)), (4095, 1, False, (3, 3)), (4096, 3, False, (0, 0)),
    (65536 + 3, 2, True, (5, 9)), (MiB + 7, 8, False, (1, 1)), (3 * MiB + 5, 16, True, (7, 3)),
    (20 * MiB + 1, 4, False, (0, 8)), (70 * MiB + 13, 8, True, (2, 2))])
def test_tile_schedules(mode, size, chunks, host, offs):
    """The three SM schedules of a direct table deliver the same bytes:
    the one-launch-slot small kernel (static tables <= small_max_bytes), the
    static one-tile-per-CTA TMA table, and dynamic claims — with chunked
    (multi-segment), misaligned and direct+host (CE) plans, replayed."""
    opts = {"small": {}, "static": {"small_max_bytes": 0}, "dynamic": {"sched": "dynamic"}}[mode]
    eng, text = _engine(2, **opts)
    _check(eng, text, size, host=host, chunks=chunks, graph=True, src_off=offs[0],
           dst_off=offs[1], seed=11, reps=2)
    eng.close()


@pytest.mark.parametrize("size,opts,kernel", [
    (4096, {}, "small_copy_kernel"), (4 * MiB, {}, "small_copy_kernel"),
    (32 * MiB, {}, "transfer_kernel<1,8>"), (160 * MiB, {}, "transfer_kernel<0,8>"),
    (32 * MiB, {"tma_peer": -1}, "transfer_kernel<0,8>"),
    (32 * MiB, {"small_max_bytes": 64 << 20}, "small_copy_kernel"),
    (4096, {"sched": "dynamic"}, "transfer_kernel<0,8>"),
    (160 * MiB, {"copy": "tma", "ctas_per_sm": 1, "threads": 128}, "transfer_kernel<1,8>")])
def test_kernel_choice_by_size(size, opts, kernel):
    """The measured per-table kernel policy (csrc/mp_engine.cu ProgKind),
    reported by the send statistics, delivering exact bytes."""
    eng, text = _engine(2, **opts)
    st = _check(eng, text, size, graph=True, seed=5)
    assert kernel in st.kernel, st.kernel
    eng.close()


@pytest.mark.parametrize("size,chunks", [(1000, 3), (3 * MiB + 17, 8), (9 * MiB, 16),
                                         (40 * MiB + 5, 5), (40 * MiB + 5, 32)])
@pytest.mark.parametrize("graph", [False, True])
def test_host_path_2d_groups(size, chunks, graph):
    """CE host path as 2-D copy groups (csrc/mp_engine.cu HostRow): a host
    share of 1/3 gives several groups, a truncated last chunk its own group;
    bytes and plan stay exact, and there are at most 2 copies per group."""
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    text = mesh_text("loop", 2, 2.0e12, 1, 2e-6, 1.0e12, 10e-6, "full")
    eng = Engine(load_topology(text), [0, 0])
    eng.configure(host="ce")
    st = _check(eng, text, size, host=True, chunks=chunks, graph=graph, reps=2, seed=13,
                src_off=3, dst_off=3)
    assert st.ce_copies <= 2 * 5
    eng.close()


@pytest.mark.parametrize("gpu_paths,host,chunks", [(1, False, 1), (1, True, 8), (2, True, 4)])
def test_huge_message_beyond_4gib(gpu_paths, host, chunks):
    """A 4.5 GiB + 5 message (byte counts past 32 bits; host chunk stride
    near the 2-D copy pitch limit), compared on the device, plan = oracle."""
    from paper_2604_22228_b200 import PathConfig
    eng, text = _engine(3)
    n = (9 << 29) + 5
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0",
                        generator=torch.Generator(device="cuda:0").manual_seed(7))
    dst = torch.bitwise_not(src)
    cfg = PathConfig(num_gpu_paths=gpu_paths, host_path_enabled=host, max_chunks=chunks,
                     graph_mode=True)
    eng.send(src, dst, n, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    assert torch.equal(src, dst)
    t = op.parse_topology(text)
    opaths = op.plan_paths(t, 0, 1, gpu_paths, host)
    ochunks = op.make_chunk_plan([p["share"] for p in opaths], n, chunks)
    _, done = eng.last_plan()
    assert [(c.path_index, c.offset, c.length, c.seq) for c in done] == ochunks
    del src, dst
    eng.close()
    torch.cuda.empty_cache()


def test_kernel_timing_is_opt_in_and_errors_reraise():
    """Streamed-mode kernel timing is off by default and on after
    set_kernel_timing(True); ABI errors raised through the CPython fast path
    keep the reference's exception classes and wording."""
    from paper_2604_22228_b200 import ChunkError, PathConfig
    from paper_2604_22228_b200._lib import EngineError
    eng, _ = _engine(2)
    src = torch.zeros(MiB, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty_like(src)
    cfg = PathConfig(max_chunks=1, graph_mode=False)
    eng.send(src, dst, MiB, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    with pytest.raises(EngineError, match="no timed kernel"):
        eng.kernel_time_ms()
    eng.set_kernel_timing(True)
    eng.send(src, dst, MiB, cfg, src_dev=0, dst_dev=1)
    assert eng.kernel_time_ms() > 0
    with pytest.raises(ChunkError, match="message size must be >= 1 byte"):
        eng.send(src, dst, 0, cfg, src_dev=0, dst_dev=1)
    eng.close()
    with pytest.raises(ValueError, match="null"):
        eng.send_ptr(src.data_ptr(), dst.data_ptr(), 16, 0, 1, cfg)


def test_prepared_send_replays_and_guards_close():
    """Engine.prepare binds a send once; calling it replays the cached graph
    (fresh bytes each time) and refuses to run after the engine is closed."""
    from paper_2604_22228_b200 import PathConfig
    from paper_2604_22228_b200._lib import EngineError
    eng, _ = _engine(2)
    n = 3 * MiB + 7
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty_like(src)
    go = eng.prepare(src, dst, n, PathConfig(max_chunks=4, graph_mode=True), src_dev=0, dst_dev=1)
    for r in range(5):
        src.copy_(torch.from_numpy(ot.pattern(n, seed=r)))
        dst.fill_(0)
        go()
        eng.sync()
        assert torch.equal(src, dst)
    assert eng.stats().cache_hits >= 4
    eng.close()
    with pytest.raises(EngineError, match="after Engine.close"):
        go()


def test_send_rejects_host_and_strided_tensors():
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(2)
    cfg = PathConfig()
    a = torch.zeros(1024, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ValueError, match="CUDA tensors"):
        eng.send(a.cpu(), a, 1024, cfg, src_dev=0, dst_dev=1)
    m = torch.zeros(64, 64, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ValueError, match="contiguous"):
        eng.send(m.t(), torch.empty_like(m), None, cfg, src_dev=0, dst_dev=1)
    eng.close()


def test_streamed_dynamic_tables_match_graph_replays():
    """Per-call (streamed) sends of a dynamic table issued back to back on a
    non-blocking stream right after the entry is built: bytes exact, and the
    launch-parity claim counters stay in step — a desynchronised counter
    makes CTAs re-claim tiles (correct bytes, ~1.5x the time), so the
    streamed rate must stay within 25% of cached-graph replays."""
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(2)
    n = 256 * MiB
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.empty_like(src)
    s = torch.cuda.Stream()
    rates = {}
    for graph in (False, True):
        cfg = PathConfig(max_chunks=1, graph_mode=graph)
        with torch.cuda.stream(s):
            for _ in range(3):
                eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
            e1.record(s)
        torch.cuda.synchronize()
        assert torch.equal(src, dst)
        rates[graph] = e0.elapsed_time(e1)
    assert rates[False] < 1.25 * rates[True], rates
    eng.close()


@pytest.mark.parametrize("pdl", [0, 1, 2, 3])
def test_chained_sends_keep_stream_order(pdl):
    """Back-to-back sends where each reads what the previous one wrote
    (a -> b, then b -> c, with a rewritten in between): with programmatic
    dependent launch the next kernel may start early, so its
    griddepcontrol.wait must order every access after the previous send."""
    from paper_2604_22228_b200 import Engine, PathConfig
    eng = Engine.loopback(2)
    eng.configure(pdl=pdl)
    cfg = PathConfig(max_chunks=1, graph_mode=True)
    for n in (4096 + 5, 65536, (1 << 20) + 3, 3 << 20, (16 << 20) + 7, (160 << 20) + 9):
        a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        b = torch.zeros_like(a)
        c = torch.zeros_like(a)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for r in range(40):
                a.fill_(r)
                eng.send(a, b, n, cfg, stream=s, src_dev=0, dst_dev=1)
                eng.send(b, c, n, cfg, stream=s, src_dev=0, dst_dev=1)
                eng.send(c, a, n, cfg, stream=s, src_dev=0, dst_dev=1)
                eng.send(a, b, n, cfg, stream=s, src_dev=0, dst_dev=1)
        s.synchronize()
        want = ("mpk::small_copy_kernel" if n < (4 << 20) else
                "mpk::transfer_kernel<1" if n < (64 << 20) else "mpk::transfer_kernel<0")
        assert eng.stats().kernel.startswith(want)
        assert bool((b == 39).all()) and bool((c == 39).all())
    eng.close()


@pytest.mark.parametrize("host,graph", [(False, True), (True, True), (True, False)])
def test_recv_orders_a_consumer_stream_after_the_send(host, graph):
    """Engine.recv (mp_wait): a consumer on ANOTHER stream that reads dst
    right after recv sees the delivered bytes — the tail of a 256 MiB
    message, the last bytes a multi-path send writes — never stale ones."""
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(2)
    n = 256 * MiB + 5
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.empty_like(src)
    tail = torch.empty(MiB, dtype=torch.uint8, device="cuda:0")
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    cfg = PathConfig(host_path_enabled=host, max_chunks=8, graph_mode=graph)
    for r in range(4):
        dst.fill_(r)
        torch.cuda.synchronize()
        eng.send(src, dst, n, cfg, stream=a, src_dev=0, dst_dev=1)
        eng.recv(dst, stream=b)
        with torch.cuda.stream(b):
            tail.copy_(dst[-MiB:])
        b.synchronize()
        assert torch.equal(tail, src[-MiB:]), f"round {r}: the consumer read before the send finished"
    eng.sync()
    eng.close()


def test_eviction_under_multi_stream_churn():
    """cache_capacity 2 with 8 buffer pairs sent round-robin from 3 streams:
    every send after the first two evicts an entry whose graph may still be
    replaying on another stream.  Each pair's last delivery must be exact."""
    from paper_2604_22228_b200 import PathConfig
    eng, _ = _engine(3)
    cfgs = [PathConfig(1, True, 4, True, cache_capacity=2), PathConfig(2, True, 3, True, cache_capacity=2),
            PathConfig(1, False, 2, False, cache_capacity=2)]
    pairs = []
    for i in range(8):
        n = (2 + i) * MiB + 13 * i
        data = ot.pattern(n, seed=40 + i)
        pairs.append((torch.from_numpy(data).to("cuda:0"), torch.empty(n, dtype=torch.uint8, device="cuda:0"),
                      n, data))
    streams = [torch.cuda.Stream() for _ in range(3)]
    for r in range(5):
        for i, (src, dst, n, _) in enumerate(pairs):
            k = (r + i) % 3
            eng.send(src, dst, n, cfgs[k], stream=streams[k], src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    eng.sync()
    assert eng.stats().cache_evictions >= 30
    for src, dst, n, data in pairs:
        assert np.array_equal(dst.cpu().numpy(), data), f"{n} B"
    eng.close()


def test_no_device_memory_leak_over_cache_churn_and_engine_cycles():
    """300 distinct cached sends (capacity 4: constant eviction, graph
    destroy) and 20 engine create / close cycles leave the device's free
    memory where it was (tile tables, claim counters, arenas, graphs freed)."""
    from paper_2604_22228_b200 import PathConfig
    n = 256 * MiB  # dynamic tables of ~4k tiles (256 KiB each): a leak per entry shows
    base = torch.empty(n + 4096, dtype=torch.uint8, device="cuda:0")
    out = torch.empty_like(base)
    torch.cuda.synchronize()

    def free():
        torch.cuda.synchronize()
        return torch.cuda.mem_get_info(0)[0]
    f0 = free()
    for cycle in range(20):
        eng, _ = _engine(3)
        cfg = PathConfig(2, True, 3, True, cache_capacity=4)
        for i in range(15 if cycle else 300):
            off = (i * 16) % 4096
            eng.send(base[off:off + n], out[off:off + n], n, cfg, src_dev=0, dst_dev=1)
        eng.sync()
        eng.close()
    f1 = free()
    assert f0 - f1 < 16 * MiB, f"device memory dropped by {(f0 - f1) / MiB:.1f} MiB"


def test_default_usage_on_the_current_stream_with_typed_tensors():
    """The minimal call a user writes: eng.send(src, dst) with float tensors,
    no config (PathConfig.from_env), no stream (the current stream), no
    devices (from the tensors), then eng.recv(dst) on the current stream."""
    from paper_2604_22228_b200 import Engine, PathConfig
    eng = Engine.loopback(2)
    src = torch.randn(3 * MiB + 5, device="cuda:0")
    dst = torch.zeros_like(src)
    eng.send(src, dst)
    eng.recv(dst)
    assert torch.equal(src, dst)
    # a multi-path config on the default stream, then a torch op that reads dst
    src2 = torch.randn(8 * MiB + 3, dtype=torch.float64, device="cuda:0")
    dst2 = torch.zeros_like(src2)
    eng.send(src2, dst2, config=PathConfig(1, True, 4, True), src_dev=0, dst_dev=1)
    eng.recv(dst2)
    assert float((dst2 - src2).abs().max()) == 0.0
    eng.close()


def test_two_engines_interleaved_on_shared_and_separate_streams():
    """Two independent engines in one process (two libraries, say) sending
    interleaved on one stream and on their own streams: separate control
    blocks, arenas and caches — every delivery exact."""
    from paper_2604_22228_b200 import PathConfig
    a, _ = _engine(3)
    b, _ = _engine(2)
    shared, sa, sb = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    bufs = []
    for i, n in enumerate([5 * MiB + 1, 7 * MiB + 3, 96 * MiB + 5, 2 * MiB]):
        data = ot.pattern(n, seed=80 + i)
        bufs.append((torch.from_numpy(data).to("cuda:0"), torch.zeros(n, dtype=torch.uint8, device="cuda:0"), n, data))
    ca, cb = PathConfig(2, True, 4, True), PathConfig(1, True, 8, False)
    for r in range(4):
        for i, (src, dst, n, _) in enumerate(bufs):
            eng, cfg = (a, ca) if (i + r) % 2 == 0 else (b, cb)
            stream = shared if r % 2 == 0 else (sa if eng is a else sb)
            eng.send(src, dst, n, cfg, stream=stream, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    a.sync()
    b.sync()
    for src, dst, n, data in bufs:
        assert np.array_equal(dst.cpu().numpy(), data), n
    a.close()
    b.close()
