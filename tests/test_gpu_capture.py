"""Engine sends inside a caller's own CUDA graph capture (torch.cuda.graph):
a cached send is recorded as graph nodes and replays byte-exact (single
kernel, direct + host with a roundtrip, streamed programs, send_many
windows); a send that would miss the plan cache is refused with a clear
error before touching the capture; and eager sends on other streams keep
working after captures (no engine event is recorded inside a capture)."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20


def _replay_ok(g, pairs, reps=3):
    for _ in range(reps):
        for src, dst in pairs:
            src.random_(0, 256)
            dst.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        if not all(torch.equal(s, d) for s, d in pairs):
            return False
    return True


@pytest.mark.parametrize("cfg_args,n", [((1, False, 1, True), 16 * MiB), ((1, True, 8, True), 64 * MiB + 3),
                                        ((1, True, 4, False), 24 * MiB + 5), ((3, True, 4, True), 8 * MiB + 1)])
def test_cached_send_captured_into_a_user_graph(cfg_args, n):
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
    eng = Engine(load_topology(mesh_text("cap", 4, 2e12, 1, 2e-6, 40e9, 1e-5, "full")), [0] * 4)
    cfg = PathConfig(*cfg_args)
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    s = torch.cuda.Stream()
    eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)  # warm: the plan is cached
    s.synchronize()
    eng.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
    assert _replay_ok(g, [(src, dst)])
    # eager sends on another stream still work after the capture
    other = torch.cuda.Stream()
    src.random_(0, 256)
    dst.zero_()
    torch.cuda.synchronize()
    eng.send(src, dst, n, cfg, stream=other, src_dev=0, dst_dev=1)
    eng.recv(dst, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    eng.sync()
    assert torch.equal(src, dst)
    eng.close()


def test_window_program_captured():
    from paper_2604_22228_b200 import Engine, PathConfig
    eng = Engine.loopback(2)
    pairs = [(torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0"),
              torch.zeros(n, dtype=torch.uint8, device="cuda:0")) for n in (MiB + 3, 4 * MiB, 9 * MiB + 1)]
    cfg = PathConfig(1, True, 4, True)
    s = torch.cuda.Stream()
    post = eng.prepare_many([(a, b, None, 0, 1) for a, b in pairs], cfg, stream=s)
    post()
    s.synchronize()
    eng.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        post()
    assert _replay_ok(g, pairs)
    eng.close()


def test_a_miss_inside_a_capture_is_refused():
    from paper_2604_22228_b200 import Engine, EngineError, PathConfig
    eng = Engine.loopback(2)
    n = 8 * MiB + 7
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(EngineError, match="capture must hit the plan cache"):
        with torch.cuda.graph(g, stream=s):
            eng.send(src, dst, n, PathConfig(1, True, 4, True), stream=s, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    # the engine is unharmed: the same send works eagerly, then captured
    eng.send(src, dst, n, PathConfig(1, True, 4, True), stream=s, src_dev=0, dst_dev=1)
    s.synchronize()
    eng.sync()
    assert torch.equal(src, dst)
    eng.close()


def test_captured_programs_are_pinned_against_eviction_and_arena_growth():
    """A captured program survives LRU eviction (its graph keeps replaying
    exactly), and a send that would have to grow the staging arenas — which
    would free the captured program's memory — is refused until clear_cache."""
    from paper_2604_22228_b200 import Engine, EngineError, PathConfig, load_topology, mesh_text
    eng = Engine(load_topology(mesh_text("pin", 3, 2e12, 1, 2e-6, 40e9, 1e-5, "full")), [0] * 3)
    relay = PathConfig(2, True, 4, True, cache_capacity=2)
    n = 4 * MiB + 3
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    s = torch.cuda.Stream()
    eng.send(src, dst, n, relay, stream=s, src_dev=0, dst_dev=1)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.send(src, dst, n, relay, stream=s, src_dev=0, dst_dev=1)
    # churn the LRU (capacity 2) with other small relay sends
    others = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda:0") for m in (MiB, 2 * MiB, 3 * MiB)]
    outs = [torch.zeros_like(o) for o in others]
    for o, d in zip(others, outs):
        eng.send(o, d, o.numel(), relay, stream=s, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    assert eng.stats().cache_evictions >= 1
    assert _replay_ok(g, [(src, dst)])
    # a much larger relay share needs bigger arenas: refused while pinned
    big = torch.randint(0, 256, (256 * MiB,), dtype=torch.uint8, device="cuda:0")
    bout = torch.zeros_like(big)
    with pytest.raises(EngineError, match="larger staging arenas"):
        eng.send(big, bout, big.numel(), relay, stream=s, src_dev=0, dst_dev=1)
    assert _replay_ok(g, [(src, dst)])  # still valid
    del g
    eng.clear_cache()  # the caller drops its graphs; now the arenas may grow
    eng.send(big, bout, big.numel(), relay, stream=s, src_dev=0, dst_dev=1)
    s.synchronize()
    eng.sync()
    assert torch.equal(big, bout)
    eng.close()


@pytest.mark.parametrize("graph_mode", [True, False])
def test_capture_of_a_program_with_copy_engine_lanes(graph_mode):
    """host = "ce": the program forks onto the engine's lane streams (2-D
    D2H / H2D copies) and joins back — inside a capture those streams join
    the caller's graph; replays are byte-exact."""
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
    eng = Engine(load_topology(mesh_text("ce", 2, 2e12, 1, 2e-6, 50e9, 1e-5, "full")), [0, 0])
    eng.configure(host="ce")
    cfg = PathConfig(1, True, 8, graph_mode)
    n = 96 * MiB + 5
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    s = torch.cuda.Stream()
    eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
    s.synchronize()
    assert eng.stats().ce_copies > 0
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
    assert _replay_ok(g, [(src, dst)])
    eng.close()


def test_send_recv_and_consumer_captured_together():
    """The pattern send -> recv -> consumer, all recorded in one capture
    after an eager send on another stream: recv inside the capture is a
    no-op (the captured send is already ordered on the capture stream), the
    capture stays valid, and replays deliver before the consumer reads."""
    from paper_2604_22228_b200 import Engine, PathConfig
    eng = Engine.loopback(2)
    n = 32 * MiB + 1
    cfg = PathConfig(1, True, 8, True)
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    tail = torch.zeros(MiB, dtype=torch.uint8, device="cuda:0")
    eng.send(src, dst, n, cfg, stream=torch.cuda.Stream(), src_dev=0, dst_dev=1)  # eager, other stream
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
        eng.recv(dst, stream=s)
        tail.copy_(dst[-MiB:])
    for _ in range(3):
        src.random_(0, 256)
        dst.zero_()
        tail.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(tail, src[-MiB:]) and torch.equal(src, dst)
    eng.close()
