"""Concurrent transfers as one program (the reference's
simulate_concurrent, sim.py:287-292): windows of messages, bidirectional
flows (BIBW) and the 4-rank Jacobi ring halo exchange with contention-free
relay planning (paths.py:210-242), all executed by one kernel per device."""

import numpy as np
import pytest

from oracle import transfer as ot

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20


def _engine(n, **opts):
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    eng = Engine(load_topology(mesh_text("loop", n, 2.0e12, 1, 2e-6, 50e9, 1e-5, "full")), [0] * n)
    if opts:
        eng.configure(**opts)
    return eng


def _bufs(sizes, seed):
    srcs, dsts, datas = [], [], []
    for i, n in enumerate(sizes):
        d = ot.pattern(n, seed=seed + i)
        s = torch.from_numpy(d).to("cuda:0")
        datas.append(d)
        srcs.append(s)
        dsts.append(torch.bitwise_not(s))
    return srcs, dsts, datas


@pytest.mark.parametrize("graph", [False, True])
def test_window_of_messages(graph):
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(2)
    sizes = [4 * MiB + 1, 3 * MiB + 7, 1, 1234567]
    srcs, dsts, datas = _bufs(sizes, 3)
    cfg = PathConfig(host_path_enabled=True, max_chunks=4, graph_mode=graph)
    for rep in range(3):
        eng.send_many([(s, d, None, 0, 1) for s, d in zip(srcs, dsts)], cfg)
        eng.sync()
        for d, want in zip(dsts, datas):
            assert np.array_equal(d.cpu().numpy(), want)
        for d in dsts:
            d.fill_(0)
    eng.close()


@pytest.mark.parametrize("host", [False, True])
def test_prepared_window(host):
    """prepare_many: a bound program resent several times is byte-exact each
    time, and refuses to run after the engine is closed."""
    from paper_2604_22228_b200 import EngineError, PathConfig
    eng = _engine(2)
    sizes = [1, 4096 + 3, 65536, MiB + 17] * 16  # a 64-message window
    srcs, dsts, datas = _bufs(sizes, 11)
    post = eng.prepare_many([(s, d, None, 0, 1) for s, d in zip(srcs, dsts)],
                            PathConfig(host_path_enabled=host, max_chunks=2, graph_mode=True))
    for rep in range(3):
        post()
        eng.sync()
        for d, want in zip(dsts, datas):
            assert np.array_equal(d.cpu().numpy(), want)
        for d in dsts:
            d.fill_(0)
    eng.close()
    with pytest.raises(EngineError):
        post()


def test_program_resend_fast_path_follows_the_cache():
    """mp_send_many remembers the last program's arguments and entry; the
    memo must follow evictions, cache clears and other programs: every
    resend is byte-exact and hit/miss is what the LRU says."""
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(2)
    srcs, dsts, datas = _bufs([4096 + 1, 70000, 3 * MiB + 5, 17], 21)
    cfg = PathConfig(max_chunks=2, graph_mode=True, cache_capacity=1)
    prog_a = [(srcs[0], dsts[0], None, 0, 1), (srcs[1], dsts[1], None, 0, 1)]
    prog_b = [(srcs[2], dsts[2], None, 0, 1), (srcs[3], dsts[3], None, 0, 1)]

    def post(prog, want_hit):
        for _, d, _, _, _ in prog:
            d.zero_()
        eng.send_many(prog, cfg)
        eng.sync()
        assert eng.stats().hit == want_hit
        for s, d, _, _, _ in prog:
            assert torch.equal(s, d)

    post(prog_a, 0)
    post(prog_a, 1)                    # fast path
    post(prog_b, 0)                    # capacity 1: evicts A
    post(prog_a, 0)                    # memo of A is stale: rebuilt
    post(prog_a, 1)
    eng.send(srcs[3], dsts[3], None, cfg, src_dev=0, dst_dev=1)   # evicts A
    eng.sync()
    post(prog_a, 0)
    eng.clear_cache()
    post(prog_a, 0)
    post(prog_a, 1)
    eng.close()


@pytest.mark.parametrize("relay", ["sm", "ce"])
def test_bidirectional_flows(relay):
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(4, relay=relay)
    srcs, dsts, datas = _bufs([8 * MiB + 5, 8 * MiB + 9], 7)
    cfg = PathConfig(num_gpu_paths=3, host_path_enabled=True, max_chunks=4, graph_mode=True,
                     share_policy="equal")
    eng.send_many([(srcs[0], dsts[0], None, 0, 1), (srcs[1], dsts[1], None, 1, 0)], cfg)
    eng.sync()
    for d, want in zip(dsts, datas):
        assert np.array_equal(d.cpu().numpy(), want)
    eng.close()


def test_jacobi_ring_contention_free():
    """Ring 0->1->2->3->0, two GPU paths each: joint planning stages every
    transfer through its source's diagonal peer (test_paths.py:88-99)."""
    import paper_2604_22228_b200 as mp
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(4)
    ring = [(0, 1), (1, 2), (2, 3), (3, 0)]
    srcs, dsts, datas = _bufs([6 * MiB + 3] * 4, 11)
    cfg = PathConfig(num_gpu_paths=2, max_chunks=4, graph_mode=True, share_policy="equal")
    joint = mp.plan_contention_free(eng.topology, [(eng.topology.device(a), eng.topology.device(b))
                                                   for a, b in ring], cfg)
    assert joint.contention_free
    assert [ps.paths[1].stage.index for ps in joint.path_sets] == [2, 3, 0, 1]
    for rep in range(2):
        eng.send_many([(s, d, None, a, b) for (a, b), s, d in zip(ring, srcs, dsts)], cfg,
                      joint=True)
        eng.sync()
        for d, want in zip(dsts, datas):
            assert np.array_equal(d.cpu().numpy(), want)
        for d in dsts:
            d.zero_()
    assert eng.stats().kernels == 1  # every transfer's tiles in one kernel (loopback)
    eng.close()


@pytest.mark.parametrize("graph", [False, True])
def test_programs_with_the_cross_device_lowering(graph):
    """fault_inject & 2 (logical GPUs lowered as separate devices: system-
    scope relay / host flags, host chunks as hop1 / hop2 tiles): a BIBW
    pair through relays + host and a 4-ring halo exchange as ONE program
    each, resent back to back, byte-exact."""
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(4, fault_inject=2)
    srcs, dsts, datas = _bufs([6 * MiB + 5, 6 * MiB + 9, 2 * MiB + 1, 2 * MiB + 3, 2 * MiB + 7, 2 * MiB + 11], 21)
    bibw = eng.prepare_many([(srcs[0], dsts[0], None, 0, 1), (srcs[1], dsts[1], None, 1, 0)],
                            PathConfig(num_gpu_paths=3, host_path_enabled=True, max_chunks=4, graph_mode=graph,
                                       share_policy="equal"))
    ring = eng.prepare_many([(srcs[2 + r], dsts[2 + r], None, r, (r + 1) % 4) for r in range(4)],
                            PathConfig(num_gpu_paths=2, host_path_enabled=True, max_chunks=3, graph_mode=graph),
                            joint=True)
    for _ in range(3):
        for d in dsts:
            d.fill_(0)
        bibw()
        ring()
        bibw()
        eng.sync()
        for d, want in zip(dsts, datas):
            assert np.array_equal(d.cpu().numpy(), want)
    eng.close()
