"""Multi-process group mode on one B200: 2-3 processes share cuda:0 through
CUDA IPC (each rank is a logical GPU).  The receiver's bytes must equal the
oracle's, over several back-to-back transfers (device barrier + flag re-arm),
in streamed and cached-graph modes, direct-only and with a relay rank."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import _dist_util  # noqa: E402

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _worker(rank, world, port, gpu_paths, graph, size, reps, host=False, host_bw=5.5e10):
    import numpy as np
    import torch.distributed as dist

    import paper_2604_22228_b200 as mp
    from oracle import planner as op
    from oracle import transfer as ot
    from paper_2604_22228_b200.group import TransferGroup
    _dist_util.init(rank, world, port)
    torch.cuda.set_device(0)
    topo = mp.load_topology(mp.mesh_text("g", world, 7.5e11, 1, 2e-6, host_bw, 1e-5, "full"))
    grp = TransferGroup(topo, device=0, stage_bytes=64 << 20)
    src = torch.empty(size + 3, dtype=torch.uint8, device="cuda:0")[3:]  # unaligned on purpose
    dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
    sb = grp.expose(src, owner=0)
    db = grp.expose(dst, owner=1)
    cfg = mp.PathConfig(num_gpu_paths=gpu_paths, host_path_enabled=host, max_chunks=4,
                        graph_mode=graph, share_policy="equal")
    for r in range(reps):
        data = ot.pattern(size, seed=100 + r)
        if rank == 0:
            src.copy_(torch.from_numpy(data))
        if rank == 1:
            dst.fill_(0xA5)
        torch.cuda.synchronize()
        dist.barrier()
        grp.transfer(sb, db, size, cfg)
        torch.cuda.synchronize()
        grp.sync()
        if rank == 1:
            got = dst.cpu().numpy()
            assert np.array_equal(got, data), f"rep {r}: mismatch"
            paths, chunks = grp.last_plan()
            ochunks = op.make_chunk_plan([p["share"] for p in op.plan_paths(
                op.parse_topology(mp.mesh_text("g", world, 7.5e11, 1, 2e-6, host_bw, 1e-5, "full")),
                0, 1, gpu_paths, host, "equal")], size, 4)
            assert [(c.path_index, c.offset, c.length, c.seq) for c in chunks] == ochunks
        dist.barrier()
    assert grp.role() == {0: 1, 1: 3}.get(rank, 2 if rank < gpu_paths + 1 else 0)
    grp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,gpu_paths", [(2, 1), (3, 2), (4, 2)])
@pytest.mark.parametrize("graph", [False, True])
def test_group_transfer(world, gpu_paths, graph):
    _dist_util.run(_worker, world, gpu_paths, graph, (4 << 20) + 12345, 3)


@pytest.mark.parametrize("world,gpu_paths", [(2, 1), (3, 2)])
@pytest.mark.parametrize("graph", [False, True])
def test_group_transfer_with_host_path(world, gpu_paths, graph):
    """Direct (+ relay) + host-staged in group mode: the sender's hop1 tiles
    write the destination rank's host inbox (POSIX shm, pinned and mapped
    in both processes) and release the chunk flag in the destination's HBM;
    the destination's kernel loads the chunk back, then waits for every byte."""
    _dist_util.run(_worker, world, gpu_paths, graph, (4 << 20) + 12345, 3, True)


def _b2b_worker(rank, world, port, gpu_paths, host, graph):
    import time

    import numpy as np
    import torch.distributed as dist

    import paper_2604_22228_b200 as mp
    from oracle import transfer as ot
    from paper_2604_22228_b200.group import TransferGroup
    _dist_util.init(rank, world, port)
    torch.cuda.set_device(0)
    size = (8 << 20) + 77
    topo = mp.load_topology(mp.mesh_text("g", world, 7.5e11, 1, 2e-6, 5.5e10, 1e-5, "full"))
    grp = TransferGroup(topo, device=0, stage_bytes=64 << 20)
    grp.configure(wait_timeout_ms=2000)
    src = torch.empty(size, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
    sb, db = grp.expose(src, owner=0), grp.expose(dst, owner=1)
    cfg = mp.PathConfig(num_gpu_paths=gpu_paths, host_path_enabled=host, max_chunks=4, graph_mode=graph)
    data = ot.pattern(size, seed=5)
    if rank == 0:
        src.copy_(torch.from_numpy(data))
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=0)
    grp.transfer(sb, db, size, cfg, stream=stream)  # first: capture / build on every rank
    stream.synchronize()
    grp.sync()
    dist.barrier()
    # every rank but the sender enqueues late, so the sender's kernels must
    # wait at the device barrier (one generation per rank per transfer)
    if rank != 0:
        time.sleep(0.2)
    for _ in range(8):
        grp.transfer(sb, db, size, cfg, stream=stream)
    stream.synchronize()
    grp.sync()  # raises if any wait timed out
    if rank == 1:
        assert np.array_equal(dst.cpu().numpy(), data)
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,gpu_paths,host", [(2, 1, False), (2, 1, True), (3, 2, False), (4, 3, True)])
@pytest.mark.parametrize("graph", [False, True])
def test_group_back_to_back_transfers(world, gpu_paths, host, graph):
    """Transfers enqueued back to back with no host sync, the receiver (and
    relay) late: the device barrier alone orders them.  Regression: the
    receiver's and idle ranks' one-warp barrier kernels once bumped their
    generation once per THREAD, so the sender ran ahead, its bytes landed
    before the previous wait re-armed the counter, and the next wait timed
    out."""
    _dist_util.run(_b2b_worker, world, gpu_paths, host, graph)


def _evict_worker(rank, world, port, graph):
    import numpy as np
    import torch.distributed as dist

    import paper_2604_22228_b200 as mp
    from oracle import transfer as ot
    from paper_2604_22228_b200.group import TransferGroup
    _dist_util.init(rank, world, port)
    torch.cuda.set_device(0)
    topo = mp.load_topology(mp.mesh_text("g", world, 7.5e11, 1, 2e-6, 5.5e10, 1e-5, "full"))
    grp = TransferGroup(topo, device=0, stage_bytes=64 << 20)
    sizes = [(3 << 20) + 5, (5 << 20) + 9]
    pairs = []
    for i, n in enumerate(sizes):
        s = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        if rank == 0:
            s.copy_(torch.from_numpy(ot.pattern(n, seed=60 + i)))
        pairs.append((grp.expose(s, owner=0), grp.expose(d, owner=1), d, n))
    torch.cuda.synchronize()
    dist.barrier()
    cfg = mp.PathConfig(num_gpu_paths=world - 1, host_path_enabled=True, max_chunks=3, graph_mode=graph,
                        cache_capacity=1)
    stream = torch.cuda.Stream(device=0)
    for _ in range(3):  # alternating pairs with capacity 1: every transfer evicts the other entry
        for sb, db, _, n in pairs:
            grp.transfer(sb, db, n, cfg, stream=stream)
    stream.synchronize()
    grp.sync()
    if rank == 1:
        for i, (_, _, d, n) in enumerate(pairs):
            assert np.array_equal(d.cpu().numpy(), ot.pattern(n, seed=60 + i))
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("graph", [False, True])
def test_group_back_to_back_with_cache_eviction(world, graph):
    """cache_capacity 1 and two alternating buffer pairs, back to back with
    no host sync: every transfer evicts (and syncs on) the other entry while
    the peers' kernels are in flight — byte-exact, no timeout."""
    _dist_util.run(_evict_worker, world, graph)


def _fuzz_worker(rank, world, port, ops, seed):
    import random

    import numpy as np
    import torch.distributed as dist

    import paper_2604_22228_b200 as mp
    from oracle import transfer as ot
    from paper_2604_22228_b200.group import TransferGroup
    _dist_util.init(rank, world, port)
    torch.cuda.set_device(0)
    topo = mp.load_topology(mp.mesh_text("gf", world, 7.5e11, 1, 2e-6, 3e10, 1e-5, "full"))
    grp = TransferGroup(topo, device=0, stage_bytes=96 << 20, host_bytes=96 << 20)
    size = (6 << 20) + 77
    mine = torch.from_numpy(ot.pattern(size, seed=900 + rank)).to("cuda:0")  # this rank's source
    inbox = torch.zeros(size, dtype=torch.uint8, device="cuda:0")           # this rank's destination
    srcs, dsts = [], []
    for q in range(world):  # collective: every rank's source and destination, in rank order
        srcs.append(grp.expose(mine, owner=q))
        dsts.append(grp.expose(inbox, owner=q))
    rng = random.Random(seed)  # the same sequence on every rank
    stream = torch.cuda.Stream(device=0)
    last_from = None  # who last wrote this rank's inbox (since the last check)
    for step in range(ops):
        a, b = rng.sample(range(world), 2)
        n = rng.choice([1, 4097, (1 << 20) + 5, size])
        cfg = mp.PathConfig(num_gpu_paths=rng.randint(1, world - 1), host_path_enabled=rng.random() < 0.5,
                            max_chunks=rng.randint(1, 6), graph_mode=rng.random() < 0.7)
        grp.transfer(srcs[a], dsts[b], n, cfg, stream=stream)
        if rank == b:
            last_from = (a, n)  # the last write into this inbox decides its first n bytes
        if rng.random() < 0.15 or step == ops - 1:  # a check point (same decision on every rank)
            stream.synchronize()
            grp.sync()
            dist.barrier()
            if last_from is not None:
                a_, n_ = last_from
                got = inbox[:n_].cpu().numpy()
                assert np.array_equal(got, ot.pattern(size, seed=900 + a_)[:n_]), (rank, step, last_from)
            inbox.zero_()
            torch.cuda.synchronize()
            last_from = None
            dist.barrier()
    grp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_group_random_transfer_sequences(world):
    """Random back-to-back group transfers between random rank pairs (random
    path counts, host path, chunking, graph / streamed), every rank taking
    its part (sender, relay, receiver or idle) — receivers' inboxes checked
    at random shared check points."""
    _dist_util.run(_fuzz_worker, world, int(os.environ.get("MP_GROUP_FUZZ_OPS", "40")),
                   int(os.environ.get("MP_GROUP_FUZZ_SEED", "7")))
