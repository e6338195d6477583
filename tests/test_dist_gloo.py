"""Multi-process host logic on CPU (gloo, world_size 2 and 3): the IPC-handle
rendezvous helpers of group.py and the plan/role agreement every rank relies
on (each rank computes the same plan independently; nothing but handles is
exchanged)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import _dist_util  # noqa: E402


def _worker_exchange(rank, world, port):
    import torch.distributed as dist

    from paper_2604_22228_b200 import group
    _dist_util.init(rank, world, port)
    blobs = group.exchange_blobs(bytes([rank]) * 256)
    assert [b[0] for b in blobs] == list(range(world))
    assert all(len(b) == 256 for b in blobs)
    payload = (b"h" * 64, 4096 + rank, 1 << 20, 3) if rank == 1 else None
    got = group.share_buffer(1, payload)
    assert got == (b"h" * 64, 4097, 1 << 20, 3)
    dist.barrier()
    dist.destroy_process_group()


def _worker_plans(rank, world, port):
    import hashlib

    import torch.distributed as dist

    import paper_2604_22228_b200 as mp
    from paper_2604_22228_b200 import group
    _dist_util.init(rank, world, port)
    topo = mp.load_topology(mp.mesh_text("g", world, 7.5e11, 1, 2e-6, 5.5e10, 1e-5, "full"))
    cfg = mp.PathConfig(num_gpu_paths=world - 1, max_chunks=8)
    r = group.roles(topo, 0, 1, cfg)
    ps = mp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    plan = mp.make_chunk_plan(ps, (64 << 20) + 5, 8)
    digest = hashlib.sha256(repr([(c.path_index, c.offset, c.length, c.seq)
                                  for c in plan.chunks]).encode()).hexdigest()
    out = [None] * world
    dist.all_gather_object(out, (sorted(r.items()), digest,
                                 mp.graph_key(0, 0, plan.total_size, cfg, ps).config_digest))
    assert all(o == out[0] for o in out)
    assert r[0] == "sender" and r[1] == "receiver"
    assert all(r[q] == "relay" for q in range(2, world))
    dist.destroy_process_group()


def test_rendezvous_helpers_world2():
    _dist_util.run(_worker_exchange, 2)


def test_every_rank_derives_the_same_plan_world3():
    _dist_util.run(_worker_plans, 3)


def test_host_path_roles_in_group_mode():
    """The host-staged path adds no rank role: the sender writes the
    destination's host inbox, the destination loads it back."""
    import paper_2604_22228_b200 as mp
    from paper_2604_22228_b200 import group
    topo = mp.load_topology(mp.mesh_text("g", 3, 7.5e11, 1, 2e-6, 5.5e10, 1e-5, "full"))
    assert group.roles(topo, 0, 1, mp.PathConfig(host_path_enabled=True)) == \
        {0: "sender", 1: "receiver", 2: "idle"}
    assert group.roles(topo, 0, 1, mp.PathConfig(2, host_path_enabled=True)) == \
        {0: "sender", 1: "receiver", 2: "relay"}
