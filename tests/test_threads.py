"""Threading contract: planning is pure and reentrant — the
C ABI releases the GIL (ctypes) and keeps its error text thread-local — and
one Engine serves sends from several threads on their own streams (the C
context is mutex-guarded; a send issued after another stream's send waits
for it on the device).  CPU: concurrent plans equal serial ones, errors do
not leak between threads.  GPU: concurrent sends are byte-exact."""

import random
import threading

import numpy as np
import pytest

from oracle import transfer as ot

MiB = 1 << 20


def _topo(n=8):
    from paper_2604_22228_b200 import load_topology, mesh_text
    return load_topology(mesh_text("thr", n, 7.5e11, 1, 2e-6, 5.5e10, 1e-5, "full"))


def _plan(topo, g, host, size, k, policy):
    from paper_2604_22228_b200 import PathConfig, make_chunk_plan, plan_paths
    cfg = PathConfig(num_gpu_paths=g, host_path_enabled=host, max_chunks=k, share_policy=policy)
    ps = plan_paths(topo, topo.device(0), topo.device(1), cfg)
    plan = make_chunk_plan(ps, size, k)
    return [p.share.hex() for p in ps.paths], [(c.path_index, c.offset, c.length, c.seq) for c in plan.chunks]


def test_concurrent_planning_equals_serial():
    topo = _topo()
    rng = random.Random(20261017)
    cases = [(rng.randint(1, 7), rng.random() < 0.5, rng.randint(1, 2**31), rng.randint(1, 32),
              rng.choice(["bandwidth_proportional", "equal"])) for _ in range(400)]
    serial = [_plan(topo, *c) for c in cases]
    out = [None] * len(cases)
    errors = []

    def worker(t):
        try:
            for i in range(t, len(cases), 8):
                out[i] = _plan(topo, *cases[i])
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append(exc)
    threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    assert out == serial


def test_error_text_is_per_thread():
    """One thread's failing call never changes the message another thread
    raises (mp_last_error is thread-local)."""
    from paper_2604_22228_b200 import ChunkError, PlanError, PathConfig, make_chunk_plan, plan_paths
    topo = _topo()
    seen = {"plan": set(), "chunk": set()}
    ps = plan_paths(topo, topo.device(0), topo.device(1), PathConfig())
    barrier = threading.Barrier(2)

    def bad_plan():
        barrier.wait()
        for _ in range(300):
            try:
                plan_paths(topo, topo.device(0), topo.device(0), PathConfig())
            except PlanError as exc:
                seen["plan"].add(str(exc))

    def bad_chunks():
        barrier.wait()
        for _ in range(300):
            try:
                make_chunk_plan(ps, 0, 4)
            except ChunkError as exc:
                seen["chunk"].add(str(exc))
    threads = [threading.Thread(target=bad_plan), threading.Thread(target=bad_chunks)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert len(seen["plan"]) == 1 and "same device" in next(iter(seen["plan"]))
    assert len(seen["chunk"]) == 1 and "size" in next(iter(seen["chunk"]))


@pytest.mark.gpu
def test_concurrent_sends_from_threads_are_byte_exact():
    torch = pytest.importorskip("torch")
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
    eng = Engine(load_topology(mesh_text("thr", 4, 2e12, 1, 2e-6, 40e9, 1e-5, "full")), [0] * 4)
    cfgs = [PathConfig(1, False, 1, True), PathConfig(1, True, 4, True), PathConfig(3, True, 8, True),
            PathConfig(2, True, 3, False)]
    sizes = [MiB + 5, 3 * MiB + 77, 17 * MiB + 1, 64 * 1024 + 3]
    jobs = []
    for t in range(4):
        n = sizes[t]
        data = ot.pattern(n, seed=100 + t)
        src = torch.from_numpy(data).to("cuda:0")
        dst = torch.bitwise_not(src)
        jobs.append((src, dst, n, cfgs[t], torch.cuda.Stream(device=0), data))
    errors = []

    def worker(src, dst, n, cfg, stream, data):
        try:
            for _ in range(30):
                eng.send(src, dst, n, cfg, stream=stream, src_dev=0, dst_dev=1)
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append(exc)
    threads = [threading.Thread(target=worker, args=j) for j in jobs]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    torch.cuda.synchronize()
    eng.sync()
    assert not errors, errors
    for src, dst, n, cfg, stream, data in jobs:
        assert np.array_equal(dst.cpu().numpy(), data), f"{n} B with {cfg} differs"
    eng.close()
