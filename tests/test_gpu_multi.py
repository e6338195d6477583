"""Real multi-GPU transfers (skipped unless >= 2 CUDA devices are visible):
GPU0 -> GPU1 over NVLink peer memory — direct, through GPU relays when a
third/fourth GPU exists, plus the host-staged path — byte-exact against the
oracle, with the plan equal to the oracle's.  Also the TMA bulk-copy kernel
on peer addresses (`tma_peer`), which the 1-GPU pool cannot verify.
On one GPU every one of these paths runs in loopback in test_gpu_transfer.py."""

import os
import sys

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs (NVLink peers)")


def _engine(n, **opts):
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    text = mesh_text("node", n, 7.7e11, 1, 2e-6, 5.5e10, 1e-5, "full")
    eng = Engine(load_topology(text), list(range(n)))
    if opts:
        eng.configure(**opts)
    return eng, text


def _check(eng, text, size, gpu_paths, host, chunks, graph, reps=2, off=0):
    from paper_2604_22228_b200 import PathConfig
    cfg = PathConfig(num_gpu_paths=gpu_paths, host_path_enabled=host, max_chunks=chunks,
                     graph_mode=graph)
    src = torch.empty(size + off, dtype=torch.uint8, device="cuda:0")[off:]
    dst = torch.empty(size + off, dtype=torch.uint8, device="cuda:1")[off:]
    t = op.parse_topology(text)
    opaths = op.plan_paths(t, 0, 1, gpu_paths, host)
    ochunks = op.make_chunk_plan([p["share"] for p in opaths], size, chunks)
    for r in range(reps):
        data = ot.pattern(size, seed=50 + r)
        src.copy_(torch.from_numpy(data))
        dst.copy_(torch.bitwise_not(torch.from_numpy(data)).to("cuda:1"))
        eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
        eng.recv(dst)
        eng.sync()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        expect = np.empty_like(data)
        ot.run(data, expect, [p["kind"] for p in opaths], ochunks, threads=4)
        assert np.array_equal(dst.cpu().numpy(), expect)
    _, done = eng.last_plan()
    assert [(c.path_index, c.offset, c.length, c.seq) for c in done] == ochunks


@needs2
@pytest.mark.parametrize("size", [4096 + 3, 3 * MiB + 5, 40 * MiB + 7, 160 * MiB + 1])
@pytest.mark.parametrize("graph", [False, True])
def test_nvlink_direct_and_host(size, graph):
    eng, text = _engine(2)
    _check(eng, text, size, 1, True, 8, graph, off=3)
    eng.close()


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs (direct + 2 relays)")
@pytest.mark.parametrize("graph", [False, True])
def test_nvlink_relays(graph):
    eng, text = _engine(4)
    _check(eng, text, 64 * MiB + 11, 3, True, 8, graph)
    eng.close()


@needs2
@pytest.mark.parametrize("size", [3 * MiB + 5, 40 * MiB + 7, 160 * MiB + 1])
def test_tma_on_peer_addresses(size):
    """tma_peer=1: the TMA bulk-copy kernels also run on tables that touch
    another GPU's memory (static TMA tables for mid sizes)."""
    eng, text = _engine(max(2, min(_ngpu(), 3)), tma_peer=True, copy="tma", ctas_per_sm=1,
                        threads=128)
    _check(eng, text, size, min(_ngpu(), 3) - 1 if _ngpu() >= 3 else 1, False, 4, True)
    eng.close()


@needs2
@pytest.mark.parametrize("host", ["sm", "ce", "auto"])
@pytest.mark.parametrize("host_bw", [1e9, 5.5e10])
def test_config1_on_real_peers(host, host_bw):
    """BASELINE config 1 on two GPUs: direct + host at 64 MiB, host hops by
    the SM kernels (hop1 helpers on GPU0, hop2 flag waits on GPU1), by copy
    engines, or the per-share automatic choice; tiny and bandwidth-sized
    host shares."""
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    text = mesh_text("node", 2, 7.7e11, 1, 2e-6, host_bw, 1e-5, "full")
    eng = Engine(load_topology(text), [0, 1])
    eng.configure(host=host)
    for k in (1, 8):
        _check(eng, text, 64 * MiB + 13, 1, True, k, True)
    eng.close()


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs (BASELINE config 3)")
def test_config3_four_gpus_two_relays_and_host():
    """BASELINE config 3: direct + relay GPU2 + relay GPU3 + host, 512 MiB."""
    eng, text = _engine(4)
    _check(eng, text, 512 * MiB, 3, True, 8, True, reps=1)
    eng.close()


@pytest.mark.skipif(_ngpu() < 8, reason="needs 8 GPUs (BASELINE config 4)")
@pytest.mark.parametrize("gpu_paths", [1, 2, 4, 7])
def test_config4_eight_gpus_relay_sweep(gpu_paths):
    """BASELINE config 4: direct + host + 0..6 relays through GPU2..GPU7, 512 MiB."""
    eng, text = _engine(8)
    _check(eng, text, 512 * MiB + 1, gpu_paths, True, 16, True, reps=1)
    eng.close()


@needs2
def test_ingress_probe_all_peers_to_one_gpu():
    """The roofline's B_ingress probe (bench.py N > 1): every other GPU
    writes GPU1 at once as ONE program; the bytes land exactly."""
    from paper_2604_22228_b200 import PathConfig
    n = min(_ngpu(), 8)
    eng, _ = _engine(n)
    size = 32 * MiB + 3
    peers = [d for d in range(n) if d != 1]
    bufs = []
    for d in peers:
        s = torch.randint(0, 256, (size,), dtype=torch.uint8, device=f"cuda:{d}")
        bufs.append((s, torch.zeros(size, dtype=torch.uint8, device="cuda:1"), d))
    eng.send_many([(s, t, None, d, 1) for s, t, d in bufs], PathConfig(1, False, 1, True))
    eng.sync()
    for s, t, _ in bufs:
        assert torch.equal(s.cpu(), t.cpu())
    eng.close()


@needs2
def test_egress_probe_one_gpu_to_all_peers():
    """The roofline's B_egress probe (bench.py N > 1): GPU0 writes every
    other GPU at once as ONE program; the bytes land exactly."""
    from paper_2604_22228_b200 import PathConfig
    n = min(_ngpu(), 8)
    eng, _ = _engine(n)
    size = 32 * MiB + 5
    bufs = []
    for d in range(1, n):
        s = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
        bufs.append((s, torch.zeros(size, dtype=torch.uint8, device=f"cuda:{d}"), d))
    eng.send_many([(s, t, None, 0, d) for s, t, d in bufs], PathConfig(1, False, 1, True))
    eng.sync()
    for s, t, _ in bufs:
        assert torch.equal(s.cpu(), t.cpu())
    eng.close()


@needs2
def test_nccl_single_process_baseline():
    """The bench's baseline-only ncclCommInitAll + ncclSend/Recv GPU0 -> GPU1
    (one process) delivers the bytes and reports a rate."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    assert bench.nccl_single_process_p2p(torch, 64 * MiB + 3, reps=5) > 0
