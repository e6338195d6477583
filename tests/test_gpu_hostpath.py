"""The host-staged path on the SM kernels, byte-exact against the oracle:

* small host chunks (<= 64 KiB) with source and destination on one device
  move as ONE roundtrip tile per chunk (hop1 into pinned host memory, a CTA
  barrier, hop2 back) — on a static TMA table by the kernel's helper warps
  beside the direct stream, on a dynamic table as ordinary tiles;
* larger host chunks are cut into hop1 / hop2 tiles handed off through the
  chunk's flag (GPU-scope release / acquire in loopback);
* traces keep the reference's chunk-level hop2-after-hop1 order.
"""

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

from test_gpu_transfer import _check

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MiB = 1 << 20


def _engine(n, host_bw, **opts):
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    text = mesh_text("loop", n, 3.2e12, 1, 2e-6, host_bw, 10e-6, "full")
    eng = Engine(load_topology(text), [0] * n)
    eng.configure(host="sm", **opts)
    return eng, text


@pytest.mark.parametrize("size", [4 * MiB + 3, 16 * MiB, 64 * MiB + 5, 200 * MiB + 1])
@pytest.mark.parametrize("host_bw", [1e9, 60e9])
@pytest.mark.parametrize("k", [1, 8])
@pytest.mark.parametrize("graph", [False, True])
def test_host_sm_roundtrip_and_flag_modes(size, host_bw, k, graph):
    eng, text = _engine(2, host_bw)
    st = _check(eng, text, size, host=True, chunks=k, graph=graph, seed=size % 97, reps=2)
    host_chunk = max(c[2] for c in op.make_chunk_plan(
        [p["share"] for p in op.plan_paths(op.parse_topology(text), 0, 1, 1, True)], size, k)
        if c[0] == 1)
    if host_chunk <= 64 << 10 and size <= 64 * MiB + 5:
        # roundtrip tiles on the helper warps: the table stays static (TMA ring)
        assert "TMA" in st.kernel, st.kernel
    assert st.kernels == 1 and st.ce_copies == 0
    eng.close()


@pytest.mark.parametrize("copy", ["vec", "tma"])
@pytest.mark.parametrize("offs", [(0, 0), (5, 5), (3, 7), (1, 2)])
def test_host_sm_roundtrip_misaligned(copy, offs):
    eng, text = _engine(2, 1e9, copy=copy, sched="dynamic")
    _check(eng, text, 3 * MiB + 11, host=True, chunks=5, src_off=offs[0], dst_off=offs[1], seed=3)
    eng.close()
    eng, text = _engine(2, 1e9, copy=copy)
    _check(eng, text, 3 * MiB + 11, host=True, chunks=5, src_off=offs[0], dst_off=offs[1], seed=4)
    eng.close()


def test_host_sm_with_relays_small_share():
    """Direct + 2 relays + host with a tiny host share: roundtrip tiles beside
    flag-handed-off relay tiles in one dynamic table."""
    eng, text = _engine(4, 1e9)
    _check(eng, text, 24 * MiB + 17, gpu_paths=3, host=True, chunks=8, graph=True, reps=3, seed=9)
    eng.close()


def test_roundtrip_keeps_hop_order_in_the_trace():
    from paper_2604_22228_b200 import PathConfig
    eng, text = _engine(2, 1e9)
    size = 16 * MiB + 777
    cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=8)
    data = ot.pattern(size, seed=5)
    src = torch.from_numpy(data).to("cuda:0")
    dst = torch.bitwise_not(src)
    plan, tl = eng.trace(src, dst, size, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    assert np.array_equal(dst.cpu().numpy(), data)
    by = {}
    for t in tl.tasks:
        by.setdefault(t.offset, {})[t.role] = t
    staged = [v for v in by.values() if "stage_hop1" in v]
    assert staged
    for v in staged:
        assert 0 <= v["stage_hop1"].start_time <= v["stage_hop1"].end_time
        assert v["stage_hop2"].start_time >= v["stage_hop1"].end_time
        assert v["stage_hop2"].end_time >= v["stage_hop2"].start_time
    eng.close()


@pytest.mark.parametrize("gpu_paths,host_bw,size,k", [(1, 1e9, 4 * MiB + 3, 8), (1, 60e9, 64 * MiB + 5, 8),
                                                      (3, 1e9, 24 * MiB + 17, 8), (4, 60e9, 100 * MiB + 1, 16)])
@pytest.mark.parametrize("graph", [False, True])
def test_cross_device_mechanics_in_loopback(gpu_paths, host_bw, size, k, graph):
    """fault_inject & 2: the lowering treats the logical devices as separate
    GPUs — relay and host flags released / acquired at system scope, host
    chunks as hop1 / hop2 tiles handed off through a flag in the
    destination's memory (never roundtrip tiles) — byte-exact on one GPU."""
    eng, text = _engine(gpu_paths + 1, host_bw, fault_inject=2)
    st = _check(eng, text, size, gpu_paths=gpu_paths, host=True, chunks=k, graph=graph, reps=2, seed=k)
    assert st.ce_copies == 0
    eng.close()
