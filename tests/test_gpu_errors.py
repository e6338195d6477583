"""A relay / host flag wait that times out never delivers stale bytes, and
the error is sticky: every later send / recv fails until `Engine.sync()`
reports and clears it (PAPER.md:385-397 assumes no silent corruption).

The timeout is forced with the engine's test-only fault injection: the first
staged chunk's hop1 tiles never signal their flag, so that chunk's hop2
tiles wait out `wait_timeout_ms` and are skipped — the destination keeps its
pre-poisoned bytes there instead of a copy of the staging buffer.
"""

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MiB = 1 << 20


def _setup(kind):
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
    text = mesh_text("loop", 3, 2.0e12, 1, 2e-6, 200e9, 10e-6, "full")
    eng = Engine(load_topology(text), [0, 0, 0])
    opts = {"wait_timeout_ms": 50, "fault_inject": 1}
    if kind == "relay_tma":
        opts["copy"] = "tma"
    if kind == "host_sm":
        opts["host"] = "sm"
        cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=4, graph_mode=True)
        gpu_paths, host = 1, True
    else:
        cfg = PathConfig(num_gpu_paths=2, host_path_enabled=False, max_chunks=4, graph_mode=True)
        gpu_paths, host = 2, False
    eng.configure(**opts)
    t = op.parse_topology(text)
    paths = op.plan_paths(t, 0, 1, gpu_paths, host)
    return eng, cfg, paths


@pytest.mark.parametrize("kind", ["relay_vec", "relay_tma", "host_sm"])
def test_timed_out_wait_is_sticky_and_never_copies_staging(kind):
    from paper_2604_22228_b200 import EngineError
    eng, cfg, paths = _setup(kind)
    size = 4 * MiB + 123
    chunks = op.make_chunk_plan([p["share"] for p in paths], size, 4)
    data = ot.pattern(size, seed=7)
    src = torch.from_numpy(data).to("cuda:0")
    dst = torch.bitwise_not(src)
    eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()  # the kernel ends: the muted chunk's wait timed out
    with pytest.raises(EngineError, match="timed out"):
        eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
    with pytest.raises(EngineError, match="timed out"):
        eng.recv(dst)
    with pytest.raises(EngineError, match="timed out"):  # programs too (mp_send_many)
        eng.send_many([(src, dst, size, 0, 1)], cfg)
    got = dst.cpu().numpy()
    staged = [c for c in chunks if paths[c[0]]["kind"] != "direct"]
    muted = staged[0]
    lo, hi = muted[1], muted[1] + muted[2]
    assert np.array_equal(got[lo:hi], ~data[lo:hi]), "a timed-out chunk received staging bytes"
    for pi, off, ln, _ in chunks:
        seg, want = got[off:off + ln], data[off:off + ln]
        if paths[pi]["kind"] == "direct":
            assert np.array_equal(seg, want)
        else:  # skipped tiles keep the poison; copied ones are exact — nothing else
            assert np.all((seg == want) | (seg == ~want))
    with pytest.raises(EngineError, match="timed out"):
        eng.sync()  # reports and clears
    eng.sync()
    eng.configure(fault_inject=0)
    dst.copy_(torch.bitwise_not(src))
    for _ in range(3):
        eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    assert torch.equal(src, dst)
    eng.close()


def test_wait_options_are_validated():
    from paper_2604_22228_b200 import Engine
    eng = Engine.loopback(2)
    with pytest.raises(ValueError):
        eng.configure(wait_timeout_ms=-1)
    with pytest.raises(ValueError):
        eng.configure(fault_inject=4)
    eng.close()
