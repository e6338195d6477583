"""Real GPU timelines: a traced send yields one record
per logical chunk-hop, in the reference's Timeline schema, and the reference's
OWN checker (integrity.check_timeline from the unmodified package installed in
baseline/_ref, when present) finds no ordering violation, full coverage and
completion on hardware data.  Channel exclusivity is reported, not asserted:
on hardware a path's consecutive chunks share its link concurrently
(DESIGN.md §10)."""

import os
import sys

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
MiB = 1 << 20


def _engine(n, **opts):
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    text = mesh_text("loop", n, 2.0e12, 1, 2e-6, 50e9, 10e-6, "full")
    eng = Engine(load_topology(text), [0] * n)
    if opts:
        eng.configure(**opts)
    return eng, text


def _ordering_ok(plan, tl):
    by = {}
    for t in tl.tasks:
        by.setdefault(t.offset, {})[t.role] = t
    for slot in by.values():
        if "stage_hop1" in slot:
            assert slot["stage_hop2"].start_time >= slot["stage_hop1"].end_time


@pytest.mark.parametrize("relay,host,fault", [("sm", "ce", 0), ("ce", "ce", 0), ("sm", "sm", 0), ("sm", "sm", 2)])
def test_trace_is_a_valid_timeline(relay, host, fault):
    """fault = 2: the cross-device lowering (system-scope flags, host chunks
    as hop1 / hop2 tiles) traced between cached sends of the same buffers."""
    from paper_2604_22228_b200 import PathConfig
    eng, text = _engine(4, relay=relay, host=host, fault_inject=fault)
    size = 16 * MiB + 777
    cfg = PathConfig(num_gpu_paths=3, host_path_enabled=True, max_chunks=4, share_policy="equal")
    data = ot.pattern(size, seed=11)
    src = torch.from_numpy(data).to("cuda:0")
    dst = torch.bitwise_not(src)
    if fault:  # cached graph sends around the traced one
        for _ in range(2):
            eng.send(src, dst, size, PathConfig(3, True, 4, True, share_policy="equal"), src_dev=0, dst_dev=1)
        eng.sync()
        dst.copy_(torch.bitwise_not(src))
    plan, tl = eng.trace(src, dst, size, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    assert np.array_equal(dst.cpu().numpy(), data)
    if fault:
        dst.zero_()
        eng.send(src, dst, size, PathConfig(3, True, 4, True, share_policy="equal"), src_dev=0, dst_dev=1)
        eng.sync()
        assert np.array_equal(dst.cpu().numpy(), data)
    # plan == oracle, one task per logical node, sane times
    paths = op.plan_paths(op.parse_topology(text), 0, 1, 3, True, "equal")
    assert [(c.path_index, c.offset, c.length, c.seq) for c in plan.chunks] == \
        op.make_chunk_plan([p["share"] for p in paths], size, 4)
    assert len(tl.tasks) == sum(len(plan.path_set.paths[c.path_index].hops) for c in plan.chunks)
    for t in tl.tasks:
        assert 0.0 <= t.start_time <= t.end_time
    _ordering_ok(plan, tl)
    csv = tl.to_csv().splitlines()
    assert csv[0] == "task_id,path,role,channel,start,end,offset,length"
    assert len(csv) == len(tl.tasks) + 1
    if os.path.isdir(os.path.join(REF, "mpsim")):
        sys.path.insert(0, REF)
        try:
            import mpsim.integrity as ref_integrity  # the unmodified reference checker
            rep = ref_integrity.check_timeline(plan, tl)
            assert rep.coverage_ok and rep.completion_ok
            assert rep.ordering_violations == []
        finally:
            sys.path.remove(REF)
            for m in [m for m in sys.modules if m == "mpsim" or m.startswith("mpsim.")]:
                del sys.modules[m]
    eng.close()
