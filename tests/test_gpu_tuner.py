"""The measured tuner (replaces the reference's simulated one,
/root/reference/pkg/src/mpsim/tuner.py:48-124): every grid point is timed on
the GPU; the table keeps the reference's CSV schema (it loads with the
reference's own TuningTable.from_csv), its configurations deliver exact
bytes, and the tuned choice is no slower than the best single arm."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MiB = 1 << 20
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _engine(n=2, host_bw=1e9):
    from paper_2604_22228_b200 import Engine, load_topology, mesh_text
    return Engine(load_topology(mesh_text("tune", n, 3.2e12, 1, 2e-6, host_bw, 1e-5, "full")),
                  [0] * n)


def _time(eng, cfg, src, dst, size, reps=30):
    from paper_2604_22228_b200.tuner import measure_makespan
    stream = torch.cuda.Stream()
    return min(measure_makespan(eng, cfg, size, src, dst, stream, reps) for _ in range(3))


def test_tune_table_round_trips_through_the_reference_and_delivers():
    from paper_2604_22228_b200 import PathConfig
    from paper_2604_22228_b200.tuner import GridPoint, TuningTable, tune
    eng = _engine(3)
    sizes = [64 << 10, 4 * MiB, 32 * MiB]
    grid = [GridPoint(g, h, c) for g in (1, 2) for h in (False, True) for c in (1, 4)]
    table = tune(eng, sizes, grid, modes=("graph", "streamed"), reps=10)
    assert len(table.entries) == len(sizes) * 2
    csv = table.to_csv()
    assert csv.splitlines()[0] == "size,mode,gpu_paths,host,max_chunks,makespan"
    again = TuningTable.from_csv(csv, table.topology)
    assert again.entries == table.entries
    if os.path.isdir(os.path.join(REF, "mpsim")):  # the unmodified reference's parser
        sys.path.insert(0, REF)
        try:
            from mpsim.tuner import TuningTable as RefTable
            ref = RefTable.from_csv(csv)
            for e, r in zip(table.entries, ref.entries):
                assert (e.size, e.mode, e.best.gpu_paths, e.best.host, e.best.max_chunks) == \
                    (r.size, r.mode, r.best.gpu_paths, r.best.host, r.best.max_chunks)
                assert r.makespan == e.makespan
        finally:
            sys.path.remove(REF)
            for m in [m for m in sys.modules if m == "mpsim" or m.startswith("mpsim.")]:
                del sys.modules[m]
    # every tuned configuration moves exact bytes
    for size in sizes:
        cfg = table.config_for(size, "graph")
        assert isinstance(cfg, PathConfig)
        src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
        dst = torch.bitwise_not(src)
        eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
        eng.sync()
        assert torch.equal(src, dst)
    eng.close()


def test_tuned_choice_is_no_slower_than_the_best_single_arm():
    from paper_2604_22228_b200 import PathConfig
    from paper_2604_22228_b200.tuner import GridPoint, tune
    eng = _engine(2)
    size = 64 * MiB
    grid = [GridPoint(1, h, c) for h in (False, True) for c in (1, 2, 8)]
    table = tune(eng, [size], grid, modes=("graph",), reps=20)
    src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
    dst = torch.empty_like(src)
    tuned = _time(eng, table.config_for(size), src, dst, size)
    arms = [_time(eng, PathConfig(1, h, c, True), src, dst, size) for h in (False, True)
            for c in (1, 2, 8)]
    assert tuned <= min(arms) * 1.05, (tuned, arms)
    eng.close()


def test_tune_engines_policy_and_calibration():
    from paper_2604_22228_b200 import PathConfig
    from paper_2604_22228_b200.tuner import calibrate_host_bandwidth, tune_engines
    eng = _engine(2)
    sizes = [256 << 10, 8 * MiB, 64 * MiB]
    rules, trials = tune_engines(eng, sizes, reps=10)
    assert rules and rules[-1][0] == 2**63 - 1
    assert all(r[1] in ("sm", "ce") and r[2] in ("sm", "ce") for r in rules)
    assert [r[0] for r in rules] == sorted(r[0] for r in rules)
    assert {t["path"] for t in trials} == {"direct", "host"}
    eng.set_size_policy(rules)
    for s in sizes:  # the policy's choices deliver exact bytes
        src = torch.randint(0, 256, (s,), dtype=torch.uint8, device="cuda:0")
        dst = torch.bitwise_not(src)
        eng.send(src, dst, s, PathConfig(1, True, 4, True), src_dev=0, dst_dev=1)
        eng.sync()
        assert torch.equal(src, dst)
    eng.set_size_policy([])
    cands = [1e9, 4e9, 16e9]
    host_bw, topo, runs = calibrate_host_bandwidth(eng, 3.2e12, 32 * MiB, 8, candidates=cands,
                                                   reps=5)
    assert host_bw in cands and len(runs) == 2 * len(cands)
    assert eng.topology is topo
    # the calibrated topology's plan (written with repr, parsed back identically)
    host_links = [ln for ln in topo.links if ln.a.is_host or ln.b.is_host]
    assert host_links and all(ln.bandwidth == host_bw for ln in host_links)
    eng.close()


def test_tune_rejects_an_infeasible_grid():
    from paper_2604_22228_b200.tuner import GridPoint, tune
    eng = _engine(2)
    with pytest.raises(ValueError, match="feasible"):
        tune(eng, [MiB], [GridPoint(3, False, 1)], modes=("graph",), reps=2)
    eng.close()


def test_probe_topology_plans_and_sends():
    """Engine.probe_topology writes a reference-schema .topo from measured
    rates (the direct link and the host-staged path's delivered rate), which
    the planner parses back and the engine sends with, byte-exact."""
    import paper_2604_22228_b200 as mp
    from paper_2604_22228_b200 import PathConfig
    eng = _engine(2)
    text = eng.probe_topology(64 * MiB, 3, name="probed2")
    link, host = eng.probe_bandwidths(64 * MiB, 3)
    assert link > 1e11 and 1e9 < host < 1e11
    topo = mp.load_topology(text)
    assert topo.name == "probed2" and len(topo.accelerators) == 2
    eng.set_topology(topo)
    n = 24 * MiB + 5
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.bitwise_not(src)
    eng.send(src, dst, n, PathConfig(1, True, 8, True), src_dev=0, dst_dev=1)
    eng.sync()
    assert torch.equal(src, dst)
    eng.close()
