"""Random parity against the LIVE reference (not only the committed goldens
or the oracle): the unmodified `mpsim` package is imported from the
reference install (baseline/_ref) or the reference tree and fed the same
random topologies / configs / sizes as the product.  Shares (as float.hex),
path kinds and hop channels, chunk plans, lane schedules, graph dumps,
graph-key digests and error messages must be identical.  Skipped where no
reference is importable (e.g. on the GPU box)."""

import os
import random
import sys

import pytest

import paper_2604_22228_b200 as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def _reference():
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "mpsim")):
            sys.path.insert(0, path)
            try:
                from mpsim import graph, paths, pipeline, topology  # noqa: F401
                return paths, pipeline, graph, topology
            except Exception:  # noqa: BLE001 - try the next location
                pass
            finally:
                sys.path.remove(path)
    return None


REF = _reference()
pytestmark = pytest.mark.skipif(REF is None, reason="the reference package is not importable here")


def _topo_text(rng, n):
    lines = [f"name fuzz{n}", "[device]"] + [f"{i} accelerator" for i in range(n)] + ["[link]"]
    for a in range(n):
        for b in range(a + 1, n):
            bw = rng.choice([rng.uniform(1e9, 9e11), float(rng.randint(1, 900)) * 1e9, 7.5e11])
            lines.append(f"{a} {b} {bw!r} {rng.choice([1e-6, 2e-6, 5e-6])!r} "
                         f"{rng.choice(['full', 'half'])} {rng.randint(1, 4)}")
    lines.append("[hostlink]")
    for d in range(n):
        lines.append(f"{d} {rng.uniform(1e9, 6e10)!r} 1e-05 {rng.choice(['full', 'half'])}")
    return "\n".join(lines) + "\n"


def _run(api, text, case):
    paths_m, pipeline_m, graph_m, topology_m = api
    n, src, dst, g, host, k, size, policy = case
    try:
        topo = topology_m.load_topology(text)
        cfg = paths_m.PathConfig(num_gpu_paths=g, host_path_enabled=host, max_chunks=k,
                                 share_policy=policy)
        ps = paths_m.plan_paths(topo, topo.device(src), topo.device(dst), cfg)
        plan = pipeline_m.make_chunk_plan(ps, size, k)
        sched = pipeline_m.lane_schedule(plan)
        eg = graph_m.build_graph(plan)
        key = graph_m.graph_key(11, 22, size, cfg, ps)
    except ValueError as exc:
        return ("error", type(exc).__name__, str(exc))
    return ([p.share.hex() for p in ps.paths], [p.kind for p in ps.paths],
            [[h.channel.id for h in p.hops] for p in ps.paths],
            [(c.path_index, c.offset, c.length, c.seq) for c in plan.chunks],
            [(l.lane_id, l.path_index, l.hop, tuple(l.chunk_ids)) for l in sched.lanes],
            eg.dump(), key.config_digest)


def test_random_plans_equal_the_live_reference():
    rng = random.Random(20261017)
    product = (mp.paths, mp.pipeline, mp.graph, mp.topology)
    checked = errors = 0
    for trial in range(120):
        n = rng.randint(2, 8)
        text = _topo_text(rng, n)
        for _ in range(12):
            src, dst = rng.sample(range(n), 2) if rng.random() < 0.95 else (0, 0)
            case = (n, src, dst, rng.randint(1, 8), rng.random() < 0.6, rng.randint(1, 40),
                    rng.choice([1, 7, 4096, rng.randint(1, 1 << 20), rng.randint(1, 1 << 34)]),
                    rng.choice(["bandwidth_proportional", "equal"]))
            want, got = _run(REF, text, case), _run(product, text, case)
            if want and want[0] == "error":
                errors += 1
                assert got[0] == "error" and got[2] == want[2], (case, want, got)
            else:
                assert got == want, case
            checked += 1
    assert checked == 1440 and 0 < errors < checked
