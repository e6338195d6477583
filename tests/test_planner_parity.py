"""The C++ planner behind the C ABI (the product) reproduces the reference
planner bit-exactly: golden vectors from the reference itself, plus random
fuzz against the oracle restatement."""

import json
import math
import os
import random

import pytest

import paper_2604_22228_b200 as mp
from oracle import planner as op
from paper_2604_22228_b200 import _lib

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


PLANNER = load("planner")
ERRORS = {"PlanError": mp.PlanError, "ChunkError": mp.ChunkError,
          "TopologyError": mp.TopologyError}


def product_plan(case):
    topo = mp.load_topology(PLANNER["topologies"][case["topology"]])
    cfg = mp.PathConfig(**case["config"])
    ps = mp.plan_paths(topo, topo.device(case["src"]), topo.device(case["dst"]), cfg)
    plan = mp.make_chunk_plan(ps, case["size"], case["max_chunks"])
    return topo, cfg, ps, plan


@pytest.mark.parametrize("case", PLANNER["cases"], ids=lambda c: f"t{c['topology']}-{c['size']}")
def test_planner_matches_reference(case):
    if "error" in case:
        with pytest.raises(ERRORS[case["error"]["type"]]) as ei:
            product_plan(case)
        assert str(ei.value) == case["error"]["message"]
        return
    topo, cfg, ps, plan = product_plan(case)
    assert [p.share.hex() for p in ps.paths] == [p["share_hex"] for p in case["paths"]]
    assert [p.kind for p in ps.paths] == [p["kind"] for p in case["paths"]]
    assert [[h.channel.id for h in p.hops] for p in ps.paths] == [p["hops"] for p in case["paths"]]
    assert [[c.path_index, c.offset, c.length, c.seq] for c in plan.chunks] == case["chunks"]
    g = mp.build_graph(plan)
    import hashlib
    assert hashlib.sha256(g.dump().encode()).hexdigest() == case["dump_sha256"]
    if "dump" in case:
        assert g.dump() == case["dump"]
        sched = mp.lane_schedule(plan)
        assert [[l.lane_id, l.path_index, l.hop, list(l.chunk_ids)] for l in sched.lanes] == \
            case["lanes"]
        assert [[a[0], a[1], b[0], b[1]] for a, b in sched.dependencies] == case["deps"]
    assert g.lane_count == case["lane_count"]
    assert mp.graph_key(1, 2, case["size"], cfg, ps).config_digest == case["digest"]


def test_lru_matches_reference():
    topo = mp.load_topology(PLANNER["topologies"][0])
    cfg = mp.PathConfig()
    ps = mp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    plan = mp.make_chunk_plan(ps, 64, 1)
    for case in load("lru")["cases"]:
        cache = mp.GraphCache(case["capacity"])
        hits = [cache.get_or_build(mp.graph_key(k, k + 1000, 64, cfg, ps), plan)[1]
                for k in case["accesses"]]
        assert hits == case["hits"]
        assert [k.src_buffer_id for k in cache.keys()] == case["final_order"]


def test_lru_failed_build_leaves_cache_unchanged():
    """graph.py:173-186: a miss builds before it inserts, so a build that
    raises leaves the cache as it was and the next access is a plain miss."""
    topo = mp.load_topology(PLANNER["topologies"][0])
    cfg = mp.PathConfig()
    ps = mp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    plan = mp.make_chunk_plan(ps, 64, 1)
    key = mp.graph_key(1, 2, 64, cfg, ps)
    other = mp.graph_key(3, 4, 64, cfg, ps)
    cache = mp.GraphCache(2)
    cache.get_or_build(other, plan)
    with pytest.raises(Exception):
        cache.get_or_build(key, None)  # build_graph(None) raises
    assert len(cache) == 1 and key not in cache
    assert [k.src_buffer_id for k in cache.keys()] == [3]
    graph, hit = cache.get_or_build(key, plan)
    assert hit is False and graph.key == key and len(cache) == 2
    assert cache.get_or_build(key, plan) == (graph, True)


@pytest.mark.parametrize("case", load("topology")["cases"], ids=lambda c: repr(c["text"][:20]))
def test_topology_parser_matches_reference(case):
    if "error" in case:
        with pytest.raises(mp.TopologyError) as ei:
            mp.load_topology(case["text"])
        assert str(ei.value) == case["error"]["message"]
    else:
        t = mp.load_topology(case["text"])
        assert t.name == case["ok"]["name"]
        assert len(t.accelerators) == case["ok"]["n"]
        assert [[c.id, c.bandwidth.hex(), c.latency.hex()] for c in t.channels()] == \
            case["ok"]["channels"]


def _fuzz_topo(rng, n):
    from paper_2604_22228_b200 import mesh_text
    lines = [f"name fz", "[device]"] + [f"{i} accelerator" for i in range(n)] + ["[link]"]
    for a in range(n):
        for b in range(a + 1, n):
            lines.append(f"{a} {b} {rng.uniform(1e9, 9e11)!r} 0 full {rng.randint(1, 4)}")
    lines.append("[hostlink]")
    lines += [f"{d} {rng.uniform(1e9, 7e10)!r} 0 {rng.choice(['full', 'half'])}"
              for d in range(n)]
    del mesh_text
    return "\n".join(lines) + "\n"


def test_fuzz_against_oracle():
    """20k random plans with measured-like float weights: C++ == oracle."""
    rng = random.Random(1234)
    n_checked = 0
    for t in range(40):
        n = rng.randint(2, 8)
        text = _fuzz_topo(rng, n)
        topo, otopo = mp.load_topology(text), op.parse_topology(text)
        for _ in range(500):
            s, d = rng.sample(range(n), 2)
            g = rng.randint(1, n - 1)
            host = rng.random() < 0.5
            pol = rng.choice(["equal", "bandwidth_proportional"])
            mc = rng.randint(1, 33)
            size = rng.choice([rng.randint(1, 100), rng.randint(1, 1 << 24),
                               rng.randint(1, 1 << 40)])
            ps = mp.plan_paths(topo, topo.device(s), topo.device(d),
                               mp.PathConfig(num_gpu_paths=g, host_path_enabled=host,
                                             share_policy=pol))
            opaths = op.plan_paths(otopo, s, d, g, host, pol)
            assert [p.share for p in ps.paths] == [p["share"] for p in opaths]
            if size < (1 << 34):
                plan = mp.make_chunk_plan(ps, size, mc)
                assert [(c.path_index, c.offset, c.length, c.seq) for c in plan.chunks] == \
                    op.make_chunk_plan([p["share"] for p in opaths], size, mc)
            n_checked += 1
    assert n_checked == 20000


def test_repr_matches_python():
    rng = random.Random(99)
    vals = [0.0, -0.0, 1.0, 0.1, 1e16, 1e-5, 1e-4, 123456789012345678.0, 5e-324,
            1.7976931348623157e308, float("inf"), -float("inf"), 0.6896551724137931,
            2.0 ** 52, 2.0 ** 53 + 2, 1e22, 1e23, 9.999999999999999e15]
    vals += [rng.uniform(0, 1) for _ in range(20000)]
    vals += [math.ldexp(rng.random(), rng.randint(-1070, 1020)) for _ in range(20000)]
    vals += [float(f"{rng.randint(1, 10**rng.randint(1, 17))}e{rng.randint(-30, 30)}")
             for _ in range(20000)]
    for v in vals:
        assert _lib.format_double(v) == repr(v), v
    assert _lib.format_double(float("nan")) == "nan"


def test_config_validation_messages():
    for kw, msg in [(dict(num_gpu_paths=0), "num_gpu_paths must be >= 1"),
                    (dict(max_chunks=0), "max_chunks must be >= 1"),
                    (dict(cache_capacity=0), "cache_capacity must be >= 1"),
                    (dict(share_policy="fastest"), "unknown share policy 'fastest'")]:
        with pytest.raises(mp.PlanError, match=msg):
            mp.PathConfig(**kw)


def test_from_env():
    cfg = mp.PathConfig.from_env({"MP_NUM_GPU_PATHS": "3", "MP_ENABLE_HOST_PATH": "on",
                                  "MP_MAX_CHUNKS": "8", "MP_ENABLE_GRAPH": "yes",
                                  "MP_GRAPH_CACHE_SIZE": "4", "MP_SHARE_POLICY": "equal"})
    assert cfg == mp.PathConfig(3, True, 8, True, 4, "equal")
    with pytest.raises(mp.PlanError, match="cannot parse flag"):
        mp.PathConfig.from_env({"MP_ENABLE_GRAPH": "maybe"})


def test_contention_free_ring():
    topo = mp.preset("beluga")
    ring = [(topo.device(a), topo.device(b)) for a, b in [(0, 1), (1, 2), (2, 3), (3, 0)]]
    plan = mp.plan_contention_free(topo, ring, mp.PathConfig(num_gpu_paths=2))
    assert plan.contention_free
    assert [ps.paths[1].stage.index for ps in plan.path_sets] == [2, 3, 0, 1]
    three = mp.plan_contention_free(topo, ring, mp.PathConfig(num_gpu_paths=3))
    assert three.shared_channel_count > 0


def test_channel_identity_shared_across_plans():
    topo = mp.preset("narval")
    cfg = mp.PathConfig(num_gpu_paths=3, host_path_enabled=True)
    a = mp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    b = mp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    assert a == b
    assert a.paths[0].hops[0].channel is topo.channel_for(topo.device(0), topo.device(1))
