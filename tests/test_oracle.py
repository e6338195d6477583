"""Pin the oracle (oracle/planner.py, oracle/transfer.py) against golden
vectors produced by the reference package itself (tests/golden/gen_golden.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


PLANNER = load("planner")
OK_CASES = [c for c in PLANNER["cases"] if "error" not in c]


def oracle_plan(case):
    topo = op.parse_topology(PLANNER["topologies"][case["topology"]])
    cfg = case["config"]
    paths = op.plan_paths(topo, case["src"], case["dst"], cfg.get("num_gpu_paths", 1),
                          cfg.get("host_path_enabled", False),
                          cfg.get("share_policy", "bandwidth_proportional"))
    chunks = op.make_chunk_plan([p["share"] for p in paths], case["size"], case["max_chunks"])
    return topo, paths, chunks


def test_golden_inventory():
    assert len(OK_CASES) >= 400
    assert PLANNER["python"].startswith("3.")


@pytest.mark.parametrize("case", OK_CASES, ids=lambda c: f"t{c['topology']}-{c['size']}")
def test_oracle_matches_reference(case):
    _, paths, chunks = oracle_plan(case)
    assert [p["share"].hex() for p in paths] == [p["share_hex"] for p in case["paths"]]
    assert [[h for h, _ in p["hops"]] for p in paths] == [p["hops"] for p in case["paths"]]
    assert [list(c) for c in chunks] == case["chunks"]
    dump = op.graph_dump(paths, chunks, case["src"], case["dst"])
    assert hashlib.sha256(dump.encode()).hexdigest() == case["dump_sha256"]
    lanes, deps = op.lane_schedule([len(p["hops"]) for p in paths], chunks)
    flat = [[lid, p, h, m] for lid, p, h, m in lanes]
    flat_deps = [[a[0], a[1], b[0], b[1]] for a, b in deps]
    assert hashlib.sha256(json.dumps([flat, flat_deps]).encode()).hexdigest() == \
        case["lanes_sha256"]
    cfg = case["config"]
    got = op.digest(cfg.get("num_gpu_paths", 1), cfg.get("host_path_enabled", False),
                    cfg.get("max_chunks", 1), cfg.get("graph_mode", False),
                    cfg.get("share_policy", "bandwidth_proportional"), case["src"], case["dst"],
                    paths)
    assert got == case["digest"]


def test_oracle_lru_matches_reference():
    for case in load("lru")["cases"]:
        lru = op.LRU(case["capacity"])
        assert [lru.access(k) for k in case["accesses"]] == case["hits"]
        assert lru.order == case["final_order"]


@pytest.mark.parametrize("case", OK_CASES[:60], ids=lambda c: f"t{c['topology']}-{c['size']}")
def test_oracle_transfer_delivers_every_byte(case):
    if case["size"] > (64 << 20):
        pytest.skip("large")
    _, paths, chunks = oracle_plan(case)
    src = ot.pattern(case["size"], seed=case["size"])
    dst = np.bitwise_not(src)
    ot.run(src, dst, [p["kind"] for p in paths], chunks, threads=2)
    assert np.array_equal(src, dst)


def test_py312_sum_matches_builtin():
    import random
    rng = random.Random(5)
    for _ in range(20000):
        xs = [rng.uniform(1e9, 9e11) * rng.choice([1, 1e-3, 1e3]) for _ in range(rng.randint(1, 9))]
        assert op.py312_sum(xs) == sum(xs)
