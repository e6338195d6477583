"""Generate golden vectors by running the REFERENCE package itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Only runnable where /root/reference exists (the build container).  Output:
tests/golden/planner.json, lru.json, topology_errors.json — committed, and
consumed by tests/test_oracle.py (oracle pinning) and
tests/test_planner_parity.py (C++ planner parity), which run anywhere.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from mpsim import graph as rg  # noqa: E402
from mpsim import paths as rp  # noqa: E402
from mpsim import pipeline as rpl  # noqa: E402
from mpsim import topology as rt  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

IDEAL = """name ideal
[device]
0 accelerator
1 accelerator
2 accelerator
3 accelerator
[link]
0 1 1e9 0 full 1
0 2 1e9 0 full 1
0 3 1e9 0 full 1
1 2 1e9 0 full 1
1 3 1e9 0 full 1
2 3 1e9 0 full 1
[hostlink]
0 0.5e9 0 half
1 0.5e9 0 half
2 0.5e9 0 half
3 0.5e9 0 half
"""


def random_topo(rng: random.Random, n: int, name: str) -> str:
    """Measured-looking bandwidths (non-round floats, repr-exact), mixed duplex."""
    lines = [f"name {name}", "[device]"] + [f"{i} accelerator" for i in range(n)] + ["[link]"]
    for a in range(n):
        for b in range(a + 1, n):
            bw = rng.uniform(6.0e11, 8.0e11)
            lines.append(f"{a} {b} {bw!r} {rng.uniform(1e-6, 3e-6)!r} "
                         f"{rng.choice(['full', 'full', 'half'])} {rng.choice([1, 1, 2])}")
    lines.append("[hostlink]")
    for d in range(n):
        lines.append(f"{d} {rng.uniform(4.0e10, 6.0e10)!r} {rng.uniform(5e-6, 2e-5)!r} "
                     f"{rng.choice(['full', 'half'])}")
    return "\n".join(lines) + "\n"


def preset_text(name: str) -> str:
    from importlib import resources
    return resources.files("mpsim.presets").joinpath(f"{name}.topo").read_text()


def run_case(topos, ti, src, dst, cfg_kw, size, mc):
    topo = rt.load_topology(topos[ti])
    case = {"topology": ti, "src": src, "dst": dst, "config": cfg_kw, "size": size,
            "max_chunks": mc}
    try:
        cfg = rp.PathConfig(**cfg_kw)
        ps = rp.plan_paths(topo, topo.device(src), topo.device(dst), cfg)
        plan = rpl.make_chunk_plan(ps, size, mc)
    except Exception as exc:  # noqa: BLE001
        case["error"] = {"type": type(exc).__name__, "message": str(exc)}
        return case
    case["paths"] = [{"kind": p.kind, "stage": None if p.stage is None else p.stage.label,
                      "share_hex": p.share.hex(), "share_repr": repr(p.share),
                      "hops": [h.channel.id for h in p.hops]} for p in ps.paths]
    case["chunks"] = [[c.path_index, c.offset, c.length, c.seq] for c in plan.chunks]
    sched = rpl.lane_schedule(plan)
    lanes = [[l.lane_id, l.path_index, l.hop, list(l.chunk_ids)] for l in sched.lanes]
    deps = [[a[0], a[1], b[0], b[1]] for a, b in sched.dependencies]
    g = rg.build_graph(plan)
    dump = g.dump()
    if len(plan.chunks) <= 40:
        case["lanes"], case["deps"], case["dump"] = lanes, deps, dump
    # digests of the full structures let big plans stay small on disk
    case["lanes_sha256"] = hashlib.sha256(json.dumps([lanes, deps]).encode()).hexdigest()
    case["dump_sha256"] = hashlib.sha256(dump.encode()).hexdigest()
    case["lane_count"] = g.lane_count
    case["digest"] = rg.graph_key(1, 2, size, cfg, ps).config_digest
    return case


def planner_cases():
    rng = random.Random(20261017)
    topos = [IDEAL, preset_text("beluga"), preset_text("narval")]
    topos += [random_topo(rng, 8, f"rand8_{i}") for i in range(6)]
    topos += [random_topo(rng, 4, f"rand4_{i}") for i in range(3)]
    cases = []
    # the survey's worked configs (§8a): C1, C3, C4 shapes and the 12 MiB golden
    fixed = [
        (1, 0, 1, dict(num_gpu_paths=1, host_path_enabled=True, max_chunks=8), 64 << 20, 8),
        (0, 0, 1, dict(num_gpu_paths=3, share_policy="equal"), 12 << 20, 4),
        (0, 0, 1, dict(num_gpu_paths=1), 1, 4),
        (0, 0, 1, dict(num_gpu_paths=3, share_policy="equal"), (10 << 20) + 12345, 8),
        (3, 0, 1, dict(num_gpu_paths=3, host_path_enabled=True, max_chunks=8), 512 << 20, 8),
        (3, 0, 1, dict(num_gpu_paths=7, host_path_enabled=True, max_chunks=16), 512 << 20, 16),
        (4, 2, 5, dict(num_gpu_paths=7, host_path_enabled=True), (1 << 30), 32),
        (3, 0, 1, dict(num_gpu_paths=7, share_policy="equal"), 30, 1),  # empty path
        (1, 1, 1, dict(), 64, 1),  # same device
        (1, 0, 1, dict(num_gpu_paths=4), 64, 1),  # insufficient staging
        (0, 0, 1, dict(), 0, 1),  # size error
        (0, 0, 1, dict(), 64, 0),  # max_chunks error
    ]
    for ti, s, d, kw, size, mc in fixed:
        cases.append(run_case(topos, ti, s, d, kw, size, mc))
    for _ in range(400):
        ti = rng.randrange(len(topos))
        n = 4 if ti < 3 or ti >= 9 else 8
        s, d = rng.sample(range(n), 2)
        kw = dict(num_gpu_paths=rng.randint(1, n - 1), host_path_enabled=rng.random() < 0.6,
                  share_policy=rng.choice(["equal", "bandwidth_proportional",
                                           "bandwidth_proportional"]),
                  graph_mode=rng.random() < 0.5)
        mc = rng.choice([1, 2, 3, 4, 5, 7, 8, 16, 32])
        kw["max_chunks"] = mc
        size = rng.choice([rng.randint(1, 4096), rng.randint(1, 1 << 20),
                           rng.randint(1, 1 << 30), 1 << rng.randint(10, 29)])
        cases.append(run_case(topos, ti, s, d, kw, size, mc))
    return topos, cases


def lru_cases():
    rng = random.Random(11)
    out = []
    topo = rt.load_topology(IDEAL)
    cfg = rp.PathConfig()
    ps = rp.plan_paths(topo, topo.device(0), topo.device(1), cfg)
    plan = rpl.make_chunk_plan(ps, 64, 1)
    for capacity in (1, 2, 3, 5, 16):
        cache = rg.GraphCache(capacity)
        seq = [rng.randrange(8) for _ in range(300)]
        hits = []
        for k in seq:
            _, hit = cache.get_or_build(rg.graph_key(k, k + 1000, 64, cfg, ps), plan)
            hits.append(hit)
        out.append({"capacity": capacity, "accesses": seq, "hits": hits,
                    "final_order": [key.src_buffer_id for key in cache.keys()]})
    return out


BAD_TOPOS = [
    "[device]\n0 accelerator\n1 gpu\n",
    "[devices]\n0 accelerator\n",
    "oops\n[device]\n0 accelerator\n",
    "[device]\n0 accelerator\n2 accelerator\n",
    "",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 1e9 0 full\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 x 1e9 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 fast 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 5 1e9 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 -1e9 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 1e9 -1 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 1e9 0 simplex 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 1e9 0 full 0\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 0 1e9 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 1e9 0 full 1\n1 0 1e9 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[hostlink]\n0 1e9 0 half\n0 1e9 0 half\n",
    "[device]\n0 accelerator\n1 accelerator\n[hostlink]\n3 1e9 0 half\n",
    "[device]\n0 accelerator\n1 accelerator\n[hostlink]\n0 1e9 0 half extra\n",
    "name a b\n[device]\n0 accelerator\n",
    "name box # comment\n[device]\n 0 accelerator # x\n1 accelerator\n[LINK]\n0 1 1_000 0 half 3\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 0x10 0 full 1\n",
    "[device]\n0 accelerator\n1 accelerator\n[link]\n0 1 inf 0 full 1\n",
    "[]\n",
    "[device]\r\n0 accelerator\r\n1 accelerator\r\n[link]\r\n0 1 2.5e10 1e-6 full 2\r\n",
]


def topology_cases():
    out = []
    for text in BAD_TOPOS:
        case = {"text": text}
        try:
            t = rt.load_topology(text)
            case["ok"] = {"name": t.name, "n": len(t.accelerators),
                          "channels": [[c.id, c.bandwidth.hex(), c.latency.hex()]
                                       for c in t.channels()]}
        except Exception as exc:  # noqa: BLE001
            case["error"] = {"type": type(exc).__name__, "message": str(exc)}
        out.append(case)
    return out


def main():
    topos, planner = planner_cases()
    for name, data, extra in (("planner", planner, {"topologies": topos}),
                              ("lru", lru_cases(), {}), ("topology", topology_cases(), {})):
        with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
            json.dump({"generator": "tests/golden/gen_golden.py",
                       "reference": "/root/reference/pkg/src/mpsim (mpsim 0.1.0)",
                       "python": sys.version.split()[0], **extra, "cases": data}, fh)
        print(name, len(data))


if __name__ == "__main__":
    main()
