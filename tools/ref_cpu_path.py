"""Time the REFERENCE package's per-message CPU path.

Runs the unmodified reference (`mpsim` installed in baseline/_ref) on one
pinned core:
  miss : plan_paths + make_chunk_plan + build_graph + graph_key
  hit  : plan_paths + graph_key + GraphCache.get_or_build (cached)
  sim  : simulate_graph on the cached graph (the reference's "execution")
Prints one JSON object.  Usage: python tools/ref_cpu_path.py <topo file> <size> <chunks>
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})

from mpsim import graph as G  # noqa: E402
from mpsim import paths as P  # noqa: E402
from mpsim import pipeline as PL  # noqa: E402
from mpsim import sim as SIM  # noqa: E402
from mpsim import topology as T  # noqa: E402


def per_call(fn, budget=1.0, min_n=20):
    fn()
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget and n >= min_n:
            return dt / n * 1e6


def main():
    text = open(sys.argv[1]).read()
    size, chunks = int(sys.argv[2]), int(sys.argv[3])
    topo = T.load_topology(text)
    cfg = P.PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=chunks,
                       graph_mode=True)
    s, d = topo.device(0), topo.device(1)

    def miss():
        ps = P.plan_paths(topo, s, d, cfg)
        plan = PL.make_chunk_plan(ps, size, chunks)
        G.build_graph(plan)
        G.graph_key(1, 2, size, cfg, ps)

    cache = G.GraphCache(16)
    ps0 = P.plan_paths(topo, s, d, cfg)
    plan0 = PL.make_chunk_plan(ps0, size, chunks)
    cache.get_or_build(G.graph_key(1, 2, size, cfg, ps0), plan0)

    def hit():
        ps = P.plan_paths(topo, s, d, cfg)
        cache.get_or_build(G.graph_key(1, 2, size, cfg, ps), plan0)

    graph, _ = cache.get_or_build(G.graph_key(1, 2, size, cfg, ps0), plan0)
    model = G.OverheadModel()

    def sim():
        SIM.simulate_graph(topo, graph, model, first_time=False)

    out = {"miss_us": per_call(miss), "hit_us": per_call(hit), "simulate_graph_us": per_call(sim),
           "nodes": graph.node_count, "cores": 1, "python": sys.version.split()[0],
           "reference": "baseline/_ref/mpsim 0.1.0 (unmodified)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
