"""direct + CE host path (max_chunks 8), osu window 64: GB/s per size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402
from paper_2604_22228_b200 import measure as M  # noqa: E402

eng = Engine(load_topology(mesh_text("l", 2, 3.17e12, 1, 2e-6, float(os.environ.get("HOST_BW", 8e9)),
                                     1e-5, "full")), [0, 0])
sizes = [1 << 20, 16 << 20, 64 << 20, 128 << 20, 512 << 20]
res = M.run_bw(M.BenchmarkSpec("omb_bw", sizes, window=64, iterations=3, warmup=2,
                               config=PathConfig(1, True, 8, True)), eng)
print(os.environ.get("TAG", ""), {r.size >> 20: round(r.value / 1e9, 1) for r in res.rows
                                  if r.metric == "bandwidth"}, flush=True)
