"""SM-driven PCIe (mapped pinned memory) vs copy engines, TMA and VEC kernels."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_22228_b200 import Engine
eng = Engine.loopback(2)
for opts in ({"copy": "tma"}, {"copy": "vec", "unroll": 8, "ctas_per_sm": 2, "threads": 256},
             {"copy": "vec", "unroll": 16, "ctas_per_sm": 1, "threads": 256},
             {"copy": "vec", "unroll": 4, "ctas_per_sm": 4, "threads": 256}):
    eng.configure(**opts)
    for nb in (8 << 20, 64 << 20):
        m = eng.measure_paths(0, 1, nb, 5)
        print(json.dumps({"opts": opts, "bytes": nb, **{k: round(v, 2) for k, v in m.items()}}), flush=True)
