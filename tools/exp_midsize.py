"""GPU experiment: single-path 8-64 MiB messages (L2-resident working sets
in back-to-back osu loops) under kernel variants: default (static TMA
table), LDG/STG kernel (copy=vec), dynamic schedule, TMA ring shapes.
µs per message, medians of 5 interleaved trials."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan, warm_up  # noqa: E402

MiB = 1 << 20
text = open("topologies/b200_loopback.topo").read()
variants = {"default": {}, "vec": {"copy": "vec"}, "dynamic": {"sched": "dynamic"},
            "tma8x16k": {"tma_stages": 8, "tma_block": 16384}, "tma2x64k": {"tma_stages": 2, "tma_block": 65536},
            "vec_dyn": {"copy": "vec", "sched": "dynamic"}}
engs = {}
for name, kw in variants.items():
    engs[name] = Engine(load_topology(text), [0, 0])
    if kw:
        engs[name].configure(**kw)
big = torch.randint(0, 256, (64 * MiB,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
st = torch.cuda.Stream()
warm_up(engs["default"], big, out, st, 1000)
cfg = PathConfig(max_chunks=1, graph_mode=True)
for n in (8 * MiB, 16 * MiB, 24 * MiB, 32 * MiB, 48 * MiB, 64 * MiB):
    res = {k: [] for k in engs}
    for _ in range(5):
        for k, e in engs.items():
            res[k].append(measure_makespan(e, cfg, n, big[:n], out[:n], st, reps=100, trials=1) * 1e6)
    med = {k: round(statistics.median(v), 2) for k, v in res.items()}
    print(n >> 20, "MiB", med, "kernel:", engs["default"].stats().kernel.split(" ")[0], flush=True)
