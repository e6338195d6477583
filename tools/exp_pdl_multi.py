"""GPU experiment: direct + host k=8 (helper-warp roundtrips) replayed as a
programmatic-dependent launch (pdl=3, default) vs as its one-kernel graph
(pdl=1: PDL only for the small-message kernel), 4-32 MiB, interleaved
trials, medians; single path (pdl=3) as the reference."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan  # noqa: E402

MiB = 1 << 20
text = open("topologies/b200_loopback.topo").read()
big = torch.randint(0, 256, (32 * MiB,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
st = torch.cuda.Stream()
engs = {}
for p in (3, 2, 1, 0):
    engs[p] = Engine(load_topology(text), [0, 0])
    engs[p].configure(pdl=p)
for size in (4 * MiB, 8 * MiB, 16 * MiB, 32 * MiB):
    res = {"single": [], **{f"multi_pdl{p}": [] for p in engs}}
    for _ in range(5):
        res["single"].append(measure_makespan(engs[3], PathConfig(max_chunks=1, graph_mode=True), size,
                                              big[:size], out[:size], st, reps=100, trials=1))
        for p, e in engs.items():
            res[f"multi_pdl{p}"].append(measure_makespan(e, PathConfig(1, True, 8, True), size, big[:size],
                                                         out[:size], st, reps=100, trials=1))
    med = {k: statistics.median(v) * 1e6 for k, v in res.items()}
    print(size >> 20, "MiB", {k: round(v, 2) for k, v in med.items()},
          {k: round(med["single"] / v, 3) for k, v in med.items() if k != "single"}, flush=True)
