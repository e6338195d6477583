"""GPU experiment: run-to-run spread of the bench's multi-over-single
sweep (bench.short_sweep) in one process, before and after allocating
(and touching) a 512 MiB pinned host buffer like the bench's e2e leg."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402

MiB = 1 << 20
eng = Engine(load_topology(open(bench.topo_file(1)).read()), [0, 0])
big = torch.randint(0, 256, (64 * MiB,), dtype=torch.uint8, device="cuda:0")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()
sizes = [4 * MiB, 16 * MiB, 64 * MiB]
for tag in ("fresh", "fresh2", "pinned512", "pinned512b"):
    if tag == "pinned512":
        h = torch.empty(512 * MiB, dtype=torch.uint8, pin_memory=True)
        big2 = torch.empty(512 * MiB, dtype=torch.uint8, device="cuda:0")
        big2.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
    rows = bench.short_sweep(torch, eng, PathConfig, big, obig, stream, sizes, 1, True, 8)
    print(tag, [(r["bytes"] >> 20, round(r["ratio"], 3), round(r["bytes"] / r["multi_gbs"] / 1e3, 2)) for r in rows],
          flush=True)
eng.close()
