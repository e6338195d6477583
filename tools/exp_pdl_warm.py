"""GPU experiment: back-to-back prepared single-path sends at 0.5-16 MiB,
repeated passes from process start (fresh engine): does the PDL-replayed
small / static kernel start in a slow state (~6.4 us = 3 launch quanta)
and speed up later?  One line per pass: µs per message per size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan  # noqa: E402

MiB = 1 << 20
sizes = [MiB // 2, MiB, 2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB]
text = open("topologies/b200_loopback.topo").read()
e = Engine(load_topology(text), [0, 0])
big = torch.empty(sizes[-1], dtype=torch.uint8, device="cuda:0")
out = torch.empty_like(big)
st = torch.cuda.Stream(device=0)
t0 = time.time()
for p in range(int(os.environ.get("PASSES", "8"))):
    row = [round(measure_makespan(e, PathConfig(max_chunks=1, graph_mode=True), s, big[:s], out[:s], st, 50) * 1e6, 2)
           for s in sizes]
    # host µs per prepared 1 MiB send (enqueue only): is the slow phase host-bound?
    go = e.prepare(big[:MiB], out[:MiB], MiB, PathConfig(max_chunks=1, graph_mode=True), stream=st,
                   src_dev=0, dst_dev=1)
    h0 = time.perf_counter()
    for _ in range(50):
        go()
    host_us = (time.perf_counter() - h0) / 50 * 1e6
    torch.cuda.synchronize()
    print(f"pass {p} t={time.time() - t0:.3f}s host_us_per_send={host_us:.2f}", row, flush=True)
    if os.environ.get("CLEAR"):
        e.clear_cache()
