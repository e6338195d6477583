"""GPU experiment: single-path sends of 128 KiB-2 MiB (the small-message
kernel) replayed as one-kernel graphs vs programmatic-dependent launches:
MP_PDL_MIN (bytes; experiment knob, read once per process) from the
command line.  µs per message, back-to-back prepared sends, median of 5."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan, warm_up  # noqa: E402

KiB = 1 << 10
e = Engine(load_topology(open("topologies/b200_loopback.topo").read()), [0, 0])
big = torch.randint(0, 256, (4 << 20,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
st = torch.cuda.Stream()
warm_up(e, big, out, st, 2000)
row = {}
for n in [int(x) * KiB for x in os.environ.get("SIZES_KIB", "128,256,384,512,768,1024,2048").split(",")]:
    v = [measure_makespan(e, PathConfig(max_chunks=1, graph_mode=True), n, big[:n], out[:n], st, reps=200, trials=1)
         for _ in range(5)]
    row[n >> 10] = round(statistics.median(v) * 1e6, 2)
print("pdl_min", os.environ.get("MP_PDL_MIN", "default"), row, flush=True)
