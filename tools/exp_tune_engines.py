"""GPU experiment: why did tune_engines time the SM single path at 1-4 MiB
at ~6.5 us (3 launch quanta) when a standalone measurement gives ~3.1 us?
Per variant: tune_engines' direct-path trials (µs), with and without a GPU
warm-up before it, and standalone measure_makespan per engine."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan, tune_engines  # noqa: E402

MiB = 1 << 20
text = open("topologies/b200_loopback.topo").read()
sizes = [MiB // 2, MiB, 2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB]
big = torch.empty(16 * MiB, dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
st = torch.cuda.Stream()


def warm(ms=300):
    x = torch.empty(256 * MiB, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    t0 = time.time()
    while time.time() - t0 < ms / 1e3:
        y.copy_(x)
    torch.cuda.synchronize()


def show(tag, trials):
    d = {}
    for t in trials:
        if t["path"] == "direct":
            d.setdefault(t["engine"], []).append(round(t["seconds"] * 1e6, 2))
    print(tag, d, flush=True)


for variant in ("cold", "warm", "warm", "cold-after-idle"):
    e = Engine(load_topology(text), [0, 0])
    if variant == "warm":
        warm()
    if variant == "cold-after-idle":
        time.sleep(2)
    rules, trials = tune_engines(e, sizes, reps=50)
    show(variant, trials)
    print("  rules", rules)
    e.close()
e = Engine(load_topology(text), [0, 0])
warm()
for name in ("sm", "ce", "sm", "ce"):
    e.configure(direct=name)
    print(name, [round(measure_makespan(e, PathConfig(max_chunks=1, graph_mode=True), s, big[:s], out[:s], st, 50)
                       * 1e6, 2) for s in sizes], flush=True)

print("--- bisect", flush=True)
for variant in ("policy+stream_dev", "policy", "stream_dev", "none", "policy+stream_dev"):
    e2 = Engine(load_topology(text), [0, 0])
    s2 = torch.cuda.Stream(device=0) if "stream_dev" in variant else torch.cuda.Stream()
    if "policy" in variant:
        e2.set_size_policy([])
    b2 = torch.empty(sizes[-1], dtype=torch.uint8, device="cuda:0")
    o2 = torch.empty_like(b2)
    e2.configure(direct="sm")
    print(variant, [round(measure_makespan(e2, PathConfig(max_chunks=1, graph_mode=True), s, b2[:s], o2[:s], s2, 50)
                          * 1e6, 2) for s in sizes], flush=True)
    e2.close()
