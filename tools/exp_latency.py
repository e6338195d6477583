"""GPU experiment: device latency of ONE send (events around it, idle GPU)
and back-to-back time per send, single path vs direct + host (SM roundtrip),
small and mid sizes.  Prints one JSON line per size."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
MiB = 1 << 20
eng = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, 1e9, 1e-5, "full")), [0, 0])
big = torch.randint(0, 256, (64 * MiB,), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
s = torch.cuda.Stream()
for size in (4096, 65536, MiB, 4 * MiB, 16 * MiB, 64 * MiB):
    row = {"size": size}
    for name, cfg in (("single", PathConfig(1, False, 1, True)), ("host_k1", PathConfig(1, True, 1, True)),
                      ("host_k8", PathConfig(1, True, 8, True))):
        go = eng.prepare(big[:size], obig[:size], size, cfg, stream=s, src_dev=0, dst_dev=1)
        for _ in range(20): go()
        torch.cuda.synchronize()
        lat = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(50):
            e0.record(s); go(); e1.record(s); e1.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
        e0.record(s)
        for _ in range(200): go()
        e1.record(s); torch.cuda.synchronize()
        row[name] = {"lat_us": round(statistics.median(lat), 2), "b2b_us": round(e0.elapsed_time(e1) * 1e3 / 200, 2),
                     "kernel": eng.stats().kernel.split(" ")[0][-5:]}
    eng.sync()
    print(json.dumps(row), flush=True)
