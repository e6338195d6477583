"""GPU experiment: back-to-back single-path sends, 256 KiB - 4 MiB, engine pdl 0..3."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
MiB = 1 << 20
big = torch.randint(0, 256, (8 * MiB,), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
s = torch.cuda.Stream()
for pdl in (0, 1, 3):
    eng = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, 1e9, 1e-5, "full")), [0, 0])
    eng.configure(pdl=pdl)
    row = {"pdl": pdl}
    for size in (256 << 10, 512 << 10, MiB, MiB + 4096, 2 * MiB, 4 * MiB):
        go = eng.prepare(big[:size], obig[:size], size, PathConfig(1, False, 1, True), stream=s, src_dev=0, dst_dev=1)
        for _ in range(20): go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record(s)
            for _ in range(200): go()
            e1.record(s); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 200)
        row[str(size)] = round(best, 2)
    print(json.dumps(row), flush=True)
    eng.close()
