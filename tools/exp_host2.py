"""SM host path (front-loaded hop1 tiles) vs CE host path, against the host share."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
from paper_2604_22228_b200.tuner import measure_makespan
MiB = 1 << 20
S = 512 * MiB
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
st = torch.cuda.Stream()
for size in (4 * MiB, 16 * MiB, 64 * MiB, 512 * MiB):
    for host in ("sm",):
        for hbw in (5e9, 10e9, 20e9, 30e9, 40e9, 55e9):
            for tile in (0,):
                e = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, hbw, 1e-5, "full")), [0, 0])
                e.configure(host=host, tile_bytes=tile if host == "sm" else 0)
                if host == "ce" and tile:
                    continue
                cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=8, graph_mode=True)
                t = measure_makespan(e, cfg, size, src[:size], dst[:size], st, reps=10)
                e.sync()
                ok = torch.equal(src[:size], dst[:size])
                print(json.dumps({"size": size, "host": host, "host_bw": hbw, "tile": tile,
                                  "gbs": size / t / 1e9, "ok": ok,
                                  "launch_us": e.stats().launch_us}), flush=True)
                e.close()
