"""GPU experiment: the host-staged path alone (98% host share, 256 MiB) on the SM
kernels vs copy engines, loopback and cross-device lowering, k = 8/16/32."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
from paper_2604_22228_b200.tuner import measure_makespan
MiB = 1 << 20
size = 256 * MiB
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda"); dst = torch.empty_like(src)
st = torch.cuda.Stream()
for fault in (0, 2):
    for host in ("sm", "ce"):
        for k in (8, 16, 32):
            e = Engine(load_topology(mesh_text("h", 2, 1e9, 1, 2e-6, 50e9, 1e-5, "full")), [0, 0])
            e.configure(fault_inject=fault, host=host)
            t = statistics.median(measure_makespan(e, PathConfig(1, True, k, True), size, src, dst, st, reps=4, trials=1) for _ in range(3))
            paths, chunks = e.last_plan()
            hb = sum(c.length for c in chunks if paths[c.path_index].kind == "host")
            e.sync(); assert torch.equal(src, dst); dst.zero_()
            print(f"fault {fault} host {host} k {k}: host share {hb/size:.3f}, host path delivers {hb/t/1e9:.1f} GB/s (total {size/t/1e9:.1f})", flush=True)
            e.close()
m = Engine.loopback(2).measure_paths(0, 1, 256 * MiB, 5)
print({k: round(v, 1) for k, v in m.items()})
