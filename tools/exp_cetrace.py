import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
MiB = 1 << 20
for hbw in (40e9,):
    topo = load_topology(mesh_text("x", 2, 600e9, 1, 2e-6, hbw, 1e-5, "full"))
    e = Engine(topo, [0, 0])
    e.configure(host="ce")
    for size in (256 * MiB,):
        src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        for k in (8, 16):
            for rep in range(3):
                plan, tl = e.trace(src, dst, size, PathConfig(1, True, k, True), 0, 1)
            assert torch.equal(src, dst)
            t0 = min(t.start_time for t in tl.tasks)
            print(f"host_bw {hbw:.0e} size {size >> 20} MiB k {k}")
            for t in sorted(tl.tasks, key=lambda t: t.start_time):
                if t.role != "direct":
                    print(f"  {t.node_id:4d} {t.role:>11} {t.engine} {t.length:9d} B  {(t.start_time - t0) * 1e6:9.1f} {(t.end_time - t0) * 1e6:9.1f} us  {t.length/(t.end_time-t.start_time)/1e9:6.1f} GB/s")
            d = [t for t in tl.tasks if t.role == "direct"]
            print("  direct end", max(t.end_time for t in d) - t0)
    e.close()
