"""GPU experiment: per chunk-hop timeline (%globaltimer) of a direct + host
send at 4 / 16 MiB, loopback, SM host path (helper roundtrips): when do the
direct chunks end, when do the host chunks' hop1 / hop2 start and end.
Trace mode launches without PDL and with a stamp kernel, so absolute
durations run longer than a cached replay; the ORDER is the point.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
for hbw in (1e9, 4e9):
    topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, hbw, 1e-5, "full"))
    e = Engine(topo, [0, 0])
    e.configure(host="sm")
    for size in (4 * MiB, 16 * MiB):
        src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        for rep in range(6):
            plan, tl = e.trace(src, dst, size, PathConfig(1, True, 8, True), 0, 1)
        assert torch.equal(src, dst)
        t0 = min(t.start_time for t in tl.tasks)
        print(f"host_bw {hbw:.0e} size {size >> 20} MiB")
        for t in sorted(tl.tasks, key=lambda t: t.start_time):
            print(f"  {t.node_id:4d} {t.role:>11} {t.length:9d} B  {(t.start_time - t0) * 1e6:8.3f} "
                  f"{(t.end_time - t0) * 1e6:8.3f} us")
    e.close()
