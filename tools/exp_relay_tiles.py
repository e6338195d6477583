"""GPU experiment: relay hop tile size (MP_RELAY_TILE experiment knob) for
relay tables in loopback — plain (GPU-scope flags) and under the cross-
device lowering (fault_inject=2: system-scope flags) — 512 MiB, direct +
1 / 2 / 6 relays + host (calibrated-small host share), k = 8 / 16.
Interleaved trials in one process (cache cleared between), medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan  # noqa: E402

MiB = 1 << 20
size = 512 * MiB
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty_like(src)
st = torch.cuda.Stream()
TILES = [int(x) << 10 for x in os.environ.get("TILES_KIB", "64,96,128,192,256").split(",")]
for fault in (0, 2):
    for g in (2, 3, 7):
        e = Engine(load_topology(mesh_text("r", 8, 3.17e12, 1, 2e-6, 1e9, 1e-5, "full")), [0] * 8)
        e.configure(fault_inject=fault)
        cfg = PathConfig(g, True, 16 if g == 7 else 8, True)
        res = {t: [] for t in TILES}
        for _ in range(3):
            for t in TILES:
                os.environ["MP_RELAY_TILE"] = str(t)
                e.clear_cache()
                res[t].append(size / measure_makespan(e, cfg, size, src, dst, st, reps=8, trials=1) / 1e9)
        e.sync()
        assert torch.equal(src, dst)
        print(f"fault {fault} relays {g - 1}: " + "  ".join(f"{t >> 10}K {statistics.median(v):.0f}"
                                                        for t, v in res.items()), flush=True)
        e.close()
