"""GPU experiment: SM host-path hop tile size (MP_HOST_TILE experiment knob)
with a bandwidth-sized host share: 2 logical GPUs on one B200, 512 MiB,
direct + host k=8 on the SM host path, host rate in the .topo 20 / 40 GB/s;
loopback (fault 0: GPU-scope flags) and cross-device lowering (fault 2).
Interleaved trials (cache cleared between), medians; bytes checked."""
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
TILES = [int(x) << 10 for x in os.environ.get("TILES_KIB", "16,32,64,128,256").split(",")]
for fault in (0, 2):
    for hbw in (20e9, 40e9):
        e = Engine(load_topology(mesh_text("h", 2, 3.17e12, 1, 2e-6, hbw, 1e-5, "full")), [0, 0])
        e.configure(fault_inject=fault, host="sm")
        cfg = PathConfig(1, True, 8, True)
        res = {t: [] for t in TILES}
        for _ in range(3):
            for t in TILES:
                os.environ["MP_HOST_TILE"] = str(t)
                e.clear_cache()
                res[t].append(size / measure_makespan(e, cfg, size, src, dst, st, reps=8, trials=1) / 1e9)
        e.sync()
        assert torch.equal(src, dst)
        print(f"fault {fault} host {hbw / 1e9:.0f} GB/s: " + "  ".join(
            f"{t >> 10}K {statistics.median(v):.0f}" for t, v in res.items()), flush=True)
        e.close()
