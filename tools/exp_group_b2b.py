"""Debug: back-to-back group transfers (no host sync between them), N = 2
ranks on one GPU.  REPS transfers of SIZE bytes direct-only; after them
every rank syncs and reports whether the engine raised, per rank."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_22228_b200 as mp  # noqa: E402
from paper_2604_22228_b200.group import TransferGroup  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
size = int(os.environ.get("SIZE", str(64 << 20)))
topo = mp.load_topology(mp.mesh_text("g", world, 1.6e12, 1, 2e-6, 1e9, 1e-5, "full"))
grp = TransferGroup(topo, device=0, stage_bytes=64 << 20, host_bytes=0 if os.environ.get("NOHOST") else 64 << 20)
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
sb, db = grp.expose(src, owner=0), grp.expose(dst, owner=1)
cfg = mp.PathConfig(1, False, 8, os.environ.get("GRAPH", "1") == "1")
stream = torch.cuda.Stream(device=0)
for reps in [int(x) for x in os.environ.get("REPS", "1,2,3,4,6,8,12,20").split(",")]:
    dist.barrier()
    t0 = time.time()
    err = None
    try:
        for i in range(reps):
            grp.transfer(sb, db, size, cfg, stream=stream)
            if os.environ.get("SYNC_EACH"):
                stream.synchronize()
        stream.synchronize()
        grp.sync()
    except Exception as exc:  # noqa: BLE001
        err = str(exc)[:90]
        try:
            grp.sync()
        except Exception:  # noqa: BLE001
            pass
    print(f"rank {rank} reps {reps} {time.time() - t0:.2f}s err={err} launches", flush=True)
    dist.barrier()
grp.close()
dist.destroy_process_group()
