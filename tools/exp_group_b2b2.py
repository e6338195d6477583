"""Debug: the exp_group_mps.py sequence with knobs to bisect a receiver
byte-count timeout in back-to-back group transfers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_22228_b200 as mp  # noqa: E402
from paper_2604_22228_b200.group import TransferGroup  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
size = 64 << 20
F = set(os.environ.get("FLAGS", "").split(","))
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
topo = mp.load_topology(mp.mesh_text("g", world, 1.6e12, 1, 2e-6, 1e9, 1e-5, "full"))
grp = TransferGroup(topo, device=0, stage_bytes=64 << 20, host_bytes=128 << 20)
sb, db = grp.expose(src, owner=0), grp.expose(dst, owner=1)
cfg = mp.PathConfig(1, False, 8, True)
stream = torch.cuda.Stream(device=0)
err = None
step = "start"
try:
    if "zero" in F:
        dst.zero_()
        torch.cuda.synchronize()
    dist.barrier()
    step = "first"
    grp.transfer(sb, db, size, cfg, stream=stream)
    stream.synchronize()
    grp.sync()
    dist.barrier()
    if "equal" in F and rank == 1:
        torch.equal(src, dst)
    step = "warm"
    for _ in range(3):
        grp.transfer(sb, db, size, cfg, stream=stream)
    stream.synchronize()
    dist.barrier()
    step = "timed"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if "events" in F:
        e0.record(stream)
    for i in range(20):
        step = f"timed {i}"
        grp.transfer(sb, db, size, cfg, stream=stream)
    if "events" in F:
        e1.record(stream)
        e1.synchronize()
    stream.synchronize()
    grp.sync()
except Exception as exc:  # noqa: BLE001
    err = str(exc)[:80]
print(f"rank {rank} flags={sorted(F)} step={step} err={err}", flush=True)
grp.close()
