"""GPU experiment: multi-process group mode (one process per logical GPU,
CUDA-IPC, device barrier) with the host-staged path through the per-rank
shared-memory inbox, N = 2 ranks sharing the one B200 under MPS (each rank
provisioned half the SMs, as separate GPUs would give each rank its own).

Rank 0 sends 512 MiB to rank 1: direct only vs direct + host planned at
several host rates; the sender's kernel runs direct + hop1 tiles, the
receiver's kernel the hop2 tiles (its own SMs) and the byte-count wait.
GB/s = bytes / the receiver's CUDA-event time over back-to-back transfers
(max over ranks); the first transfer of each config is checked byte-exact.

    torchrun --nproc-per-node 2 tools/exp_group_mps.py   (under MPS: tools/gpu_group_mps.sh)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_22228_b200 as mp  # noqa: E402
from paper_2604_22228_b200.group import TransferGroup  # noqa: E402

MiB = 1 << 20


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    size = int(os.environ.get("SIZE", str(512 * MiB)))
    reps = int(os.environ.get("REPS", "20"))
    link = float(os.environ.get("LINK_BW", "1.6e12"))
    src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda:0",
                        generator=torch.Generator(device="cuda:0").manual_seed(7))
    dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
    rows = []
    for host_bw in [0.0] + [float(x) * 1e9 for x in os.environ.get("HOST_BWS", "10,20,40").split(",")]:
        topo = mp.load_topology(mp.mesh_text("g", world, link, 1, 2e-6, host_bw or 1e9, 1e-5, "full"))
        grp = TransferGroup(topo, device=0, stage_bytes=512 << 20, host_bytes=128 << 20)
        sb = grp.expose(src, owner=0)
        db = grp.expose(dst, owner=1)
        gp = int(os.environ.get("GPU_PATHS", "1"))  # 1 + relay ranks (<= world - 1)
        cfg = mp.PathConfig(num_gpu_paths=gp, host_path_enabled=host_bw > 0, max_chunks=8,
                            graph_mode=os.environ.get("GRAPH", "1") == "1")
        stream = torch.cuda.Stream(device=0)
        dst.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        grp.transfer(sb, db, size, cfg, stream=stream)
        stream.synchronize()
        grp.sync()
        dist.barrier()
        ok = torch.equal(src, dst) if rank == 1 else None
        for _ in range(3):
            grp.transfer(sb, db, size, cfg, stream=stream)
        stream.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            grp.transfer(sb, db, size, cfg, stream=stream)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        t = [None] * world
        dist.all_gather_object(t, ms)
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        grp.sync()
        if rank == 0:
            paths, chunks = grp.last_plan()
            kinds = [pth.kind for pth in paths]
            host_bytes = sum(c.length for c in chunks if kinds[c.path_index] == "host")
            rows.append({"world": world, "gpu_paths": gp, "host_plan_gbs": host_bw / 1e9, "host_share": round(host_bytes / size, 4),
                         "gbs": round(reps * size / (max(t) / 1e3) / 1e9, 1), "bytes_ok": oks[1]})
            print(json.dumps(rows[-1]), flush=True)
        grp.close()
        dist.barrier()
    if rank == 0:
        base = rows[0]["gbs"]
        for r in rows[1:]:
            r["over_direct_only"] = round(r["gbs"] / base, 3)
        print(json.dumps({"summary": rows}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
