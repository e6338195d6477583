"""GPU experiment: multi-path vs single path when an osu_bw window of W
non-blocking messages is posted as ONE program (Engine.prepare_many, W
distinct buffer pairs): the host path's PCIe round trip of each message
then overlaps the other messages' direct copies instead of ending every
message.  Loopback, host rate in the .topo = HOST_BW (1 GB/s = the
calibrated planning rate), k = 8, direct + host on the SM host path.
Per size: µs per message (window time / W) for single path vs direct + host,
posted one message at a time (prepare) and as W-message programs.
Output: gpurun_out/exp_window_multi.jsonl
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
os.makedirs("gpurun_out", exist_ok=True)
SIZES = [int(s) for s in os.environ.get("SIZES", "").split(",") if s] or \
    [MiB, 4 * MiB, 8 * MiB, 16 * MiB, 32 * MiB, 64 * MiB]
W = int(os.environ.get("W", "8"))
HOST_BW = float(os.environ.get("HOST_BW", "1e9"))
TRIALS = 5
stream = torch.cuda.Stream()


def timed(post, n_msgs, reps):
    for _ in range(10):
        post()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        post()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n_msgs)


topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, HOST_BW, 1e-5, "full"))
e = Engine(topo, [0, 0])
e.configure(host="sm")
with open("gpurun_out/exp_window_multi.jsonl", "a") as out:
    for size in SIZES:
        srcs = [torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda") for _ in range(W)]
        dsts = [torch.empty_like(s) for s in srcs]
        reps = max(20, min(400, (256 * MiB) // (size * W)))
        res = {}
        for name, cfg in (("single", PathConfig(max_chunks=1, graph_mode=True)),
                          ("multi", PathConfig(1, True, 8, True))):
            one = e.prepare(srcs[0], dsts[0], size, cfg, stream=stream, src_dev=0, dst_dev=1)
            win = e.prepare_many([(s, d, size, 0, 1) for s, d in zip(srcs, dsts)], cfg, stream=stream)
            a, b = [], []
            for _ in range(TRIALS):
                a.append(timed(one, 1, reps * W))
                b.append(timed(win, W, reps))
            e.sync()
            for s, d in zip(srcs, dsts):
                assert torch.equal(s, d)
            res[f"{name}_msg_us"] = round(statistics.median(a), 3)
            res[f"{name}_win_us"] = round(statistics.median(b), 3)
            res[f"{name}_win_kernel"] = e.stats().kernel.split(" ")[0]
        row = {"bytes": size, "W": W, "host_bw": HOST_BW, **res,
               "ratio_msg": round(res["single_msg_us"] / res["multi_msg_us"], 3),
               "ratio_win": round(res["single_win_us"] / res["multi_win_us"], 3)}
        print(json.dumps(row), flush=True)
        out.write(json.dumps(row) + "\n")
        del srcs, dsts
e.close()
