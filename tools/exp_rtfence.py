"""GPU experiment: helper-warp host roundtrips with / without a trailing
system-scope fence (TILE_FENCE), per message size, static TMA tables,
loopback: direct + host k=8 at the calibrated planning rate (1 GB/s) vs
single path; MP_RT_FENCE_MIN switched between interleaved trials in one
process (the cache is cleared, so each trial lowers afresh); medians.
Output: gpurun_out/exp_rtfence.jsonl"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
SIZES = [int(s) * MiB for s in os.environ.get("SIZES_MIB", "8,16,24,32,48,64,92").split(",")]
VARIANTS = {"never": str(1 << 62), "always": "0"}
TRIALS = int(os.environ.get("TRIALS", "5"))
big = torch.randint(0, 256, (max(SIZES),), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()


def rate(eng, cfg, size, reps=100):
    src, dst = big[:size], obig[:size]
    go = eng.prepare(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(20):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        go()
    e1.record(stream)
    torch.cuda.synchronize()
    eng.sync()
    assert torch.equal(src, dst)
    return e0.elapsed_time(e1) * 1e3 / reps


e = Engine(load_topology(open("topologies/b200_loopback.topo").read()), [0, 0])
rate(e, PathConfig(1, True, 8, True), max(SIZES), reps=200)
with open("gpurun_out/exp_rtfence.jsonl", "a") as out:
    for size in SIZES:
        res = {"single": []} | {v: [] for v in VARIANTS}
        for _ in range(TRIALS):
            res["single"].append(rate(e, PathConfig(max_chunks=1, graph_mode=True), size))
            for name, val in VARIANTS.items():
                os.environ["MP_RT_FENCE_MIN"] = val
                e.clear_cache()
                res[name].append(rate(e, PathConfig(1, True, 8, True), size))
        row = {"bytes": size, **{f"{k}_us": round(statistics.median(v), 3) for k, v in res.items()}}
        for name in VARIANTS:
            row[f"ratio_{name}"] = round(row["single_us"] / row[f"{name}_us"], 3)
        row["kernel"] = e.stats().kernel.split(" ")[0]
        print(json.dumps(row), flush=True)
        out.write(json.dumps(row) + "\n")
e.close()
