"""GPU experiment: small host roundtrips in bins (one CTA per bin) vs one
roundtrip tile per CTA (MP_RT_BIN=0), static TMA tables, loopback.

Per message size and host rate in the .topo (HOST_BWS; 1 GB/s = the
calibrated planning rate, 4 GB/s gives ~4x larger host chunks): single path
k=1 and direct + host k=8 (SM host path), with MP_RT_BIN switched between
interleaved trials inside one process (the cache is cleared between them,
so each trial lowers afresh).  Back-to-back prepared sends, bytes checked;
median over trials.  Output: gpurun_out/exp_rtbin.jsonl
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
    [4 * MiB, 8 * MiB, 16 * MiB, 32 * MiB, 64 * MiB]
HOST_BWS = [float(s) for s in os.environ.get("HOST_BWS", "1e9,4e9").split(",")]
BINS = os.environ.get("BINS", "0,2048,4096").split(",")
TRIALS = int(os.environ.get("TRIALS", "7"))
K = int(os.environ.get("K", "8"))
big = torch.randint(0, 256, (max(SIZES),), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()


def rate(eng, cfg, size, reps=200):
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


with open("gpurun_out/exp_rtbin.jsonl", "a") as out:
    for hbw in HOST_BWS:
        topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, hbw, 1e-5, "full"))
        e = Engine(topo, [0, 0])
        e.configure(host="sm")
        rate(e, PathConfig(1, True, K, True), max(SIZES), reps=2000)  # clocks up
        for size in SIZES:
            res = {"single": []} | {b: [] for b in BINS}
            for _ in range(TRIALS):
                res["single"].append(rate(e, PathConfig(max_chunks=1, graph_mode=True), size))
                for b in BINS:
                    os.environ["MP_RT_BIN"] = b
                    e.clear_cache()
                    res[b].append(rate(e, PathConfig(1, True, K, True), size))
            row = {"host_bw": hbw, "bytes": size, "k": K,
                   **{f"{n}_us": round(statistics.median(v), 3) for n, v in res.items()}}
            for b in BINS:
                row[f"ratio_{b}"] = round(row["single_us"] / row[f"{b}_us"], 3)
            print(json.dumps(row), flush=True)
            out.write(json.dumps(row) + "\n")
        e.close()
