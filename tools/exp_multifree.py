"""GPU experiment: where does direct + host multi-path lose to single path?

Per message size, back-to-back cached sends (loopback, logical GPU0/GPU1 on
cuda:0) of: single path k=1; direct only k=8 (chunking cost); direct + host
k=8 with the host path on copy engines and on the SM kernels (host rate in
the .topo = HOST_BW, default 1 GB/s = the calibrated planning rate).
Output: gpurun_out/exp_multifree.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
os.makedirs("gpurun_out", exist_ok=True)
out = open("gpurun_out/exp_multifree.jsonl", "a")
HOST_BW = float(os.environ.get("HOST_BW", "1e9"))
SIZES = [int(s) for s in os.environ.get("SIZES", "").split(",") if s] or \
    [4 * MiB, 16 * MiB, 64 * MiB, 128 * MiB, 256 * MiB]
TAG = os.environ.get("TAG", "")


def emit(**kw):
    kw["tag"] = TAG
    print(json.dumps(kw), flush=True)
    out.write(json.dumps(kw) + "\n")
    out.flush()


big = torch.randint(0, 256, (max(SIZES),), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()


def rate(eng, cfg, size, reps, trials=3):
    src, dst = big[:size], obig[:size]
    go = eng.prepare(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(10):
        go()
    torch.cuda.synchronize()
    eng.sync()
    best = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(trials):
        e0.record(stream)
        for _ in range(reps):
            go()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        best = t if best is None else min(best, t)
    eng.sync()
    assert torch.equal(src, dst)
    st = eng.stats()
    return {"gbs": size / best / 1e9, "us": best * 1e6, "kernel": st.kernel.split(" ")[0],
            "kernels": st.kernels, "ce": st.ce_copies, "nodes_phys": st.nodes_physical}


topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, HOST_BW, 1e-5, "full"))
for size in SIZES:
    reps = 200 if size <= 64 * MiB else 40
    arms = {}
    e = Engine(topo, [0, 0])
    arms["single"] = rate(e, PathConfig(max_chunks=1, graph_mode=True), size, reps)
    arms["direct_k8"] = rate(e, PathConfig(1, False, 8, True), size, reps)
    for host in ("ce", "sm"):
        e.configure(host=host)
        arms[f"host_{host}_k8"] = rate(e, PathConfig(1, True, 8, True), size, reps)
        arms[f"host_{host}_k8_stream"] = rate(e, PathConfig(1, True, 8, False), size, reps)
    e.close()
    emit(size=size, host_bw=HOST_BW, **arms)
out.close()
