"""Where does the direct + host send lose at 4-16 MiB?  Back-to-back cached
sends (loopback) of: single path; direct k=8 (small kernel / forced TMA
static table); direct + host k=8 with SM roundtrips, PDL on/off, at several
host planning rates (host chunk sizes).  One JSON line per (size, arm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
SIZES = [int(s) for s in os.environ.get("SIZES", "").split(",") if s] or [4 * MiB, 8 * MiB, 16 * MiB]
big = torch.randint(0, 256, (max(SIZES),), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()


def rate(eng, cfg, size, reps=300, trials=5):
    src, dst = big[:size], obig[:size]
    go = eng.prepare(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(20):
        go()
    torch.cuda.synchronize()
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
    kms = eng.kernel_bench(src, dst, size, PathConfig(cfg.num_gpu_paths, cfg.host_path_enabled,
                                                      cfg.max_chunks, False), 0, 1, reps=50)
    paths, chunks = eng.last_plan()
    hb = [c.length for c in chunks if c.path_index != 0]
    return {"us": round(best * 1e6, 3), "kernel_us": round(kms * 1e3, 3),
            "kernel": st.kernel.split(" ")[0], "host_chunks": hb[:3], "n_host": len(hb)}


for size in SIZES:
    for hbw in [float(x) for x in os.environ.get("HBWS", "0.1e9,1e9,4e9").split(",")]:
        topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, hbw, 1e-5, "full"))
        arms = {}
        e = Engine(topo, [0, 0])
        if hbw == 1e9 and not os.environ.get("HOST_ONLY"):
            arms["single"] = rate(e, PathConfig(max_chunks=1, graph_mode=True), size)
            arms["direct_k8"] = rate(e, PathConfig(1, False, 8, True), size)
            e.configure(small_max_bytes=0)
            arms["direct_k8_tma"] = rate(e, PathConfig(1, False, 8, True), size)
            e.configure(small_max_bytes=4 * MiB)
        e.configure(host="sm")
        arms["host_sm_k8"] = rate(e, PathConfig(1, True, 8, True), size)
        if not os.environ.get("HOST_ONLY"):
            arms["host_sm_k1"] = rate(e, PathConfig(1, True, 1, True), size)
            e.configure(pdl=0)
            arms["host_sm_k8_nopdl"] = rate(e, PathConfig(1, True, 8, True), size)
        e.close()
        for k, v in arms.items():
            print(json.dumps({"size": size, "host_bw": hbw, "arm": k, **v}), flush=True)
