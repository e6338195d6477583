"""GPU experiment: does multi-path ADD bandwidth when the direct path is the
bottleneck?  On one B200 in loopback the "direct" path is an HBM copy
(~3.3 TB/s) that the host path cannot add to (a host-staged byte is read
from and written to the same HBM).  Here the process runs under MPS with
CUDA_MPS_ACTIVE_THREAD_PERCENTAGE = P (set by the caller), which caps the SM
transfer kernel — a stand-in for a link-limited direct path (P ~ 20 % gives
an NVLink-class ~0.7 TB/s) — while the copy engines of the host path are not
capped, like PCIe beside NVLink on a real node.

Per P: the measured per-path rates (SM direct, PCIe D2H / H2D).  Two
planning topologies: (a) "probed": the raw probes as the .topo link / host
rates; (b) "calibrated": tuner.calibrate_host_bandwidth at 512 MiB (the host
rate and host mechanism, CE or SM, that maximise measured direct + host
throughput; its curve is written too).  Then at 64 / 128 / 256 / 512 MiB:
single path (SM kernel, k = 1) vs direct + host (k = 8), back-to-back
cached sends; bytes checked.  R = direct + min(D2H, H2D).
Output: gpurun_out/exp_linkcap.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402
from paper_2604_22228_b200.tuner import calibrate_host_bandwidth  # noqa: E402

MiB = 1 << 20
os.makedirs("gpurun_out", exist_ok=True)
P = os.environ.get("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE", "100")
K = int(os.environ.get("K", "8"))
ONLY_CAL = os.environ.get("ONLY_CAL", "") == "1"
TAG = os.environ.get("TAG", "")
SIZES = [64 * MiB, 128 * MiB, 256 * MiB, 512 * MiB]
stream = torch.cuda.Stream()
big = torch.randint(0, 256, (max(SIZES),), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)


def rate(eng, cfg, size, reps):
    src, dst = big[:size], obig[:size]
    go = eng.prepare(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(5):
        go()
    torch.cuda.synchronize()
    best = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e0.record(stream)
        for _ in range(reps):
            go()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        best = t if best is None else min(best, t)
    eng.sync()
    assert torch.equal(src, dst)
    return size / best / 1e9


probe_eng = Engine(load_topology(mesh_text("p", 2, 1e12, 1, 2e-6, 55e9, 1e-5, "full")), [0, 0])
m = probe_eng.measure_paths(0, 1, 256 * MiB, 5)
probe_eng.close()
direct, pcie = m["direct_sm"], min(m["d2h"], m["h2d"])
probed = load_topology(mesh_text("linkcap", 2, direct * 1e9, 1, 2e-6, pcie * 1e9, 1e-5, "full"))
eng = Engine(probed, [0, 0])
eng.configure(host="ce")
plans = [] if ONLY_CAL else [("probed", probed, "ce", pcie)]
cal = Engine(probed, [0, 0])
hbw, ctopo, trials = calibrate_host_bandwidth(cal, direct * 1e9, 512 * MiB, K, reps=5, name="linkcap_cal")
host_engine = {0: "sm", 1: "ce", 2: "auto"}[cal.options()["host_engine"]]
cal.close()
with open("gpurun_out/exp_linkcap.jsonl", "a") as out:
    out.write(json.dumps({"mps_pct": P, "calibration": [(h, round(b / 1e9, 1), round(g, 1)) for h, b, g in trials],
                          "picked_gbs": hbw / 1e9, "picked_engine": host_engine}) + "\n")
    plans.append(("calibrated", ctopo, host_engine, hbw / 1e9))
    for plan_name, topo, hengine, host_plan in plans:
        eng.set_topology(topo)
        eng.configure(host=hengine)
        for size in SIZES:
            reps = max(10, (2 << 30) // size)
            single = rate(eng, PathConfig(max_chunks=1, graph_mode=True), size, reps)
            multi = rate(eng, PathConfig(1, True, K, True), size, reps)
            paths, chunks = eng.last_plan()
            host_bytes = sum(c.length for c in chunks if c.path_index == 1)
            row = {"tag": TAG, "k": K, "mps_pct": P, "plan": plan_name, "host_engine": hengine, "host_plan_gbs": round(host_plan, 1),
                   "bytes": size, "direct_probe_gbs": round(direct, 1), "pcie_probe_gbs": round(pcie, 1),
                   "host_share": round(host_bytes / size, 4), "single_gbs": round(single, 1),
                   "multi_gbs": round(multi, 1), "multi_over_single": round(multi / single, 3),
                   "R_gbs": round(direct + pcie, 1), "frac_R": round(multi / (direct + pcie), 3)}
            print(json.dumps(row), flush=True)
            out.write(json.dumps(row) + "\n")
eng.close()
