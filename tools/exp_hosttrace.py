"""GPU experiment: per chunk-hop timeline (Engine.trace, %globaltimer) of a
direct + host send with the host path on the SM kernels — where the host
round trip sits against the direct stream.  Output: gpurun_out/exp_hosttrace.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20
os.makedirs("gpurun_out", exist_ok=True)
out = open("gpurun_out/exp_hosttrace.jsonl", "a")
HOST_BW = float(os.environ.get("HOST_BW", "1e9"))
topo = load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, HOST_BW, 1e-5, "full"))
eng = Engine(topo, [0, 0])
eng.configure(host=os.environ.get("HOST", "sm"))
SIZES = [int(x) for x in os.environ.get("SIZES", "").split(",") if x] or [4 * MiB, 16 * MiB, 128 * MiB]
K = int(os.environ.get("K", "8"))
for size in SIZES:
    src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    cfg = PathConfig(1, True, K, False)
    for _ in range(5):
        plan, tl = eng.trace(src, dst, size, cfg, src_dev=0, dst_dev=1)
    rows = []
    for t in tl.tasks:
        rows.append({"node": t.node_id, "role": t.role, "start": round(t.start_time * 1e6, 2),
                     "end": round(t.end_time * 1e6, 2), "len": t.length})
    rec = {"size": size, "host": os.environ.get("HOST", "sm"), "rows": rows}
    print(json.dumps({"size": size, "k": K, "host_bw": HOST_BW, "direct": [(r["start"], r["end"]) for r in rows if r["role"] == "direct"],
                      "hop1": [(r["start"], r["end"]) for r in rows if r["role"] == "stage_hop1"],
                      "hop2": [(r["start"], r["end"]) for r in rows if r["role"] == "stage_hop2"]}),
          flush=True)
    out.write(json.dumps(rec) + "\n")
out.close()
