"""GPU experiment: loopback relay tables (8 logical GPUs on one B200,
direct + 0..6 relays + host, max_chunks 16, 512 MiB) — GB/s and fraction of
the loopback roofline (a relayed byte costs two HBM copies)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
MiB = 1 << 20
S = int(os.environ.get("SIZE", 512 * MiB))
K = int(os.environ.get("K", 16))
eng = Engine(load_topology(mesh_text("r", 8, 3.17e12, 1, 2e-6, 1e9, 1e-5, "full")), [0] * 8)
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
s = torch.cuda.Stream()
hbm = 6555.5 / 2
row = {"delay": os.environ.get("MP_HOP2_DELAY", "3"), "size": S, "k": K}
for g in range(1, 8):
    cfg = PathConfig(g, True, K, True)
    go = eng.prepare(src, dst, S, cfg, stream=s, src_dev=0, dst_dev=1)
    for _ in range(5): go()
    torch.cuda.synchronize()
    best = 1e9
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e0.record(s)
        for _ in range(10): go()
        e1.record(s); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3 / 10)
    eng.sync()
    assert torch.equal(src, dst)
    share = sum(p.share for p in eng.last_plan()[0] if p.kind == "gpu")
    r = 1.0 / ((1 - share) / hbm + 2 * share / hbm)
    row[f"g{g}"] = [round(S / best / 1e9, 1), round(S / best / 1e9 / r, 3)]
print(json.dumps(row), flush=True)
