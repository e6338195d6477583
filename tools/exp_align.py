"""GPU experiment: cost of misaligned chunk boundaries (direct only) and of
the host path, with PDL replays and with ordinary launches (kernel_bench)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
MiB = 1 << 20
big = torch.randint(0, 256, (257 * MiB,), dtype=torch.uint8, device="cuda")
obig = torch.empty_like(big)
stream = torch.cuda.Stream()
def rate(eng, cfg, size, reps=60):
    go = eng.prepare(big[:size], obig[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(10): go()
    torch.cuda.synchronize()
    best = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e0.record(stream)
        for _ in range(reps): go()
        e1.record(stream); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / reps
        best = t if best is None else min(best, t)
    kb = eng.kernel_bench(big[:size], obig[:size], size, PathConfig(cfg.num_gpu_paths, cfg.host_path_enabled, cfg.max_chunks, False), 0, 1, reps=reps) * 1e3
    eng.sync()
    return round(best, 2), round(kb, 2)
for hb in (1e9,):
    e = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, hb, 1e-5, "full")), [0, 0])
    e.configure(host="sm")
    for base in (16 * MiB, 64 * MiB, 128 * MiB, 256 * MiB):
        for extra in (0, 12345):
            s = base + extra
            row = {"size": s}
            for name, cfg in (("single", PathConfig(1, False, 1, True)), ("k8", PathConfig(1, False, 8, True)),
                              ("k9", PathConfig(1, False, 9, True)), ("host_k8", PathConfig(1, True, 8, True))):
                row[name] = rate(e, cfg, s)
            print(json.dumps(row), flush=True)
