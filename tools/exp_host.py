"""GPU experiment: host-staged path by SM kernels vs copy engines, and the
multi-path makespan against the host share (host link bandwidth in the .topo)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text

MiB = 1 << 20
out = open("gpurun_out/exp_host.jsonl", "w")
def emit(**kw):
    print(json.dumps(kw), flush=True); out.write(json.dumps(kw) + "\n"); out.flush()

S = 512 * MiB
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
stream = torch.cuda.Stream()

def rate(eng, cfg, size, reps=10):
    for _ in range(3):
        eng.send(src[:size], dst[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        eng.send(src[:size], dst[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
    e1.record(stream); torch.cuda.synchronize(); eng.sync()
    assert torch.equal(src[:size], dst[:size])
    return size * reps / (e0.elapsed_time(e1) / 1e3) / 1e9

for size in (64 * MiB, 512 * MiB):
    eng1 = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, 50e9, 1e-5, "full")), [0, 0])
    emit(exp="single", size=size, gbs=rate(eng1, PathConfig(max_chunks=1, graph_mode=True), size))
    eng1.close()
    for host in ("sm", "ce"):
        for host_bw in (2e9, 5e9, 10e9, 20e9, 30e9, 40e9, 55e9, 3.2e12):
            for k in (8,):
                e = Engine(load_topology(mesh_text("x", 2, 3.2e12, 1, 2e-6, host_bw, 1e-5, "full")), [0, 0])
                e.configure(host=host)
                cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=k, graph_mode=True)
                try:
                    emit(exp="multi", host=host, size=size, host_bw=host_bw, k=k, gbs=rate(e, cfg, size))
                except Exception as ex:
                    emit(exp="multi", host=host, size=size, host_bw=host_bw, k=k, error=str(ex))
                e.close()
out.close()
