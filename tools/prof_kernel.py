"""Profiling driver: the bench's headline send (512 MiB, direct + host, k=8,
graph replay) a few times, nothing else — so `ncu -s 2 -c 1` lands on a
full-size transfer_kernel launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
S = int(os.environ.get("PROF_BYTES", 512 << 20))
host_bw = float(os.environ.get("PROF_HOST_BW", 20e9))
eng = Engine(load_topology(mesh_text("b200_loopback", 2, 3.2e12, 1, 2e-6, host_bw, 1e-5, "full")), [0, 0])
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=8, graph_mode=True)
for _ in range(int(os.environ.get("PROF_ITERS", 5))):
    eng.send(src, dst, S, cfg, src_dev=0, dst_dev=1)
eng.sync(); torch.cuda.synchronize()
assert torch.equal(src, dst)
print("ok")
