"""Profiling driver: a 512 MiB loopback send over direct + N relays (+ host),
max_chunks 16 (BASELINE config 3/4 shape), graph replay; `ncu -s 2 -c 1`
lands on a full-size relay-table transfer_kernel launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

S = int(os.environ.get("PROF_BYTES", 512 << 20))
g = int(os.environ.get("PROF_GPU_PATHS", 2))
eng = Engine(load_topology(mesh_text("l8", 8, 3.17e12, 1, 2e-6, 6e9, 1e-5, "full")), [0] * 8)
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
cfg = PathConfig(num_gpu_paths=g, host_path_enabled=True, max_chunks=16, graph_mode=True)
for _ in range(int(os.environ.get("PROF_ITERS", 4))):
    eng.send(src, dst, S, cfg, src_dev=0, dst_dev=1)
eng.sync()
torch.cuda.synchronize()
assert torch.equal(src, dst)
print("ok", eng.stats().kernel)
