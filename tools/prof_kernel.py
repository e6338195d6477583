"""Profiling driver: one send configuration a few times, nothing else — so
`ncu -k regex:transfer_kernel -s 2 -c 1` lands on a steady-state launch.
Defaults: the bench's headline (512 MiB, direct + host, k=8, graph replay).
Env: PROF_BYTES, PROF_K, PROF_HOST (1/0), PROF_HOST_BW, PROF_HOST_ENGINE (sm/ce/auto),
PROF_ITERS, PROF_DEVICES ("0,1": logical GPU0/GPU1 on two physical GPUs; default loopback),
PROF_GPU_PATHS (1 = direct only; > 1 adds relays through the next logical GPUs),
PROF_TOPO (a .topo file to plan on instead of the generated mesh, e.g. the bench's)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
S = int(os.environ.get("PROF_BYTES", 512 << 20))
host_bw = float(os.environ.get("PROF_HOST_BW", 1e9))
dmap = [int(x) for x in os.environ.get("PROF_DEVICES", "0,0").split(",")]
gp = int(os.environ.get("PROF_GPU_PATHS", 1))
n = max(len(dmap), gp + 1)
dmap = (dmap * n)[:n] if len(dmap) < n else dmap
topo = (open(os.environ["PROF_TOPO"]).read() if os.environ.get("PROF_TOPO") else
        mesh_text("prof", n, 3.2e12 if len(set(dmap)) == 1 else 7.7e11, 1, 2e-6, host_bw, 1e-5, "full"))
eng = Engine(load_topology(topo), dmap)
if os.environ.get("PROF_HOST_ENGINE"):
    eng.configure(host=os.environ["PROF_HOST_ENGINE"])
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty(S, dtype=torch.uint8, device=f"cuda:{dmap[1]}")
cfg = PathConfig(num_gpu_paths=gp, host_path_enabled=os.environ.get("PROF_HOST", "1") == "1",
                 max_chunks=int(os.environ.get("PROF_K", 8)), graph_mode=True)
for _ in range(int(os.environ.get("PROF_ITERS", 5))):
    eng.send(src, dst, S, cfg, src_dev=0, dst_dev=1)
eng.sync(); torch.cuda.synchronize()
assert torch.equal(src.cpu(), dst.cpu())
print("ok")
