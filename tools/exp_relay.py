"""Relay sweep in loopback (BASELINE config 4 shape): GB/s per relay count
for the current engine build; env knobs select variants."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

size = int(os.environ.get("SIZE", 512 << 20))
eng = Engine(load_topology(mesh_text("l8", 8, 3.17e12, 1, 2e-6, 6e9, 1e-5, "full")), [0] * 8)
if os.environ.get("ENGINE_OPTS"):
    eng.configure(**json.loads(os.environ["ENGINE_OPTS"]))
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
s = torch.cuda.Stream()
out = {}
for g in (1, 2, 3, 5, 7):
    cfg = PathConfig(num_gpu_paths=g, host_path_enabled=True, max_chunks=16, graph_mode=True)
    for _ in range(4):
        eng.send(src, dst, size, cfg, stream=s, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        eng.send(src, dst, size, cfg, stream=s, src_dev=0, dst_dev=1)
    e1.record(s)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    out[g - 1] = round(10 * size / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
print(os.environ.get("TAG", ""), json.dumps(out), flush=True)
