"""Runs the README's quick-start snippet verbatim (plus a byte check)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

eng = Engine.loopback(2)
src = torch.randint(0, 256, (512 << 20,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty_like(src)
cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=8, graph_mode=True)
eng.send(src, dst, config=cfg, src_dev=0, dst_dev=1)
go = eng.prepare(src, dst, config=cfg, src_dev=0, dst_dev=1)
go()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    eng.send(src, dst, config=cfg, src_dev=0, dst_dev=1)
dst.zero_()
g.replay()
torch.cuda.synchronize()
eng.sync()
print("README snippet ok:", torch.equal(src, dst))
