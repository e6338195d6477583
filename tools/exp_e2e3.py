"""e2e breakdown: the checksum's cost and bench.e2e_run as the bench runs it."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402

MiB = 1 << 20
size = 512 * MiB
text = open(bench.topo_file(1)).read()
eng = Engine(load_topology(text), [0, 0])
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("sum_u8_i64", lambda: dst.sum(dtype=torch.int64)),
                 ("sum_view_i64", lambda: dst.view(torch.int64).sum()),
                 ("sum_view_i32_i64", lambda: dst.view(torch.int32).sum(dtype=torch.int64))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, "ms", e0.elapsed_time(e1) / 10, flush=True)
args = types.SimpleNamespace(size=size, window=64, steps=20, warmup=5)
cfg = PathConfig(1, True, 8, True)
for _ in range(2):
    print("bench e2e_run", bench.e2e_run(torch, eng, cfg, src, dst, args), flush=True)
print("bench e2e_run steps=10", bench.e2e_run(torch, eng, cfg, src, dst, args, steps=10), flush=True)
