"""512 MiB single-path copies with the destination at different offsets from
the source inside one allocation: does the src/dst address relationship
(HBM channel / L2 slice mapping) move the copy rate?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

MiB = 1 << 20
n = 512 * MiB
eng = Engine.loopback(2)
buf = torch.empty(2048 * MiB, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
cfg = PathConfig(max_chunks=1, graph_mode=True)
for off in (512 * MiB, 512 * MiB + 64 * 1024, 576 * MiB, 640 * MiB, 768 * MiB, 1024 * MiB,
            1024 * MiB + 4 * MiB, 1536 * MiB - 2 * MiB):
    src, dst = buf[:n], buf[off:off + n]
    for _ in range(10):
        eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(40):
        eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 40
    e0.record(s)
    for _ in range(40):
        dst.copy_(src)
    e1.record(s)
    torch.cuda.synchronize()
    tus = e0.elapsed_time(e1) * 1e3 / 40
    print(f"dst - src = {off / MiB:8.3f} MiB: engine {us:7.2f} us ({n / us / 1e3:6.0f} GB/s), "
          f"torch copy_ {tus:7.2f} us ({n / tus / 1e3:6.0f} GB/s)", flush=True)
