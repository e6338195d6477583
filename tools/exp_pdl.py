"""PDL on/off A/B through the engine: back-to-back prepared single-path sends
(cached graph mode) per size, GPU us per message."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

sizes = [4 << 10, 64 << 10, 1 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20]
big = torch.randint(0, 256, (max(sizes),), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
s = torch.cuda.Stream()
for pdl in (0, 2, 0, 2):
    eng = Engine.loopback(2)
    eng.configure(pdl=pdl)
    row = []
    for n in sizes:
        go = eng.prepare(big[:n], out[:n], n, PathConfig(max_chunks=1, graph_mode=True), stream=s,
                         src_dev=0, dst_dev=1)
        for _ in range(20):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(2000):
            go()
        e1.record(s)
        torch.cuda.synchronize()
        row.append(f"{n >> 10}K={e0.elapsed_time(e1) / 2000 * 1e3:.2f}us")
    assert torch.equal(big, out)
    print(f"pdl={pdl} kernel={eng.stats().kernel.split(' ')[0]}: " + "  ".join(row), flush=True)
    eng.close()
