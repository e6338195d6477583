"""GPU experiment: can a user capture Engine.send into their OWN CUDA graph
(torch.cuda.graph) and replay it?  Cached single-kernel sends (PDL launch
path), cached graph sends with a host path, and a cache miss inside the
capture.  Prints what happens per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

MiB = 1 << 20
eng = Engine.loopback(2)
for name, cfg, n, warm in [("single 16MiB cached", PathConfig(max_chunks=1, graph_mode=True), 16 * MiB, True),
                           ("direct+host 64MiB cached", PathConfig(1, True, 8, True), 64 * MiB, True),
                           ("single 8MiB streamed cached", PathConfig(1, False, 1, False), 8 * MiB, True),
                           ("miss inside capture", PathConfig(1, True, 4, True), 24 * MiB + 3, False)]:
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    s = torch.cuda.Stream()
    try:
        if warm:
            eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
            s.synchronize()
            eng.sync()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
        for r in range(3):
            src.random_(0, 256)
            dst.zero_()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            ok = torch.equal(src, dst)
            if not ok:
                break
        eng.sync()
        print(f"{name}: captured, replays byte-exact={ok}", flush=True)
    except Exception as exc:  # noqa: BLE001
        print(f"{name}: {type(exc).__name__}: {str(exc)[:160]}", flush=True)
        try:
            torch.cuda.synchronize()
            eng.sync()
        except Exception as exc2:  # noqa: BLE001
            print("   after:", str(exc2)[:120])
eng.close()
