"""Host cost per send through the Python API layers (Engine.send with tensors,
Engine.send_ptr with raw pointers) next to the GPU time per message, for
cached-graph replay at small sizes.  One JSON line per (size, layer).

    python tools/py_latency.py [iters]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    eng = Engine.loopback(2, 0)
    big = torch.zeros(4 << 20, dtype=torch.uint8, device="cuda:0")
    out = torch.empty_like(big)
    s = torch.cuda.Stream()
    cfg = PathConfig(max_chunks=1, graph_mode=True)
    for n in (4096, 65536, 1 << 20):
        src, dst = big[:n], out[:n]
        prepared = eng.prepare(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1)
        layers = {
            "send": lambda: eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1),
            "prepare": prepared,
            "send_ptr": lambda: eng.send_ptr(src.data_ptr(), dst.data_ptr(), n, 0, 1, cfg,
                                             s.cuda_stream),
        }
        for name, fn in layers.items():
            for _ in range(50):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            t0 = time.perf_counter()
            for _ in range(iters):
                fn()
            t1 = time.perf_counter()
            e1.record(s)
            torch.cuda.synchronize()
            gpu_us = e0.elapsed_time(e1) * 1e3 / iters
            print(json.dumps({"layer": name, "bytes": n, "host_us": (t1 - t0) * 1e6 / iters,
                              "gpu_us_per_msg": gpu_us, "gbs": n / gpu_us / 1e3}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
