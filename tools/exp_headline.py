"""The bench headline loop (512 MiB, direct + host, k=8, cached graph, 64
messages per window) against single path, with and without the NVML clock
sampler running, to locate per-message overheads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

size, W, steps = 512 << 20, 64, 10
host_bw = float(os.environ.get("HOST_BW", 8e9))
eng = Engine(load_topology(mesh_text("b200_loopback", 2, 3.17e12, 1, 2e-6, host_bw, 1e-5,
                                     "full")), [0, 0])
if os.environ.get("HOST"):
    eng.configure(host=os.environ["HOST"])
if os.environ.get("PROBE"):  # the bench's order: probe the paths before the buffers exist
    eng.probe_bandwidths(256 << 20, 5, host_bytes=8 << 20)
if os.environ.get("ALLOC") == "bench":  # bench.py's allocation and fill sequence
    src = torch.empty(size, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    src.copy_(torch.randint(0, 256, (size,), dtype=torch.uint8,
                            generator=torch.Generator().manual_seed(20261017)).to(src.device))
    dst.copy_(torch.bitwise_not(src))
else:
    src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
stream = torch.cuda.Stream()


def run(cfg, clocks):
    for _ in range(3 * W):
        eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = bench.Clocks(0) if clocks else None
    if ctx:
        ctx.__enter__()
    e0.record(stream)
    for _ in range(steps * W):
        eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    e1.record(stream)
    torch.cuda.synchronize()
    if ctx:
        ctx.__exit__(None, None, None)
    return steps * W * size / (e0.elapsed_time(e1) / 1e3) / 1e9


multi = PathConfig(1, True, 8, True)
single = PathConfig(max_chunks=1, graph_mode=True)
for clocks in (False, True):
    print(f"host_bw={host_bw:g} host={os.environ.get('HOST', 'ce')} clocks={clocks}: "
          f"multi {run(multi, clocks):.1f}  single {run(single, clocks):.1f}  "
          f"multi {run(multi, clocks):.1f}", flush=True)
st = eng.stats()
print("graph nodes", st.nodes_physical, "kernel", st.kernel)
