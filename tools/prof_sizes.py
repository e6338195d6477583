"""Per-size single-path SM sends (graph mode): event time per message, and the
transfer kernel's own duration (streamed mode, events on its stream).
Run plain, or under `ncu --metrics gpu__time_duration.sum` for a launch list."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

MiB = 1 << 20
sizes = [int(x) for x in os.environ.get("SIZES", "").split(",") if x] or \
    [1 * MiB, 4 * MiB, 16 * MiB, 32 * MiB, 64 * MiB, 128 * MiB, 512 * MiB]
reps = int(os.environ.get("REPS", 20))
eng = Engine.loopback(2)
eng.set_kernel_timing(True)
opts = os.environ.get("ENGINE_OPTS")
if opts:
    eng.configure(**json.loads(opts))
big = torch.randint(0, 256, (max(sizes),), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
s = torch.cuda.Stream()
g = PathConfig(max_chunks=1, graph_mode=True)
st = PathConfig(max_chunks=1, graph_mode=False)
for n in sizes:
    a, b = big[:n], out[:n]
    for _ in range(3):
        eng.send(a, b, n, g, stream=s, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        eng.send(a, b, n, g, stream=s, src_dev=0, dst_dev=1)
    e1.record(s)
    torch.cuda.synchronize()
    per_msg = e0.elapsed_time(e1) / reps * 1e3
    ks = []
    for _ in range(5):
        eng.send(a, b, n, st, stream=s, src_dev=0, dst_dev=1)
        ks.append(eng.kernel_time_ms() * 1e3)
    assert torch.equal(a, b)
    print(json.dumps({"bytes": n, "us_per_msg_graph": per_msg, "kernel_us": sorted(ks)[2],
                      "gbs_graph": n / per_msg / 1e3, "gbs_kernel": n / sorted(ks)[2] / 1e3}),
          flush=True)
