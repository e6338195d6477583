"""GPU experiment: L2 cache hints on the LDG/STG copy loop (build variants
via MP_NVCC_EXTRA: -DMP_LD16_NC=... / -DMP_ST16=...): the 512 MiB headline
kernel (ordinary launches, mp_kernel_bench) and back-to-back sends at
128 / 256 / 512 MiB.  Prints one line per variant (VARIANT env)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200.tuner import measure_makespan, warm_up  # noqa: E402

MiB = 1 << 20
e = Engine(load_topology(open("topologies/b200_loopback.topo").read()), [0, 0])
big = torch.randint(0, 256, (512 * MiB,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
st = torch.cuda.Stream()
warm_up(e, big, out, st, 1000)
cfg = PathConfig(1, True, 8, True)
res = {}
for _ in range(3):
    res.setdefault("kernel512_us", []).append(
        e.kernel_bench(big, out, 512 * MiB, PathConfig(1, True, 8, False), 0, 1, reps=20) * 1e3)
    for n in (128, 256, 512):
        res.setdefault(f"send{n}_gbs", []).append(
            n * MiB / measure_makespan(e, cfg, n * MiB, big[:n * MiB], out[:n * MiB], st, reps=20, trials=1) / 1e9)
print(os.environ.get("VARIANT", "?"), {k: round(statistics.median(v), 2) for k, v in res.items()}, flush=True)
