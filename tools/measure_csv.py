"""The reference-schema CSV (bench.py:33) of the measured harnesses at the
current code, loopback (one B200): osu_bw (windows 1 / 16 / 64, per-call
sends and window-as-program), BIBW, latency with the lifecycle phases, and
the Jacobi ring halo exchange — single path and direct + host multi-path.

    python tools/measure_csv.py > gpurun_out/measure.csv
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402
from paper_2604_22228_b200 import measure as M  # noqa: E402

KiB, MiB = 1 << 10, 1 << 20
eng = Engine(load_topology(open("topologies/b200_loopback.topo").read()), [0, 0])
sizes = [4 * KiB, 64 * KiB, MiB, 16 * MiB, 128 * MiB]
rows = [M.CSV_HEADER]


def add(res):
    rows.extend(res.to_csv().splitlines()[1:])


for cfg in (PathConfig(1, False, 1, True), PathConfig(1, True, 8, True)):
    for w in (1, 16, 64):
        add(M.run_bw(M.BenchmarkSpec("omb_bw", sizes, window=w, iterations=5, warmup=2, config=cfg,
                                     topology="b200_loopback"), eng))
        add(M.run_bw(M.BenchmarkSpec("omb_bw_program", sizes, window=w, iterations=5, warmup=2, config=cfg,
                                     topology="b200_loopback"), eng, program=True))
    add(M.run_bibw(M.BenchmarkSpec("omb_bibw", sizes, window=16, iterations=5, warmup=2, config=cfg,
                                   topology="b200_loopback"), eng))
    add(M.run_latency(M.BenchmarkSpec("latency", sizes[:4], iterations=20, warmup=3, config=cfg,
                                      topology="b200_loopback"), eng))
eng.close()
ring = Engine.loopback(4)
spec = M.JacobiSpec(nx_values=[2 ** 24, 2 ** 27], iterations=1000, timed=10)
for cfg in (PathConfig(1, False, 1, True), PathConfig(2, False, 8, True), PathConfig(1, True, 8, True)):
    add(M.run_jacobi(spec, cfg, ring, compute="kernel"))
ring.close()
print("\n".join(rows))
