"""Window posted as one send_many program vs W per-call sends (W distinct
buffer pairs): GB/s per size and window."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402
from paper_2604_22228_b200 import measure as M  # noqa: E402

eng = Engine.loopback(2)
sizes = [1 << 10, 4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20]
for w in (4, 16, 64):
    for prog in (False, True):
        ps = [s for s in sizes if s * w <= 2 << 30]
        r = M.run_bw(M.BenchmarkSpec("omb_bw", ps, window=w, iterations=5, warmup=3,
                                     config=PathConfig(1, False, 1, True)), eng, program=prog)
        print(f"W={w:2d} {'program' if prog else 'per-call'}: " + "  ".join(
            f"{s >> 10}K={r.value(s, 'bandwidth') / 1e9:.1f}" for s in ps), flush=True)
eng.close()
