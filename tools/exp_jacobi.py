"""Measured Jacobi ring halo exchange (measure.run_jacobi, bench.py:355-390)
on a 4-logical-GPU engine: CSV rows in the reference schema per config.

    python tools/exp_jacobi.py [nx ...]     (default nx = 2^24, 2^27)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402
from paper_2604_22228_b200 import measure as M  # noqa: E402


def main():
    nxs = [int(a) for a in sys.argv[1:]] or [2 ** 24, 2 ** 27]
    n = torch.cuda.device_count()
    eng = (Engine.loopback(4) if n < 4 else
           Engine(load_topology(mesh_text("b200x4", 4, 750e9, 1, 2e-6, 55e9, 1e-5, "full")),
                  list(range(4))))
    spec = M.JacobiSpec(nx_values=nxs, iterations=1000, timed=10)
    configs = [PathConfig(1, False, 1, graph_mode=True), PathConfig(2, False, 8, graph_mode=True),
               PathConfig(3, False, 8, graph_mode=True), PathConfig(1, True, 8, graph_mode=True),
               PathConfig(2, True, 8, graph_mode=True)]
    out = []
    for cfg in configs:
        res = M.run_jacobi(spec, cfg, eng, compute="kernel")
        out.extend(res.to_csv().splitlines()[0 if not out else 1:])
    print("\n".join(out))
    eng.close()


if __name__ == "__main__":
    main()
