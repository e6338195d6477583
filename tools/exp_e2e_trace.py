"""Host roundtrip timing under a concurrent 512 MiB H2D upload (the e2e
step's PCIe load): per chunk-hop trace of a 512 MiB direct + host send with
and without the upload running on another stream."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402

MiB = 1 << 20
size = 512 * MiB
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
eng = Engine(load_topology(open(os.path.join(root, "topologies/b200_loopback.topo")).read()), [0, 0])
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
up = torch.empty(4 * size, dtype=torch.uint8, device="cuda")
hsrc = torch.empty(4 * size, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
cfg = PathConfig(1, True, 8, False)
for upload in (False, True, False, True):
    if upload:
        with torch.cuda.stream(cs):
            up.copy_(hsrc, non_blocking=True)  # ~40 ms of H2D
        torch.cuda._sleep(1000000)
    plan, tl = eng.trace(src, dst, size, cfg, src_dev=0, dst_dev=1)
    rows = [(t.role, round(t.start_time * 1e6, 1), round(t.end_time * 1e6, 1)) for t in tl.tasks]
    d = [r for r in rows if r[0] == "direct"]
    h1 = [r for r in rows if r[0] == "stage_hop1"]
    h2 = [r for r in rows if r[0] == "stage_hop2"]
    print(json.dumps({"upload": upload, "direct_span": [min(r[1] for r in d), max(r[2] for r in d)],
                      "hop1": [r[1:] for r in h1], "hop2": [r[1:] for r in h2]}), flush=True)
    torch.cuda.synchronize()
eng.sync()
