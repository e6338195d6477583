"""GPU experiment: host µs per prepared send (1 MiB single path, enqueue
only, the stream blocked behind a spin so nothing waits on the GPU), the
C-level BoundSend (round 2) vs the earlier Python closure around it,
alternating in one process."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, _mpfast, load_topology  # noqa: E402
from paper_2604_22228_b200._lib import check  # noqa: E402

MiB = 1 << 20
e = Engine(load_topology(open("topologies/b200_loopback.topo").read()), [0, 0])
src = torch.empty(MiB, dtype=torch.uint8, device="cuda:0")
dst = torch.empty_like(src)
st = torch.cuda.Stream()
cfg = PathConfig(max_chunks=1, graph_mode=True)
direct = e.prepare(src, dst, MiB, cfg, stream=st, src_dev=0, dst_dev=1)
raw = _mpfast.bind(e._ctx_addr, src.data_ptr(), dst.data_ptr(), MiB, 0, 1, cfg.abi_addr(), st.cuda_stream,
                   (src, dst, cfg, st))
ctx = e._ctx_addr


def closure():  # the round-1 prepare(): a Python function around the raw binding
    if e._ctx_addr != ctx:
        raise RuntimeError("closed")
    rc = raw()
    if rc:
        check(rc)


for fn in (direct, closure):
    for _ in range(2000):
        fn()
torch.cuda.synchronize()
res = {"bound_c": [], "closure": []}
for rep in range(20):
    for name, fn in (("bound_c", direct), ("closure", closure)):
        torch.cuda.synchronize()
        torch.cuda._sleep(3_000_000)  # keep the stream busy: the calls only enqueue
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        res[name].append((time.perf_counter() - t0) / 200 * 1e6)
torch.cuda.synchronize()
for k, v in res.items():
    v.sort()
    print(k, "median host us per send", round(v[len(v) // 2], 3))
e.close()
