"""e2e experiment (round 2): why an H2D upload slows down beside the copy
kernel, and which upload shape / kernel shape keeps it at PCIe rate.

For each variant: the 512 MiB upload alone, the 64 sends alone, and both
started together on two streams (each stream's own completion time).
Prints one JSON line per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology  # noqa: E402

MiB = 1 << 20
size, W = 512 * MiB, 64
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
text = open(os.path.join(root, "topologies/b200_loopback.topo")).read()
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
up = torch.empty_like(src)
hsrc = torch.empty(size, dtype=torch.uint8, pin_memory=True)
hsrc.copy_(src.cpu())
cur = torch.cuda.current_stream()
ups = [torch.cuda.Stream() for _ in range(4)]


def ev():
    return torch.cuda.Event(enable_timing=True)


def upload(pieces, nstreams, start):
    """The 512 MiB upload as `pieces` copies spread over `nstreams` streams;
    returns the end events."""
    n = size // pieces
    ends = []
    for s in range(nstreams):
        ups[s].wait_event(start)
    for p in range(pieces):
        st = ups[p % nstreams]
        with torch.cuda.stream(st):
            up[p * n:(p + 1) * n].copy_(hsrc[p * n:(p + 1) * n], non_blocking=True)
    for s in range(nstreams):
        e = ev()
        e.record(ups[s])
        ends.append(e)
    return ends


def run(name, eng, cfg, pieces=1, nstreams=1, sends=W):
    go = eng.prepare(src, dst, size, cfg, stream=cur, src_dev=0, dst_dev=1)
    for _ in range(8):
        go()
    torch.cuda.synchronize()
    res = {"variant": name, "pieces": pieces, "streams": nstreams}
    # upload alone
    s0 = ev()
    s0.record(cur)
    ends = upload(pieces, nstreams, s0)
    torch.cuda.synchronize()
    t_up = max(s0.elapsed_time(e) for e in ends) / 1e3
    res["upload_alone_gbs"] = size / t_up / 1e9
    # sends alone
    s0, s1 = ev(), ev()
    s0.record(cur)
    for _ in range(sends):
        go()
    s1.record(cur)
    torch.cuda.synchronize()
    t_s = s0.elapsed_time(s1) / 1e3
    res["sends_alone_gbs"] = sends * size / t_s / 1e9
    res["sends_alone_ms"] = t_s * 1e3
    # together
    s0, s1 = ev(), ev()
    s0.record(cur)
    ends = upload(pieces, nstreams, s0)
    for _ in range(sends):
        go()
    s1.record(cur)
    torch.cuda.synchronize()
    t_u2 = max(s0.elapsed_time(e) for e in ends) / 1e3
    t_s2 = s0.elapsed_time(s1) / 1e3
    res["upload_conc_gbs"] = size / t_u2 / 1e9
    res["upload_conc_ms"] = t_u2 * 1e3
    res["sends_conc_ms"] = t_s2 * 1e3
    res["step_ms"] = max(t_u2, t_s2) * 1e3
    res["e2e_gbs"] = sends * size / max(t_u2, t_s2) / 1e9
    eng.sync()
    print(json.dumps(res), flush=True)


from paper_2604_22228_b200 import mesh_text  # noqa: E402
HBWS = [float(x) for x in os.environ.get("HBWS", "0.1e9,0.5e9,1e9,2e9").split(",")]
for hbw in HBWS:
    eng = Engine(load_topology(mesh_text("x", 2, 3.17e12, 1, 2e-6, hbw, 1e-5, "full")), [0, 0])
    run(f"direct+host k8 host_bw={hbw:g}", eng, PathConfig(1, True, 8, True), 1, 1)
    run(f"direct+host k1 host_bw={hbw:g}", eng, PathConfig(1, True, 1, True), 1, 1)
    eng.close()
