"""e2e pipeline experiment: H2D of each window's input overlapping the
previous window's sends, with the host-staged path on copy engines vs on the
SM kernels (mapped pinned memory).  Prints GB/s per variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

size, W, steps = 512 << 20, 64, 4
HOST_BWS = [float(x) * 1e9 for x in os.environ.get("HOST_BWS", "4").split(",")]
src = torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
hsrc = torch.empty(size, dtype=torch.uint8, pin_memory=True)
hsrc.copy_(src.cpu())
cur = torch.cuda.current_stream()
cs = torch.cuda.Stream()
variants = [(h, "direct+host", bw) for h in ("ce", "sm") for bw in HOST_BWS] + \
    [("ce", "direct", 4e9)]
for host, paths, hbw in variants:
    if True:
        topo = mesh_text("b200_loopback", 2, 3.17e12, 1, 2e-6, hbw, 1e-5, "full")
        eng = Engine(load_topology(topo), [0, 0])
        eng.configure(host=host)
        cfg = PathConfig(1, paths == "direct+host", 8, True)
        bufs = [src, torch.empty_like(src)]
        landed = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        for ev in consumed:
            ev.record(cur)

        def run(n):
            for i in range(n):
                b = i % 2
                with torch.cuda.stream(cs):
                    cs.wait_event(consumed[b])
                    bufs[b].copy_(hsrc, non_blocking=True)
                    landed[b].record(cs)
                cur.wait_event(landed[b])
                for _ in range(W):
                    eng.send(bufs[b], dst, size, cfg, stream=cur, src_dev=0, dst_dev=1)
                consumed[b].record(cur)
        run(2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        cs.wait_event(e0)
        run(steps)
        e1.record(cur)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        # sends alone
        e0.record(cur)
        for _ in range(steps * W):
            eng.send(src, dst, size, cfg, stream=cur, src_dev=0, dst_dev=1)
        e1.record(cur)
        torch.cuda.synchronize()
        t2 = e0.elapsed_time(e1) / 1e3
        print(f"host={host} {paths} host_bw={hbw / 1e9:g}: e2e {steps * W * size / t / 1e9:.1f} GB/s, "
              f"sends alone {steps * W * size / t2 / 1e9:.1f} GB/s", flush=True)
        eng.close()
