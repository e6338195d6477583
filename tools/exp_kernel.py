"""GPU experiment: transfer-kernel shape sweep + host-path pipeline analysis.

Prints one JSON object per line into gpurun_out/exp_kernel.jsonl.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

MiB = 1 << 20
out = open("gpurun_out/exp_kernel.jsonl", "w")


def emit(**kw):
    print(json.dumps(kw), flush=True)
    out.write(json.dumps(kw) + "\n")
    out.flush()


S = 512 * MiB
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
stream = torch.cuda.Stream()


def kernel_rate(eng, cfg, size=S, reps=6):
    ts = []
    for _ in range(reps):
        eng.send(src[:size], dst[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
        ts.append(eng.kernel_time_ms())
    eng.sync()
    assert torch.equal(src[:size], dst[:size])
    t = sorted(ts[1:])[len(ts[1:]) // 2]
    return size / (t / 1e3) / 1e9, t


def send_rate(eng, cfg, size=S, reps=10):
    for _ in range(3):
        eng.send(src[:size], dst[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        eng.send(src[:size], dst[:size], size, cfg, stream=stream, src_dev=0, dst_dev=1)
    e1.record(stream)
    torch.cuda.synchronize()
    assert torch.equal(src[:size], dst[:size])
    return size * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


single = PathConfig(max_chunks=1, graph_mode=False)
eng = Engine.loopback(2)
eng.set_kernel_timing(True)

# 1. vec variants
for unroll in (4, 8, 16):
    for ctas in (1, 2, 4):
        if unroll == 16 and ctas > 1:
            continue
        for tile in (64 << 10, 256 << 10, 0):
            for threads in (128, 256):
                try:
                    eng.configure(copy="vec", unroll=unroll, ctas_per_sm=ctas, tile_bytes=tile,
                                  threads=threads)
                    gbs, ms = kernel_rate(eng, single)
                    emit(exp="vec", unroll=unroll, ctas=ctas, tile=tile, threads=threads,
                         gbs=gbs, ms=ms)
                except Exception as e:  # noqa: BLE001
                    emit(exp="vec", unroll=unroll, ctas=ctas, tile=tile, threads=threads,
                         error=str(e))
# 2. TMA variants
for stages, block in ((4, 32768), (6, 32768), (4, 49152), (8, 16384), (3, 65536), (2, 65536)):
    for ctas in (1, 2):
        if stages * block * ctas > 200 * 1024:
            continue
        for tile in (256 << 10, 1 << 20, 0):
            try:
                eng.configure(copy="tma", tma_stages=stages, tma_block=block, ctas_per_sm=ctas,
                              tile_bytes=tile, threads=128)
                gbs, ms = kernel_rate(eng, single)
                emit(exp="tma", stages=stages, block=block, ctas=ctas, tile=tile, gbs=gbs, ms=ms)
            except Exception as e:  # noqa: BLE001
                emit(exp="tma", stages=stages, block=block, ctas=ctas, tile=tile, error=str(e))
# 3. CE direct
eng.configure(direct="ce", copy="vec", unroll=8, ctas_per_sm=2, tile_bytes=0, threads=256)
emit(exp="ce_direct", gbs=send_rate(eng, single))
eng.configure(direct="sm")
emit(exp="sm_direct_graph", gbs=send_rate(eng, PathConfig(max_chunks=1, graph_mode=True)))

# 4. host path: isolated and concurrent copies
h = torch.empty(64 * MiB, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(64 * MiB, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for nbytes in (1 * MiB, 9 * MiB, 64 * MiB):
    def t(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps
    d2h = t(lambda: h[:nbytes].copy_(src[:nbytes], non_blocking=True))
    h2d = t(lambda: dst[:nbytes].copy_(h[:nbytes], non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            h[:nbytes].copy_(src[:nbytes], non_blocking=True)
        with torch.cuda.stream(s2):
            dst[:nbytes].copy_(h2[:nbytes], non_blocking=True)
    bd = t(both)
    emit(exp="pcie", bytes=nbytes, d2h_gbs=nbytes / d2h / 1e9, h2d_gbs=nbytes / h2d / 1e9,
         concurrent_each_gbs=nbytes / bd / 1e9)

# 5. multi-path direct+host at several host link bandwidths (shares)
from paper_2604_22228_b200 import load_topology, mesh_text  # noqa: E402
for host_bw in (20e9, 40e9, 55e9):
    for k in (4, 8, 16, 32):
        topo = load_topology(mesh_text("x", 2, 3.1e12, 1, 2e-6, host_bw, 1e-5, "full"))
        e2 = Engine(topo, [0, 0])
        cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=k, graph_mode=True)
        emit(exp="multi", host_bw=host_bw, k=k, gbs=send_rate(e2, cfg))
        e2.configure(direct="ce")
        emit(exp="multi_ce", host_bw=host_bw, k=k, gbs=send_rate(e2, cfg))
        e2.close()
out.close()
