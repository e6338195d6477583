"""NVLink probe for a box with >= 2 GPUs (the 1-GPU pool cannot run it):
GPU0 -> GPU1 bandwidth per message size for the copy engine (per-call
cudaMemcpyAsync = the reference's BASELINE_CONFIG), the LDG/STG peer kernel
(default), the TMA kernels on peer addresses (tma_peer=1), direct + host,
and direct + 1..N-2 GPU relays at 512 MiB (the NVSwitch ingress question).
One JSON line per measurement; byte-exactness checked on every arm.

    python tools/nvlink_probe.py [max_relays]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text  # noqa: E402

MiB = 1 << 20


def rate(eng, cfg, src, dst, n, reps):
    s = torch.cuda.Stream(device=0)
    for _ in range(3):
        eng.send(src[:n], dst[:n], n, cfg, stream=s, src_dev=0, dst_dev=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        eng.send(src[:n], dst[:n], n, cfg, stream=s, src_dev=0, dst_dev=1)
    e1.record(s)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    assert torch.equal(src[:n].to("cuda:1"), dst[:n]), "bytes differ"
    return reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        print(json.dumps({"unavailable": f"{ngpu} GPU visible; needs >= 2"}))
        return
    relays = min(int(sys.argv[1]) if len(sys.argv) > 1 else 6, ngpu - 2)
    n_log = 2 + relays
    text = mesh_text("probe", n_log, 7.7e11, 1, 2e-6, 5.5e10, 1e-5, "full")
    src = torch.randint(0, 256, (512 * MiB,), dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(512 * MiB, dtype=torch.uint8, device="cuda:1")
    arms = {"ce": dict(direct="ce"), "ldg_stg": {}, "tma_peer": dict(tma_peer=True)}
    for name, opts in arms.items():
        eng = Engine(load_topology(text), list(range(n_log)))
        if opts:
            eng.configure(**opts)
        cfg = PathConfig(max_chunks=1, graph_mode=name != "ce")
        for n in (64 << 10, MiB, 16 * MiB, 64 * MiB, 512 * MiB):
            reps = 200 if n <= 16 * MiB else 20
            print(json.dumps({"arm": name, "bytes": n, "gbs": rate(eng, cfg, src, dst, n, reps),
                              "kernel": eng.stats().kernel}), flush=True)
        eng.close()
    eng = Engine(load_topology(text), list(range(n_log)))
    for g in range(1, relays + 2):
        for host in (False, True):
            cfg = PathConfig(num_gpu_paths=g, host_path_enabled=host, max_chunks=8, graph_mode=True)
            print(json.dumps({"arm": "multi", "relays": g - 1, "host": host, "bytes": 512 * MiB,
                              "gbs": rate(eng, cfg, src, dst, 512 * MiB, 20)}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
