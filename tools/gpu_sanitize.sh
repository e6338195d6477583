#!/bin/bash
# compute-sanitizer over a small multi-path workload: relays + host (TMA and
# LDG/STG, CE and SM host paths), the small-message, static-TMA and dynamic
# kernels, the forced peer path; graph and streamed mode
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
cat > /tmp/san_work.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2604_22228_b200 as mp
text = mp.mesh_text("s", 4, 2e12, 1, 2e-6, 40e9, 1e-5, "full")
MiB = 1 << 20
# (engine options, gpu paths, host, size): relay + host tables (dynamic
# claims, flag waits) with both dynamic kernels and both host mechanisms;
# direct-only tables on the small-message kernel, the static TMA table and
# the dynamic LDG/STG kernel; the forced peer launch path
cases = [(dict(copy=copy, host=host), 3, True, 2 * MiB + 7)
         for copy in ("tma", "vec") for host in ("ce", "sm")]
cases += [({}, 1, False, 4096 + 3), ({}, 1, False, 3 * MiB + 5), ({}, 1, False, 24 * MiB + 9),
          (dict(sched="dynamic"), 1, False, 24 * MiB + 9), (dict(tma_peer=-1), 2, True, 5 * MiB + 1)]
# round 2: host roundtrip tiles (calibrated-small host share) on the static
# TMA table's helper warps and on dynamic tables, with and without relays
small = mp.mesh_text("s1", 4, 2e12, 1, 2e-6, 1e9, 1e-5, "full")
cases += [(dict(host="sm", _topo=small), 1, True, 24 * MiB + 9),
          (dict(host="sm", sched="dynamic", _topo=small), 1, True, 24 * MiB + 9),
          (dict(host="auto", _topo=small), 3, True, 6 * MiB + 3),
          (dict(host="sm", copy="tma", _topo=small), 2, True, 130 * MiB + 1)]
for opts, g, host, n in cases:
    opts = dict(opts)
    eng = mp.Engine(mp.load_topology(opts.pop("_topo", text)), [0] * 4)
    eng.configure(**opts)
    src = torch.randint(0, 256, (n + 5,), dtype=torch.uint8, device="cuda")[5:]
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    for graph in (False, True):
        cfg = mp.PathConfig(num_gpu_paths=g, host_path_enabled=host, max_chunks=4, graph_mode=graph)
        for _ in range(2):
            eng.send(src, dst, n, cfg, src_dev=0, dst_dev=1)
    eng.sync()
    assert torch.equal(src, dst), (opts, g, host, n)
    print(opts, g, host, n, eng.stats().kernel, flush=True)
    eng.close()
print("workload ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_work.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
