#!/bin/bash
# compute-sanitizer over a small multi-path workload (relays + host, TMA and VEC)
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
cat > /tmp/san_work.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2604_22228_b200 as mp
text = mp.mesh_text("s", 4, 2e12, 1, 2e-6, 40e9, 1e-5, "full")
for copy in ("tma", "vec"):
    for host in ("ce", "sm"):
        eng = mp.Engine(mp.load_topology(text), [0] * 4)
        eng.configure(copy=copy, host=host)
        n = (2 << 20) + 7
        src = torch.randint(0, 256, (n + 5,), dtype=torch.uint8, device="cuda")[5:]
        dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
        for graph in (False, True):
            cfg = mp.PathConfig(num_gpu_paths=3, host_path_enabled=True, max_chunks=4, graph_mode=graph)
            for _ in range(2):
                eng.send(src, dst, n, cfg, src_dev=0, dst_dev=1)
        eng.sync()
        assert torch.equal(src, dst), (copy, host)
        eng.close()
print("workload ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=transfer_kernel --print-limit 20 python /tmp/san_work.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
