#!/bin/bash
# Everything a >= 2-GPU B200 node would settle, in one run:
# the real-peer GPU tests, the bench at N = 2 / 4 / 8 (as many as the node
# has) with the reference arm, the NVLink per-size probe (CE vs LDG/STG vs
# TMA on peers, relay sweep), and the ncu NVLink / PCIe / DRAM bytes of a
# GPU0 -> GPU1 send.  Outputs land in gpurun_out/; on the 1-GPU pool it
# exits after saying so.
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
if [ "$NG" -lt 2 ]; then echo "one GPU visible: nothing to settle here"; exit 0; fi
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -2 gpurun_out/multi_tests.log
NS=""; for n in 2 4 8; do [ "$n" -le "$NG" ] && NS="$NS $n"; done
WINDOW=64 STEPS=10 NS="$NS" bash tools/gpu_bench_n.sh
timeout 900 python tools/nvlink_probe.py > gpurun_out/nvlink_probe.txt 2>&1; echo "nvlink probe rc=$?"
TAG=nvlink_paths PROF_DEVICES=0,1 PROF_BYTES=536870912 timeout 600 bash tools/ncu_paths.sh; echo "ncu paths rc=$?"
