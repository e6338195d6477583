#!/bin/bash
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
python tools/prof_sizes.py > gpurun_out/sizes_tma.jsonl 2>&1
ENGINE_OPTS='{"copy": "vec", "unroll": 4, "ctas_per_sm": 4, "threads": 256}' python tools/prof_sizes.py > gpurun_out/sizes_vec.jsonl 2>&1
ENGINE_OPTS='{"direct": "ce"}' python tools/prof_sizes.py > gpurun_out/sizes_ce.jsonl 2>&1
SIZES=33554432 REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:transfer_kernel -s 4 -c 1 -o gpurun_out/transfer_32m python tools/prof_sizes.py > /dev/null 2>&1
echo "tma"; cat gpurun_out/sizes_tma.jsonl; echo vec; cat gpurun_out/sizes_vec.jsonl; echo ce; cat gpurun_out/sizes_ce.jsonl
