#!/bin/bash
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/exp_smhost.py > gpurun_out/exp_smhost.jsonl 2>&1; cat gpurun_out/exp_smhost.jsonl
timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or probe_node" 2>&1 | tail -3
