#!/bin/bash
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/exp_host2.py > gpurun_out/exp_host2.jsonl 2>&1; cat gpurun_out/exp_host2.jsonl
timeout 600 python -m pytest tests -m gpu -q -x -k "relays or war or trace or concurrent" 2>&1 | tail -2
