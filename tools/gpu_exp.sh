#!/bin/bash
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python tools/exp_kernel.py > gpurun_out/exp_kernel.log 2>&1; echo "exp rc=$?"
tail -3 gpurun_out/exp_kernel.log
