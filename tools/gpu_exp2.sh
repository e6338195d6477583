#!/bin/bash
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/exp_host.py > gpurun_out/exp_host.log 2>&1; echo "exp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:transfer_kernel -s 2 -c 1 -o gpurun_out/transfer_512m python tools/prof_kernel.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python tools/prof_kernel.py > /dev/null 2>&1; echo "ncu list rc=$?"
