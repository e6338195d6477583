#!/bin/bash
# one gpurun call: build check, GPU tests, smoke, short bench, launch list
set -x
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/smoke.log | tail -3
cat gpurun_out/bench.json | head -c 3000
