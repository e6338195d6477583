#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, the default bench line
# and the reference arm, the ncu launch list of the bench's headline windows,
# one ncu --set full capture of the headline send's dominant kernel (planned
# on the bench's topology) and its link-level DRAM / PCIe bytes.
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
export PROF_TOPO=topologies/b200_loopback.topo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:transfer_kernel -s 2 -c 1 \
    -o gpurun_out/headline_512m python tools/prof_kernel.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/headline_512m.ncu-rep gpurun_out/transfer_kernel_ncu.json > /dev/null 2>&1; echo "summary rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --quick --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench list rc=$?"
TAG=headline_paths PROF_BYTES=536870912 timeout 300 bash tools/ncu_paths.sh; echo "ncu paths rc=$?"
