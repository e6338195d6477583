#!/bin/bash
# host cost per send: plain-C ABI consumer (3 engine variants) + Python layers
mkdir -p gpurun_out _build
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/abi_latency.cu -o _build/abi_latency \
  -L paper_2604_22228_b200 -lmpb200 -Xlinker -rpath,'$ORIGIN/../paper_2604_22228_b200' || exit 1
out=gpurun_out/abi_latency${TAG:-}.jsonl; : > $out
for v in tma vec ce; do ENGINE=$v timeout 300 ./_build/abi_latency ${ITERS:-10000} | tee -a $out; done
for v in tma vec; do SCHED=dynamic ENGINE=$v timeout 300 ./_build/abi_latency ${ITERS:-10000} | tee -a $out; done
[ -n "${NOPY:-}" ] || timeout 300 python tools/py_latency.py ${ITERS:-10000} | tee gpurun_out/py_latency${TAG:-}.jsonl
