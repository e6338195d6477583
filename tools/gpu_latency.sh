#!/bin/bash
# Per-message GPU time and host cost per send: the plain-C ABI consumer
# (tools/abi_latency.cu) over engine variants, the launch-slot probe
# (tools/kexp.cu), and the Python layers (tools/py_latency.py).
mkdir -p gpurun_out _build
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/abi_latency.cu -o _build/abi_latency \
  -L paper_2604_22228_b200 -lmpb200 -Xlinker -rpath,'$ORIGIN/../paper_2604_22228_b200' || exit 1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -I paper_2604_22228_b200/csrc \
  tools/kexp.cu -o _build/kexp || exit 1
out=gpurun_out/abi_latency${TAG:-}.jsonl; : > $out
for v in default ring peer ce; do ENGINE=$v timeout 300 ./_build/abi_latency ${ITERS:-10000} >> $out; done
SCHED=dynamic SMALL=0 timeout 300 ./_build/abi_latency ${ITERS:-10000} >> $out
timeout 300 ./_build/kexp > gpurun_out/launch_slots${TAG:-}.txt
[ -n "${NOPY:-}" ] || timeout 300 python tools/py_latency.py ${ITERS:-10000} > gpurun_out/py_latency${TAG:-}.jsonl
echo done
