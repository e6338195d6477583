#!/bin/bash
# group-mode bench with N ranks sharing the one visible GPU (IPC path check)
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for N in 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29${N}11 bench.py --gpus $N --steps 3 --warmup 3 --window 8 --size 67108864 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "N=$N rc=$?"; cat gpurun_out/bench_n$N.json | head -c 700; echo; tail -3 gpurun_out/bench_n$N.err
done
