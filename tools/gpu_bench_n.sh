#!/bin/bash
# bench.py at N > 1 under torchrun on whatever GPUs the box has (ranks share
# GPU 0 when there are fewer GPUs than ranks: rank 0 drives every logical GPU
# of the node topology, mapped onto the visible devices).
mkdir -p gpurun_out
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for N in ${NS:-2 4 8}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29${N}31 bench.py --gpus $N --steps ${STEPS:-3} --warmup 3 --window ${WINDOW:-8} ${BENCH_ARGS:-} > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "N=$N rc=$?"; tail -c 400 gpurun_out/bench_n$N.json; echo; grep -i "error" gpurun_out/bench_n$N.err | tail -2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29${N}41 bench.py --impl reference --gpus $N --steps 1 --warmup 1 --window 2 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err; echo "ref N=$N rc=$?"; tail -c 300 gpurun_out/bench_ref_n$N.json; echo
done
