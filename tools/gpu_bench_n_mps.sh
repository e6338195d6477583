#!/bin/bash
# group-mode bench with N ranks sharing the one visible GPU under MPS (kernels
# of different processes then run concurrently, as one rank per GPU would)
mkdir -p gpurun_out
which nvidia-cuda-mps-control || { echo "no MPS control binary"; exit 0; }
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "MPS started"
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for N in ${NS:-2 3 4}; do
# each rank gets 1/N of the SMs (MPS execution-resource provisioning): a
# relay rank's flag-waiting CTAs then cannot occupy the SMs the sender's
# CTAs need, as on separate GPUs
export CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=$((100 / N))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29${N}21 bench.py --gpus $N --steps 3 --warmup 3 --window 8 --size 67108864 > gpurun_out/bench_mps_n$N.json 2> gpurun_out/bench_mps_n$N.err; echo "N=$N rc=$?"; head -c 600 gpurun_out/bench_mps_n$N.json; echo; grep -i "error" gpurun_out/bench_mps_n$N.err | tail -2
done
echo quit | nvidia-cuda-mps-control
