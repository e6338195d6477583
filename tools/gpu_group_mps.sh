#!/bin/bash
# tools/exp_group_mps.py: 2 ranks (one per logical GPU) sharing the one B200
# under MPS, each provisioned half the SMs; MPS is stopped at the end
mkdir -p gpurun_out
which nvidia-cuda-mps-control || { echo "no MPS control binary"; exit 0; }
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
nvidia-cuda-mps-control -d && echo "MPS started"
export CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=${PCT:-50}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${WORLD:-2} --master-addr 127.0.0.1 \
    --master-port 29581 tools/exp_group_mps.py > gpurun_out/exp_group_mps.jsonl 2> gpurun_out/exp_group_mps.err
echo "rc=$?"; cat gpurun_out/exp_group_mps.jsonl; grep -iE "error|Traceback" gpurun_out/exp_group_mps.err | tail -3
echo quit | nvidia-cuda-mps-control
