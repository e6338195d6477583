#!/bin/bash
# exp_linkcap.py under MPS at several SM percentages (a link-limited direct
# path beside uncapped copy engines); MPS is stopped at the end
mkdir -p gpurun_out
which nvidia-cuda-mps-control || { echo "no MPS control binary"; exit 0; }
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
nvidia-cuda-mps-control -d && echo "MPS started"
rm -f gpurun_out/exp_linkcap.jsonl
for p in ${PCTS:-10 20 35 100}; do
  CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=$p timeout 300 python tools/exp_linkcap.py 2> gpurun_out/exp_linkcap_$p.err || tail -3 gpurun_out/exp_linkcap_$p.err
done
echo quit | nvidia-cuda-mps-control
