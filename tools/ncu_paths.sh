#!/bin/bash
# Link-level evidence for one send configuration (tools/prof_kernel.py env):
# per launch of the transfer kernel its duration, DRAM bytes, PCIe bytes
# (the host-staged hops) and NVLink TX/RX bytes (peer paths, >= 2 GPUs),
# then a summary with achieved GB/s per link.  Usage (under gpurun, 1 process):
#   TAG=r02_headline PROF_BYTES=536870912 bash tools/ncu_paths.sh
#   TAG=r02_nvlink PROF_DEVICES=0,1 bash tools/ncu_paths.sh      # on a >= 2-GPU box
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
ncu --metrics $M --clock-control none -k regex:"transfer_kernel|small_copy" -s ${SKIP:-3} -c ${COUNT:-2} --csv \
    --log-file gpurun_out/${TAG:-paths}_ncu.csv python tools/prof_kernel.py > /dev/null 2>&1
python tools/ncu_paths_summary.py gpurun_out/${TAG:-paths}_ncu.csv gpurun_out/${TAG:-paths}_ncu.json
