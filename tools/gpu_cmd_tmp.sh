bash tools/gpu_tests.sh | tail -3
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/abi_latency.cu -o _build/abi_latency -L paper_2604_22228_b200 -lmpb200 -Xlinker -rpath,'$ORIGIN/../paper_2604_22228_b200'
MODES=3 ./_build/abi_latency 10000 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'engine' in d and d['mode']=='single_stream': print(d['mode'], d['bytes'], round(d['gpu_us_per_msg'],2), round(d['host_us_mean'],2))
"
