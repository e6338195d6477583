mkdir -p gpurun_out _build
bash tools/gpu_tests.sh | tail -3
SMALL=4194304 MODES=2 ENGINE=tma ./_build/abi_latency 10000 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'engine' in d: print(d['engine'], d['mode'], d['bytes'], round(d['gpu_us_per_msg'],2), round(d['gbs'],1))
"
