mkdir -p gpurun_out _build
bash tools/gpu_tests.sh | tail -3
for v in default ring peer; do MODES=2 ENGINE=$v ./_build/abi_latency 10000 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'engine' in d: print(d['engine'], d['mode'], d['bytes'], round(d['gpu_us_per_msg'],2), round(d['gbs'],1))
"; done
