mkdir -p gpurun_out _build
python paper_2604_22228_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
for cfg in "65536 4 8" "131072 4 8" "262144 4 8" "131072 2 8" "131072 4 4" "262144 2 16" "131072 3 8" "524288 4 8"; do set -- $cfg
MP_TAIL_PIECE=0 TILE=$1 CTAS=$2 UNROLL=$3 MODES=1 ./_build/abi_latency 10000 | python -c "
import json,sys
out=[]
for l in sys.stdin:
    d=json.loads(l)
    if 'engine' in d and d['bytes']>=(16<<20): out.append('%d:%.2f' % (d['bytes']>>20, d['gpu_us_per_msg']))
print('tile $1 ctas $2 unroll $3', ' '.join(out))
"; done
