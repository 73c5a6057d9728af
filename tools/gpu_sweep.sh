#!/bin/bash
# p sweep + per-kernel split. usage: bash tools/gpu_sweep.sh <tag> "<cfg:p cfg:p ...>"
T=${1:-v}; LIST=${2:-"c3:4 c3:8 c3:16 c4:4 c4:8 c4:16 c2:8 c5:16"}
mkdir -p gpurun_out
for cp in $LIST; do
  c=${cp%%:*}; p=${cp##*:}
  timeout 900 python bench.py --config $c --p $p --steps 5 --warmup 3 --no-cpu --no-e2e $BARGS > gpurun_out/sweep_${c}_p${p}$T.json 2> gpurun_out/sweep_${c}_p${p}$T.err
  python - "$c p$p" "gpurun_out/sweep_${c}_p${p}$T.json" <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[2]) if l.startswith('{')][-1])
    r=d['roofline']
    ks=' '.join('%s %.3fms %.2f'%(k['kernel'],k['ms'],k['frac']) for k in r['kernels'])
    print(sys.argv[1], 'ms %.3f'%d['ms_per_step'], 'Eps %.3e'%d['value'], 'items', r['items'], ks, d.get('parity',{}).get('match'))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
done
