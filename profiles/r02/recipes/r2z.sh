# graph engine decomposition: no exchange / copy-engine traffic only / full exchange
set -x
O=gpurun_out/r2z; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --train-no-sync --out $O/train_full.json > /dev/null 2>&1
FMX_HOOK_NOOP=3 timeout 600 $T --out $O/train_noop3.json > $O/train_noop3.log 2>&1
for f in $O/train_*.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']
print('$f', r['img_s'], r['ms_per_step'], r['replicas_agree'], (r.get('no_sync') or {}).get('ms_per_step'))"; done
tail -n 2 $O/train_noop3.log | cut -c1-300
