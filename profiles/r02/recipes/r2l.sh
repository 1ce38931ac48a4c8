# DP: host enqueue time; bucket readiness on the GPU clock with and without the exchange
set -x
O=gpurun_out/r2l; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --out $O/train_base.json > $O/train_base.log 2>&1
FMX_HOOK_STAMP=1 timeout 600 $T --stamps $O/stamps_sync.json --out $O/train_st_sync.json > /dev/null 2>&1
FMX_HOOK_STAMP=1 FMX_HOOK_NOOP=1 timeout 600 $T --stamps $O/stamps_noop.json --out $O/train_st_noop.json > /dev/null 2>&1
FMX_HOOK_NOOP=1 timeout 600 $T --out $O/train_noop.json > /dev/null 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'], r.get('host'))"; done
