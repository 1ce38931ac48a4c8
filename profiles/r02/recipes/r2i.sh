# DP knobs: hook stream priority, reduce grid cap, bucket size
set -x
O=gpurun_out/r2i; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --out $O/train_base_1.json > /dev/null 2>&1
FMX_HOOK_PRIORITY=0 timeout 600 $T --out $O/train_prio0.json > /dev/null 2>&1
FMX_REDUCE_CTAS=40 timeout 600 $T --out $O/train_ctas40.json > /dev/null 2>&1
FMX_REDUCE_CTAS=160 timeout 600 $T --out $O/train_ctas160.json > /dev/null 2>&1
timeout 600 $T --bucket-mb 6 --out $O/train_b6.json > /dev/null 2>&1
timeout 600 $T --bucket-mb 12 --out $O/train_b12.json > /dev/null 2>&1
timeout 600 $T --out $O/train_base_2.json > /dev/null 2>&1
FMX_HOOK_PRIORITY=0 FMX_REDUCE_CTAS=40 timeout 600 $T --out $O/train_prio0_ctas40.json > /dev/null 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'])"; done
