# ResNet-50 graph engine: cap the LAST bucket (the step's tail) instead of the first
set -x
O=gpurun_out/r4m; mkdir -p $O
run() {  # tag env
  env $2 timeout 600 python bench.py --train-only --train-model resnet50 --out $O/$1.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['resnet50']
print('$1', round(r['img_s']), round(r['ms_per_step'],2), r['replicas_agree'])"
}
for rep in 1 2; do
run def_$rep FMX_X=0
run last1_$rep FMX_LAST_BUCKET_MB=1
run last2_$rep FMX_LAST_BUCKET_MB=2
run last4_$rep FMX_LAST_BUCKET_MB=4
done
