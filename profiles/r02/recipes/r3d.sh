# graph engine: defer x bucket size, BERT-base and ResNet-50
set -x
O=gpurun_out/r3d; mkdir -p $O
for m in bert resnet50; do for d in 0 1; do for b in 25 50; do
FMX_DEFER=$d timeout 600 python bench.py --train-only --train-model $m --train-engine graph --bucket-mb $b --out $O/train_${m}_d${d}_b${b}.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/train_${m}_d${d}_b${b}.json').read().splitlines()[-1]); r=d['$m']; u=[k for k in r if k.endswith('_s')][0]
print('$m defer=$d bucket=$b', round(r[u]), round(r['ms_per_step'],2), r['replicas_agree'])"
done; done; done
