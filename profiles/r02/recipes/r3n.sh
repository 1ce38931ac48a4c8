# ResNet-50 graph engine: bucket cap / first bucket sweep (defer on)
set -x
O=gpurun_out/r3n; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
for cfg in "12 1" "14 1" "16 1" "20 1" "12 1" "14 1" "16 1" "8 1"; do
set -- $cfg
timeout 600 $T --bucket-mb $1 --first-bucket-mb $2 --out $O/train_b$1_f$2.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/train_b$1_f$2.json').read().splitlines()[-1]); r=d['resnet50']
print('bucket=$1 first=$2', round(r['img_s']), round(r['ms_per_step'],2), r['replicas_agree'])"
done
