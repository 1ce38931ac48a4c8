# the SGD step fused into the collective vs torch's optimizer after it (graph engine)
set -x
O=gpurun_out/r4b; mkdir -p $O
run() {  # tag args
  timeout 600 python bench.py --train-only $2 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); k=list(d)[0]; r=d[k]; u=[x for x in r if x.endswith('_s')][0]
print('$1', k, round(r[u]), round(r['ms_per_step'],2), r['replicas_agree'], r['optimizer'])"
}
for rep in 1 2; do
run r50_$rep "--train-model resnet50"
run r50_fused_$rep "--train-model resnet50 --fused-sgd"
run mnv2_$rep "--train-model mobilenet_v2 --ranks-per-gpu 4"
run mnv2_fused_$rep "--train-model mobilenet_v2 --ranks-per-gpu 4 --fused-sgd"
done
tail -n 3 $O/r50_fused_1.log | cut -c1-300
