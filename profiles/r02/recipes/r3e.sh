# defaults after the bucket / engine change: BERT-base (graph, 25 MiB) and MobileNetV2 legs
set -x
O=gpurun_out/r3e; mkdir -p $O
timeout 600 python bench.py --train-only --train-model bert --train-no-sync --out $O/train_bert.json > $O/train_bert.log 2>&1
timeout 600 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $O/train_mobilenet_v2.json > $O/train_mnv2.log 2>&1
timeout 600 python bench.py --train-only --train-model mobilenet_v2 --out $O/train_mobilenet_v2_7.json > $O/train_mnv2_7.log 2>&1
for f in $O/train_*.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); k=list(d)[0]; r=d[k]; u=[x for x in r if x.endswith('_s')][0]
print('$f', k, round(r[u]), round(r['ms_per_step'],2), r['replicas_agree'], r['instances'], r.get('bucket_mb'), (r.get('no_sync') or {}).get(u))"; done
