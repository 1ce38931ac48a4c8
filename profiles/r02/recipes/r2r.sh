# graph engine: strided bucket views; GPU-clock timeline of one replayed step; other models
set -x
O=gpurun_out/r2r; mkdir -p $O
timeout 500 python -m pytest tests/test_graph_dp_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
T="python bench.py --train-only"
timeout 600 $T --train-model resnet50 --train-no-sync --out $O/train_resnet50.json > $O/train_resnet50.log 2>&1
FMX_HOOK_STAMP=1 timeout 600 $T --train-model resnet50 --stamps $O/stamps_graph.json --out $O/train_stamps.json > $O/train_stamps.log 2>&1
timeout 600 $T --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $O/train_mobilenet_v2.json > $O/train_mnv2.log 2>&1
timeout 600 $T --train-model bert --train-no-sync --out $O/train_bert.json > $O/train_bert.log 2>&1
for f in $O/train_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); k=list(d)[0]; r=d[k]; u=[x for x in r if x.endswith('_s')][0]
print(k, r[u], r['ms_per_step'], r['replicas_agree'], (r.get('no_sync') or {}).get(u))"; done
tail -3 $O/pytest.log; tail -3 $O/train_bert.log
