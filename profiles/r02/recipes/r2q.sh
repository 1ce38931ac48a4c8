# DP training with the whole step captured as one CUDA graph (ddp.ShmDataParallel) vs eager DDP
set -x
O=gpurun_out/r2q; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --out $O/train_graph.json > $O/train_graph.log 2>&1
timeout 600 $T --train-no-sync --out $O/train_graph_ns.json > $O/train_graph_ns.log 2>&1
timeout 600 $T --train-engine ddp --out $O/train_ddp.json > $O/train_ddp.log 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'], r.get('no_sync',{}).get('img_s'))"; done
tail -5 $O/train_graph.log
