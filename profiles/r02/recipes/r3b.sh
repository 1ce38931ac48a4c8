# BERT-base DP graph engine with the fused AdamW
set -x
O=gpurun_out/r3b; mkdir -p $O
T="python bench.py --train-only --train-model bert"
timeout 600 $T --train-engine graph --train-no-sync --out $O/train_bert_graph.json > $O/train_bert_graph.log 2>&1
for f in $O/train_*.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['bert']
print('$f', r['seq_s'], r['ms_per_step'], r['replicas_agree'], (r.get('no_sync') or {}).get('seq_s'))"; done
tail -n 3 $O/train_bert_graph.log | cut -c1-300
