# BERT-base DP graph engine knobs (defer, bucket sizes) vs eager DDP
set -x
O=gpurun_out/r3c; mkdir -p $O
T="python bench.py --train-only --train-model bert --train-engine graph"
FMX_DEFER=0 timeout 600 $T --out $O/train_nodefer.json > /dev/null 2>&1
timeout 600 $T --bucket-mb 25 --out $O/train_b25.json > /dev/null 2>&1
timeout 600 $T --first-bucket-mb 8 --out $O/train_fb8.json > /dev/null 2>&1
timeout 600 python bench.py --train-only --train-model bert --train-engine ddp --out $O/train_ddp.json > /dev/null 2>&1
for f in $O/train_*.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['bert']
print('$f', r['seq_s'], r['ms_per_step'], r['replicas_agree'])"; done
