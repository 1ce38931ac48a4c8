# DP: which part of the exchange slows the backward pass on the GPU?  copy-engine traffic
# alone (noop=3) vs the reduction kernels alone (noop=4), against no exchange (noop=1)
set -x
O=gpurun_out/r2n; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
FMX_HOOK_NOOP=1 timeout 600 $T --out $O/train_noop1.json > /dev/null 2>&1
FMX_HOOK_NOOP=3 timeout 600 $T --out $O/train_noop3.json > $O/train_noop3.log 2>&1
FMX_HOOK_NOOP=4 timeout 600 $T --out $O/train_noop4.json > $O/train_noop4.log 2>&1
timeout 600 $T --out $O/train_sync.json > /dev/null 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['host'])"; done
tail -3 $O/train_noop3.log
