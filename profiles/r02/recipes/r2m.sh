# DP host-side breakdown: where does the exchanging step's extra host enqueue time go?
# + ZC load/store contention probe
set -x
O=gpurun_out/r2m; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --out $O/train_sync.json > $O/train_sync.log 2>&1
FMX_HOOK_NOOP=1 timeout 600 $T --out $O/train_noop1.json > /dev/null 2>&1
FMX_HOOK_NOOP=2 timeout 600 $T --out $O/train_noop2.json > /dev/null 2>&1
FMX_HOOK_THREAD=1 timeout 600 $T --out $O/train_thread.json > /dev/null 2>&1
timeout 120 python tools/probe_zc_contention.py > $O/probe_zc_full.jsonl 2>&1
CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=14 timeout 120 python tools/with_mps.py python tools/probe_zc_contention.py > $O/probe_zc_mps14.jsonl 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'], r.get('host'))"; done
cat $O/probe_zc_*.jsonl
