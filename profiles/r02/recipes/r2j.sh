# DP: hardware work-queue aliasing hypothesis (CUDA_DEVICE_MAX_CONNECTIONS), no extra lane streams
set -x
O=gpurun_out/r2j; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
timeout 600 $T --out $O/train_base_1.json > /dev/null 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 600 $T --out $O/train_cdmc8.json > $O/train_cdmc8.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=16 timeout 600 $T --out $O/train_cdmc16.json > $O/train_cdmc16.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=4 timeout 600 $T --out $O/train_cdmc4.json > $O/train_cdmc4.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 600 $T --out $O/train_cdmc1.json > $O/train_cdmc1.log 2>&1
FMX_LANES=1 timeout 600 $T --out $O/train_lanes1.json > /dev/null 2>&1
timeout 600 $T --train-no-sync --out $O/train_base_nosync.json > /dev/null 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'], r.get('no_sync',{}).get('ms_per_step'))"; done
