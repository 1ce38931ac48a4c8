# DP train leg at the north_star's 4-GPU shape on ONE B200: 28 instance ranks over 4 torchrun
# processes (4 logical GPUs) - functional check of the multi-GPU training path, NOT a scaling number
set -x
O=gpurun_out/r3o; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655"
FMX_DEVICE_MAP=0,0,0,0 FMX_FAKE_BUS=1 timeout 1200 $TR bench.py --gpus 4 --train-only --train-model resnet50 --train-steps 5 --train-warmup 3 --out $O/train_4lgpu.json > $O/train_4lgpu.log 2>&1; echo "rc=$?" >> $O/train_4lgpu.log
python -c "
import json; d=json.loads(open('$O/train_4lgpu.json').read().splitlines()[-1]); r=d['resnet50']
print('28 ranks', r['img_s'], r['ms_per_step'], r['replicas_agree'], r['instances'], r['n_gpus'])"
tail -n 3 $O/train_4lgpu.log | cut -c1-400
