# BASELINE configs' DP legs at their own rank splits on logical GPUs of ONE B200 (functional:
# the multi-GPU communicator, rank order and training path; not scaling numbers):
# C3 MobileNetV2 4 instances 2+2, C4 BERT-base bf16 14 instances 7+7
set -x
O=gpurun_out/r3y; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29677"
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 900 $TR bench.py --gpus 2 --ranks-per-gpu 2 --train-only --train-model mobilenet_v2 --train-steps 5 --train-warmup 3 --out $O/train_c3.json > $O/train_c3.log 2>&1; echo "c3 rc=$?" >> $O/log.txt
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 1200 $TR bench.py --gpus 2 --ranks-per-gpu 7 --train-only --train-model bert --train-steps 5 --train-warmup 3 --out $O/train_c4.json > $O/train_c4.log 2>&1; echo "c4 rc=$?" >> $O/log.txt
cat $O/log.txt
for f in $O/train_c3.json $O/train_c4.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); k=list(d)[0]; r=d[k]; u=[x for x in r if x.endswith('_s')][0]
print('$f', k, round(r[u]), round(r['ms_per_step'],2), r['replicas_agree'], r['instances'], r.get('n_gpus'))"; done
tail -n 3 $O/train_c4.log | cut -c1-300
