#!/bin/bash
# torchrun N=2 orchestration on one B200 (two logical GPUs x 5 ranks: the reference caps a bus at 10); DDP bucket size.
OUT=gpurun_out/r1y; mkdir -p $OUT
FMX_DEVICE_MAP=0,0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --ranks-per-gpu 5 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_n2.log 2>&1; echo "torchrun n2 rc=$?" >> $OUT/log.txt
for b in 5 8 15; do
  timeout 600 python bench.py --train-only --train-model resnet50 --bucket-mb $b --out $OUT/train_r50_b$b.json > $OUT/train_r50_b$b.log 2>&1; echo "train r50 b$b rc=$?" >> $OUT/log.txt
done
timeout 600 python bench.py --train-only --train-model bert --bucket-mb 10 --out $OUT/train_bert_b10.json > $OUT/train_bert_b10.log 2>&1; echo "train bert b10 rc=$?" >> $OUT/log.txt
