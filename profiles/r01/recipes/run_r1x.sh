#!/bin/bash
# DDP hook on a side stream: parity, then the three DP legs.
OUT=gpurun_out/r1x; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
