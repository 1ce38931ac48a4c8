#!/bin/bash
OUT=gpurun_out/r2n; mkdir -p $OUT
for m in resnet50 bert; do for b in 4 8; do
  timeout 600 python bench.py --train-only --train-model $m --bucket-mb $b --out $OUT/train_${m}_b$b.json > $OUT/train_${m}_b$b.log 2>&1; echo "train $m b$b rc=$?" >> $OUT/log.txt
done; done
