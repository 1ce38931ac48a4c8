#!/bin/bash
OUT=gpurun_out/r2d; mkdir -p $OUT
for cfg in "4 1" "2 1"; do
  set -- $cfg; tag=mr$1-ramp$2
  FMX_MIN_ROUNDS=$1 FMX_RAMP=$2 timeout 300 python bench.py --sweep --sweep-max 67108864 --out $OUT/sweep_$tag.jsonl > $OUT/sweep_$tag.log 2>&1; echo "sweep $tag rc=$?" >> $OUT/log.txt
  FMX_MIN_ROUNDS=$1 FMX_RAMP=$2 timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_$tag.json > $OUT/train_$tag.log 2>&1; echo "train $tag rc=$?" >> $OUT/log.txt
done
