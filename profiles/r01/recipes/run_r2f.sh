#!/bin/bash
# AUTO transport per collective (ZC <= 4 MiB, CE above): parity, sweep, DP legs.
OUT=gpurun_out/r2f; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --out $OUT/sweep_auto.jsonl > $OUT/sweep_auto.log 2>&1; echo "sweep rc=$?" >> $OUT/log.txt
for b in 4 8; do
  timeout 400 python bench.py --train-only --train-model resnet50 --bucket-mb $b --out $OUT/train_r50_b$b.json > $OUT/train_r50_b$b.log 2>&1; echo "train r50 b$b rc=$?" >> $OUT/log.txt
done
FMX_ZC_MAX=16777216 timeout 400 python bench.py --train-only --train-model resnet50 --bucket-mb 8 --out $OUT/train_r50_b8_zc16.json > $OUT/train_r50_b8_zc16.log 2>&1; echo "train r50 b8 zc16 rc=$?" >> $OUT/log.txt
