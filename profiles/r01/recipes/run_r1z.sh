#!/bin/bash
# Size sweeps of reduce-scatter / all-gather / broadcast; DP legs (8 MiB buckets) with no-sync bound.
OUT=gpurun_out/r1z; mkdir -p $OUT
for op in reduce_scatter allgather broadcast; do
  timeout 400 python bench.py --sweep --sweep-op $op --out $OUT/sweep_${op}_n7.jsonl > $OUT/sweep_$op.log 2>&1; echo "sweep $op rc=$?" >> $OUT/log.txt
done
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
