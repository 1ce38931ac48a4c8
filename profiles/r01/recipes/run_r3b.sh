#!/bin/bash
# Copy fence on by default: GPU suite, default bench, DP legs, bucketed probe, sweep.
OUT=gpurun_out/r3b; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json --stamps $OUT/stamps.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --out $OUT/bench_b13.json > $OUT/bench_b13.log 2>&1; echo "b13 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --out $OUT/sweep_n7.jsonl > $OUT/sweep_n7.log 2>&1; echo "sweep rc=$?" >> $OUT/log.txt
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
