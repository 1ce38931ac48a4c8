#!/bin/bash
# Hardware work queues per context (CUDA_DEVICE_MAX_CONNECTIONS) under MPS.
OUT=gpurun_out/r2s; mkdir -p $OUT
for c in 2 4 16 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_c$c.json > $OUT/bench_c$c.log 2>&1; echo "bench c$c rc=$?" >> $OUT/log.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_c$c.json > $OUT/train_c$c.log 2>&1; echo "train c$c rc=$?" >> $OUT/log.txt
done
