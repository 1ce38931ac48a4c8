#!/bin/bash
OUT=gpurun_out/r2z; mkdir -p $OUT
for nop in 0 1 2; do
FMX_NOP=$nop timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --out $OUT/bench_b13_nop$nop.json > $OUT/bench_b13_nop$nop.log 2>&1; echo "b13 nop$nop rc=$?" >> $OUT/log.txt
done
FMX_NOP=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_nop1.json > $OUT/bench_nop1.log 2>&1; echo "plain nop1 rc=$?" >> $OUT/log.txt
FMX_NOP=1 timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_nop1.json > $OUT/train_r50_nop1.log 2>&1; echo "r50 nop1 rc=$?" >> $OUT/log.txt
