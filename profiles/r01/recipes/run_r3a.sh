#!/bin/bash
OUT=gpurun_out/r3a; mkdir -p $OUT
for nop in 3 5; do
FMX_NOP=$nop timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --out $OUT/bench_b13_nop$nop.json > $OUT/bench_b13_nop$nop.log 2>&1; echo "b13 nop$nop rc=$?" >> $OUT/log.txt
done
for nop in 2 3; do
FMX_NOP=$nop timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_nop$nop.json > $OUT/bench_nop$nop.log 2>&1; echo "plain nop$nop rc=$?" >> $OUT/log.txt
FMX_NOP=$nop timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_nop$nop.json > $OUT/train_r50_nop$nop.log 2>&1; echo "r50 nop$nop rc=$?" >> $OUT/log.txt
FMX_NOP=$nop timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_nop$nop.json > $OUT/train_bert_nop$nop.log 2>&1; echo "bert nop$nop rc=$?" >> $OUT/log.txt
done
