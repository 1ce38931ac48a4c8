#!/bin/bash
# Pipeline depth for DDP buckets (join-stream overlap): slots x bucket size.
OUT=gpurun_out/r2m; mkdir -p $OUT
for cfg in "2 8" "3 8" "4 8" "4 4" "4 16"; do
  set -- $cfg; tag=s$1-b$2
  FMX_SLOTS=$1 timeout 400 python bench.py --train-only --train-model resnet50 --bucket-mb $2 --out $OUT/train_r50_$tag.json > $OUT/train_r50_$tag.log 2>&1; echo "train r50 $tag rc=$?" >> $OUT/log.txt
done
FMX_SLOTS=4 timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_s4.json > $OUT/train_bert_s4.log 2>&1; echo "train bert s4 rc=$?" >> $OUT/log.txt
FMX_SLOTS=4 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_s4.json > $OUT/bench_s4.log 2>&1; echo "bench s4 rc=$?" >> $OUT/log.txt
