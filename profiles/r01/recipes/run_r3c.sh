#!/bin/bash
# Same-box A/B of the copy fence in DP training (box-to-box variance is ~5%).
OUT=gpurun_out/r3c; mkdir -p $OUT
for rep in 1 2; do for f in 1 0; do
  FMX_COPY_FENCE=$f timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_f${f}_$rep.json > $OUT/train_r50_f${f}_$rep.log 2>&1; echo "r50 f$f rep$rep rc=$?" >> $OUT/log.txt
done; done
for f in 1 0; do
  FMX_COPY_FENCE=$f timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_f$f.json > $OUT/train_bert_f$f.log 2>&1; echo "bert f$f rc=$?" >> $OUT/log.txt
done
