#!/bin/bash
OUT=gpurun_out/r3t; mkdir -p $OUT
for rep in 1 2; do
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_base$rep.json > $OUT/train_base$rep.log 2>&1; echo "base rc=$?" >> $OUT/log.txt
FMX_BUCKET_VIEW=1 timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_view$rep.json > $OUT/train_view$rep.log 2>&1; echo "view rc=$?" >> $OUT/log.txt
done
FMX_BUCKET_VIEW=1 timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_view.json > $OUT/train_bert_view.log 2>&1; echo "bert view rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_base.json > $OUT/train_bert_base.log 2>&1; echo "bert base rc=$?" >> $OUT/log.txt
