#!/bin/bash
OUT=gpurun_out/r2k; mkdir -p $OUT
timeout 400 python bench.py --train-only --train-model resnet50 --stamps $OUT/stamps_r50.json --out $OUT/train_r50_st.json > $OUT/train_r50_st.log 2>&1; echo "train r50 stamps rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "train r50 rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "train bert rc=$?" >> $OUT/log.txt
