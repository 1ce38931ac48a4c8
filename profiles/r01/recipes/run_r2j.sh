#!/bin/bash
OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 400 python bench.py --train-only --train-model resnet50 --stamps $OUT/stamps_r50.json --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "train r50 rc=$?" >> $OUT/log.txt
