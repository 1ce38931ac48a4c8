#!/bin/bash
# Join-stream mode (cross-collective overlap): parity, DDP legs, train timeline.
OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --stamps $OUT/stamps_r50.json --out $OUT/train_r50_st.json > $OUT/train_r50_st.log 2>&1; echo "train r50 st rc=$?" >> $OUT/log.txt
for b in 8 25; do
timeout 400 python bench.py --train-only --train-model resnet50 --bucket-mb $b --out $OUT/train_r50_b$b.json > $OUT/train_r50_b$b.log 2>&1; echo "train r50 b$b rc=$?" >> $OUT/log.txt
done
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "train bert rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --out $OUT/train_mbv2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
