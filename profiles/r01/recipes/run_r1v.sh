#!/bin/bash
# Stock-NCCL duplicate-GPU check; MobileNetV2 (4 instances) and BERT-base bf16 (7 instances) DP legs.
OUT=gpurun_out/r1v; mkdir -p $OUT
timeout 300 python -m pytest tests/test_nccl_duplicate_gpu.py -x -q > $OUT/pytest_nccl.log 2>&1; echo "nccl dup rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --out $OUT/train_mbv2.json > $OUT/train_mbv2.log 2>&1; echo "mbv2 rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "bert rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "r50 rc=$?" >> $OUT/log.txt
