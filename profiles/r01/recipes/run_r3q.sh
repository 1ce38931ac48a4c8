#!/bin/bash
OUT=gpurun_out/r3q; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q > $OUT/pytest_ddp.log 2>&1; echo "ddp rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --compress bf16 --out $OUT/train_r50_bf16.json > $OUT/train_r50_bf16.log 2>&1; echo "r50 bf16 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "r50 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --compress bf16 --out $OUT/train_mbv2_bf16.json > $OUT/train_mbv2_bf16.log 2>&1; echo "mbv2 bf16 rc=$?" >> $OUT/log.txt
