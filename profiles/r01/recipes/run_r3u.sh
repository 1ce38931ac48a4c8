#!/bin/bash
OUT=gpurun_out/r3u; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q > $OUT/pytest_ddp.log 2>&1; echo "ddp rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --train-no-sync --out $OUT/train_resnet50.json > $OUT/train_r50.log 2>&1; echo "r50 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --compress bf16 --out $OUT/train_resnet50_bf16.json > $OUT/train_r50b.log 2>&1; echo "r50 bf16 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "mbv2 rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --train-no-sync --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "bert rc=$?" >> $OUT/log.txt
