#!/bin/bash
# Enqueue thread for the DDP hook: parity, then ResNet-50 / BERT A/B on one lease.
OUT=gpurun_out/r3y; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q -k threaded > $OUT/pytest_ddp.log 2>&1; echo "ddp rc=$?" >> $OUT/log.txt
for rep in 1 2; do
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_base$rep.json > $OUT/train_base$rep.log 2>&1; echo "base rc=$?" >> $OUT/log.txt
FMX_HOOK_THREAD=1 timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50_thr$rep.json > $OUT/train_thr$rep.log 2>&1; echo "thr rc=$?" >> $OUT/log.txt
done
FMX_HOOK_THREAD=1 timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert_thr.json > $OUT/train_bert_thr.log 2>&1; echo "bert thr rc=$?" >> $OUT/log.txt
