#!/bin/bash
# Join-stream mode on one stream: bucketed probe, DDP parity, DP legs.
OUT=gpurun_out/r2x; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py tests/test_allreduce_gpu.py -k "ddp or join_stream" -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --out $OUT/bench_b13.json > $OUT/bench_b13.log 2>&1; echo "b13 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --stamps $OUT/stamps_r50.json --out $OUT/train_r50_st.json > $OUT/train_r50_st.log 2>&1; echo "r50 st rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "r50 rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "bert rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --out $OUT/train_mbv2.json > $OUT/train_mbv2.log 2>&1; echo "mbv2 rc=$?" >> $OUT/log.txt
