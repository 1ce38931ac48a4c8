#!/bin/bash
# Join-stream calls complete on the gather lane (fetch of bucket k+1 overlaps gather of k).
OUT=gpurun_out/r2u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_ddp_gpu.py tests/test_failure_handling.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --stamps $OUT/stamps_r50.json --out $OUT/train_r50_st.json > $OUT/train_r50_st.log 2>&1; echo "r50 st rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --out $OUT/train_r50.json > $OUT/train_r50.log 2>&1; echo "r50 rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --train-only --train-model bert --out $OUT/train_bert.json > $OUT/train_bert.log 2>&1; echo "bert rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
