#!/bin/bash
# Fused stage + STAGED signal in the zero-copy copy kernel.
OUT=gpurun_out/r3m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_stress_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --sweep-max 4194304 --out $OUT/sweep_fused.jsonl > $OUT/sweep_fused.log 2>&1; echo "sweep fused rc=$?" >> $OUT/log.txt
FMX_FUSE_SIGNAL=0 timeout 300 python bench.py --sweep --sweep-max 4194304 --out $OUT/sweep_plain.jsonl > $OUT/sweep_plain.log 2>&1; echo "sweep plain rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --sweep-max 4194304 --ranks-per-gpu 2 --out $OUT/sweep_fused_n2.jsonl > $OUT/sweep_fused_n2.log 2>&1; echo "sweep fused n2 rc=$?" >> $OUT/log.txt
