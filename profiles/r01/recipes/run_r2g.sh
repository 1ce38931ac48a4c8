#!/bin/bash
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q > $OUT/pytest_ddp.log 2>&1; echo "pytest ddp rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --ranks-per-gpu 2 --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1; echo "sweep n2 rc=$?" >> $OUT/log.txt
