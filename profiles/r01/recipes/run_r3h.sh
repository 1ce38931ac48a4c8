#!/bin/bash
OUT=gpurun_out/r3h; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_stress_gpu.py -x -q > $OUT/pytest_stress.log 2>&1; echo "stress rc=$?" >> $OUT/log.txt
