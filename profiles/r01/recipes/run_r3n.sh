#!/bin/bash
OUT=gpurun_out/r3n; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_stress_gpu.py -x -q -k wide > $OUT/pytest_wide.log 2>&1; echo "wide rc=$?" >> $OUT/log.txt
