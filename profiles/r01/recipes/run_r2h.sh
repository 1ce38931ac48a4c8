#!/bin/bash
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 300 python -m pytest tests/test_failure_handling.py -x -q > $OUT/pytest_fail.log 2>&1; echo "pytest fail rc=$?" >> $OUT/log.txt
