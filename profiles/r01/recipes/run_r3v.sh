#!/bin/bash
OUT=gpurun_out/r3v; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ddp_gpu.py -x -q -k zero > $OUT/pytest_zero.log 2>&1; echo "zero rc=$?" >> $OUT/log.txt
