#!/bin/bash
# After the source split + spill fix: GPU suite, default bench, ncu full of the reduce kernel.
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full python tools/reduce_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/log.txt
