#!/bin/bash
OUT=gpurun_out/r4c; mkdir -p $OUT
start=$(date +%s); timeout 1700 python tools/soak.py 28 4 mps 105 40 > $OUT/soak_28.log 2>&1; echo "28 rc=$? secs=$(( $(date +%s) - start ))" >> $OUT/log.txt
