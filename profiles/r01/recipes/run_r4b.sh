#!/bin/bash
# Extended soak: long random programs at 7 (MPS, green), 14 and 28 ranks.
OUT=gpurun_out/r4b; mkdir -p $OUT
timeout 1500 python tools/soak.py 7 1 mps 101 300 > $OUT/soak_7_mps.log 2>&1; echo "7 mps rc=$?" >> $OUT/log.txt
timeout 1200 python tools/soak.py 5 1 green 102 120 > $OUT/soak_5_green.log 2>&1; echo "5 green rc=$?" >> $OUT/log.txt
timeout 1500 python tools/soak.py 14 2 mps 103 150 > $OUT/soak_14.log 2>&1; echo "14 rc=$?" >> $OUT/log.txt
timeout 1800 python tools/soak.py 28 4 mps 104 100 > $OUT/soak_28.log 2>&1; echo "28 rc=$?" >> $OUT/log.txt
