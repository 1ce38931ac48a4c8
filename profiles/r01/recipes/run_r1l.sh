#!/bin/bash
# Message-size sweep 1 KiB - 1 GiB (BASELINE configs[4]) at 7 and 2 ranks on one B200.
OUT=gpurun_out/r1l; mkdir -p $OUT
timeout 400 python bench.py --sweep --mode mps --out $OUT/sweep_mps_n7.jsonl > $OUT/sweep_mps_n7.log 2>&1; echo "mps n7 rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --mode mps --ranks-per-gpu 2 --out $OUT/sweep_mps_n2.jsonl > $OUT/sweep_mps_n2.log 2>&1; echo "mps n2 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --mode green --out $OUT/sweep_green_n7.jsonl > $OUT/sweep_green_n7.log 2>&1; echo "green n7 rc=$?" >> $OUT/log.txt
