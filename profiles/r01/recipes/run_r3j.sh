#!/bin/bash
# AUTO threshold re-check with the copy fence: CE-only and ZC-only sweeps to 64 MiB.
OUT=gpurun_out/r3j; mkdir -p $OUT
FMX_ZC_MAX=0 timeout 400 python bench.py --sweep --sweep-max 67108864 --out $OUT/sweep_ce.jsonl > $OUT/sweep_ce.log 2>&1; echo "ce rc=$?" >> $OUT/log.txt
FMX_ZC_MAX=1073741824 timeout 400 python bench.py --sweep --sweep-max 67108864 --out $OUT/sweep_zc.jsonl > $OUT/sweep_zc.log 2>&1; echo "zc rc=$?" >> $OUT/log.txt
