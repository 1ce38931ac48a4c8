#!/bin/bash
OUT=gpurun_out/r3i; mkdir -p $OUT
start=$(date +%s); timeout 900 python bench.py > $OUT/bench.out 2> $OUT/bench.err; echo "bench rc=$? secs=$(( $(date +%s) - start ))" >> $OUT/log.txt
start=$(date +%s); timeout 300 python bench.py --impl reference > $OUT/ref.out 2> $OUT/ref.err; echo "ref rc=$? secs=$(( $(date +%s) - start ))" >> $OUT/log.txt
