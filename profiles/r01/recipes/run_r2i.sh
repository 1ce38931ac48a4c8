#!/bin/bash
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 300 python bench.py --count 256 --steps 50 --warmup 5 --no-e2e --no-train --no-cpu-baseline --stamps $OUT/stamps_small.json --out $OUT/bench_small.json > $OUT/bench_small.log 2>&1; echo "small rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --count 256 --steps 50 --warmup 5 --no-e2e --no-train --no-cpu-baseline --ranks-per-gpu 2 --stamps $OUT/stamps_small2.json --out $OUT/bench_small2.json > $OUT/bench_small2.log 2>&1; echo "small2 rc=$?" >> $OUT/log.txt
