#!/bin/bash
# Does compute on the instances' SMs slow the allreduce? (in-training comm is 50 ms vs 30)
OUT=gpurun_out/r2v; mkdir -p $OUT
for l in 0 400; do
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --load $l --out $OUT/bench_load$l.json > $OUT/bench_load$l.log 2>&1; echo "load $l rc=$?" >> $OUT/log.txt
done
