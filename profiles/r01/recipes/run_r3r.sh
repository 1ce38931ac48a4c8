#!/bin/bash
OUT=gpurun_out/r3r; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
for rep in 1 2 3; do
ENVS= run eq$rep
ENVS=FMX_RAMP=3 run q$rep
done
