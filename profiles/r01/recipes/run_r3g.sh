#!/bin/bash
# Equal-round geometry (new default): slice size, slots, lanes.
OUT=gpurun_out/r3g; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
for rep in 1 2; do
ENVS= run def$rep
ENVS= run 3M$rep --slice-bytes 3145728
ENVS= run 6M$rep --slice-bytes 6291456
ENVS= run 8M$rep --slice-bytes 8388608
ENVS=FMX_SLOTS=3 run k3$rep
ENVS=FMX_LANES=1 run l1$rep
done
