#!/bin/bash
# GPU-clock pipeline timelines (bench --stamps): default, 8 MiB x 4 slots.
OUT=gpurun_out/r1r; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train "$@" --stamps $OUT/stamps_$tag.json --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run default
ENVS=FMX_SLOTS=4 run s4-8M --slice-bytes 8388608
