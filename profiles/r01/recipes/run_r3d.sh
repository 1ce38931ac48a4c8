#!/bin/bash
# Schedule knobs re-measured with the copy fence (earlier runs were confounded by the CE->memop slow path).
OUT=gpurun_out/r3d; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run default
ENVS= run 8M --slice-bytes 8388608
ENVS= run 2M --slice-bytes 2097152
ENVS=FMX_SLOTS=3 run k3
ENVS=FMX_LANES=1 run lanes1
ENVS=FMX_LANES=2 run lanes2
ENVS=FMX_RAMP=0 run noramp
ENVS= run default2
