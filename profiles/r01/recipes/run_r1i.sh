#!/bin/bash
OUT=gpurun_out/r1i; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run green --no-e2e --no-train --mode green --timeline $OUT/tl_green.json
ENVS= run mps --no-e2e --no-train --mode mps --timeline $OUT/tl_mps.json
ENVS=FMX_GATHER_GRAIN=fine run mps-gfine --no-e2e --no-train --mode mps
ENVS=FMX_RAMP=0 run mps-noramp --no-e2e --no-train --mode mps
ENVS= run mpsgreen --mode mps+green --train-mode mps+green
ENVS= run mps-train --no-e2e --mode mps --train-mode mps
