#!/bin/bash
# GPU-clock timelines: default (4 MiB, ramp, 2 slots), 4 MiB x 3 slots, 2 MiB.
OUT=gpurun_out/r1s; mkdir -p $OUT
nvidia-smi -q | grep -iE "Link|Gen|Width|Product Name|Bus Id" | head -20 > $OUT/smi.txt
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train "$@" --stamps $OUT/stamps_$tag.json --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run default
ENVS=FMX_SLOTS=3 run s3
ENVS= run 2M --slice-bytes 2097152
