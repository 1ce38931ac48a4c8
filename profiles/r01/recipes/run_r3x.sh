#!/bin/bash
# Per-contributor flags in the first round only (shorter pipeline fill), same lease x3.
OUT=gpurun_out/r3x; mkdir -p $OUT
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
for rep in 1 2 3; do
ENVS= run def$rep
ENVS=FMX_GRAIN=first run first$rep
done
FMX_GRAIN=first timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --stamps $OUT/stamps_first.json --out $OUT/bench_first_st.json > $OUT/bench_first_st.log 2>&1; echo "stamps rc=$?" >> $OUT/log.txt
