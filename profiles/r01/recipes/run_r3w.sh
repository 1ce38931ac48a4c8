#!/bin/bash
OUT=gpurun_out/r3w; mkdir -p $OUT
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_ce$rep.json > $OUT/bench_ce$rep.log 2>&1; echo "ce rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --transport zc --out $OUT/bench_zc$rep.json > $OUT/bench_zc$rep.log 2>&1; echo "zc rc=$?" >> $OUT/log.txt
done
