#!/bin/bash
OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --stamps $OUT/stamps_b13.json --out $OUT/bench_b13.json > $OUT/bench_b13.log 2>&1; echo "b13 rc=$?" >> $OUT/log.txt
FMX_LANES=1 timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --bucket-serial --stamps $OUT/stamps_b13s1.json --out $OUT/bench_b13s1.json > $OUT/bench_b13s1.log 2>&1; echo "b13 serial lanes1 rc=$?" >> $OUT/log.txt
