#!/bin/bash
OUT=gpurun_out/r2q; mkdir -p $OUT
FMX_STAMP_STEPS=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_def.json --stamps $OUT/stamps_def.json > $OUT/bench_def.log 2>&1; echo "def rc=$?" >> $OUT/log.txt
FMX_LANE1_USER=1 FMX_STAMP_STEPS=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_l1u.json --stamps $OUT/stamps_l1u.json > $OUT/bench_l1u.log 2>&1; echo "l1u rc=$?" >> $OUT/log.txt
FMX_LANES=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_lanes1.json > $OUT/bench_lanes1.log 2>&1; echo "lanes1 rc=$?" >> $OUT/log.txt
