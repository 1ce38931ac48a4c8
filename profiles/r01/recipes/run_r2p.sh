#!/bin/bash
OUT=gpurun_out/r2p; mkdir -p $OUT
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_p0.json --stamps $OUT/stamps_p0.json > $OUT/bench_p0.log 2>&1; echo "p0 rc=$?" >> $OUT/log.txt
FMX_LANE_PRIORITY=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_p1.json > $OUT/bench_p1.log 2>&1; echo "p1 rc=$?" >> $OUT/log.txt
FMX_LANES=2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --out $OUT/bench_l2.json > $OUT/bench_l2.log 2>&1; echo "l2 rc=$?" >> $OUT/log.txt
