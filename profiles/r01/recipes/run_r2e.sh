#!/bin/bash
# ZC transport (SM zero-copy loads/stores) under MPS vs CE.
OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --transport zc --out $OUT/bench_zc.json --stamps $OUT/stamps_zc.json > $OUT/bench_zc.log 2>&1; echo "zc rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --transport ce --out $OUT/bench_ce.json > $OUT/bench_ce.log 2>&1; echo "ce rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --transport zc --sweep-max 16777216 --out $OUT/sweep_zc.jsonl > $OUT/sweep_zc.log 2>&1; echo "sweep zc rc=$?" >> $OUT/log.txt
