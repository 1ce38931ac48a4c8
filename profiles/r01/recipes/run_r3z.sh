#!/bin/bash
# Rarely used bench paths: --inproc (ranks as threads), --timeline, --dtype bf16, --transport zc e2e.
OUT=gpurun_out/r3z; mkdir -p $OUT
timeout 300 python bench.py --inproc --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --out $OUT/bench_inproc.json > $OUT/bench_inproc.log 2>&1; echo "inproc rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e --timeline $OUT/tl.json --out $OUT/bench_tl.json > $OUT/bench_tl.log 2>&1; echo "timeline rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --dtype bf16 --out $OUT/bench_bf16.json > $OUT/bench_bf16.log 2>&1; echo "bf16 rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-train --impl reference --dtype bf16 > $OUT/ref_bf16.log 2>&1; echo "ref bf16 rc=$?" >> $OUT/log.txt
