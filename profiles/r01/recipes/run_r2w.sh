#!/bin/bash
# 102 MB gradient as 13 x 8 MB buckets: join-stream overlap vs serial completion.
OUT=gpurun_out/r2w; mkdir -p $OUT
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --out $OUT/bench_b13.json --stamps $OUT/stamps_b13.json > $OUT/bench_b13.log 2>&1; echo "b13 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 13 --bucket-serial --out $OUT/bench_b13s.json > $OUT/bench_b13s.log 2>&1; echo "b13 serial rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --buckets 4 --out $OUT/bench_b4.json > $OUT/bench_b4.log 2>&1; echo "b4 rc=$?" >> $OUT/log.txt
