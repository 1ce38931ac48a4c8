#!/bin/bash
OUT=gpurun_out/r3k; mkdir -p $OUT
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --ranks-per-gpu 2 --stamps $OUT/stamps_n2.json --out $OUT/bench_n2.json > $OUT/bench_n2.log 2>&1; echo "n2 rc=$?" >> $OUT/log.txt
FMX_SLOTS=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --ranks-per-gpu 2 --out $OUT/bench_n2_k3.json > $OUT/bench_n2_k3.log 2>&1; echo "n2 k3 rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --ranks-per-gpu 2 --slice-bytes 16777216 --out $OUT/bench_n2_16M.json > $OUT/bench_n2_16M.log 2>&1; echo "n2 16M rc=$?" >> $OUT/log.txt
FMX_SLOTS=4 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --ranks-per-gpu 2 --slice-bytes 16777216 --out $OUT/bench_n2_16M_k4.json > $OUT/bench_n2_16M_k4.log 2>&1; echo "n2 16M k4 rc=$?" >> $OUT/log.txt
