#!/bin/bash
OUT=gpurun_out/r1h; mkdir -p $OUT
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --mode mps --train-mode mps --out $OUT/bench_mps.json > $OUT/bench_mps.log 2>&1; echo "bench mps rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/ref.log 2>&1; echo "ref rc=$?" >> $OUT/log.txt
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train > $OUT/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> $OUT/log.txt
timeout 400 ncu --target-processes all --set full --clock-control none --import-source on -k regex:fmx_reduce -s 10 -c 1 -o $OUT/reduce_prof python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-train > $OUT/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> $OUT/log.txt
