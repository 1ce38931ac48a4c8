#!/bin/bash
OUT=gpurun_out/r1e; mkdir -p $OUT
timeout 700 python -m pytest tests/test_allreduce_gpu.py -x -q --timeout 200 > $OUT/gputest.log 2>&1; echo "gputest rc=$?" >> $OUT/log.txt
for sb in 4194304 8388608 2097152 1048576; do
  timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --slice-bytes $sb --out $OUT/bench_$sb.json > $OUT/bench_$sb.log 2>&1; echo "bench $sb rc=$?" >> $OUT/log.txt
done
timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --mode mps --out $OUT/bench_mps.json > $OUT/bench_mps.log 2>&1; echo "bench mps rc=$?" >> $OUT/log.txt
timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --transport zc --out $OUT/bench_zc.json > $OUT/bench_zc.log 2>&1; echo "bench zc rc=$?" >> $OUT/log.txt
