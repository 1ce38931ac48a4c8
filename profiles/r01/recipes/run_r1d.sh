#!/bin/bash
OUT=gpurun_out/r1d; mkdir -p $OUT
timeout 400 python -m pytest tests/test_ddp_gpu.py -x -q --timeout 200 > $OUT/gputest.log 2>&1; echo "ddp test rc=$?" >> $OUT/log.txt
timeout 420 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
for sb in 2097152 8388608; do
  timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --slice-bytes $sb --out $OUT/bench_$sb.json > $OUT/bench_$sb.log 2>&1; echo "bench $sb rc=$?" >> $OUT/log.txt
done
FMX_RESULT_VIA_CE=1 timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --out $OUT/bench_viace.json > $OUT/bench_viace.log 2>&1; echo "bench viace rc=$?" >> $OUT/log.txt
timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --mode mps --out $OUT/bench_mps.json > $OUT/bench_mps.log 2>&1; echo "bench mps rc=$?" >> $OUT/log.txt
