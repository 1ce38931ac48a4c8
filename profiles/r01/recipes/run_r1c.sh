#!/bin/bash
OUT=gpurun_out/r1c; mkdir -p $OUT
timeout 60 python tools/debug_ar.py --layout procs --transport ce --mode green --n 2 --count 16777216 --rounds 20 > $OUT/debug.log 2>&1; echo "debug rc=$?" >> $OUT/log.txt
timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_ddp_gpu.py -x -q --timeout 240 > $OUT/gputest.log 2>&1; echo "gputest rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
for sb in 2097152 8388608; do
  timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --slice-bytes $sb --out $OUT/bench_$sb.json > $OUT/bench_$sb.log 2>&1; echo "bench $sb rc=$?" >> $OUT/log.txt
done
FMX_RESULT_VIA_CE=1 timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --out $OUT/bench_viace.json > $OUT/bench_viace.log 2>&1; echo "bench viace rc=$?" >> $OUT/log.txt
