#!/bin/bash
OUT=gpurun_out/r1g; mkdir -p $OUT
timeout 200 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_ddp_gpu.py -x -q --timeout 200 > $OUT/gputest.log 2>&1; echo "gputest rc=$?" >> $OUT/log.txt
for cfg in "default 4194304" "FMX_RAMP=0 4194304" "FMX_GRAIN=fine 4194304" "default 8388608" "FMX_LANES=1 4194304" "default 2097152"; do
  set -- $cfg
  tag=$(echo $1 | tr '=' '-')-$2
  env $([ "$1" != default ] && echo $1) timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --slice-bytes $2 --timeline $OUT/tl_$tag.json --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt
done
