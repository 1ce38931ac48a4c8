#!/bin/bash
# Parity of the 2-lane pipeline + config sweep.
OUT=gpurun_out/sweep2; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py -x -q --timeout 300 > $OUT/gputest.log 2>&1
echo "gputest rc=$?" >> $OUT/log.txt
run() {  # tag, env..., args...
  tag=$1; shift
  echo "== $tag" >> $OUT/log.txt
  env "$@" timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --out $OUT/tmp.json ${BENCH_ARGS} >> $OUT/log.txt 2>&1
  echo "rc=$?" >> $OUT/log.txt
  [ -f $OUT/tmp.json ] && python -c "
import json; d=json.load(open('$OUT/tmp.json')); d['sweep']='$tag'; print(json.dumps(d))" >> $OUT/sweep.jsonl; rm -f $OUT/tmp.json
}
BENCH_ARGS="--slice-bytes 4194304" run green-ce-4M FMX_X=0
BENCH_ARGS="--slice-bytes 4194304" run green-ce-4M-viace FMX_RESULT_VIA_CE=1
BENCH_ARGS="--slice-bytes 2097152" run green-ce-2M FMX_X=0
BENCH_ARGS="--slice-bytes 8388608" run green-ce-8M FMX_X=0
BENCH_ARGS="--slice-bytes 4194304" run green-ce-4M-no2d FMX_COPY2D=0
BENCH_ARGS="--slice-bytes 4194304 --transport zc" run green-zc-4M FMX_X=0
BENCH_ARGS="--slice-bytes 4194304 --mode mps" run mps-ce-4M FMX_X=0
BENCH_ARGS="--slice-bytes 4194304 --mode mps --transport zc" run mps-zc-4M FMX_X=0
BENCH_ARGS="--slice-bytes 2097152 --mode mps" run mps-ce-2M FMX_X=0
