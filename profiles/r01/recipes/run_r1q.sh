#!/bin/bash
# Host path with early fetch-slot release; result-slot via CE; slice sizes with e2e.
OUT=gpurun_out/r1q; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py -x -q -k "host or seven" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run default
ENVS= run default2
ENVS=FMX_RESULT_VIA_CE=1 run viace --no-e2e
ENVS= run 8M --slice-bytes 8388608
ENVS= run 16M --slice-bytes 16777216
ENVS=FMX_SLOTS=4 run s4-8M --slice-bytes 8388608 --no-e2e
ENVS=FMX_SLOTS=3 run s3-16M --slice-bytes 16777216 --no-e2e
