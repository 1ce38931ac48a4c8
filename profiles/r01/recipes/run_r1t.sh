#!/bin/bash
# New ramp geometry: slice 4/8/16 MiB, slots 2/3, device + e2e.
OUT=gpurun_out/r1t; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run 4M
ENVS= run 8M --slice-bytes 8388608 --stamps $OUT/stamps_8M.json
ENVS= run 16M --slice-bytes 16777216
ENVS=FMX_SLOTS=3 run s3-8M --slice-bytes 8388608
ENVS=FMX_SLOTS=4 run s4-8M --slice-bytes 8388608
ENVS= run 4M-b
