#!/bin/bash
# Host path with the push lane: parity + e2e timing + stamps.
OUT=gpurun_out/r1u; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py -x -q -k "host" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
run() { tag=$1; shift; env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
ENVS= run l3 --stamps $OUT/stamps_l3.json
ENVS=FMX_LANES=2 run l2
ENVS= run l3-8M --slice-bytes 8388608
ENVS= run l3-2M --slice-bytes 2097152
