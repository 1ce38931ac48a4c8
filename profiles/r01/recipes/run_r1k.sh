#!/bin/bash
# Three-lane schedule (gather on its own lane): parity, then lanes x mode x slice sweep.
OUT=gpurun_out/r1k; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py tests/test_ddp_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
run() { tag=$1; shift; env $ENVS timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
for mode in mps green; do
  ENVS=FMX_LANES=3 run $mode-l3 --no-e2e --mode $mode --timeline $OUT/tl_$mode-l3.json
  ENVS=FMX_LANES=2 run $mode-l2 --no-e2e --mode $mode
done
ENVS=FMX_LANES=3 run mps-l3-8M --no-e2e --mode mps --slice-bytes 8388608
ENVS=FMX_LANES=3 run mps-l3-2M --no-e2e --mode mps --slice-bytes 2097152
ENVS="FMX_LANES=3 FMX_RAMP=0" run mps-l3-noramp --no-e2e --mode mps
ENVS=FMX_LANES=3 run mps-l3-e2e --mode mps
